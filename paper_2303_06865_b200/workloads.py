"""Workload shapes (BASELINE.json configs) and the byte / token accounting of
the hot path.  Pure arithmetic on sizes -- no kernels, no method arithmetic.

Paper anchors: memory formulas weights l(8 h1^2 + 4 h1 h2) and KV peak
4 b l h1 (s + n) in fp16 bytes; per-layer decode KV I/O
4 bls (s + n/2) h1; generation throughput b n / t.
Compressed storage: 4-bit codes + fp16 (scale, min) per 64 elements =
4.5 bits per element.
"""
from __future__ import annotations

from dataclasses import dataclass

BITS, GROUP = 4, 64
COMPRESSED_BYTES_PER_ELEM = BITS / 8 + 4 / GROUP        # 0.5625 B = 4.5 bits


@dataclass(frozen=True)
class Workload:
    name: str
    batch: int          # b (effective batch)
    heads: int
    head_dim: int
    prompt_len: int     # s
    gen_len: int        # n
    layers: int         # l
    h2: int = 0         # MLP hidden (weight accounting only)

    @property
    def h1(self) -> int:
        return self.heads * self.head_dim

    @property
    def t_cap(self) -> int:
        return self.prompt_len + self.gen_len


# BASELINE.json configs; layer counts are the OPT family values (l = 96 for 175B)
CONFIGS = {
    "tiny": Workload("tiny", 4, 12, 64, 512, 1, 1),
    "opt-6.7b": Workload("opt-6.7b", 64, 32, 128, 512, 32, 32, 16384),
    "opt-30b": Workload("opt-30b", 144, 56, 128, 1024, 32, 48, 28672),
    "opt-175b": Workload("opt-175b", 144, 96, 128, 512, 32, 96, 49152),
}


def weight_bytes_fp16(w: Workload) -> int:
    """l (8 h1^2 + 4 h1 h2) bytes."""
    return w.layers * (8 * w.h1 ** 2 + 4 * w.h1 * w.h2)


def kv_peak_bytes_fp16(w: Workload, batch: int | None = None) -> int:
    """4 b l h1 (s + n) bytes."""
    b = w.batch if batch is None else batch
    return 4 * b * w.layers * w.h1 * (w.prompt_len + w.gen_len)


def kv_cache_bytes_compressed(w: Workload, batch: int | None = None) -> int:
    """Bytes of the 4-bit cache as allocated (codes + fp16 (scale, min)), all layers."""
    b = w.batch if batch is None else batch
    elems = 2 * b * w.layers * w.h1 * w.t_cap
    return elems // 2 + elems // GROUP * 4


def attention_bytes(batch: int, h1: int, cur_len: int) -> int:
    """Algorithmic HBM bytes of one decode-attention launch (one layer):
    K and V codes + meta for cur_len tokens (1.125 B per hidden element per
    token) plus q in and out (2 B each): (1.125 cur_len + 4) h1 per sequence."""
    per_seq = 2 * cur_len * (h1 // 2 + h1 // GROUP * 4) + 2 * h1 * 2
    return batch * per_seq


def append_bytes(batch: int, h1: int, n_new: int = 1) -> int:
    """One append launch: read K, V fp16, write codes + meta (5.125 B per element pair)."""
    elems = 2 * batch * h1 * n_new
    return elems * 2 + elems // 2 + elems // GROUP * 4


def attention_flops(batch: int, h1: int, cur_len: int) -> int:
    """4 cur_len h1 per sequence (QK^T and PV)."""
    return 4 * batch * h1 * cur_len

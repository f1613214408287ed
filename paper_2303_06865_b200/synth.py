"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic (no quantization, no
attention): it only draws fp16 tensors.  The generator is counter based and
uses integer torch ops whose results are exact in int64 (32-bit values times
31-bit constants), so the same call gives bit-identical tensors on the CPU and
on the GPU.  That lets a test generate a full-size cache on the device and
regenerate any sampled (b, h) slice on the host for the oracle, without ever
copying an oracle input back from the CUDA path.

Recipe: the paper uses synthetic equal-length
prompts and dummy weights.  Default values are Irwin-Hall(4) sums
of 22-bit uniforms, x = (u1+u2+u3+u4 - 2^23) * 2^-21 in [-4, 4), exact in fp32,
then rounded to fp16 (sigma ~ 1.15).  Value-set variants shape the data:
``outliers`` (channels 7 and 77 of every head x16), ``peaky`` q (x16 / x64),
``ties`` (x = k/2), ``extreme`` (constant groups, +-65504, subnormals, every
finite fp16 bit pattern).
"""
from __future__ import annotations

import torch

M32 = 0xFFFFFFFF
_C1 = 0x7FEB352D  # odd multipliers < 2^31: products with a 32-bit value stay < 2^63
_C2 = 0x6B43A9B5
_C3 = 0x5BD1E995

# tensor kinds for tensor_id()
K_PROMPT, V_PROMPT, Q, K_NEW, V_NEW, WEIGHT = range(6)
BASE_SEED = 230306865


def tensor_id(layer: int, kind: int, step: int = 0) -> int:
    return ((layer * 8 + kind) * 4096 + step) & M32


def _hash32(x: torch.Tensor) -> torch.Tensor:
    """32-bit integer mixer on int64 tensors holding values in [0, 2^32)."""
    x = x ^ (x >> 16)
    x = (x * _C1) & M32
    x = x ^ (x >> 15)
    x = (x * _C2) & M32
    x = x ^ (x >> 13)
    x = (x * _C3) & M32
    x = x ^ (x >> 16)
    return x


def _key(seed: int, tid: int) -> int:
    t = torch.tensor([(seed & M32) ^ ((tid * 0x9E3779B1) & M32)], dtype=torch.int64)
    return int(_hash32(_hash32(t) ^ (tid & M32))[0])


def uniform32(seed: int, tid: int, idx: torch.Tensor) -> torch.Tensor:
    """32-bit uniform integers (int64 tensor) for counters idx (int64, < 2^32)."""
    k = _key(seed, tid)
    return _hash32(_hash32((idx & M32) ^ k) ^ ((idx >> 32) & M32) ^ (k >> 1))


def irwin_hall(seed: int, tid: int, idx: torch.Tensor) -> torch.Tensor:
    """Default value set at counters idx -> fp16 tensor (same device as idx)."""
    s = torch.zeros_like(idx)
    for k in range(4):
        s = s + (uniform32(seed, tid, idx * 4 + k) >> 10)      # 22-bit uniforms
    x = (s - (1 << 23)).to(torch.float32) * (2.0 ** -21)          # exact in fp32
    return x.to(torch.float16)                                    # RNE


def fill(seed: int, tid: int, shape, device="cpu", chunk: int = 1 << 25) -> torch.Tensor:
    """Full fp16 tensor of `shape`, element i drawn at counter i (chunked)."""
    n = 1
    for d in shape:
        n *= int(d)
    out = torch.empty(n, dtype=torch.float16, device=device)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        idx = torch.arange(s, e, dtype=torch.int64, device=device)
        out[s:e] = irwin_hall(seed, tid, idx)
    return out.view(*shape)


def fill_rows(seed: int, tid: int, shape, row0: int, row1: int, device="cpu", chunk: int = 1 << 25) -> torch.Tensor:
    """Rows [row0, row1) of the leading dimension of fill(seed, tid, shape), drawn directly
    (same counters): a rank generates its shard of a global batch without the rest."""
    rs = 1
    for d in shape[1:]:
        rs *= int(d)
    n = (row1 - row0) * rs
    out = torch.empty(n, dtype=torch.float16, device=device)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        idx = torch.arange(row0 * rs + s, row0 * rs + e, dtype=torch.int64, device=device)
        out[s:e] = irwin_hall(seed, tid, idx)
    return out.view(row1 - row0, *shape[1:])


def gather(seed: int, tid: int, shape, index_slices) -> torch.Tensor:
    """Host (CPU) regeneration of a sub-block of fill(seed, tid, shape).

    index_slices: one python slice / int / list per dim.  Returns the same
    values fill() would have produced at those positions."""
    grids = []
    for d, sl in zip(shape, index_slices):
        if isinstance(sl, slice):
            grids.append(torch.arange(d, dtype=torch.int64)[sl])
        elif isinstance(sl, int):
            grids.append(torch.tensor([sl], dtype=torch.int64))
        else:
            grids.append(torch.as_tensor(sl, dtype=torch.int64))
    strides = []
    acc = 1
    for d in reversed(shape):
        strides.append(acc)
        acc *= int(d)
    strides = strides[::-1]
    idx = torch.zeros([len(g) for g in grids], dtype=torch.int64)
    for k, g in enumerate(grids):
        view = [1] * len(grids)
        view[k] = len(g)
        idx = idx + g.view(view) * strides[k]
    return irwin_hall(seed, tid, idx)


# ---------------------------------------------------------------- value sets
def with_outliers(x: torch.Tensor, channels=(7, 77)) -> torch.Tensor:
    """Channels c mod D of every head scaled x16 (exact in fp16 for |x| < 4096)."""
    y = x.clone()
    D = x.shape[-1]
    for c in channels:
        y[..., c % D] = y[..., c % D] * 16
    return y


def peaky(q: torch.Tensor, factor: int) -> torch.Tensor:
    """q scaled by a power of two (exact in fp16): sharpens the softmax."""
    return q * factor


def ties(seed: int, tid: int, shape) -> torch.Tensor:
    """x = k/2, k uniform in [0, 30]: many exact .5 ties in (x-min)/(max-min)*15."""
    n = 1
    for d in shape:
        n *= int(d)
    u = uniform32(seed, tid, torch.arange(n, dtype=torch.int64))
    return ((u % 31).to(torch.float32) * 0.5).to(torch.float16).view(*shape)


def extreme(seed: int, tid: int, rows: int, cols: int, group: int = 64) -> torch.Tensor:
    """Per group, one of: constant, +-65504 mix, subnormals, any finite fp16 pattern."""
    n = rows * cols
    idx = torch.arange(n, dtype=torch.int64)
    u = uniform32(seed, tid, idx)
    kind = (uniform32(seed, tid ^ 0x55, idx // group) % 5)
    bits = u & 0xFFFF
    # any finite pattern: force exponent field != 31
    finite = torch.where(((bits >> 10) & 0x1F) == 0x1F, bits & 0xFBFF, bits)
    subn = bits & 0x83FF                                  # exponent 0: subnormals / zeros
    big = torch.where((u >> 16) & 1 == 1, torch.full_like(u, 0x7BFF), torch.full_like(u, 0xFBFF))
    const = (uniform32(seed, tid ^ 0xAA, idx // group) & 0x7BFF)
    mixed = torch.where((u >> 17) % 3 == 0, big, finite)
    out = torch.where(kind == 0, const,
          torch.where(kind == 1, big,
          torch.where(kind == 2, subn,
          torch.where(kind == 3, finite, mixed))))
    out = torch.where(out >= 32768, out - 65536, out)          # bit pattern as signed int16
    return out.to(torch.int16).view(torch.float16).view(rows, cols)

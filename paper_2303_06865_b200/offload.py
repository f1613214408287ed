"""Host-offloaded compressed KV cache with FlexGen's overlapped block schedule.

FlexGen keeps the KV cache of large-batch decoding off the GPU (1.2 TB for OPT-175B
at b = 512) and overlaps its I/O with compute: Alg. 1 walks layers j and GPU batches
k, and while batch k computes it loads the cache of batch k + 1 and stores the cache of batch
k - 1.  Re-based on B200: the compressed cache of every (layer, GPU batch) lives in pinned host
memory; a device ring of `slots` cache buffers is fed by a load stream (host -> device copy
engine) and drained by a store stream (device -> host); the compute stream runs the fused
append + decode attention kernel (flexq_append_decode_attention) on the resident buffer.

Only the chunk that received the new token goes back to the host (one strided 2-D copy per
K / V buffer: batch * heads rows of one chunk), since the decode step appends one token per
(b, h) and leaves every other byte of the cache unchanged.

This module is host-side plumbing (streams, events, copies); every step of the method runs in
libflexq's kernels, and nothing here computes on the CPU.
"""
from __future__ import annotations

import torch
from cuda.bindings import runtime as _rt

from . import flexq as fq


def _check_rt(err, what):
    e = err[0] if isinstance(err, tuple) else err
    if e != _rt.cudaError_t.cudaSuccess:
        raise RuntimeError(f"{what}: {e}")


class OffloadedKV:
    """Compressed KV caches of `layers` x `gpu_batches` blocks in pinned host memory, streamed
    through `slots` device buffers in Alg. 1's (layer, GPU batch) order."""

    def __init__(self, layers: int, gpu_batches: int, batch: int, heads: int, head_dim: int, prompt_len: int,
                 gen_len: int, device, slots: int = 2):
        self.layers, self.gpu_batches, self.slots = layers, gpu_batches, slots
        self.device = torch.device(device)
        self.host = [[self._pinned(batch, heads, head_dim, prompt_len, gen_len) for _ in range(gpu_batches)]
                     for _ in range(layers)]
        self.dev = [fq.KVCache(batch, heads, head_dim, prompt_len, gen_len, device=self.device)
                    for _ in range(slots)]
        self.ws = [fq.make_workspace(c) for c in self.dev]
        self.load_stream = torch.cuda.Stream(device=self.device)
        self.store_stream = torch.cuda.Stream(device=self.device)
        self.loaded = [torch.cuda.Event() for _ in range(slots)]
        self.computed = [torch.cuda.Event() for _ in range(slots)]
        self.stored = [torch.cuda.Event() for _ in range(slots)]
        self.chunk_bytes = self.dev[0].k.shape[-1]
        self.rows = batch * heads
        self.row_pitch = self.dev[0].chunks * self.chunk_bytes

    @staticmethod
    def _pinned(batch, heads, head_dim, prompt_len, gen_len) -> fq.KVCache:
        c = fq.KVCache(batch, heads, head_dim, prompt_len, gen_len, device="cpu")
        c.k = c.k.pin_memory()
        c.v = c.v.pin_memory()
        return c

    def block_bytes(self) -> int:
        """Bytes of one (layer, GPU batch) cache (K + V): what one load moves host -> device."""
        return self.dev[0].nbytes()

    def items(self):
        """Alg. 1's order: for each layer, each GPU batch."""
        return [(j, k) for j in range(self.layers) for k in range(self.gpu_batches)]

    # ------------------------------------------------------------------ copies
    def _load(self, slot: int, j: int, k: int):
        h, d = self.host[j][k], self.dev[slot]
        with torch.cuda.stream(self.load_stream):
            d.k.copy_(h.k, non_blocking=True)
            d.v.copy_(h.v, non_blocking=True)

    def _store_chunk(self, slot: int, j: int, k: int, chunk: int):
        """Copy chunk `chunk` of every (b, h) -- the one holding the new token -- back to the host."""
        h, d = self.host[j][k], self.dev[slot]
        off = chunk * self.chunk_bytes
        for hb, db in ((h.k, d.k), (h.v, d.v)):
            err = _rt.cudaMemcpy2DAsync(hb.data_ptr() + off, self.row_pitch, db.data_ptr() + off, self.row_pitch,
                                        self.chunk_bytes, self.rows, _rt.cudaMemcpyKind.cudaMemcpyDeviceToHost,
                                        self.store_stream.cuda_stream)
            _check_rt(err, "cudaMemcpy2DAsync")

    def prefill(self, k_prompt, v_prompt, stream=None):
        """Quantize each block's prompt K / V on the device and write the whole cache to the host.
        k_prompt(j, k) / v_prompt(j, k) -> fp16 [B][H][s][D] device tensors."""
        stream = stream or torch.cuda.current_stream(self.device)
        d = self.dev[0]
        for j, k in self.items():
            d.k.zero_()
            d.v.zero_()
            fq.flexq_append_kv(k_prompt(j, k), v_prompt(j, k), d, pos=0, stream=stream)
            stream.synchronize()
            self.host[j][k].k.copy_(d.k)
            self.host[j][k].v.copy_(d.v)

    # ------------------------------------------------------------------ one decode step
    def decode_step(self, cur_len: int, q, k_new, v_new, out, stream=None):
        """Append token cur_len - 1 and attend over [0, cur_len) for every (layer, GPU batch).
        q / k_new / v_new / out: callables (j, k) -> fp16 [B][H][D] device tensors.
        All work is enqueued on streams; returns after enqueueing (the caller syncs)."""
        stream = stream or torch.cuda.current_stream(self.device)
        items = self.items()
        chunk = (cur_len - 1) // fq.CHUNK
        S = self.slots
        # prologue: the first S - 1 loads
        for i in range(min(S - 1, len(items))):
            self.load_stream.wait_event(self.stored[i % S])
            self._load(i % S, *items[i])
            self.loaded[i % S].record(self.load_stream)
        for i, (j, k) in enumerate(items):
            slot = i % S
            nxt = i + S - 1
            if nxt < len(items):                  # load_cache(i, j, k + 1) (Alg. 1)
                ns = nxt % S
                self.load_stream.wait_event(self.stored[ns])     # the slot's previous block is home
                self._load(ns, *items[nxt])
                self.loaded[ns].record(self.load_stream)
            stream.wait_event(self.loaded[slot])                 # compute(i, j, k)
            fq.flexq_append_decode_attention(q(j, k), k_new(j, k), v_new(j, k), self.dev[slot], cur_len,
                                             out=out(j, k), workspace=self.ws[slot], stream=stream)
            self.computed[slot].record(stream)
            self.store_stream.wait_event(self.computed[slot])    # store_cache(i, j, k - 1)
            self._store_chunk(slot, j, k, chunk)
            self.stored[slot].record(self.store_stream)
        stream.wait_event(self.stored[(len(items) - 1) % S])

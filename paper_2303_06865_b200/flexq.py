"""Thin Python binding over the C ABI in include/flexq.h (libflexq.so).

Argument marshalling only: torch tensors are passed as data pointers plus
torch's current CUDA stream; every step of the path runs in the library's
CUDA kernels.  There is no CPU fallback: if libflexq.so is missing and cannot
be built, every call raises.
"""
from __future__ import annotations

import ctypes
import os
import re

import torch

from . import build as _build

_lib = None
HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "flexq.h")

FLEXQ_OK, FLEXQ_ERR_NULL, FLEXQ_ERR_ARG, FLEXQ_ERR_ALIGN, FLEXQ_ERR_UNSUPPORTED, FLEXQ_ERR_WORKSPACE, \
    FLEXQ_ERR_CUDA = range(7)
BITS, GROUP = 4, 64
KV_DENSE, KV_TOKEN_MAJOR = 0, 1   # flexq_kv_layout (include/flexq.h)
LAYOUTS = {"dense": KV_DENSE, "token_major": KV_TOKEN_MAJOR}


class FlexqError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {lib().flexq_status_string(status).decode()} (status {status})")


def lib():
    """Load libflexq.so (building it in-tree with nvcc if it is missing)."""
    global _lib
    if _lib is None:
        path = os.environ.get("FLEXQ_LIB", _build.LIB)   # FLEXQ_LIB: A/B tuning builds only
        if not os.path.exists(path):
            try:
                _build.build()
            except Exception as e:  # noqa: BLE001
                raise RuntimeError(f"libflexq.so is not built and the build failed: {e}") from e
        L = ctypes.CDLL(path)
        P, I, I64, SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
        L.flexq_abi_version.restype = I
        L.flexq_status_string.argtypes = [I]
        L.flexq_status_string.restype = ctypes.c_char_p
        L.flexq_quantize.argtypes = [P, I64, I64, I, I, P, P, P]
        L.flexq_dequantize.argtypes = [P, P, I64, I64, I, I, P, P]
        L.flexq_kv_cache_bytes.argtypes = [I] * 7 + [ctypes.POINTER(SZ), ctypes.POINTER(I)]
        L.flexq_append_kv.argtypes = [P, P] + [I] * 10 + [P, P, P]
        L.flexq_decode_attention_workspace_size.argtypes = [I] * 8
        L.flexq_decode_attention_workspace_size.restype = SZ
        L.flexq_decode_attention_topk_workspace_size.argtypes = [I] * 8
        L.flexq_decode_attention_topk_workspace_size.restype = SZ
        L.flexq_decode_attention.argtypes = [P, P, P] + [I] * 9 + [P, P, SZ, P]
        L.flexq_decode_attention_topk.argtypes = [P, P, P] + [I] * 10 + [P, P, P, SZ, P]
        L.flexq_append_decode_attention.argtypes = [P] * 5 + [I] * 9 + [P, P, SZ, P]
        L.flexq_dequant_gemm_workspace_size.argtypes = [I64, I64, I64, I, I]
        L.flexq_dequant_gemm_workspace_size.restype = SZ
        L.flexq_dequant_gemm.argtypes = [P, P, I64, I64, I64, I, I, P, P, SZ, P]
        L.flexq_gemm_panel_bytes.argtypes = [I64, I64, I, I]
        L.flexq_gemm_panel_bytes.restype = SZ
        L.flexq_pack_weight.argtypes = [P, P, I64, I64, I, I, P, P]
        L.flexq_kv_import.argtypes = [P] * 4 + [I] * 11 + [P, P, P]
        L.flexq_kv_export.argtypes = [P, P] + [I] * 11 + [P] * 5
        for f in ("flexq_quantize", "flexq_dequantize", "flexq_kv_cache_bytes", "flexq_append_kv",
                  "flexq_decode_attention", "flexq_decode_attention_topk", "flexq_append_decode_attention",
                  "flexq_dequant_gemm", "flexq_pack_weight", "flexq_kv_import", "flexq_kv_export"):
            getattr(L, f).restype = I
        if hasattr(L, "flexq_debug_attn_trace"):   # tuning build only
            L.flexq_debug_attn_trace.argtypes = [P, I]
            L.flexq_debug_attn_trace.restype = I
        _lib = L
    return _lib


def header_symbols() -> list[str]:
    """Names of the functions declared in include/flexq.h."""
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(flexq_[a-z0-9_]+)\s*\(", src)))


def _check(status: int, what: str):
    if status != FLEXQ_OK:
        raise FlexqError(status, what)


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream, device=None) -> int:
    """The cudaStream_t to pass: the given stream, else torch's current stream of `device`
    (the tensors' device, not necessarily the current one)."""
    if stream is None:
        return torch.cuda.current_stream(device).cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _cross_stream(stream, device, *tensors):
    """When a call runs on a torch stream other than the current one: order it after the current
    stream's pending work (e.g. the zero-fill of arrays allocated here) and mark the tensors as used
    on it, so the caching allocator does not hand their memory out again before it is done."""
    if stream is None or not isinstance(stream, torch.cuda.Stream):
        return
    cur = torch.cuda.current_stream(device)
    if stream == cur:
        return
    stream.wait_stream(cur)
    for t in tensors:
        t.record_stream(stream)


def _need(t: torch.Tensor, dtype, name: str, shape=None, device=None):
    """A contiguous CUDA tensor of `dtype` (and `shape` / on `device` when given); the C ABI
    takes raw pointers, so a mismatch must be caught here, not as an illegal address."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != dtype or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous CUDA {dtype} tensor")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")


# ---------------------------------------------------------------- quantizer
def flexq_quantize(x: torch.Tensor, codes=None, meta=None, bits: int = BITS, group_size: int = GROUP,
                   stream=None):
    """x fp16 [rows][cols] -> (codes u8 [rows][cols*bits/8] (bit stream),
    meta fp16 [rows][cols/g][2] = (scale, min))."""
    _need(x, torch.float16, "x")
    rows, cols = x.shape
    if codes is None:
        codes = torch.empty(rows, cols * bits // 8, dtype=torch.uint8, device=x.device)
    if meta is None:
        meta = torch.empty(rows, cols // group_size, 2, dtype=torch.float16, device=x.device)
    _need(codes, torch.uint8, "codes", (rows, cols * bits // 8), x.device)
    _need(meta, torch.float16, "meta", (rows, cols // group_size, 2), x.device)
    with torch.cuda.device(x.device):
        _check(lib().flexq_quantize(x.data_ptr(), rows, cols, bits, group_size, codes.data_ptr(),
                                    meta.data_ptr(), _stream(stream, x.device)), "flexq_quantize")
    return codes, meta


def flexq_dequantize(codes: torch.Tensor, meta: torch.Tensor, out=None, bits: int = BITS,
                     group_size: int = GROUP, stream=None) -> torch.Tensor:
    _need(codes, torch.uint8, "codes")
    rows, nbytes = codes.shape
    cols = nbytes * 8 // bits
    dev = codes.device
    _need(meta, torch.float16, "meta", (rows, cols // group_size, 2), dev)
    if out is None:
        out = torch.empty(rows, cols, dtype=torch.float16, device=dev)
    _need(out, torch.float16, "out", (rows, cols), dev)
    with torch.cuda.device(dev):
        _check(lib().flexq_dequantize(codes.data_ptr(), meta.data_ptr(), rows, cols, bits, group_size,
                                      out.data_ptr(), _stream(stream, dev)), "flexq_dequantize")
    return out


# ---------------------------------------------------------------- KV cache
CHUNK = 32   # tokens per cache chunk (include/flexq.h)


def token_stride(t_cap: int) -> int:
    """Token stride of the cache layout: capacity rounded up to a chunk (include/flexq.h)."""
    return (t_cap + CHUNK - 1) // CHUNK * CHUNK


class KVCache:
    """One layer's compressed KV cache in the chunked layout of include/flexq.h:
    `k` and `v` are u8 [B][H][T_stride/32][32*(CB+MB)], chunk = [codes 32 x CB][meta 32 x MB], CB = D*bits/8,
    MB = 4*D/group (18*D per chunk at bits 4, group 64)
    (K codes token-major; V codes quad-interleaved at (4, 64) in the default "dense" layout,
    token-major like K in the "token_major" layout -- Top-K's -- and for the variants).
    The *_codes() / *_meta() accessors are layout views (copies) for tests and
    inspection, over tokens [0, T_stride)."""

    def __init__(self, batch: int, heads: int, head_dim: int, prompt_len: int, gen_len: int,
                 device="cuda", bits: int = BITS, group_size: int = GROUP, layout: str = "dense"):
        if layout not in LAYOUTS:
            raise ValueError(f"layout must be one of {sorted(LAYOUTS)}")
        self.layout = layout
        self.kv_layout = LAYOUTS[layout]
        self.batch, self.heads, self.head_dim = batch, heads, head_dim
        self.prompt_len, self.gen_len = prompt_len, gen_len
        self.bits, self.group_size = bits, group_size
        self.t_cap = prompt_len + gen_len
        self.t_stride = token_stride(self.t_cap)
        self.chunks = self.t_stride // CHUNK
        self.code_bytes = head_dim * bits // 8          # CB: one token's codes (bit stream)
        self.meta_bytes = 4 * head_dim // group_size     # MB: one token's half2 (scale, min) per group
        self.k = torch.zeros(batch, heads, self.chunks, CHUNK * (self.code_bytes + self.meta_bytes),
                             dtype=torch.uint8, device=device)
        self.v = torch.zeros_like(self.k)

    def nbytes(self) -> int:
        return self.k.numel() + self.v.numel()

    def _part(self, buf: torch.Tensor, offset: int, per_token: int) -> torch.Tensor:
        B, H, NC = self.batch, self.heads, self.chunks
        x = buf[..., offset:offset + CHUNK * per_token].reshape(B, H, NC, CHUNK, per_token)
        return x.reshape(B, H, NC * CHUNK, per_token)

    def variant(self) -> bool:
        """(bits, group) other than P:846's (4, 64): token-major K and V rows, variant kernels."""
        return (self.bits, self.group_size) != (BITS, GROUP)

    def _codes(self, buf) -> torch.Tensor:        # u8 [B][H][T_stride][D*bits/8]
        return self._part(buf, 0, self.code_bytes)

    def _meta(self, buf) -> torch.Tensor:         # fp16 [B][H][T_stride][D/g][2] = (scale, min)
        m = self._part(buf, CHUNK * self.code_bytes, self.meta_bytes)
        return m.contiguous().view(torch.float16).view(self.batch, self.heads, self.t_stride, -1, 2)

    def k_codes(self):
        return self._codes(self.k)

    def v_codes(self):
        """V codes as token-major rows.  In memory each chunk's V codes are
        quad-interleaved and swizzled: word (quad, column pair i ^ ((quad & 3) << 3)) holds
        token 4 quad + k in byte k (include/flexq.h)."""
        if self.variant() or self.kv_layout == KV_TOKEN_MAJOR:
            return self._codes(self.v)
        B, H, NC, cb = self.batch, self.heads, self.chunks, self.head_dim // 2
        x = self.v[..., :CHUNK * cb].reshape(B, H, NC, CHUNK // 4, cb, 4)
        quad = torch.arange(CHUNK // 4, device=x.device).view(-1, 1)
        pair = torch.arange(cb, device=x.device).view(1, -1)
        src = pair ^ ((quad & 3) << 3)                                  # [quad][logical pair] -> stored pair
        x = torch.gather(x, 4, src.view(1, 1, 1, CHUNK // 4, cb, 1).expand(B, H, NC, CHUNK // 4, cb, 4))
        return x.permute(0, 1, 2, 3, 5, 4).reshape(B, H, NC * CHUNK, cb)

    def k_meta(self):
        return self._meta(self.k)

    def v_meta(self):
        return self._meta(self.v)


def _plain_shapes(cache: "KVCache", plain_tokens: int):
    B, H, D = cache.batch, cache.heads, cache.head_dim
    return (B, H, plain_tokens, D * cache.bits // 8), (B, H, plain_tokens, D // cache.group_size, 2)


def flexq_kv_import(cache: "KVCache", k_codes, k_meta, v_codes, v_meta, t0: int = 0, n_tok=None, stream=None):
    """Plain quantized KV (flexq_quantize's rows per head: codes u8 [B][H][T][D*bits/8], meta fp16
    [B][H][T][D/g][2]) -> cache tokens [t0, t0 + n_tok) (include/flexq.h)."""
    T = k_codes.shape[2]
    n_tok = T - t0 if n_tok is None else n_tok
    cs, ms = _plain_shapes(cache, T)
    for t, name, dt, shp in ((k_codes, "k_codes", torch.uint8, cs), (v_codes, "v_codes", torch.uint8, cs),
                             (k_meta, "k_meta", torch.float16, ms), (v_meta, "v_meta", torch.float16, ms)):
        _need(t, dt, name)
        if tuple(t.shape) != shp:
            raise ValueError(f"{name} must have shape {shp}, got {tuple(t.shape)}")
    dev = cache.k.device
    for t in (k_codes, k_meta, v_codes, v_meta):
        if t.device != dev:
            raise ValueError(f"plain arrays must be on {dev}")
    _cross_stream(stream, dev, k_codes, k_meta, v_codes, v_meta, cache.k, cache.v)
    with torch.cuda.device(dev):
        _check(lib().flexq_kv_import(_ptr(k_codes), _ptr(k_meta), _ptr(v_codes), _ptr(v_meta), cache.batch, cache.heads,
                                     cache.head_dim, cache.prompt_len, cache.gen_len, T, t0, n_tok, cache.bits,
                                     cache.group_size, cache.kv_layout, _ptr(cache.k), _ptr(cache.v),
                                     _stream(stream, dev)),
               "flexq_kv_import")


def flexq_kv_export(cache: "KVCache", t0: int = 0, n_tok=None, plain_tokens=None, stream=None):
    """Cache tokens [t0, t0 + n_tok) -> plain (k_codes, k_meta, v_codes, v_meta) arrays with
    plain_tokens (default t0 + n_tok) token rows; rows outside the range are zero."""
    n_tok = cache.t_cap - t0 if n_tok is None else n_tok
    T = t0 + n_tok if plain_tokens is None else plain_tokens
    cs, ms = _plain_shapes(cache, T)
    dev = cache.k.device
    kc, vc = torch.zeros(cs, dtype=torch.uint8, device=dev), torch.zeros(cs, dtype=torch.uint8, device=dev)
    km, vm = torch.zeros(ms, dtype=torch.float16, device=dev), torch.zeros(ms, dtype=torch.float16, device=dev)
    _cross_stream(stream, dev, kc, km, vc, vm)
    with torch.cuda.device(dev):
        _check(lib().flexq_kv_export(_ptr(cache.k), _ptr(cache.v), cache.batch, cache.heads, cache.head_dim,
                                     cache.prompt_len, cache.gen_len, T, t0, n_tok, cache.bits, cache.group_size,
                                     cache.kv_layout, _ptr(kc), _ptr(km), _ptr(vc), _ptr(vm), _stream(stream, dev)),
               "flexq_kv_export")
    return kc, km, vc, vm


def flexq_kv_cache_bytes(batch, heads, head_dim, prompt_len, gen_len, bits=BITS, group_size=GROUP):
    """-> (bytes of one cache buffer (K or V) of one layer, token stride)."""
    c, t = ctypes.c_size_t(), ctypes.c_int()
    _check(lib().flexq_kv_cache_bytes(batch, heads, head_dim, prompt_len, gen_len, bits, group_size,
                                      ctypes.byref(c), ctypes.byref(t)), "flexq_kv_cache_bytes")
    return c.value, t.value


def flexq_append_kv(k_new: torch.Tensor, v_new: torch.Tensor, cache: KVCache, pos: int, stream=None):
    """k_new, v_new fp16 [B][H][n_new][D] -> cache tokens [pos, pos + n_new)."""
    dev = cache.k.device
    _need(k_new, torch.float16, "k_new", device=dev)
    if k_new.dim() != 4 or (k_new.shape[0], k_new.shape[1], k_new.shape[3]) != (cache.batch, cache.heads,
                                                                                cache.head_dim):
        raise ValueError(f"k_new must be [B={cache.batch}][H={cache.heads}][n_new][D={cache.head_dim}], "
                         f"got {tuple(k_new.shape)}")
    _need(v_new, torch.float16, "v_new", k_new.shape, dev)
    B, H, n_new, D = k_new.shape
    with torch.cuda.device(dev):
        _check(lib().flexq_append_kv(k_new.data_ptr(), v_new.data_ptr(), B, H, D, cache.prompt_len,
                                     cache.gen_len, pos, n_new, cache.bits, cache.group_size, cache.kv_layout,
                                     cache.k.data_ptr(), cache.v.data_ptr(), _stream(stream, dev)), "flexq_append_kv")


def flexq_decode_attention_workspace_size(batch, heads, head_dim, prompt_len, gen_len, bits=BITS,
                                          group_size=GROUP, kv_layout=KV_DENSE) -> int:
    return int(lib().flexq_decode_attention_workspace_size(batch, heads, head_dim, prompt_len, gen_len,
                                                           bits, group_size, kv_layout))


def make_workspace(cache: KVCache) -> torch.Tensor:
    n = flexq_decode_attention_workspace_size(cache.batch, cache.heads, cache.head_dim, cache.prompt_len,
                                              cache.gen_len, cache.bits, cache.group_size, cache.kv_layout)
    return torch.zeros(n, dtype=torch.uint8, device=cache.k.device)


def flexq_decode_attention(q: torch.Tensor, cache: KVCache, cur_len: int, out=None, workspace=None,
                           stream=None) -> torch.Tensor:
    """q fp16 [B][H][D] -> out fp16 [B][H][D] over cache tokens [0, cur_len)."""
    dev, shp = cache.k.device, (cache.batch, cache.heads, cache.head_dim)
    _need(q, torch.float16, "q", shp, dev)
    if out is None:
        out = torch.empty_like(q)
    if workspace is None:
        workspace = make_workspace(cache)
    _need(out, torch.float16, "out", shp, dev)
    _need(workspace, torch.uint8, "workspace", device=dev)
    with torch.cuda.device(dev):
        _check(lib().flexq_decode_attention(q.data_ptr(), cache.k.data_ptr(), cache.v.data_ptr(), cache.batch,
                                            cache.heads, cache.head_dim, cache.prompt_len, cache.gen_len,
                                            cur_len, cache.bits, cache.group_size, cache.kv_layout, out.data_ptr(),
                                            workspace.data_ptr(), workspace.numel(), _stream(stream, dev)),
               "flexq_decode_attention")
    return out


def flexq_append_decode_attention(q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor, cache: KVCache,
                                  cur_len: int, out=None, workspace=None, stream=None) -> torch.Tensor:
    """One layer's decode step in one launch (NEXT-3): append k_new / v_new fp16 [B][H][D] (or
    [B][H][1][D]) at position cur_len - 1, then attend over [0, cur_len).  Same cache bytes as
    flexq_append_kv, same output bound as flexq_decode_attention."""
    dev, shp = cache.k.device, (cache.batch, cache.heads, cache.head_dim)
    _need(q, torch.float16, "q", shp, dev)
    _need(k_new, torch.float16, "k_new", device=dev)
    _need(v_new, torch.float16, "v_new", device=dev)
    if k_new.numel() != q.numel() or v_new.numel() != q.numel():
        raise ValueError("k_new / v_new must hold one token per (batch, head): [B][H][D]")
    if out is None:
        out = torch.empty_like(q)
    if workspace is None:
        workspace = make_workspace(cache)
    _need(out, torch.float16, "out", shp, dev)
    _need(workspace, torch.uint8, "workspace", device=dev)
    with torch.cuda.device(dev):
        _check(lib().flexq_append_decode_attention(q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(),
                                                   cache.k.data_ptr(), cache.v.data_ptr(), cache.batch, cache.heads,
                                                   cache.head_dim, cache.prompt_len, cache.gen_len, cur_len,
                                                   cache.bits, cache.group_size, cache.kv_layout, out.data_ptr(),
                                                   workspace.data_ptr(), workspace.numel(), _stream(stream, dev)),
               "flexq_append_decode_attention")
    return out


def topk_keep(cur_len: int, fraction: float = 0.1) -> int:
    """Tokens kept by FlexGen's Top-K sparse attention: ceil(fraction * cur_len)."""
    import math
    return max(1, min(cur_len, math.ceil(fraction * cur_len - 1e-9)))


def make_topk_workspace(cache: KVCache) -> torch.Tensor:
    n = int(lib().flexq_decode_attention_topk_workspace_size(cache.batch, cache.heads, cache.head_dim,
                                                             cache.prompt_len, cache.gen_len, cache.bits,
                                                             cache.group_size, cache.kv_layout))
    if n == 0:
        raise FlexqError(FLEXQ_ERR_UNSUPPORTED, "flexq_decode_attention_topk_workspace_size")
    return torch.zeros(n, dtype=torch.uint8, device=cache.k.device)


def flexq_decode_attention_topk(q: torch.Tensor, cache: KVCache, cur_len: int, keep: int, out=None, sel=None,
                                workspace=None, stream=None) -> torch.Tensor:
    """Top-K sparse decode attention.  sel: optional int32 [B][H][keep] output
    receiving the kept token indices (ascending).  workspace: make_topk_workspace(cache)."""
    dev, shp = cache.k.device, (cache.batch, cache.heads, cache.head_dim)
    _need(q, torch.float16, "q", shp, dev)
    if out is None:
        out = torch.empty_like(q)
    if workspace is None:
        workspace = make_topk_workspace(cache)
    _need(out, torch.float16, "out", shp, dev)
    _need(workspace, torch.uint8, "workspace", device=dev)
    if sel is not None:
        _need(sel, torch.int32, "sel", (cache.batch, cache.heads, keep), dev)
    with torch.cuda.device(dev):
        _check(lib().flexq_decode_attention_topk(q.data_ptr(), cache.k.data_ptr(), cache.v.data_ptr(), cache.batch,
                                                 cache.heads, cache.head_dim, cache.prompt_len, cache.gen_len,
                                                 cur_len, keep, cache.bits, cache.group_size, cache.kv_layout,
                                                 out.data_ptr(),
                                                 _ptr(sel), workspace.data_ptr(), workspace.numel(),
                                                 _stream(stream, dev)),
               "flexq_decode_attention_topk")
    return out


# ---------------------------------------------------------------- decode linear layer (NEXT-2)
def flexq_gemm_panel_bytes(k: int, n: int, bits: int = BITS, group_size: int = GROUP) -> int:
    return int(lib().flexq_gemm_panel_bytes(k, n, bits, group_size))


def flexq_pack_weight(codes: torch.Tensor, meta: torch.Tensor, out=None, bits: int = BITS, group_size: int = GROUP,
                      stream=None) -> torch.Tensor:
    """One-time re-layout of a quantized [k][n] weight (codes u8 [k][n/2], meta [k][n/g][2])
    into the GEMM's panel format (u8, same total size)."""
    _need(codes, torch.uint8, "codes")
    k, half_n = codes.shape
    n = half_n * 2
    dev = codes.device
    _need(meta, torch.float16, "meta", (k, n // group_size, 2), dev)
    if out is None:
        out = torch.empty(max(flexq_gemm_panel_bytes(k, n, bits, group_size), 16), dtype=torch.uint8, device=dev)
    _need(out, torch.uint8, "panels", device=dev)
    if out.numel() < flexq_gemm_panel_bytes(k, n, bits, group_size):
        raise ValueError("panels buffer smaller than flexq_gemm_panel_bytes(k, n)")
    with torch.cuda.device(dev):
        _check(lib().flexq_pack_weight(codes.data_ptr(), meta.data_ptr(), k, n, bits, group_size, out.data_ptr(),
                                       _stream(stream, dev)), "flexq_pack_weight")
    return out


def flexq_dequant_gemm_workspace_size(m: int, k: int, n: int, bits: int = BITS, group_size: int = GROUP) -> int:
    return int(lib().flexq_dequant_gemm_workspace_size(m, k, n, bits, group_size))


def make_gemm_workspace(m: int, k: int, n: int, device) -> torch.Tensor:
    """Zeroed workspace for flexq_dequant_gemm (every call leaves its tickets zeroed)."""
    return torch.zeros(max(flexq_dequant_gemm_workspace_size(m, k, n), 16), dtype=torch.uint8, device=device)


def flexq_dequant_gemm(x: torch.Tensor, panels: torch.Tensor, n: int, out=None, workspace=None, bits: int = BITS,
                       group_size: int = GROUP, stream=None) -> torch.Tensor:
    """y fp16 [m][n] = x fp16 [m][k] . w^; panels = flexq_pack_weight(codes, meta)."""
    _need(x, torch.float16, "x")
    m, k = x.shape
    dev = x.device
    _need(panels, torch.uint8, "panels", device=dev)
    if panels.numel() < flexq_gemm_panel_bytes(k, n, bits, group_size):
        raise ValueError("panels smaller than flexq_gemm_panel_bytes(k, n): packed for another shape?")
    if out is None:
        out = torch.empty(m, n, dtype=torch.float16, device=dev)
    if workspace is None:
        workspace = make_gemm_workspace(m, k, n, dev)
    _need(out, torch.float16, "out", (m, n), dev)
    _need(workspace, torch.uint8, "workspace", device=dev)
    with torch.cuda.device(dev):
        _check(lib().flexq_dequant_gemm(x.data_ptr(), panels.data_ptr(), m, k, n, bits, group_size, out.data_ptr(),
                                        workspace.data_ptr(), workspace.numel(), _stream(stream, dev)),
               "flexq_dequant_gemm")
    return out

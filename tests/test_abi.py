"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/flexq.h declares, and rejects bad arguments on the host before
any CUDA call (include/flexq.h "Conventions")."""
import ctypes

import pytest

from paper_2303_06865_b200 import flexq as fq

A = 0x10000          # fake 16-byte-aligned "device" pointers: validation never dereferences
U = 0x10008          # misaligned


@pytest.fixture(scope="module")
def L():
    return fq.lib()


def test_exports_every_header_symbol(L):
    syms = fq.header_symbols()
    assert {"flexq_quantize", "flexq_dequantize", "flexq_append_kv", "flexq_decode_attention",
            "flexq_decode_attention_workspace_size", "flexq_status_string", "flexq_abi_version",
            "flexq_kv_cache_bytes"} <= set(syms)
    for s in syms:
        assert hasattr(L, s), s


def test_version_and_status_strings(L):
    assert L.flexq_abi_version() == 2
    for s in range(-2, 10):
        assert L.flexq_status_string(s)            # never NULL


def test_quantize_validation(L):
    q = L.flexq_quantize
    assert q(A, -1, 128, 4, 64, A, A, None) == fq.FLEXQ_ERR_ARG
    assert q(A, 4, 128, 0, 64, A, A, None) == fq.FLEXQ_ERR_ARG      # bits < 1
    assert q(A, 4, 128, 9, 64, A, A, None) == fq.FLEXQ_ERR_ARG      # bits > 8
    assert q(A, 4, 128, 4, 0, A, A, None) == fq.FLEXQ_ERR_ARG
    assert q(A, 4, 128, 5, 64, A, A, None) == fq.FLEXQ_ERR_UNSUPPORTED   # b = 5: legal, not built
    assert q(A, 4, 128, 1, 64, A, A, None) == fq.FLEXQ_ERR_UNSUPPORTED
    assert q(A, 4, 128, 4, 16, A, A, None) == fq.FLEXQ_ERR_UNSUPPORTED   # g = 16: legal, not built
    assert q(A, 4, 96, 4, 48, A, A, None) == fq.FLEXQ_ERR_UNSUPPORTED
    assert q(A, 4, 96, 3, 64, A, A, None) == fq.FLEXQ_ERR_UNSUPPORTED    # partial group (reading I)
    assert q(A, 4, 100, 4, 64, A, A, None) == fq.FLEXQ_ERR_UNSUPPORTED   # partial group (reading I)
    assert q(None, 4, 128, 4, 64, A, A, None) == fq.FLEXQ_ERR_NULL
    assert q(A, 4, 128, 4, 64, None, A, None) == fq.FLEXQ_ERR_NULL
    assert q(U, 4, 128, 4, 64, A, A, None) == fq.FLEXQ_ERR_ALIGN
    assert q(A, 0, 128, 4, 64, None, None, None) == fq.FLEXQ_OK      # empty: no-op, no launch
    assert q(A, 4, 0, 4, 64, None, None, None) == fq.FLEXQ_OK


def test_dequantize_validation(L):
    d = L.flexq_dequantize
    assert d(A, A, 4, 128, 4, 65, A, None) == fq.FLEXQ_ERR_UNSUPPORTED
    assert d(A, A, 4, 128, 6, 64, A, None) == fq.FLEXQ_ERR_UNSUPPORTED
    assert d(A, A, 4, 96, 8, 64, A, None) == fq.FLEXQ_ERR_UNSUPPORTED
    assert d(A, A, 4, 128, 10, 64, A, None) == fq.FLEXQ_ERR_ARG
    assert d(A, None, 4, 128, 4, 64, A, None) == fq.FLEXQ_ERR_NULL
    assert d(A, A, 4, 128, 4, 64, U, None) == fq.FLEXQ_ERR_ALIGN
    assert d(A, A, 0, 128, 4, 64, A, None) == fq.FLEXQ_OK


def test_append_validation(L):
    f = L.flexq_append_kv

    def call(B=2, H=3, D=128, s=8, n=4, pos=0, nn=1, bits=4, g=64, k=A, kv=A, lay=0):
        return f(k, A, B, H, D, s, n, pos, nn, bits, g, lay, A, kv, None)
    assert call(B=0) == fq.FLEXQ_ERR_ARG
    assert call(pos=-1) == fq.FLEXQ_ERR_ARG
    assert call(pos=12) == fq.FLEXQ_ERR_ARG            # pos + n_new > s + n
    assert call(pos=10, nn=3) == fq.FLEXQ_ERR_ARG
    assert call(nn=0) == fq.FLEXQ_ERR_ARG
    assert call(D=96) == fq.FLEXQ_ERR_UNSUPPORTED
    assert call(bits=5) == fq.FLEXQ_ERR_UNSUPPORTED       # legal, not built
    assert call(g=16) == fq.FLEXQ_ERR_UNSUPPORTED
    assert call(D=64, bits=2, g=128) == fq.FLEXQ_ERR_UNSUPPORTED   # head_dim % group != 0
    assert call(bits=9) == fq.FLEXQ_ERR_ARG
    assert call(bits=3, g=32, k=None) == fq.FLEXQ_ERR_NULL          # a built variant gets to the pointer checks
    assert call(k=None) == fq.FLEXQ_ERR_NULL
    assert call(kv=None) == fq.FLEXQ_ERR_NULL
    assert call(kv=U) == fq.FLEXQ_ERR_ALIGN
    assert call(lay=2) == fq.FLEXQ_ERR_ARG           # flexq_kv_layout: 0 dense, 1 token-major
    assert call(lay=-1) == fq.FLEXQ_ERR_ARG
    assert call(lay=1, k=None) == fq.FLEXQ_ERR_NULL


def test_attention_validation(L):
    f = L.flexq_decode_attention
    ws = L.flexq_decode_attention_workspace_size(2, 3, 128, 8, 4, 4, 64, 0)
    assert ws > 0
    assert L.flexq_decode_attention_workspace_size(0, 3, 128, 8, 4, 4, 64, 0) == 0
    assert L.flexq_decode_attention_workspace_size(2, 3, 128, 8, 4, 4, 64, 7) == 0   # no such layout
    # (4, 64) token-major: the variant kernel's workspace or the dense one, whichever is larger
    wt = L.flexq_decode_attention_workspace_size(2, 3, 128, 8, 4, 4, 64, 1)
    assert wt == max(ws, 256 + (6 * 1 * 130 * 4 + 15) // 16 * 16)

    def call(cur=5, D=128, q=A, kv=A, out=A, w=A, wb=ws, g=64, lay=0):
        return f(q, A, kv, 2, 3, D, 8, 4, cur, 4, g, lay, out, w, wb, None)
    assert call(cur=0) == fq.FLEXQ_ERR_ARG
    assert call(cur=13) == fq.FLEXQ_ERR_ARG             # cur_len > s + n
    assert call(D=32) == fq.FLEXQ_ERR_UNSUPPORTED
    assert call(g=16) == fq.FLEXQ_ERR_UNSUPPORTED
    assert call(D=64, g=128) == fq.FLEXQ_ERR_UNSUPPORTED
    assert call(q=None) == fq.FLEXQ_ERR_NULL
    assert call(kv=None) == fq.FLEXQ_ERR_NULL
    assert call(out=U) == fq.FLEXQ_ERR_ALIGN
    assert call(lay=3) == fq.FLEXQ_ERR_ARG
    assert call(lay=1, wb=wt - 1) == fq.FLEXQ_ERR_WORKSPACE
    # variants (NEXT-3): their own workspace size, 256 B + (D + 2) floats per (b, h, 128-token tile)
    wv = L.flexq_decode_attention_workspace_size(2, 3, 128, 8, 4, 3, 32, 0)
    assert wv == 256 + (6 * 1 * 130 * 4 + 15) // 16 * 16
    assert L.flexq_decode_attention_workspace_size(2, 3, 128, 8, 4, 3, 32, 1) == wv   # same layout
    assert L.flexq_decode_attention_workspace_size(2, 3, 128, 300, 0, 8, 128, 0) == 256 + 6 * 3 * 130 * 4
    assert f(A, A, A, 2, 3, 128, 8, 4, 5, 3, 32, 0, A, A, wv - 1, None) == fq.FLEXQ_ERR_WORKSPACE
    assert f(None, A, A, 2, 3, 128, 8, 4, 5, 3, 32, 0, A, A, wv, None) == fq.FLEXQ_ERR_NULL
    assert call(w=None) == fq.FLEXQ_ERR_WORKSPACE
    assert call(wb=ws - 1) == fq.FLEXQ_ERR_WORKSPACE


def test_kv_cache_bytes(L):
    c, t = fq.flexq_kv_cache_bytes(144, 96, 128, 512, 32)
    assert t == 544                                   # 544 = 17 chunks of 32: no padding
    assert c == 144 * 96 * 17 * 18 * 128              # one buffer (K or V)
    assert c * 8 == 144 * 96 * 544 * 128 * 4.5        # 4.5 bits per element
    c, t = fq.flexq_kv_cache_bytes(4, 12, 64, 512, 1)
    assert t == 544 and c == 4 * 12 * 17 * 18 * 64
    # variants: chunk = 32 x (D b / 8 code bytes + 4 D / g meta bytes)
    c, t = fq.flexq_kv_cache_bytes(144, 96, 128, 512, 32, bits=3, group_size=32)
    assert c == 144 * 96 * 17 * 32 * (48 + 16)
    c, _ = fq.flexq_kv_cache_bytes(2, 2, 64, 40, 0, bits=8, group_size=64)
    assert c == 2 * 2 * 2 * 32 * (64 + 4)
    c, _ = fq.flexq_kv_cache_bytes(2, 2, 128, 40, 0, bits=2, group_size=128)
    assert c == 2 * 2 * 2 * 32 * (32 + 4)
    assert fq.token_stride(513) == 544 and fq.token_stride(1) == 32 and fq.token_stride(32) == 32
    with __import__("pytest").raises(fq.FlexqError):
        fq.flexq_kv_cache_bytes(1, 1, 96, 8, 8)


def test_topk_validation(L):
    f = L.flexq_decode_attention_topk
    L.flexq_decode_attention_topk_workspace_size.restype = ctypes.c_size_t
    ws = L.flexq_decode_attention_topk_workspace_size(2, 3, 128, 8, 4, 4, 64, 1)
    assert ws == 2048 + 2 * 3 * 12 * 8          # counters + (index, weight) per (b, h, token)
    assert L.flexq_decode_attention_topk_workspace_size(2, 3, 128, 8, 4, 4, 64, 0) == ws
    assert L.flexq_decode_attention_topk_workspace_size(2, 3, 128, 8, 4, 3, 32, 0) == 0   # b = 4, g = 64 only

    def call(cur=5, keep=2, D=128, q=A, out=A, sel=None, w=A, s=8, n=4, lay=1):
        return f(q, A, A, 2, 3, D, s, n, cur, keep, 4, 64, lay, out, sel, w, ws, None)
    assert call(keep=0) == fq.FLEXQ_ERR_ARG
    assert call(keep=6) == fq.FLEXQ_ERR_ARG          # keep > cur_len
    assert call(cur=13) == fq.FLEXQ_ERR_ARG
    assert call(D=96) == fq.FLEXQ_ERR_UNSUPPORTED
    assert call(cur=1153, keep=5, s=1200, n=0) == fq.FLEXQ_ERR_UNSUPPORTED   # beyond the score buffer
    assert f(A, A, A, 2, 3, 128, 8, 4, 5, 2, 3, 32, 0, A, None, A, ws, None) == fq.FLEXQ_ERR_UNSUPPORTED   # b = 4, g = 64 only
    assert call(lay=2) == fq.FLEXQ_ERR_ARG
    assert call(lay=0, q=None) == fq.FLEXQ_ERR_NULL    # the dense layout is accepted too
    assert call(q=None) == fq.FLEXQ_ERR_NULL
    assert call(sel=U) == fq.FLEXQ_ERR_ALIGN
    assert call(w=None) == fq.FLEXQ_ERR_WORKSPACE
    assert f(A, A, A, 2, 3, 128, 8, 4, 5, 2, 4, 64, 1, A, None, A, ws - 1, None) == fq.FLEXQ_ERR_WORKSPACE
    assert fq.topk_keep(543) == 55 and fq.topk_keep(130) == 13 and fq.topk_keep(5) == 1


def test_append_attention_validation(L):
    f = L.flexq_append_decode_attention
    ws = L.flexq_decode_attention_workspace_size(2, 3, 128, 8, 4, 4, 64, 0)

    def call(cur=5, D=128, q=A, kn=A, vn=A, kv=A, out=A, w=A, wb=ws, g=64, lay=0):
        return f(q, kn, vn, kv, A, 2, 3, D, 8, 4, cur, 4, g, lay, out, w, wb, None)
    assert call(cur=0) == fq.FLEXQ_ERR_ARG
    assert call(cur=13) == fq.FLEXQ_ERR_ARG
    assert call(D=96) == fq.FLEXQ_ERR_UNSUPPORTED
    assert call(g=16) == fq.FLEXQ_ERR_UNSUPPORTED
    assert call(kn=None) == fq.FLEXQ_ERR_NULL
    assert call(vn=None) == fq.FLEXQ_ERR_NULL
    assert call(kv=None) == fq.FLEXQ_ERR_NULL
    assert call(vn=U) == fq.FLEXQ_ERR_ALIGN
    assert call(w=None) == fq.FLEXQ_ERR_WORKSPACE
    assert call(wb=ws - 1) == fq.FLEXQ_ERR_WORKSPACE
    assert call(lay=5) == fq.FLEXQ_ERR_ARG


def test_dequant_gemm_validation(L):
    f = L.flexq_dequant_gemm
    ws = L.flexq_dequant_gemm_workspace_size(144, 12288, 49152, 4, 64)
    assert ws > 0
    assert L.flexq_dequant_gemm_workspace_size(144, 12288, 49152, 4, 32) == 0
    assert L.flexq_dequant_gemm_workspace_size(144, 100, 49152, 4, 64) == 0
    # panels are a re-layout: the bytes of codes + meta, plus a 16-byte flag trailer per panel
    assert L.flexq_gemm_panel_bytes(12288, 49152, 4, 64) == (12288 * 49152 // 2 + 12288 * 49152 // 64 * 4
                                                             + 16 * (49152 // 256) * (12288 // 64))
    assert L.flexq_gemm_panel_bytes(12288, 100, 4, 64) == 0

    def call(m=144, k=12288, n=49152, x=A, pn=A, y=A, w=A, wb=ws, b=4, g=64):
        return f(x, pn, m, k, n, b, g, y, w, wb, None)
    assert call(m=-1) == fq.FLEXQ_ERR_ARG
    assert call(k=-1) == fq.FLEXQ_ERR_ARG
    assert call(b=9) == fq.FLEXQ_ERR_ARG
    assert call(g=0) == fq.FLEXQ_ERR_ARG
    assert call(b=3) == fq.FLEXQ_ERR_UNSUPPORTED
    assert call(g=128) == fq.FLEXQ_ERR_UNSUPPORTED
    assert call(n=100) == fq.FLEXQ_ERR_UNSUPPORTED      # partial group (reading I)
    assert call(n=192) == fq.FLEXQ_ERR_UNSUPPORTED      # n % 256 != 0: not built
    assert call(k=96) == fq.FLEXQ_ERR_UNSUPPORTED       # k % 64 != 0: not built
    assert call(k=0) == fq.FLEXQ_ERR_UNSUPPORTED
    assert call(x=None) == fq.FLEXQ_ERR_NULL
    assert call(pn=None) == fq.FLEXQ_ERR_NULL
    assert call(y=U) == fq.FLEXQ_ERR_ALIGN
    assert call(w=None) == fq.FLEXQ_ERR_WORKSPACE
    assert call(wb=ws - 1) == fq.FLEXQ_ERR_WORKSPACE
    assert call(m=0, x=None, pn=None, y=None, w=None) == fq.FLEXQ_OK   # empty: no-op
    pk = L.flexq_pack_weight
    assert pk(A, A, 128, 100, 4, 64, A, None) == fq.FLEXQ_ERR_UNSUPPORTED
    assert pk(A, A, 128, 256, 4, 32, A, None) == fq.FLEXQ_ERR_UNSUPPORTED
    assert pk(A, None, 128, 256, 4, 64, A, None) == fq.FLEXQ_ERR_NULL
    assert pk(A, A, 128, 256, 4, 64, U, None) == fq.FLEXQ_ERR_ALIGN
    assert pk(A, A, 0, 256, 4, 64, None, None) == fq.FLEXQ_OK

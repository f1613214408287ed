"""Pins for the oracle's decode linear layer over a 4-bit weight (G1), CPU only.

y = t . w^ where w^ is the weight "converted back to FP16 before
computation" from groups of 64 along the output channel (reading J).

Pinned against, none of which calls the oracle's own G1 code path:
  * numpy: the fp16 weight rebuilt in numpy from codes/meta (c*s is exact in fp32, so
    f32(c*s) + f32(min) rounds once, like fmaf), then float64 matmul;
  * closed forms: one-hot rows of t select rows of w^; a weight whose groups hold exactly
    representable levels reconstructs exactly, so y = t . w bit-for-bit in f64;
  * all-zero codes: y[m][n] = sum_k t[m][k] * min[k][n/64] (the offset term alone);
  * linearity in t, and the group index (a transposed or mis-grouped weight fails these).
"""
import numpy as np
import pytest

from paper_2303_06865_b200 import synth


def numpy_dequant_f16(codes, meta, group=64):
    """Independent O7 in numpy: f16(clip(f32(c*s) + f32(min))) -- c*s is exact in fp32."""
    s = meta[..., 0].view(np.float16).astype(np.float32)
    m = meta[..., 1].view(np.float16).astype(np.float32)
    s = np.repeat(s, group, axis=-1)
    m = np.repeat(m, group, axis=-1)
    v = codes.astype(np.float32) * s + m
    return np.clip(v, -65504, 65504).astype(np.float16)


def make(orc, M, K, N, seed):
    w = synth.fill(seed, 1, (K, N)).numpy()
    x = synth.fill(seed, 2, (M, K)).numpy()
    codes, meta = orc.quantize(w, 4, 64)
    return x, w, codes, meta


@pytest.mark.parametrize("M,K,N", [(3, 64, 64), (5, 130, 192), (16, 256, 128)])
def test_matches_numpy(orc, M, K, N):
    x, _, codes, meta = make(orc, M, K, N, seed=31)
    got = orc.dequant_gemm_f64(x, codes, meta)
    wq = numpy_dequant_f16(codes, meta).astype(np.float64)
    ref = x.astype(np.float64) @ wq
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_weight_is_the_dequantize_output(orc):
    """The operand is O7's fp16 value: one-hot rows of t pick rows of w^ exactly."""
    K, N = 96, 128
    _, _, codes, meta = make(orc, 1, K, N, seed=32)
    x = np.zeros((K, K), np.float16)
    x[np.arange(K), np.arange(K)] = 1.0
    got = orc.dequant_gemm_f64(x, codes, meta)
    wq = orc.dequantize(codes, meta).astype(np.float64)
    assert np.array_equal(got, wq)
    # and the numpy rebuild agrees bit for bit
    assert np.array_equal(wq, numpy_dequant_f16(codes, meta).astype(np.float64))


def test_exact_levels_give_exact_product(orc):
    """Groups holding min + j*step (j = 0..15, step a power of two) quantize and reconstruct
    exactly, so y equals t . w computed directly from w."""
    K, N = 64, 128
    rng = np.random.default_rng(7)
    lv = rng.integers(0, 16, size=(K, N))
    lv[:, ::64] = 0
    lv[:, 1::64] = 15                              # every group spans the full 0..15 range
    mins = rng.integers(-8, 8, size=(K, N // 64)).astype(np.float64)
    step = 2.0 ** rng.integers(-6, -1, size=(K, N // 64))
    w = (np.repeat(mins, 64, axis=1) + lv * np.repeat(step, 64, axis=1)).astype(np.float16)
    codes, meta = orc.quantize(w, 4, 64)
    assert np.array_equal(codes, lv)
    x = synth.fill(33, 2, (4, K)).numpy()
    got = orc.dequant_gemm_f64(x, codes, meta)
    ref = x.astype(np.float64) @ w.astype(np.float64)
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-13)


def test_zero_codes_leave_the_offset_term(orc):
    K, N, M = 64, 192, 3
    codes = np.zeros((K, N), np.uint8)
    meta = np.zeros((K, N // 64, 2), np.uint16)
    rng = np.random.default_rng(9)
    mins = rng.standard_normal((K, N // 64)).astype(np.float16)
    meta[..., 0] = np.float16(0.5).view(np.uint16)
    meta[..., 1] = mins.view(np.uint16)
    x = synth.fill(34, 2, (M, K)).numpy()
    got = orc.dequant_gemm_f64(x, codes, meta)
    ref = x.astype(np.float64) @ np.repeat(mins.astype(np.float64), 64, axis=1)
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-13)
    # group n/64: column 64 takes group 1's min, not group 0's
    assert np.allclose(got[:, 64], x.astype(np.float64) @ mins[:, 1].astype(np.float64))


def test_linear_in_t(orc):
    x, _, codes, meta = make(orc, 4, 128, 128, seed=35)
    a = orc.dequant_gemm_f64(x, codes, meta)
    x2 = (x.astype(np.float32) * 2).astype(np.float16)        # exact
    b = orc.dequant_gemm_f64(x2, codes, meta)
    assert np.array_equal(b, 2 * a)
    xs = np.concatenate([x[2:], x[:2]])
    c = orc.dequant_gemm_f64(xs, codes, meta)
    assert np.array_equal(c, np.concatenate([a[2:], a[:2]]))


def test_rejects_bad_group(orc):
    x, _, codes, meta = make(orc, 2, 64, 64, seed=36)
    with pytest.raises(ValueError):
        orc.dequant_gemm_f64(x, codes[:, :48], meta)

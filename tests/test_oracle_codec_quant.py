"""Pins for the oracle's fp16 codec (O1) and quantizer (O2-O7), CPU only.

Each pin checks the oracle against something other than itself: numpy's fp16
conversion (a library routine), exact rational arithmetic (Python Fractions),
a brute-force nearest-level search, hand-worked cases under tests/golden/
(with citations), and the invariants the paper / north_star fix (P:841-848,
S:469-477).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from paper_2303_06865_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------- O1 codec
def test_f16_to_f32_all_patterns(orc):
    """Every one of the 65,536 fp16 bit patterns decodes like numpy's float16."""
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ref = bits.view(np.float16).astype(np.float32)
    got = np.array([orc.f16_to_f32(int(b)) for b in bits], np.float32)
    fin = np.isfinite(ref)
    assert np.array_equal(got[fin].view(np.uint32), ref[fin].view(np.uint32))
    assert np.all(np.isnan(got[np.isnan(ref)]))
    assert np.array_equal(got[np.isinf(ref)], ref[np.isinf(ref)])


def test_f32_to_f16_matches_numpy(orc):
    """RNE conversion incl. ties, subnormal edge and the 65504/65520 overflow edge."""
    rng = np.random.default_rng(1)
    vals = [0.0, -0.0, 65504.0, 65519.99, 65520.0, 65536.0, 1e9, -65520.0,
            2.0 ** -24, 2.0 ** -25, 3 * 2.0 ** -26, 2.0 ** -14, 2.0 ** -14 - 2.0 ** -25,
            1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11, 2049.0, 2051.0, 0.1, 1 / 3]
    # exact midpoints between adjacent fp16 values (ties) across the whole range
    h = np.arange(0, 0x7BFF, 7, dtype=np.uint16)
    lo = h.view(np.float16).astype(np.float64)
    hi = (h + 1).view(np.float16).astype(np.float64)
    mids = ((lo + hi) / 2).astype(np.float32)
    rand = (rng.standard_normal(20000) * np.exp2(rng.integers(-26, 17, 20000))).astype(np.float32)
    xs = np.concatenate([np.array(vals, np.float32), mids, -mids, rand])
    ref = xs.astype(np.float16).view(np.uint16)
    got = np.array([orc.f32_to_f16(float(x)) for x in xs], np.uint16)
    assert np.array_equal(got, ref)


# ----------------------------------------------------------------- golden cases
def test_golden_closed_forms(orc):
    g = json.load(open(os.path.join(GOLDEN, "quantize_closed_forms.json")))
    for case in g["cases"]:
        x = np.array(case["x"], np.float16)[None, :]
        codes, meta = orc.quantize(x, bits=case["bits"], group=x.shape[1])
        assert codes[0].tolist() == case["codes"], case["name"]
        scale = float(meta[0, 0, 0:1].view(np.float16)[0])
        mn = float(meta[0, 0, 1:2].view(np.float16)[0])
        assert abs(scale - case["scale"]) < 1e-8, case["name"]
        assert mn == case["min"], case["name"]
    p = g["pack4"]
    assert orc.pack4(np.array(p["codes"], np.uint8)).tolist() == p["bytes"]
    assert orc.unpack4(np.array(p["bytes"], np.uint8)).tolist() == p["codes"]


# ----------------------------------------------------------------- exact-rational pin
def _exact_codes(xg: np.ndarray, bits: int):
    """Exact rational code for every element: RNE((x-min)/(max-min)*(2^b-1)).
    Returns (codes, t_exact) computed with Fractions (no floating point)."""
    L = (1 << bits) - 1
    vals = [Fraction(float(v)) for v in xg.astype(np.float64)]
    mn, mx = min(vals), max(vals)
    if mx == mn:
        return [0] * len(vals), [Fraction(0)] * len(vals)
    codes, ts = [], []
    for v in vals:
        t = (v - mn) / (mx - mn) * L
        k = int(t)                     # floor (t >= 0)
        d = t - k
        c = k + 1 if d > Fraction(1, 2) else k if d < Fraction(1, 2) else (k if k % 2 == 0 else k + 1)
        codes.append(c)
        ts.append(t)
    return codes, ts


def _f32_exact(x: float) -> bool:
    return float(np.float32(x)) == x


@pytest.mark.parametrize("bits", [4, 2, 8])
def test_quantize_equals_exact_rational(orc, bits):
    """O4 in fp32 equals the exact rational RNE code wherever x-min and max-min
    are exact in fp32 and t is not within 4 ulps of a half-integer without being one."""
    x = synth.fill(11, 3, (64, 64)).numpy()
    x = np.concatenate([x, synth.ties(11, 4, (32, 64)).numpy(),
                        synth.with_outliers(synth.fill(11, 5, (32, 128))).numpy().reshape(64, 64)])
    codes, _ = orc.quantize(x, bits=bits, group=64)
    flagged = checked = 0
    for r in range(x.shape[0]):
        ex, ts = _exact_codes(x[r], bits)
        xv = x[r].astype(np.float64)
        mn, mx = xv.min(), xv.max()
        for j in range(64):
            if not (_f32_exact(xv[j] - mn) and _f32_exact(mx - mn)):
                continue
            t = ts[j]
            frac = t - int(t)
            if frac != Fraction(1, 2) and abs(frac - Fraction(1, 2)) < Fraction(4, 2 ** 20):
                flagged += 1
                continue
            checked += 1
            assert codes[r, j] == ex[j], (r, j, float(t))
    assert checked > 0.95 * x.size
    assert flagged <= 2


def test_quantize_nearest_level_bruteforce(orc):
    """Brute force: each code is the index of the nearest of the 2^b levels
    min + k*(max-min)/(2^b-1) (exact rationals), ties to the even index."""
    for bits in (1, 2, 3):
        L = (1 << bits) - 1
        x = synth.fill(12, bits, (40, 8)).numpy()
        codes, _ = orc.quantize(x, bits=bits, group=8)
        for r in range(x.shape[0]):
            vals = [Fraction(float(v)) for v in x[r].astype(np.float64)]
            mn, mx = min(vals), max(vals)
            for j, v in enumerate(vals):
                dists = [abs(v - (mn + k * (mx - mn) / L)) for k in range(L + 1)]
                best = min(dists)
                ks = [k for k, d in enumerate(dists) if d == best]
                want = ks[0] if len(ks) == 1 else [k for k in ks if k % 2 == 0][0]
                assert codes[r, j] == want


# ----------------------------------------------------------------- invariants
def test_minmax_recovered_and_endpoints(orc):
    """north_star: group min recovered exactly (min16 bit-equal), argmin -> 0, argmax -> 2^b-1."""
    x = np.concatenate([synth.fill(13, 1, (200, 128)).numpy(),
                        synth.with_outliers(synth.fill(13, 2, (50, 128))).numpy()])
    codes, meta = orc.quantize(x, 4, 64)
    g = x.reshape(-1, 64)
    c = codes.reshape(-1, 64)
    m = meta.reshape(-1, 2)
    mins = g.min(axis=1)
    mins = np.where(mins == 0, np.float16(0), mins)       # reading P: -0 -> +0
    assert np.array_equal(m[:, 1], mins.view(np.uint16))
    rows = np.arange(g.shape[0])
    assert np.all(c[rows, g.argmin(axis=1)] == 0)
    assert np.all(c[rows, g.argmax(axis=1)] == 15)
    # max value reconstructed within 15*|scale16 - r/15| + half an fp16 ulp (reading F iv)
    deq = orc.dequantize(codes, meta, 4, 64).reshape(-1, 64).astype(np.float64)
    r = g.max(axis=1).astype(np.float64) - g.min(axis=1).astype(np.float64)
    s16 = m[:, 0].view(np.float16).astype(np.float64)
    err = np.abs(deq[rows, g.argmax(axis=1)] - g.max(axis=1).astype(np.float64))
    assert np.all(err <= 15 * np.abs(s16 - r / 15) + np.abs(g.max(axis=1)).astype(np.float64) * 2.0 ** -11 + 1e-12)


def test_reconstruction_bound(orc):
    """S:472 / north_star: |x - (min + c*r/15)| <= (r/15)/2 with the exact step (reading G),
    over 10^5 elements; and the stored-scale bound for dequantize()."""
    x = synth.fill(14, 1, (1600, 64)).numpy()          # 102,400 elements
    codes, meta = orc.quantize(x, 4, 64)
    xv = x.astype(np.float64)
    mn = xv.min(axis=1, keepdims=True)
    r = xv.max(axis=1, keepdims=True) - mn
    recon = mn + codes.astype(np.float64) * r / 15
    assert np.all(np.abs(xv - recon) <= r / 30 * (1 + 2.0 ** -20))
    assert np.abs(xv - recon).max() > 0.45 * (r / 30).max() * 0.5    # bound is not vacuous
    deq = orc.dequantize(codes, meta, 4, 64).astype(np.float64)
    s16 = meta[:, 0, 0].view(np.float16).astype(np.float64)[:, None]
    bound = r / 30 + 15 * np.abs(s16 - r / 15) + np.abs(deq) * 2.0 ** -11 + 1e-12
    assert np.all(np.abs(xv - deq) <= bound)


def test_idempotence(orc):
    """quantize(dequantize(quantize(x))) reproduces the codes."""
    x = np.concatenate([synth.fill(15, 1, (300, 64)).numpy(),
                        synth.with_outliers(synth.fill(15, 2, (100, 128))).numpy().reshape(200, 64)])
    c1, m1 = orc.quantize(x, 4, 64)
    c2, _ = orc.quantize(orc.dequantize(c1, m1, 4, 64), 4, 64)
    assert np.array_equal(c1, c2)


def test_degenerate_and_extreme(orc):
    """Reading C (constant groups reconstruct exactly), R (clamp at +-65504), and
    codes always in range on every finite fp16 pattern."""
    x = synth.extreme(16, 1, 256, 128).numpy()
    codes, meta = orc.quantize(x, 4, 64)
    assert codes.max() <= 15
    deq = orc.dequantize(codes, meta, 4, 64)
    assert np.all(np.isfinite(deq.astype(np.float32)))
    g = x.reshape(-1, 64)
    const = (g == g[:, :1]).all(axis=1) & (g[:, 0] != 0)
    assert const.sum() > 10
    assert np.array_equal(deq.reshape(-1, 64)[const], g[const])
    assert np.all(codes.reshape(-1, 64)[const] == 0)


def test_unsupported_and_bad_args(orc):
    with pytest.raises(ValueError):
        orc.quantize(np.zeros((2, 100), np.float16), 4, 64)     # partial group (reading I)
    with pytest.raises(ValueError):
        orc.quantize(np.zeros((2, 64), np.float16), 9, 64)      # bits out of [1, 8]


# ---------------------------------------------------------------- O6 for any b (NEXT-3 variants)
def test_pack_bits_golden_bytes(orc):
    """Hand-worked little-endian bit streams."""
    # b = 2: codes [1, 2, 3, 0] -> bits 10 01 11 00 (LSB first) -> 0b00111001 = 0x39
    assert orc.pack_bits(np.array([1, 2, 3, 0], np.uint8), 2).tolist() == [0x39]
    # b = 3: codes [5, 3, 7, 1, 0, 2, 6, 4] -> stream (LSB of each code first)
    #   101 110 111 100 000 010 011 001
    #   byte 0 = stream bits 0..7   = 1,0,1,1,1,0,1,1 -> 0xDD
    #   byte 1 = stream bits 8..15  = 1,1,0,0,0,0,0,0 -> 0x03
    #   byte 2 = stream bits 16..23 = 1,0,0,1,1,0,0,1 -> 0x99
    assert orc.pack_bits(np.array([5, 3, 7, 1, 0, 2, 6, 4], np.uint8), 3).tolist() == [0xDD, 0x03, 0x99]
    # b = 8: identity; b = 4: oracle_pack4's nibble order
    c = np.arange(16, dtype=np.uint8)
    assert np.array_equal(orc.pack_bits(c, 8), c)
    c4 = np.random.default_rng(3).integers(0, 16, 64).astype(np.uint8)
    assert np.array_equal(orc.pack_bits(c4, 4), orc.pack4(c4))


@pytest.mark.parametrize("bits", [1, 2, 3, 4, 5, 7, 8])
def test_pack_bits_round_trip_and_numpy(orc, bits):
    rng = np.random.default_rng(bits)
    c = rng.integers(0, 1 << bits, size=(3, 64)).astype(np.uint8)
    p = orc.pack_bits(c, bits)
    assert p.shape == (3, 64 * bits // 8)
    assert np.array_equal(orc.unpack_bits(p, 64, bits), c)
    # independent numpy bit stream: unpackbits (little) of each code's b low bits, concatenated
    ref = np.packbits(np.unpackbits(c[..., None], axis=-1, bitorder="little")[..., :bits].reshape(3, -1),
                      axis=-1, bitorder="little")
    assert np.array_equal(p, ref)

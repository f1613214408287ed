"""GPU parity for the decode linear layer over a 4-bit weight (NEXT-2, flexq_dequant_gemm)
against the oracle's G1 (oracle_dequant_gemm_f64), through the C ABI.

The kernel's weight operand is one fp16 FMA, min(RN16(c*scale + min), 65504) (DESIGN.md reading
G2); the oracle uses O7's fp16 value (RN16 of the fp32 fmaf).  They differ by at most one fp16
ulp and only where RN32 of the exact value is an fp16 tie; the bound below covers it.

Tolerance ("dequant-GEMM tolerance"): fp16 x fp16 products are exact in fp32;
the tensor core accumulates each 16-term MMA into the fp32 accumulator, K/16 accumulations
per output, plus at most a handful of fp32 split-k partial additions; y is rounded once to
fp16.  Elementwise:
    |y - o| <= 2^-11 |o| + (K/16 + 8) * 2^-22 * S,   S = sum_k |x_mk| |w^_kn|
(half an fp16 ulp, plus a worst-case bound of one fp32 rounding of a partial sum bounded
by S per accumulation, with a 2x margin).  Normwise the result must also be within
2^-9 max|o| -- the fp16 rounding with a 4x margin -- which a dropped k-block, a wrong group
or a transposed operand all violate by orders of magnitude.
Oracle inputs are regenerated on the host by synth (never copied back from the device).
"""
import numpy as np
import pytest
import torch

from paper_2303_06865_b200 import flexq as fq
from paper_2303_06865_b200 import synth

pytestmark = pytest.mark.gpu


def check_gemm(got, x, codes, meta, orc, what=""):
    """got: fp16 [M][n] (numpy); x fp16 [M][K]; codes u8 [K][n] unpacked; meta [K][n/64][2]."""
    ref = orc.dequant_gemm_f64(x, codes, meta)
    wq = orc.dequantize(codes, meta).astype(np.float64)
    S = np.abs(x.astype(np.float64)) @ np.abs(wq)
    K = x.shape[1]
    g = got.astype(np.float64)
    err = np.abs(g - ref)
    tol = 2.0 ** -11 * np.abs(ref) + (K / 16 + 8) * 2.0 ** -22 * S
    bad = err > tol
    assert not bad.any(), f"{what}: {bad.sum()} of {bad.size} out of tolerance; max err {err.max():.3e}"
    assert err.max() <= 2.0 ** -9 * max(np.abs(ref).max(), 1e-30), f"{what}: normwise {err.max():.3e}"


def quantized(w, cuda):
    """flexq_quantize + flexq_pack_weight on the device -> panels."""
    codes, meta = fq.flexq_quantize(w.to(cuda))
    return fq.flexq_pack_weight(codes, meta), codes, meta


def weights(seed, K, N, outliers=False):
    w = synth.fill(seed, 1, (K, N))
    if outliers:
        w = synth.with_outliers(w)
    return w


GEMM_CASES = [
    # name, M, K, N
    ("m1_one_tile", 1, 64, 256),
    ("m5_two_tiles", 5, 128, 512),
    ("m144_split_k", 144, 640, 512),        # 10 k-blocks x 2 tiles over 148 CTAs: every tile split
    ("m16_deep_k", 16, 4096, 256),          # one tile, 64 k-blocks shared by 64 CTAs
    ("m33_ragged_rows", 33, 192, 768),      # rows not a multiple of 16
    ("m160_max_rows", 160, 128, 256),
    ("m256_two_row_chunks", 256, 128, 256),
    ("m300_two_row_chunks", 300, 256, 512),
    ("m16_remainder_split", 16, 256, 256 * 150),   # one full wave + 2 remainder tiles split 4 ways
    # small batches (M <= 16) take the panel-streaming kernel (dequant_gemv.cu): stream-K ranges
    # that start and end inside tiles, one- and two-block rows (M <= 8, 9..16)
    ("m9_two_row_blocks", 9, 320, 768),
    ("m1_stream_k_split", 1, 2048, 512),        # 64 panels < 148 CTAs: one panel per CTA
    ("m3_ranges_cut_tiles", 3, 640, 256 * 160),  # 1600 panels over 148 CTAs: ranges cut tiles
    ("m17_first_tcgen05_row", 17, 256, 512),
]


@pytest.mark.parametrize("case", GEMM_CASES, ids=[c[0] for c in GEMM_CASES])
def test_dequant_gemm_parity(orc, cuda, case):
    name, M, K, N = case
    seed = 4100 + M + K + N
    w = weights(seed, K, N)
    x = synth.fill(seed, 2, (M, K))
    panels, _, _ = quantized(w, cuda)
    ws = fq.make_gemm_workspace(M, K, N, cuda)
    y = fq.flexq_dequant_gemm(x.to(cuda), panels, N, workspace=ws)
    torch.cuda.synchronize()
    oc, om = orc.quantize(w.numpy(), 4, 64)
    check_gemm(y.cpu().numpy(), x.numpy(), oc, om, orc, name)
    assert int(ws[:(N // 256) * 4].count_nonzero()) == 0, "tile tickets must be left zeroed"
    # a second call reuses the (zeroed) workspace and reproduces the result bit for bit
    y2 = fq.flexq_dequant_gemm(x.to(cuda), panels, N, workspace=ws)
    assert torch.equal(y, y2)


def test_dequant_gemm_outliers_and_peaky_x(orc, cuda):
    M, K, N = 24, 256, 512
    w = weights(4201, K, N, outliers=True)
    x = synth.peaky(synth.fill(4201, 2, (M, K)), 16)
    panels, _, _ = quantized(w, cuda)
    y = fq.flexq_dequant_gemm(x.to(cuda), panels, N)
    oc, om = orc.quantize(w.numpy(), 4, 64)
    check_gemm(y.cpu().numpy(), x.numpy(), oc, om, orc, "outliers")


def test_dequant_gemm_extreme_weights(orc, cuda):
    """Constant groups, +-65504, subnormals (synth.extreme): w^ is O7's clamped fp16 value."""
    M, K, N = 8, 128, 256
    w = synth.extreme(4202, 3, K, N)
    x = (synth.fill(4202, 2, (M, K)).float() * 2.0 ** -12).half()    # keep y finite
    panels, _, _ = quantized(w, cuda)
    y = fq.flexq_dequant_gemm(x.to(cuda), panels, N)
    oc, om = orc.quantize(w.numpy(), 4, 64)
    check_gemm(y.cpu().numpy(), x.numpy(), oc, om, orc, "extreme")


def test_dequant_gemm_one_hot_rows_are_dequantize(cuda):
    """x = rows of the identity: y = the kernel's fp16 weight operand, which must be
    flexq_dequantize's (O7) value up to reading G2's double-rounding ties (<= 1 ulp, rare)."""
    K, N = 128, 512
    w = weights(4203, K, N)
    panels, codes, meta = quantized(w, cuda)
    x = torch.eye(K, dtype=torch.float16, device=cuda)
    y = fq.flexq_dequant_gemm(x, panels, N)
    d = fq.flexq_dequantize(codes, meta)
    ulps = (y.view(torch.int16).int() - d.view(torch.int16).int()).abs()
    assert int(ulps.max()) <= 1
    assert int((ulps > 0).sum()) <= K * N // 10000


@pytest.mark.parametrize("kind", ["normal", "extreme"])
def test_pack_weight_layout(cuda, kind):
    """flexq_pack_weight is a pure re-layout (plus the clamp-flag trailer): rebuild it in numpy from
    the documented layout, for ordinary weights (flag 0) and +-65504 groups (flag 1 where needed)."""
    K, N = 128, 512
    w = weights(4205, K, N) if kind == "normal" else synth.extreme(4205, 9, K, N)
    panels, codes, meta = quantized(w, cuda)
    P = panels.cpu().numpy()
    c = codes.cpu().numpy()
    full = np.zeros((K, N), np.uint8)
    full[:, 0::2] = c & 15
    full[:, 1::2] = c >> 4
    mt = meta.cpu().numpy().view(np.uint16)          # [K][N/64][2]
    KB = K // 64
    pos_of = [0, 4, 1, 5, 2, 6, 3, 7]                  # nibble position of k offset e in a word
    for t in range(N // 256):
        for kb in range(KB):
            pi = t * KB + kb
            blob = P[pi * 9216:(pi + 1) * 9216]
            # flag (after all panels): some code may reconstruct above 65504 (15 * scale + min > 65504)
            flag = P[(N // 256) * KB * 9216 + pi * 16:(N // 256) * KB * 9216 + (pi + 1) * 16]
            sc = mt[kb * 64:(kb + 1) * 64, t * 4:(t + 1) * 4, 0].view(np.float16).astype(np.float64)
            mn = mt[kb * 64:(kb + 1) * 64, t * 4:(t + 1) * 4, 1].view(np.float16).astype(np.float64)
            assert flag[:4].view(np.uint32)[0] == int((15 * sc + mn > 65504).any())
            assert not flag[4:].any()
            words = blob[:8192].view(np.uint32).reshape(2, 256, 4)
            for hk in range(2):
                for j in range(4):
                    k0 = kb * 64 + hk * 32 + 8 * j
                    ref = np.zeros(256, np.uint32)
                    for e in range(8):
                        ref |= full[k0 + e, t * 256:(t + 1) * 256].astype(np.uint32) << (4 * pos_of[e])
                    assert np.array_equal(words[hk, :, j], ref)
            mb = blob[8192:9216].view(np.uint16).reshape(4, 32, 2, 2)   # [g][kp][scale|min pair][k, k+1]
            for g in range(4):
                for kp in range(32):
                    k = kb * 64 + 2 * kp
                    assert mb[g, kp, 0, 0] == mt[k, t * 4 + g, 0] and mb[g, kp, 0, 1] == mt[k + 1, t * 4 + g, 0]
                    assert mb[g, kp, 1, 0] == mt[k, t * 4 + g, 1] and mb[g, kp, 1, 1] == mt[k + 1, t * 4 + g, 1]


def test_dequant_gemm_cuda_graph(orc, cuda):
    M, K, N = 40, 256, 512
    w = weights(4204, K, N)
    x = synth.fill(4204, 2, (M, K)).to(cuda)
    panels, _, _ = quantized(w, cuda)
    ws = fq.make_gemm_workspace(M, K, N, cuda)
    y = torch.empty(M, N, dtype=torch.float16, device=cuda)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fq.flexq_dequant_gemm(x, panels, N, out=y, workspace=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fq.flexq_dequant_gemm(x, panels, N, out=y, workspace=ws)
    y.zero_()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    oc, om = orc.quantize(w.numpy(), 4, 64)
    check_gemm(y.cpu().numpy(), x.cpu().numpy(), oc, om, orc, "graph")


@pytest.mark.parametrize("N", [49152, 12288])
def test_opt175b_weight_full_size_sampled(orc, cuda, N):
    """BASELINE configs[4] matrices at full size (w1 12288 x 49152, w_Q-class 12288 x 12288)
    with the bench's batch M = 144, the launch configuration bench.py times; the oracle
    recomputes sampled 64-column blocks from host-regenerated weights."""
    M, K = 144, 12288
    seed = synth.BASE_SEED + 4
    w = synth.fill(seed, 10 + N // 12288, (K, N), device=cuda)
    codes, meta = fq.flexq_quantize(w)
    del w
    panels = fq.flexq_pack_weight(codes, meta)
    del codes, meta
    x = synth.fill(seed, 20, (M, K))
    y = fq.flexq_dequant_gemm(x.to(cuda), panels, N).cpu().numpy()
    rng = np.random.default_rng(11)
    blocks = sorted({0, N // 64 - 1, *[int(b) for b in rng.integers(0, N // 64, size=4)]})
    for b in blocks:
        wb = synth.gather(seed, 10 + N // 12288, (K, N), [slice(None), slice(64 * b, 64 * b + 64)])
        oc, om = orc.quantize(wb.numpy(), 4, 64)
        check_gemm(y[:, 64 * b:64 * b + 64], x.numpy(), oc, om, orc, f"N={N} block {b}")


@pytest.mark.parametrize("M", [1, 16])
def test_small_batch_full_size_sampled(orc, cuda, M):
    """Batch-1 / batch-16 decode (the panel-streaming kernel) on the OPT-175B w1 matrix
    (12288 x 49152, BASELINE configs[4]); sampled 64-column blocks against the oracle."""
    K, N = 12288, 49152
    seed = synth.BASE_SEED + 5
    w = synth.fill(seed, 12, (K, N), device=cuda)
    codes, meta = fq.flexq_quantize(w)
    del w
    panels = fq.flexq_pack_weight(codes, meta)
    del codes, meta
    x = synth.fill(seed, 21 + M, (M, K))
    y = fq.flexq_dequant_gemm(x.to(cuda), panels, N).cpu().numpy()
    rng = np.random.default_rng(12 + M)
    blocks = sorted({0, N // 64 - 1, *[int(b) for b in rng.integers(0, N // 64, size=3)]})
    for b in blocks:
        wb = synth.gather(seed, 12, (K, N), [slice(None), slice(64 * b, 64 * b + 64)])
        oc, om = orc.quantize(wb.numpy(), 4, 64)
        check_gemm(y[:, 64 * b:64 * b + 64], x.numpy(), oc, om, orc, f"M={M} block {b}")


def test_pair_kernel_matches_single(cuda, tmp_path):
    """The opt-in CTA-pair kernel (cta_group::2, FLEXQ_GEMM_PAIR=1) splits the MMA's M across two
    SMs without changing any sum: its output must equal the single-CTA kernel's bit for bit, at
    a full tile wave, a split-k remainder and two row chunks."""
    import os
    import subprocess
    import sys
    script = tmp_path / "pair_case.py"
    script.write_text(
        "import sys, torch\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        "from paper_2303_06865_b200 import flexq as fq, synth\n"
        "dev = torch.device('cuda:0')\n"
        "out = []\n"
        "for M, K, N in ((144, 640, 512), (16, 256, 256 * 150), (300, 256, 1024)):\n"
        "    w = synth.fill(4300 + N, 1, (K, N), device=dev)\n"
        "    c, m = fq.flexq_quantize(w)\n"
        "    p = fq.flexq_pack_weight(c, m)\n"
        "    y = fq.flexq_dequant_gemm(synth.fill(4300 + N, 2, (M, K), device=dev), p, N)\n"
        "    out.append(y.cpu())\n"
        "torch.save(out, sys.argv[1])\n")
    res = {}
    for mode in ("0", "1"):
        f = tmp_path / f"y{mode}.pt"
        env = dict(os.environ, FLEXQ_GEMM_PAIR=mode)
        r = subprocess.run([sys.executable, str(script), str(f)], env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        res[mode] = torch.load(f)
    for a, b in zip(res["0"], res["1"]):
        assert torch.equal(a, b)

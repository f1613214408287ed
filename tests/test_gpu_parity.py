"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Codes, metadata and dequantized values must be
byte-identical (north_star, SURVEY 8(c) "GPU parity contract"); attention
outputs must satisfy |gpu - oracle_f64| <= max(2e-3, 1e-2 |oracle|)
elementwise (reading Q).  Oracle inputs are regenerated on the host by
synth (never copied back from the device)."""
import numpy as np
import pytest
import torch

from paper_2303_06865_b200 import flexq as fq
from paper_2303_06865_b200 import synth

pytestmark = pytest.mark.gpu

ATOL, RTOL = 2e-3, 1e-2


def assert_attn_close(got: np.ndarray, ref: np.ndarray, what=""):
    got = got.astype(np.float64)
    err = np.abs(got - ref)
    bad = err > np.maximum(ATOL, RTOL * np.abs(ref))
    assert not bad.any(), (f"{what}: {bad.sum()} of {bad.size} elements out of tolerance; "
                           f"max abs err {err.max():.3e}")


# ---------------------------------------------------------------- quantize
QUANT_CASES = [
    ("default", lambda: synth.fill(31, 1, (37, 192))),
    ("ragged_rows_wide", lambda: synth.fill(31, 2, (5, 4096))),
    ("outliers", lambda: synth.with_outliers(synth.fill(31, 3, (300, 128)))),
    ("ties", lambda: synth.ties(31, 4, (257, 64))),
    ("extreme", lambda: synth.extreme(31, 5, 512, 128)),
    ("one_group", lambda: synth.fill(31, 6, (1, 64))),
]


@pytest.mark.parametrize("name,make", QUANT_CASES, ids=[c[0] for c in QUANT_CASES])
def test_quantize_bit_exact(orc, cuda, name, make):
    x = make()
    codes, meta = fq.flexq_quantize(x.to(cuda))
    torch.cuda.synchronize()
    oc, om = orc.quantize(x.numpy(), 4, 64)
    assert np.array_equal(codes.cpu().numpy(), orc.pack4(oc)), name
    assert np.array_equal(meta.cpu().numpy().view(np.uint16), om), name


def test_quantize_large_grid_stride(orc, cuda):
    """More groups than the grid's threads: exercises the grid-stride loop."""
    rows, cols = 4099, 1024
    x = synth.fill(32, 1, (rows, cols))
    codes, meta = fq.flexq_quantize(x.to(cuda))
    oc, om = orc.quantize(x.numpy(), 4, 64)
    assert np.array_equal(codes.cpu().numpy(), orc.pack4(oc))
    assert np.array_equal(meta.cpu().numpy().view(np.uint16), om)


@pytest.mark.parametrize("name,make", QUANT_CASES, ids=[c[0] for c in QUANT_CASES])
def test_dequantize_bit_exact(orc, cuda, name, make):
    x = make()
    oc, om = orc.quantize(x.numpy(), 4, 64)
    codes = torch.from_numpy(orc.pack4(oc)).to(cuda)
    meta = torch.from_numpy(om.view(np.float16)).to(cuda)
    out = fq.flexq_dequantize(codes, meta)
    ref = orc.dequantize(oc, om, 4, 64)
    assert np.array_equal(out.cpu().numpy().view(np.uint16), ref.view(np.uint16)), name


# ---------------------------------------------------------------- append
@pytest.mark.parametrize("D", [64, 128])
def test_append_kv_bit_exact(orc, cuda, D):
    B, H, s, n = 3, 5, 70, 6
    k = synth.fill(33, synth.tensor_id(0, synth.K_PROMPT), (B, H, s, D))
    v = synth.with_outliers(synth.fill(33, synth.tensor_id(0, synth.V_PROMPT), (B, H, s, D)))
    cache = fq.KVCache(B, H, D, s, n, device=cuda)
    fq.flexq_append_kv(k.to(cuda), v.to(cuda), cache, pos=0)
    okc, ovc = orc.empty_cache(B, H, s + n, D), orc.empty_cache(B, H, s + n, D)
    orc.append_kv(k.numpy(), v.numpy(), okc, ovc, 0)
    for step in range(1, 4):
        kn = synth.fill(33, synth.tensor_id(0, synth.K_NEW, step), (B, H, 1, D))
        vn = synth.fill(33, synth.tensor_id(0, synth.V_NEW, step), (B, H, 1, D))
        fq.flexq_append_kv(kn.to(cuda), vn.to(cuda), cache, pos=s + step - 1)
        orc.append_kv(kn.numpy(), vn.numpy(), okc, ovc, s + step - 1)
    torch.cuda.synchronize()
    T = s + n
    assert cache.t_stride % 32 == 0 and cache.t_stride >= T
    assert np.array_equal(cache.k_codes()[:, :, :T].cpu().numpy(), orc.pack4(okc[0]))
    assert np.array_equal(cache.v_codes()[:, :, :T].cpu().numpy(), orc.pack4(ovc[0]))
    assert np.array_equal(cache.k_meta()[:, :, :T].cpu().numpy().view(np.uint16), okc[1])
    assert np.array_equal(cache.v_meta()[:, :, :T].cpu().numpy().view(np.uint16), ovc[1])
    # untouched positions (incl. the stride padding) stay zero
    assert int(cache.k_codes()[:, :, s + 3:].sum()) == 0 and int(cache.v_meta()[:, :, s + 3:].abs().sum()) == 0


# ---------------------------------------------------------------- attention
def build_case(orc, cuda, B, H, D, s, n, n_steps, seed, outliers=False, qfactor=1, layout="dense"):
    """Prompt fill + n_steps single-token appends on both sides; returns the
    GPU cache (in `layout`), the oracle caches, q (fp16) and cur_len = s + n_steps."""
    k = synth.fill(seed, synth.tensor_id(0, synth.K_PROMPT), (B, H, s, D))
    v = synth.fill(seed, synth.tensor_id(0, synth.V_PROMPT), (B, H, s, D))
    if outliers:
        k, v = synth.with_outliers(k), synth.with_outliers(v)
    cache = fq.KVCache(B, H, D, s, n, device=cuda, layout=layout)
    okc, ovc = orc.empty_cache(B, H, s + n, D), orc.empty_cache(B, H, s + n, D)
    if s > 0:
        fq.flexq_append_kv(k.to(cuda), v.to(cuda), cache, pos=0)
        orc.append_kv(k.numpy(), v.numpy(), okc, ovc, 0)
    for step in range(1, n_steps + 1):
        kn = synth.fill(seed, synth.tensor_id(0, synth.K_NEW, step), (B, H, 1, D))
        vn = synth.fill(seed, synth.tensor_id(0, synth.V_NEW, step), (B, H, 1, D))
        fq.flexq_append_kv(kn.to(cuda), vn.to(cuda), cache, pos=s + step - 1)
        orc.append_kv(kn.numpy(), vn.numpy(), okc, ovc, s + step - 1)
    q = synth.peaky(synth.fill(seed, synth.tensor_id(0, synth.Q, n_steps), (B, H, D)), qfactor)
    return cache, okc, ovc, q, s + n_steps


ATTN_CASES = [
    # name, B, H, D, s, n, steps, outliers, qfactor
    ("tiny_config", 4, 12, 64, 512, 1, 1, False, 1),          # BASELINE configs[0], in full
    ("tiny_outliers_peaky16", 4, 12, 64, 512, 1, 1, True, 16),
    ("d128_ragged_split", 2, 3, 128, 100, 8, 3, False, 1),     # cur_len 103: ragged tail, split-K
    ("d128_peaky64_outliers", 2, 4, 128, 300, 4, 2, True, 64),
    ("d128_one_token", 3, 2, 128, 0, 4, 1, False, 1),           # cur_len = 1
    ("d128_stage_multiple", 1, 2, 128, 64, 32, 0, False, 16),   # cur_len 64 = 2 full stages
    ("d64_long", 1, 3, 64, 1024, 32, 2, True, 16),
    ("d128_many_heads_nosplit", 24, 128, 128, 40, 2, 1, False, 1),  # B*H = 3072: no split
    ("d128_full_capacity_odd", 3, 5, 128, 100, 3, 3, False, 4),      # cur_len = T_cap = 103 (stride 104)
    ("d64_full_capacity_odd", 2, 3, 64, 60, 1, 1, True, 16),         # cur_len = T_cap = 61 (stride 64)
    ("d128_opt30b_len", 2, 4, 128, 1024, 32, 31, False, 1),          # cur_len 1055: the 1088-token buffer
    ("d128_beyond_buffer", 1, 3, 128, 1500, 8, 2, True, 16),         # cur_len 1502 > 1088: context split
    ("d64_beyond_buffer", 1, 2, 64, 2000, 1, 1, False, 4),           # cur_len 2001
    # about one head per warp (first ticket = warp index, residency capped at ceil(heads / SMs)):
    ("d128_one_per_warp", 3, 100, 128, 300, 8, 3, False, 1),         # 300 heads: 2 CTAs per SM
    ("d128_one_chunk_heads", 8, 40, 128, 30, 4, 2, True, 16),        # cur_len 32: one stage per head
    ("d128_576", 4, 80, 128, 574, 2, 2, False, 4),                   # cur_len 576: the score buffer, full
    ("d64_one_per_warp", 10, 32, 64, 200, 4, 2, True, 16),
]


def test_attention_q_wide_dynamic_range(orc, cuda):
    """q with one channel per head at 2^12 x the rest (the pass-1 fixed-point q of
    each lane is scaled to its own max, so the small channels are represented to
    2^-24 of that max): still within reading Q's tolerance."""
    B, H, D, s, n = 2, 4, 128, 200, 4
    cache, okc, ovc, q, cur = build_case(orc, cuda, B, H, D, s, n, 2, seed=44)
    q = q.clone()
    q[..., 5] = torch.where(q[..., 5] >= 0, 1.0, -1.0).to(torch.float16) * 4096   # |q| ~ 2^12 vs ~1
    q = (q.float() * 0.001).to(torch.float16)                                      # keep the softmax O(1)
    out = fq.flexq_decode_attention(q.to(cuda), cache, cur)
    ref = orc.attention_f64(q.numpy(), okc, ovc, cur)
    assert_attn_close(out.cpu().numpy(), ref, "wide-range q")


@pytest.mark.parametrize("case", ATTN_CASES, ids=[c[0] for c in ATTN_CASES])
def test_attention_parity(orc, cuda, case):
    name, B, H, D, s, n, steps, outl, qf = case
    cache, okc, ovc, q, cur = build_case(orc, cuda, B, H, D, s, n, steps, seed=40, outliers=outl, qfactor=qf)
    ws = fq.make_workspace(cache)
    out = fq.flexq_decode_attention(q.to(cuda), cache, cur, workspace=ws)
    torch.cuda.synchronize()
    ref = orc.attention_f64(q.numpy(), okc, ovc, cur)
    assert_attn_close(out.cpu().numpy(), ref, name)
    ctrl = 256 + 4 * B * H           # ticket counter + per-(b, h) split tickets (include/flexq.h)
    assert int(ws[:ctrl].sum()) == 0, "workspace control words must be restored to zero"
    # a second call on the same workspace gives the identical result
    out2 = fq.flexq_decode_attention(q.to(cuda), cache, cur, workspace=ws)
    assert torch.equal(out, out2)


def test_attention_every_cur_len_small(orc, cuda):
    """cur_len sweeps 1..70 over one cache (stage boundaries at 32, 64)."""
    B, H, D, s, n = 1, 2, 128, 64, 6
    cache, okc, ovc, q, _ = build_case(orc, cuda, B, H, D, s, n, 6, seed=41)
    ws = fq.make_workspace(cache)
    for cur in list(range(1, 71)):
        out = fq.flexq_decode_attention(q.to(cuda), cache, cur, workspace=ws)
        ref = orc.attention_f64(q.numpy(), okc, ovc, cur)
        assert_attn_close(out.cpu().numpy(), ref, f"cur_len={cur}")


def test_attention_cuda_graph_replay(orc, cuda):
    """append + attention captured in a CUDA graph give the same bytes on replay."""
    B, H, D, s, n = 2, 8, 128, 200, 4
    cache, okc, ovc, q, cur = build_case(orc, cuda, B, H, D, s, n, 0, seed=42)
    kn = synth.fill(42, 99, (B, H, 1, D)).to(cuda)
    vn = synth.fill(42, 98, (B, H, 1, D)).to(cuda)
    qd = q.to(cuda)
    ws = fq.make_workspace(cache)
    out = torch.empty_like(qd)
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fq.flexq_append_kv(kn, vn, cache, pos=s)
        fq.flexq_decode_attention(qd, cache, s + 1, out=out, workspace=ws)
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    eager = out.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fq.flexq_append_kv(kn, vn, cache, pos=s)
        fq.flexq_decode_attention(qd, cache, s + 1, out=out, workspace=ws)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)
    orc.append_kv(kn.cpu().numpy(), vn.cpu().numpy(), okc, ovc, s)
    assert_attn_close(out.cpu().numpy(), orc.attention_f64(q.numpy(), okc, ovc, s + 1), "graph")


# ---------------------------------------------------------------- full size, sampled
@pytest.mark.parametrize("cfg", [("opt175b", 144, 96, 128, 512, 32, 3), ("opt30b", 144, 56, 128, 1024, 32, 2)],
                         ids=["opt175b", "opt30b"])
def test_full_size_sampled(orc, cuda, cfg):
    """BASELINE configs[3] (OPT-175B: B=144, H=96, s=512) and configs[2] (OPT-30B: B=144, H=56,
    s=1024) at full size on one GPU, step 31 (cur_len 543 / 1055), the launch configuration
    bench.py times; the oracle recomputes 12 sampled (b, h) heads from host-regenerated inputs."""
    _, B, H, D, s, n, cfg_index = cfg
    seed = synth.BASE_SEED + cfg_index
    cache = fq.KVCache(B, H, D, s, n, device=cuda)
    k = synth.fill(seed, synth.tensor_id(0, synth.K_PROMPT), (B, H, s, D), device=cuda)
    v = synth.fill(seed, synth.tensor_id(0, synth.V_PROMPT), (B, H, s, D), device=cuda)
    fq.flexq_append_kv(k, v, cache, pos=0)
    del k, v
    steps = 31
    for step in range(1, steps + 1):
        kn = synth.fill(seed, synth.tensor_id(0, synth.K_NEW, step), (B, H, 1, D), device=cuda)
        vn = synth.fill(seed, synth.tensor_id(0, synth.V_NEW, step), (B, H, 1, D), device=cuda)
        fq.flexq_append_kv(kn, vn, cache, pos=s + step - 1)
    q = synth.fill(seed, synth.tensor_id(0, synth.Q, steps), (B, H, D), device=cuda)
    out = fq.flexq_decode_attention(q, cache, s + steps).cpu().numpy()
    kc_all = cache.k_codes().cpu().numpy()
    vm_all = cache.v_meta().cpu().numpy().view(np.uint16)
    rng = np.random.default_rng(7)
    samples = [(0, 0), (B - 1, H - 1)] + [(int(rng.integers(B)), int(rng.integers(H))) for _ in range(10)]
    for b, h in samples:
        kp = synth.gather(seed, synth.tensor_id(0, synth.K_PROMPT), (B, H, s, D), [b, h, slice(None), slice(None)])
        vp = synth.gather(seed, synth.tensor_id(0, synth.V_PROMPT), (B, H, s, D), [b, h, slice(None), slice(None)])
        okc, ovc = orc.empty_cache(1, 1, s + n, D), orc.empty_cache(1, 1, s + n, D)
        orc.append_kv(kp.numpy(), vp.numpy(), okc, ovc, 0)
        for step in range(1, steps + 1):
            kn = synth.gather(seed, synth.tensor_id(0, synth.K_NEW, step), (B, H, 1, D), [b, h, slice(None), slice(None)])
            vn = synth.gather(seed, synth.tensor_id(0, synth.V_NEW, step), (B, H, 1, D), [b, h, slice(None), slice(None)])
            orc.append_kv(kn.numpy(), vn.numpy(), okc, ovc, s + step - 1)
        # codes of this head are bit-exact ...
        assert np.array_equal(kc_all[b, h, :s + steps], orc.pack4(okc[0][0, 0, :s + steps]))
        assert np.array_equal(vm_all[b, h, :s + steps], ovc[1][0, 0, :s + steps])
        # ... and the attention output is in tolerance
        qh = synth.gather(seed, synth.tensor_id(0, synth.Q, steps), (B, H, D), [b, h, slice(None)])
        ref = orc.attention_f64(qh.numpy(), okc, ovc, s + steps)
        assert_attn_close(out[b:b + 1, h:h + 1], ref, f"(b={b}, h={h})")


def test_full_size_fused_sampled(orc, cuda):
    """The launch bench.py times: OPT-175B (B=144, H=96, D=128, s=512, n=32) at full size, every
    decode step i = 1..31 through flexq_append_decode_attention (cur_len 513..543, one fused launch
    per step).  For 12 sampled heads the oracle replays prompt fill + the 31 appends and
    recomputes the outputs of steps 1 (cur_len 513) and 31 (cur_len 543); K codes, K meta, V codes
    and V meta of those heads must be byte-identical over all 543 tokens."""
    B, H, D, s, n = 144, 96, 128, 512, 32
    seed = synth.BASE_SEED + 3
    cache = fq.KVCache(B, H, D, s, n, device=cuda)
    k = synth.fill(seed, synth.tensor_id(0, synth.K_PROMPT), (B, H, s, D), device=cuda)
    v = synth.fill(seed, synth.tensor_id(0, synth.V_PROMPT), (B, H, s, D), device=cuda)
    fq.flexq_append_kv(k, v, cache, pos=0)
    del k, v
    ws = fq.make_workspace(cache)
    outs = {}
    steps = n - 1
    for step in range(1, steps + 1):
        kn = synth.fill(seed, synth.tensor_id(0, synth.K_NEW, step), (B, H, D), device=cuda)
        vn = synth.fill(seed, synth.tensor_id(0, synth.V_NEW, step), (B, H, D), device=cuda)
        q = synth.fill(seed, synth.tensor_id(0, synth.Q, step), (B, H, D), device=cuda)
        o = fq.flexq_append_decode_attention(q, kn, vn, cache, s + step, workspace=ws)
        if step in (1, steps):
            outs[step] = o.cpu().numpy()
    T = s + steps
    kc_all, vc_all = cache.k_codes().cpu().numpy(), cache.v_codes().cpu().numpy()
    km_all = cache.k_meta().cpu().numpy().view(np.uint16)
    vm_all = cache.v_meta().cpu().numpy().view(np.uint16)
    assert int(ws[:256 + 4 * B * H].sum()) == 0
    rng = np.random.default_rng(11)
    samples = [(0, 0), (B - 1, H - 1)] + [(int(rng.integers(B)), int(rng.integers(H))) for _ in range(10)]
    sl = lambda b, h, *rest: [b, h, *rest]   # noqa: E731
    for b, h in samples:
        okc, ovc = orc.empty_cache(1, 1, s + n, D), orc.empty_cache(1, 1, s + n, D)
        kp = synth.gather(seed, synth.tensor_id(0, synth.K_PROMPT), (B, H, s, D), sl(b, h, slice(None), slice(None)))
        vp = synth.gather(seed, synth.tensor_id(0, synth.V_PROMPT), (B, H, s, D), sl(b, h, slice(None), slice(None)))
        orc.append_kv(kp.numpy(), vp.numpy(), okc, ovc, 0)
        for step in range(1, steps + 1):
            kn = synth.gather(seed, synth.tensor_id(0, synth.K_NEW, step), (B, H, D), sl(b, h, slice(None)))
            vn = synth.gather(seed, synth.tensor_id(0, synth.V_NEW, step), (B, H, D), sl(b, h, slice(None)))
            orc.append_kv(kn.numpy().reshape(1, 1, 1, D), vn.numpy().reshape(1, 1, 1, D), okc, ovc, s + step - 1)
            if step in outs:
                qh = synth.gather(seed, synth.tensor_id(0, synth.Q, step), (B, H, D), sl(b, h, slice(None)))
                ref = orc.attention_f64(qh.numpy().reshape(1, 1, D), okc, ovc, s + step)
                assert_attn_close(outs[step][b:b + 1, h:h + 1], ref, f"step {step} (b={b}, h={h})")
        assert np.array_equal(kc_all[b, h, :T], orc.pack4(okc[0][0, 0, :T])), (b, h)
        assert np.array_equal(vc_all[b, h, :T], orc.pack4(ovc[0][0, 0, :T])), (b, h)
        assert np.array_equal(km_all[b, h, :T], okc[1][0, 0, :T]), (b, h)
        assert np.array_equal(vm_all[b, h, :T], ovc[1][0, 0, :T]), (b, h)


# ---------------------------------------------------------------- NEXT-1: Top-K sparse attention
def test_topk_full_size_sampled(orc, cuda):
    """The Top-K launch bench.py times (topk_sparse): OPT-175B at full size (B=144, H=96, D=128),
    token-major cache, cur_len 543, keep = ceil(0.1 * 543) = 55.  For 12 sampled heads
    the oracle quantizes the head's 543 K / V rows and recomputes scores, kept set and output: the
    head's cache bytes are identical, the GPU's kept set is a valid top-55 set of the oracle's
    scores (it may differ from the oracle's only at near-ties), and the output is within reading Q
    of the oracle evaluated on the GPU's set."""
    B, H, D, T = 144, 96, 128, 543
    seed = synth.BASE_SEED + 5
    cache = fq.KVCache(B, H, D, T, 1, device=cuda, layout="token_major")
    k = synth.fill(seed, synth.tensor_id(0, synth.K_PROMPT), (B, H, T, D), device=cuda)
    v = synth.fill(seed, synth.tensor_id(0, synth.V_PROMPT), (B, H, T, D), device=cuda)
    fq.flexq_append_kv(k, v, cache, pos=0)
    del k, v
    q = synth.fill(seed, synth.tensor_id(0, synth.Q, 1), (B, H, D), device=cuda)
    keep = fq.topk_keep(T)
    assert keep == 55
    sel = torch.full((B, H, keep), -1, dtype=torch.int32, device=cuda)
    out = fq.flexq_decode_attention_topk(q, cache, T, keep, sel=sel).cpu().numpy()
    sel = sel.cpu().numpy()
    kc_all, vc_all = cache.k_codes().cpu().numpy(), cache.v_codes().cpu().numpy()
    rng = np.random.default_rng(12)
    samples = [(0, 0), (B - 1, H - 1)] + [(int(rng.integers(B)), int(rng.integers(H))) for _ in range(10)]
    sl = lambda b, h, *rest: [b, h, *rest]   # noqa: E731
    mismatched = 0
    for b, h in samples:
        okc, ovc = orc.empty_cache(1, 1, T + 1, D), orc.empty_cache(1, 1, T + 1, D)
        kp = synth.gather(seed, synth.tensor_id(0, synth.K_PROMPT), (B, H, T, D), sl(b, h, slice(None), slice(None)))
        vp = synth.gather(seed, synth.tensor_id(0, synth.V_PROMPT), (B, H, T, D), sl(b, h, slice(None), slice(None)))
        orc.append_kv(kp.numpy(), vp.numpy(), okc, ovc, 0)
        assert np.array_equal(kc_all[b, h, :T], orc.pack4(okc[0][0, 0, :T])), (b, h)
        assert np.array_equal(vc_all[b, h, :T], orc.pack4(ovc[0][0, 0, :T])), (b, h)
        qh = synth.gather(seed, synth.tensor_id(0, synth.Q, 1), (B, H, D), sl(b, h, slice(None))).numpy()
        _, omask, scores = orc.attention_topk_f64(qh.reshape(1, 1, D), okc, ovc, T, keep)
        idx = sel[b, h]
        assert np.all(np.diff(idx) > 0) and idx.min() >= 0 and idx.max() < T, (b, h)
        mask = np.zeros((1, 1, T), np.uint8)
        mask[0, 0, idx] = 1
        sc = scores[0, 0]
        eps = 1e-4 * max(1.0, np.abs(sc).max())
        assert sc[idx].min() >= sc[mask[0, 0] == 0].max() - eps, (b, h)
        mismatched += int((mask != omask).sum())
        ref, _, _ = orc.attention_topk_f64(qh.reshape(1, 1, D), okc, ovc, T, keep, sel=mask)
        assert_attn_close(out[b:b + 1, h:h + 1], ref, f"(b={b}, h={h})")
    assert mismatched <= 2 * len(samples)   # differences only at near-ties


@pytest.mark.parametrize("layout", ["dense", "token_major"])
@pytest.mark.parametrize("D", [64, 128])
def test_topk_exact_ties_bit_exact(orc, cuda, D, layout):
    """Selection is index work: on exactly tied scores (K rows drawn from 3
    distinct rows, so identical codes + meta give identical scores on both sides) the GPU's
    kept set must equal the oracle's -- score descending, then lowest token index -- with zero
    mismatches; the output is then within reading Q of the oracle on that set."""
    for T in (150, 300):   # ~50 copies of each score (ranked directly), ~100 (refined digit by digit)
        _topk_ties_case(orc, cuda, D, layout, T)


def _topk_ties_case(orc, cuda, D, layout, T):
    B, H = 2, 3
    base = synth.fill(59, 1, (B, H, 3, D))
    cls = torch.stack([torch.arange(T) % 3, 2 - torch.arange(T) % 3, (torch.arange(T) // 7) % 3])
    k = torch.stack([torch.stack([base[b, h][cls[h]] for h in range(H)]) for b in range(B)])
    v = synth.fill(59, 2, (B, H, T, D))
    cache = fq.KVCache(B, H, D, T, 1, device=cuda, layout=layout)
    fq.flexq_append_kv(k.to(cuda), v.to(cuda), cache, pos=0)
    okc, ovc = orc.empty_cache(B, H, T, D), orc.empty_cache(B, H, T, D)
    orc.append_kv(k.numpy(), v.numpy(), okc, ovc, 0)
    q = synth.fill(59, 3, (B, H, D))
    for keep in (1, 15, 50, 73, T - 1):
        sel = torch.full((B, H, keep), -1, dtype=torch.int32, device=cuda)
        out = fq.flexq_decode_attention_topk(q.to(cuda), cache, T, keep, sel=sel)
        torch.cuda.synchronize()
        ref, omask, _ = orc.attention_topk_f64(q.numpy(), okc, ovc, T, keep)
        mask = np.zeros((B, H, T), np.uint8)
        for b in range(B):
            for h in range(H):
                mask[b, h, sel.cpu().numpy()[b, h]] = 1
        assert int((mask != omask).sum()) == 0, f"keep={keep}: kept sets differ"
        assert_attn_close(out.cpu().numpy(), ref, f"ties keep={keep}")


@pytest.mark.parametrize("layout", ["dense", "token_major"])
def test_topk_repeated_tail(orc, cuda, layout):
    """The bench's decode step rewrites one k_new row per layer, so its caches end in 31 copies of
    one K row: a group of equal scores that often lands in the select's threshold bin.  The kept
    set must be a valid top-`keep` set (ties inside the group broken by lowest index) and the output
    within reading Q on it."""
    B, H, D, s, rep = 3, 16, 128, 512, 31
    T = s + rep
    k = synth.fill(64, 1, (B, H, T, D))
    v = synth.fill(64, 2, (B, H, T, D))
    k[:, :, s:] = k[:, :, s:s + 1]
    v[:, :, s:] = v[:, :, s:s + 1]
    cache = fq.KVCache(B, H, D, T, 1, device=cuda, layout=layout)
    fq.flexq_append_kv(k.to(cuda), v.to(cuda), cache, pos=0)
    okc, ovc = orc.empty_cache(B, H, T, D), orc.empty_cache(B, H, T, D)
    orc.append_kv(k.numpy(), v.numpy(), okc, ovc, 0)
    for qs in (0, 1, 2):
        q = synth.fill(65 + qs, 3, (B, H, D))
        keep = fq.topk_keep(T)
        sel = torch.full((B, H, keep), -1, dtype=torch.int32, device=cuda)
        out = fq.flexq_decode_attention_topk(q.to(cuda), cache, T, keep, sel=sel)
        torch.cuda.synchronize()
        sel_np = sel.cpu().numpy()
        _, omask, scores = orc.attention_topk_f64(q.numpy(), okc, ovc, T, keep)
        mask = np.zeros((B, H, T), np.uint8)
        for b in range(B):
            for h in range(H):
                idx = sel_np[b, h]
                assert np.all(np.diff(idx) > 0) and idx.min() >= 0 and idx.max() < T, (b, h)
                mask[b, h, idx] = 1
                sc = scores[b, h]
                eps = 1e-4 * max(1.0, np.abs(sc).max())
                assert sc[idx].min() >= sc[mask[b, h] == 0].max() - eps, (b, h)
                grp = mask[b, h, s:]            # equal scores: the kept part of the group is a prefix
                assert np.all(np.diff(grp.astype(np.int8)) <= 0), (b, h, grp)
        assert (mask != omask).sum() <= 2 * B * H
        ref, _, _ = orc.attention_topk_f64(q.numpy(), okc, ovc, T, keep, sel=mask)
        assert_attn_close(out.cpu().numpy(), ref, f"repeated tail q{qs}")


TOPK_CASES = [
    # name, B, H, D, s, n, steps, outliers, qfactor, keep fraction
    ("d128_10pct", 3, 8, 128, 300, 4, 3, False, 4, 0.1),
    ("d64_10pct_outliers", 2, 6, 64, 512, 1, 1, True, 16, 0.1),
    ("d128_keep_all", 1, 4, 128, 70, 2, 1, False, 1, 1.0),
    ("d128_keep_one", 2, 3, 128, 90, 2, 2, False, 8, 0.0),
    ("d128_opt175b_len", 2, 16, 128, 512, 32, 31, False, 1, 0.1),
    ("d128_long_1152_buffer", 1, 4, 128, 1100, 2, 1, True, 4, 0.1),   # cur_len 1101: 36 keys per lane
    ("d64_peaky_half", 2, 5, 64, 400, 2, 1, False, 64, 0.5),
    ("d128_flat_q_crowded_bin", 2, 4, 128, 300, 2, 1, False, 1 / 256, 0.1),   # one 1/16 bin: radix refine
]


@pytest.mark.parametrize("layout", ["dense", "token_major"])
@pytest.mark.parametrize("case", TOPK_CASES, ids=[c[0] for c in TOPK_CASES])
def test_topk_attention_parity(orc, cuda, case, layout):
    """The GPU's kept set must be a valid top-`keep` set of the oracle's scores
    (several sets are correct when scores tie within rounding), and the output
    must match the oracle evaluated on that set within reading Q's tolerance."""
    name, B, H, D, s, n, steps, outl, qf, frac = case
    cache, okc, ovc, q, cur = build_case(orc, cuda, B, H, D, s, n, steps, seed=60, outliers=outl, qfactor=qf,
                                         layout=layout)
    if layout == "token_major":   # the cache bytes of the token-major layout: V rows like K rows
        T = cur
        assert np.array_equal(cache.v_codes()[:, :, :T].cpu().numpy(), orc.pack4(ovc[0][:, :, :T]))
        assert np.array_equal(cache.v_meta()[:, :, :T].cpu().numpy().view(np.uint16), ovc[1][:, :, :T])
        assert np.array_equal(cache.k_codes()[:, :, :T].cpu().numpy(), orc.pack4(okc[0][:, :, :T]))
    keep = fq.topk_keep(cur, frac) if frac > 0 else 1
    sel = torch.full((B, H, keep), -1, dtype=torch.int32, device=cuda)
    out = fq.flexq_decode_attention_topk(q.to(cuda), cache, cur, keep, sel=sel)
    torch.cuda.synchronize()
    sel = sel.cpu().numpy()
    _, omask, scores = orc.attention_topk_f64(q.numpy(), okc, ovc, cur, keep)
    mask = np.zeros((B, H, cur), np.uint8)
    for b in range(B):
        for h in range(H):
            idx = sel[b, h]
            assert np.all(np.diff(idx) > 0) and idx.min() >= 0 and idx.max() < cur, (b, h)
            mask[b, h, idx] = 1
            sc = scores[b, h]
            eps = 1e-4 * max(1.0, np.abs(sc).max())
            if keep < cur:
                assert sc[idx].min() >= sc[mask[b, h] == 0].max() - eps, (b, h)
    assert (mask != omask).sum() <= 2 * B * H          # differences only at near-ties
    ref, _, _ = orc.attention_topk_f64(q.numpy(), okc, ovc, cur, keep, sel=mask)
    assert_attn_close(out.cpu().numpy(), ref, name)


@pytest.mark.parametrize("layout", ["dense", "token_major"])
def test_topk_workspace_reuse(orc, cuda, layout):
    """Every call leaves the Top-K workspace's scheduler counters zero (include/flexq.h): calls on
    one workspace, with different q and keep, give the bytes a fresh zeroed workspace gives, and the
    workspace's control area is zero again afterwards."""
    B, H, D, s, n, steps = 3, 40, 128, 300, 4, 3
    cache, okc, ovc, q, cur = build_case(orc, cuda, B, H, D, s, n, steps, seed=61, layout=layout)
    ws = fq.make_topk_workspace(cache)
    gen = torch.Generator().manual_seed(7)
    for rep, frac in enumerate([0.1, 0.3, 0.1, 0.05]):
        qq = (q + 0.25 * rep * torch.randn(q.shape, generator=gen).to(q.dtype)).to(cuda)
        keep = fq.topk_keep(cur, frac)
        got = fq.flexq_decode_attention_topk(qq, cache, cur, keep, workspace=ws)
        ref = fq.flexq_decode_attention_topk(qq, cache, cur, keep)
        torch.cuda.synchronize()
        assert torch.equal(got.view(torch.int16), ref.view(torch.int16)), rep
        assert int(ws[:2048].count_nonzero()) == 0, rep   # the select kernel's tickets


# ---------------------------------------------------------------- fused append + attention (NEXT-3)
FUSED_CASES = [
    # name, B, H, D, s, n, steps (fused decode steps after the prompt), outliers, qfactor
    ("d128_split_ragged", 2, 3, 128, 100, 8, 3, False, 1),        # split-K, token in a ragged last stage
    ("d128_first_token_of_chunk", 2, 4, 128, 95, 4, 2, True, 16),  # cur_len 96, 97: chunk boundary
    ("d128_one_token", 3, 2, 128, 0, 2, 1, False, 1),             # cur_len = 1: the new token alone
    ("d128_no_split", 24, 128, 128, 40, 2, 1, False, 4),          # B*H = 3072 units
    ("d128_fused_one_per_warp", 3, 100, 128, 290, 4, 3, True, 4),
    ("d64_fused_chunk_edge", 10, 32, 64, 127, 2, 2, False, 1),    # cur_len 128, 129
    ("d128_opt175b_shard_b18", 18, 96, 128, 541, 2, 2, False, 1),  # the N = 8 shard, cur_len 542, 543
    ("d64_tiny", 4, 12, 64, 512, 1, 1, False, 1),                 # configs[0] with the fused step
    ("d64_full_capacity", 2, 3, 64, 60, 3, 3, True, 16),          # last step: cur_len = T_cap
]


@pytest.mark.parametrize("case", FUSED_CASES, ids=[c[0] for c in FUSED_CASES])
def test_append_attention_fused(orc, cuda, case):
    """flexq_append_decode_attention == flexq_append_kv(pos = cur_len - 1) then attention:
    the cache bytes bit-exact against the oracle's append, the output within reading Q."""
    name, B, H, D, s, n, steps, outl, qf = case
    cache, okc, ovc, _, cur = build_case(orc, cuda, B, H, D, s, n, 0, seed=45, outliers=outl)
    ws = fq.make_workspace(cache)
    for step in range(1, steps + 1):
        kn = synth.fill(45, synth.tensor_id(1, synth.K_NEW, step), (B, H, D))
        vn = synth.fill(45, synth.tensor_id(1, synth.V_NEW, step), (B, H, D))
        if outl:
            kn, vn = synth.with_outliers(kn), synth.with_outliers(vn)
        q = synth.peaky(synth.fill(45, synth.tensor_id(1, synth.Q, step), (B, H, D)), qf)
        cur = s + step
        out = fq.flexq_append_decode_attention(q.to(cuda), kn.to(cuda), vn.to(cuda), cache, cur, workspace=ws)
        orc.append_kv(kn.numpy()[:, :, None], vn.numpy()[:, :, None], okc, ovc, cur - 1)
        torch.cuda.synchronize()
        assert_attn_close(out.cpu().numpy(), orc.attention_f64(q.numpy(), okc, ovc, cur), f"{name} step {step}")
    T = s + n
    assert np.array_equal(cache.k_codes()[:, :, :T].cpu().numpy(), orc.pack4(okc[0]))
    assert np.array_equal(cache.v_codes()[:, :, :T].cpu().numpy(), orc.pack4(ovc[0]))
    assert np.array_equal(cache.k_meta()[:, :, :T].cpu().numpy().view(np.uint16), okc[1])
    assert np.array_equal(cache.v_meta()[:, :, :T].cpu().numpy().view(np.uint16), ovc[1])
    assert int(ws[:256 + 4 * B * H].sum()) == 0


def test_append_attention_fused_matches_two_launches(cuda):
    """The fused step and the two-launch step (append, then attention) leave
    byte-identical caches; outputs agree to reading Q (same kernel, same data)."""
    B, H, D, s, n = 16, 12, 128, 300, 4
    k = synth.fill(46, synth.tensor_id(0, synth.K_PROMPT), (B, H, s, D)).to(cuda)
    v = synth.fill(46, synth.tensor_id(0, synth.V_PROMPT), (B, H, s, D)).to(cuda)
    c1, c2 = fq.KVCache(B, H, D, s, n, device=cuda), fq.KVCache(B, H, D, s, n, device=cuda)
    fq.flexq_append_kv(k, v, c1, pos=0)
    fq.flexq_append_kv(k, v, c2, pos=0)
    for step in range(1, n + 1):
        kn = synth.fill(46, synth.tensor_id(1, synth.K_NEW, step), (B, H, D)).to(cuda)
        vn = synth.fill(46, synth.tensor_id(1, synth.V_NEW, step), (B, H, D)).to(cuda)
        q = synth.fill(46, synth.tensor_id(1, synth.Q, step), (B, H, D)).to(cuda)
        o1 = fq.flexq_append_decode_attention(q, kn, vn, c1, s + step)
        fq.flexq_append_kv(kn.view(B, H, 1, D), vn.view(B, H, 1, D), c2, pos=s + step - 1)
        o2 = fq.flexq_decode_attention(q, c2, s + step)
        assert torch.equal(o1, o2), f"step {step}"
    assert torch.equal(c1.k, c2.k) and torch.equal(c1.v, c2.v)


@pytest.mark.parametrize("D", [64, 128])
def test_attention_extreme_cache(orc, cuda, D):
    """Pathological KV groups (synth.extreme: constant groups -> scale 0, +-65504 mixes, subnormal
    groups, any finite pattern), scaled by powers of two so the softmax stays finite: the
    fixed-point q and weight paths must still land within reading Q of the f64 oracle."""
    B, H, s, n = 2, 3, 150, 4
    rows = B * H * s
    k = (synth.extreme(4401, 1, rows, D).float() * 2.0 ** -10).half().view(B, H, s, D)
    v = (synth.extreme(4401, 2, rows, D).float() * 2.0 ** -4).half().view(B, H, s, D)
    cache = fq.KVCache(B, H, D, s, n, device=cuda)
    okc, ovc = orc.empty_cache(B, H, s + n, D), orc.empty_cache(B, H, s + n, D)
    fq.flexq_append_kv(k.to(cuda), v.to(cuda), cache, pos=0)
    orc.append_kv(k.numpy(), v.numpy(), okc, ovc, 0)
    for qf in (1, 16):
        q = synth.peaky(synth.fill(4401, 3 + qf, (B, H, D)), qf)
        out = fq.flexq_decode_attention(q.to(cuda), cache, s)
        ref = orc.attention_f64(q.numpy(), okc, ovc, s)
        assert_attn_close(out.cpu().numpy(), ref, f"extreme D={D} q x{qf}")
    # and one fused append + attention step with a pathological new token
    kn = (synth.extreme(4401, 10, B * H, D).float() * 2.0 ** -10).half().view(B, H, D)
    vn = (synth.extreme(4401, 20, B * H, D).float() * 2.0 ** -4).half().view(B, H, D)
    q = synth.fill(4401, 30, (B, H, D))
    out = fq.flexq_append_decode_attention(q.to(cuda), kn.to(cuda), vn.to(cuda), cache, s + 1)
    orc.append_kv(kn.view(B, H, 1, D).numpy(), vn.view(B, H, 1, D).numpy(), okc, ovc, s)
    ref = orc.attention_f64(q.numpy(), okc, ovc, s + 1)
    assert_attn_close(out.cpu().numpy(), ref, f"extreme fused D={D}")
    assert np.array_equal(cache.k_codes()[:, :, :s + 1].cpu().numpy(), orc.pack4(okc[0][:, :, :s + 1]))


# ---------------------------------------------------------------- the token-major (4, 64) layout
@pytest.mark.parametrize("D", [64, 128])
def test_token_major_layout(orc, cuda, D):
    """FLEXQ_KV_TOKEN_MAJOR at (4, 64): V rows are laid out like K rows (byte-exact against the
    oracle's append), dense decode attention over it (the CUDA-core kernel) and the one-call
    decode step are within reading Q, and export / import move the same plain bytes as for the
    dense layout."""
    B, H, s, n = 2, 5, 200, 4
    cache, okc, ovc, q, cur = build_case(orc, cuda, B, H, D, s, n, 2, seed=61, outliers=True, qfactor=4,
                                         layout="token_major")
    T = cur
    assert np.array_equal(cache.k_codes()[:, :, :T].cpu().numpy(), orc.pack4(okc[0][:, :, :T]))
    assert np.array_equal(cache.v_codes()[:, :, :T].cpu().numpy(), orc.pack4(ovc[0][:, :, :T]))
    assert np.array_equal(cache.v_meta()[:, :, :T].cpu().numpy().view(np.uint16), ovc[1][:, :, :T])
    # raw V bytes equal raw K-layout bytes of the same rows: token-major like K
    vchunk = cache.v[..., :16 * D].reshape(B, H, -1, D // 2)      # each chunk's [codes 32 x D/2]
    assert torch.equal(vchunk[:, :, :T].cpu(), cache.v_codes()[:, :, :T].cpu())
    out = fq.flexq_decode_attention(q.to(cuda), cache, cur)
    torch.cuda.synchronize()
    assert_attn_close(out.cpu().numpy(), orc.attention_f64(q.numpy(), okc, ovc, cur), "token-major attention")
    kn = synth.fill(61, 90, (B, H, 1, D))
    vn = synth.fill(61, 91, (B, H, 1, D))
    out2 = fq.flexq_append_decode_attention(q.to(cuda), kn[:, :, 0].to(cuda), vn[:, :, 0].to(cuda), cache, cur + 1)
    orc.append_kv(kn.numpy(), vn.numpy(), okc, ovc, cur)
    torch.cuda.synchronize()
    assert_attn_close(out2.cpu().numpy(), orc.attention_f64(q.numpy(), okc, ovc, cur + 1), "token-major fused step")
    assert np.array_equal(cache.v_codes()[:, :, :cur + 1].cpu().numpy(), orc.pack4(ovc[0][:, :, :cur + 1]))
    # the same plain bytes leave both layouts
    dense, _, _, _, _ = build_case(orc, cuda, B, H, D, s, n, 2, seed=61, outliers=True, qfactor=4)
    fq.flexq_append_kv(kn.to(cuda), vn.to(cuda), dense, pos=cur)
    for a, b in zip(fq.flexq_kv_export(cache, 0, cur + 1), fq.flexq_kv_export(dense, 0, cur + 1)):
        assert torch.equal(a, b)


@pytest.mark.parametrize("layout", ["dense", "token_major"])
def test_topk_short_contexts(orc, cuda, layout):
    """Contexts of one 64-token stage or less (a select unit of a single stage: the next unit's q
    is issued before this unit has read its own) and the stage boundary, through the full path
    against the oracle on the GPU's kept set."""
    B, H, D = 3, 7, 128
    for cur in (1, 2, 31, 64, 65, 129):
        cache, okc, ovc, q, cur_len = build_case(orc, cuda, B, H, D, cur, 1, 0, seed=62, layout=layout)
        keep = fq.topk_keep(cur_len)
        sel = torch.full((B, H, keep), -1, dtype=torch.int32, device=cuda)
        out = fq.flexq_decode_attention_topk(q.to(cuda), cache, cur_len, keep, sel=sel)
        torch.cuda.synchronize()
        mask = np.zeros((B, H, cur_len), np.uint8)
        for b in range(B):
            for h in range(H):
                mask[b, h, sel.cpu().numpy()[b, h]] = 1
        assert int(mask.sum()) == B * H * keep
        ref, _, _ = orc.attention_topk_f64(q.numpy(), okc, ovc, cur_len, keep, sel=mask)
        assert_attn_close(out.cpu().numpy(), ref, f"short context {cur_len}")


def test_schedule_variants_within_tolerance(orc, cuda, tmp_path):
    """The tuning schedules (static stream-K, whole-head tickets, ticket pieces, the static prefix
    + ticket hybrid, one ticket counter, the 3-stage ring, no residency cap, no programmatic dependent launch) all compute the same attention: each,
    forced through its environment switch in a fresh process, is within reading Q of the oracle
    on a launch whose heads get split (B*H = 40 over ~2,400 warps) and on one whose heads do not."""
    import os
    import subprocess
    import sys
    script = tmp_path / "sched_case.py"
    script.write_text(
        "import sys, numpy as np, torch\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        "from paper_2303_06865_b200 import flexq as fq, synth\n"
        "dev = torch.device('cuda:0')\n"
        "outs = []\n"
        "for (B, H, s) in ((2, 20, 600), (16, 160, 300)):\n"
        "    c = fq.KVCache(B, H, 128, s, 2, device=dev)\n"
        "    k = synth.fill(63, 1, (B, H, s, 128), device=dev)\n"
        "    v = synth.fill(63, 2, (B, H, s, 128), device=dev)\n"
        "    fq.flexq_append_kv(k, v, c, pos=0)\n"
        "    q = synth.fill(63, 3, (B, H, 128), device=dev)\n"
        "    kn = synth.fill(63, 4, (B, H, 128), device=dev)\n"
        "    vn = synth.fill(63, 5, (B, H, 128), device=dev)\n"
        "    outs.append(fq.flexq_append_decode_attention(q, kn, vn, c, s + 1).cpu().numpy())\n"
        "np.savez(sys.argv[1], *outs)\n")
    envs = {"default": {}, "static": {"FLEXQ_ATTN_SPLIT": "100000,0,0"}, "tickets": {"FLEXQ_ATTN_SPLIT": "0,0,0"},
            "ticket_pieces": {"FLEXQ_ATTN_SPLIT": "0,100,3"}, "hybrid": {"FLEXQ_ATTN_SPLIT": "100000,0,0", "FLEXQ_ATTN_HYBRID": "70,4"},
            "one_counter": {"FLEXQ_ATTN_CTRS": "1", "FLEXQ_ATTN_SPLIT": "0,0,0"}, "ring3": {"FLEXQ_ATTN_RING": "3"},
            "cap_off": {"FLEXQ_ATTN_CAP": "0"}, "pdl_off": {"FLEXQ_PDL": "0"}}
    refs = []
    for (B, H, s) in ((2, 20, 600), (16, 160, 300)):
        k = synth.fill(63, 1, (B, H, s, 128))
        v = synth.fill(63, 2, (B, H, s, 128))
        kn = synth.fill(63, 4, (B, H, 1, 128))
        vn = synth.fill(63, 5, (B, H, 1, 128))
        okc, ovc = orc.empty_cache(B, H, s + 2, 128), orc.empty_cache(B, H, s + 2, 128)
        orc.append_kv(k.numpy(), v.numpy(), okc, ovc, 0)
        orc.append_kv(kn.numpy(), vn.numpy(), okc, ovc, s)
        refs.append(orc.attention_f64(synth.fill(63, 3, (B, H, 128)).numpy(), okc, ovc, s + 1))
    for name, extra in envs.items():
        f = tmp_path / f"{name}.npz"
        r = subprocess.run([sys.executable, str(script), str(f)], env=dict(os.environ, **extra), capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        got = np.load(f)
        for i, ref in enumerate(refs):
            assert_attn_close(got[f"arr_{i}"], ref, f"schedule {name}, case {i}")

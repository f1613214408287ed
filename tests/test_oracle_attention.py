"""Pins for the oracle's decode attention (O8) and KV append (A4), CPU only.

Pinned against: softmax weights summing to 1 (north_star), closed forms
(cur_len = 1, identical keys -> mean of V, dominant key),
invariants (V scaling, token permutation), an independent numpy/scipy
evaluation on inputs whose dequantized values are exact, the f32 twin, and
the append layout (quantize rows of the new tokens).
"""
import numpy as np
import pytest
import scipy.special

from paper_2303_06865_b200 import synth


def make_cache(orc, B, H, D, T, seed, group=64, outliers=False, T_cap=None):
    T_cap = T_cap or T
    k = synth.fill(seed, synth.tensor_id(0, synth.K_PROMPT), (B, H, T, D))
    v = synth.fill(seed, synth.tensor_id(0, synth.V_PROMPT), (B, H, T, D))
    if outliers:
        k, v = synth.with_outliers(k), synth.with_outliers(v)
    kc, vc = orc.empty_cache(B, H, T_cap, D, group), orc.empty_cache(B, H, T_cap, D, group)
    orc.append_kv(k.numpy(), v.numpy(), kc, vc, pos=0, group=group)
    q = synth.fill(seed, synth.tensor_id(0, synth.Q), (B, H, D))
    return q.numpy(), kc, vc, k.numpy(), v.numpy()


def deq_f32(orc, cache):
    """K^ as fp32 fmaf(c, scale, min) -- via the codes/meta and numpy float64 fma
    (exact product+sum of fp32 values in float64, then one rounding to fp32)."""
    codes, meta = cache
    g = codes.shape[-1] // meta.shape[-2]
    s = meta[..., 0].view(np.float16).astype(np.float64)
    m = meta[..., 1].view(np.float16).astype(np.float64)
    s = np.repeat(s, g, axis=-1)
    m = np.repeat(m, g, axis=-1)
    return (codes.astype(np.float64) * s + m).astype(np.float32)   # exact in f64, one RN to f32


def test_append_kv_layout(orc):
    """A4: append writes quantize(rows) at [pos, pos+n_new) and touches nothing else."""
    B, H, D, T_cap = 2, 3, 128, 20
    kn = synth.fill(21, 1, (B, H, 5, D)).numpy()
    vn = synth.fill(21, 2, (B, H, 5, D)).numpy()
    kc, vc = orc.empty_cache(B, H, T_cap, D), orc.empty_cache(B, H, T_cap, D)
    kc[0][:] = 7
    orc.append_kv(kn, vn, kc, vc, pos=9)
    c, m = orc.quantize(kn.reshape(-1, D), 4, 64)
    assert np.array_equal(kc[0][:, :, 9:14].reshape(-1, D), c)
    assert np.array_equal(kc[1][:, :, 9:14].reshape(-1, 2, 2), m)
    assert np.all(kc[0][:, :, :9] == 7) and np.all(kc[0][:, :, 14:] == 7)
    c, m = orc.quantize(vn.reshape(-1, D), 4, 64)
    assert np.array_equal(vc[0][:, :, 9:14].reshape(-1, D), c)
    with pytest.raises(ValueError):
        orc.append_kv(kn, vn, kc, vc, pos=16)          # pos + n_new > T_cap


@pytest.mark.parametrize("D,T", [(64, 37), (128, 130)])
def test_softmax_rows_sum_to_one(orc, D, T):
    q, kc, vc, _, _ = make_cache(orc, 2, 3, D, T, seed=22)
    _, p = orc.attention_f64(q, kc, vc, T, want_probs=True)
    assert np.all(p >= 0)
    assert np.abs(p.sum(axis=-1) - 1).max() <= 2 * T * 2.0 ** -52 * 4


def test_matches_independent_numpy_scipy(orc):
    """Independent evaluation: numpy dequant (exact in f64) + scipy softmax."""
    B, H, D, T = 2, 2, 128, 50
    q, kc, vc, _, _ = make_cache(orc, B, H, D, T, seed=23, outliers=True)
    K = deq_f32(orc, kc).astype(np.float64)
    V = deq_f32(orc, vc).astype(np.float64)
    qf = q.astype(np.float64)
    s = np.einsum("bhd,bhtd->bht", qf, K) / np.sqrt(D)
    ref = np.einsum("bht,bhtd->bhd", scipy.special.softmax(s, axis=-1), V)
    got = orc.attention_f64(q, kc, vc, T)
    assert np.abs(got - ref).max() <= 1e-10 * max(1.0, np.abs(V).max())


def test_cur_len_one_returns_v0(orc):
    q, kc, vc, _, _ = make_cache(orc, 1, 2, 64, 8, seed=24)
    got = orc.attention_f64(q, kc, vc, 1)
    V = deq_f32(orc, vc).astype(np.float64)
    assert np.array_equal(got, V[:, :, 0, :])


def test_identical_keys_give_mean_of_v(orc):
    """all keys identical -> uniform weights -> o = mean of V^ rows."""
    B, H, D, T = 1, 2, 128, 33
    k1 = synth.fill(25, 1, (B, H, 1, D)).numpy()
    k = np.repeat(k1, T, axis=2)
    v = synth.fill(25, 2, (B, H, T, D)).numpy()
    kc, vc = orc.empty_cache(B, H, T, D), orc.empty_cache(B, H, T, D)
    orc.append_kv(k, v, kc, vc, 0)
    q = synth.fill(25, 3, (B, H, D)).numpy()
    got, p = orc.attention_f64(q, kc, vc, T, want_probs=True)
    assert np.abs(p - 1.0 / T).max() < 1e-15
    V = deq_f32(orc, vc).astype(np.float64)
    assert np.abs(got - V.mean(axis=2)).max() < 1e-12


def test_dominant_key(orc):
    """q parallel to k_0 with a large norm -> o ~= v^_0."""
    B, H, D, T = 1, 1, 64, 16
    k = synth.fill(26, 1, (B, H, T, D)).numpy() * np.float16(0.01)
    k[0, 0, 0] = np.float16(1.0)
    k[0, 0, 0, ::2] = np.float16(-1.0)
    v = synth.fill(26, 2, (B, H, T, D)).numpy()
    kc, vc = orc.empty_cache(B, H, T, D), orc.empty_cache(B, H, T, D)
    orc.append_kv(k, v, kc, vc, 0)
    q = (k[:, :, 0, :].astype(np.float32) * 8).astype(np.float16)
    got = orc.attention_f64(q, kc, vc, T)
    V = deq_f32(orc, vc).astype(np.float64)
    assert np.abs(got[0, 0] - V[0, 0, 0]).max() < 1e-6


def test_v_scaling_and_permutation_invariance(orc):
    B, H, D, T = 1, 2, 128, 40
    q, kc, vc, _, _ = make_cache(orc, B, H, D, T, seed=27)
    o = orc.attention_f64(q, kc, vc, T)
    # scaling V's (scale, min) by 2 (exact in fp16) doubles the output exactly
    vm2 = (vc[1].view(np.float16) * np.float16(2)).view(np.uint16)
    o2 = orc.attention_f64(q, kc, (vc[0], vm2), T)
    assert np.array_equal(o2, 2 * o)
    # jointly permuting token rows of K and V leaves the output unchanged
    perm = np.random.default_rng(0).permutation(T)
    kp = (np.ascontiguousarray(kc[0][:, :, perm]), np.ascontiguousarray(kc[1][:, :, perm]))
    vp = (np.ascontiguousarray(vc[0][:, :, perm]), np.ascontiguousarray(vc[1][:, :, perm]))
    op = orc.attention_f64(q, kp, vp, T)
    assert np.abs(op - o).max() < 1e-12 * max(1, np.abs(o).max())


@pytest.mark.parametrize("factor,outliers", [(1, False), (16, False), (64, True)])
def test_f32_twin_agrees_with_f64(orc, factor, outliers):
    """SURVEY O8 pin (2): f32 evaluation of the same definition within 1e-4*max|V^|."""
    B, H, D, T = 2, 4, 128, 300
    q, kc, vc, _, _ = make_cache(orc, B, H, D, T, seed=28, outliers=outliers)
    q = (q.astype(np.float32) * factor).astype(np.float16)
    o64 = orc.attention_f64(q, kc, vc, T)
    o32 = orc.attention_f32(q, kc, vc, T)
    vmax = np.abs(deq_f32(orc, vc)).max()
    assert np.abs(o64 - o32).max() <= 1e-4 * max(1.0, vmax)


def test_cur_len_prefix_only(orc):
    """Tokens at positions >= cur_len never influence the output."""
    B, H, D, T = 1, 2, 64, 30
    q, kc, vc, _, _ = make_cache(orc, B, H, D, T, seed=29)
    o = orc.attention_f64(q, kc, vc, 20)
    kc[0][:, :, 20:] = 15
    vc[0][:, :, 20:] = 15
    assert np.array_equal(orc.attention_f64(q, kc, vc, 20), o)


# ---------------------------------------------------------------- NEXT-1: Top-K sparse attention
def test_topk_keep_all_equals_dense(orc):
    """keep fraction 1.0 -> identical to dense attention."""
    q, kc, vc, _, _ = make_cache(orc, 2, 3, 128, 77, seed=51)
    dense = orc.attention_f64(q, kc, vc, 77)
    sparse, mask, _ = orc.attention_topk_f64(q, kc, vc, 77, keep=77)
    assert mask.all()
    assert np.abs(sparse - dense).max() < 1e-12


def test_topk_selection_is_top_scores(orc):
    """The kept set is exactly the `keep` largest scores (independent numpy argsort)."""
    q, kc, vc, _, _ = make_cache(orc, 2, 2, 64, 130, seed=52)
    keep = 13                                         # ceil(0.1 * 130), "top 10%"
    _, mask, scores = orc.attention_topk_f64(q, kc, vc, 130, keep=keep)
    K = deq_f32(orc, kc).astype(np.float64)
    s_ref = np.einsum("bhd,bhtd->bht", q.astype(np.float64), K) / np.sqrt(64)
    assert np.abs(scores - s_ref).max() < 1e-9
    for b in range(2):
        for h in range(2):
            order = np.lexsort((np.arange(130), -scores[b, h]))   # score desc, index asc
            want = np.zeros(130, np.uint8)
            want[order[:keep]] = 1
            assert np.array_equal(mask[b, h], want)
            assert mask[b, h].sum() == keep


def tied_topk_case(orc, B=1, H=2, D=64, T=40, seed=57):
    """K rows drawn from 3 distinct rows (token t gets row t % 3, reversed in head 1), so the
    scores take 3 values with exact ties (identical codes and meta give bit-identical sums)."""
    base = synth.fill(seed, 1, (B, H, 3, D)).numpy()
    k = np.empty((B, H, T, D), np.float16)
    for h in range(H):
        cls = np.arange(T) % 3 if h == 0 else (2 - np.arange(T) % 3)
        k[:, h] = base[:, h][:, cls]
    v = synth.fill(seed, 2, (B, H, T, D)).numpy()
    kc, vc = orc.empty_cache(B, H, T, D), orc.empty_cache(B, H, T, D)
    orc.append_kv(k, v, kc, vc, 0)
    q = synth.fill(seed, 3, (B, H, D)).numpy()
    return q, kc, vc, base


def test_topk_exact_ties_keep_lowest_index(orc):
    """Selection is index work: on exactly tied scores the kept set is
    the definition's -- score descending, then token index ascending (flexq.h).  The class
    order comes from an independent numpy evaluation of the 3 distinct rows; the expected
    set is then built by counting, not from the oracle's own ranking."""
    B, H, D, T = 1, 2, 64, 40
    q, kc, vc, _ = tied_topk_case(orc, B, H, D, T)
    K = deq_f32(orc, kc).astype(np.float64)
    for keep in (1, 5, 14, 20, 27, 39):
        _, mask, scores = orc.attention_topk_f64(q, kc, vc, T, keep=keep)
        for h in range(H):
            cls_of = np.arange(T) % 3 if h == 0 else (2 - np.arange(T) % 3)
            s_cls = np.array([q[0, h].astype(np.float64) @ K[0, h, list(cls_of).index(c)] for c in range(3)])
            assert len(set(s_cls.tolist())) == 3                          # three distinct values
            for c in range(3):                                            # ties are exact
                assert len(set(scores[0, h, cls_of == c].tolist())) == 1
            want = np.zeros(T, np.uint8)
            left = keep
            for c in np.argsort(-s_cls):                                   # best class first
                idx = np.flatnonzero(cls_of == c)                          # ascending token index
                take = idx[:left]
                want[take] = 1
                left -= len(take)
            assert np.array_equal(mask[0, h], want), (keep, h)
    # all-identical keys: the kept set is the first `keep` tokens
    k = np.repeat(synth.fill(58, 1, (1, 1, 1, D)).numpy(), T, axis=2)
    kc1, vc1 = orc.empty_cache(1, 1, T, D), orc.empty_cache(1, 1, T, D)
    orc.append_kv(k, synth.fill(58, 2, (1, 1, T, D)).numpy(), kc1, vc1, 0)
    _, mask, _ = orc.attention_topk_f64(synth.fill(58, 3, (1, 1, D)).numpy(), kc1, vc1, T, keep=9)
    assert mask[0, 0].tolist() == [1] * 9 + [0] * (T - 9)


def test_topk_renormalised_and_dominant_key(orc):
    """one dominant key and keep = 1 -> output = that key's V^ row; weights
    renormalised over the kept set sum to 1 (checked through V = constant rows)."""
    B, H, D, T = 1, 1, 64, 20
    k = synth.fill(53, 1, (B, H, T, D)).numpy() * np.float16(0.01)
    k[0, 0, 5] = np.float16(1.0)
    v = synth.fill(53, 2, (B, H, T, D)).numpy()
    kc, vc = orc.empty_cache(B, H, T, D), orc.empty_cache(B, H, T, D)
    orc.append_kv(k, v, kc, vc, 0)
    q = (k[:, :, 5, :].astype(np.float32) * 4).astype(np.float16)
    out, mask, _ = orc.attention_topk_f64(q, kc, vc, T, keep=1)
    assert mask[0, 0].tolist() == [int(t == 5) for t in range(T)]
    V = deq_f32(orc, vc).astype(np.float64)
    assert np.abs(out[0, 0] - V[0, 0, 5]).max() < 1e-12
    # constant V rows -> output equals the constant for any kept set (weights sum to 1)
    vconst = np.full((B, H, T, D), np.float16(1.5))
    vc2 = orc.empty_cache(B, H, T, D)
    orc.append_kv(k, vconst, orc.empty_cache(B, H, T, D), vc2, 0)
    out2, _, _ = orc.attention_topk_f64(q, kc, vc2, T, keep=7)
    assert np.abs(out2 - 1.5).max() < 1e-12


def test_topk_converges_to_dense(orc):
    """SPEC 'Invariants': max deviation from dense is non-increasing as the kept
    fraction grows (0.1, 0.25, 0.5, 1.0) on a fixed instance."""
    q, kc, vc, _, _ = make_cache(orc, 1, 4, 128, 200, seed=54)
    q = (q.astype(np.float32) * 4).astype(np.float16)
    dense = orc.attention_f64(q, kc, vc, 200)
    devs = [np.abs(orc.attention_topk_f64(q, kc, vc, 200, keep=int(np.ceil(f * 200)))[0] - dense).max()
            for f in (0.1, 0.25, 0.5, 1.0)]
    assert all(devs[i + 1] <= devs[i] + 1e-15 for i in range(3)), devs
    assert devs[-1] < 1e-12


@pytest.mark.parametrize("bits,group", [(2, 32), (3, 128), (8, 64), (4, 32)])
def test_variant_cache_append_and_attention(orc, bits, group):
    """NEXT-3 variants (reading V): append writes quantize(rows, bits, group) per token row, and the
    attention dequantizes with the row's (D / group) meta pairs -- checked against an independent
    numpy dequant (exact in f64) + scipy softmax, and the closed form of cur_len = 1."""
    B, H, D, T = 2, 2, 128, 40
    k = synth.with_outliers(synth.fill(26, 1, (B, H, T, D))).numpy()
    v = synth.fill(26, 2, (B, H, T, D)).numpy()
    kc, vc = orc.empty_cache(B, H, T, D, group), orc.empty_cache(B, H, T, D, group)
    orc.append_kv(k, v, kc, vc, 0, bits, group)
    c, m = orc.quantize(k.reshape(-1, D), bits, group)
    assert np.array_equal(kc[0].reshape(-1, D), c) and np.array_equal(kc[1].reshape(-1, D // group, 2), m)
    assert kc[0].max() <= 2 ** bits - 1
    q = synth.fill(26, 3, (B, H, D)).numpy()
    K = deq_f32(orc, kc).astype(np.float64)
    V = deq_f32(orc, vc).astype(np.float64)
    s = np.einsum("bhd,bhtd->bht", q.astype(np.float64), K) / np.sqrt(D)
    ref = np.einsum("bht,bhtd->bhd", scipy.special.softmax(s, axis=-1), V)
    got = orc.attention_f64(q, kc, vc, T, group)
    assert np.abs(got - ref).max() <= 1e-10 * max(1.0, np.abs(V).max())
    assert np.array_equal(orc.attention_f64(q, kc, vc, 1, group), V[:, :, 0, :])

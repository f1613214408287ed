"""GPU parity of the KV-cache path for the NEXT-3 variants b in {2, 3, 4, 8} x g in {32, 64, 128}
(the b = 4, g = 64 cache is covered by test_gpu_parity.py).  Through the C ABI:
  - flexq_append_kv: cache codes (each token's row as a little-endian bit stream) and
    (scale, min) metadata byte-identical to the oracle's quantizer (reading B with 2^b - 1 levels);
  - flexq_decode_attention / flexq_append_decode_attention: |gpu - oracle_f64| <=
    max(2e-3, 1e-2 |oracle|) elementwise (reading Q), the oracle's caches built by the oracle.
Oracle inputs are regenerated on the host by synth, never copied back from the device."""
import numpy as np
import pytest
import torch

from paper_2303_06865_b200 import flexq as fq
from paper_2303_06865_b200 import synth

pytestmark = pytest.mark.gpu

ATOL, RTOL = 2e-3, 1e-2
VARIANTS = [(b, g) for b in (2, 3, 4, 8) for g in (32, 64, 128) if (b, g) != (4, 64)]


def close(got, ref, what):
    got = got.astype(np.float64)
    err = np.abs(got - ref)
    bad = err > np.maximum(ATOL, RTOL * np.abs(ref))
    assert not bad.any(), f"{what}: {bad.sum()} of {bad.size} out of tolerance; max abs err {err.max():.3e}"


def build(orc, cuda, B, H, D, s, n, steps, bits, group, seed, outliers=False, qfactor=1):
    k = synth.fill(seed, synth.tensor_id(0, synth.K_PROMPT), (B, H, s, D))
    v = synth.fill(seed, synth.tensor_id(0, synth.V_PROMPT), (B, H, s, D))
    if outliers:
        k, v = synth.with_outliers(k), synth.with_outliers(v)
    cache = fq.KVCache(B, H, D, s, n, device=cuda, bits=bits, group_size=group)
    okc, ovc = orc.empty_cache(B, H, s + n, D, group), orc.empty_cache(B, H, s + n, D, group)
    if s > 0:
        fq.flexq_append_kv(k.to(cuda), v.to(cuda), cache, pos=0)
        orc.append_kv(k.numpy(), v.numpy(), okc, ovc, 0, bits, group)
    for step in range(1, steps + 1):
        kn = synth.fill(seed, synth.tensor_id(0, synth.K_NEW, step), (B, H, 1, D))
        vn = synth.fill(seed, synth.tensor_id(0, synth.V_NEW, step), (B, H, 1, D))
        fq.flexq_append_kv(kn.to(cuda), vn.to(cuda), cache, pos=s + step - 1)
        orc.append_kv(kn.numpy(), vn.numpy(), okc, ovc, s + step - 1, bits, group)
    q = synth.peaky(synth.fill(seed, synth.tensor_id(0, synth.Q, steps), (B, H, D)), qfactor)
    return cache, okc, ovc, q, s + steps


def check_cache(orc, cache, okc, ovc, T, bits):
    assert np.array_equal(cache.k_codes()[:, :, :T].cpu().numpy(), orc.pack_bits(okc[0][:, :, :T], bits))
    assert np.array_equal(cache.v_codes()[:, :, :T].cpu().numpy(), orc.pack_bits(ovc[0][:, :, :T], bits))
    assert np.array_equal(cache.k_meta()[:, :, :T].cpu().numpy().view(np.uint16), okc[1][:, :, :T])
    assert np.array_equal(cache.v_meta()[:, :, :T].cpu().numpy().view(np.uint16), ovc[1][:, :, :T])


@pytest.mark.parametrize("bits,group", VARIANTS, ids=[f"b{b}g{g}" for b, g in VARIANTS])
@pytest.mark.parametrize("D", [64, 128])
def test_append_variant_bit_exact(orc, cuda, bits, group, D):
    if D % group:
        pytest.skip("head_dim % group != 0 (FLEXQ_ERR_UNSUPPORTED)")
    B, H, s, n = 3, 5, 70, 6
    cache, okc, ovc, _, cur = build(orc, cuda, B, H, D, s, n, 3, bits, group, seed=60, outliers=True)
    torch.cuda.synchronize()
    check_cache(orc, cache, okc, ovc, s + n, bits)
    # untouched positions (incl. the stride padding) stay zero
    assert int(cache.k_codes()[:, :, cur:].sum()) == 0 and int(cache.v_meta()[:, :, cur:].abs().sum()) == 0


ATTN = [
    # name, B, H, D, s, n, steps, outliers, qfactor
    ("d128_ragged_split", 2, 3, 128, 300, 4, 2, False, 1),      # cur 302: 3 tiles, split-K + combine
    ("d128_peaky_outliers", 2, 4, 128, 200, 4, 1, True, 32),
    ("d64_long_split", 1, 3, 64, 1000, 8, 2, True, 8),          # cur 1002: 8 tiles
    ("d128_one_token", 3, 2, 128, 0, 4, 1, False, 1),            # cur_len = 1
    ("d128_many_heads_nosplit", 16, 96, 128, 130, 2, 1, False, 4),   # B*H = 1536: one CTA per head
]


@pytest.mark.parametrize("bits,group", VARIANTS, ids=[f"b{b}g{g}" for b, g in VARIANTS])
@pytest.mark.parametrize("case", ATTN, ids=[c[0] for c in ATTN])
def test_attention_variant_parity(orc, cuda, bits, group, case):
    name, B, H, D, s, n, steps, outl, qf = case
    if D % group:
        pytest.skip("head_dim % group != 0")
    cache, okc, ovc, q, cur = build(orc, cuda, B, H, D, s, n, steps, bits, group, seed=61, outliers=outl,
                                    qfactor=qf)
    ws = fq.make_workspace(cache)
    out = fq.flexq_decode_attention(q.to(cuda), cache, cur, workspace=ws)
    torch.cuda.synchronize()
    ref = orc.attention_f64(q.numpy(), okc, ovc, cur, group)
    close(out.cpu().numpy(), ref, f"{name} b{bits} g{group}")
    out2 = fq.flexq_decode_attention(q.to(cuda), cache, cur, workspace=ws)
    assert torch.equal(out, out2)


@pytest.mark.parametrize("bits,group", [(3, 32), (2, 128), (8, 64)])
def test_attention_variant_every_cur_len(orc, cuda, bits, group):
    """cur_len 1..140 over one cache: chunk boundaries at 32, 64, 96, the tile boundary at 128."""
    B, H, D, s, n = 1, 2, 128, 130, 10
    cache, okc, ovc, q, _ = build(orc, cuda, B, H, D, s, n, 10, bits, group, seed=62)
    ws = fq.make_workspace(cache)
    for cur in range(1, 141):
        out = fq.flexq_decode_attention(q.to(cuda), cache, cur, workspace=ws)
        ref = orc.attention_f64(q.numpy(), okc, ovc, cur, group)
        close(out.cpu().numpy(), ref, f"cur_len={cur}")


@pytest.mark.parametrize("bits,group", [(2, 32), (3, 64), (8, 128), (4, 32)])
def test_append_decode_attention_variant(orc, cuda, bits, group):
    """The one-call decode step (append of token cur_len - 1, then attention) on a variant cache:
    the cache bytes equal flexq_append_kv's, the output is within reading Q."""
    B, H, D, s, n = 2, 6, 128, 150, 4
    cache, okc, ovc, q, cur = build(orc, cuda, B, H, D, s, n, 0, bits, group, seed=63)
    kn = synth.fill(63, synth.tensor_id(0, synth.K_NEW, 1), (B, H, 1, D))
    vn = synth.fill(63, synth.tensor_id(0, synth.V_NEW, 1), (B, H, 1, D))
    out = fq.flexq_append_decode_attention(q.to(cuda), kn[:, :, 0].to(cuda), vn[:, :, 0].to(cuda), cache, s + 1)
    torch.cuda.synchronize()
    orc.append_kv(kn.numpy(), vn.numpy(), okc, ovc, s, bits, group)
    check_cache(orc, cache, okc, ovc, s + n, bits)
    ref = orc.attention_f64(q.numpy(), okc, ovc, s + 1, group)
    close(out.cpu().numpy(), ref, f"fused b{bits} g{group}")


def test_variant_full_size_sampled(orc, cuda):
    """OPT-175B decode shape (batch 144, 96 heads, D 128, cur_len 543) at b = 3, g = 32, the launch
    configuration the bench's variant sweep times: the cache is built on the device from seeded
    inputs; the oracle rebuilds sampled heads from the same inputs regenerated on the host."""
    B, H, D, s, n, bits, group = 144, 96, 128, 543, 1, 3, 32
    seed = 64
    cache = fq.KVCache(B, H, D, s, n, device=cuda, bits=bits, group_size=group)
    k = synth.fill(seed, synth.tensor_id(0, synth.K_PROMPT), (B, H, s, D), device=cuda)
    v = synth.fill(seed, synth.tensor_id(0, synth.V_PROMPT), (B, H, s, D), device=cuda)
    fq.flexq_append_kv(k, v, cache, pos=0)
    del k, v
    q = synth.fill(seed, synth.tensor_id(0, synth.Q, 0), (B, H, D), device=cuda)
    out = fq.flexq_decode_attention(q, cache, s).cpu().numpy()
    q = q.cpu()
    for b, h in [(0, 0), (B - 1, H - 1), (17, 40), (71, 3)]:
        kp = synth.gather(seed, synth.tensor_id(0, synth.K_PROMPT), (B, H, s, D), [b, h, slice(None), slice(None)])
        vp = synth.gather(seed, synth.tensor_id(0, synth.V_PROMPT), (B, H, s, D), [b, h, slice(None), slice(None)])
        okc, ovc = orc.empty_cache(1, 1, s + n, D, group), orc.empty_cache(1, 1, s + n, D, group)
        orc.append_kv(kp.reshape(1, 1, s, D).numpy(), vp.reshape(1, 1, s, D).numpy(), okc, ovc, 0, bits, group)
        ref = orc.attention_f64(q[b:b + 1, h:h + 1].numpy(), okc, ovc, s, group)
        close(out[b:b + 1, h:h + 1], ref, f"head ({b}, {h})")


@pytest.mark.parametrize("bits,group", [(2, 32), (3, 128), (8, 32), (4, 128)])
def test_attention_variant_extreme_cache(orc, cuda, bits, group):
    """Pathological KV groups (synth.extreme, per group of the variant: constant groups -> scale 0,
    +-65504 mixes, subnormal groups, any finite pattern) scaled by powers of two so the softmax stays
    finite; cache bytes identical to the oracle's, output within reading Q, plus one pathological
    one-call decode step."""
    B, H, D, s, n = 2, 3, 128, 150, 4
    rows = B * H * s
    k = (synth.extreme(4402, 1, rows, D, group).float() * 2.0 ** -10).half().view(B, H, s, D)
    v = (synth.extreme(4402, 2, rows, D, group).float() * 2.0 ** -4).half().view(B, H, s, D)
    cache = fq.KVCache(B, H, D, s, n, device=cuda, bits=bits, group_size=group)
    okc, ovc = orc.empty_cache(B, H, s + n, D, group), orc.empty_cache(B, H, s + n, D, group)
    fq.flexq_append_kv(k.to(cuda), v.to(cuda), cache, pos=0)
    orc.append_kv(k.numpy(), v.numpy(), okc, ovc, 0, bits, group)
    for qf in (1, 16):
        q = synth.peaky(synth.fill(4402, 3 + qf, (B, H, D)), qf)
        out = fq.flexq_decode_attention(q.to(cuda), cache, s)
        close(out.cpu().numpy(), orc.attention_f64(q.numpy(), okc, ovc, s, group), f"extreme q x{qf}")
    kn = (synth.extreme(4402, 10, B * H, D, group).float() * 2.0 ** -10).half().view(B, H, D)
    vn = (synth.extreme(4402, 20, B * H, D, group).float() * 2.0 ** -4).half().view(B, H, D)
    q = synth.fill(4402, 30, (B, H, D))
    out = fq.flexq_append_decode_attention(q.to(cuda), kn.to(cuda), vn.to(cuda), cache, s + 1)
    orc.append_kv(kn.view(B, H, 1, D).numpy(), vn.view(B, H, 1, D).numpy(), okc, ovc, s, bits, group)
    close(out.cpu().numpy(), orc.attention_f64(q.numpy(), okc, ovc, s + 1, group), "extreme fused")
    check_cache(orc, cache, okc, ovc, s + 1, bits)


@pytest.mark.parametrize("bits,group", [(2, 32), (8, 128), (4, 128)])
def test_attention_variant_q_wide_dynamic_range(orc, cuda, bits, group):
    """q with one channel per head at 2^12 x the rest: the IDP.4A K pass holds q in 22-bit fixed point
    relative to the head's max |q| (the small channels to 2^-22 of that max); still within reading Q."""
    B, H, D, s, n = 2, 4, 128, 200, 4
    cache, okc, ovc, q, cur = build(orc, cuda, B, H, D, s, n, 2, bits, group, seed=65)
    q = q.clone()
    q[..., 5] = torch.where(q[..., 5] >= 0, 1.0, -1.0).to(torch.float16) * 4096
    q = (q.float() * 0.001).to(torch.float16)
    out = fq.flexq_decode_attention(q.to(cuda), cache, cur)
    close(out.cpu().numpy(), orc.attention_f64(q.numpy(), okc, ovc, cur, group), f"wide-range q b{bits} g{group}")

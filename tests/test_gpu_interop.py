"""flexq_kv_import / flexq_kv_export: the plain quantized KV layout (flexq_quantize's rows per
head) <-> the chunked cache, byte-exact against the oracle's append layout (A4) and
against flexq_append_kv's cache bytes; partial token ranges leave every other byte alone."""
import numpy as np
import pytest
import torch

from paper_2303_06865_b200 import flexq as fq
from paper_2303_06865_b200 import synth

pytestmark = pytest.mark.gpu

CASES = [(4, 64, 128), (4, 64, 64), (3, 32, 128), (2, 32, 64), (8, 128, 128)]


def oracle_plain(orc, k, v, T_cap, bits, group):
    """Oracle append (A4) of the full token range -> plain arrays (codes packed as S:520's bit stream)."""
    B, H, T, D = k.shape
    okc, ovc = orc.empty_cache(B, H, T_cap, D, group), orc.empty_cache(B, H, T_cap, D, group)
    orc.append_kv(k.numpy(), v.numpy(), okc, ovc, 0, bits, group)
    pack = (lambda c: orc.pack4(c)) if bits == 4 else (lambda c: orc.pack_bits(c, bits))
    return (pack(okc[0]), okc[1].view(np.float16), pack(ovc[0]), ovc[1].view(np.float16))


@pytest.mark.parametrize("bits,group,D", CASES, ids=[f"b{b}g{g}d{d}" for b, g, d in CASES])
def test_import_export_byte_exact(orc, cuda, bits, group, D):
    B, H, s, n = 2, 3, 70, 5
    T = s + n
    k = synth.with_outliers(synth.fill(81, 1, (B, H, T, D)))
    v = synth.fill(81, 2, (B, H, T, D))
    pk, pkm, pv, pvm = oracle_plain(orc, k, v, T, bits, group)
    # the reference cache: flexq_append_kv of the same fp16 rows
    ref = fq.KVCache(B, H, D, s, n, device=cuda, bits=bits, group_size=group)
    fq.flexq_append_kv(k.to(cuda), v.to(cuda), ref, pos=0)
    # import the oracle's plain arrays into an empty cache: identical bytes (padding stays zero)
    got = fq.KVCache(B, H, D, s, n, device=cuda, bits=bits, group_size=group)
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(cuda)  # noqa: E731
    fq.flexq_kv_import(got, t(pk), t(pkm), t(pv), t(pvm))
    torch.cuda.synchronize()
    assert torch.equal(got.k, ref.k) and torch.equal(got.v, ref.v)
    # export the appended cache: the oracle's plain arrays, byte for byte
    kc, km, vc, vm = fq.flexq_kv_export(ref)
    assert np.array_equal(kc.cpu().numpy(), pk) and np.array_equal(vc.cpu().numpy(), pv)
    assert np.array_equal(km.cpu().numpy().view(np.uint16), pkm.view(np.uint16))
    assert np.array_equal(vm.cpu().numpy().view(np.uint16), pvm.view(np.uint16))


@pytest.mark.parametrize("bits,group", [(4, 64), (3, 32)])
def test_partial_range_touches_nothing_else(orc, cuda, bits, group):
    """Import tokens [37, 74) (crossing a 32-token chunk and splitting 4-token quads) over a
    cache holding other data: those tokens equal a fresh append, every other byte is unchanged;
    export of the same range writes only those plain rows."""
    B, H, D, s, n = 2, 2, 128, 90, 6
    T = s + n
    t0, nt = 37, 37
    k1, v1 = synth.fill(82, 1, (B, H, T, D)), synth.fill(82, 2, (B, H, T, D))
    k2, v2 = synth.fill(82, 3, (B, H, T, D)), synth.fill(82, 4, (B, H, T, D))
    base = fq.KVCache(B, H, D, s, n, device=cuda, bits=bits, group_size=group)
    fq.flexq_append_kv(k1.to(cuda), v1.to(cuda), base, pos=0)
    before_k, before_v = base.k.clone(), base.v.clone()
    pk, pkm, pv, pvm = oracle_plain(orc, k2, v2, T, bits, group)
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(cuda)  # noqa: E731
    fq.flexq_kv_import(base, t(pk), t(pkm), t(pv), t(pvm), t0=t0, n_tok=nt)
    # expected: the cache of k1 with tokens [t0, t0 + nt) of k2 appended over it
    exp = fq.KVCache(B, H, D, s, n, device=cuda, bits=bits, group_size=group)
    fq.flexq_append_kv(k1.to(cuda), v1.to(cuda), exp, pos=0)
    fq.flexq_append_kv(k2[:, :, t0:t0 + nt].contiguous().to(cuda), v2[:, :, t0:t0 + nt].contiguous().to(cuda), exp,
                       pos=t0)
    torch.cuda.synchronize()
    assert torch.equal(base.k, exp.k) and torch.equal(base.v, exp.v)
    assert not torch.equal(base.k, before_k)
    kc, km, vc, vm = fq.flexq_kv_export(base, t0=t0, n_tok=nt, plain_tokens=T)
    assert int(kc[:, :, :t0].sum()) == 0 and int(kc[:, :, t0 + nt:].sum()) == 0
    assert np.array_equal(kc[:, :, t0:t0 + nt].cpu().numpy(), pk[:, :, t0:t0 + nt])
    assert np.array_equal(vc[:, :, t0:t0 + nt].cpu().numpy(), pv[:, :, t0:t0 + nt])
    assert np.array_equal(vm[:, :, t0:t0 + nt].cpu().numpy().view(np.uint16), pvm[:, :, t0:t0 + nt].view(np.uint16))


def test_imported_cache_attends_like_appended(orc, cuda):
    """A cache filled by import from flexq_quantize's own output is the attention kernel's input:
    same output as the appended cache (identical bytes -> identical result)."""
    B, H, D, s, n = 3, 4, 128, 200, 2
    T = s + n
    k, v = synth.fill(83, 1, (B, H, T, D)).to(cuda), synth.fill(83, 2, (B, H, T, D)).to(cuda)
    kc, km = fq.flexq_quantize(k.view(-1, D))
    vc, vm = fq.flexq_quantize(v.view(-1, D))
    imp = fq.KVCache(B, H, D, s, n, device=cuda)
    fq.flexq_kv_import(imp, kc.view(B, H, T, D // 2), km.view(B, H, T, D // 64, 2), vc.view(B, H, T, D // 2),
                       vm.view(B, H, T, D // 64, 2))
    app = fq.KVCache(B, H, D, s, n, device=cuda)
    fq.flexq_append_kv(k, v, app, pos=0)
    q = synth.fill(83, 3, (B, H, D)).to(cuda)
    assert torch.equal(fq.flexq_decode_attention(q, imp, T), fq.flexq_decode_attention(q, app, T))


def test_export_import_on_a_side_stream(cuda):
    """Export / import issued on a stream other than the current one (bench.py's token-major
    copies): the binding orders the calls after the current stream's zero-fill of the arrays it
    allocates and keeps their memory alive for the side stream, so every copy is complete --
    before the fix some of the copies came out empty."""
    B, H, D, s, n = 16, 12, 128, 300, 4
    srcs = []
    for j in range(4):
        c = fq.KVCache(B, H, D, s, n, device=cuda)
        fq.flexq_append_kv(synth.fill(82, 2 * j, (B, H, s + n, D), device=cuda),
                           synth.fill(82, 2 * j + 1, (B, H, s + n, D), device=cuda), c, pos=0)
        srcs.append(c)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    outs = []
    for c in srcs:
        t = fq.KVCache(B, H, D, s, n, device=cuda, layout="token_major")
        plain = fq.flexq_kv_export(c, stream=side)
        fq.flexq_kv_import(t, *plain, stream=side)
        del plain
        outs.append(t)
    side.synchronize()
    for c, t in zip(srcs, outs):
        for a, b in zip(fq.flexq_kv_export(c), fq.flexq_kv_export(t)):
            assert torch.equal(a, b)

"""NEXT-4: host-offloaded compressed KV with Alg. 1's overlap.  The offloaded
pipeline runs the same kernels on the same bytes as the device-resident path, so its outputs
and the host copies of the caches must be bit-identical to a device-resident run; the first
step's outputs are also checked against the oracle."""
import numpy as np
import pytest
import torch

from paper_2303_06865_b200 import flexq as fq
from paper_2303_06865_b200 import synth
from paper_2303_06865_b200.offload import OffloadedKV

pytestmark = pytest.mark.gpu


def test_offloaded_decode_matches_resident(orc, cuda):
    L, KB, B, H, D, s, n = 3, 2, 3, 8, 128, 100, 8
    seed = 6100

    def t(kind, j, k, step, shape):
        return synth.fill(seed, synth.tensor_id(j * 16 + k, kind, step), shape, device=cuda)

    off = OffloadedKV(L, KB, B, H, D, s, n, cuda, slots=2)
    off.prefill(lambda j, k: t(synth.K_PROMPT, j, k, 0, (B, H, s, D)),
                lambda j, k: t(synth.V_PROMPT, j, k, 0, (B, H, s, D)))
    res = {}
    for j, k in off.items():
        c = fq.KVCache(B, H, D, s, n, device=cuda)
        fq.flexq_append_kv(t(synth.K_PROMPT, j, k, 0, (B, H, s, D)), t(synth.V_PROMPT, j, k, 0, (B, H, s, D)), c, 0)
        res[j, k] = c
    outs = {jk: torch.empty(B, H, D, dtype=torch.float16, device=cuda) for jk in off.items()}
    for step in range(1, 4):
        cur = s + step
        q = lambda j, k: t(synth.Q, j, k, step, (B, H, D))            # noqa: E731
        kn = lambda j, k: t(synth.K_NEW, j, k, step, (B, H, D))       # noqa: E731
        vn = lambda j, k: t(synth.V_NEW, j, k, step, (B, H, D))       # noqa: E731
        off.decode_step(cur, q, kn, vn, lambda j, k: outs[j, k])
        torch.cuda.synchronize()
        for j, k in off.items():
            ref = fq.flexq_append_decode_attention(q(j, k), kn(j, k), vn(j, k), res[j, k], cur)
            assert torch.equal(outs[j, k], ref), (step, j, k)
    torch.cuda.synchronize()
    for j, k in off.items():
        assert torch.equal(off.host[j][k].k, res[j, k].k.cpu()), (j, k)
        assert torch.equal(off.host[j][k].v, res[j, k].v.cpu()), (j, k)
    # and against the oracle for one block at the last step (host-regenerated inputs)
    j, k = 2, 1
    okc, ovc = orc.empty_cache(B, H, s + n, D), orc.empty_cache(B, H, s + n, D)
    cpu = lambda kind, st, shape: synth.fill(seed, synth.tensor_id(j * 16 + k, kind, st), shape).numpy()  # noqa
    orc.append_kv(cpu(synth.K_PROMPT, 0, (B, H, s, D)), cpu(synth.V_PROMPT, 0, (B, H, s, D)), okc, ovc, 0)
    for st in range(1, 4):
        orc.append_kv(cpu(synth.K_NEW, st, (B, H, 1, D)), cpu(synth.V_NEW, st, (B, H, 1, D)), okc, ovc, s + st - 1)
    ref = orc.attention_f64(cpu(synth.Q, 3, (B, H, D)), okc, ovc, s + 3)
    got = outs[j, k].cpu().numpy().astype(np.float64)
    assert (np.abs(got - ref) <= np.maximum(2e-3, 1e-2 * np.abs(ref))).all()

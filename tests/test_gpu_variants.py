"""GPU parity for the quantizer variants (b in {2, 3, 8}, g in {32, 128}),
through the C ABI, against the oracle's general-b quantizer (O2-O5) and bit-stream packing (O6,
S:520): codes, metadata and dequantized values byte-identical."""
import numpy as np
import pytest
import torch

from paper_2303_06865_b200 import flexq as fq
from paper_2303_06865_b200 import synth

pytestmark = pytest.mark.gpu

VARIANTS = [(b, g) for b in (2, 3, 4, 8) for g in (32, 64, 128) if (b, g) != (4, 64)]
SETS = [
    ("default", lambda g: synth.fill(51, 1, (37, 3 * 128))),
    ("outliers", lambda g: synth.with_outliers(synth.fill(51, 2, (64, 256)))),
    ("ties", lambda g: synth.ties(51, 3, (129, 128))),
    ("extreme", lambda g: synth.extreme(51, 4, 256, 128, group=g)),
    ("one_row", lambda g: synth.fill(51, 5, (1, 128))),
]


@pytest.mark.parametrize("bits,group", VARIANTS, ids=[f"b{b}g{g}" for b, g in VARIANTS])
@pytest.mark.parametrize("name,make", SETS, ids=[s[0] for s in SETS])
def test_quantize_variant_bit_exact(orc, cuda, bits, group, name, make):
    x = make(group)
    codes, meta = fq.flexq_quantize(x.to(cuda), bits=bits, group_size=group)
    deq = fq.flexq_dequantize(codes, meta, bits=bits, group_size=group)
    torch.cuda.synchronize()
    oc, om = orc.quantize(x.numpy(), bits, group)
    assert np.array_equal(codes.cpu().numpy(), orc.pack_bits(oc, bits)), f"codes b={bits} g={group} {name}"
    assert np.array_equal(meta.cpu().numpy().view(np.uint16), om), f"meta b={bits} g={group} {name}"
    od = orc.dequantize(oc, om, bits, group)
    assert np.array_equal(deq.cpu().numpy().view(np.uint16), od.view(np.uint16)), f"dequant {name}"


@pytest.mark.parametrize("bits,group", [(2, 32), (3, 128), (8, 64)])
def test_quantize_variant_large_grid_stride(orc, cuda, bits, group):
    """More groups than the grid's threads (grid-stride loop), at a ragged row count."""
    x = synth.fill(52, bits * 1000 + group, (3001, 1024))
    codes, meta = fq.flexq_quantize(x.to(cuda), bits=bits, group_size=group)
    oc, om = orc.quantize(x.numpy(), bits, group)
    assert np.array_equal(codes.cpu().numpy(), orc.pack_bits(oc, bits))
    assert np.array_equal(meta.cpu().numpy().view(np.uint16), om)

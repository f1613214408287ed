"""Byte accounting pinned to the paper's printed example and SPEC's
exact byte counts."""
from paper_2303_06865_b200 import workloads as wl


def test_opt175b_memory_example():
    w = wl.Workload("opt-175b-b512", 512, 96, 128, 512, 32, 96, 49152)
    # weights "325 GB", KV cache "1.2 TB, which is 3.8x the model weights"
    assert wl.weight_bytes_fp16(w) == 347_892_350_976
    assert wl.kv_peak_bytes_fp16(w) == 1_314_259_992_576
    assert round(wl.weight_bytes_fp16(w) / 2 ** 30) == 324
    assert abs(wl.kv_peak_bytes_fp16(w) / 1e12 - 1.3) < 0.02
    assert round(wl.kv_peak_bytes_fp16(w) / wl.weight_bytes_fp16(w), 1) == 3.8


def test_compression_ratio():
    assert wl.COMPRESSED_BYTES_PER_ELEM * 8 == 4.5
    w = wl.CONFIGS["opt-175b"]
    assert wl.kv_cache_bytes_compressed(w) * 16 == wl.kv_peak_bytes_fp16(w) * 4.5


def test_attention_bytes_formula():
    # 1.125 cur_len h1 + 4 h1 per (sequence, layer, step)
    h1 = 12288
    assert wl.attention_bytes(1, h1, 543) == 1.125 * 543 * h1 + 4 * h1
    # fp16 equivalent of the paper's per-layer KV I/O 4 bls (s + n/2) h1
    assert wl.attention_bytes(144, h1, 528) - 144 * 4 * h1 == 4 * 144 * 528 * h1 * 0.28125

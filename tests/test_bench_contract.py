"""The committed bench lines (profiles/) against the bench contract and the byte arithmetic of
SURVEY 8(d), derived here by hand from the cache layout (no GPU; host logic only).

Per (b, h) and cached token, the 4-bit cache holds D/2 code bytes and D/64 (scale, min) fp16 pairs
(4 B each) for K and again for V (north_star "group 64, fp16 scale/min pairs"): 144 B at
D = 128.  A fused decode launch at cur_len T also reads q and the new token's fp16 K / V rows,
writes the output and the new token's 144 B of cache (roofline)."""
import json
import os

import pytest

from paper_2303_06865_b200 import workloads as wl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LINES = ["profiles/r2_bench_reentry.json", "profiles/r2_bench.json"]
B, H, D, S, N, L = 144, 96, 128, 512, 32, 96          # OPT-175B, BASELINE configs[1]
HEADS = B * H


def per_token_bytes(d: int) -> int:
    return 2 * (d // 2 + (d // 64) * 4)               # K and V: codes + (scale, min) pairs


def fused_launch_bytes(cur_len: int) -> int:
    q_out = 2 * (2 * D)                               # q in, out, fp16
    new_rows = 2 * (2 * D)                            # k_new, v_new, fp16
    return HEADS * (cur_len * per_token_bytes(D) + q_out + new_rows + per_token_bytes(D))


def load(path):
    with open(os.path.join(ROOT, path)) as f:
        return json.load(f)


def test_hand_formula_matches_workloads():
    """workloads.py's attention / append bytes equal the hand derivation at every cur_len of the
    bench's cycle (the append's bytes: the fp16 rows read + the quantized token written)."""
    for cur in range(S + 1, S + N):
        got = wl.attention_bytes(B, H * D, cur) + wl.append_bytes(B, H * D)
        assert got == fused_launch_bytes(cur), cur


@pytest.mark.parametrize("path", LINES)
def test_bench_line_contract(path):
    d = load(path)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "cpu_baseline",
              "clocks", "gpu_launches"):
        assert k in d, k
    assert d["warmup"] >= 3 and d["steps"] >= 1 and d["n_gpus"] == 1
    assert d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert "workload" in d["config"] and d["config"]["global_batch"] == B
    # one fused launch per layer and step, all of them the library's
    assert d["gpu_launches"] == L * d["steps"]
    # value: the step's algorithmic bytes over its time; with 31 steps every cur_len of the
    # cycle 513..543 runs once, so value / tokens_per_s = the cycle's mean step bytes / B
    assert d["steps"] % (N - 1) == 0
    mean_step = L * sum(fused_launch_bytes(c) for c in range(S + 1, S + N)) / (N - 1)
    assert d["value"] * 1e9 / d["tokens_per_s"] == pytest.approx(mean_step / B, rel=2e-3)
    assert d["ms_per_step"] == pytest.approx(mean_step / (d["value"] * 1e9) * 1e3, rel=2e-3)


@pytest.mark.parametrize("path", LINES)
def test_bench_line_roofline(path):
    r = load(path)["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak_kind"] == "measured"
    # the per-launch pass runs at the cycle's longest context
    assert r["bytes_per_launch"] == fused_launch_bytes(S + N - 1)
    assert r["achieved"] == pytest.approx(r["bytes_per_launch"] / (r["us_per_launch"] * 1e-6) / 1e9, rel=2e-3)
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], abs=2e-4)
    # ncu's DRAM traffic of the same launch shape is the algorithmic bytes, no re-reads
    assert 1.0 <= r["traffic"] / r["bytes_per_launch"] <= 1.01


@pytest.mark.parametrize("path", LINES)
def test_bench_line_e2e_and_clocks(path):
    d = load(path)
    e = d["e2e"]
    # every step: q, k_new, v_new (fp16) of every layer in; the last layer's output back
    assert e["h2d_bytes_per_step"] == L * HEADS * 3 * 2 * D
    assert e["d2h_bytes_per_step"] == HEADS * 2 * D
    assert e["unit"] == "GB/s" and 0 < e["value"] < d["value"]
    c = d["clocks"]
    assert not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(c["reasons"])
    assert 0 < c["sm_mhz"] <= c["sm_max_mhz"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0


def test_reference_arm_line():
    """The reference arm (the oracle on the host's cores): same metric, unit
    and workload as the device line, its own value in cpu_baseline and e2e, no transfers."""
    d, dev = load("profiles/r2_bench_reference.json"), load(LINES[0])
    assert d["impl"] == "reference"
    for k in ("metric", "unit", "higher_is_better", "dtype", "scaling"):
        assert d[k] == dev[k], k
    assert d["config"]["global_batch"] == dev["config"]["global_batch"] and d["warmup"] >= 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0
    # bytes per sampled token: the sample's unit is one 96-head sequence at cur_len 543
    assert d["value"] * 1e9 / d["tokens_per_s"] == pytest.approx(L * fused_launch_bytes(S + N - 1) / B, rel=0.05)

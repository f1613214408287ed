#!/usr/bin/env python
"""bench.py -- decode-step throughput of the compressed-KV hot path on B200.

One step = one decode step of the whole model (Alg. 1's token -> layer loop
order): for each of the l layers, flexq_append_kv (quantize the new
token's K/V into the cache) then flexq_decode_attention over the
cur_len = s + i cached tokens.  Steps cycle i = 1..n-1.  The
workload at N = 1 is OPT-175B (BASELINE.json configs[3]: 96 heads x 128,
s = 512, n = 32, batch 144, l = 96 -> 104 GB of compressed cache resident in
HBM).  metric: algorithmic compressed-KV GB/s of the step (whole job), with
tokens/s alongside.

    python bench.py [--gpus N --steps K --warmup W] [--config opt-175b] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, weak scaling)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compressed-KV decode attention GB/s and tokens/s vs HBM roofline at 1/2/4/8 B200"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=31)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="flexq", choices=["flexq", "reference"])
    ap.add_argument("--config", default="opt-175b")
    ap.add_argument("--layers", type=int, default=0, help="override model depth (0 = full)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--step", default="fused", choices=["fused", "two"],
                    help="per layer: one fused append+attention launch (NEXT-3) or append_kv then attention")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-offload", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget")
    ap.add_argument("--same-device", action="store_true",
                    help="all ranks on cuda:0 with gloo (functional test of the N > 1 path on one GPU)")
    return ap.parse_args()


# ---------------------------------------------------------------- helpers
_T0 = time.time()


_NVTX = [False]


def log(msg: str):
    """Progress line on stderr; also an NVTX range per bench phase (visible in nsys / ncu --nvtx)."""
    sys.stderr.write(f"[bench {time.time() - _T0:7.1f}s] {msg}\n")
    sys.stderr.flush()
    try:
        import torch
        if torch.cuda.is_available():
            if _NVTX[0]:
                torch.cuda.nvtx.range_pop()
            torch.cuda.nvtx.range_push(f"bench:{msg}")
            _NVTX[0] = True
    except Exception:  # noqa: BLE001 -- tracing is best effort
        pass


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return FALLBACK_HBM_GBS, "fallback"


def bf16_peak_tflops() -> float:
    """Measured dense bf16 (= fp16) tensor peak, burst (MEASURED_PEAKS.json), else the guide's fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["bf16_tflops"])
    return 1590.0


class ClockSampler:
    """NVML SM clock / throttle-reason sampling during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def result(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.same_device:          # functional test of the multi-rank path on one GPU (gloo)
        local = 0
    pg = None
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "flexq" and not args.same_device else "gloo"
        if args.impl == "flexq":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
        pg = dist
    return world, rank, local, pg


# ---------------------------------------------------------------- CPU oracle baseline
_ORACLE_STATE = {}


def _oracle_task(_):
    """One sequence (all heads) of one decode step through the oracle: append the
    new token (quantize) then attention_f64 over cur_len tokens
    (P:271-274).  Inputs are prepared in the parent before the fork (numpy
    only in the workers: no torch thread pool after fork); only the step is timed."""
    import oracle
    kc, vc, kn, vn, q, cur_len = _ORACLE_STATE["inputs"]
    t0 = time.perf_counter()
    oracle.append_kv(kn, vn, kc, vc, cur_len - 1)
    oracle.attention_f64(q, kc, vc, cur_len)
    return time.perf_counter() - t0


_POOL = None


def cpu_oracle_baseline(w, budget_s: float, bytes_fn):
    """Time the oracle, as it stands, on a bounded sample of the workload on all
    host cores: one worker process per core, each task = one sequence x all
    heads x one layer of one decode step at cur_len = s + n - 1.  Throughput =
    sample bytes / (sum of per-task step times / cores).  Returns
    (GB/s, sequence-layers/s, cores, sample description)."""
    global _POOL
    import multiprocessing as mp
    import oracle
    from paper_2303_06865_b200 import synth
    oracle.build()
    cores = os.cpu_count() or 1
    cur_len = w.prompt_len + w.gen_len - 1
    H, D = w.heads, w.head_dim
    if _POOL is None:
        import atexit
        seed = synth.BASE_SEED + 77
        kc, vc = oracle.empty_cache(1, H, cur_len, D), oracle.empty_cache(1, H, cur_len, D)
        kp = synth.fill(seed, synth.tensor_id(0, synth.K_PROMPT), (1, H, cur_len - 1, D)).numpy()
        vp = synth.fill(seed, synth.tensor_id(0, synth.V_PROMPT), (1, H, cur_len - 1, D)).numpy()
        oracle.append_kv(kp, vp, kc, vc, 0)
        kn = synth.fill(seed, synth.tensor_id(0, synth.K_NEW), (1, H, 1, D)).numpy()
        vn = synth.fill(seed, synth.tensor_id(0, synth.V_NEW), (1, H, 1, D)).numpy()
        q = synth.fill(seed, synth.tensor_id(0, synth.Q), (1, H, D)).numpy()
        _ORACLE_STATE["inputs"] = (kc, vc, kn, vn, q, cur_len)
        _POOL = mp.get_context("fork").Pool(cores)
        atexit.register(_POOL.terminate)
    t1 = statistics.median(_POOL.map(_oracle_task, range(cores), chunksize=1))
    n_tasks = max(cores, int(budget_s / max(t1, 1e-4)) * cores)
    n_tasks = min(n_tasks, 256 * cores)
    times = _POOL.map(_oracle_task, range(n_tasks), chunksize=1)
    busy = sum(times) / cores
    nbytes = bytes_fn(n_tasks, cur_len)
    gbs = nbytes / busy / 1e9
    sample = (f"{n_tasks} tasks x (1 sequence x {H} heads x 1 layer: append 1 token + attention_f64 at "
              f"cur_len {cur_len}); {t1 * 1e3:.1f} ms per task; {cores} worker processes; "
              f"rate = bytes / (sum task time / cores)")
    return gbs, n_tasks / busy, cores, sample


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    world, rank, local, pg = dist_setup(args)
    if rank != 0:
        return
    from paper_2303_06865_b200 import workloads as wl
    w = wl.CONFIGS[args.config]
    if args.layers:
        w = wl.Workload(w.name, w.batch, w.heads, w.head_dim, w.prompt_len, w.gen_len, args.layers, w.h2)
    per = lambda n, cur: n * (wl.attention_bytes(1, w.h1, cur) + wl.append_bytes(1, w.h1))  # noqa: E731
    budget = max(2.0, min(args.cpu_seconds, 120.0 / max(1, args.steps + args.warmup)))
    vals = []
    for i in range(args.warmup + args.steps):
        gbs, seqs, cores, sample = cpu_oracle_baseline(w, budget, per)
        if i >= args.warmup:
            vals.append((gbs, seqs))
    gbs = statistics.median(v[0] for v in vals)
    seqs = statistics.median(v[1] for v in vals)
    tok_s = seqs / w.layers
    line = {"metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u4+f16->f32",
            "data": "synthetic", "tokens_per_s": round(tok_s, 4),
            "config": {"workload": f"{w.name}: batch {w.batch}, {w.heads}x{w.head_dim}, s={w.prompt_len}, "
                                   f"n={w.gen_len}, l={w.layers}; oracle on a bounded per-step sample",
                       "global_batch": w.batch, "seq_len": w.prompt_len + w.gen_len},
            "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- flexq arm
def run_flexq(args):
    import torch
    from paper_2303_06865_b200 import flexq as fq
    from paper_2303_06865_b200 import synth
    from paper_2303_06865_b200 import workloads as wl

    world, rank, local, pg = dist_setup(args)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    fq.lib()

    w = wl.CONFIGS[args.config]
    if args.layers:
        w = wl.Workload(w.name, w.batch, w.heads, w.head_dim, w.prompt_len, w.gen_len, args.layers, w.h2)
    from paper_2303_06865_b200 import dist as fd
    B_total = w.batch * (world if args.scaling == "weak" else 1)
    B = fd.rank_batch(w.batch, world, rank, args.scaling)
    if B == 0:
        raise SystemExit(f"--scaling strong needs batch ({w.batch}) >= ranks ({world})")
    H, D, s, n, L = w.heads, w.head_dim, w.prompt_len, w.gen_len, w.layers
    h1 = H * D
    seed = synth.BASE_SEED + 3 + 1000 * rank
    stream = torch.cuda.Stream(device=dev)

    # ---- setup: compressed caches for all layers resident in HBM
    log("setup")
    with torch.cuda.stream(stream):
        caches = [fq.KVCache(B, H, D, s, n, device=dev) for _ in range(L)]
        kp = synth.fill(seed, synth.tensor_id(0, synth.K_PROMPT), (B, H, s, D), device=dev)
        vp = synth.fill(seed, synth.tensor_id(0, synth.V_PROMPT), (B, H, s, D), device=dev)
        for c in caches:                                  # prompt fill (prefill's KV, quantized)
            fq.flexq_append_kv(kp, vp, c, pos=0)
        del kp, vp
        qs = synth.fill(seed, synth.tensor_id(0, synth.Q), (L, B, H, D), device=dev)
        kn = synth.fill(seed, synth.tensor_id(0, synth.K_NEW), (L, B, H, 1, D), device=dev)
        vn = synth.fill(seed, synth.tensor_id(0, synth.V_NEW), (L, B, H, 1, D), device=dev)
        outs = torch.empty(L, B, H, D, dtype=torch.float16, device=dev)
        ws = fq.make_workspace(caches[0])
    torch.cuda.synchronize()
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    cache_bytes = sum(c.nbytes() for c in caches)

    fused = args.step == "fused"

    def layer_step(j, cur, q, k_new, v_new, out, st):
        """One layer of decode step cur_len = cur: append the token, attend (one or two launches)."""
        if fused:
            fq.flexq_append_decode_attention(q, k_new, v_new, caches[j], cur, out=out, workspace=ws, stream=st)
        else:
            fq.flexq_append_kv(k_new.view(B, H, 1, D), v_new.view(B, H, 1, D), caches[j], pos=cur - 1, stream=st)
            fq.flexq_decode_attention(q, caches[j], cur, out=out, workspace=ws, stream=st)

    def step_calls(i, st):
        cur = s + i
        for j in range(L):
            layer_step(j, cur, qs[j], kn[j], vn[j], outs[j], st)

    # one CUDA graph per decode step i = 1..n-1
    log("prompt fill done; capturing graphs")
    steps_i = list(range(1, n))
    graphs = {}
    with torch.cuda.stream(stream):
        step_calls(1, stream)                              # warm the launch path before capture
    torch.cuda.synchronize()
    for i in steps_i:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            step_calls(i, stream)
        graphs[i] = g
    torch.cuda.synchronize()

    def seq_of(k):
        return steps_i[k % len(steps_i)]

    step_bytes = {i: L * (wl.attention_bytes(B, h1, s + i) + wl.append_bytes(B, h1)) for i in steps_i}

    def barrier():
        if pg:
            pg.barrier()
        torch.cuda.synchronize()

    # ---- warmup + timed region (device events on the launching stream)
    log("graphs captured; timing")
    for k in range(args.warmup):
        graphs[seq_of(k)].replay()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for k in range(args.steps):
                i = seq_of(args.warmup + k)
                graphs[i].replay()
            ev1.record(stream)
        barrier()
    ms = fd.max_over_ranks(ev0.elapsed_time(ev1), device=dev)
    ms_step = ms / args.steps
    job_bytes = B_total * sum(L * (wl.attention_bytes(1, h1, s + seq_of(args.warmup + k)) + wl.append_bytes(1, h1))
                              for k in range(args.steps))
    value_gbs = job_bytes / (ms / 1e3) / 1e9
    tokens_per_s = B_total * args.steps / (ms / 1e3)

    # ---- N > 1: gather every rank's outputs of one layer-step (NCCL all-gather),
    # outside the timed data path and timed on its own; checked against each rank's own block
    allgather = None
    if world > 1:
        torch.cuda.synchronize()
        # same-device functional runs use gloo, which gathers host tensors
        src = outs[L - 1].cpu() if args.same_device else outs[L - 1]
        G_out = B_total if args.scaling == "strong" else B * world
        per = (G_out + world - 1) // world
        full = fd.gather_outputs(src, G_out)
        ok = bool(torch.equal(full[rank * per: rank * per + B], src))
        barrier()
        t0 = time.perf_counter()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        for _ in range(20):
            fd.gather_outputs(src, G_out)
        g1.record()
        torch.cuda.synchronize()
        ag_us = (g0.elapsed_time(g1) if not args.same_device else (time.perf_counter() - t0) * 1e3) / 20 * 1e3
        ag_us = fd.max_over_ranks(ag_us, device=dev)
        ok_all = fd.max_over_ranks(0.0 if ok else 1.0, device=dev) == 0.0
        allgather = {"what": "all_gather_into_tensor of one layer-step's fp16 outputs [B][H][D] per rank",
                     "bytes_per_rank": int(src.numel() * 2), "us": round(ag_us, 1),
                     "matches_rank_blocks": ok_all, "in_timed_region": False,
                     "backend": "gloo (same-device functional run)" if args.same_device else "nccl"}
        del full

    # ---- dominant kernel: attention alone, one graph of L launches at cur_len = s + n - 1
    log("timed; per-kernel pass")
    cur_last = s + n - 1
    ga = torch.cuda.CUDAGraph()
    with torch.cuda.graph(ga, stream=stream):
        for j in range(L):
            fq.flexq_decode_attention(qs[j], caches[j], cur_last, out=outs[j], workspace=ws, stream=stream)
    gapp = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gapp, stream=stream):
        for j in range(L):
            fq.flexq_append_kv(kn[j], vn[j], caches[j], pos=cur_last - 1, stream=stream)
    gfu = torch.cuda.CUDAGraph()          # fused append + attention (rewrites the same token: idempotent)
    with torch.cuda.graph(gfu, stream=stream):
        for j in range(L):
            fq.flexq_append_decode_attention(qs[j], kn[j], vn[j], caches[j], cur_last, out=outs[j], workspace=ws,
                                             stream=stream)
    reps = 5
    for g in (ga, gapp, gfu):
        g.replay()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    with torch.cuda.stream(stream):
        e[0].record(stream)
        for _ in range(reps):
            ga.replay()
        e[1].record(stream)
        for _ in range(reps):
            gapp.replay()
        e[2].record(stream)
        for _ in range(reps):
            gfu.replay()
        e[3].record(stream)
    torch.cuda.synchronize()
    attn_us = e[0].elapsed_time(e[1]) * 1e3 / (reps * L)
    app_us = e[1].elapsed_time(e[2]) * 1e3 / (reps * L)
    fused_us = e[2].elapsed_time(e[3]) * 1e3 / (reps * L)
    attn_bytes = wl.attention_bytes(B, h1, cur_last)
    fused_bytes = attn_bytes + wl.append_bytes(B, h1)
    peak, peak_kind = peaks()
    # the dominant kernel is the one the step launches per layer
    k_us, k_bytes = (fused_us, fused_bytes) if fused else (attn_us, attn_bytes)
    achieved = k_bytes / (k_us * 1e-6) / 1e9

    # ---- NEXT-1: Top-K sparse attention (keep 10%) at the same shape
    topk = None
    if cur_last <= 1152:
        keep = fq.topk_keep(cur_last)
        gt = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gt, stream=stream):
            for j in range(L):
                fq.flexq_decode_attention_topk(qs[j], caches[j], cur_last, keep, out=outs[j], workspace=ws,
                                               stream=stream)
        gt.replay()
        torch.cuda.synchronize()
        t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            t0e.record(stream)
            for _ in range(reps):
                gt.replay()
            t1e.record(stream)
        torch.cuda.synchronize()
        tk_us = t0e.elapsed_time(t1e) * 1e3 / (reps * L)
        kv_row = h1 // 2 + h1 // 64 * 4                      # one token's K (or V) bytes over all heads
        tk_bytes = B * (cur_last * kv_row + keep * kv_row + 2 * h1 * 2)
        topk = {"keep": keep, "cur_len": cur_last, "us_per_launch": round(tk_us, 2),
                "algorithmic_bytes_per_launch": tk_bytes, "GBps": round(tk_bytes / (tk_us * 1e-6) / 1e9, 1),
                "speedup_vs_dense": round(attn_us / tk_us, 3),
                "note": "bytes = K for all tokens + V for the kept 10% (P:856) + q + out; the V gather "
                        "reads each kept token's 4-token quad row"}
    traffic = None
    tp = os.path.join(ROOT, "profiles", "attention_traffic.json")
    if os.path.exists(tp) and w.name == "opt-175b" and B == 144:
        traffic = json.load(open(tp)).get("fused_dram_bytes_per_launch" if fused else "dram_bytes_per_launch")

    # ---- e2e: host buffers through the public API, H2D of the step's inputs and D2H of its outputs
    log("e2e")
    e2e = None
    if not args.no_e2e:
        # one pinned block per layer holding (q, k_new, v_new): one H2D copy per layer
        hin = torch.stack([qs, kn.view(qs.shape), vn.view(qs.shape)], dim=1).cpu().pin_memory()   # [L][3][B][H][D]
        outh = torch.empty(outs.shape, dtype=outs.dtype).pin_memory()
        NB = 6                                     # device slots: H2D runs up to NB layers ahead
        din = [torch.empty_like(hin[0], device=dev) for _ in range(NB)]
        dout = [torch.empty_like(outs[0]) for _ in range(NB)]
        h2d = torch.cuda.Stream(device=dev)       # one stream per copy direction: both copy engines busy
        d2h = torch.cuda.Stream(device=dev)
        ready = [torch.cuda.Event() for _ in range(NB)]
        consumed = [torch.cuda.Event() for _ in range(NB)]
        drained = [torch.cuda.Event() for _ in range(NB)]
        gl = [0]                                   # global layer counter (slot = gl % NB)

        def e2e_step(i):
            cur = s + i
            for j in range(L):
                g = gl[0]
                gl[0] += 1
                b = g % NB
                with torch.cuda.stream(h2d):
                    if g >= NB:
                        h2d.wait_event(consumed[b])        # slot b's inputs consumed by layer g - NB
                    din[b].copy_(hin[j], non_blocking=True)
                    ready[b].record(h2d)
                stream.wait_event(ready[b])
                if g >= NB:
                    stream.wait_event(drained[b])          # slot b's output copied out
                layer_step(j, cur, din[b][0], din[b][1], din[b][2], dout[b], stream)
                consumed[b].record(stream)
                with torch.cuda.stream(d2h):
                    d2h.wait_event(consumed[b])
                    outh[j].copy_(dout[b], non_blocking=True)
                    drained[b].record(d2h)

        for k in range(2):
            e2e_step(seq_of(k))
        barrier()
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2e_bytes = 0
        ke = max(3, min(args.steps, 10))
        x0.record(stream)
        for k in range(ke):
            i = seq_of(k)
            e2e_step(i)
            e2e_bytes += step_bytes[i]
        stream.wait_stream(d2h)                    # the last outputs are home
        x1.record(stream)
        barrier()
        ems = fd.max_over_ranks(x0.elapsed_time(x1), device=dev)
        e2e_job = e2e_bytes * (B_total / B if B else 0)
        e2e = {"value": round(e2e_job / (ems / 1e3) / 1e9, 2),
               "unit": "GB/s", "h2d_bytes_per_step": int(hin.nbytes),
               "d2h_bytes_per_step": int(outh.nbytes), "ms_per_step": round(ems / ke, 3),
               "tokens_per_s": round(B_total * ke / (ems / 1e3), 2),
               "how": "pinned host (q, k_new, v_new) block per layer -> one H2D copy on a copy stream, D2H of the "
                      "output on another, 6 device slots so copies run ahead of compute; append+attention via the "
                      "C ABI, D2H of every layer's output; CUDA events, max over ranks"}

    # ---- weight quantize / dequantize sweep (BASELINE configs[4]), rank 0
    log("sweep")
    sweep = gemm = None
    if rank == 0 and not args.no_sweep:
        sweep, gemm = {}, {}
        bf16_peak = bf16_peak_tflops()
        for (r, c) in ((12288, 49152), (12288, 12288)):
            x = synth.fill(seed, synth.tensor_id(0, synth.WEIGHT, c), (r, c), device=dev)
            codes = torch.empty(r, c // 2, dtype=torch.uint8, device=dev)
            meta = torch.empty(r, c // 64, 2, dtype=torch.float16, device=dev)
            y = torch.empty_like(x)
            # each op as a CUDA graph of 10 launches (no host launch gaps inside the timing)
            def graph_of(fn):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for _ in range(10):
                        fn()
                return g
            with torch.cuda.stream(stream):
                fq.flexq_quantize(x, codes, meta, stream=stream)
                fq.flexq_dequantize(codes, meta, y, stream=stream)
            torch.cuda.synchronize()
            gq = graph_of(lambda: fq.flexq_quantize(x, codes, meta, stream=stream))
            gd = graph_of(lambda: fq.flexq_dequantize(codes, meta, y, stream=stream))
            tq, td = [], []
            with torch.cuda.stream(stream):
                for _ in range(5):
                    a0, a1, a2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                    a0.record(stream)
                    gq.replay()
                    a1.record(stream)
                    gd.replay()
                    a2.record(stream)
                    a2.synchronize()
                    tq.append(a0.elapsed_time(a1) / 10)
                    td.append(a1.elapsed_time(a2) / 10)
            # NEXT-2: the decode linear layer y = t . w^ over this 4-bit weight at the decode batch
            # (M = 144), through flexq_pack_weight + flexq_dequant_gemm (tcgen05 kernel),
            # beside two library baselines: flexq_dequantize + cuBLAS, and cuBLAS on the fp16 weight.
            M = 144
            panels = fq.flexq_pack_weight(codes, meta)
            xt = synth.fill(seed, synth.tensor_id(0, synth.WEIGHT, c + 1), (M, r), device=dev)
            yt = torch.empty(M, c, dtype=torch.float16, device=dev)
            wsg = fq.make_gemm_workspace(M, r, c, dev)
            with torch.cuda.stream(stream):
                fq.flexq_dequant_gemm(xt, panels, c, out=yt, workspace=wsg, stream=stream)
                torch.matmul(xt, y, out=yt)
            torch.cuda.synchronize()
            gg = graph_of(lambda: fq.flexq_dequant_gemm(xt, panels, c, out=yt, workspace=wsg, stream=stream))
            gb1 = graph_of(lambda: (fq.flexq_dequantize(codes, meta, y, stream=stream), torch.matmul(xt, y, out=yt)))
            gb2 = graph_of(lambda: torch.matmul(xt, x, out=yt))
            tg, tb1, tb2 = [], [], []
            with torch.cuda.stream(stream):
                for _ in range(5):
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                    ev[0].record(stream)
                    gg.replay()
                    ev[1].record(stream)
                    gb1.replay()
                    ev[2].record(stream)
                    gb2.replay()
                    ev[3].record(stream)
                    ev[3].synchronize()
                    tg.append(ev[0].elapsed_time(ev[1]) / 10)
                    tb1.append(ev[1].elapsed_time(ev[2]) / 10)
                    tb2.append(ev[2].elapsed_time(ev[3]) / 10)
            fl = 2.0 * M * r * c
            tgm = statistics.median(tg) * 1e-3
            gemm[f"{M}x{r}x{c}"] = {
                "us": round(tgm * 1e6, 1), "tflops": round(fl / tgm / 1e12, 1),
                "tensor_frac_of_measured_bf16": round(fl / tgm / 1e12 / bf16_peak, 4),
                "weight_gbs": round((r * c // 2 + r * c // 64 * 4) / tgm / 1e9, 1),
                "dequantize_then_cublas_us": round(statistics.median(tb1) * 1e3, 1),
                "cublas_fp16_weight_us": round(statistics.median(tb2) * 1e3, 1)}
            del panels, xt, yt, wsg, gg, gb1, gb2
            nb = r * c * 2 + r * c // 2 + r * c // 64 * 4
            sweep[f"{r}x{c}"] = {"quantize_us": round(statistics.median(tq) * 1e3, 1),
                                 "quantize_gbs": round(nb / (statistics.median(tq) * 1e-3) / 1e9, 1),
                                 "dequantize_us": round(statistics.median(td) * 1e3, 1),
                                 "dequantize_gbs": round(nb / (statistics.median(td) * 1e-3) / 1e9, 1)}
            del x, codes, meta, y, gq, gd

    # ---- the other BASELINE configs (OPT-6.7B, OPT-30B shapes): decode attention alone at the last
    # step's context, 4 layers of fresh caches, one CUDA graph -- per-launch time and GB/s (rank 0)
    other = None
    if rank == 0 and not args.no_sweep and w.name == "opt-175b":
        other = {}
        for cname in ("opt-6.7b", "opt-30b"):
            cw = wl.CONFIGS[cname]
            cl, cB = 4, cw.batch
            ccaches = [fq.KVCache(cB, cw.heads, cw.head_dim, cw.prompt_len, cw.gen_len, device=dev) for _ in range(cl)]
            for j in range(cl):
                kp = synth.fill(seed + 7, synth.tensor_id(j, synth.K_PROMPT), (cB, cw.heads, cw.prompt_len, cw.head_dim),
                                device=dev)
                fq.flexq_append_kv(kp, kp, ccaches[j], pos=0)
                del kp
            ccur = cw.prompt_len + cw.gen_len - 1
            cq = synth.fill(seed + 7, synth.tensor_id(0, synth.Q), (cB, cw.heads, cw.head_dim), device=dev)
            cout = torch.empty_like(cq)
            cws = fq.make_workspace(ccaches[0])
            gc = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gc, stream=stream):
                for j in range(cl):
                    fq.flexq_decode_attention(cq, ccaches[j], ccur, out=cout, workspace=cws, stream=stream)
            gc.replay()
            torch.cuda.synchronize()
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                c0.record(stream)
                for _ in range(10):
                    gc.replay()
                c1.record(stream)
            torch.cuda.synchronize()
            cus = c0.elapsed_time(c1) * 1e3 / (10 * cl)
            cbytes = wl.attention_bytes(cB, cw.h1, ccur)
            other[cname] = {"batch": cB, "heads": cw.heads, "cur_len": ccur, "us_per_launch": round(cus, 2),
                            "bytes_per_launch": cbytes, "GBps": round(cbytes / (cus * 1e-6) / 1e9, 1),
                            "frac_of_measured_hbm": round(cbytes / (cus * 1e-6) / 1e9 / peak, 4)}
            del ccaches, cq, cout, cws, gc

    # ---- NEXT-3 variants of the KV cache (rank 0): decode attention on the OPT-175B shape at the
    # last step's context for three (b, g), 2 layers of fresh caches each, one CUDA graph
    kv_variants = None
    if rank == 0 and not args.no_sweep and w.name == "opt-175b":
        kv_variants = {}
        vcur = s + n - 1
        vk = synth.fill(seed + 9, synth.tensor_id(0, synth.K_PROMPT), (B, H, vcur, D), device=dev)
        vq = synth.fill(seed + 9, synth.tensor_id(0, synth.Q), (B, H, D), device=dev)
        vout = torch.empty_like(vq)
        for vb, vg in ((2, 32), (3, 64), (8, 128)):
            vcaches = [fq.KVCache(B, H, D, s, n, device=dev, bits=vb, group_size=vg) for _ in range(2)]
            for vc in vcaches:
                fq.flexq_append_kv(vk, vk, vc, pos=0)
            vws = fq.make_workspace(vcaches[0])
            gv = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gv, stream=stream):
                for vc in vcaches:
                    fq.flexq_decode_attention(vq, vc, vcur, out=vout, workspace=vws, stream=stream)
            gv.replay()
            torch.cuda.synchronize()
            v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                v0.record(stream)
                for _ in range(10):
                    gv.replay()
                v1.record(stream)
            torch.cuda.synchronize()
            vus = v0.elapsed_time(v1) * 1e3 / (10 * len(vcaches))
            vbytes = 2 * B * H * vcur * (D * vb // 8 + 4 * D // vg) + 2 * B * H * D * 2
            kv_variants[f"b{vb}g{vg}"] = {"cur_len": vcur, "us_per_launch": round(vus, 2), "bytes_per_launch": vbytes,
                                          "GBps": round(vbytes / (vus * 1e-6) / 1e9, 1),
                                          "frac_of_measured_hbm": round(vbytes / (vus * 1e-6) / 1e9 / peak, 4),
                                          "kernel": "attention_variant_kernel (CUDA cores)"}
            del vcaches, vws, gv
        del vk, vq, vout

    # ---- NEXT-4: host-offloaded compressed KV, Alg. 1 overlap (rank 0): 2 OPT-175B layers of
    # batch 144 in pinned host memory, streamed through a 2-slot device ring
    log("offload")
    offload = None
    if rank == 0 and not args.no_offload and w.name == "opt-175b":
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        import offload_bench
        offload = offload_bench.run(layers=2, gpu_batches=1, B=B, H=H, D=D, s=s, n=n, steps=3, dev=str(dev))
        offload["bound"] = "pcie"
        offload["how"] = ("per (layer, GPU batch) in Alg. 1 order: H2D of the whole compressed block on a load "
                          "stream, fused append+attention on the compute stream, D2H of the new token's chunk "
                          "on a store stream; value = H2D bytes / device time, vs a pinned 1 GiB H2D copy")

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    log("cpu baseline")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        per = lambda nseq, cur: nseq * (wl.attention_bytes(1, h1, cur) + wl.append_bytes(1, h1))  # noqa: E731
        gbs, seqs, cores, sample = cpu_oracle_baseline(w, args.cpu_seconds, per)
        cpu = {"value": round(gbs, 4), "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value_gbs, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "u4+f16->f32", "data": "synthetic (counter-based Irwin-Hall fp16, P:41/P:44)",
            "tokens_per_s": round(tokens_per_s, 2),
            "attention_tokens_per_s_per_layer": round(tokens_per_s * L, 1),
            "config": {"workload": f"{w.name} decode step: batch {B} per GPU (global {B_total}), {H} heads x {D}, "
                                   f"s={s}, n={n}, l={L} layers, "
                                   + ("fused append+attention (one launch) per layer, " if fused else
                                      "append_kv + decode_attention per layer, ") +
                                   f"steps cycle cur_len {s + 1}..{s + n - 1}",
                       "global_batch": B_total, "seq_len": s + n, "parallelism": f"dp{world} (sequences)",
                       "l2": f"working set {cache_bytes / 1e9:.1f} GB per GPU >> {l2 / 1e6:.0f} MB L2; no flush"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "traffic_source": "profiles/attention_traffic.json (ncu --set full, same launch shape)",
                         "kernel": "decode_attention_kernel<128>" + (" (fused append)" if fused else ""),
                         "peak_kind": peak_kind,
                         "bytes_per_launch": k_bytes, "us_per_launch": round(k_us, 2),
                         # the step's algorithmic bytes at this kernel's measured rate, over the step time
                         # (the per-launch pass runs at the longest context, cur_len = s + n - 1, so
                         # k_us * L would overstate a step whose contexts run s + 1 .. s + n - 1)
                         "share_of_step": round(value_gbs / (achieved * world) if fused else
                                                attn_us * L / (ms_step * 1e3), 4),
                         "attention_only_us_per_launch": round(attn_us, 2),
                         "attention_only_GBps": round(attn_bytes / (attn_us * 1e-6) / 1e9, 1),
                         "append_us_per_launch": round(app_us, 2),
                         "fused_us_per_launch": round(fused_us, 2)},
            "gpu_launches": args.steps * L * (1 if fused else 2),
            "clocks": clk.result(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "weight_sweep": sweep,
            "topk_sparse": topk,
            "dequant_gemm": gemm,
            "offload": offload,
            "allgather": allgather,
            "other_configs": other,
            "kv_variants": kv_variants,
        }
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_flexq(args)


if __name__ == "__main__":
    main()

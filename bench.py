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
    python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

`--gpus N` without torchrun re-launches itself under torch.distributed.run with N ranks.
Scaling: OPT-175B is strong-scaled by default (BASELINE configs[3]: an effective batch of 144
sharded across the GPUs); a weak-scaling run (every rank its own batch of 144) is
reported beside it as `weak_scaling`.
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
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="default: strong for opt-175b (global batch 144 sharded), weak otherwise")
    ap.add_argument("--no-weak", action="store_true", help="skip the weak-scaling secondary run (N > 1)")
    ap.add_argument("--step", default="fused", choices=["fused", "two"],
                    help="per layer: one fused append+attention launch (NEXT-3) or append_kv then attention")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-offload", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget")
    ap.add_argument("--same-device", action="store_true",
                    help="all ranks on cuda:0 with gloo (functional test of the N > 1 path on one GPU)")
    a = ap.parse_args()
    if a.scaling is None:
        a.scaling = "strong" if a.config == "opt-175b" else "weak"
    return a


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
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
                         f"(python -m torch.distributed.run --nproc-per-node {args.gpus} bench.py --gpus "
                         f"{args.gpus} ...), or run without torchrun and let bench.py launch it")
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
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u4+f16->f32",
            "data": "synthetic", "tokens_per_s": round(tok_s, 4),
            "config": {"workload": f"{w.name}: batch {w.batch}, {w.heads}x{w.head_dim}, s={w.prompt_len}, "
                                   f"n={w.gen_len}, l={w.layers}; oracle on a bounded per-step sample",
                       "global_batch": w.batch, "seq_len": w.prompt_len + w.gen_len},
            "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- flexq arm
def rank_rows(B_total: int, world: int, rank: int, scaling: str, per_gpu: int) -> tuple[int, int]:
    """Global sequence rows [b0, b1) of `rank`: its shard of the fixed global batch (strong) or
    its own block of per_gpu sequences (weak).  Inputs are drawn per global row, so any
    sharding sees the same sequences a single process would."""
    from paper_2303_06865_b200 import dist as fd
    if scaling == "strong":
        return fd.shard(B_total, world, rank)
    return rank * per_gpu, (rank + 1) * per_gpu


class DecodeModel:
    """The compressed KV caches of every layer for sequences [b0, b1) of a global batch, with
    the step's per-layer inputs (q, k_new, v_new) and one CUDA graph per decode step i."""

    def __init__(self, w, L, B_total, b0, b1, seed, dev, stream, fused=True):
        import torch
        from paper_2303_06865_b200 import flexq as fq
        from paper_2303_06865_b200 import synth
        self.fq, self.w, self.L, self.B = fq, w, L, b1 - b0
        self.b0, self.b1, self.B_total, self.stream, self.fused = b0, b1, B_total, stream, fused
        H, D, s, n = w.heads, w.head_dim, w.prompt_len, w.gen_len
        self.steps_i = list(range(1, n)) if n > 1 else [1]
        with torch.cuda.stream(stream):
            self.caches = [fq.KVCache(self.B, H, D, s, max(n, 1), device=dev) for _ in range(L)]
            kp = synth.fill_rows(seed, synth.tensor_id(0, synth.K_PROMPT), (B_total, H, s, D), b0, b1, device=dev)
            vp = synth.fill_rows(seed, synth.tensor_id(0, synth.V_PROMPT), (B_total, H, s, D), b0, b1, device=dev)
            for c in self.caches:                                  # prompt fill (prefill's KV, quantized)
                fq.flexq_append_kv(kp, vp, c, pos=0, stream=stream)
            del kp, vp
            rows = lambda kind, j: synth.fill_rows(seed, synth.tensor_id(j, kind), (B_total, H, D), b0, b1,  # noqa: E731
                                                   device=dev)
            self.qs = torch.stack([rows(synth.Q, j) for j in range(L)])
            self.kn = torch.stack([rows(synth.K_NEW, j) for j in range(L)])
            self.vn = torch.stack([rows(synth.V_NEW, j) for j in range(L)])
            self.outs = torch.empty(L, self.B, H, D, dtype=torch.float16, device=dev)
            self.ws = fq.make_workspace(self.caches[0])
        torch.cuda.synchronize()
        self.graphs = {}

    def nbytes(self):
        return sum(c.nbytes() for c in self.caches)

    def layer_step(self, j, cur, q, k_new, v_new, out, st):
        """One layer of decode step cur_len = cur: append the token, attend (one or two launches)."""
        fq, B, H, D = self.fq, self.B, self.w.heads, self.w.head_dim
        if self.fused:
            fq.flexq_append_decode_attention(q, k_new, v_new, self.caches[j], cur, out=out, workspace=self.ws,
                                             stream=st)
        else:
            fq.flexq_append_kv(k_new.view(B, H, 1, D), v_new.view(B, H, 1, D), self.caches[j], pos=cur - 1,
                               stream=st)
            fq.flexq_decode_attention(q, self.caches[j], cur, out=out, workspace=self.ws, stream=st)

    def step_calls(self, i, st):
        cur = self.w.prompt_len + i
        for j in range(self.L):
            self.layer_step(j, cur, self.qs[j], self.kn[j], self.vn[j], self.outs[j], st)

    def capture(self):
        import torch
        with torch.cuda.stream(self.stream):
            self.step_calls(self.steps_i[0], self.stream)          # warm the launch path before capture
        torch.cuda.synchronize()
        for i in self.steps_i:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                self.step_calls(i, self.stream)
            self.graphs[i] = g
        torch.cuda.synchronize()

    def seq_of(self, k):
        return self.steps_i[k % len(self.steps_i)]

    def step_bytes(self, i, rows):
        from paper_2303_06865_b200 import workloads as wl
        h1 = self.w.h1
        return self.L * (wl.attention_bytes(rows, h1, self.w.prompt_len + i) + wl.append_bytes(rows, h1))

    def time_steps(self, warmup, steps, barrier, clocks=None):
        """W untimed steps, then K timed steps (CUDA events on the launching stream)."""
        import torch
        for k in range(warmup):
            self.graphs[self.seq_of(k)].replay()
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx = clocks if clocks is not None else _Null()
        with ctx:
            with torch.cuda.stream(self.stream):
                ev0.record(self.stream)
                for k in range(steps):
                    self.graphs[self.seq_of(warmup + k)].replay()
                ev1.record(self.stream)
            barrier()
        return ev0.elapsed_time(ev1), [self.seq_of(warmup + k) for k in range(steps)]

    def per_launch(self, cur, which, reps=5, layers=None):
        """Average launch time (us) of `which` in {attn, append, fused, topk} over one CUDA graph of
        `layers` launches (one per layer cache) at cur_len = cur."""
        import torch
        fq, st = self.fq, self.stream
        L = self.L if layers is None else min(layers, self.L)
        keep = fq.topk_keep(cur)
        if which == "topk_tm":           # build the token-major copies and the workspace outside the capture
            for j in range(L):
                self.tm_cache(j)
        if which in ("topk", "topk_tm"):
            self.topk_ws()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for j in range(L):
                if which == "attn":
                    fq.flexq_decode_attention(self.qs[j], self.caches[j], cur, out=self.outs[j], workspace=self.ws,
                                              stream=st)
                elif which == "append":
                    fq.flexq_append_kv(self.kn[j].unsqueeze(2), self.vn[j].unsqueeze(2), self.caches[j],
                                       pos=cur - 1, stream=st)
                elif which in ("topk", "topk_tm"):
                    c = self.caches[j] if which == "topk" else self.tm_cache(j)
                    fq.flexq_decode_attention_topk(self.qs[j], c, cur, keep, out=self.outs[j],
                                                   workspace=self.topk_ws(), stream=st)
                else:                   # fused: rewrites the same token at cur - 1 (idempotent)
                    fq.flexq_append_decode_attention(self.qs[j], self.kn[j], self.vn[j], self.caches[j], cur,
                                                     out=self.outs[j], workspace=self.ws, stream=st)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st)
            for _ in range(reps):
                g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / (reps * L)

    def topk_ws(self):
        if getattr(self, "tws", None) is None:
            self.tws = self.fq.make_topk_workspace(self.caches[0])
        return self.tws

    def tm_cache(self, j):
        """Layer j's cache in the token-major layout (Top-K's): the same bytes moved with
        flexq_kv_export / flexq_kv_import (no requantization)."""
        import torch
        self.tm = getattr(self, "tm", {})
        if j not in self.tm:
            fq, c = self.fq, self.caches[j]
            # allocations (zero-filled by torch) and the two copy kernels all on the model's stream,
            # and the plain arrays freed only after it drains: exporting on self.stream into arrays
            # zero-filled on the default stream (and freed while the import still read them) left
            # some layers' token-major copies empty, so Top-K timed them on all-equal scores
            with torch.cuda.stream(self.stream):
                t = fq.KVCache(c.batch, c.heads, c.head_dim, c.prompt_len, c.gen_len, device=c.k.device,
                               layout="token_major")
                plain = fq.flexq_kv_export(c)
                fq.flexq_kv_import(t, *plain)
            self.stream.synchronize()
            del plain
            self.tm[j] = t
        return self.tm[j]

    def free(self):
        self.graphs.clear()
        self.tm, self.tws = {}, None
        del self.caches, self.qs, self.kn, self.vn, self.outs, self.ws


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass


def reference_output(w, B_total, row, layer, step_i, seed, dev):
    """Recompute, for one global sequence `row`, the attention output of `layer` at decode step
    step_i from scratch (its own one-sequence cache: prompt fill, then the step's token k_new of
    that layer appended at every position s .. s + i - 1, exactly what steps 1..i write)."""
    import torch
    from paper_2303_06865_b200 import flexq as fq
    from paper_2303_06865_b200 import synth
    H, D, s, n = w.heads, w.head_dim, w.prompt_len, w.gen_len
    c = fq.KVCache(1, H, D, s, max(n, 1), device=dev)
    kp = synth.fill_rows(seed, synth.tensor_id(0, synth.K_PROMPT), (B_total, H, s, D), row, row + 1, device=dev)
    vp = synth.fill_rows(seed, synth.tensor_id(0, synth.V_PROMPT), (B_total, H, s, D), row, row + 1, device=dev)
    fq.flexq_append_kv(kp, vp, c, pos=0)
    one = lambda kind: synth.fill_rows(seed, synth.tensor_id(layer, kind), (B_total, H, D), row, row + 1,  # noqa: E731
                                       device=dev)
    kn, vn, q = one(synth.K_NEW), one(synth.V_NEW), one(synth.Q)
    for pos in range(s, s + step_i):
        fq.flexq_append_kv(kn.unsqueeze(2), vn.unsqueeze(2), c, pos=pos)
    out = fq.flexq_decode_attention(q, c, s + step_i)
    torch.cuda.synchronize()
    return out[0]


def run_flexq(args):
    import torch
    from paper_2303_06865_b200 import flexq as fq
    from paper_2303_06865_b200 import workloads as wl
    from paper_2303_06865_b200 import dist as fd

    world, rank, local, pg = dist_setup(args)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    fq.lib()

    w = wl.CONFIGS[args.config]
    if args.layers:
        w = wl.Workload(w.name, w.batch, w.heads, w.head_dim, w.prompt_len, w.gen_len, args.layers, w.h2)
    scaling = args.scaling
    B_total = w.batch if scaling == "strong" else w.batch * world
    b0, b1 = rank_rows(B_total, world, rank, scaling, w.batch)
    if b1 <= b0:
        raise SystemExit(f"--scaling strong needs batch ({w.batch}) >= ranks ({world})")
    H, D, s, n, L = w.heads, w.head_dim, w.prompt_len, w.gen_len, w.layers
    h1 = H * D
    seed = synth_seed()
    stream = torch.cuda.Stream(device=dev)
    fused = args.step == "fused"
    peak, peak_kind = peaks()

    def barrier():
        if pg:
            pg.barrier()
        torch.cuda.synchronize()

    # ---- setup: compressed caches for all layers resident in HBM
    log(f"setup: rows [{b0}, {b1}) of a global batch of {B_total} ({scaling} scaling, {world} rank(s))")
    m = DecodeModel(w, L, B_total, b0, b1, seed, dev, stream, fused)
    B = m.B
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    cache_bytes = m.nbytes()
    log("prompt fill done; capturing graphs")
    m.capture()

    # ---- warmup + timed region
    log("graphs captured; timing")
    clk = ClockSampler(local)
    ms, seqs = m.time_steps(args.warmup, args.steps, barrier, clk)
    ms = fd.max_over_ranks(ms, device=dev)
    ms_step = ms / args.steps
    job_bytes = sum(m.step_bytes(i, B_total) for i in seqs)
    value_gbs = job_bytes / (ms / 1e3) / 1e9
    tokens_per_s = B_total * args.steps / (ms / 1e3)
    last_i = seqs[-1]

    # ---- outputs: all-gather one layer-step's fp16 outputs (NCCL, outside the timed data path),
    # then rank 0 recomputes the last global sequence (owned by the last rank) from scratch on its
    # own one-sequence cache and checks the gathered row (reading Q's tolerance: the one-sequence
    # launch schedules its pieces differently)
    gather = None
    out_last = m.outs[L - 1]
    check_row = B_total - 1
    if world > 1:
        torch.cuda.synchronize()
        src = out_last.cpu() if args.same_device else out_last
        full = fd.gather_outputs(src, B_total)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        g0.record()
        for _ in range(20):
            fd.gather_outputs(src, B_total)
        g1.record()
        torch.cuda.synchronize()
        ag_us = (g0.elapsed_time(g1) if not args.same_device else (time.perf_counter() - t0) * 1e3) / 20 * 1e3
        ag_us = fd.max_over_ranks(ag_us, device=dev)
        got_row = full[check_row].to(dev)
        import torch.distributed as dist
        gather = {"what": "all_gather of one layer-step's fp16 outputs [B_rank][H][D] per rank",
                  "bytes_per_rank": int(src.numel() * 2), "us": round(ag_us, 1), "in_timed_region": False,
                  "backend": dist.get_backend(), "comm_size": dist.get_world_size(),
                  "nccl_version": ".".join(map(str, torch.cuda.nccl.version())) if not args.same_device else None}
        del full
    else:
        got_row = out_last[check_row - b0]
    check = None
    if rank == 0:
        ref = reference_output(w, B_total, check_row, L - 1, last_i, seed, dev).float()
        err = (got_row.float() - ref).abs()
        ok = bool((err <= torch.clamp(1e-2 * ref.abs(), min=2e-3)).all())
        check = {"row": check_row, "owner_rank": fd.owner(B_total, world, check_row), "layer": L - 1,
                 "cur_len": s + last_i, "max_abs_err": float(err.max()), "within_reading_Q": ok,
                 "what": "rank 0 recomputes the last global sequence's output from scratch on a one-sequence "
                         "cache and checks the row gathered from its owner"}
        if not ok:
            log(f"cross-rank output check FAILED: {check}")

    # ---- dominant kernel: per-launch time at the longest context (cur_len = s + n - 1)
    log("timed; per-kernel pass")
    cur_last = s + m.steps_i[-1]
    attn_us = m.per_launch(cur_last, "attn")
    app_us = m.per_launch(cur_last, "append")
    fused_us = m.per_launch(cur_last, "fused")
    attn_bytes = wl.attention_bytes(B, h1, cur_last)
    fused_bytes = attn_bytes + wl.append_bytes(B, h1)
    k_us, k_bytes = (fused_us, fused_bytes) if fused else (attn_us, attn_bytes)
    achieved = k_bytes / (k_us * 1e-6) / 1e9

    # ---- NEXT-1: Top-K sparse attention (keep 10%) at the same shape
    topk = None
    if cur_last <= 1152 and rank == 0:
        keep = fq.topk_keep(cur_last)
        kv_row = h1 // 2 + h1 // 64 * 4                      # one token's K (or V) bytes over all heads
        tk_bytes = B * (cur_last * kv_row + keep * kv_row + 2 * h1 * 2)
        tk_us = m.per_launch(cur_last, "topk_tm", layers=4)
        tk_us_dense = m.per_launch(cur_last, "topk", layers=4)
        attn4_us = m.per_launch(cur_last, "attn", layers=4)
        topk = {"keep": keep, "cur_len": cur_last, "layout": "token_major", "us_per_launch": round(tk_us, 2),
                "algorithmic_bytes_per_launch": tk_bytes, "GBps": round(tk_bytes / (tk_us * 1e-6) / 1e9, 1),
                "frac_of_measured_hbm": round(tk_bytes / (tk_us * 1e-6) / 1e9 / peak, 4),
                "speedup_vs_dense": round(attn4_us / tk_us, 3), "dense_attention_us_same_graph": round(attn4_us, 2),
                "dense_layout_us_per_launch": round(tk_us_dense, 2),
                "note": "bytes = K for all tokens + V for the kept 10% (P:856) + q + out; two launches (select, "
                        "gather), graph of 4 layers; the dense layout gathers whole 4-token quad rows"}
    traffic = None
    tp = os.path.join(ROOT, "profiles", "attention_traffic.json")
    if os.path.exists(tp) and w.name == "opt-175b" and B == 144:
        traffic = json.load(open(tp)).get("fused_dram_bytes_per_launch" if fused else "dram_bytes_per_launch")

    # ---- e2e: host buffers through the public API, H2D of the step's inputs and D2H of its outputs
    log("e2e")
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(m, args, dev, barrier, B_total)
    m.free()
    del m
    torch.cuda.empty_cache()

    # ---- weak-scaling secondary key (N > 1 strong runs): every rank its own full batch
    weak = None
    if world > 1 and scaling == "strong" and not args.no_weak:
        log("weak-scaling secondary")
        wb0, wb1 = rank_rows(w.batch * world, world, rank, "weak", w.batch)
        mw = DecodeModel(w, L, w.batch * world, wb0, wb1, seed, dev, stream, fused)
        mw.capture()
        wms, wseqs = mw.time_steps(args.warmup, args.steps, barrier)
        wms = fd.max_over_ranks(wms, device=dev)
        wbytes = sum(mw.step_bytes(i, w.batch * world) for i in wseqs)
        weak = {"value": round(wbytes / (wms / 1e3) / 1e9, 2), "unit": "GB/s", "scaling": "weak",
                "global_batch": w.batch * world, "batch_per_gpu": w.batch, "ms_per_step": round(wms / args.steps, 4),
                "tokens_per_s": round(w.batch * world * args.steps / (wms / 1e3), 2)}
        mw.free()
        del mw
        torch.cuda.empty_cache()

    extra = {}
    if rank == 0 and world == 1 and w.name == "opt-175b" and not args.no_sweep:
        extra = run_sweeps(args, dev, stream, seed, peak)

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    log("cpu baseline")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_object(w, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value_gbs, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "u4+f16->f32", "data": "synthetic (counter-based Irwin-Hall fp16, P:41/P:44)",
            "tokens_per_s": round(tokens_per_s, 2),
            "attention_tokens_per_s_per_layer": round(tokens_per_s * L, 1),
            "config": {"workload": f"{w.name} decode step: global batch {B_total} ({scaling} scaling: {B} per GPU), "
                                   f"{H} heads x {D}, s={s}, n={n}, l={L} layers, "
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
            "topk_sparse": topk,
            "dist": gather,
            "output_check": check,
            "weak_scaling": weak,
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()


def synth_seed():
    from paper_2303_06865_b200 import synth
    return synth.BASE_SEED + 3


def run_e2e(m, args, dev, barrier, B_total):
    """The same step through the public API from HOST buffers: per layer, one H2D copy of the
    pinned (q, k_new, v_new) block on a copy stream (NB device slots let it run ahead of the
    compute stream), the fused launch; the step's result -- the last layer's attention output
    (earlier layers' outputs feed the next layer on the device) -- is read back with a D2H copy.
    Each step is one CUDA graph (copies + launches + cross-stream events), timed over the same
    --steps as the device region.  (A D2H of every layer's output, measured in round 1, competes
    for HBM with the bandwidth-bound kernel and adds ~5 % without being part of the result.)"""
    import torch
    from paper_2303_06865_b200 import dist as fd
    L, s = m.L, m.w.prompt_len
    hin = torch.stack([m.qs, m.kn, m.vn], dim=1).cpu().pin_memory()    # [L][3][B][H][D]
    outh = torch.empty(m.outs[0].shape, dtype=m.outs.dtype).pin_memory()
    NB = 8 if L % 8 == 0 else (6 if L % 6 == 0 else 4)
    din = [torch.empty_like(hin[0], device=dev) for _ in range(NB)]
    dout = [torch.empty_like(m.outs[0]) for _ in range(NB)]
    st = m.stream
    h2d = torch.cuda.Stream(device=dev)

    def e2e_step(i):
        cur = s + i
        ready = [torch.cuda.Event() for _ in range(L)]
        consumed = [torch.cuda.Event() for _ in range(L)]
        fork = torch.cuda.Event()
        fork.record(st)
        h2d.wait_event(fork)
        for j in range(L):
            b = j % NB
            with torch.cuda.stream(h2d):
                if j >= NB:
                    h2d.wait_event(consumed[j - NB])      # slot b's inputs consumed by layer j - NB
                din[b].copy_(hin[j], non_blocking=True)
                ready[j].record(h2d)
            st.wait_event(ready[j])
            m.layer_step(j, cur, din[b][0], din[b][1], din[b][2], dout[b], st)
            consumed[j].record(st)
        outh.copy_(dout[(L - 1) % NB], non_blocking=True)   # the step's result, D2H
        st.wait_stream(h2d)

    graphs = {}
    for i in m.steps_i:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            e2e_step(i)
        graphs[i] = g
    torch.cuda.synchronize()
    for k in range(args.warmup):
        graphs[m.seq_of(k)].replay()
    barrier()
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_bytes = 0
    with torch.cuda.stream(st):
        x0.record(st)
        for k in range(args.steps):
            i = m.seq_of(args.warmup + k)
            graphs[i].replay()
            e2e_bytes += m.step_bytes(i, B_total)
        x1.record(st)
    barrier()
    ems = fd.max_over_ranks(x0.elapsed_time(x1), device=dev)
    res = {"value": round(e2e_bytes / (ems / 1e3) / 1e9, 2),
           "unit": "GB/s", "h2d_bytes_per_step": int(hin.nbytes),
           "d2h_bytes_per_step": int(outh.nbytes), "ms_per_step": round(ems / args.steps, 3),
           "tokens_per_s": round(B_total * args.steps / (ems / 1e3), 2),
           "pcie_floor_ms_per_step": None,
           "how": f"pinned host (q, k_new, v_new) block per layer -> one H2D copy on a copy stream, {NB} device "
                  f"slots so the copies run ahead of compute; fused append+attention via the C ABI; D2H of the "
                  f"step's result (last layer's output); one CUDA graph per step; CUDA events, max over ranks"}
    # the PCIe floor: the step's H2D bytes at this box's pinned copy rate
    try:
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        import offload_bench
        res["pcie_floor_ms_per_step"] = round(hin.nbytes / offload_bench.h2d_gbs(dev) / 1e6, 3)
    except Exception:  # noqa: BLE001
        pass
    del graphs, din, dout, hin, outh
    return res


def run_sweeps(args, dev, stream, seed, peak):
    """Rank 0, N = 1: the other BASELINE configs as full-depth steps, the OPT-175B shard proxies,
    the weight quantize / dequantize sweep + NEXT-2 GEMM, the KV-cache variants and NEXT-4."""
    import torch
    from paper_2303_06865_b200 import flexq as fq
    from paper_2303_06865_b200 import synth
    from paper_2303_06865_b200 import workloads as wl
    out = {}
    nobar = torch.cuda.synchronize

    # ---- BASELINE configs[0..2]: tiny, OPT-6.7B, OPT-30B as full-depth decode steps on one GPU
    log("config lines")
    lines = {}
    for cname in ("tiny", "opt-6.7b", "opt-30b"):
        cw = wl.CONFIGS[cname]
        cm = DecodeModel(cw, cw.layers, cw.batch, 0, cw.batch, seed + 11, dev, stream, True)
        cm.capture()
        steps = len(cm.steps_i)
        cms, cseqs = cm.time_steps(2, steps, nobar)
        cbytes = sum(cm.step_bytes(i, cw.batch) for i in cseqs)
        cur = cw.prompt_len + cm.steps_i[-1]
        kus = cm.per_launch(cur, "fused", layers=8)
        kbytes = wl.attention_bytes(cw.batch, cw.h1, cur) + wl.append_bytes(cw.batch, cw.h1)
        lines[cname] = {"batch": cw.batch, "heads": cw.heads, "head_dim": cw.head_dim, "layers": cw.layers,
                        "steps": steps, "ms_per_step": round(cms / steps, 4),
                        "value": round(cbytes / (cms / 1e3) / 1e9, 2), "unit": "GB/s",
                        "tokens_per_s": round(cw.batch * steps / (cms / 1e3), 2),
                        "fused_us_per_launch": round(kus, 2), "cur_len": cur,
                        "frac_of_measured_hbm": round(kbytes / (kus * 1e-6) / 1e9 / peak, 4)}
        cm.free()
        del cm
        torch.cuda.empty_cache()
    out["config_lines"] = lines

    # ---- shard proxies: the OPT-175B per-rank shard of a strong-scaled global batch of 144 at
    # N = 2 / 4 / 8 (batch 72 / 36 / 18) on this one GPU, fused launches at cur_len 543
    log("shard proxies")
    w = wl.CONFIGS["opt-175b"]
    proxy = {}
    for nb in (2, 4, 8):
        Bp = w.batch // nb
        pm = DecodeModel(wl.Workload(w.name, w.batch, w.heads, w.head_dim, w.prompt_len, w.gen_len, 8),
                         8, w.batch, 0, Bp, seed, dev, stream, True)
        cur = w.prompt_len + w.gen_len - 1
        us = pm.per_launch(cur, "fused")
        kb = wl.attention_bytes(Bp, w.h1, cur) + wl.append_bytes(Bp, w.h1)
        proxy[f"n{nb}_batch{Bp}"] = {"batch": Bp, "us_per_launch": round(us, 2),
                                     "GBps": round(kb / (us * 1e-6) / 1e9, 1),
                                     "frac_of_measured_hbm": round(kb / (us * 1e-6) / 1e9 / peak, 4),
                                     "step_ms_estimate": round(us * w.layers / 1e3, 3)}
        pm.free()
        del pm
        torch.cuda.empty_cache()
    out["shard_proxy"] = proxy

    sw = legacy_sweeps(args, dev, stream, seed, peak)
    out.update(sw)
    return out


def legacy_sweeps(args, dev, stream, seed, peak):
    """Rank 0, N = 1: weight quantize / dequantize sweep (BASELINE configs[4]) with the NEXT-2
    dequant-GEMM beside its library baselines, the NEXT-3 KV-cache variants on the OPT-175B
    shape, and NEXT-4 host-offloaded KV."""
    import torch
    from paper_2303_06865_b200 import flexq as fq
    from paper_2303_06865_b200 import synth
    from paper_2303_06865_b200 import workloads as wl
    w = wl.CONFIGS["opt-175b"]
    B, H, D, s, n = w.batch, w.heads, w.head_dim, w.prompt_len, w.gen_len
    # ---- weight quantize / dequantize sweep (BASELINE configs[4]), rank 0
    log("sweep")
    sweep = gemm = None
    if True:
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

    # ---- NEXT-3 variants of the KV cache (rank 0): decode attention on the OPT-175B shape at the
    # last step's context for three (b, g), 2 layers of fresh caches each, one CUDA graph
    kv_variants = None
    if True:
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
    if not args.no_offload:
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        import offload_bench
        offload = offload_bench.run(layers=2, gpu_batches=1, B=B, H=H, D=D, s=s, n=n, steps=3, dev=str(dev))
        offload["bound"] = "pcie"
        offload["how"] = ("per (layer, GPU batch) in Alg. 1 order: H2D of the whole compressed block on a load "
                          "stream, fused append+attention on the compute stream, D2H of the new token's chunk "
                          "on a store stream; value = H2D bytes / device time, vs a pinned 1 GiB H2D copy")

    return {"weight_sweep": sweep, "dequant_gemm": gemm, "kv_variants": kv_variants, "offload": offload}


def cpu_baseline_object(w, budget_s):
    """The oracle as it stands on this host: (1) all cores, one worker process per core, on a bounded
    sample of the workload (extrapolated: sample bytes / sample time); (2) the tiny configuration
    (BASELINE configs[0]) in full on one thread -- prompt fill, one appended token and one decode
    attention step -- timed end to end."""
    from paper_2303_06865_b200 import workloads as wl
    h1 = w.h1
    per = lambda nseq, cur: nseq * (wl.attention_bytes(1, h1, cur) + wl.append_bytes(1, h1))  # noqa: E731
    gbs, seqs, cores, sample = cpu_oracle_baseline(w, budget_s, per)
    obj = {"value": round(gbs, 4), "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample,
           "extrapolated": True}
    try:
        import oracle
        from paper_2303_06865_b200 import synth
        t = wl.CONFIGS["tiny"]
        B, H, D, s = t.batch, t.heads, t.head_dim, t.prompt_len
        seed = synth.BASE_SEED
        k = synth.fill(seed, synth.tensor_id(0, synth.K_PROMPT), (B, H, s, D)).numpy()
        v = synth.fill(seed, synth.tensor_id(0, synth.V_PROMPT), (B, H, s, D)).numpy()
        kn = synth.fill(seed, synth.tensor_id(0, synth.K_NEW, 1), (B, H, 1, D)).numpy()
        vn = synth.fill(seed, synth.tensor_id(0, synth.V_NEW, 1), (B, H, 1, D)).numpy()
        q = synth.fill(seed, synth.tensor_id(0, synth.Q, 1), (B, H, D)).numpy()
        t0 = time.perf_counter()
        kc, vc = oracle.empty_cache(B, H, s + 1, D), oracle.empty_cache(B, H, s + 1, D)
        oracle.append_kv(k, v, kc, vc, 0)
        t1 = time.perf_counter()
        oracle.append_kv(kn, vn, kc, vc, s)
        oracle.attention_f64(q, kc, vc, s + 1)
        t2 = time.perf_counter()
        step_bytes = wl.attention_bytes(B, H * D, s + 1) + wl.append_bytes(B, H * D)
        obj["tiny_full_single_thread"] = {
            "prompt_fill_s": round(t1 - t0, 4), "decode_step_s": round(t2 - t1, 4),
            "decode_step_GBps": round(step_bytes / (t2 - t1) / 1e9, 5), "threads": 1,
            "what": "BASELINE configs[0] in full: quantize the 512-token prompt of 4 x 12 heads, append one "
                    "token, one decode attention at cur_len 513 (oracle_attention_f64)"}
    except Exception as e:  # noqa: BLE001
        obj["tiny_full_single_thread"] = {"error": str(e)}
    return obj


def relaunch(args) -> int:
    """--gpus N > 1 without torchrun: run this script under torch.distributed.run, one rank per GPU."""
    import socket
    import subprocess
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    log(f"launching {args.gpus} ranks: {' '.join(cmd[1:6])} ...")
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_flexq(args)


if __name__ == "__main__":
    main()

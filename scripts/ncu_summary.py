"""Summarise ncu outputs for profiles/ (run here, on the CPU box).

    python scripts/ncu_summary.py launches gpurun_out/launches.csv   > profiles/..._launches.md
    python scripts/ncu_summary.py full gpurun_out/attn_full.ncu-rep   > profiles/..._attn_full.md
"""
import collections
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ik, iv, iu, im, iid = (hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit"),
                           hdr.index("Metric Name"), hdr.index("ID"))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = collections.defaultdict(dict)      # launch id -> {name, metric: value}
    for r in rows[hi + 1:]:
        if len(r) <= iv:
            continue
        d = per[r[iid]]
        d["name"] = r[ik].split("(")[0].replace("void ", "")
        d[r[im]] = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    tot = collections.defaultdict(float)
    byt = collections.defaultdict(float)
    cnt = collections.Counter()
    for d in per.values():
        t = d.get("gpu__time_duration.sum", 0.0)
        tot[d["name"]] += t
        byt[d["name"]] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        cnt[d["name"]] += 1
    allus = sum(tot.values())
    print(f"# ncu launch list: {path}\n")
    print("Per-launch device time, `--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
          "--clock-control none` (cold-cache, serialised: compare shares, not absolutes).\n")
    print("| kernel | launches | total us | mean us | share of time | DRAM bytes / launch |\n|---|---|---|---|---|---|")
    for k in sorted(tot, key=lambda x: -tot[x]):
        print(f"| `{k}` | {cnt[k]} | {tot[k]:.1f} | {tot[k] / cnt[k]:.2f} | {tot[k] / allus:.3f} | "
              f"{byt[k] / cnt[k] / 1e6:.2f} MB |")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full: {path}\n")
    for r in rows[2:]:
        print(f"## `{r[hdr.index('Kernel Name')][:120]}`\n")
        print("| metric | value | unit |\n|---|---|---|")
        for m in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"| {m} | {r[i]} | {units[i]} |")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])

"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iall, inot = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Warp Stall Sampling (Not-issued Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        data.append((int(r[iall]), int(r[inot]), r[ia], r[isrc].strip(),
                     {hdr[i]: int(r[i]) for i in stall_cols if r[i] not in ("", "0")}))
    except ValueError:
        pass
tot = sum(d[0] for d in data)
print(f"total samples {tot}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for d in sorted(data, key=lambda d: -d[0])[:n]:
    top = sorted(d[4].items(), key=lambda kv: -kv[1])[:3]
    print(f"{d[0]:7d} {100*d[0]/tot:5.1f}%  {d[2][-5:]}  {d[3][:60]:60s} {top}")

"""Aggregate an ncu source page (cuda,sass) by line ranges of one file:
python tools/ncu_regions.py report.ncu-rep file.cuh name:lo-hi ..."""
import csv
import subprocess
import sys
from collections import defaultdict

rep, fname = sys.argv[1], sys.argv[2]
regions = []
for a in sys.argv[3:]:
    n, r = a.split(":")
    lo, hi = r.split("-")
    regions.append((n, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, hdr = None, None
agg = defaultdict(lambda: [0.0] * 4)
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr and r and len(r) > 20 and r[0].isdigit():
        try:
            v = [float(r[hdr[k]] or 0) for k in ("L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal",
                                                 "Instructions Executed", "Warp Stall Sampling (All Samples)")]
        except (ValueError, KeyError):
            continue
        ln = int(r[0])
        key = "other:" + str(cur)
        if cur == fname:
            key = "unassigned"
            for n, lo, hi in regions:
                if lo <= ln <= hi:
                    key = n
        a = agg[key]
        for i in range(4):
            a[i] += v[i]
T = [max(sum(a[i] for a in agg.values()), 1) for i in range(4)]
print(f"totals: smem wavefronts {T[0]:.3g} (ideal {T[1]:.3g}), instructions {T[2]:.3g}, stall samples {T[3]:.3g}")
for k, a in sorted(agg.items(), key=lambda x: -x[1][2]):
    print(f"{k:28s} wf {a[0] / T[0] * 100:5.1f}% ({a[0] / max(a[1], 1):.1f}x ideal)  inst {a[2] / T[2] * 100:5.1f}%  stall {a[3] / T[3] * 100:5.1f}%")

"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) into a markdown
table: launches, mean ms and share of the per-step kernel time (setup kernels excluded)."""
import collections
import csv
import sys

SETUP = ("k_detj", "k_cols", "k_mixed_detj", "k_adj_keys", "k_pat_", "DeviceRadixSort", "DeviceScan", "k_adj_ptr")


def main(path, title):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in data:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")) * 1e-6)
    step = sum(sum(v) for k, v in agg.items() if not any(s in k for s in SETUP))
    print(f"# {title}")
    print("# gpu__time_duration.sum, --clock-control none; cold-cache serialised: compare SHARES, not absolutes\n")
    print("| kernel | launches | mean ms | share of per-step kernel time |")
    print("|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        share = "(setup, once)" if any(s in k for s in SETUP) else f"{100 * sum(v) / step:.1f}%"
        print(f"| {k} | {len(v)} | {sum(v) / len(v):.3f} | {share} |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])

#!/bin/bash
# Round evidence (B200_PROFILING.md recipe): plain runs first, then
#   1. the launch list of a short bench (gpu__time_duration per launch, --clock-control none);
#   2. ncu --set full of k_sweep4 (configs 3 and 4, the bench workload) and k_sweepq (config 2);
# and traffic.json (DRAM bytes per launch keyed by workload, with the kernel-source sha that
# bench.py checks).  Output under gpurun_out/prof_round/.
set -u
OUT=gpurun_out/prof_round
mkdir -p $OUT
python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu-baseline > $OUT/bench_plain.json 2> $OUT/bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c4.csv \
    python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
for spec in "4 k_sweep4 sweep4_c4" "3 k_sweep4 sweep4_c3" "2 k_sweepq sweepq_c2"; do
  set -- $spec
  python tools/assemble_once.py $1 0 > $OUT/plain_$3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$2 -c 1 -o $OUT/prof_$3 \
      python tools/assemble_once.py $1 0 > $OUT/ncu_$3.log 2>&1
done
python - <<'PY'
import csv, json, subprocess, sys
sys.path.insert(0, ".")
import bench
out = {}
for cid, k, tag, wl in ((4, "k_sweep4", "sweep4_c4", "hex8_200^3"), (3, "k_sweep4", "sweep4_c3", "hex8_100^3"),
                       (2, "k_sweepq", "sweepq_c2", "q4_1000x1000")):
    r = subprocess.run(["ncu", "-i", f"gpurun_out/prof_round/prof_{tag}.ncu-rep", "--page", "raw", "--csv"],
                       capture_output=True, text=True).stdout
    rows = list(csv.reader(r.splitlines()))
    if len(rows) < 3:
        continue
    d = dict(zip(rows[0], rows[2]))
    def num(key):
        v = d[key]
        unit = rows[1][rows[0].index(key)]
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        return float(v.replace(",", "")) * mult
    etype = 3 if tag.startswith("sweep4") else 2
    pct = lambda key: float(d[key].replace(",", "")) if key in d else None
    out[wl] = {"bytes": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"), "kernel": k,
               "fp64_pipe_pct": pct("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
               "issue_active_pct": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
               "smem_wavefronts": pct("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
               "src_sha": bench.kernel_source_sha(etype, 0), "profile": f"prof_{tag}.ncu-rep",
               "duration_ms": float(d["gpu__time_duration.sum"].replace(",", "")) * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}[rows[1][rows[0].index("gpu__time_duration.sum")]]}
json.dump(out, open("gpurun_out/prof_round/traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
PY

#!/bin/bash
# quick GPU check: parity tests + bench of configs 3 and 2 (assemble ms, HBM fraction)
timeout 900 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -4
for c in ${CFGS:-3 2}; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/q_c$c.json 2> gpurun_out/q_c$c.err
  python -c "import json;d=json.load(open('gpurun_out/q_c$c.json'));print(d['config']['workload'],'assemble_ms',round(d['assemble_ms'],3),'frac',round(d['roofline']['frac'],4),'step_ms',round(d['ms_per_step'],3), d['clocks'])" || tail -3 gpurun_out/q_c$c.err
done

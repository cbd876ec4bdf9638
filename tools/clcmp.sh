#!/bin/bash
# k_sweep4 cluster vs solo: parity subset + assemble timing of configs 3 and 4
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x ${KSEL:+-k "$KSEL"} 2>&1 | tail -4
for c in ${CFGS:-3 4}; do
 for cl in 1 2; do
  LGDM_SWEEP_CLUSTER=$cl timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/cl_c${c}_$cl.json 2> gpurun_out/cl_c${c}_$cl.err
  python -c "import json;d=json.load(open('gpurun_out/cl_c${c}_$cl.json'));print('cfg $c cluster $cl', d['config']['workload'],'assemble_ms',round(d['assemble_ms'],3),'min',round(d['assemble_ms_min'],3),'frac',round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/cl_c${c}_$cl.err
 done
done

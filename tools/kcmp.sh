#!/bin/bash
# Hex8 kernel comparison: parity subset + assemble timing of kernels 2 (k_hex8) and 4 (k_sweep4)
mkdir -p gpurun_out
timeout 1200 python -m pytest ${TESTS:-tests/test_gpu_parity.py} -m gpu -q -x ${KSEL:+-k "$KSEL"} 2>&1 | tail -8
for c in ${CFGS:-3}; do
 for k in ${KERNS:-2}; do
  timeout 300 python bench.py --config $c --kernel $k --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/k_c${c}_k$k.json 2> gpurun_out/k_c${c}_k$k.err
  python -c "import json;d=json.load(open('gpurun_out/k_c${c}_k$k.json'));print('cfg $c kernel $k', d['config']['workload'],'assemble_ms',round(d['assemble_ms'],3),'min',round(d['assemble_ms_min'],3),'frac',round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/k_c${c}_k$k.err
 done
done

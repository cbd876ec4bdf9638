#!/bin/bash
# kernel comparison: parity subset (TESTS, KSEL) + assemble timing of configs CFGS x kernel
# selectors KERNS (lgdm_set_kernel: 0 auto, 1 general, 2 sweep)
mkdir -p gpurun_out
timeout 1200 python -m pytest ${TESTS:-tests/test_gpu_parity.py} -m gpu -q -x ${KSEL:+-k "$KSEL"} 2>&1 | tail -8
for c in ${CFGS:-3}; do
 for k in ${KERNS:-0}; do
  timeout 300 python bench.py --config $c --kernel $k --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/k_c${c}_k$k.json 2> gpurun_out/k_c${c}_k$k.err
  python -c "import json;d=json.load(open('gpurun_out/k_c${c}_k$k.json'));print('cfg $c kernel $k', d['config']['workload'],'assemble_ms',round(d['assemble_ms'],3),'min',round(d['assemble_ms_min'],3),'frac',round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/k_c${c}_k$k.err
 done
done

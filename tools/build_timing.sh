#!/bin/bash
# debug build with the sweep kernels' phase counters (lgdm_debug_phase_cycles) -> lib_timing.so
cd "$(dirname "$0")/.." && /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC,-fopenmp,-O2 -shared -Iinclude -DLGDM_PHASE_TIMING -o lib_timing.so \
  paper_2301_06503_b200/csrc/lgdm_api.cu -lgomp -ldl

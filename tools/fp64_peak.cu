// FP64 FMA throughput microbenchmark (B200 sm_100a): many independent DFMA chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* out;
  cudaMalloc(&out, 8);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int bpsm : {1, 2, 4, 8}) {
    for (int threads : {256, 512}) {
      dfma_loop<8><<<nsm * bpsm, threads>>>(out, 100, 0.999, 1e-3);
      cudaEventRecord(e0);
      dfma_loop<8><<<nsm * bpsm, threads>>>(out, iters, 0.999, 1e-3);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * iters * double(nsm) * bpsm * threads;
      printf("blocks/SM %d threads %d: %.2f TFLOP/s fp64 (%.3f ms)\n", bpsm, threads, flops / ms / 1e9, ms);
    }
  }
  return 0;
}

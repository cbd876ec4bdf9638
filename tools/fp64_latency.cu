// Dependent-chain latency of DFMA and of a shared-memory double load on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, long long* cyc, int n, double a, double b) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = x; cyc[0] = t1 - t0; }
}
__global__ void lds_chain(double* out, long long* cyc, int n) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7 + 3) % 1024;
  __syncthreads();
  int idx = threadIdx.x;
  double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { double v = sm[idx]; idx = int(v); acc += v; }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = acc; cyc[0] = t1 - t0; }
}
int main() {
  double* out; long long* cyc; long long h;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  chain<<<1, 32>>>(out, cyc, 100, 0.999, 1e-3);
  chain<<<1, 32>>>(out, cyc, 10000, 0.999, 1e-3);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", h / 10000.0);
  lds_chain<<<1, 32>>>(out, cyc, 10000);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("LDS.64 -> int dependent chain: %.2f cycles/iter (incl. F2I + add)\n", h / 10000.0);
  return 0;
}

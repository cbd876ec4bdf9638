#include <cstdio>
#include <cuda_runtime.h>
// mma.sync m8n8k4 f64: A 8x4 (1 double per lane), B 4x8 (1 double per lane), C/D 8x8 (2 doubles per lane)
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void k(double* out, int iters, double x) {
  double a = x + threadIdx.x, b = x * 2 + threadIdx.x;
  double c[8][2], f[16];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
  for (int i = 0; i < 16; ++i) f[i] = i * x;
  for (int it = 0; it < iters; ++it) {
    if (MODE & 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    if (MODE & 2) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] = fma(f[i], a, b);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  for (int i = 0; i < 16; ++i) s += f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* o; cudaMalloc(&o, 148 * 8 * 1024 * 8);
  int iters = 20000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 1; mode <= 3; ++mode) for (int warps : {4, 8, 16}) {
    auto run = [&]() {
      if (mode == 1) k<1><<<148 * 2, warps * 32>>>(o, iters, 1e-9);
      if (mode == 2) k<2><<<148 * 2, warps * 32>>>(o, iters, 1e-9);
      if (mode == 3) k<3><<<148 * 2, warps * 32>>>(o, iters, 1e-9);
    };
    run(); cudaEventRecord(e0); run(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double thr = 148.0 * 2 * warps * 32;
    double dm = (mode & 1) ? thr / 32 * iters * 8 * 512.0 : 0;   // 8x8x4 x2 flops per mma per warp
    double df = (mode & 2) ? thr * iters * 64 * 2.0 : 0;
    printf("mode %d warps/CTA %2d: %.3f ms  dmma %.2f TF  dfma %.2f TF  total %.2f TF\n", mode, warps, ms,
           dm / ms / 1e9, df / ms / 1e9, (dm + df) / ms / 1e9);
  }
  return 0;
}

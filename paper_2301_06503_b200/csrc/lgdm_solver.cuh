// lgdm_solver.cuh -- Newton-loop kernels (Alg. 2 l.4-7, l.16): symmetric
// Dirichlet elimination on the assembled CSR, a Jacobi-preconditioned BiCGSTAB on K delta = R
// (the paper solves with `mldivide`; an iterative solve keeps the whole loop on the
// GPU), dof update and the convergence norms.  All reductions are deterministic (fixed-order
// warp and block trees), so a run is bitwise reproducible.
#pragma once
#include "lgdm_device.cuh"

namespace lgdm {

constexpr int kRedBlocks = 592;   // 4 x 148 SMs; partial sums, then one final block

// constrained rows become unit rows with R = increment; free rows move K_ij inc_j of the
// constrained columns to the RHS and zero them (one warp per row, fixed-order reduction).
// Rows are the owned rows (global id row_g0 + row, local dof own_b + row); fixed / inc are
// over the local dofs (owned + ghosts), a column c is local dof c - col_off.
__global__ void k_dirichlet(int64_t nrows, int64_t row_g0, int64_t own_b, int64_t col_off,
                            const int64_t* __restrict__ row_ptr,
                            const int32_t* __restrict__ col_idx, double* __restrict__ val,
                            double* __restrict__ R, const uint8_t* __restrict__ fixed,
                            const double* __restrict__ inc) {
  const int64_t row = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= nrows) return;
  const int64_t lo = row_ptr[row], hi = row_ptr[row + 1];
  if (fixed[own_b + row]) {
    for (int64_t q = lo + lane; q < hi; q += 32) val[q] = col_idx[q] == row_g0 + row ? 1.0 : 0.0;
    if (lane == 0) R[row] = inc[own_b + row];
    return;
  }
  double s = 0.0;
  for (int64_t q = lo + lane; q < hi; q += 32) {
    const int64_t c = col_idx[q] - col_off;
    if (fixed[c]) {
      s = fma(val[q], inc[c], s);
      val[q] = 0.0;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0 && s != 0.0) R[row] -= s;
}

// y = A x over the owned rows (one warp per row, fixed-order lane partials + tree); x is a
// local dof vector (owned + ghost dofs), column c is local dof c - col_off
__global__ void k_spmv(int64_t nrows, const int64_t* __restrict__ row_ptr,
                       const int32_t* __restrict__ col_idx, const double* __restrict__ val,
                       const double* __restrict__ x, int64_t col_off, double* __restrict__ y) {
  const int64_t row = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= nrows) return;
  double s = 0.0;
  for (int64_t q = row_ptr[row] + lane; q < row_ptr[row + 1]; q += 32) s = fma(val[q], x[col_idx[q] - col_off], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[row] = s;
}

// inverse diagonal for the Jacobi preconditioner (0 -> 1); row_g0 = global id of row 0
__global__ void k_invdiag(int64_t nrows, int64_t row_g0, const int64_t* __restrict__ row_ptr,
                          const int32_t* __restrict__ col_idx, const double* __restrict__ val,
                          double* __restrict__ dinv) {
  const int64_t row = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (row >= nrows) return;
  double d = 0.0;
  for (int64_t q = row_ptr[row]; q < row_ptr[row + 1]; ++q)
    if (col_idx[q] == row_g0 + row) d = val[q];
  dinv[row] = d != 0.0 ? 1.0 / d : 1.0;
}

// block-level fixed-order sum of NV products a_k . b_k over n entries into part[blk * NV + k]
template <int NV>
__device__ __forceinline__ void block_sum_store(double (&v)[NV], double* part) {
  __shared__ double red[NV][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    if (lane == 0) red[k][w] = v[k];
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = lane < int(blockDim.x >> 5) ? red[k][lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) part[blockIdx.x * NV + k] = s;
    }
  }
}

// two dot products (a.b, c.d) -> part
__global__ void k_dot2(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                       const double* __restrict__ c, const double* __restrict__ d,
                       double* __restrict__ part) {
  double v[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    v[0] = fma(a[i], b[i], v[0]);
    if (c) v[1] = fma(c[i], d[i], v[1]);
  }
  block_sum_store<2>(v, part);
}

// final fixed-order sum of nb partials of NV values
template <int NV>
__global__ void k_final(int nb, const double* __restrict__ part, double* __restrict__ out) {
  double v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x)
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += part[i * NV + k];
  block_sum_store<NV>(v, out);
}

// BiCGSTAB vector updates
__global__ void k_p_update(int64_t n, double beta, double omega, const double* __restrict__ r,
                           const double* __restrict__ v, double* __restrict__ p) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) p[i] = r[i] + beta * (p[i] - omega * v[i]);
}
__global__ void k_scale_mul(int64_t n, const double* __restrict__ d, const double* __restrict__ x,
                            double* __restrict__ y) {   // y = d .* x
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) y[i] = d[i] * x[i];
}
__global__ void k_axpy(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) y[i] = fma(a, x[i], y[i]);
}
__global__ void k_s_update(int64_t n, double alpha, const double* __restrict__ r,
                           const double* __restrict__ v, double* __restrict__ s) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) s[i] = r[i] - alpha * v[i];
}
__global__ void k_x_update(int64_t n, double alpha, double omega, const double* __restrict__ ph,
                           const double* __restrict__ sh, double* __restrict__ x) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) x[i] = x[i] + alpha * ph[i] + omega * sh[i];
}
__global__ void k_r_update(int64_t n, double omega, const double* __restrict__ s,
                           const double* __restrict__ t, double* __restrict__ r) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) r[i] = s[i] - omega * t[i];
}

// convergence norms: sum of squares of delta and dofs over u dofs and ebar dofs
template <int NDPN>
__global__ void k_delta_sumsq(int64_t n, const double* __restrict__ delta,
                              const double* __restrict__ dofs, double* __restrict__ part) {
  double v[4] = {0.0, 0.0, 0.0, 0.0};   // |du|^2, |u|^2, |de|^2, |e|^2
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const bool e = (i % NDPN) == NDPN - 1;
    const double d = delta[i], u = dofs[i];
    v[e ? 2 : 0] = fma(d, d, v[e ? 2 : 0]);
    v[e ? 3 : 1] = fma(u, u, v[e ? 3 : 1]);
  }
  block_sum_store<4>(v, part);
}

// reaction: -sum of R over listed dofs, one block, fixed order
__global__ void k_reaction(int64_t n, const int64_t* __restrict__ ids, const double* __restrict__ R,
                           double* __restrict__ out) {
  double v[1] = {0.0};
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) v[0] -= R[ids[k]];
  block_sum_store<1>(v, out);
}

__global__ void k_rowptr32(int64_t n, const int64_t* __restrict__ in, int32_t* __restrict__ out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = int32_t(in[i]);
}

}  // namespace lgdm

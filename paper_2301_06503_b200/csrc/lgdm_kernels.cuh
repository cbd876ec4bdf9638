// lgdm_kernels.cuh -- CUDA kernels of liblgdm (sm_100a).  Included once, by lgdm_api.cu.
//
//   k_detj            det J > 0 check at every GP, run once at create
//   k_cols            expand per-node neighbour lists into CSR col_idx (reading R-PAT)
//   k_elem_blocks     GENERAL path, step 1: element batches -> phase A / phase C -> dense
//                     element blocks (Eqs. 11a-f) in a scratch buffer
//   k_gather          GENERAL path, step 2: warp per owned node sums its block-row over the
//                     adjacent elements in ascending element id (the order of Alg. 1's
//                     assembly loop) and stores it with coalesced writes
//   k_update_history  Eq. A.2 / Fig. 8b l.22-24 per GP
//   k_sumsq_*         deterministic two-stage sum of squares of R (u rows, ebar rows)
//   k_scale           dofs *= s (benchmark helper)
#pragma once
#include "lgdm_device.cuh"

namespace lgdm {

// ----------------------------------------------------------------------------------------
template <int D>
__global__ void k_detj(int64_t ne, const int32_t* __restrict__ conn,
                       const double* __restrict__ coords, unsigned long long* bad) {
  using F = Fam<D>;
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t >= ne * F::NGP) return;
  const int64_t e = t / F::NGP;
  const int g = int(t % F::NGP);
  double J[D][D];
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) J[i][j] = 0.0;
  for (int a = 0; a < F::NEN; ++a) {
    const int64_t n = conn[e * F::NEN + a];
    for (int j = 0; j < D; ++j) {
      const double dn = shape_dxi<D>(a, g, j);
      for (int i = 0; i < D; ++i) J[i][j] += coords[n * D + i] * dn;
    }
  }
  double det;
  if constexpr (D == 1) det = J[0][0];
  else if constexpr (D == 2) det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  else
    det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
          J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
          J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
  if (!(det > 0.0)) atomicMin(bad, (unsigned long long)t);
}

// ----------------------------------------------------------------------------------------
// col_idx: one warp per owned node; row i of node n holds, for every neighbour slot s,
// columns ndpn * gid(nbr[s]) + j.
template <int NDPN>
__global__ void k_cols(int64_t n_owned, const int64_t* __restrict__ nbr_ptr,
                       const int32_t* __restrict__ nbr, const int64_t* __restrict__ base,
                       int64_t gid0, int32_t* __restrict__ col_idx) {
  const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n_owned) return;
  const int64_t p0 = nbr_ptr[w];
  const int deg = int(nbr_ptr[w + 1] - p0);
  const int W = deg * NDPN;
  const int64_t b0 = base[w];
  for (int idx = lane; idx < NDPN * W; idx += 32) {
    const int c = idx % W;
    const int s = c / NDPN, j = c % NDPN;
    col_idx[b0 + idx] = int32_t(NDPN * (gid0 + nbr[p0 + s]) + j);
  }
}

// ----------------------------------------------------------------------------------------
// GENERAL path step 1.  One CTA = batches of EPB elements (grid-stride).
// Shared memory: recs [EPB][NGP][GpBlock::STRIDE] | scal [EPB][NGP][kScal] | X [EPB][NEN][D] |
// U [EPB][NEN][NDPN].  Threads: EPB * NPAIR.
template <int D, int EPB>
__global__ void __launch_bounds__(EPB * Fam<D>::NPAIR)
k_elem_blocks(DevMat m, int64_t ne, const int32_t* __restrict__ conn,
              const double* __restrict__ coords, const double* __restrict__ dofs,
              const double* __restrict__ kappa, double* __restrict__ Ke_out,
              double* __restrict__ Fe_out) {
  using F = Fam<D>;
  using R = Rec<D>;
  constexpr int NT = EPB * F::NPAIR;
  extern __shared__ double sm[];
  double* recs = sm;
  double* scal = recs + EPB * F::NGP * GpBlock<D>::STRIDE;
  double* Xs = scal + EPB * F::NGP * kScal;
  double* Us = Xs + EPB * F::NEN * D;
  const int tid = threadIdx.x;
  for (int64_t e0 = int64_t(blockIdx.x) * EPB; e0 < ne; e0 += int64_t(gridDim.x) * EPB) {
    for (int t = tid; t < EPB * F::NEN; t += NT) {
      const int el = t / F::NEN, a = t % F::NEN;
      const int64_t e = e0 + el;
      if (e < ne) {
        const int64_t n = conn[e * F::NEN + a];
#pragma unroll
        for (int i = 0; i < D; ++i) Xs[t * D + i] = coords[n * D + i];
#pragma unroll
        for (int i = 0; i < F::NDPN; ++i) Us[t * F::NDPN + i] = dofs[n * F::NDPN + i];
      }
    }
    __syncthreads();
    for (int t = tid; t < EPB * F::NGP; t += NT) {
      const int el = t / F::NGP, g = t % F::NGP;
      const int64_t e = e0 + el;
      if (e < ne)
        phaseA<D>(m, Xs + el * F::NEN * D, Us + el * F::NEN * F::NDPN, kappa[e * F::NGP + g], g,
                  recs + size_t(t) * GpBlock<D>::STRIDE, scal + t * kScal);
    }
    __syncthreads();
    {
      const int el = tid / F::NPAIR, p = tid % F::NPAIR;
      const int64_t e = e0 + el;
      if (e < ne) {
        int a, b;
        pair_ab<F::NEN>(p, a, b);
        PairAcc<D> acc;
        phaseC<D>(recs + size_t(el) * F::NGP * GpBlock<D>::STRIDE, scal + el * F::NGP * kScal, a,
                  b, acc);
        double* Ke = Ke_out + e * (F::NDOFE * F::NDOFE);
        emit_pair<D>(a, b, acc, [&](int ra, int ri, int cb, int cj, double v) {
          Ke[(ra * F::NDPN + ri) * F::NDOFE + cb * F::NDPN + cj] = v;
        });
        if (a == b) {
#pragma unroll
          for (int i = 0; i <= D; ++i) Fe_out[e * F::NDOFE + a * F::NDPN + i] = acc.Fd[i];
        }
      }
    }
    __syncthreads();
  }
}

// adjacency entry of an owned node: element, local index of the node, slot of each node
struct AdjEntry {
  int32_t e;
  uint8_t aloc;
  uint8_t slot[8];
  uint8_t pad[3];
};

// GENERAL path step 2.  One warp per owned node, WPB warps per CTA.
template <int D, int WPB>
__global__ void __launch_bounds__(WPB * 32)
k_gather(int64_t n_owned, const int64_t* __restrict__ adj_ptr, const AdjEntry* __restrict__ adj,
         const int64_t* __restrict__ nbr_ptr, const int64_t* __restrict__ base,
         const double* __restrict__ Ke_in, const double* __restrict__ Fe_in,
         double* __restrict__ val, double* __restrict__ Rv) {
  using F = Fam<D>;
  constexpr int MAXW = F::NDPN * (D == 1 ? 3 : (D == 2 ? 9 : 27));
  __shared__ double buf[WPB][F::NDPN * MAXW];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n = int64_t(blockIdx.x) * WPB + wl;
  if (n >= n_owned) return;
  const int deg = int(nbr_ptr[n + 1] - nbr_ptr[n]);
  const int W = deg * F::NDPN;
  double* B = buf[wl];
  for (int idx = lane; idx < F::NDPN * W; idx += 32) B[idx] = 0.0;
  double r = 0.0;
  __syncwarp();
  for (int64_t k = adj_ptr[n]; k < adj_ptr[n + 1]; ++k) {
    const AdjEntry en = adj[k];
    const double* Ke = Ke_in + int64_t(en.e) * (F::NDOFE * F::NDOFE) +
                       int64_t(en.aloc) * F::NDPN * F::NDOFE;
    for (int idx = lane; idx < F::NDPN * F::NDOFE; idx += 32) {
      const int i = idx / F::NDOFE, c = idx % F::NDOFE;
      const int b = c / F::NDPN, j = c % F::NDPN;
      B[i * W + en.slot[b] * F::NDPN + j] += Ke[idx];
    }
    if (lane < F::NDPN) r += Fe_in[int64_t(en.e) * F::NDOFE + en.aloc * F::NDPN + lane];
  }
  __syncwarp();
  double* out = val + base[n];
  for (int idx = lane; idx < F::NDPN * W; idx += 32) out[idx] = B[idx];
  if (lane < F::NDPN) Rv[n * F::NDPN + lane] = r;
}

// ----------------------------------------------------------------------------------------
template <int D>
__global__ void k_update_history(int64_t ne, const int32_t* __restrict__ conn,
                                 const double* __restrict__ dofs, double* __restrict__ kappa) {
  using F = Fam<D>;
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t >= ne * F::NGP) return;
  const int64_t e = t / F::NGP;
  const int g = int(t % F::NGP);
  double eb = 0.0;
#pragma unroll
  for (int a = 0; a < F::NEN; ++a)
    eb = fma(shapeN<D>(a, g), dofs[int64_t(conn[e * F::NEN + a]) * F::NDPN + D], eb);
  const double k = kappa[t];
  if ((eb - k) > 1e-10) kappa[t] = eb;  // Fig. 8b l.22-23
}

constexpr int kSumBlocks = 592;   // 4 x 148 SMs
constexpr int kSumThreads = 256;

__global__ void k_sumsq_partial(int64_t n_rows, int ndpn, int dim, const double* __restrict__ R,
                                double* __restrict__ part) {
  __shared__ double su[kSumThreads], se[kSumThreads];
  double u = 0.0, e = 0.0;
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n_rows;
       r += int64_t(gridDim.x) * blockDim.x) {
    const double v = R[r];
    if (int(r % ndpn) == dim) e = fma(v, v, e);
    else u = fma(v, v, u);
  }
  su[threadIdx.x] = u;
  se[threadIdx.x] = e;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      su[threadIdx.x] += su[threadIdx.x + s];
      se[threadIdx.x] += se[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = su[0];
    part[2 * blockIdx.x + 1] = se[0];
  }
}

__global__ void k_sumsq_final(int nparts, const double* __restrict__ part, double* __restrict__ out) {
  __shared__ double su[kSumThreads], se[kSumThreads];
  double u = 0.0, e = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
    u += part[2 * i];
    e += part[2 * i + 1];
  }
  su[threadIdx.x] = u;
  se[threadIdx.x] = e;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      su[threadIdx.x] += su[threadIdx.x + s];
      se[threadIdx.x] += se[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = su[0];
    out[1] = se[0];
  }
}

__global__ void k_scale(int64_t n, double s, double* __restrict__ x) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) x[i] *= s;
}

}  // namespace lgdm

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
              const double* __restrict__ kappa, const double* __restrict__ k0g,
              const double* __restrict__ alg, double* __restrict__ Ke_out,
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
      if (e < ne) {
        const int64_t q = e * F::NGP + g;   // per-GP damage parameters (defect fields)
        phaseA<D>(m, Xs + el * F::NEN * D, Us + el * F::NEN * F::NDPN, kappa[q],
                  k0g ? k0g[q] : m.kappa0, alg ? alg[q] : m.alpha, g,
                  recs + size_t(t) * GpBlock<D>::STRIDE, scal + t * kScal);
      }
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
         const double* __restrict__ Ke_in, const double* __restrict__ Fe_in, int max_deg,
         double* __restrict__ val, double* __restrict__ Rv) {
  using F = Fam<D>;
  extern __shared__ double gbuf[];   // [WPB][NDPN x max_deg NDPN]: sized by the largest degree
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n = int64_t(blockIdx.x) * WPB + wl;
  if (n >= n_owned) return;
  const int deg = int(nbr_ptr[n + 1] - nbr_ptr[n]);
  const int W = deg * F::NDPN;
  double* B = gbuf + size_t(wl) * F::NDPN * max_deg * F::NDPN;
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
// Blocked DOF order [u; ebar]: P K P^T and P R of the
// node-interleaved CSR, one warp per blocked row.  Interleaved row (o, i) of node o with deg
// neighbours holds, from base[o] + i deg ndpn, the columns (neighbour k, comp) at k ndpn + comp;
// blocked row (u rows first: r = o dim + i, then e rows: r = n dim + o) holds the u columns
// (k, comp < dim) then the e columns (k, comp = dim) -- ascending blocked column ids.
template <int DIM, int NDPN>
__global__ void k_blocked(int64_t no, const int64_t* __restrict__ nbr_ptr,
                          const int64_t* __restrict__ base, const int32_t* __restrict__ col_idx,
                          const double* __restrict__ val, const double* __restrict__ R,
                          int64_t* __restrict__ rp_b, int32_t* __restrict__ ci_b,
                          double* __restrict__ val_b, double* __restrict__ R_b) {
  const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nrows = no * NDPN;
  if (warp >= nrows) return;
  const bool urow = warp < no * DIM;
  const int64_t o = urow ? warp / DIM : warp - no * DIM;
  const int i = urow ? int(warp % DIM) : DIM;
  const int64_t deg = nbr_ptr[o + 1] - nbr_ptr[o];
  const int64_t start = urow ? nbr_ptr[o] * NDPN * DIM + i * deg * NDPN
                             : nbr_ptr[no] * NDPN * DIM + nbr_ptr[o] * NDPN;
  const int64_t src0 = base[o] + i * deg * NDPN;
  for (int64_t j = lane; j < deg * NDPN; j += 32) {
    const bool ucol = j < deg * DIM;
    const int64_t k = ucol ? j / DIM : j - deg * DIM;
    const int comp = ucol ? int(j % DIM) : DIM;
    const int64_t src = src0 + k * NDPN + comp;
    const int64_t mnode = col_idx[src] / NDPN;
    ci_b[start + j] = int32_t(ucol ? mnode * DIM + comp : no * DIM + mnode);
    val_b[start + j] = val[src];
  }
  if (lane == 0) {
    rp_b[warp] = start;
    R_b[warp] = R[o * NDPN + i];
    if (warp == nrows - 1) rp_b[nrows] = nbr_ptr[no] * NDPN * NDPN;
  }
}

// ----------------------------------------------------------------------------------------
// State-variable update (Alg. 2 l.8-14, Fig. 9a update_variables, P:288-295,
// P:359-390), one thread per (element, GP): record [eps_v (NV, Voigt, engineering shear),
// d eeq / d eps_v (NV, Eq. A.3), sigma (NV, Eq. 2 with the h_sigma term of reading R-11a),
// eeq, ebar, kappa, D (Eq. A.1), g (Eq. A.4)] and the history commit of k_update_history.
// Per-GP k0g / alg: defect fields, NULL = material values.
template <int D> struct StateW {
  static constexpr int NV = D == 1 ? 1 : (D == 2 ? 3 : 6);
  static constexpr int W = 3 * NV + 5;
};
// State record of one GP from the displacement gradient Gu and ebar (shared by k_update_state
// and the mixed-order k_mixed_state): [eps_v, d eeq/d eps_v, sigma (Eq. 2), eeq, ebar, kappa,
// D (Eq. A.1), g (Eq. A.4)]; the trial kappa (Fig. 9a l.22-24) is returned in *kap_out.
template <int D>
__device__ __forceinline__ void state_record(const DevMat& m, const double (&Gu)[D][D], double ebar,
                                             double kh, double k0, double al, double* out,
                                             double* kap_out) {
  constexpr int NV = StateW<D>::NV;
  // Voigt strain (engineering shear): 2D [xx, yy, xy], 3D [xx, yy, zz, xy, yz, xz]
  double ev[NV], dv[NV], eeq;
  if constexpr (D == 1) {
    ev[0] = Gu[0][0];
    eeq = ev[0];                                   // reading R-1D
    dv[0] = 1.0;
  } else {
    constexpr int P[6] = {0, 1, 2, 0, 1, 0}, Q[6] = {0, 1, 2, 1, 2, 2};
    double mv[NV], sv[NV];
#pragma unroll
    for (int V = 0; V < NV; ++V) {
      const int p = (D == 2 && V == 2) ? 0 : P[V], q = (D == 2 && V == 2) ? 1 : Q[V];
      ev[V] = V < D ? Gu[p][p] : Gu[p][q] + Gu[q][p];
      mv[V] = V < D ? 1.0 : 0.0;
    }
    double I1 = 0.0;
#pragma unroll
    for (int V = 0; V < D; ++V) I1 += ev[V];
    // J2 = 1/2 dev:dev on the 3x3 tensor (plane strain eps33 = 0, reading R-PS; shear gamma/2)
    double J2 = 0.0;
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      const double dp = (p < D ? ev[p] : 0.0) - I1 / 3.0;
      J2 += 0.5 * dp * dp;
      if (p < D) sv[p] = dp;
    }
#pragma unroll
    for (int V = D; V < NV; ++V) {
      J2 += 0.25 * ev[V] * ev[V];
      sv[V] = 0.5 * ev[V];
    }
    const double Qv = m.c2 * I1 * I1 + m.c3 * J2;
    const double sQ = sqrt(Qv);
    eeq = m.c1 * I1 + sQ * m.i2k;
    const double r4k = Qv < 1e-30 ? 0.0 : m.i4k / sQ;   // reading R-SQ: no sqrt term
#pragma unroll
    for (int V = 0; V < NV; ++V)
      dv[V] = m.c1 * mv[V] + (2.0 * m.c2 * I1 * mv[V] + m.c3 * sv[V]) * r4k;
  }
  // history (Fig. 9a l.22-24), damage (Eq. A.1, l.27-31), interaction (Eq. A.4)
  const double kap = (ebar - kh) > 1e-10 ? ebar : kh;
  double Dm = 0.0;
  if (!((kap - k0) < 1e-10)) Dm = 1.0 - (k0 / kap) * (1.0 - al + al * exp(-m.beta * (kap - k0)));
  const double gI = m.ga * exp(-m.n * Dm) + m.gb;
  *kap_out = kap;
  if (out) {
    // Eq. 2: sigma = (1 - D) C eps + h_sigma (eeq - ebar) d
    const double hr = m.hs * (eeq - ebar);
    double tr = 0.0;
#pragma unroll
    for (int U2 = 0; U2 < D; ++U2) tr += ev[U2];
#pragma unroll
    for (int V = 0; V < NV; ++V) {
      const double ce = D == 1 ? m.E * ev[0] : (V < D ? m.lam * tr + 2.0 * m.mu * ev[V] : m.mu * ev[V]);
      out[V] = ev[V];
      out[NV + V] = dv[V];
      out[2 * NV + V] = fma(1.0 - Dm, ce, hr * dv[V]);
    }
    out[3 * NV + 0] = eeq;
    out[3 * NV + 1] = ebar;
    out[3 * NV + 2] = kap;
    out[3 * NV + 3] = Dm;
    out[3 * NV + 4] = gI;
  }
}

template <int D>
__global__ void __launch_bounds__(128, 5)   // 5 CTAs/SM: 96 registers (+80 B stack) measured 5 % faster than 4
k_update_state(DevMat m, int64_t ne, const int32_t* __restrict__ conn,
               const double* __restrict__ coords, const double* __restrict__ dofs,
               double* __restrict__ kappa, const double* __restrict__ k0g,
               const double* __restrict__ alg, double* __restrict__ sdv) {
  using F = Fam<D>;
  constexpr int W = StateW<D>::W;
  // a warp = 32 consecutive GPs = EPW whole elements = exactly 32 (element, node) slots
  constexpr int EPW = 32 / F::NGP, NV = D + F::NDPN;   // node values: coords, dofs
  static_assert(EPW * F::NEN == 32, "one node per lane");
  extern __shared__ double stage[];   // [blockDim][W]: records, written out coalesced; then
                                      // per warp [32][NV] node values
  double* nodes = stage + blockDim.x * W + (threadIdx.x >> 5) * (32 * NV);   // [EPW][NEN][NV]
  const int lane = threadIdx.x & 31;
  const int64_t t0 = int64_t(blockIdx.x) * blockDim.x;
  const int64_t t = t0 + threadIdx.x;
  const int64_t ngp = ne * F::NGP;
  {
    // each lane gathers one node of the warp's elements (one conn load, NV value loads),
    // instead of every GP thread loading all nodes of its element
    const int64_t ew = (t0 + (threadIdx.x & ~31)) / F::NGP + lane / F::NEN;
    if (ew < ne) {
      const int64_t n = conn[ew * F::NEN + lane % F::NEN];
#pragma unroll
      for (int i = 0; i < D; ++i) nodes[lane * NV + i] = __ldg(coords + n * D + i);
#pragma unroll
      for (int i = 0; i < F::NDPN; ++i) nodes[lane * NV + D + i] = __ldg(dofs + n * F::NDPN + i);
    }
    __syncwarp();
  }
  if (t < ngp) {
    const int g = int(t % F::NGP);
    const double* en = nodes + (lane / F::NGP) * (F::NEN * NV);   // this element's nodes
    // geometry: J_ij = sum_a X_ai dN_a/dxi_j
    double J[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) J[i][j] = 0.0;
#pragma unroll
    for (int a = 1; a < F::NEN; ++a) {        // relative to node 0 (reading R-REL)
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const double x = en[a * NV + i] - en[i];
#pragma unroll
        for (int j = 0; j < D; ++j) J[i][j] = fma(x, shape_dxi<D>(a, g, j), J[i][j]);
      }
    }
    double Ji[D][D];
    if constexpr (D == 1) {
      Ji[0][0] = 1.0 / J[0][0];
    } else if constexpr (D == 2) {
      const double r = 1.0 / (J[0][0] * J[1][1] - J[0][1] * J[1][0]);
      Ji[0][0] = J[1][1] * r;
      Ji[0][1] = -J[0][1] * r;
      Ji[1][0] = -J[1][0] * r;
      Ji[1][1] = J[0][0] * r;
    } else {
      const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
      const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
      const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
      const double r = 1.0 / (J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02);
      Ji[0][0] = c00 * r;
      Ji[1][0] = c01 * r;
      Ji[2][0] = c02 * r;
      Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * r;
      Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * r;
      Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * r;
      Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * r;
      Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * r;
      Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * r;
    }
    // displacement gradient Gu_ij = sum_a u_ai dN_a/dx_j and ebar = sum_a N_a e_a
    double Gu[D][D], ebar = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) Gu[i][j] = 0.0;
#pragma unroll
    for (int a = 0; a < F::NEN; ++a) {
      double gn[D];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) s = fma(Ji[k][j], shape_dxi<D>(a, g, k), s);
        gn[j] = s;
      }
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const double u = en[a * NV + D + i] - en[D + i];
#pragma unroll
        for (int j = 0; j < D; ++j) Gu[i][j] = fma(u, gn[j], Gu[i][j]);
      }
      ebar = fma(shapeN<D>(a, g), en[a * NV + D + D], ebar);
    }
    double kap;
    state_record<D>(m, Gu, ebar, kappa[t], k0g ? k0g[t] : m.kappa0, alg ? alg[t] : m.alpha,
                    sdv ? stage + threadIdx.x * W : nullptr, &kap);
    kappa[t] = kap;
  }
  if (sdv) {   // the block's records are one contiguous range of the output: coalesced copy
    __syncthreads();
    const int64_t nrec = min(int64_t(blockDim.x), ngp - t0);
    const int n = int(nrec) * W;
    double* dst = sdv + t0 * W;   // 16-byte aligned: 128 W doubles per block, even
    const int n2 = n >> 1;
    for (int k = threadIdx.x; k < n2; k += blockDim.x)
      __stcs(reinterpret_cast<double2*>(dst) + k, reinterpret_cast<const double2*>(stage)[k]);
    if ((n & 1) && threadIdx.x == 0) __stcs(dst + n - 1, stage[n - 1]);
  }
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

// lgdm_mixed.cuh -- mixed-order elements: quadratic u with linear ebar, the
// paper's own discretisation ("shape functions for displacement (u) are taken as
// quadratic, and for micro-equivalent strain as linear"; 1D bar P:418; 2D SEN P:466).
//   LGDM_BAR3  (4): 3-node quadratic bar for u (local nodes xi = -1, +1, 0), linear ebar on
//                   the two end nodes, 3-point Gauss.
//   LGDM_QUAD8 (5): 8-node serendipity quad for u (corners counter-clockwise, then midsides
//                   (0,-1), (1,0), (0,1), (-1,0)), bilinear ebar on the corners, 3x3 Gauss
//                   (readings R-Q8, R-GEO, R-GP3, R-ORDM).
// Local element dofs are node-major: corner a < NENE holds (u_0..u_{D-1}, ebar) at a (D+1);
// midside a >= NENE holds (u_0..u_{D-1}) at NENE (D+1) + (a - NENE) D.  Global dof of node n,
// component c = doff[n] + c.
//
// Two kernels, as the general equal-order path (k_elem_blocks + k_gather):
//   k_mixed_blocks  one warp per two elements (mixed_elements): GP cores of both at once (the
//                   constitutive part is gpLaw of lgdm_device.cuh), per-(GP, node) records in
//                   shared memory, node-pair Gauss sums (one lane per pair a < b, both
//                   directions), diagonal blocks by the row-sum identity -> element blocks
//                   Ke [NDOFE][NDOFE], Fe [NDOFE] in HBM;
//   k_mixed_gather  one warp per owned node: the node's CSR block-row accumulated in shared
//                   memory over its adjacent elements in ascending element id (atomic-free,
//                   bitwise reproducible; the element row-blocks arrive by cp.async, all of a
//                   node's elements in flight at once), then written once, coalesced.
// Gradients use coordinates / dofs relative to the element's node 0 (reading R-REL).  Also
// here: k_mixed_state (state records), k_mixed_history, k_mixed_detj, k_blocked_mixed and the
// dof-kind reductions of the residual / increment norms.
#pragma once
#include <cstdint>

namespace lgdm {

template <int T> struct MFam;
template <> struct MFam<4> {
  static constexpr int DIM = 1, NENU = 3, NENE = 2, NGP = 3, NS = 1, NDOFE = 5;
};
template <> struct MFam<5> {
  static constexpr int DIM = 2, NENU = 8, NENE = 4, NGP = 9, NS = 3, NDOFE = 20;
};

template <int T> __host__ __device__ constexpr int mldof(int a) {
  using F = MFam<T>;
  return a < F::NENE ? a * (F::DIM + 1) : F::NENE * (F::DIM + 1) + (a - F::NENE) * F::DIM;
}
// local dof -> (node, component)
template <int T> __host__ __device__ constexpr int mdof_node(int c) {
  using F = MFam<T>;
  return c < F::NENE * (F::DIM + 1) ? c / (F::DIM + 1) : F::NENE + (c - F::NENE * (F::DIM + 1)) / F::DIM;
}
template <int T> __host__ __device__ constexpr int mdof_comp(int c) {
  using F = MFam<T>;
  return c < F::NENE * (F::DIM + 1) ? c % (F::DIM + 1) : (c - F::NENE * (F::DIM + 1)) % F::DIM;
}

// Shape-function values at the Gauss points, tabulated once on the host (lgdm_api.cu,
// mixed_tables) into constant memory: every lane of a warp reads the same GP row.
template <int T> struct MShape {
  using F = MFam<T>;
  double w[F::NGP];
  double Nu[F::NGP][F::NENU], dNu[F::NGP][F::NENU][F::DIM];
  double Ne[F::NGP][F::NENE], dNe[F::NGP][F::NENE][F::DIM];
};
__constant__ MShape<4> c_shape4;
__constant__ MShape<5> c_shape5;
template <int T> __device__ __forceinline__ const MShape<T>& mshape();
template <> __device__ __forceinline__ const MShape<4>& mshape<4>() { return c_shape4; }
template <> __device__ __forceinline__ const MShape<5>& mshape<5>() { return c_shape5; }

// per-(GP, u node) record: grad N, S grad N, W' grad N, Dt' grad N, Sigma' grad N (the Kuu
// column factors t1 = lam* gN + Ams SgN, t2 = Ams gN + Ass SgN are formed in the pair loop:
// 4 D fewer doubles of shared memory per record -> more resident elements)
template <int D> struct MURec {
  static constexpr int GN = 0, SGN = D, WGN = 2 * D, DGN = 3 * D, FU = 4 * D,
                       STRIDE = 5 * D + 1;   // odd: spreads banks
};
// per-(GP, ebar node) record: N, grad N, hN N + gvec . grad N (Kee), fe0 N + fvec . grad N (Fe)
template <int D> struct MERec {
  static constexpr int N = 0, GN = 1, E = 1 + D, FE = 2 + D, STRIDE = 3 + D + ((3 + D) % 2 == 0);
};

// per-warp shared memory of mixed_elements (doubles): coordinates + element dofs and the GP
// cores of two elements, the records of one element (reused as the block staging
// [NENU][NENU][D+1][D+1] once the pair sums are done), the coupling sums U, V of the corners
template <int T> struct MSmem {
  using F = MFam<T>;
  static constexpr int D = F::DIM;
  static constexpr int NPE = F::NENU * D + F::NDOFE;             // X [NENU][D], U [NDOFE]
  static constexpr int XU = 0, CORE = XU + 2 * NPE, CS = F::NGP * Core<D>::STRIDE,
                       UR = CORE + 2 * CS,
                       ER = UR + F::NGP * F::NENU * MURec<D>::STRIDE,
                       UV = ER + F::NGP * F::NENE * MERec<D>::STRIDE,
                       SIZE = (UV + F::NENE * (D + 1) + 1) & ~1;
  static constexpr int ST = F::NDOFE * F::NDOFE;   // staging of Ke (row-major), at UR
  static_assert(ST <= ER - UR, "block staging fits in the record area");
  static_assert(UR % 2 == 0 && SIZE % 2 == 0, "16-byte aligned staging");
  static constexpr int NP = F::NENU * (F::NENU - 1) / 2;             // node pairs a < b
  static_assert(NP + F::NENE <= 32, "one lane per pair plus the coupling lanes");
};

// Element tangent Ke [NDOFE][NDOFE] (local dof order, row-major) and residual Fe [NDOFE] of up
// to two elements (e1 < 0: one), by one warp, from their coordinates / dofs staged in sm[XU]
// (MInputs::store + __syncwarp).  out(k, Ke, Fe) supplies element k's output pointers (HBM
// scratch or shared memory).
//   * GP cores of both elements in one pass: lanes 16 k + g (two elements' 2 x NGP lanes);
//   * per element: per-(GP, node) records; one lane per node pair a < b Gauss-sums K_ab and
//     K_ba together (Kuu_ba = Kuu_ab^T: the integrand lam gA gB^T + Ams (gA SgB^T + SgA gB^T) +
//     Ass SgA SgB^T + mu (gB gA^T + gA.gB I) is symmetric under a <-> b with transposition);
//   * diagonal blocks by the partition-of-unity row-sum identity, as in the sweeps (sum_b N_b
//     = 1 for the u and the ebar families alike): Kuu_aa = -sum_{b!=a} Kuu_ab,
//     Keu_aa = -sum_{b!=a} Keu_ab, Kue_aa = U_a - sum_{b!=a corner} Kue_ab with
//     U_a = sum_g W' grad N_a, Kee_aa = V_a - sum_{b!=a corner} Kee_ab with V_a = sum_g E_a.
// Inputs of an element pair, software-pipelined by the caller: each lane holds <= 3 of the
// 2 x NPE values (coordinates, element dofs); the gather indices are loaded one pass before
// the values, the values one pass before they are used.
template <int T> struct MInputs {
  static constexpr int NPE = MSmem<T>::NPE, NQ = (2 * NPE + 31) / 32;
  int64_t idx[NQ];
  double v[NQ];
  // global index of value t of the pair (e0, e1): coords or dofs offset, -1 = none
  __device__ __forceinline__ void load_idx(int lane, int64_t e0, int64_t e1, const int32_t* __restrict__ conn,
                                           const int32_t* __restrict__ gdof) {
    constexpr int D = MFam<T>::DIM, NENU = MFam<T>::NENU, ND = MFam<T>::NDOFE;
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
      const int t = lane + 32 * u;
      const int k = t >= NPE ? 1 : 0, q = t - k * NPE;
      const int64_t e = k ? e1 : e0;
      idx[u] = -1;
      if (t < 2 * NPE && e >= 0)
        idx[u] = q < NENU * D ? int64_t(conn[e * NENU + q / D]) * D + q % D : int64_t(gdof[e * ND + q - NENU * D]);
    }
  }
  __device__ __forceinline__ void load_vals(int lane, const double* __restrict__ coords,
                                            const double* __restrict__ dofs) {
    constexpr int D = MFam<T>::DIM, NENU = MFam<T>::NENU;
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
      const int q = (lane + 32 * u) % NPE;
      v[u] = idx[u] < 0 ? 0.0 : (q < NENU * D ? coords[idx[u]] : dofs[idx[u]]);
    }
  }
  __device__ __forceinline__ void store(int lane, double* sm) const {
#pragma unroll
    for (int u = 0; u < NQ; ++u)
      if (lane + 32 * u < 2 * NPE) sm[MSmem<T>::XU + lane + 32 * u] = v[u];
  }
};

template <int T, class OUT>
__device__ __forceinline__ void mixed_elements(const DevMat& m, const MShape<T>& S, double* sm, int lane,
                                               int64_t e0, int64_t e1,
                                               const double* __restrict__ kappa,
                                               const double* __restrict__ k0g,
                                               const double* __restrict__ alg, OUT&& out) {
  using F = MFam<T>;
  constexpr int D = F::DIM, NGP = F::NGP, NENU = F::NENU, NENE = F::NENE, ND = F::NDOFE;
  constexpr int DB = D + 1;
  using SM = MSmem<T>;
  using UR = MURec<D>;
  using ER = MERec<D>;
  using Co = Core<D>;
  // (coordinates and element dofs of both elements are in sm[XU], see MInputs)
  // GP cores: geometry on the u nodes (R-GEO), kinematics, Appendix A law
  {
    const int k = lane >> 4, g = lane & 15;
    const int64_t e = k ? e1 : e0;
    if (g < NGP && e >= 0) {
      const double* X = sm + SM::XU + k * SM::NPE;
      const double* U = X + NENU * D;
      double J[D][D];
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) J[i][j] = 0.0;
      // J = sum_a (X_a - X_0) dN_a/dxi (sum_a dN_a = 0): coordinates relative to node 0
      // (exact differences) remove the cancellation of |X| >> element size (R-REL)
#pragma unroll
      for (int a = 1; a < NENU; ++a)
#pragma unroll
        for (int j = 0; j < D; ++j)
#pragma unroll
          for (int i = 0; i < D; ++i) J[i][j] = fma(X[a * D + i] - X[i], S.dNu[g][a][j], J[i][j]);
      double detJ, Ji[D][D];
      if constexpr (D == 1) {
        detJ = J[0][0];
        Ji[0][0] = 1.0 / detJ;
      } else {
        detJ = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        const double r = 1.0 / detJ;
        Ji[0][0] = J[1][1] * r;
        Ji[0][1] = -J[0][1] * r;
        Ji[1][0] = -J[1][0] * r;
        Ji[1][1] = J[0][0] * r;
      }
      const double dV = S.w[g] * detJ * m.t;
      double eps[D][D], ebar = 0.0, gb[D];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        gb[i] = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) eps[i][j] = 0.0;
      }
#pragma unroll
      for (int a = 1; a < NENU; ++a) {       // gradients from differences to node 0, likewise
        double gn[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < D; ++j) s = fma(Ji[j][i], S.dNu[g][a][j], s);
          gn[i] = s;
        }
#pragma unroll
        for (int i = 0; i < D; ++i) {
          const double ua = U[mldof<T>(a) + i] - U[i];
#pragma unroll
          for (int j = 0; j < D; ++j) eps[i][j] = fma(ua, gn[j], eps[i][j]);
        }
      }
#pragma unroll
      for (int a = 0; a < NENE; ++a) {
        const double ea = U[mldof<T>(a) + D];
        ebar = fma(S.Ne[g][a], ea, ebar);
        if (a == 0) continue;
        const double da = ea - U[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < D; ++j) s = fma(Ji[j][i], S.dNe[g][a][j], s);
          gb[i] = fma(s, da, gb[i]);
        }
      }
      double es[F::NS];
      if constexpr (D == 1) {
        es[0] = eps[0][0];
      } else {
        es[0] = eps[0][0];
        es[1] = eps[1][1];
        es[2] = 0.5 * (eps[0][1] + eps[1][0]);
      }
      const int64_t q = e * NGP + g;
      gpLaw<D>(m, Ji, dV, es, ebar, gb, kappa[q], k0g ? k0g[q] : m.kappa0, alg ? alg[q] : m.alpha,
               sm + SM::CORE + k * SM::CS + g * Co::STRIDE);
    }
  }
  __syncwarp();
  // this lane's node pair a < b (lanes < NP)
  int pa = 0, pb = 0;
  {
    int r = lane;
    for (int a = 0; a < NENU - 1; ++a) {
      if (r < NENU - 1 - a) {
        pa = a;
        pb = a + 1 + r;
        break;
      }
      r -= NENU - 1 - a;
    }
  }
  for (int k = 0; k < 2; ++k) {
    if ((k ? e1 : e0) < 0) continue;
    const double* cores = sm + SM::CORE + k * SM::CS;
    // per-(GP, node) records
    for (int t = lane; t < NGP * NENU; t += 32) {
      const int g = t / NENU, a = t % NENU;
      const double* core = cores + g * Co::STRIDE;
      double* r = sm + SM::UR + t * UR::STRIDE;
      double gn[D], SgN[D], WgN[D], DgN[D], fu[D];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) s = fma(core[Co::JI + j * D + i], S.dNu[g][a][j], s);
        gn[i] = s;
      }
      symv<D>(core + Co::S, gn, SgN);
      symv<D>(core + Co::WT, gn, WgN);
      symv<D>(core + Co::DT, gn, DgN);
      symv<D>(core + Co::SG, gn, fu);
#pragma unroll
      for (int i = 0; i < D; ++i) {
        r[UR::GN + i] = gn[i];
        r[UR::SGN + i] = SgN[i];
        r[UR::WGN + i] = WgN[i];
        r[UR::DGN + i] = DgN[i];
        r[UR::FU + i] = fu[i];
      }
    }
    for (int t = lane; t < NGP * NENE; t += 32) {
      const int g = t / NENE, a = t % NENE;
      const double* core = cores + g * Co::STRIDE;
      double* r = sm + SM::ER + t * ER::STRIDE;
      double gvd = 0.0, fvd = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) s = fma(core[Co::JI + j * D + i], S.dNe[g][a][j], s);
        r[ER::GN + i] = s;
        gvd = fma(core[Co::GV + i], s, gvd);
        fvd = fma(core[Co::FV + i], s, fvd);
      }
      const double Na = S.Ne[g][a];
      r[ER::N] = Na;
      r[ER::E] = fma(core[Co::HN], Na, gvd);
      r[ER::FE] = fma(core[Co::FE0], Na, fvd);
    }
    __syncwarp();
    // node-pair Gauss sums (Eqs. 11a-d), both directions
    double Kuu[D][D], Kue_ab[D], Kue_ba[D], Keu_ab[D], Keu_ba[D], Kee_ab = 0.0, Kee_ba = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      Kue_ab[i] = Kue_ba[i] = Keu_ab[i] = Keu_ba[i] = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) Kuu[i][j] = 0.0;
    }
    const bool ca = pa < NENE, cb = pb < NENE;   // corners carry ebar (cb implies ca)
    if (lane < SM::NP) {
#pragma unroll 1
      for (int g = 0; g < NGP; ++g) {
        const double* A = sm + SM::UR + (g * NENU + pa) * UR::STRIDE;
        const double* B = sm + SM::UR + (g * NENU + pb) * UR::STRIDE;
        const double* core = cores + g * Co::STRIDE;
        const double mu = core[Co::MU];
        const double lamS = core[Co::LAM], Ams = core[Co::AMS], Ass = core[Co::ASS];
        double t1[D], t2[D];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          t1[j] = fma(lamS, B[UR::GN + j], Ams * B[UR::SGN + j]);
          t2[j] = fma(Ams, B[UR::GN + j], Ass * B[UR::SGN + j]);
        }
        double dot = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) dot = fma(A[UR::GN + i], B[UR::GN + i], dot);
#pragma unroll
        for (int i = 0; i < D; ++i) {
          const double ub = mu * B[UR::GN + i];
#pragma unroll
          for (int j = 0; j < D; ++j) {
            double v = Kuu[i][j];
            v = fma(A[UR::GN + i], t1[j], v);
            v = fma(A[UR::SGN + i], t2[j], v);
            v = fma(A[UR::GN + j], ub, v);
            Kuu[i][j] = v;
          }
          Kuu[i][i] = fma(mu, dot, Kuu[i][i]);
        }
        if (ca) {
          const double* EA = sm + SM::ER + (g * NENE + pa) * ER::STRIDE;
          const double NA = EA[ER::N];
#pragma unroll
          for (int i = 0; i < D; ++i) {
            Kue_ba[i] = fma(NA, B[UR::WGN + i], Kue_ba[i]);
            Keu_ab[i] = fma(NA, B[UR::DGN + i], Keu_ab[i]);
          }
          if (cb) {
            const double* EBr = sm + SM::ER + (g * NENE + pb) * ER::STRIDE;
            const double NB = EBr[ER::N];
#pragma unroll
            for (int i = 0; i < D; ++i) {
              Kue_ab[i] = fma(NB, A[UR::WGN + i], Kue_ab[i]);
              Keu_ba[i] = fma(NB, A[UR::DGN + i], Keu_ba[i]);
            }
            double dote = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) dote = fma(EA[ER::GN + i], EBr[ER::GN + i], dote);
            const double gd = core[Co::GHC] * dote;
            Kee_ab = fma(NB, EA[ER::E], gd + Kee_ab);
            Kee_ba = fma(NA, EBr[ER::E], gd + Kee_ba);
          }
        }
      }
    } else if (lane < SM::NP + NENE) {   // coupling sums of corner a: U_a = sum W' grad N_a, V_a = sum E_a
      const int a = lane - SM::NP;
      double u[D], v = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) u[i] = 0.0;
      for (int g = 0; g < NGP; ++g) {
#pragma unroll
        for (int i = 0; i < D; ++i) u[i] += sm[SM::UR + (g * NENU + a) * UR::STRIDE + UR::WGN + i];
        v += sm[SM::ER + (g * NENE + a) * ER::STRIDE + ER::E];
      }
#pragma unroll
      for (int i = 0; i < D; ++i) sm[SM::UV + a * DB + i] = u[i];
      sm[SM::UV + a * DB + D] = v;
    }
    // residual (Eqs. 11e, 11f), from the records before the staging overwrites them
    double* Ke;
    double* Fe;
    out(k, Ke, Fe);
    if (lane < ND) {
      const int a = mdof_node<T>(lane), i = mdof_comp<T>(lane);
      double f = 0.0;
      if (i < D) {
#pragma unroll
        for (int g = 0; g < NGP; ++g) f += sm[SM::UR + (g * NENU + a) * UR::STRIDE + UR::FU + i];
      } else {
#pragma unroll
        for (int g = 0; g < NGP; ++g) f += sm[SM::ER + (g * NENE + a) * ER::STRIDE + ER::FE];
      }
      Fe[lane] = f;
    }
    __syncwarp();
    // off-diagonal blocks into the staging: Ke itself (local dof order, row-major)
    double* st = sm + SM::UR;
    auto stg = [&](int a, int b, int i, int j) -> double& { return st[(mldof<T>(a) + i) * ND + mldof<T>(b) + j]; };
    if (lane < SM::NP) {
#pragma unroll
      for (int i = 0; i < D; ++i) {
#pragma unroll
        for (int j = 0; j < D; ++j) {
          stg(pa, pb, i, j) = Kuu[i][j];
          stg(pb, pa, j, i) = Kuu[i][j];
        }
        if (cb) stg(pa, pb, i, D) = Kue_ab[i];
        if (ca) stg(pb, pa, i, D) = Kue_ba[i];
        if (ca) stg(pa, pb, D, i) = Keu_ab[i];
        if (cb) stg(pb, pa, D, i) = Keu_ba[i];
      }
      if (cb) {
        stg(pa, pb, D, D) = Kee_ab;
        stg(pb, pa, D, D) = Kee_ba;
      }
    }
    __syncwarp();
    // diagonal blocks: coupling - the row's other blocks, ascending b.  Entries (a, i, j):
    // corners DB x DB, midsides D x D, enumerated corners first
    constexpr int NDG = NENE * DB * DB + (NENU - NENE) * D * D;
    for (int t = lane; t < NDG; t += 32) {
      int a, i, j;
      if (t < NENE * DB * DB) {
        a = t / (DB * DB);
        i = (t / DB) % DB;
        j = t % DB;
      } else {
        const int u = t - NENE * DB * DB;
        a = NENE + u / (D * D);
        i = (u / D) % D;
        j = u % D;
      }
      const double* row = st + (mldof<T>(a) + i) * ND + j;
      double sum = 0.0;
#pragma unroll
      for (int b = 0; b < NENU; ++b)   // ebar columns (j == D): corners only
        if (b != a && (j < D || b < NENE)) sum += row[mldof<T>(b)];
      const double c = j == D ? sm[SM::UV + a * DB + i] : 0.0;
      st[(mldof<T>(a) + i) * ND + mldof<T>(a) + j] = c - sum;
    }
    __syncwarp();
    // Ke out: a straight copy of the staging (16-byte vectors, coalesced)
    if constexpr ((ND * ND) % 2 == 0) {   // QUAD8: every element's Ke is 16-byte aligned
      const double2* s2 = reinterpret_cast<const double2*>(st);
      double2* k2 = reinterpret_cast<double2*>(Ke);
      for (int t = lane; t < ND * ND / 2; t += 32) k2[t] = s2[t];
    } else {
      for (int t = lane; t < ND * ND; t += 32) Ke[t] = st[t];
    }
    __syncwarp();
  }
}

template <int T, int WPB>
__global__ void __launch_bounds__(WPB * 32)
k_mixed_blocks(DevMat m, int64_t ne, const int32_t* __restrict__ conn, const double* __restrict__ coords,
               const int32_t* __restrict__ gdof, const double* __restrict__ dofs,
               const double* __restrict__ kappa, const double* __restrict__ k0g,
               const double* __restrict__ alg, double* __restrict__ EB, double* __restrict__ EF) {
  using F = MFam<T>;
  constexpr int ND = F::NDOFE;
  using SM = MSmem<T>;
  extern __shared__ double smem_mx[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // the shape table in shared memory: lanes read different Gauss points (divergent constant
  // cache reads would serialise)
  MShape<T>& S = *reinterpret_cast<MShape<T>*>(smem_mx);
  constexpr int TBL = (int(sizeof(MShape<T>)) / 8 + 1) & ~1;
  for (int k = threadIdx.x; k < int(sizeof(MShape<T>)) / 8; k += blockDim.x)
    smem_mx[k] = reinterpret_cast<const double*>(&mshape<T>())[k];
  __syncthreads();
  double* sm = smem_mx + TBL + w * SM::SIZE;
  // two elements per warp pass (e, e + stride); inputs pipelined (MInputs)
  const int64_t stride = int64_t(gridDim.x) * WPB;
  auto second = [&](int64_t e) { return e < ne && e + stride < ne ? e + stride : int64_t(-1); };
  auto first = [&](int64_t e) { return e < ne ? e : int64_t(-1); };
  int64_t e = int64_t(blockIdx.x) * WPB + w;
  MInputs<T> in;
  in.load_idx(lane, first(e), second(e), conn, gdof);
  in.load_vals(lane, coords, dofs);
  in.load_idx(lane, first(e + 2 * stride), second(e + 2 * stride), conn, gdof);
  for (; e < ne; e += 2 * stride) {
    const int64_t e1 = second(e);
    in.store(lane, sm);
    __syncwarp();
    in.load_vals(lane, coords, dofs);                                          // pass + 1
    in.load_idx(lane, first(e + 4 * stride), second(e + 4 * stride), conn, gdof);   // pass + 2
    mixed_elements<T>(m, S, sm, lane, e, e1, kappa, k0g, alg,
                      [&](int k, double*& Ke, double*& Fe) {
                        const int64_t ek = k ? e1 : e;
                        Ke = EB + ek * (ND * ND);
                        Fe = EF + ek * ND;
                      });
  }
}

// node -> adjacent element map of the gather: element, local index of the node, and the
// column offset (within the node's block-row) of each local node's first dof
struct MixAdj {
  int32_t e;
  int32_t aloc;
  int32_t coff[8];
};
// per-node gather metadata, one 32-byte load: first value of the block-row, first row,
// first adjacency entry, block-row width, rows, adjacent elements
struct NodeMeta {
  int64_t base, r0, k0;
  int32_t W;
  int16_t nr, nk;
};

// async global -> shared copies (no registers held while the loads are in flight)
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = unsigned(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
}

// per-warp staging of the gather: MXS element row-blocks ((D+1) x NDOFE doubles, padded to
// 32-multiples) + their residual entries
template <int T> struct MGStage {
  static constexpr int MXS = 4;
  static constexpr int RB = ((MFam<T>::DIM + 1) * MFam<T>::NDOFE + 31) / 32 * 32;
  static constexpr int SIZE = MXS * (RB + 4 + 4);   // row-blocks, F, column offsets (8 x int32)
};

template <int T, int WPB>
__global__ void __launch_bounds__(WPB * 32, 4)
k_mixed_gather(int64_t nn, const NodeMeta* __restrict__ meta, const MixAdj* __restrict__ adj,
               const double* __restrict__ EB, const double* __restrict__ EF, int max_row,
               double* __restrict__ val, double* __restrict__ R) {
  using F = MFam<T>;
  using SG = MGStage<T>;
  constexpr int ND = F::NDOFE;
  constexpr int NQ = SG::RB / 32;                     // entries of one element's rows per lane
  extern __shared__ double smem_mg[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* buf = smem_mg + w * (max_row + SG::SIZE);
  double* stg = buf + max_row;                        // [MXS][RB] row-blocks, then [MXS][4] F
  double* stf = stg + SG::MXS * SG::RB;
  int32_t* sco = reinterpret_cast<int32_t*>(stf + SG::MXS * 4);   // [MXS][8] column offsets
  const int64_t stride = int64_t(gridDim.x) * WPB;
  int64_t n = int64_t(blockIdx.x) * WPB + w;
  int qb[NQ], qrow[NQ], qcomp[NQ];   // local node, row and component of this lane's entries
#pragma unroll
  for (int t = 0; t < NQ; ++t) {
    const int q = lane + 32 * t, c = q % ND;
    qb[t] = mdof_node<T>(c);
    qrow[t] = q / ND;
    qcomp[t] = mdof_comp<T>(c);
  }
  NodeMeta nx{};
  if (n < nn) nx = meta[n];
  for (; n < nn; n += stride) {
    const NodeMeta md = nx;
    if (n + stride < nn) nx = meta[n + stride];      // prefetch the next node's metadata
    const int64_t r0 = md.r0, base = md.base;
    const int nr = md.nr, W = md.W;
    const int tot = nr * W;
    for (int k = lane; k < tot; k += 32) buf[k] = 0.0;
    // this lane's entries (row i, element dof c) of an element block: row * W + component of
    // the node's block-row (-1: no entry); qb / qrow / qcomp depend on the lane only
    int qoff[NQ];
#pragma unroll
    for (int t = 0; t < NQ; ++t) qoff[t] = lane + 32 * t < nr * ND ? qrow[t] * W + qcomp[t] : -1;
    double rsum = 0.0;
    const int64_t k0 = md.k0, k1 = md.k0 + md.nk;
    for (int64_t k = k0; k < k1; k += SG::MXS) {
      const int kk = int(k1 - k < SG::MXS ? k1 - k : SG::MXS);
      // the round's adjacency entries in one parallel load (lane u), then every row-block of
      // the round in flight at once, straight into shared memory
      int2 ea = make_int2(0, 0);
      if (lane < kk) ea = *reinterpret_cast<const int2*>(adj + k + lane);   // (e, aloc)
      for (int u = 0; u < kk; ++u) {
        const int64_t e = __shfl_sync(0xffffffffu, ea.x, u);
        const int lr = mldof<T>(__shfl_sync(0xffffffffu, ea.y, u));
        const double* src = EB + e * (ND * ND) + lr * ND;
#pragma unroll
        for (int t = 0; t < NQ; ++t)
          if (qoff[t] >= 0) cp_async8(stg + u * SG::RB + lane + 32 * t, src + lane + 32 * t);
        if (lane < nr) cp_async8(stf + u * 4 + lane, EF + e * ND + lr + lane);
      }
      // the round's column offsets (8 int32 per adjacency entry) join the same async group
      if (lane < 8 * kk) {
        const unsigned d = unsigned(__cvta_generic_to_shared(sco + lane));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(&adj[k + (lane >> 3)].coff[lane & 7]) : "memory");
      }
      cp_async_wait_all();
      __syncwarp();
      // accumulate in ascending element order
      for (int u = 0; u < kk; ++u) {
#pragma unroll
        for (int t = 0; t < NQ; ++t)
          if (qoff[t] >= 0) buf[qoff[t] + sco[u * 8 + qb[t]]] += stg[u * SG::RB + lane + 32 * t];
        if (lane < nr) rsum += stf[u * 4 + lane];
        __syncwarp();
      }
    }
    for (int k = lane; k < tot; k += 32) val[base + k] = buf[k];
    if (lane < nr) R[r0 + lane] = rsum;
    __syncwarp();
  }
}

template <int T>
__global__ void k_mixed_detj(int64_t ne, const int32_t* __restrict__ conn,
                             const double* __restrict__ coords, unsigned long long* bad) {
  using F = MFam<T>;
  constexpr int D = F::DIM;
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t >= ne * F::NGP) return;
  const int64_t e = t / F::NGP;
  const int g = int(t % F::NGP);
  const MShape<T>& S = mshape<T>();
  double J[D][D];
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) J[i][j] = 0.0;
  for (int a = 0; a < F::NENU; ++a) {
    const int64_t n = conn[e * F::NENU + a];
    for (int j = 0; j < D; ++j)
      for (int i = 0; i < D; ++i) J[i][j] += coords[n * D + i] * S.dNu[g][a][j];
  }
  double det;
  if constexpr (D == 1) det = J[0][0];
  else det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  if (!(det > 0.0)) atomicMin(bad, (unsigned long long)t);
}

// Eq. A.2 with Fig. 8b l.19-24: ebar at the GP from the linear ebar field
template <int T>
__global__ void k_mixed_history(int64_t ne, const int32_t* __restrict__ conn,
                                const int64_t* __restrict__ doff, const double* __restrict__ dofs,
                                double* __restrict__ kappa) {
  using F = MFam<T>;
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t >= ne * F::NGP) return;
  const int64_t e = t / F::NGP;
  const int g = int(t % F::NGP);
  const MShape<T>& S = mshape<T>();
  double eb = 0.0;
#pragma unroll
  for (int a = 0; a < F::NENE; ++a) eb = fma(S.Ne[g][a], dofs[doff[conn[e * F::NENU + a]] + F::DIM], eb);
  const double k = kappa[t];
  if ((eb - k) > 1e-10) kappa[t] = eb;
}

// State-variable update (Alg. 2 l.8-14, Fig. 9a) for mixed elements: one thread per
// (element, GP), u gradient from the quadratic field, ebar from the linear field, the record
// of state_record (lgdm_kernels.cuh), history commit; records staged and written coalesced.
template <int T>
__global__ void __launch_bounds__(128)
k_mixed_state(DevMat m, int64_t ne, const int32_t* __restrict__ conn,
              const double* __restrict__ coords, const int64_t* __restrict__ doff,
              const double* __restrict__ dofs, double* __restrict__ kappa,
              const double* __restrict__ k0g, const double* __restrict__ alg,
              double* __restrict__ sdv) {
  using F = MFam<T>;
  constexpr int D = F::DIM, W = StateW<D>::W;
  extern __shared__ double smem_ms[];
  MShape<T>& S = *reinterpret_cast<MShape<T>*>(smem_ms);
  constexpr int TBL = (int(sizeof(MShape<T>)) / 8 + 1) & ~1;
  for (int k = threadIdx.x; k < int(sizeof(MShape<T>)) / 8; k += blockDim.x)
    smem_ms[k] = reinterpret_cast<const double*>(&mshape<T>())[k];
  __syncthreads();
  double* stage = smem_ms + TBL;
  const int64_t t0 = int64_t(blockIdx.x) * blockDim.x;
  const int64_t t = t0 + threadIdx.x;
  const int64_t ngp = ne * F::NGP;
  if (t < ngp) {
    const int64_t e = t / F::NGP;
    const int g = int(t % F::NGP);
    const int32_t* ce = conn + e * F::NENU;
    double J[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) J[i][j] = 0.0;
    const int64_t n0 = ce[0];
#pragma unroll
    for (int a = 1; a < F::NENU; ++a) {      // relative to node 0 (see k_mixed_blocks)
      const int64_t n = ce[a];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const double x = __ldg(coords + n * D + i) - __ldg(coords + n0 * D + i);
#pragma unroll
        for (int j = 0; j < D; ++j) J[i][j] = fma(x, S.dNu[g][a][j], J[i][j]);
      }
    }
    double Ji[D][D];
    if constexpr (D == 1) {
      Ji[0][0] = 1.0 / J[0][0];
    } else {
      const double r = 1.0 / (J[0][0] * J[1][1] - J[0][1] * J[1][0]);
      Ji[0][0] = J[1][1] * r;
      Ji[0][1] = -J[0][1] * r;
      Ji[1][0] = -J[1][0] * r;
      Ji[1][1] = J[0][0] * r;
    }
    double Gu[D][D], ebar = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) Gu[i][j] = 0.0;
    const int64_t o0 = __ldg(doff + n0);
#pragma unroll
    for (int a = 0; a < F::NENU; ++a) {
      const int64_t o = __ldg(doff + ce[a]);
      double gn[D];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) s = fma(Ji[k][j], S.dNu[g][a][k], s);
        gn[j] = s;
      }
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const double u = __ldg(dofs + o + i) - __ldg(dofs + o0 + i);
#pragma unroll
        for (int j = 0; j < D; ++j) Gu[i][j] = fma(u, gn[j], Gu[i][j]);
      }
      if (a < F::NENE) ebar = fma(S.Ne[g][a], __ldg(dofs + o + D), ebar);
    }
    double kap;
    state_record<D>(m, Gu, ebar, kappa[t], k0g ? k0g[t] : m.kappa0, alg ? alg[t] : m.alpha,
                    sdv ? stage + threadIdx.x * W : nullptr, &kap);
    kappa[t] = kap;
  }
  if (sdv) {
    __syncthreads();
    const int64_t nrec = min(int64_t(blockDim.x), ngp - t0);
    const int n = int(nrec) * W;
    double* dst = sdv + t0 * W;
    for (int k = threadIdx.x; k < n; k += blockDim.x) __stcs(dst + k, stage[k]);
  }
}

// Blocked order [u; ebar] of a mixed-order system: one warp per
// blocked row r' (source row perm[r']); the row's u columns first, then its ebar columns, each
// group in source order -- ascending blocked ids, since inv preserves the order within a kind.
// rp_b is built on the host (row lengths are permuted, not changed).  Values move unchanged.
__global__ void k_blocked_mixed(int64_t n, int dim, const int64_t* __restrict__ perm,
                                const int32_t* __restrict__ inv, const uint8_t* __restrict__ kind,
                                const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                const double* __restrict__ val, const double* __restrict__ R,
                                const int64_t* __restrict__ rp_b, int32_t* __restrict__ ci_b,
                                double* __restrict__ val_b, double* __restrict__ R_b) {
  const int64_t r = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  const int64_t src = perm[r];
  const int64_t lo = row_ptr[src], hi = row_ptr[src + 1];
  int nu = 0;   // u columns of the row
  for (int64_t q = lo + lane; q - lane < hi; q += 32) {
    const bool u = q < hi && kind[col_idx[q]] < dim;
    nu += __popc(__ballot_sync(0xffffffffu, u));
  }
  const int64_t dst0 = rp_b[r];
  int cu = 0, ce = 0;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t q = lo + lane; q - lane < hi; q += 32) {
    const bool in = q < hi;
    const int32_t c = in ? col_idx[q] : 0;
    const bool u = in && kind[c] < dim;
    const unsigned bu = __ballot_sync(0xffffffffu, u), be = __ballot_sync(0xffffffffu, in && !u);
    if (in) {
      const int64_t d = dst0 + (u ? cu + __popc(bu & lt) : nu + ce + __popc(be & lt));
      ci_b[d] = inv[c];
      val_b[d] = val[q];
    }
    cu += __popc(bu);
    ce += __popc(be);
  }
  if (lane == 0) R_b[r] = R[src];
}

// ||R_u||^2, ||R_e||^2 by dof kind (kind[i] = component; ebar = dim)
__global__ void k_sumsq_kind(int64_t n, int dim, const uint8_t* __restrict__ kind,
                             const double* __restrict__ R, double* __restrict__ part) {
  double v[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double x = R[i];
    if (kind[i] == dim) v[1] = fma(x, x, v[1]);
    else v[0] = fma(x, x, v[0]);
  }
  block_sum_store<2>(v, part);
}

__global__ void k_delta_sumsq_kind(int64_t n, int dim, const uint8_t* __restrict__ kind,
                                   const double* __restrict__ delta, const double* __restrict__ dofs,
                                   double* __restrict__ part) {
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const bool e = kind[i] == dim;
    const double d = delta[i], u = dofs[i];
    v[e ? 2 : 0] = fma(d, d, v[e ? 2 : 0]);
    v[e ? 3 : 1] = fma(u, u, v[e ? 3 : 1]);
  }
  block_sum_store<4>(v, part);
}

}  // namespace lgdm

// lgdm_device.cuh -- device-side arithmetic of the LGDM K/R assembly (sm_100a, FP64).
//
// The element work is split into three phases so that each FP64 product is formed once:
//   phase A  (one thread per element x Gauss point): geometry (Fig. 3 / Fig. 6: J, det J,
//            grad N), kinematics (Fig. 8b l.7, l.19: eps = B u, ebar = N e, grad ebar),
//            constitutive update (Appendix A; Fig. 8b condition vectors) and the per-node
//            "expansions" of the Voigt tangent into gradient space (NodeRec below);
//   phase C  (one thread per element x node pair a<=b): the Gauss sums of Eqs. 11a-f for the
//            4x4 (Hex8) / 3x3 (Q4) / 2x2 (bar) node-pair blocks (a,b) and (b,a), using the
//            symmetry of Kuu (every term is B^T X B with X symmetric).
// The Voigt tangent of Eq. 11a plus the term of reading R-11a,
//     X = (1-D) C + h_sigma (d d^T + (eeq - ebar) H),
// is isotropic-plus-rank-2 in the basis {m = dI1/deps, s = dJ2/deps}, so
//     Kuu_ab[i][j] = lam* dNa_i dNb_j + mu* (dNa_j dNb_i + delta_ij gNa.gNb)
//                  + Ams (dNa_i (S gNb)_j + (S gNa)_i dNb_j) + Ass (S gNa)_i (S gNb)_j,
// with S the deviatoric strain tensor.  This is the B200 formulation of the paper's
// B_mat' * D_mat * B_mat product (Fig. 7): no B matrix is ever materialised.
#pragma once
#include <cstdint>

namespace lgdm {

// Material constants derived once on the host (Eq. 1, A.1, A.3, A.4).
struct DevMat {
  double E, lam, mu;       // 1D: E; 2D plane strain / 3D: Lame constants
  double k, kappa0, alpha, beta;
  double h, hs, c;         // h, h_sigma, c
  double n, ga, gb;        // g(D) = ga * exp(-n D) + gb   (Eq. A.4 rearranged)
  double t;                // area (1D) / thickness
  double c1, c2, c3;       // Eq. A.3 constants (reading R-A3)
  double i2k, i4k;         // 1 / (2k), 1 / (4k) (host-side; the state record's law)
};

template <int D> struct Fam;
template <> struct Fam<1> {
  static constexpr int DIM = 1, NEN = 2, NDPN = 2, NGP = 2, NS = 1, NPAIR = 3, NDOFE = 4;
};
template <> struct Fam<2> {
  static constexpr int DIM = 2, NEN = 4, NDPN = 3, NGP = 4, NS = 3, NPAIR = 10, NDOFE = 12;
};
template <> struct Fam<3> {
  static constexpr int DIM = 3, NEN = 8, NDPN = 4, NGP = 8, NS = 6, NPAIR = 36, NDOFE = 32;
};

// Per (element, GP, node) record produced by phase A (offsets in doubles, by accessor):
//   gN   grad N_a                    SgN  S grad N_a
//   t1   lam* gN + Ams SgN           t2   Ams gN + Ass SgN
//   WgN  W' grad N_a   (Kue)         DgN  Dt' grad N_a  (Keu)
//   N    N_a                          E    hN N_a + gvec . gN_a   (Kee)
//   F    (Sigma' gN_a, fe0 N_a + fvec . gN_a)   (Fu, Fe)
// All coefficients carry dV and the signs of Eq. 11, so phase C only multiplies and adds.
// Hex8 layout pairs the fields read together so phase C uses 16-byte shared loads:
//   [gN0 gN1][gN2 N][SgN0 SgN1][SgN2 E][t1_0 t1_1][t2_0 t2_1][t1_2 t2_2][WgN0 WgN1]
//   [WgN2 DgN2][DgN0 DgN1][F0 F1][F2 F3][pad pad]     (26 doubles = 13 x 16 B: odd, so
//   8 distinct records of a quarter-warp hit distinct 16-byte bank groups)
template <int D> struct Rec;
template <> struct Rec<3> {
  static constexpr int N = 3, E = 7, STRIDE = 26;
  __host__ __device__ static constexpr int gn(int i) { return i; }
  __host__ __device__ static constexpr int sgn(int i) { return 4 + i; }
  __host__ __device__ static constexpr int t1(int i) { return i < 2 ? 8 + i : 12; }
  __host__ __device__ static constexpr int t2(int i) { return i < 2 ? 10 + i : 13; }
  __host__ __device__ static constexpr int wgn(int i) { return 14 + i; }
  __host__ __device__ static constexpr int dgn(int i) { return i < 2 ? 18 + i : 17; }
  __host__ __device__ static constexpr int f(int i) { return 20 + i; }
};
template <> struct Rec<2> {  // 18 doubles = 9 x 16 B
  static constexpr int N = 12, E = 13, STRIDE = 18;
  __host__ __device__ static constexpr int gn(int i) { return i; }
  __host__ __device__ static constexpr int sgn(int i) { return 2 + i; }
  __host__ __device__ static constexpr int t1(int i) { return 4 + i; }
  __host__ __device__ static constexpr int t2(int i) { return 6 + i; }
  __host__ __device__ static constexpr int wgn(int i) { return 8 + i; }
  __host__ __device__ static constexpr int dgn(int i) { return 10 + i; }
  __host__ __device__ static constexpr int f(int i) { return 14 + i; }
};
template <> struct Rec<1> {  // 10 doubles = 5 x 16 B
  static constexpr int N = 6, E = 7, STRIDE = 10;
  __host__ __device__ static constexpr int gn(int i) { return i; }
  __host__ __device__ static constexpr int sgn(int i) { return 1 + i; }
  __host__ __device__ static constexpr int t1(int i) { return 2 + i; }
  __host__ __device__ static constexpr int t2(int i) { return 3 + i; }
  __host__ __device__ static constexpr int wgn(int i) { return 4 + i; }
  __host__ __device__ static constexpr int dgn(int i) { return 5 + i; }
  __host__ __device__ static constexpr int f(int i) { return 8 + i; }
};
// per (element, GP) scalars used by phase C: mu*, ghc
constexpr int kScal = 2;
// doubles per (element, GP) record block: NEN records, padded to an odd number of 16-byte
// units so consecutive (e,g) blocks start in different bank groups
template <int D> struct GpBlock {
  static constexpr int N = Fam<D>::NEN * Rec<D>::STRIDE;
  static constexpr int STRIDE = ((N / 2) % 2 == 1) ? N : N + 2;
};

// reference node sign r_ak (SURVEY 8c.1 node order) and Gauss point sign s_gk (xi fastest)
template <int D> __device__ __forceinline__ int node_sign(int a, int k) {
  if constexpr (D == 1) return a == 0 ? -1 : 1;
  if (k == 0) return ((a & 3) == 1 || (a & 3) == 2) ? 1 : -1;
  if (k == 1) return ((a & 3) >= 2) ? 1 : -1;
  return a >= 4 ? 1 : -1;
}
__device__ __forceinline__ int gp_sign(int g, int k) { return ((g >> k) & 1) ? 1 : -1; }

// 1D Lagrange factors at xi = +-1/sqrt(3): (1 + r s/sqrt3)/2
#define LGDM_P 0.78867513459481288225   // (1 + 1/sqrt(3)) / 2
#define LGDM_M 0.21132486540518711775   // (1 - 1/sqrt(3)) / 2

template <int D> __device__ __forceinline__ double shapeN(int a, int g) {
  double v = 1.0;
#pragma unroll
  for (int k = 0; k < D; ++k) v *= (node_sign<D>(a, k) == gp_sign(g, k)) ? LGDM_P : LGDM_M;
  return v;
}
template <int D> __device__ __forceinline__ double shape_dxi(int a, int g, int k) {
  double v = 0.5 * node_sign<D>(a, k);
#pragma unroll
  for (int l = 0; l < D; ++l)
    if (l != k) v *= (node_sign<D>(a, l) == gp_sign(g, l)) ? LGDM_P : LGDM_M;
  return v;
}

// symmetric tensor (sym storage 1D [xx]; 2D [xx,yy,xy]; 3D [xx,yy,zz,xy,yz,xz]) times vector
template <int D> __device__ __forceinline__ void symv(const double* T, const double* v, double* o) {
  if constexpr (D == 1) {
    o[0] = T[0] * v[0];
  } else if constexpr (D == 2) {
    o[0] = T[0] * v[0] + T[2] * v[1];
    o[1] = T[2] * v[0] + T[1] * v[1];
  } else {
    o[0] = T[0] * v[0] + T[3] * v[1] + T[5] * v[2];
    o[1] = T[3] * v[0] + T[1] * v[1] + T[4] * v[2];
    o[2] = T[5] * v[0] + T[4] * v[1] + T[2] * v[2];
  }
}

// Compact per-(element, GP) state produced by the core of phase A (offsets in doubles):
//   JI[D*D]  J^-1 (row j, col i = Ji[j][i])     S, WT, DT, SG [NS]  S, W', Dt', Sigma'
//   LAM, AMS, ASS, HN, FE0, MU, GHC               GV[D], FV[D]
template <int D> struct Core {
  static constexpr int NS = Fam<D>::NS;
  static constexpr int JI = 0, S = D * D, WT = S + NS, DT = WT + NS, SG = DT + NS,
                       LAM = SG + NS, AMS = LAM + 1, ASS = AMS + 1, HN = ASS + 1, FE0 = HN + 1,
                       MU = FE0 + 1, GHC = MU + 1, GV = GHC + 1, FV = GV + D;
  static constexpr int USED = FV + D;
  static constexpr int STRIDE = (USED % 2 == 1) ? USED : USED + 1;
};

// Constitutive part of the GP core (Appendix A, Eqs. 2-4, 11a-f coefficients): from the
// Voigt-tensor strain es (tensor shear), ebar, grad ebar, the history kh, the GP's kappa0 /
// alpha, dV and J^-1 to the compact GP state (Core<D> layout).  Shared by the equal-order
// core below and the mixed-order elements (lgdm_mixed.cuh).
template <int D>
__device__ __forceinline__ void gpLaw(const DevMat& m, const double (&Ji)[D][D], double dV,
                                      const double* es, double ebar, const double* gb, double kh,
                                      double k0, double al, double* __restrict__ core) {
  using Co = Core<D>;
  constexpr int NS = Fam<D>::NS;
  // ---- Appendix A: equivalent strain, history, damage, interaction ----
  double I1, eeq, dm, ds;  // d = dm * m + ds * s
  double S[NS];            // deviatoric strain tensor (in-plane part in 2D)
  double A2 = 0.0, Bq = 0.0;  // H = A2 (2 c2 m m^T + c3 P) - Bq q q^T
  if constexpr (D == 1) {
    I1 = es[0];
    eeq = es[0];  // reading R-1D
    dm = 1.0;
    ds = 0.0;
    S[0] = 0.0;
  } else {
    I1 = (D == 2) ? es[0] + es[1] : es[0] + es[1] + es[2];
    const double third = I1 * (1.0 / 3.0);
    double J2;
    if constexpr (D == 2) {
      S[0] = es[0] - third;
      S[1] = es[1] - third;
      S[2] = es[2];
      J2 = 0.5 * (S[0] * S[0] + S[1] * S[1] + third * third) + S[2] * S[2];  // dev_zz = -I1/3
    } else {
      S[0] = es[0] - third;
      S[1] = es[1] - third;
      S[2] = es[2] - third;
      S[3] = es[3];
      S[4] = es[4];
      S[5] = es[5];
      J2 = 0.5 * (S[0] * S[0] + S[1] * S[1] + S[2] * S[2]) + S[3] * S[3] + S[4] * S[4] +
           S[5] * S[5];
    }
    const double Q = m.c2 * I1 * I1 + m.c3 * J2;
    if (Q < 1e-30) {  // reading R-SQ
      eeq = m.c1 * I1 + sqrt(Q) / (2.0 * m.k);
      dm = m.c1;
      ds = 0.0;
    } else {
      const double sQ = sqrt(Q);
      const double r4k = 1.0 / (4.0 * m.k * sQ);
      eeq = m.c1 * I1 + sQ / (2.0 * m.k);
      dm = m.c1 + 2.0 * m.c2 * I1 * r4k;
      ds = m.c3 * r4k;
      A2 = r4k;                       // 1/(4 k sqrt Q)
      Bq = r4k / (2.0 * Q);           // 1/(8 k Q sqrt Q)
    }
  }
  const bool L = (ebar - kh) > 1e-10;                  // Fig. 8b l.22 cond1
  const double kap = L ? ebar : kh;
  double Dm = 0.0, dD = 0.0;
  if (!((kap - k0) < 1e-10)) {                         // Fig. 8b l.27 cond2 (negated)
    const double ex = exp(-m.beta * (kap - k0));
    const double br = 1.0 - al + al * ex;
    const double r = k0 / kap;
    Dm = 1.0 - r * br;                                 // Eq. A.1
    dD = (r / kap) * br + r * al * m.beta * ex;
  }
  const double enD = exp(-m.n * Dm);
  const double gI = m.ga * enD + m.gb;                 // Eq. A.4
  const double gp = -m.n * m.ga * enD * dD;            // dg/dkappa
  const double Lf = L ? 1.0 : 0.0;
  const double rho = eeq - ebar;

  // ---- coefficients of the gradient-space tangent (all x dV, signs of Eq. 11) ----
  double lamS, muS, Ams, Ass;
  double Wt[NS], Dt[NS], Sg[NS];
  if constexpr (D == 1) {
    lamS = dV * (m.E * (1.0 - Dm) + m.hs);
    muS = 0.0;
    Ams = 0.0;
    Ass = 0.0;
    const double Ce = m.E * es[0];
    Wt[0] = -dV * (Ce * dD * Lf + m.hs);
    Dt[0] = -m.h * dV;
    Sg[0] = -dV * ((1.0 - Dm) * Ce + m.hs * rho);
  } else {
    const double c2I1 = 2.0 * m.c2 * I1;
    lamS = dV * (m.lam * (1.0 - Dm) +
                 m.hs * (dm * dm + rho * (A2 * (2.0 * m.c2 - m.c3 * (1.0 / 3.0)) - Bq * c2I1 * c2I1)));
    muS = dV * (m.mu * (1.0 - Dm) + m.hs * rho * A2 * m.c3 * 0.5);
    Ams = dV * m.hs * (dm * ds - rho * Bq * c2I1 * m.c3);
    Ass = dV * m.hs * (ds * ds - rho * Bq * m.c3 * m.c3);
    // C eps as a tensor: lam I1 I + 2 mu eps
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      const bool diag = q < D;
      const double Ce = (diag ? m.lam * I1 : 0.0) + 2.0 * m.mu * es[q];
      const double dt = (diag ? dm : 0.0) + ds * S[q];  // tensor form of d
      Wt[q] = -dV * (Ce * dD * Lf + m.hs * dt);           // Kue (11b)
      Dt[q] = -m.h * dV * dt;                              // Keu (11c)
      Sg[q] = -dV * ((1.0 - Dm) * Ce + m.hs * rho * dt);   // Fu  (11e), sigma of Eq. 2
    }
  }
  const double hN = m.h * dV;
  const double ghc = gI * m.h * m.c * dV;
  const double fe0 = m.h * dV * rho;
  double gv[D], fv[D];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    gv[i] = m.h * m.c * gp * Lf * dV * gb[i];  // Kee gradient term (11d, reading R-kappa')
    fv[i] = -ghc * gb[i];                      // Fe gradient term (11f, reading R-11f)
  }
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int i = 0; i < D; ++i) core[Co::JI + j * D + i] = Ji[j][i];
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    core[Co::S + q] = S[q];
    core[Co::WT + q] = Wt[q];
    core[Co::DT + q] = Dt[q];
    core[Co::SG + q] = Sg[q];
  }
  core[Co::LAM] = lamS;
  core[Co::AMS] = Ams;
  core[Co::ASS] = Ass;
  core[Co::HN] = hN;
  core[Co::FE0] = fe0;
  core[Co::MU] = muS;
  core[Co::GHC] = ghc;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    core[Co::GV + i] = gv[i];
    core[Co::FV + i] = fv[i];
  }
}

// ---------------------------------------------------------------------------------------
// Phase A, part 1 ("core"): one Gauss point g of one element.  X [NEN][D] coords,
// U [NEN][NDPN] dofs, kh = kappa_hist.  Writes the compact GP state (Core<D> layout) to core.
// Returns det J (caller treats <= 0 as an inverted element).
// ---------------------------------------------------------------------------------------
// Shape values are supplied by SHD(a, j) = dN_a/dxi_j and SHN(a) = N_a at the Gauss point
// (gpCore below passes the closed forms; kernels may pass register copies of a table).
// k0 / al: the GP's damage threshold kappa0 and alpha (defect regions; the material's
// values unless per-GP fields are set, lgdm_set_defects).
template <int D, class XF, class UF, class SD, class SN>
__device__ __forceinline__ double gpCoreSK(const DevMat& m, XF&& X, UF&& U, double kh, double k0,
                                           double al, SD&& SHD, SN&& SHN, double* __restrict__ core) {
  using F = Fam<D>;
  constexpr int NEN = F::NEN, NS = F::NS;

  // geometry: J_ij = sum_a X_ai dN_a/dxi_j = sum_{a>0} (X_ai - X_0i) dN_a/dxi_j (reading R-REL:
  // sum_a dN_a = 0; exact differences instead of the cancellation of |X| >> element size)
  double J[D][D];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) J[i][j] = 0.0;
#pragma unroll
  for (int a = 1; a < NEN; ++a)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double dn = SHD(a, j);
#pragma unroll
      for (int i = 0; i < D; ++i) J[i][j] = fma(X(a, i) - X(0, i), dn, J[i][j]);
    }
  double detJ, Ji[D][D];
  if constexpr (D == 1) {
    detJ = J[0][0];
    Ji[0][0] = 1.0 / detJ;
  } else if constexpr (D == 2) {
    detJ = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    const double r = 1.0 / detJ;
    Ji[0][0] = J[1][1] * r;
    Ji[0][1] = -J[0][1] * r;
    Ji[1][0] = -J[1][0] * r;
    Ji[1][1] = J[0][0] * r;
  } else {
    const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    detJ = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    const double r = 1.0 / detJ;
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
  const double dV = detJ * m.t;  // Gauss weights are 1

  // grad N_a = J^-T dN/dxi (recomputed where needed instead of kept live); kinematics
  auto gradN = [&](int a, double* gn) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) s = fma(Ji[j][i], SHD(a, j), s);
      gn[i] = s;
    }
  };
  double eps[D][D], ebar = 0.0, gb[D];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    gb[i] = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) eps[i][j] = 0.0;
  }
  ebar = SHN(0) * U(0, D);
#pragma unroll
  for (int a = 1; a < NEN; ++a) {     // gradients from differences to node 0 (R-REL)
    double gn[D];
    gradN(a, gn);
    const double ea = U(a, D);
    ebar = fma(SHN(a), ea, ebar);
    const double de = ea - U(0, D);
#pragma unroll
    for (int i = 0; i < D; ++i) {
      gb[i] = fma(gn[i], de, gb[i]);
      {
        const double ua = U(a, i) - U(0, i);
#pragma unroll
        for (int j = 0; j < D; ++j) eps[i][j] = fma(ua, gn[j], eps[i][j]);
      }
    }
  }
  // symmetrise: eps_ij = (du_i/dx_j + du_j/dx_i)/2
  double es[NS];
  if constexpr (D == 1) {
    es[0] = eps[0][0];
  } else if constexpr (D == 2) {
    es[0] = eps[0][0];
    es[1] = eps[1][1];
    es[2] = 0.5 * (eps[0][1] + eps[1][0]);
  } else {
    es[0] = eps[0][0];
    es[1] = eps[1][1];
    es[2] = eps[2][2];
    es[3] = 0.5 * (eps[0][1] + eps[1][0]);
    es[4] = 0.5 * (eps[1][2] + eps[2][1]);
    es[5] = 0.5 * (eps[0][2] + eps[2][0]);
  }

  gpLaw<D>(m, Ji, dV, es, ebar, gb, kh, k0, al, core);
  return detJ;
}


template <int D, class XF, class UF, class SD, class SN>
__device__ __forceinline__ double gpCoreS(const DevMat& m, XF&& X, UF&& U, double kh, SD&& SHD,
                                          SN&& SHN, double* __restrict__ core) {
  return gpCoreSK<D>(m, X, U, kh, m.kappa0, m.alpha, SHD, SHN, core);
}

// Core of one GP with the closed-form shape functions at Gauss point g.
template <int D, class XF, class UF>
__device__ __forceinline__ double gpCore(const DevMat& m, XF&& X, UF&& U, double kh, int g,
                                         double* __restrict__ core) {
  return gpCoreS<D>(m, X, U, kh, [&](int a, int j) { return shape_dxi<D>(a, g, j); },
                    [&](int a) { return shapeN<D>(a, g); }, core);
}

// Phase A, part 2 ("expansion"): the record of node a at GP g from the compact state.
template <int D>
__device__ __forceinline__ void gpExpand(const double* __restrict__ core, int a, int g,
                                         double* __restrict__ r) {
  using Co = Core<D>;
  using R = Rec<D>;
  double gn[D], SgN[D], WgN[D], DgN[D], fu[D];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) s = fma(core[Co::JI + j * D + i], shape_dxi<D>(a, g, j), s);
    gn[i] = s;
  }
  symv<D>(core + Co::S, gn, SgN);
  symv<D>(core + Co::WT, gn, WgN);
  symv<D>(core + Co::DT, gn, DgN);
  symv<D>(core + Co::SG, gn, fu);
  const double Na = shapeN<D>(a, g);
  const double lamS = core[Co::LAM], Ams = core[Co::AMS], Ass = core[Co::ASS];
  double gvd = 0.0, fvd = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    r[R::gn(i)] = gn[i];
    r[R::sgn(i)] = SgN[i];
    r[R::t1(i)] = fma(lamS, gn[i], Ams * SgN[i]);
    r[R::t2(i)] = fma(Ams, gn[i], Ass * SgN[i]);
    r[R::wgn(i)] = WgN[i];
    r[R::dgn(i)] = DgN[i];
    r[R::f(i)] = fu[i];
    gvd = fma(core[Co::GV + i], gn[i], gvd);
    fvd = fma(core[Co::FV + i], gn[i], fvd);
  }
  r[R::N] = Na;
  r[R::E] = fma(core[Co::HN], Na, gvd);
  r[R::f(D)] = fma(core[Co::FE0], Na, fvd);
}

// Phase A for one GP, all nodes (general path): core into registers, then expansions.
template <int D>
__device__ __forceinline__ double phaseA(const DevMat& m, const double* __restrict__ X,
                                         const double* __restrict__ U, double kh, double k0,
                                         double al, int g, double* __restrict__ rec,
                                         double* __restrict__ scal) {
  double core[Core<D>::STRIDE];
  const double detJ = gpCoreSK<D>(
      m, [&](int a, int i) { return X[a * D + i]; },
      [&](int a, int i) { return U[a * Fam<D>::NDPN + i]; }, kh, k0, al,
      [&](int a, int j) { return shape_dxi<D>(a, g, j); }, [&](int a) { return shapeN<D>(a, g); },
      core);
#pragma unroll
  for (int a = 0; a < Fam<D>::NEN; ++a) gpExpand<D>(core, a, g, rec + a * Rec<D>::STRIDE);
  scal[0] = core[Core<D>::MU];
  scal[1] = core[Core<D>::GHC];
  return detJ;
}

// pair index -> (a, b), a <= b, row-major upper triangle
template <int NEN> __device__ __forceinline__ void pair_ab(int p, int& a, int& b) {
  int aa = 0, rem = p;
  while (rem >= NEN - aa) {
    rem -= NEN - aa;
    ++aa;
  }
  a = aa;
  b = aa + rem;
}

// Phase C accumulators for one node pair (a,b), a <= b.
template <int D> struct PairAcc {
  double Kuu[D][D];     // Kuu_ab (Kuu_ba = transpose)
  double Kue_ab[D], Kue_ba[D], Keu_ab[D], Keu_ba[D];
  double Kee_ab, Kee_ba;
  double Fd[D + 1];     // F of node a (diagonal pairs only)
};

// Gauss sum of one node pair: recs [NGP][GpBlock::STRIDE], per-GP scalars (mu*, ghc) at
// scal[g * SCAL_STRIDE + MU_OFF / GHC_OFF].
template <int D> struct PairIn {
  double gA[D], sA[D], wA[D], dA[D], NA, EA;   // row node a
  double gB[D], t1[D], t2[D], wB[D], dB[D], NB, EB;   // column node b
};
template <int D>
__device__ __forceinline__ void load_pair(const double* __restrict__ A, const double* __restrict__ B,
                                          PairIn<D>& in) {
  using R = Rec<D>;
  if constexpr (D == 3) {
    const double2* A2 = reinterpret_cast<const double2*>(A);
    const double2* B2 = reinterpret_cast<const double2*>(B);
    double2 v;
    v = A2[0]; in.gA[0] = v.x; in.gA[1] = v.y;
    v = A2[1]; in.gA[2] = v.x; in.NA = v.y;
    v = A2[2]; in.sA[0] = v.x; in.sA[1] = v.y;
    v = A2[3]; in.sA[2] = v.x; in.EA = v.y;
    v = A2[7]; in.wA[0] = v.x; in.wA[1] = v.y;
    v = A2[8]; in.wA[2] = v.x; in.dA[2] = v.y;
    v = A2[9]; in.dA[0] = v.x; in.dA[1] = v.y;
    v = B2[0]; in.gB[0] = v.x; in.gB[1] = v.y;
    v = B2[1]; in.gB[2] = v.x; in.NB = v.y;
    v = B2[4]; in.t1[0] = v.x; in.t1[1] = v.y;
    v = B2[5]; in.t2[0] = v.x; in.t2[1] = v.y;
    v = B2[6]; in.t1[2] = v.x; in.t2[2] = v.y;
    v = B2[7]; in.wB[0] = v.x; in.wB[1] = v.y;
    v = B2[8]; in.wB[2] = v.x; in.dB[2] = v.y;
    v = B2[9]; in.dB[0] = v.x; in.dB[1] = v.y;
    in.EB = B[R::E];
  } else {
#pragma unroll
    for (int i = 0; i < D; ++i) {
      in.gA[i] = A[R::gn(i)]; in.sA[i] = A[R::sgn(i)]; in.wA[i] = A[R::wgn(i)]; in.dA[i] = A[R::dgn(i)];
      in.gB[i] = B[R::gn(i)]; in.t1[i] = B[R::t1(i)]; in.t2[i] = B[R::t2(i)];
      in.wB[i] = B[R::wgn(i)]; in.dB[i] = B[R::dgn(i)];
    }
    in.NA = A[R::N]; in.EA = A[R::E]; in.NB = B[R::N]; in.EB = B[R::E];
  }
}

template <int D>
__device__ __forceinline__ void accumulate_pair(const PairIn<D>& in, double mu, double ghc,
                                                PairAcc<D>& acc) {
  double dot = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) dot = fma(in.gA[i], in.gB[i], dot);
#pragma unroll
  for (int i = 0; i < D; ++i) {
    const double ub = mu * in.gB[i];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double v = acc.Kuu[i][j];
      v = fma(in.gA[i], in.t1[j], v);
      v = fma(in.sA[i], in.t2[j], v);
      v = fma(in.gA[j], ub, v);
      acc.Kuu[i][j] = v;
    }
    acc.Kuu[i][i] = fma(mu, dot, acc.Kuu[i][i]);
  }
#pragma unroll
  for (int i = 0; i < D; ++i) {
    acc.Kue_ab[i] = fma(in.NB, in.wA[i], acc.Kue_ab[i]);
    acc.Kue_ba[i] = fma(in.NA, in.wB[i], acc.Kue_ba[i]);
    acc.Keu_ab[i] = fma(in.NA, in.dB[i], acc.Keu_ab[i]);
    acc.Keu_ba[i] = fma(in.NB, in.dA[i], acc.Keu_ba[i]);
  }
  acc.Kee_ab = fma(in.NB, in.EA, fma(ghc, dot, acc.Kee_ab));
  acc.Kee_ba = fma(in.NA, in.EB, fma(ghc, dot, acc.Kee_ba));
}

template <int D, int SCAL_STRIDE = kScal, int MU_OFF = 0, int GHC_OFF = 1>
__device__ __forceinline__ void phaseC(const double* __restrict__ recs,
                                       const double* __restrict__ scal, int a, int b,
                                       PairAcc<D>& acc) {
  using F = Fam<D>;
  using R = Rec<D>;
  constexpr int GB = GpBlock<D>::STRIDE;
#pragma unroll
  for (int i = 0; i < D; ++i) {
#pragma unroll
    for (int j = 0; j < D; ++j) acc.Kuu[i][j] = 0.0;
    acc.Kue_ab[i] = acc.Kue_ba[i] = acc.Keu_ab[i] = acc.Keu_ba[i] = 0.0;
  }
  acc.Kee_ab = acc.Kee_ba = 0.0;
#pragma unroll
  for (int i = 0; i <= D; ++i) acc.Fd[i] = 0.0;
  const double* Ab = recs + a * R::STRIDE;
  const double* Bb = recs + b * R::STRIDE;
#pragma unroll 2
  for (int g = 0; g < F::NGP; ++g) {
    PairIn<D> in;
    load_pair<D>(Ab + g * GB, Bb + g * GB, in);
    accumulate_pair<D>(in, scal[g * SCAL_STRIDE + MU_OFF], scal[g * SCAL_STRIDE + GHC_OFF], acc);
  }
  if (a == b) {
#pragma unroll 1
    for (int g = 0; g < F::NGP; ++g)
#pragma unroll
      for (int i = 0; i <= D; ++i) acc.Fd[i] += Ab[g * GB + R::f(i)];
  }
}

// Element-block entry (row r, col c) setter for an accumulated pair, via callback
// put(a_local, i, b_local, j, value).
template <int D, class Put>
__device__ __forceinline__ void emit_pair(int a, int b, const PairAcc<D>& acc, Put&& put) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
      put(a, i, b, j, acc.Kuu[i][j]);
      if (a != b) put(b, j, a, i, acc.Kuu[i][j]);
    }
    put(a, i, b, D, acc.Kue_ab[i]);
    put(a, D, b, i, acc.Keu_ab[i]);
    if (a != b) {
      put(b, i, a, D, acc.Kue_ba[i]);
      put(b, D, a, i, acc.Keu_ba[i]);
    }
  }
  put(a, D, b, D, acc.Kee_ab);
  if (a != b) put(b, D, a, D, acc.Kee_ba);
}

}  // namespace lgdm

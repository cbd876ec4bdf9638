// lgdm_oracle.cpp -- plain, slow, obviously-correct CPU oracle for the LGDM K/R assembly.
//
// TEST INFRASTRUCTURE ONLY (see lgdm_oracle.h).  Nothing under paper_2301_06503_b200/ or
// include/ uses this file; it shares no code with the CUDA path.
//
// Structure follows Algorithm 1 of PAPER.md: loop over elements, loop over Gauss
// points, form K_local / F_local from Eqs. 11a-f with the constitutive laws of
// Appendix A, then assemble.  Dense matrices are used throughout (B_u, N, B_e,
// C, the Voigt tangent X) so that each line can be checked against the printed equations.
// The readings of garbled / ambiguous passages are the ones listed in DESIGN.md
// ("Readings of the paper"): R-A3 (de Vree eq. strain), R-PS, R-SH, R-1D, R-11a (h_sigma),
// R-11f (sign), R-kappa' (L factor in 11b and 11d), R-TH (Fig. 8b thresholds), R-SQ, R-PAT.
//
// Compiled with -O2 -ffp-contract=off (no fused multiply-add, no fast-math).
#include "lgdm_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <set>
#include <vector>

#include <omp.h>

namespace {

const double kTolHist = 1e-10;  // Fig. 8b l.22: cond1 = (gp_e_eqv - k0) > 1D-10
const double kTolDam = 1e-10;   // Fig. 8b l.27: cond2 = (k_gp - ki) < 1D-10

struct Fam {
  int dim, nen, ndpn, nv, ngp, ndofe;
};

bool family(int type, Fam* f) {
  switch (type) {
    case 1: *f = {1, 2, 2, 1, 2, 4}; return true;     // 2-node bar, (u, ebar) per node
    case 2: *f = {2, 4, 3, 3, 4, 12}; return true;    // Q4 plane strain, (ux, uy, ebar)
    case 3: *f = {3, 8, 4, 6, 8, 32}; return true;    // Hex8, (ux, uy, uz, ebar)
    default: return false;
  }
}

// Reference node coordinates: bar -1,+1; Q4 counter-clockwise; Hex8 bottom
// face counter-clockwise then top face.
void ref_node(int type, int a, double* xa) {
  static const double q[4][2] = {{-1, -1}, {1, -1}, {1, 1}, {-1, 1}};
  if (type == 1) {
    xa[0] = a == 0 ? -1.0 : 1.0;
  } else if (type == 2) {
    xa[0] = q[a][0];
    xa[1] = q[a][1];
  } else {
    xa[0] = q[a % 4][0];
    xa[1] = q[a % 4][1];
    xa[2] = a < 4 ? -1.0 : 1.0;
  }
}

// Voigt layout of the engineering strain: 1D [e]; 2D [xx, yy, gxy]; 3D [xx, yy, zz, gxy, gyz, gxz].
// voigt_pair(dim, V) gives the tensor index pair (p, q) of Voigt component V.
void voigt_pair(int dim, int V, int* p, int* q) {
  static const int p2[3][2] = {{0, 0}, {1, 1}, {0, 1}};
  static const int p3[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {1, 2}, {0, 2}};
  if (dim == 1) { *p = 0; *q = 0; return; }
  const int(*t)[2] = dim == 2 ? p2 : p3;
  *p = t[V][0];
  *q = t[V][1];
}

// Elasticity matrix C (Voigt, engineering shear).  1D: E.  2D: plane strain.  3D: isotropic.
void elasticity(const oracle_material* m, int dim, double* C) {
  if (dim == 1) { C[0] = m->E; return; }
  const double lam = m->E * m->nu / ((1.0 + m->nu) * (1.0 - 2.0 * m->nu));
  const double mu = m->E / (2.0 * (1.0 + m->nu));
  const int nv = dim == 2 ? 3 : 6;
  for (int V = 0; V < nv * nv; ++V) C[V] = 0.0;
  for (int V = 0; V < nv; ++V) {
    int p, q;
    voigt_pair(dim, V, &p, &q);
    if (p == q) {
      for (int W = 0; W < nv; ++W) {
        int r, s;
        voigt_pair(dim, W, &r, &s);
        if (r == s) C[V * nv + W] = lam;
      }
      C[V * nv + V] = lam + 2.0 * mu;
    } else {
      C[V * nv + V] = mu;
    }
  }
}

}  // namespace

extern "C" {

// Eq. A.1 with the Fig. 8b threshold: D = 0 when kappa - kappa0 < 1e-10.
void oracle_damage(const oracle_material* m, double kappa, double* D, double* dD) {
  if (kappa - m->kappa0 < kTolDam) {
    *D = 0.0;
    *dD = 0.0;
    return;
  }
  const double ex = std::exp(-m->beta * (kappa - m->kappa0));
  const double brace = 1.0 - m->alpha + m->alpha * ex;
  *D = 1.0 - (m->kappa0 / kappa) * brace;
  // d/dkappa of 1 - (k0/kappa)*brace  =  (k0/kappa^2)*brace + (k0/kappa)*alpha*beta*ex
  *dD = (m->kappa0 / (kappa * kappa)) * brace + (m->kappa0 / kappa) * m->alpha * m->beta * ex;
}

// Eq. A.4: g(D) = ((1-R) e^{-nD} + R - e^{-n}) / (1 - e^{-n}).
void oracle_interaction(const oracle_material* m, double D, double* g, double* dgdD) {
  const double en = std::exp(-m->n);
  const double enD = std::exp(-m->n * D);
  *g = ((1.0 - m->R) * enD + m->R - en) / (1.0 - en);
  *dgdD = -m->n * (1.0 - m->R) * enD / (1.0 - en);
}

// Eq. A.3, de Vree reading R-A3 (eq_variant 0) or the printed constants (1):
//   eeq = c1 I1 + 1/(2k) sqrt(c2 I1^2 + c3 J2),  I1 = tr eps,  J2 = 1/2 dev(eps):dev(eps)
//   c1 = (k-1)/(2k(1-2nu)),  c2 = ((k-1)/(1-2nu))^2,  c3 = 12k/(1+nu)^2  [literal: 2k/(1-nu)^2].
// The strain tensor is rebuilt from Voigt (plane strain: eps33 = 0, reading R-PS; tensor
// shear = gamma/2, reading R-SH).  d and H are the first and second derivatives with respect
// to the Voigt vector, by the chain rule through I1 and J2.  1D: eeq = eps (reading R-1D).
void oracle_eqstrain(const oracle_material* m, int dim, const double* ev, double* eeq, double* d,
                     double* H) {
  if (dim == 1) {
    *eeq = ev[0];
    d[0] = 1.0;
    H[0] = 0.0;
    return;
  }
  const int nv = dim == 2 ? 3 : 6;
  double eps[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int V = 0; V < nv; ++V) {
    int p, q;
    voigt_pair(dim, V, &p, &q);
    if (p == q) {
      eps[p][p] = ev[V];
    } else {
      eps[p][q] = 0.5 * ev[V];
      eps[q][p] = 0.5 * ev[V];
    }
  }
  const double I1 = eps[0][0] + eps[1][1] + eps[2][2];
  double dev[3][3];
  for (int p = 0; p < 3; ++p)
    for (int q = 0; q < 3; ++q) dev[p][q] = eps[p][q] - (p == q ? I1 / 3.0 : 0.0);
  double J2 = 0.0;
  for (int p = 0; p < 3; ++p)
    for (int q = 0; q < 3; ++q) J2 += 0.5 * dev[p][q] * dev[p][q];

  const double k = m->k, nu = m->nu;
  const double c1 = (k - 1.0) / (2.0 * k * (1.0 - 2.0 * nu));
  const double c2 = ((k - 1.0) / (1.0 - 2.0 * nu)) * ((k - 1.0) / (1.0 - 2.0 * nu));
  const double c3 = m->eq_variant == 1 ? 2.0 * k / ((1.0 - nu) * (1.0 - nu))
                                       : 12.0 * k / ((1.0 + nu) * (1.0 + nu));
  const double Q = c2 * I1 * I1 + c3 * J2;
  const double sQ = std::sqrt(Q);
  *eeq = c1 * I1 + sQ / (2.0 * k);

  // dI1/deps_v = mvec; dJ2/deps_v = svec; d2J2/deps_v^2 = P.
  double mvec[6], svec[6], P[36];
  for (int V = 0; V < nv; ++V) {
    int p, q;
    voigt_pair(dim, V, &p, &q);
    mvec[V] = p == q ? 1.0 : 0.0;
    svec[V] = p == q ? dev[p][p] : eps[p][q];  // d(1/2 dev:dev)/d eps_pp = dev_pp; /d gamma = eps_pq
    for (int W = 0; W < nv; ++W) {
      int r, s;
      voigt_pair(dim, W, &r, &s);
      double v = 0.0;
      if (p == q && r == s) v = (p == r ? 1.0 : 0.0) - 1.0 / 3.0;
      if (p != q && V == W) v = 0.5;
      P[V * nv + W] = v;
    }
  }
  if (Q < 1e-30) {  // reading R-SQ: sqrt term not differentiable at zero strain
    for (int V = 0; V < nv; ++V) {
      d[V] = c1 * mvec[V];
      for (int W = 0; W < nv; ++W) H[V * nv + W] = 0.0;
    }
    return;
  }
  double qv[6];
  for (int V = 0; V < nv; ++V) qv[V] = 2.0 * c2 * I1 * mvec[V] + c3 * svec[V];  // dQ/deps_v
  for (int V = 0; V < nv; ++V) {
    d[V] = c1 * mvec[V] + qv[V] / (4.0 * k * sQ);
    for (int W = 0; W < nv; ++W) {
      const double dq = 2.0 * c2 * mvec[V] * mvec[W] + c3 * P[V * nv + W];
      H[V * nv + W] = dq / (4.0 * k * sQ) - qv[V] * qv[W] / (8.0 * k * Q * sQ);
    }
  }
}

int oracle_gauss(int type, double* xi, double* w) {
  Fam f;
  if (!family(type, &f)) return -1;
  const double a = 1.0 / std::sqrt(3.0);
  for (int g = 0; g < f.ngp; ++g) {
    for (int k = 0; k < f.dim; ++k) xi[g * f.dim + k] = ((g >> k) & 1) ? a : -a;  // xi fastest
    w[g] = 1.0;
  }
  return f.ngp;
}

void oracle_shape(int type, const double* xi, double* N, double* dNdxi) {
  Fam f;
  if (!family(type, &f)) return;
  const double scale = 1.0 / double(1 << f.dim);
  for (int a = 0; a < f.nen; ++a) {
    double xa[3];
    ref_node(type, a, xa);
    double prod = scale;
    for (int k = 0; k < f.dim; ++k) prod *= (1.0 + xa[k] * xi[k]);
    N[a] = prod;
    for (int k = 0; k < f.dim; ++k) {
      double v = scale * xa[k];
      for (int l = 0; l < f.dim; ++l)
        if (l != k) v *= (1.0 + xa[l] * xi[l]);
      dNdxi[a * f.dim + k] = v;
    }
  }
}

int oracle_element(int type, const oracle_material* m, const double* Xe, const double* Ue,
                   const double* kap, double* Ke, double* Fe, double* Fabs, double* sig,
                   int32_t* guard) {
  return oracle_element_d(type, m, Xe, Ue, kap, nullptr, nullptr, Ke, Fe, Fabs, sig, guard);
}

// Same, with per-GP damage threshold kappa0 and alpha (defect regions; the code's
// per-GP `ki` and `alpha_var`, Fig. 9a l.3-4 / P:380-389).  NULL = the material's value.
int oracle_element_d(int type, const oracle_material* m0, const double* Xe, const double* Ue,
                     const double* kap, const double* k0g, const double* alg, double* Ke,
                     double* Fe, double* Fabs, double* sig, int32_t* guard) {
  oracle_material mg = *m0;   // per-GP damage parameters (defect fields) set in the GP loop
  const oracle_material* m = &mg;
  Fam f;
  if (!family(type, &f)) return -1000;
  const int dim = f.dim, nen = f.nen, ndpn = f.ndpn, nv = f.nv, nd = f.ndofe;
  double xi[24], w[8];
  oracle_gauss(type, xi, w);
  double C[36];
  elasticity(m, dim, C);
  for (int r = 0; r < nd * nd; ++r) Ke[r] = 0.0;
  for (int r = 0; r < nd; ++r) Fe[r] = 0.0, Fabs[r] = 0.0;

  for (int g = 0; g < f.ngp; ++g) {  // Alg. 1 line 5: for igp = 1..ngp
    // ---- geometry (Fig. 3, gp_data): J, det J, grad N ----
    double N[8], dNdxi[24];
    oracle_shape(type, xi + g * dim, N, dNdxi);
    // J = sum_a X_a dN_a/dxi with coordinates relative to node 0 (reading R-REL: the same sum,
    // sum_a dN_a/dxi = 0; exact differences instead of the cancellation of |X| >> element size)
    double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int a = 0; a < nen; ++a)
      for (int i = 0; i < dim; ++i)
        for (int j = 0; j < dim; ++j) J[i][j] += (Xe[a * dim + i] - Xe[i]) * dNdxi[a * dim + j];
    double detJ, Ji[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    if (dim == 1) {
      detJ = J[0][0];
      Ji[0][0] = 1.0 / J[0][0];
    } else if (dim == 2) {
      detJ = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      Ji[0][0] = J[1][1] / detJ;
      Ji[0][1] = -J[0][1] / detJ;
      Ji[1][0] = -J[1][0] / detJ;
      Ji[1][1] = J[0][0] / detJ;
    } else {
      detJ = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
             J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
             J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
      Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / detJ;
      Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / detJ;
      Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / detJ;
      Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / detJ;
      Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / detJ;
      Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / detJ;
      Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / detJ;
      Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / detJ;
      Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / detJ;
    }
    if (!(detJ > 0.0)) return -(g + 1);
    double gradN[8][3];  // dN_a/dx_i = sum_j Jinv[j][i] dN_a/dxi_j   (grad_x N = J^-T grad_xi N)
    for (int a = 0; a < nen; ++a)
      for (int i = 0; i < dim; ++i) {
        double s = 0.0;
        for (int j = 0; j < dim; ++j) s += Ji[j][i] * dNdxi[a * dim + j];
        gradN[a][i] = s;
      }
    const double dV = w[g] * detJ * m->t;

    // ---- full-width operators over the element dof vector (node-interleaved) ----
    // Bu [nv x nd] (strain-displacement, Voigt, engineering shear), Ne [nd], Be [dim x nd].
    double Bu[6][32], Ne[32], Be[3][32];
    for (int r = 0; r < nd; ++r) {
      Ne[r] = 0.0;
      for (int V = 0; V < 6; ++V) Bu[V][r] = 0.0;
      for (int i = 0; i < 3; ++i) Be[i][r] = 0.0;
    }
    for (int a = 0; a < nen; ++a) {
      for (int V = 0; V < nv; ++V) {
        int p, q;
        voigt_pair(dim, V, &p, &q);
        if (p == q) {
          Bu[V][a * ndpn + p] = gradN[a][p];
        } else {
          Bu[V][a * ndpn + p] = gradN[a][q];
          Bu[V][a * ndpn + q] = gradN[a][p];
        }
      }
      Ne[a * ndpn + dim] = N[a];
      for (int i = 0; i < dim; ++i) Be[i][a * ndpn + dim] = gradN[a][i];
    }

    // ---- kinematics (Fig. 5b l.12, l.17): eps = B u, ebar = N e, grad ebar = B_e e ----
    // (R-REL: B u and grad ebar on the dofs relative to node 0's -- B annihilates constants;
    // ebar = N e on the absolute values)
    double Ur[32];
    for (int r = 0; r < nd; ++r) Ur[r] = Ue[r] - Ue[r % ndpn];
    double ev[6] = {0, 0, 0, 0, 0, 0}, ebar = 0.0, gbar[3] = {0, 0, 0};
    for (int r = 0; r < nd; ++r) {
      for (int V = 0; V < nv; ++V) ev[V] += Bu[V][r] * Ur[r];
      ebar += Ne[r] * Ue[r];
      for (int i = 0; i < dim; ++i) gbar[i] += Be[i][r] * Ur[r];
    }

    // ---- constitutive (Appendix A; Fig. 8b condition vectors) ----
    mg.kappa0 = k0g ? k0g[g] : m0->kappa0;
    mg.alpha = alg ? alg[g] : m0->alpha;
    double eeq, dv[6], H[36];
    oracle_eqstrain(m, dim, ev, &eeq, dv, H);
    const double kh = kap[g];
    const bool L = (ebar - kh) > kTolHist;                    // cond1
    const double kappa = L ? ebar : kh;
    double D, dD;
    oracle_damage(m, kappa, &D, &dD);                         // cond2 inside
    double gI, dgdD;
    oracle_interaction(m, D, &gI, &dgdD);
    const double gprime = dgdD * dD;                          // dg/dkappa
    const double Lf = L ? 1.0 : 0.0;                          // d kappa / d ebar (reading R-kappa')
    if (guard) {
      const double sc = 1e-14 * std::max(std::fabs(ebar), m->kappa0);
      guard[g] = (std::fabs(ebar - kh - kTolHist) < sc ||
                  std::fabs(kappa - m->kappa0 - kTolDam) < sc) ? 1 : 0;
    }

    // Eq. 2: sigma = (1-D) C eps + h_sigma (eeq - ebar) d
    double Ceps[6], sv[6];
    for (int V = 0; V < nv; ++V) {
      double s = 0.0;
      for (int W = 0; W < nv; ++W) s += C[V * nv + W] * ev[W];
      Ceps[V] = s;
      sv[V] = (1.0 - D) * Ceps[V] + m->h_sigma * (eeq - ebar) * dv[V];
    }
    if (sig)
      for (int V = 0; V < nv; ++V) sig[g * nv + V] = sv[V];

    // Voigt tangent of Eq. 11a with the term of reading R-11a:
    //   X = (1-D) C + h_sigma (d d^T + (eeq - ebar) H)
    double X[36];
    for (int V = 0; V < nv; ++V)
      for (int W = 0; W < nv; ++W)
        X[V * nv + W] = (1.0 - D) * C[V * nv + W] +
                        m->h_sigma * (dv[V] * dv[W] + (eeq - ebar) * H[V * nv + W]);
    // Eq. 11b: w = C eps dD/dkappa dkappa/debar + h_sigma d
    double wv[6];
    for (int V = 0; V < nv; ++V) wv[V] = Ceps[V] * dD * Lf + m->h_sigma * dv[V];

    // XB = X Bu  [nv x nd]
    double XB[6][32];
    for (int V = 0; V < nv; ++V)
      for (int c = 0; c < nd; ++c) {
        double s = 0.0;
        for (int W = 0; W < nv; ++W) s += X[V * nv + W] * Bu[W][c];
        XB[V][c] = s;
      }

    for (int r = 0; r < nd; ++r) {
      double btw = 0.0, btsig = 0.0, btsig_abs = 0.0, bg = 0.0, bg_abs = 0.0;
      for (int V = 0; V < nv; ++V) {
        btw += Bu[V][r] * wv[V];
        btsig += Bu[V][r] * sv[V];
        btsig_abs += std::fabs(Bu[V][r]) * (std::fabs((1.0 - D) * Ceps[V]) +
                                            std::fabs(m->h_sigma * (eeq - ebar) * dv[V]));
      }
      for (int i = 0; i < dim; ++i) {
        bg += Be[i][r] * gbar[i];
        bg_abs += std::fabs(Be[i][r]) * std::fabs(gbar[i]);
      }
      for (int c = 0; c < nd; ++c) {
        double kuu = 0.0, bb = 0.0;
        for (int V = 0; V < nv; ++V) kuu += Bu[V][r] * XB[V][c];  // 11a: Bu^T X Bu
        for (int i = 0; i < dim; ++i) bb += Be[i][r] * Be[i][c];
        double kue = -btw * Ne[c];                                // 11b: -Bu^T w N
        double keu = 0.0;                                         // 11c: -N^T h d^T Bu
        for (int V = 0; V < nv; ++V) keu += -Ne[r] * m->h * dv[V] * Bu[V][c];
        double kee = m->h * Ne[r] * Ne[c]                         // 11d: N^T h N
                     + m->h * m->c * gprime * Lf * bg * Ne[c]     //      + B^T h c g' grad ebar N
                     + gI * m->h * m->c * bb;                     //      + B^T g h c B
        Ke[r * nd + c] += dV * (kuu + kue + keu + kee);
      }
      // 11e (t = 0): -Bu^T sigma;  11f (reading R-11f): N h (eeq-ebar) - B^T g h c grad ebar
      Fe[r] += dV * (-btsig + m->h * Ne[r] * (eeq - ebar) - gI * m->h * m->c * bg);
      Fabs[r] += dV * (btsig_abs + m->h * std::fabs(Ne[r] * (eeq - ebar)) +
                       gI * m->h * m->c * bg_abs);
    }
  }
  return 0;
}

// ---------------- pattern (reading R-PAT) ----------------

static void node_neighbours(int type, int64_t n_nodes, int64_t n_elems, const int64_t* conn,
                            std::vector<std::set<int64_t>>* nb) {
  Fam f;
  family(type, &f);
  nb->assign(n_nodes, std::set<int64_t>());
  for (int64_t e = 0; e < n_elems; ++e)
    for (int a = 0; a < f.nen; ++a)
      for (int b = 0; b < f.nen; ++b) (*nb)[conn[e * f.nen + a]].insert(conn[e * f.nen + b]);
}

int64_t oracle_pattern_nnz(int type, int64_t n_nodes, int64_t n_elems, const int64_t* conn) {
  Fam f;
  if (!family(type, &f)) return -1;
  std::vector<std::set<int64_t>> nb;
  node_neighbours(type, n_nodes, n_elems, conn, &nb);
  int64_t nnz = 0;
  for (int64_t a = 0; a < n_nodes; ++a) nnz += int64_t(nb[a].size()) * f.ndpn * f.ndpn;
  return nnz;
}

int oracle_pattern(int type, int64_t n_nodes, int64_t n_elems, const int64_t* conn,
                   int64_t* row_ptr, int32_t* col_idx) {
  Fam f;
  if (!family(type, &f)) return -1;
  std::vector<std::set<int64_t>> nb;
  node_neighbours(type, n_nodes, n_elems, conn, &nb);
  int64_t pos = 0;
  row_ptr[0] = 0;
  for (int64_t a = 0; a < n_nodes; ++a)
    for (int i = 0; i < f.ndpn; ++i) {
      for (int64_t b : nb[a])  // std::set iterates in ascending order
        for (int j = 0; j < f.ndpn; ++j) col_idx[pos++] = int32_t(f.ndpn * b + j);
      row_ptr[a * f.ndpn + i + 1] = pos;
    }
  return 0;
}

static int64_t find_col(const int64_t* row_ptr, const int32_t* col_idx, int64_t row, int64_t col) {
  const int32_t* lo = col_idx + row_ptr[row];
  const int32_t* hi = col_idx + row_ptr[row + 1];
  const int32_t* it = std::lower_bound(lo, hi, int32_t(col));
  if (it == hi || *it != col) return -1;
  return it - col_idx;
}

static void gather(const Fam& f, int64_t e, const int64_t* conn, const double* coords,
                   const double* dofs, double* Xe, double* Ue) {
  for (int a = 0; a < f.nen; ++a) {
    const int64_t n = conn[e * f.nen + a];
    for (int i = 0; i < f.dim; ++i) Xe[a * f.dim + i] = coords[n * f.dim + i];
    for (int i = 0; i < f.ndpn; ++i) Ue[a * f.ndpn + i] = dofs[n * f.ndpn + i];
  }
}

// Alg. 1 lines 4-11; Fig. 2: element loop, K_local, unroll, assemble.
int oracle_assemble(int type, const oracle_material* m, int64_t n_nodes, const double* coords,
                    int64_t n_elems, const int64_t* conn, const double* dofs, const double* kappa,
                    const int64_t* row_ptr, const int32_t* col_idx, double* val, double* R,
                    double* S, int64_t* n_guard) {
  return oracle_assemble_d(type, m, n_nodes, coords, n_elems, conn, dofs, kappa, nullptr, nullptr,
                           row_ptr, col_idx, val, R, S, n_guard);
}

// One element of Alg. 1 lines 5-10: K_local, F_local, then the scatter into K and R.
static int assemble_one(const Fam& f, int type, const oracle_material* m, int64_t e,
                        const double* coords, const int64_t* conn, const double* dofs,
                        const double* kappa, const double* kappa0_gp, const double* alpha_gp,
                        const int64_t* row_ptr, const int32_t* col_idx, double* val, double* R,
                        double* S, double* Ke, double* Fe, double* Fa, int64_t* ng) {
  const int nd = f.ndofe;
  double Xe[24], Ue[32];
  int32_t guard[8];
  gather(f, e, conn, coords, dofs, Xe, Ue);
  const int rc = oracle_element_d(type, m, Xe, Ue, kappa + e * f.ngp,
                                  kappa0_gp ? kappa0_gp + e * f.ngp : nullptr,
                                  alpha_gp ? alpha_gp + e * f.ngp : nullptr, Ke, Fe, Fa, nullptr,
                                  guard);
  if (rc != 0) return -2;  // det J <= 0
  for (int g = 0; g < f.ngp; ++g) *ng += guard[g];
  for (int a = 0; a < f.nen; ++a)
    for (int i = 0; i < f.ndpn; ++i) {
      const int64_t row = f.ndpn * conn[e * f.nen + a] + i;
      const int r = a * f.ndpn + i;
      R[row] += Fe[r];
      S[row] += Fa[r];
      for (int b = 0; b < f.nen; ++b)
        for (int j = 0; j < f.ndpn; ++j) {
          const int64_t col = f.ndpn * conn[e * f.nen + b] + j;
          const int64_t p = find_col(row_ptr, col_idx, row, col);
          if (p < 0) return -3;
          val[p] += Ke[r * nd + b * f.ndpn + j];
        }
    }
  return 0;
}

int oracle_assemble_d(int type, const oracle_material* m, int64_t n_nodes, const double* coords,
                      int64_t n_elems, const int64_t* conn, const double* dofs,
                      const double* kappa, const double* kappa0_gp, const double* alpha_gp,
                      const int64_t* row_ptr, const int32_t* col_idx, double* val, double* R,
                      double* S, int64_t* n_guard) {
  Fam f;
  if (!family(type, &f)) return -1;
  const int nd = f.ndofe;
  const int64_t ndof = n_nodes * f.ndpn;
  std::fill(val, val + row_ptr[ndof], 0.0);
  std::fill(R, R + ndof, 0.0);
  std::fill(S, S + ndof, 0.0);
  std::vector<double> Ke(nd * nd), Fe(nd), Fa(nd);
  int64_t ng = 0;
  for (int64_t e = 0; e < n_elems; ++e) {
    const int rc = assemble_one(f, type, m, e, coords, conn, dofs, kappa, kappa0_gp, alpha_gp,
                                row_ptr, col_idx, val, R, S, Ke.data(), Fe.data(), Fa.data(), &ng);
    if (rc != 0) return rc;
  }
  if (n_guard) *n_guard = ng;
  return 0;
}

// The same element loop on all host cores (SURVEY 8d oracle timing (b); used for the CPU
// baseline only -- parity uses the serial loop above): elements are visited colour by colour;
// elements of one colour share no node (caller's colouring, e.g. the 2^d parities of a
// structured grid), so the scatter of one colour is race-free.  Entries are summed in
// (colour, element) order instead of element order.  Returns the thread count used in *threads.
int oracle_assemble_colored(int type, const oracle_material* m, int64_t n_nodes,
                            const double* coords, int64_t n_elems, const int64_t* conn,
                            const double* dofs, const double* kappa, const int32_t* colour,
                            int n_colours, const int64_t* row_ptr, const int32_t* col_idx,
                            double* val, double* R, double* S, int nthreads, int* threads) {
  Fam f;
  if (!family(type, &f)) return -1;
  const int nd = f.ndofe;
  const int64_t ndof = n_nodes * f.ndpn;
  std::fill(val, val + row_ptr[ndof], 0.0);
  std::fill(R, R + ndof, 0.0);
  std::fill(S, S + ndof, 0.0);
  std::vector<std::vector<int64_t>> by(n_colours);
  for (int64_t e = 0; e < n_elems; ++e) {
    if (colour[e] < 0 || colour[e] >= n_colours) return -4;
    by[colour[e]].push_back(e);
  }
  if (nthreads > 0) omp_set_num_threads(nthreads);
  int used = 1, rc_all = 0;
  for (int c = 0; c < n_colours; ++c) {
    const std::vector<int64_t>& el = by[c];
#pragma omp parallel
    {
      std::vector<double> Ke(nd * nd), Fe(nd), Fa(nd);
      int64_t ng = 0;
#pragma omp single
      used = omp_get_num_threads();
#pragma omp for schedule(static)
      for (int64_t k = 0; k < int64_t(el.size()); ++k) {
        const int rc = assemble_one(f, type, m, el[k], coords, conn, dofs, kappa, nullptr, nullptr,
                                    row_ptr, col_idx, val, R, S, Ke.data(), Fe.data(), Fa.data(), &ng);
        if (rc != 0) {
#pragma omp critical
          rc_all = rc;
        }
      }
    }
    if (rc_all != 0) return rc_all;
  }
  if (threads) *threads = used;
  return 0;
}

// Sampled rows: the same sums restricted to the block-rows of selected nodes.
static void adjacency(const Fam& f, int64_t n_nodes, int64_t n_elems, const int64_t* conn,
                      std::vector<std::vector<int64_t>>* adj, const std::vector<char>& want) {
  adj->assign(n_nodes, std::vector<int64_t>());
  for (int64_t e = 0; e < n_elems; ++e)
    for (int a = 0; a < f.nen; ++a) {
      const int64_t n = conn[e * f.nen + a];
      if (want[n]) (*adj)[n].push_back(e);  // ascending e by construction
    }
}

int64_t oracle_rows_nnz(int type, int64_t n_nodes, int64_t n_elems, const int64_t* conn,
                        int64_t n_sel, const int64_t* sel) {
  Fam f;
  if (!family(type, &f)) return -1;
  std::vector<char> want(n_nodes, 0);
  for (int64_t s = 0; s < n_sel; ++s) want[sel[s]] = 1;
  std::vector<std::vector<int64_t>> adj;
  adjacency(f, n_nodes, n_elems, conn, &adj, want);
  int64_t nnz = 0;
  for (int64_t s = 0; s < n_sel; ++s) {
    std::set<int64_t> nb;
    for (int64_t e : adj[sel[s]])
      for (int b = 0; b < f.nen; ++b) nb.insert(conn[e * f.nen + b]);
    nnz += int64_t(nb.size()) * f.ndpn * f.ndpn;
  }
  return nnz;
}

int oracle_assemble_rows(int type, const oracle_material* m, int64_t n_nodes, const double* coords,
                         int64_t n_elems, const int64_t* conn, const double* dofs,
                         const double* kappa, int64_t n_sel, const int64_t* sel,
                         int64_t* row_ptr_sel, int32_t* col_idx_sel, double* val_sel,
                         double* R_sel, double* S_sel) {
  Fam f;
  if (!family(type, &f)) return -1;
  const int nd = f.ndofe;
  std::vector<char> want(n_nodes, 0);
  for (int64_t s = 0; s < n_sel; ++s) want[sel[s]] = 1;
  std::vector<std::vector<int64_t>> adj;
  adjacency(f, n_nodes, n_elems, conn, &adj, want);
  std::vector<double> Ke(nd * nd), Fe(nd), Fa(nd);
  double Xe[24], Ue[32];
  int64_t pos = 0;
  row_ptr_sel[0] = 0;
  for (int64_t s = 0; s < n_sel; ++s) {
    const int64_t a0 = sel[s];
    std::set<int64_t> nbset;
    for (int64_t e : adj[a0])
      for (int b = 0; b < f.nen; ++b) nbset.insert(conn[e * f.nen + b]);
    std::vector<int64_t> nb(nbset.begin(), nbset.end());
    const int64_t width = int64_t(nb.size()) * f.ndpn;
    const int64_t base = pos;
    for (int i = 0; i < f.ndpn; ++i) {
      for (int64_t b : nb)
        for (int j = 0; j < f.ndpn; ++j) {
          col_idx_sel[pos] = int32_t(f.ndpn * b + j);
          val_sel[pos] = 0.0;
          ++pos;
        }
      row_ptr_sel[s * f.ndpn + i + 1] = pos;
      R_sel[s * f.ndpn + i] = 0.0;
      S_sel[s * f.ndpn + i] = 0.0;
    }
    for (int64_t e : adj[a0]) {
      gather(f, e, conn, coords, dofs, Xe, Ue);
      if (oracle_element(type, m, Xe, Ue, kappa + e * f.ngp, Ke.data(), Fe.data(), Fa.data(),
                         nullptr, nullptr) != 0)
        return -2;
      for (int a = 0; a < f.nen; ++a) {
        if (conn[e * f.nen + a] != a0) continue;
        for (int i = 0; i < f.ndpn; ++i) {
          const int r = a * f.ndpn + i;
          R_sel[s * f.ndpn + i] += Fe[r];
          S_sel[s * f.ndpn + i] += Fa[r];
          for (int b = 0; b < f.nen; ++b) {
            const int64_t slot =
                std::lower_bound(nb.begin(), nb.end(), conn[e * f.nen + b]) - nb.begin();
            for (int j = 0; j < f.ndpn; ++j)
              val_sel[base + i * width + slot * f.ndpn + j] += Ke[r * nd + b * f.ndpn + j];
          }
        }
      }
    }
  }
  return 0;
}

// Eq. A.2 with Fig. 8b l.19-24:
//   ebar_gp = N(xi_g) e;  cond1 = (ebar_gp - kappa) > 1e-10;  kappa(cond1) = ebar_gp.
int oracle_update_history(int type, int64_t n_nodes, int64_t n_elems, const int64_t* conn,
                          const double* dofs, double* kappa) {
  Fam f;
  if (!family(type, &f)) return -1;
  (void)n_nodes;
  double xi[24], w[8], N[8], dNdxi[24];
  oracle_gauss(type, xi, w);
  for (int64_t e = 0; e < n_elems; ++e)
    for (int g = 0; g < f.ngp; ++g) {
      oracle_shape(type, xi + g * f.dim, N, dNdxi);
      double ebar = 0.0;
      for (int a = 0; a < f.nen; ++a) ebar += N[a] * dofs[conn[e * f.nen + a] * f.ndpn + f.dim];
      double& k = kappa[e * f.ngp + g];
      if ((ebar - k) > kTolHist) k = ebar;
    }
  return 0;
}

// J^-1 by cofactors (as in oracle_element); false if det J <= 0.
static bool invert(int dim, const double (&J)[3][3], double (&Ji)[3][3]) {
  double detJ;
  if (dim == 1) {
    detJ = J[0][0];
    Ji[0][0] = 1.0 / detJ;
  } else if (dim == 2) {
    detJ = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    Ji[0][0] = J[1][1] / detJ;
    Ji[0][1] = -J[0][1] / detJ;
    Ji[1][0] = -J[1][0] / detJ;
    Ji[1][1] = J[0][0] / detJ;
  } else {
    detJ = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
           J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
           J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / detJ;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / detJ;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / detJ;
    Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / detJ;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / detJ;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / detJ;
    Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / detJ;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / detJ;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / detJ;
  }
  return detJ > 0.0;
}

// State-variable update (Alg. 2 l.8-14, Fig. 9a `update_variables`),
// one record of oracle_sdv_width(type) doubles per (element, GP):
//   [strain eps_v (nv, Voigt, engineering shear; Fig. 9a l.7 `B_mat_u*udof`)]
//   [d eeq / d eps_v (nv; Alg. 2 l.11, Eq. A.3)]
//   [sigma (nv; Eq. 2 with the reading-R-11a term h_sigma (eeq - ebar) d)]
//   [eeq (Eq. A.3, Fig. 9a l.11-16), ebar (Fig. 9a l.19), kappa (history, l.22-24),
//    D (Eq. A.1, l.27-31), g (Eq. A.4, Alg. 2 l.12)]
// and commits the history kappa <- kappa (as oracle_update_history).  kappa0_gp / alpha_gp:
// per-GP damage threshold and alpha (defect regions), NULL = material value.
int oracle_sdv_width(int type) {
  Fam f;
  if (!family(type, &f)) return -1;
  return 3 * f.nv + 5;
}

int oracle_update_state(int type, const oracle_material* m, int64_t n_nodes, const double* coords,
                        int64_t n_elems, const int64_t* conn, const double* dofs, double* kappa,
                        const double* kappa0_gp, const double* alpha_gp, double* sdv) {
  Fam f;
  if (!family(type, &f)) return -1;
  (void)n_nodes;
  const int dim = f.dim, nen = f.nen, ndpn = f.ndpn, nv = f.nv;
  const int W = 3 * nv + 5;
  double xi[24], w[8], C[36];
  oracle_gauss(type, xi, w);
  elasticity(m, dim, C);
  double Xe[24], Ue[32];
  for (int64_t e = 0; e < n_elems; ++e) {
    gather(f, e, conn, coords, dofs, Xe, Ue);
    for (int g = 0; g < f.ngp; ++g) {
      double N[8], dNdxi[24];
      oracle_shape(type, xi + g * dim, N, dNdxi);
      // J_ij = sum_a X_ai dN_a/dxi_j; grad_x N = J^-T grad_xi N (as oracle_element)
      double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, Ji[3][3];
      for (int a = 0; a < nen; ++a)   // relative to node 0 (R-REL)
        for (int i = 0; i < dim; ++i)
          for (int j = 0; j < dim; ++j) J[i][j] += (Xe[a * dim + i] - Xe[i]) * dNdxi[a * dim + j];
      if (!invert(dim, J, Ji)) return -2;
      double gradN[8][3];
      for (int a = 0; a < nen; ++a)
        for (int i = 0; i < dim; ++i) {
          double s = 0.0;
          for (int j = 0; j < dim; ++j) s += Ji[j][i] * dNdxi[a * dim + j];
          gradN[a][i] = s;
        }
      // strain (Voigt, engineering shear) and ebar at the GP
      double ev[6] = {0, 0, 0, 0, 0, 0}, ebar = 0.0;
      for (int a = 0; a < nen; ++a) {
        for (int V = 0; V < nv; ++V) {
          int p, q;
          voigt_pair(dim, V, &p, &q);
          if (p == q) ev[V] += gradN[a][p] * (Ue[a * ndpn + p] - Ue[p]);
          else ev[V] += gradN[a][q] * (Ue[a * ndpn + p] - Ue[p]) + gradN[a][p] * (Ue[a * ndpn + q] - Ue[q]);
        }
        ebar += N[a] * Ue[a * ndpn + dim];
      }
      oracle_material mg = *m;
      if (kappa0_gp) mg.kappa0 = kappa0_gp[e * f.ngp + g];
      if (alpha_gp) mg.alpha = alpha_gp[e * f.ngp + g];
      double eeq, dv[6], H[36];
      oracle_eqstrain(&mg, dim, ev, &eeq, dv, H);
      double& kh = kappa[e * f.ngp + g];
      const double kap = (ebar - kh) > kTolHist ? ebar : kh;   // Fig. 9a l.22-24
      double D, dD, gI, dg;
      oracle_damage(&mg, kap, &D, &dD);
      oracle_interaction(&mg, D, &gI, &dg);
      double* out = sdv + (e * f.ngp + g) * W;
      for (int V = 0; V < nv; ++V) {
        double ce = 0.0;
        for (int U = 0; U < nv; ++U) ce += C[V * nv + U] * ev[U];
        out[V] = ev[V];
        out[nv + V] = dv[V];
        out[2 * nv + V] = (1.0 - D) * ce + m->h_sigma * (eeq - ebar) * dv[V];   // Eq. 2
      }
      out[3 * nv + 0] = eeq;
      out[3 * nv + 1] = ebar;
      out[3 * nv + 2] = kap;
      out[3 * nv + 3] = D;
      out[3 * nv + 4] = gI;
      kh = kap;
    }
  }
  return 0;
}

// ||R restricted to u-rows||_2 and ||R restricted to ebar-rows||_2.
void oracle_residual_norms(int type, int64_t n_rows, const double* R, double* out2) {
  Fam f;
  family(type, &f);
  double su = 0.0, se = 0.0;
  for (int64_t r = 0; r < n_rows; ++r) {
    if (r % f.ndpn == f.dim) se += R[r] * R[r];
    else su += R[r] * R[r];
  }
  out2[0] = std::sqrt(su);
  out2[1] = std::sqrt(se);
}

}  // extern "C"

// =========================================================================================
// Mixed-order elements: quadratic u with linear ebar, the paper's own
// discretisation ("shape functions for displacement (u) are taken as quadratic, and for
// micro-equivalent strain as linear"; 1D bar P:418; 2D SEN P:466).
//   type 4 = BAR3:  3-node quadratic bar for u (local nodes xi = -1, +1, 0), ebar on the two
//                   end nodes (linear), 3-point Gauss.
//   type 5 = QUAD8: 8-node serendipity quad for u (corners counter-clockwise, then midsides
//                   (0,-1), (1,0), (0,1), (-1,0)), ebar bilinear on the 4 corners, 3x3 Gauss
//                   (reading R-Q8: the paper's "biquadratic" with Fig. 6's 8 shape rows).
// Geometry is isoparametric on the u nodes (reading R-GEO).  The corner ("ebar") nodes are
// the first nene local nodes.  Local element dofs are node-major: corner node a has
// (u_0..u_{d-1}, ebar) at a*(d+1); midside node a >= nene has (u_0..u_{d-1}) at
// nene*(d+1) + (a-nene)*d.  Global dofs are node-interleaved with a variable count per node:
// dof = doff[node] + comp, doff the prefix sum of (d+1 for ebar-carrying nodes, d otherwise)
// (reading R-ORD extended).
// =========================================================================================
namespace {

struct MFam {
  int dim, nenu, nene, nv, ngp, ndofe;
};

bool mfamily(int type, MFam* f) {
  switch (type) {
    case 4: *f = {1, 3, 2, 1, 3, 5}; return true;      // 3 u + 2 ebar dofs
    case 5: *f = {2, 8, 4, 3, 9, 20}; return true;     // 16 u + 4 ebar dofs
    default: return false;
  }
}

int mldof(const MFam& f, int a) {
  return a < f.nene ? a * (f.dim + 1) : f.nene * (f.dim + 1) + (a - f.nene) * f.dim;
}

// reference coordinates of the u nodes
void mref_node(int type, int a, double* xa) {
  static const double q8[8][2] = {{-1, -1}, {1, -1}, {1, 1}, {-1, 1},
                                  {0, -1},  {1, 0},  {0, 1}, {-1, 0}};
  if (type == 4) xa[0] = a == 0 ? -1.0 : (a == 1 ? 1.0 : 0.0);
  else { xa[0] = q8[a][0]; xa[1] = q8[a][1]; }
}

}  // namespace

extern "C" {

int oracle_mixed_family(int type, int32_t* out6) {
  MFam f;
  if (!mfamily(type, &f)) return -1;
  out6[0] = f.dim; out6[1] = f.nenu; out6[2] = f.nene; out6[3] = f.nv; out6[4] = f.ngp;
  out6[5] = f.ndofe;
  return 0;
}

// 3-point Gauss-Legendre per direction: xi = -sqrt(3/5), 0, +sqrt(3/5); w = 5/9, 8/9, 5/9
// (xi fastest in 2D).
int oracle_mixed_gauss(int type, double* xi, double* w) {
  MFam f;
  if (!mfamily(type, &f)) return -1;
  const double p[3] = {-std::sqrt(3.0 / 5.0), 0.0, std::sqrt(3.0 / 5.0)};
  const double q[3] = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
  for (int g = 0; g < f.ngp; ++g) {
    const int gx = g % 3, gy = g / 3;
    xi[g * f.dim] = p[gx];
    w[g] = q[gx];
    if (f.dim == 2) {
      xi[g * f.dim + 1] = p[gy];
      w[g] *= q[gy];
    }
  }
  return f.ngp;
}

// u shape functions.  BAR3: N = xi(xi-1)/2, xi(xi+1)/2, 1-xi^2.  QUAD8 serendipity:
// corner  N = 1/4 (1+xi xa)(1+eta ea)(xi xa + eta ea - 1);
// midside xa = 0: N = 1/2 (1-xi^2)(1+eta ea);  ea = 0: N = 1/2 (1+xi xa)(1-eta^2).
void oracle_mixed_shape_u(int type, const double* xi, double* N, double* dNdxi) {
  if (type == 4) {
    const double x = xi[0];
    N[0] = 0.5 * x * (x - 1.0);
    N[1] = 0.5 * x * (x + 1.0);
    N[2] = 1.0 - x * x;
    dNdxi[0] = x - 0.5;
    dNdxi[1] = x + 0.5;
    dNdxi[2] = -2.0 * x;
    return;
  }
  const double x = xi[0], y = xi[1];
  for (int a = 0; a < 8; ++a) {
    double r[2];
    mref_node(type, a, r);
    const double xa = r[0], ea = r[1];
    if (a < 4) {
      N[a] = 0.25 * (1.0 + x * xa) * (1.0 + y * ea) * (x * xa + y * ea - 1.0);
      dNdxi[a * 2 + 0] = 0.25 * xa * (1.0 + y * ea) * (2.0 * x * xa + y * ea);
      dNdxi[a * 2 + 1] = 0.25 * ea * (1.0 + x * xa) * (x * xa + 2.0 * y * ea);
    } else if (xa == 0.0) {
      N[a] = 0.5 * (1.0 - x * x) * (1.0 + y * ea);
      dNdxi[a * 2 + 0] = -x * (1.0 + y * ea);
      dNdxi[a * 2 + 1] = 0.5 * ea * (1.0 - x * x);
    } else {
      N[a] = 0.5 * (1.0 + x * xa) * (1.0 - y * y);
      dNdxi[a * 2 + 0] = 0.5 * xa * (1.0 - y * y);
      dNdxi[a * 2 + 1] = -y * (1.0 + x * xa);
    }
  }
}

// ebar shape functions: linear on the corners (BAR2 / Q4 of the corner nodes).
void oracle_mixed_shape_e(int type, const double* xi, double* N, double* dNdxi) {
  MFam f;
  if (!mfamily(type, &f)) return;
  for (int a = 0; a < f.nene; ++a) {
    double r[2];
    mref_node(type, a, r);
    if (f.dim == 1) {
      N[a] = 0.5 * (1.0 + r[0] * xi[0]);
      dNdxi[a] = 0.5 * r[0];
    } else {
      N[a] = 0.25 * (1.0 + r[0] * xi[0]) * (1.0 + r[1] * xi[1]);
      dNdxi[a * 2 + 0] = 0.25 * r[0] * (1.0 + r[1] * xi[1]);
      dNdxi[a * 2 + 1] = 0.25 * r[1] * (1.0 + r[0] * xi[0]);
    }
  }
}

// Element blocks of Eqs. 11a-f for a mixed element: identical integrands to
// oracle_element_d; B_u from the u shape functions over the u dofs, N_e / B_e from the ebar
// shape functions over the ebar dofs; dV = w_g det J t.
int oracle_mixed_element(int type, const oracle_material* m0, const double* Xe, const double* Ue,
                         const double* kap, const double* k0g, const double* alg, double* Ke,
                         double* Fe, double* Fabs, double* sig) {
  oracle_material mg = *m0;
  const oracle_material* m = &mg;
  MFam f;
  if (!mfamily(type, &f)) return -1000;
  const int dim = f.dim, nv = f.nv, nd = f.ndofe;
  double xi[18], w[9];
  oracle_mixed_gauss(type, xi, w);
  double C[36];
  elasticity(m, dim, C);
  for (int r = 0; r < nd * nd; ++r) Ke[r] = 0.0;
  for (int r = 0; r < nd; ++r) Fe[r] = 0.0, Fabs[r] = 0.0;

  for (int g = 0; g < f.ngp; ++g) {
    double Nu[8], dNu[16], Nn[4], dNe[8];
    oracle_mixed_shape_u(type, xi + g * dim, Nu, dNu);
    oracle_mixed_shape_e(type, xi + g * dim, Nn, dNe);
    // J = sum_a X_a dN_a/dxi, with the coordinates taken relative to node 0 (reading R-REL:
    // the same sum since sum_a dN_a/dxi = 0; exact differences instead of the cancellation of
    // |X| >> element size)
    double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, Ji[3][3];
    for (int a = 0; a < f.nenu; ++a)
      for (int i = 0; i < dim; ++i)
        for (int j = 0; j < dim; ++j) J[i][j] += (Xe[a * dim + i] - Xe[i]) * dNu[a * dim + j];
    const double detJ = dim == 1 ? J[0][0] : J[0][0] * J[1][1] - J[0][1] * J[1][0];
    if (!invert(dim, J, Ji)) return -(g + 1);
    double gNu[8][3], gNe[4][3];
    for (int a = 0; a < f.nenu; ++a)
      for (int i = 0; i < dim; ++i) {
        double s = 0.0;
        for (int j = 0; j < dim; ++j) s += Ji[j][i] * dNu[a * dim + j];
        gNu[a][i] = s;
      }
    for (int a = 0; a < f.nene; ++a)
      for (int i = 0; i < dim; ++i) {
        double s = 0.0;
        for (int j = 0; j < dim; ++j) s += Ji[j][i] * dNe[a * dim + j];
        gNe[a][i] = s;
      }
    const double dV = w[g] * detJ * m->t;

    // full-width operators over the element dof vector
    double Bu[6][20], Ne[20], Be[3][20];
    for (int r = 0; r < nd; ++r) {
      Ne[r] = 0.0;
      for (int V = 0; V < 6; ++V) Bu[V][r] = 0.0;
      for (int i = 0; i < 3; ++i) Be[i][r] = 0.0;
    }
    for (int a = 0; a < f.nenu; ++a) {
      const int o = mldof(f, a);
      for (int V = 0; V < nv; ++V) {
        int p, q;
        voigt_pair(dim, V, &p, &q);
        if (p == q) {
          Bu[V][o + p] = gNu[a][p];
        } else {
          Bu[V][o + p] = gNu[a][q];
          Bu[V][o + q] = gNu[a][p];
        }
      }
    }
    for (int a = 0; a < f.nene; ++a) {
      const int o = mldof(f, a) + dim;
      Ne[o] = Nn[a];
      for (int i = 0; i < dim; ++i) Be[i][o] = gNe[a][i];
    }

    // eps = B_u u, grad ebar = B_e e on the dofs relative to node 0's (R-REL: B annihilates
    // constants); ebar = N_e e on the absolute values
    double Ur[20];
    for (int r = 0; r < nd; ++r) {
      const int a = r < f.nene * (dim + 1) ? r / (dim + 1) : f.nene + (r - f.nene * (dim + 1)) / dim;
      const int comp = r - mldof(f, a);
      Ur[r] = Ue[r] - Ue[comp];   // node 0 is a corner: (u_0.., ebar_0) at local dofs 0..dim
    }
    double ev[6] = {0, 0, 0, 0, 0, 0}, ebar = 0.0, gbar[3] = {0, 0, 0};
    for (int r = 0; r < nd; ++r) {
      for (int V = 0; V < nv; ++V) ev[V] += Bu[V][r] * Ur[r];
      ebar += Ne[r] * Ue[r];
      for (int i = 0; i < dim; ++i) gbar[i] += Be[i][r] * Ur[r];
    }

    mg.kappa0 = k0g ? k0g[g] : m0->kappa0;
    mg.alpha = alg ? alg[g] : m0->alpha;
    double eeq, dv[6], H[36];
    oracle_eqstrain(m, dim, ev, &eeq, dv, H);
    const double kh = kap[g];
    const bool L = (ebar - kh) > kTolHist;
    const double kappa = L ? ebar : kh;
    double D, dD;
    oracle_damage(m, kappa, &D, &dD);
    double gI, dgdD;
    oracle_interaction(m, D, &gI, &dgdD);
    const double gprime = dgdD * dD;
    const double Lf = L ? 1.0 : 0.0;

    double Ceps[6], sv[6];
    for (int V = 0; V < nv; ++V) {
      double s = 0.0;
      for (int W = 0; W < nv; ++W) s += C[V * nv + W] * ev[W];
      Ceps[V] = s;
      sv[V] = (1.0 - D) * Ceps[V] + m->h_sigma * (eeq - ebar) * dv[V];
    }
    if (sig)
      for (int V = 0; V < nv; ++V) sig[g * nv + V] = sv[V];
    double X[36];
    for (int V = 0; V < nv; ++V)
      for (int W = 0; W < nv; ++W)
        X[V * nv + W] = (1.0 - D) * C[V * nv + W] +
                        m->h_sigma * (dv[V] * dv[W] + (eeq - ebar) * H[V * nv + W]);
    double wv[6];
    for (int V = 0; V < nv; ++V) wv[V] = Ceps[V] * dD * Lf + m->h_sigma * dv[V];
    double XB[6][20];
    for (int V = 0; V < nv; ++V)
      for (int c = 0; c < nd; ++c) {
        double s = 0.0;
        for (int W = 0; W < nv; ++W) s += X[V * nv + W] * Bu[W][c];
        XB[V][c] = s;
      }
    for (int r = 0; r < nd; ++r) {
      double btw = 0.0, btsig = 0.0, btsig_abs = 0.0, bg = 0.0, bg_abs = 0.0;
      for (int V = 0; V < nv; ++V) {
        btw += Bu[V][r] * wv[V];
        btsig += Bu[V][r] * sv[V];
        btsig_abs += std::fabs(Bu[V][r]) * (std::fabs((1.0 - D) * Ceps[V]) +
                                            std::fabs(m->h_sigma * (eeq - ebar) * dv[V]));
      }
      for (int i = 0; i < dim; ++i) {
        bg += Be[i][r] * gbar[i];
        bg_abs += std::fabs(Be[i][r]) * std::fabs(gbar[i]);
      }
      for (int c = 0; c < nd; ++c) {
        double kuu = 0.0, bb = 0.0;
        for (int V = 0; V < nv; ++V) kuu += Bu[V][r] * XB[V][c];       // 11a
        for (int i = 0; i < dim; ++i) bb += Be[i][r] * Be[i][c];
        double kue = -btw * Ne[c];                                     // 11b
        double keu = 0.0;                                              // 11c
        for (int V = 0; V < nv; ++V) keu += -Ne[r] * m->h * dv[V] * Bu[V][c];
        double kee = m->h * Ne[r] * Ne[c] + m->h * m->c * gprime * Lf * bg * Ne[c] +
                     gI * m->h * m->c * bb;                            // 11d
        Ke[r * nd + c] += dV * (kuu + kue + keu + kee);
      }
      Fe[r] += dV * (-btsig + m->h * Ne[r] * (eeq - ebar) - gI * m->h * m->c * bg);   // 11e, 11f
      Fabs[r] += dV * (btsig_abs + m->h * std::fabs(Ne[r] * (eeq - ebar)) +
                       gI * m->h * m->c * bg_abs);
    }
  }
  return 0;
}

// Global dof offsets: doff[n] = first dof of node n, doff[n_nodes] = ndof.  A node carries
// ebar iff it is a corner (local index < nene) of its elements.  Returns ndof, or -1 when a
// node is a corner of one element and a midside node of another, or is referenced by none.
int64_t oracle_mixed_dofs(int type, int64_t n_nodes, int64_t n_elems, const int64_t* conn,
                          int64_t* doff) {
  MFam f;
  if (!mfamily(type, &f)) return -1;
  std::vector<int> kind(n_nodes, 0);   // 0 unused, 1 corner, 2 midside
  for (int64_t e = 0; e < n_elems; ++e)
    for (int a = 0; a < f.nenu; ++a) {
      const int k = a < f.nene ? 1 : 2;
      int& s = kind[conn[e * f.nenu + a]];
      if (s != 0 && s != k) return -1;
      s = k;
    }
  doff[0] = 0;
  for (int64_t n = 0; n < n_nodes; ++n) {
    if (kind[n] == 0) return -1;
    doff[n + 1] = doff[n] + (kind[n] == 1 ? f.dim + 1 : f.dim);
  }
  return doff[n_nodes];
}

// Pattern (reading R-PAT): every dof pair of two nodes sharing an element (explicit zeros
// kept); rows in dof order, ascending global columns.
int64_t oracle_mixed_pattern(int type, int64_t n_nodes, int64_t n_elems, const int64_t* conn,
                             const int64_t* doff, int64_t* row_ptr, int32_t* col_idx) {
  MFam f;
  if (!mfamily(type, &f)) return -1;
  std::vector<std::set<int64_t>> nb(n_nodes);
  for (int64_t e = 0; e < n_elems; ++e)
    for (int a = 0; a < f.nenu; ++a)
      for (int b = 0; b < f.nenu; ++b) nb[conn[e * f.nenu + a]].insert(conn[e * f.nenu + b]);
  int64_t pos = 0;
  if (row_ptr) row_ptr[0] = 0;
  for (int64_t a = 0; a < n_nodes; ++a)
    for (int64_t r = doff[a]; r < doff[a + 1]; ++r) {
      for (int64_t b : nb[a])
        for (int64_t c = doff[b]; c < doff[b + 1]; ++c) {
          if (col_idx) col_idx[pos] = int32_t(c);
          ++pos;
        }
      if (row_ptr) row_ptr[r + 1] = pos;
    }
  return pos;
}

// Alg. 1 l.4-11 for mixed elements: element loop, K_local, scatter into the pattern.
int oracle_mixed_assemble(int type, const oracle_material* m, int64_t n_nodes,
                          const double* coords, int64_t n_elems, const int64_t* conn,
                          const int64_t* doff, const double* dofs, const double* kappa,
                          const double* kappa0_gp, const double* alpha_gp,
                          const int64_t* row_ptr, const int32_t* col_idx, double* val, double* R,
                          double* S) {
  MFam f;
  if (!mfamily(type, &f)) return -1;
  const int nd = f.ndofe;
  const int64_t ndof = doff[n_nodes];
  std::fill(val, val + row_ptr[ndof], 0.0);
  std::fill(R, R + ndof, 0.0);
  std::fill(S, S + ndof, 0.0);
  std::vector<double> Ke(nd * nd), Fe(nd), Fa(nd);
  double Xe[16], Ue[20];
  int64_t gdof[20];
  for (int64_t e = 0; e < n_elems; ++e) {
    for (int a = 0; a < f.nenu; ++a) {
      const int64_t n = conn[e * f.nenu + a];
      for (int i = 0; i < f.dim; ++i) Xe[a * f.dim + i] = coords[n * f.dim + i];
      const int nda = a < f.nene ? f.dim + 1 : f.dim;
      for (int i = 0; i < nda; ++i) {
        gdof[mldof(f, a) + i] = doff[n] + i;
        Ue[mldof(f, a) + i] = dofs[doff[n] + i];
      }
    }
    if (oracle_mixed_element(type, m, Xe, Ue, kappa + e * f.ngp,
                             kappa0_gp ? kappa0_gp + e * f.ngp : nullptr,
                             alpha_gp ? alpha_gp + e * f.ngp : nullptr, Ke.data(), Fe.data(),
                             Fa.data(), nullptr) != 0)
      return -2;
    for (int r = 0; r < nd; ++r) {
      R[gdof[r]] += Fe[r];
      S[gdof[r]] += Fa[r];
      for (int c = 0; c < nd; ++c) {
        const int64_t p = find_col(row_ptr, col_idx, gdof[r], gdof[c]);
        if (p < 0) return -3;
        val[p] += Ke[r * nd + c];
      }
    }
  }
  return 0;
}

// Eq. A.2 with Fig. 8b l.19-24 for mixed elements: ebar_gp from the linear ebar field.
int oracle_mixed_update_history(int type, int64_t n_elems, const int64_t* conn,
                                const int64_t* doff, const double* dofs, double* kappa) {
  MFam f;
  if (!mfamily(type, &f)) return -1;
  double xi[18], w[9], N[4], dN[8];
  oracle_mixed_gauss(type, xi, w);
  for (int64_t e = 0; e < n_elems; ++e)
    for (int g = 0; g < f.ngp; ++g) {
      oracle_mixed_shape_e(type, xi + g * f.dim, N, dN);
      double ebar = 0.0;
      for (int a = 0; a < f.nene; ++a) ebar += N[a] * dofs[doff[conn[e * f.nenu + a]] + f.dim];
      double& k = kappa[e * f.ngp + g];
      if ((ebar - k) > kTolHist) k = ebar;
    }
  return 0;
}

}  // extern "C"

extern "C" {

// State-variable update (Alg. 2 l.8-14, Fig. 9a) for mixed elements: the record of
// oracle_update_state ([eps_v, d eeq/d eps_v, sigma, eeq, ebar, kappa, D, g], oracle_sdv_width
// of the equal-order family of the same dimension) with eps from the quadratic u field and
// ebar from the linear field; commits kappa.
int oracle_mixed_update_state(int type, const oracle_material* m, int64_t n_nodes,
                              const double* coords, int64_t n_elems, const int64_t* conn,
                              const int64_t* doff, const double* dofs, double* kappa,
                              const double* kappa0_gp, const double* alpha_gp, double* sdv) {
  MFam f;
  if (!mfamily(type, &f)) return -1;
  (void)n_nodes;
  const int dim = f.dim, nv = f.nv, W = 3 * f.nv + 5;
  double xi[18], w[9], C[36];
  oracle_mixed_gauss(type, xi, w);
  elasticity(m, dim, C);
  for (int64_t e = 0; e < n_elems; ++e) {
    const int64_t* c = conn + e * f.nenu;
    for (int g = 0; g < f.ngp; ++g) {
      double Nu[8], dNu[16], Ne[4], dNe[8];
      oracle_mixed_shape_u(type, xi + g * dim, Nu, dNu);
      oracle_mixed_shape_e(type, xi + g * dim, Ne, dNe);
      double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, Ji[3][3];
      for (int a = 0; a < f.nenu; ++a)
        for (int i = 0; i < dim; ++i)   // relative to node 0 (R-REL)
          for (int j = 0; j < dim; ++j)
            J[i][j] += (coords[c[a] * dim + i] - coords[c[0] * dim + i]) * dNu[a * dim + j];
      if (!invert(dim, J, Ji)) return -2;
      double ev[6] = {0, 0, 0, 0, 0, 0}, ebar = 0.0;
      for (int a = 0; a < f.nenu; ++a) {
        double gN[3];
        for (int i = 0; i < dim; ++i) {
          double s = 0.0;
          for (int j = 0; j < dim; ++j) s += Ji[j][i] * dNu[a * dim + j];
          gN[i] = s;
        }
        const double* ua = dofs + doff[c[a]];
        const double* u0 = dofs + doff[c[0]];
        for (int V = 0; V < nv; ++V) {
          int p, q;
          voigt_pair(dim, V, &p, &q);
          if (p == q) ev[V] += gN[p] * (ua[p] - u0[p]);
          else ev[V] += gN[q] * (ua[p] - u0[p]) + gN[p] * (ua[q] - u0[q]);
        }
      }
      for (int a = 0; a < f.nene; ++a) ebar += Ne[a] * dofs[doff[c[a]] + dim];
      oracle_material mg = *m;
      if (kappa0_gp) mg.kappa0 = kappa0_gp[e * f.ngp + g];
      if (alpha_gp) mg.alpha = alpha_gp[e * f.ngp + g];
      double eeq, dv[6], H[36];
      oracle_eqstrain(&mg, dim, ev, &eeq, dv, H);
      double& kh = kappa[e * f.ngp + g];
      const double kap = (ebar - kh) > kTolHist ? ebar : kh;
      double D, dD, gI, dg;
      oracle_damage(&mg, kap, &D, &dD);
      oracle_interaction(&mg, D, &gI, &dg);
      double* out = sdv + (e * f.ngp + g) * W;
      for (int V = 0; V < nv; ++V) {
        double ce = 0.0;
        for (int U = 0; U < nv; ++U) ce += C[V * nv + U] * ev[U];
        out[V] = ev[V];
        out[nv + V] = dv[V];
        out[2 * nv + V] = (1.0 - D) * ce + m->h_sigma * (eeq - ebar) * dv[V];
      }
      out[3 * nv + 0] = eeq;
      out[3 * nv + 1] = ebar;
      out[3 * nv + 2] = kap;
      out[3 * nv + 3] = D;
      out[3 * nv + 4] = gI;
      kh = kap;
    }
  }
  return 0;
}

}  // extern "C"

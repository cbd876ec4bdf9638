/* lgdm_oracle.h -- CPU oracle for the LGDM K/R assembly path (arXiv 2301.06503).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2301_06503_b200/, include/lgdm.h) never links, loads or calls it, and it
 * shares no code, header, table or constant with the CUDA path.
 *
 * Plain, slow, element-by-element FP64 implementation following Algorithm 1 of
 * PAPER.md ("for el ... for igp ... Compute K_local, F_local ... Assemble"),
 * with the readings listed in DESIGN.md section "Readings of the paper".
 *
 * Element types: 1 = 2-node bar (d=1), 2 = Q4 plane strain (d=2), 3 = Hex8 (d=3).
 * DOFs are node-interleaved: dof = ndpn*node + comp, comp = (u_x[,u_y[,u_z]], ebar).
 */
#ifndef LGDM_ORACLE_H
#define LGDM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double E, nu;        /* elasticity (Eq. 1, 4C); plane strain in 2D            */
  double k;            /* compressive/tensile strength ratio (Eq. A.3)            */
  double kappa0;       /* damage threshold kappa_0 (Eq. A.1; code `ki`)          */
  double alpha, beta;  /* damage law parameters (Eq. A.1)                         */
  double h;            /* coupling modulus (Eq. 1)                                */
  double h_sigma;      /* coefficient of Eq. 2's h-term (reading R-11a)           */
  double c;            /* gradient parameter (Eq. 1)                              */
  double R, n;         /* interaction function parameters (Eq. A.4)               */
  double t;            /* cross-section area (1D) / thickness (2D, 3D: 1)         */
  int32_t eq_variant;  /* 0 = de Vree modified von Mises (reading R-A3), 1 = A.3 literal */
  int32_t pad_;
} oracle_material;

/* ---- pointwise laws (Appendix A) ---- */
void oracle_damage(const oracle_material* m, double kappa, double* D, double* dD);
void oracle_interaction(const oracle_material* m, double D, double* g, double* dgdD);
/* eps_v: Voigt strain (1D: [e]; 2D: [xx,yy,gxy]; 3D: [xx,yy,zz,gxy,gyz,gxz]) engineering shear.
 * Outputs eeq, d[nv] = d eeq/d eps_v, H[nv*nv] = d2 eeq / d eps_v^2 (row-major). */
void oracle_eqstrain(const oracle_material* m, int dim, const double* eps_v,
                     double* eeq, double* d, double* H);

/* ---- element machinery ---- */
int  oracle_gauss(int type, double* xi /*[ngp*dim]*/, double* w /*[ngp]*/);
void oracle_shape(int type, const double* xi, double* N /*[nen]*/, double* dNdxi /*[nen*dim]*/);

/* Element blocks (Eqs. 11a-f with the DESIGN.md readings).
 * Xe [nen*dim] node coords, Ue [nen*ndpn] node-interleaved dofs, kap [ngp] kappa_hist.
 * Ke [ndofe*ndofe] row-major (K = -dR/dx), Fe [ndofe] (R = F of Eq. 11),
 * Fabs [ndofe] = sum over GPs of |per-GP contribution to Fe| (tolerance scale, reading R-TOL),
 * sig [ngp*nv] (optional) macro stress per GP, guard [ngp] (optional) 1 where a threshold
 * decision is within 1e-14 relative of its switch.  Returns 0, or -(g+1) if det J <= 0 at GP g. */
int oracle_element(int type, const oracle_material* m, const double* Xe, const double* Ue,
                   const double* kap, double* Ke, double* Fe, double* Fabs,
                   double* sig, int32_t* guard);
/* Same with per-GP damage threshold k0g [ngp] and alpha alg [ngp] (defect regions);
 * NULL = the material's kappa0 / alpha. */
int oracle_element_d(int type, const oracle_material* m, const double* Xe, const double* Ue,
                     const double* kap, const double* k0g, const double* alg, double* Ke,
                     double* Fe, double* Fabs, double* sig, int32_t* guard);

/* ---- pattern (reading R-PAT) ---- */
int64_t oracle_pattern_nnz(int type, int64_t n_nodes, int64_t n_elems, const int64_t* conn);
int oracle_pattern(int type, int64_t n_nodes, int64_t n_elems, const int64_t* conn,
                   int64_t* row_ptr /*[ndof+1]*/, int32_t* col_idx /*[nnz]*/);

/* ---- assembly (Alg. 1 lines 4-11) into the pattern above ---- */
int oracle_assemble(int type, const oracle_material* m, int64_t n_nodes, const double* coords,
                    int64_t n_elems, const int64_t* conn, const double* dofs, const double* kappa,
                    const int64_t* row_ptr, const int32_t* col_idx,
                    double* val, double* R, double* S, int64_t* n_guard);

/* With per-GP defect fields kappa0_gp, alpha_gp [n_elems*ngp] (NULL = material). */
int oracle_assemble_d(int type, const oracle_material* m, int64_t n_nodes, const double* coords,
                      int64_t n_elems, const int64_t* conn, const double* dofs,
                      const double* kappa, const double* kappa0_gp, const double* alpha_gp,
                      const int64_t* row_ptr, const int32_t* col_idx,
                      double* val, double* R, double* S, int64_t* n_guard);
/* The same element loop on all host cores, colour by colour (elements of one colour share no
 * node; colour[e] in [0, n_colours)); CPU-baseline timing only.  *threads = threads used. */
int oracle_assemble_colored(int type, const oracle_material* m, int64_t n_nodes,
                            const double* coords, int64_t n_elems, const int64_t* conn,
                            const double* dofs, const double* kappa, const int32_t* colour,
                            int n_colours, const int64_t* row_ptr, const int32_t* col_idx,
                            double* val, double* R, double* S, int nthreads, int* threads);

/* Sampled rows: the block-rows of the n_sel listed nodes only, each computed from the
 * elements adjacent to that node (ascending element id).  Output per selected node s is
 * packed: rows ndpn*s .. ndpn*s+ndpn-1 of a compact CSR (row_ptr_sel[n_sel*ndpn+1]). */
int64_t oracle_rows_nnz(int type, int64_t n_nodes, int64_t n_elems, const int64_t* conn,
                        int64_t n_sel, const int64_t* sel);
int oracle_assemble_rows(int type, const oracle_material* m, int64_t n_nodes, const double* coords,
                         int64_t n_elems, const int64_t* conn, const double* dofs,
                         const double* kappa, int64_t n_sel, const int64_t* sel,
                         int64_t* row_ptr_sel, int32_t* col_idx_sel, double* val_sel,
                         double* R_sel, double* S_sel);

/* ---- history (Eq. A.2, Fig. 8b l.22-24) and residual norms ---- */
int oracle_update_history(int type, int64_t n_nodes, int64_t n_elems, const int64_t* conn,
                          const double* dofs, double* kappa);
void oracle_residual_norms(int type, int64_t n_rows, const double* R, double* out2);

/* ---- state-variable update (Alg. 2 l.8-14, Fig. 9a) ----
 * sdv [n_elems*ngp*oracle_sdv_width(type)]: per GP [eps_v (nv), d eeq/d eps_v (nv),
 * sigma (nv), eeq, ebar, kappa, D, g]; commits kappa.  kappa0_gp / alpha_gp nullable. */
int oracle_sdv_width(int type);
int oracle_update_state(int type, const oracle_material* m, int64_t n_nodes, const double* coords,
                        int64_t n_elems, const int64_t* conn, const double* dofs, double* kappa,
                        const double* kappa0_gp, const double* alpha_gp, double* sdv);

/* ---- mixed-order elements ----
 * type 4 = BAR3 (quadratic u on 3 nodes [xi=-1, +1, 0], linear ebar on the 2 end nodes,
 * 3-point Gauss); type 5 = QUAD8 (8-node serendipity u [corners ccw, midsides (0,-1), (1,0),
 * (0,1), (-1,0)], bilinear ebar on the corners, 3x3 Gauss).  Local dofs node-major, corners
 * (u..., ebar) first, then midsides (u...).  Global dof = doff[node] + comp. */
int oracle_mixed_family(int type, int32_t* out6 /* dim, nenu, nene, nv, ngp, ndofe */);
int oracle_mixed_gauss(int type, double* xi, double* w);
void oracle_mixed_shape_u(int type, const double* xi, double* N, double* dNdxi);
void oracle_mixed_shape_e(int type, const double* xi, double* N, double* dNdxi);
int oracle_mixed_element(int type, const oracle_material* m, const double* Xe, const double* Ue,
                         const double* kap, const double* k0g, const double* alg, double* Ke,
                         double* Fe, double* Fabs, double* sig);
int64_t oracle_mixed_dofs(int type, int64_t n_nodes, int64_t n_elems, const int64_t* conn,
                          int64_t* doff /*[n_nodes+1]*/);
/* row_ptr / col_idx may be NULL (count only); returns nnz */
int64_t oracle_mixed_pattern(int type, int64_t n_nodes, int64_t n_elems, const int64_t* conn,
                             const int64_t* doff, int64_t* row_ptr, int32_t* col_idx);
int oracle_mixed_assemble(int type, const oracle_material* m, int64_t n_nodes,
                          const double* coords, int64_t n_elems, const int64_t* conn,
                          const int64_t* doff, const double* dofs, const double* kappa,
                          const double* kappa0_gp, const double* alpha_gp,
                          const int64_t* row_ptr, const int32_t* col_idx, double* val, double* R,
                          double* S);
int oracle_mixed_update_history(int type, int64_t n_elems, const int64_t* conn,
                                const int64_t* doff, const double* dofs, double* kappa);
/* state records (layout of oracle_update_state, nv of the dimension) + history commit */
int oracle_mixed_update_state(int type, const oracle_material* m, int64_t n_nodes,
                              const double* coords, int64_t n_elems, const int64_t* conn,
                              const int64_t* doff, const double* dofs, double* kappa,
                              const double* kappa0_gp, const double* alpha_gp, double* sdv);
#ifdef __cplusplus
}
#endif
#endif

/* lgdm.h -- C ABI of the B200-native LGDM K/R assembly library (liblgdm.so).
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, arXiv 2301.06503):
 *   For every element and Gauss point (Alg. 1 lines 4-8; Alg. 2 lines 4-5)
 *   the tangent blocks Kuu, Kue, Keu, Kee (Eqs. 11a-d) and residuals Fu, Fe
 *   (Eqs. 11e-f) of the localizing gradient damage method, with the damage law
 *   (Eq. A.1), history (Eq. A.2), modified von Mises equivalent strain
 *   (Eq. A.3) and interaction function (Eq. A.4), assembled into a
 *   global CSR matrix K and vector R (Alg. 1 line 11; Fig. 2 lines 28-30).
 *   Readings of garbled/ambiguous passages: DESIGN.md "Readings of the paper"
 *   (R-A3, R-PS, R-SH, R-1D, R-11a, R-11f, R-kappa', R-TH, R-HIST, R-SQ, R-PAT, R-ORD).
 *
 * Conventions (frozen):
 *   - FP64 everywhere.  DOFs are node-interleaved: dof = ndpn*global_node + comp,
 *     comp = (u_x[, u_y[, u_z]], ebar); ndpn = d+1.
 *   - K = -dR/dx (so K*dx = R is the Newton step of Eq. 11), R = F of Eq. 11 (t = zeta = 0).
 *   - CSR: row_ptr int64 (config 4 has > 2^31 nonzeros), col_idx int32 holding GLOBAL dof
 *     ids, columns ascending, structural pattern with explicit zeros (every node pair that
 *     shares an element, x ndpn^2).  A rank's CSR is the row slice of its owned nodes.
 *   - Element local node order: bar2 (-1, +1); Q4 counter-clockwise from (-1,-1); Hex8
 *     bottom face (zeta=-1) counter-clockwise, then top face.  Gauss points 2 / 2x2 / 2x2x2
 *     at +-1/sqrt(3), xi fastest.  2D is plane strain with unit thickness; 1D uses the area.
 *
 * Errors: every call returns lgdm_status; no exception crosses the ABI.  On error outputs
 * are untouched and lgdm_last_error() (thread-local) describes the failure.
 * Threading: a mesh is not thread-safe; distinct meshes are independent.
 * Ownership: host inputs are copied; all device buffers are owned by the mesh and freed by
 * lgdm_destroy.  Pointers returned by lgdm_assemble stay valid until the next
 * lgdm_assemble / lgdm_destroy of that mesh.
 * Asynchrony: create/set_state/assemble/update_history enqueue work on the mesh's CUDA
 * stream and return without synchronising (create synchronises once for its checks);
 * lgdm_residual_norms and lgdm_get_kappa synchronise that stream.
 */
#ifndef LGDM_H
#define LGDM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LGDM_OK = 0,
  LGDM_ERR_INVALID_ARGUMENT = 1,  /* bad type, size, material (S:173 invariants), null ptr */
  LGDM_ERR_INVERTED_ELEMENT = 2,  /* det J <= 0 at a Gauss point; message names it  */
  LGDM_ERR_INVALID_STATE = 3,     /* assemble before set_state, size mismatch      */
  LGDM_ERR_OUT_OF_MEMORY = 4,
  LGDM_ERR_CUDA = 5,
  LGDM_ERR_NCCL = 6,
  LGDM_ERR_UNSUPPORTED = 7,       /* e.g. NCCL not loadable                                 */
  LGDM_ERR_NOT_CONVERGED = 8      /* lgdm_solve: residual above tolerance after max_iter    */
} lgdm_status;

/* Equal-order families (u and ebar on the same nodes; node-interleaved dofs, ndpn = d + 1) and
 * the paper's mixed-order families ("shape functions for displacement
 * (u) are taken as quadratic, and for micro-equivalent strain as linear"):
 *   LGDM_BAR3  = 4: 3-node quadratic bar for u, local nodes (xi = -1, +1, 0); linear ebar on
 *                   the two end nodes; 3-point Gauss.
 *   LGDM_QUAD8 = 5: 8-node serendipity quad for u (corners counter-clockwise, then midsides
 *                   (0,-1), (1,0), (0,1), (-1,0)); bilinear ebar on the corners; 3x3 Gauss;
 *                   plane strain.
 * Mixed meshes: a node carries ebar iff it is a corner (local index < 2 / < 4) of its
 * elements (a node that is a corner of one element and a midside node of another, or no
 * element's node, is INVALID_ARGUMENT).  Dofs stay node-interleaved with a variable count
 * per node: dof = doff[node] + comp, comp = (u_x[, u_y][, ebar]), doff = prefix sum of
 * (d + 1 for corner nodes, d for midside nodes), see lgdm_dof_offsets.  Slabs through
 * lgdm_create_mesh_mixed (global dof offset); assemble uses the element-block
 * + gather kernels (lgdm_set_kernel 0 or 1); lgdm_update_state writes the records of the
 * equal-order family of the same dimension (lgdm_sdv_width); lgdm_get_blocked returns the
 * u dofs (node order) then the ebar dofs (node order).  Gradients are evaluated on coordinates / dofs relative to each
 * element's node 0 (reading R-REL). */
typedef enum { LGDM_BAR2 = 1, LGDM_QUAD4 = 2, LGDM_HEX8 = 3, LGDM_BAR3 = 4, LGDM_QUAD8 = 5 } lgdm_elem_type;

/* Material (Eq. 1 4C, Eqs. 2-4, Appendix A).  Validated at create:
 * E > 0, 0 <= nu < 0.5, k >= 1, kappa0 > 0, 0 < alpha <= 1, beta > 0, h > 0,
 * h_sigma >= 0, c > 0, 0 < R < 1, n > 0, thickness_or_area > 0. */
typedef struct {
  double E, nu;             /* Young's modulus [MPa], Poisson ratio                         */
  double k;                 /* compressive/tensile strength ratio (Eq. A.3)                 */
  double kappa0;            /* damage threshold (Eq. A.1; `ki` in Fig. 8b)                  */
  double alpha, beta;       /* damage law parameters (Eq. A.1)                              */
  double h;                 /* coupling modulus (Eq. 1)                                     */
  double h_sigma;           /* coefficient of Eq. 2's h-term (reading R-11a: h = R1, 0 = R2) */
  double c;                 /* gradient parameter [mm^2] (Eq. 1)                            */
  double R, n;              /* interaction function parameters (Eq. A.4)                    */
  double thickness_or_area; /* 1D: bar area [mm^2]; 2D/3D: 1                                */
  int32_t eq_variant;       /* 0: de Vree constants (reading R-A3); 1: A.3 as printed        */
  int32_t reserved;         /* must be 0                                                    */
} lgdm_material;

typedef struct lgdm_mesh_s* lgdm_mesh;

/* Equal-order meshes: the row / column counts below with ndpn = d + 1.  Mixed-order meshes
 * (LGDM_BAR3 / LGDM_QUAD8): n_rows = dofs of the owned nodes, n_cols = n_global_dofs,
 * first_row = global dof of the first owned node (lgdm_create_mesh_mixed). */
typedef struct {
  int64_t n_rows;           /* owned rows = ndpn * (owned_node_end - owned_node_begin)      */
  int64_t n_cols;           /* ndpn * n_global_nodes                                        */
  int64_t nnz;
  int64_t first_row;        /* global row id of local row 0 = ndpn*(offset+owned_begin)     */
  const int64_t* row_ptr;   /* device, [n_rows+1], row_ptr[0] = 0                           */
  const int32_t* col_idx;   /* device, [nnz], global dof ids, ascending per row             */
  double* val;              /* device, [nnz]                                                */
} lgdm_csr;

typedef struct {   /* mixed-order meshes: nen = u nodes, ndpn = dofs of a corner node */
  int32_t elem_type, dim, nen, ndpn, ngp, structured;   /* structured: 1 = sweep kernel path  */
  int64_t n_nodes, n_elems, n_owned_nodes, n_rows, nnz;
  int64_t nx, ny, nz;                                    /* element counts if structured      */
  int64_t device_bytes;                                  /* device memory owned by the mesh  */
} lgdm_info;

/* Create a mesh (a whole mesh, or one rank's slab).  S:44-70, S:82 (immutable mesh).
 *   coords  host [n_nodes][d] f64 (copied)           conn host [n_elems][nen] LOCAL node ids
 *   global_node_offset: global id of local node 0 -- local nodes are the contiguous global
 *     range [offset, offset+n_nodes) (true for z-slabs of Hex8 / y-slabs of Q4 under x-fastest
 *     numbering); 0 on one GPU.   n_global_nodes: sets n_cols.
 *   owned_node_begin/end: local node range whose rows this mesh assembles (the rest are ghost
 *     nodes of ghost elements, recomputed here so K needs no communication).
 *   device: CUDA ordinal; cuda_stream: cudaStream_t (NULL = legacy default stream).
 * Builds the CSR pattern (reading R-PAT) and the element->CSR maps once.  det J <= 0 at any
 * GP -> LGDM_ERR_INVERTED_ELEMENT.  Connectivity of an x-fastest structured grid (any
 * coordinates) is detected and enables the fused sweep kernels.  Rejected with
 * LGDM_ERR_INVALID_ARGUMENT before any device work: an empty mesh (n_elems < 1 or n_nodes < 2),
 * an empty or out-of-range owned range, conn entries outside [0, n_nodes), NULL inputs, an
 * unknown type, an invalid material; no CUDA device -> LGDM_ERR_CUDA (there is no CPU path). */
lgdm_status lgdm_create_mesh(lgdm_elem_type type, int64_t n_nodes, const double* coords,
                             int64_t n_elems, const int64_t* conn, const lgdm_material* mat,
                             int64_t global_node_offset, int64_t n_global_nodes,
                             int64_t owned_node_begin, int64_t owned_node_end, int device,
                             void* cuda_stream, lgdm_mesh* out);

/* Mixed-order mesh or slab (LGDM_BAR3 / LGDM_QUAD8) with its place in the global dof
 * numbering: as lgdm_create_mesh, plus global_dof_offset = global dof id of the slab's local
 * dof 0 (its first local node's first dof) and n_global_dofs (the K column count).  Local
 * dofs are numbered by lgdm_dof_offsets; a slab's local nodes must be a contiguous global node
 * range whose node kinds (corner / midside) are those of the whole mesh, so global dof =
 * global_dof_offset + local dof.  Rows are those of the owned nodes [owned_node_begin,
 * owned_node_end); the elements touching them (ghosts included) are local and recomputed, so
 * stitched slab rows equal the whole-mesh rows bitwise (ascending element order is kept when
 * the slab's elements are a contiguous, ordered global range).  lgdm_create_mesh accepts the
 * mixed types for whole meshes only.  Errors as lgdm_create_mesh; n_global_dofs < offset +
 * local dofs -> LGDM_ERR_INVALID_ARGUMENT. */
lgdm_status lgdm_create_mesh_mixed(lgdm_elem_type type, int64_t n_nodes, const double* coords,
                                   int64_t n_elems, const int64_t* conn, const lgdm_material* mat,
                                   int64_t global_node_offset, int64_t n_global_nodes,
                                   int64_t owned_node_begin, int64_t owned_node_end,
                                   int64_t global_dof_offset, int64_t n_global_dofs, int device,
                                   void* cuda_stream, lgdm_mesh* out);

/* State of the current Newton iterate (Alg. 2 line 7): dofs [n_nodes][ndpn] node-
 * interleaved, kappa [n_elems][ngp] = history kappa_hist at the start of the increment.
 * src_on_device: 1 if both pointers are device pointers (D2D copy), 0 for host (H2D; pinned
 * host memory makes the copy asynchronous).  Size mismatch -> LGDM_ERR_INVALID_STATE.
 * kappa may be NULL to keep the mesh's current history (dofs-only update). */
lgdm_status lgdm_set_state(lgdm_mesh mesh, const double* dofs, int64_t n_dofs,
                           const double* kappa, int64_t n_kappa, int src_on_device);

/* Overlapped input transfer for a stream of iterates: lgdm_prefetch_dofs starts copying the
 * NEXT iterate's dofs (host, pinned for asynchrony; n_dofs as in lgdm_set_state) into a second
 * device buffer on an internal copy stream, concurrently with the work already enqueued on the
 * mesh stream; lgdm_set_state_prefetched makes that buffer the current dofs (the mesh stream
 * waits for the copy; the two buffers are swapped, nothing is copied again).  At most one
 * prefetch may be pending: a second call before lgdm_set_state_prefetched, or
 * lgdm_set_state_prefetched without a pending prefetch -> LGDM_ERR_INVALID_STATE.  The history
 * kappa must have been set before (lgdm_set_state).  The host buffer must stay valid until the
 * copy completes (next lgdm_set_state_prefetched returns after enqueuing the wait, so keep it
 * until the following synchronisation of the mesh stream). */
lgdm_status lgdm_prefetch_dofs(lgdm_mesh mesh, const double* host_dofs, int64_t n_dofs);
lgdm_status lgdm_set_state_prefetched(lgdm_mesh mesh);

/* Assemble K (owned rows) and R = F (owned rows) for the current state (Eqs. 11a-f with the
 * trial kappa = cond1 ? ebar : kappa_hist, Fig. 8b; history is NOT written, reading R-HIST).
 * K and *R point to mesh-owned device memory. */
lgdm_status lgdm_assemble(lgdm_mesh mesh, lgdm_csr* K, double** R);

/* Commit the history: kappa_hist <- (ebar_gp - kappa_hist > 1e-10) ? ebar_gp : kappa_hist for
 * every local GP (owned and ghost), Eq. A.2 with Fig. 8b lines 22-24. */
lgdm_status lgdm_update_history(lgdm_mesh mesh);

/* ---- state-variable update and defect fields ----
 *
 * Doubles per (element, GP) record of lgdm_update_state: 3 nv + 5 with nv = 1 / 3 / 6 Voigt
 * components (bar / Q4 / Hex8): 8 / 14 / 23; -1 for an unknown type. */
int lgdm_sdv_width(lgdm_elem_type type);

/* Per-GP damage threshold kappa0 and damage parameter alpha of Eq. A.1 (defect regions,
 * PAPER.md P:418; the code's per-GP `ki` and `alpha_var`, Fig. 9a l.3-4 / P:380-389), each an
 * array [n_elems][ngp] (n = n_elems * ngp) or NULL = the material's value (NULL clears a
 * previously set field).  src_on_device: 1 device pointers (async D2D copy on the mesh stream),
 * 0 host (copied before return).  Values are not validated (kappa0 > 0, 0 <= alpha <= 1 are
 * the caller's responsibility).  With a field set, lgdm_assemble uses it in the general
 * kernel and the default sweeps (kernels 0, 1, 4; the experimental sweep kernels 2, 3, 5
 * return LGDM_ERR_INVALID_ARGUMENT) and lgdm_update_state uses it.  n mismatch -> LGDM_ERR_INVALID_STATE. */
lgdm_status lgdm_set_defects(lgdm_mesh mesh, const double* kappa0_gp, const double* alpha_gp,
                             int64_t n, int src_on_device);

/* State-variable update of Alg. 2 lines 8-14 (Fig. 9a update_variables,
 * P:359-390) for the current state: per (element, GP), in element-major order, the record
 *   [eps_v (nv, Voigt, engineering shear: bar [e]; Q4 [xx, yy, xy]; Hex8 [xx, yy, zz, xy, yz, xz]),
 *    d eeq / d eps_v (nv, Eq. A.3 with reading R-A3 / R-SQ),
 *    sigma (nv, Eq. 2 with the h_sigma (eeq - ebar) d term of reading R-11a),
 *    eeq (Eq. A.3), ebar (Fig. 9a l.19), kappa (history, l.22-24), D (Eq. A.1), g (Eq. A.4)]
 * and commits the history kappa_hist <- kappa (as lgdm_update_history).  sdv: n_sdv =
 * n_elems * ngp * lgdm_sdv_width doubles, device (dst_on_device = 1, async on the mesh stream)
 * or host (synchronises the stream), or NULL to commit the history only.
 * Before set_state -> LGDM_ERR_INVALID_STATE; n_sdv mismatch -> LGDM_ERR_INVALID_STATE. */
lgdm_status lgdm_update_state(lgdm_mesh mesh, double* sdv, int64_t n_sdv, int dst_on_device);

/* The last assembled K and R in the paper's blocked DOF order [u; ebar] (PAPER.md P:345-346,
 * `u(1:ndof_u)` then the ebar dofs): rows and columns permuted by
 * blocked r < n dim -> interleaved ndpn (r / dim) + r % dim, r >= n dim -> ndpn (r - n dim) + dim,
 * i.e. P K P^T and P R, columns ascending per row, the same nnz (explicit zeros kept).  Mesh-
 * owned device memory, valid until the next lgdm_get_blocked / lgdm_destroy; async on the
 * mesh stream (a pure permutation of lgdm_assemble's output: bit-identical values).  Needs a
 * single-rank whole mesh (no slab offset / ownership) -> else LGDM_ERR_INVALID_ARGUMENT;
 * before lgdm_assemble -> LGDM_ERR_INVALID_STATE. */
lgdm_status lgdm_get_blocked(lgdm_mesh mesh, lgdm_csr* K, double** R);

/* ---- Newton loop pieces (Alg. 2 lines 4-7 and 16) ----
 * A whole mesh on one rank, or row-owned slabs with a communicator (lgdm_set_comm): rank p
 * owns a contiguous node range that follows rank p-1's; its ghost dofs below are rank p-1's
 * last owned dofs and rank p-1's ghosts above are rank p's first owned dofs (the slab
 * partitions of slabs.py: one node layer each way for equal order; two lattice rows below and
 * one above for mixed order -- the exchange counts need not match).  lgdm_set_comm checks it;
 * a slab mesh without a validated layout -> LGDM_ERR_UNSUPPORTED.  Across ranks: dof ids are GLOBAL (every
 * rank passes the same lists), delta vectors are LOCAL dof vectors (the mesh's owned + ghost
 * dofs in node order, lgdm_dof_offsets), their ghost dofs filled from the neighbouring slabs by
 * an NCCL send / recv halo exchange, and every sum is an NCCL allreduce.  All work runs on the
 * mesh stream; the calls below synchronise it where they return host values.
 *
 * Symmetric Dirichlet elimination on the last assembled K, R (in place; the paper does not
 * state its scheme -- SPEC.md apply_dirichlet): constrained u dofs dof_ids[n_fixed] (host,
 * node-interleaved global ids; a rank uses those among its local dofs) get unit rows and R = increments[k] (the step's prescribed increment
 * on the first iteration, 0 afterwards, since Eq. 11 solves for increments); every free row
 * moves K_ij increments_j to its RHS and zeroes K_ij.  An ebar dof or an id out of range ->
 * LGDM_ERR_INVALID_ARGUMENT; before lgdm_assemble -> LGDM_ERR_INVALID_STATE. */
lgdm_status lgdm_apply_dirichlet(lgdm_mesh mesh, int64_t n_fixed, const int64_t* dof_ids,
                                 const double* increments);

/* Solve K delta = R (Alg. 2 l.6; the paper uses a direct `mldivide`) with
 * Jacobi-preconditioned BiCGSTAB on the GPU, across the ranks of a communicator (owned-row
 * SpMV after a ghost-dof halo exchange, allreduced dot products): delta (device, local dofs =
 * lgdm_dof_offsets' last entry doubles, ghost dofs filled on return) from 0 until
 * ||R - K delta|| <= tol ||R||; iters / relres (host, nullable) report the iterations and the
 * true relative residual.  Not within 10 tol after max_iter -> LGDM_ERR_NOT_CONVERGED (delta
 * holds the last iterate).  Reductions are fixed-order: bitwise reproducible. */
lgdm_status lgdm_solve(lgdm_mesh mesh, double* delta, double tol, int max_iter, int* iters,
                       double* relres);

/* Direct solve of K delta = R on the GPU (the paper's `mldivide`; single-rank whole
 * meshes only, else LGDM_ERR_UNSUPPORTED -- across ranks use lgdm_solve): sparse QR of
 * cuSOLVER (cusolverSpDcsrlsvqr with symrcm reordering; libcusolver / libcusparse dlopen'ed,
 * missing -> LGDM_ERR_UNSUPPORTED; nnz >= 2^31 -> LGDM_ERR_UNSUPPORTED).  delta device;
 * singularity (host, nullable) = -1 or the first rank-deficient pivot, in which case
 * LGDM_ERR_NOT_CONVERGED is returned.  Synchronises the mesh stream. */
lgdm_status lgdm_solve_direct(lgdm_mesh mesh, double* delta, int* singularity);

/* First global dof of every node (mixed-order meshes: variable dofs per node; equal-order:
 * ndpn * node): host_out [n_nodes + 1], the last entry = number of dofs.  n must equal
 * n_nodes + 1, else LGDM_ERR_INVALID_ARGUMENT. */
lgdm_status lgdm_dof_offsets(lgdm_mesh mesh, int64_t* host_out, int64_t n);

/* Reaction of a displacement-controlled problem (the load of the paper's load-displacement
 * curves, Fig. 11 / P:418; SPEC reaction_force): -sum of the last assembled R over the listed
 * dofs (host, global ids; summed over the ranks that own them), to be called after
 * lgdm_assemble and BEFORE lgdm_apply_dirichlet.  Host out. */
lgdm_status lgdm_reaction(lgdm_mesh mesh, int64_t n, const int64_t* dof_ids, double* out);

/* dofs += alpha * delta (delta device, the local dofs incl. ghosts; Alg. 2 l.7). */
lgdm_status lgdm_add_dofs(lgdm_mesh mesh, const double* delta, double alpha);

/* Convergence sums of Alg. 1 l.26 / Alg. 2 l.16 (host out4): {sum du^2, sum u^2, sum de^2,
 * sum e^2} over the owned u and ebar dofs of delta (device) and of the current dofs, summed
 * over the ranks. */
lgdm_status lgdm_delta_norms(lgdm_mesh mesh, const double* delta, double out4[4]);

/* Convergence test of Alg. 1 l.26 / Alg. 2 l.16: out2 = {||du||/||u||,
 * ||de||/||e||} (host) from the sums of lgdm_delta_norms, a zero iterate norm counted as
 * 1e-16; *converged = 1 when both ratios are <= tol.  tol <= 0 -> INVALID_ARGUMENT; the other
 * errors are lgdm_delta_norms'.  Synchronises the mesh stream. */
lgdm_status lgdm_delta_ratios(lgdm_mesh mesh, const double* delta, double tol, double out2[2],
                              int* converged);

/* Sums of squares of the last assembled R over owned rows: out2 = {sum Fu^2, sum Fe^2}.
 * out2 is a device pointer (2 doubles) when on_device = 1 (stream-ordered, no sync; for a
 * caller-side allreduce), else a host pointer (synchronises). */
lgdm_status lgdm_residual_sumsq(lgdm_mesh mesh, double* out2, int on_device);

/* Global norms {||Fu||_2, ||Fe||_2}: the convergence quantities of P:297 in residual form.
 * Local (owned rows) unless lgdm_set_comm was called, then NCCL allreduce(sum) over ranks.
 * out2 is host memory; synchronises. */
lgdm_status lgdm_residual_norms(lgdm_mesh mesh, double out2[2]);

/* One pass of the hot path per Newton iteration (Alg. 2 l.4-5 and the
 * residual check of l.16): lgdm_assemble -> sums of squares of R (u rows, ebar rows)
 * -> ncclAllReduce of the 2 sums when a communicator is set -> out2 = {||Fu||, ||Fe||} (host)
 * -> with LGDM_STEP_HISTORY also lgdm_update_history.  With LGDM_STEP_GRAPH the pass is captured
 * once into a CUDA graph on the mesh stream (per dofs buffer, kernel selector, defect fields,
 * communicator and flags; at most two kept) and replayed on later calls -- the first call runs
 * eagerly.  K and R stay on the device (as after lgdm_assemble).  Synchronises the mesh stream.
 * Errors: those of lgdm_assemble / lgdm_residual_norms / lgdm_update_history; unknown flags ->
 * INVALID_ARGUMENT; a failed capture -> LGDM_ERR_CUDA. */
enum { LGDM_STEP_GRAPH = 1, LGDM_STEP_HISTORY = 2 };
lgdm_status lgdm_step(lgdm_mesh mesh, int flags, double out2[2]);

/* Attach an NCCL communicator (ncclUniqueId bytes from rank 0, e.g. broadcast through
 * torch.distributed).  NCCL is loaded at run time (dlopen libnccl.so.2). */
lgdm_status lgdm_set_comm(lgdm_mesh mesh, const void* nccl_unique_id, int nranks, int rank);

/* Fill out (>= 128 bytes) with a fresh ncclUniqueId (call on rank 0, broadcast to the others
 * through any channel, e.g. torch.distributed.broadcast_object_list). */
lgdm_status lgdm_nccl_unique_id(void* out, int64_t out_bytes);

/* Copy the current kappa_hist [n_elems][ngp] to host (tests).  Synchronises. */
lgdm_status lgdm_get_kappa(lgdm_mesh mesh, double* host_out);

/* dofs *= s on device (benchmark helper: dofs_t = (1 + 0.05 t) dofs_0, SURVEY 8d cfg 2). */
lgdm_status lgdm_scale_dofs(lgdm_mesh mesh, double s);

/* Select the assembly kernel (all produce the same K and R up to rounding, parity-tested):
 *   0 = automatic: structured meshes (x-fastest grids, whole owned layers) -> 2, else 1
 *   1 = general (element-batch + node gather, any connectivity)
 *   2 = structured sweep: Q4 k_sweepq, Hex8 k_sweep4 (row-sum diagonals)
 * Kernel 2 needs a structured mesh: LGDM_ERR_INVALID_ARGUMENT otherwise; any other
 * selector value: LGDM_ERR_INVALID_ARGUMENT. */
lgdm_status lgdm_set_kernel(lgdm_mesh mesh, int kernel);

lgdm_status lgdm_get_info(lgdm_mesh mesh, lgdm_info* info);

/* Number of kernel launches issued by this mesh since creation (launch accounting). */
int64_t lgdm_launch_count(lgdm_mesh mesh);

#ifdef LGDM_PHASE_TIMING
/* Debug builds only (compiled with -DLGDM_PHASE_TIMING; not exported otherwise): cycles per
 * phase of the sweep kernels' instrumentation points, summed over CTAs (16 counters, host
 * out16); reset != 0 clears them.  Synchronises the device. */
int lgdm_debug_phase_cycles(unsigned long long* out16, int reset);
#endif

const char* lgdm_last_error(void);
void lgdm_destroy(lgdm_mesh mesh);

#ifdef __cplusplus
}
#endif
#endif /* LGDM_H */

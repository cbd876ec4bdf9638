// lgdm_sweep.cuh -- fused structured-sweep assembly (Q4 and Hex8), the hot kernels.
//
// Included by lgdm_api.cu after the definition of lgdm_mesh_s.
//
// Mapping (B200-first redesign of Alg. 2's "Compute and Assemble K, F"):
//   * One CTA owns a tile of node COLUMNS and a chunk of node LAYERS along the sweep axis
//     (Hex8: z; Q4: y).  It writes exactly the CSR block-rows of the nodes it owns, so no two
//     CTAs ever touch the same entry (atomic-free).
//   * It sweeps the element layers that touch its nodes.  In each layer the elements around
//     the tile (owned columns + one halo element on each side, recomputed) are processed in
//     colour batches -- parity of the element's (i, j) -- so no two elements of a batch share
//     a node and every block-row entry receives at most one add per batch.
//   * Per-entry summation order = (element layer, colour) -- a function of global indices
//     only, so any tiling / slabbing gives bitwise identical K and R.
// Kernels: k_sweep4 (Hex8, lgdm_sweep4.cuh), k_sweepq (Q4, lgdm_sweepq.cuh).
#pragma once

namespace lgdm {

#ifdef LGDM_PHASE_TIMING
// debug build only: cycles spent per phase by thread 0 of each role, summed over CTAs
__device__ unsigned long long g_phase[16];
#define PT_DECL unsigned long long pt_t0 = clock64();
#define PT_MARK(slot, cond)                                          \
  do {                                                               \
    if (cond) {                                                      \
      const unsigned long long pt_t1 = clock64();                    \
      atomicAdd(&g_phase[slot], pt_t1 - pt_t0);                      \
      pt_t0 = pt_t1;                                                 \
    }                                                                \
  } while (0)
#else
#define PT_DECL
#define PT_MARK(slot, cond) do {} while (0)
#endif

struct SweepGeom {
  int64_t nx, nyE, nyN, nl;        // elements in x; elements / nodes in y (D=2: 1 / 1); layers
  int64_t lay_own_b, lay_own_e;    // owned node layers [b, e) (local)
  int64_t own_node_b;              // local id of the first owned node
  int64_t chunk_len;               // owned node layers per CTA chunk
  int tiles_x, tiles_y, chunks;
  const double* k0g;               // per-GP kappa0 / alpha (defect fields) or NULL
  const double* alg;               //   (read by k_sweep4 / k_sweepq only)
};

template <int D> __device__ __forceinline__ void node_off(int a, int& ox, int& oy, int& oz) {
  // element local node -> (x, y, layer) offset; D=2: the element's second axis is the layer
  ox = node_sign<D>(a, 0) > 0;
  if constexpr (D == 3) {
    oy = node_sign<D>(a, 1) > 0;
    oz = node_sign<D>(a, 2) > 0;
  } else {
    oy = 0;
    oz = node_sign<D>(a, 1) > 0;
  }
}

// in-plane slot of offset (dx, dy)
template <int D> __device__ __forceinline__ int plane_slot(int dx, int dy) {
  if constexpr (D == 3) return (dy + 1) * 3 + (dx + 1);
  else return dx + 1;
}

}  // namespace lgdm

#include "lgdm_sweep4.cuh"
#include "lgdm_sweepq.cuh"

namespace {

bool sweep_supported(lgdm_mesh m) {
  if (!m->structured || m->f.dim < 2) return false;
  const int64_t per_layer = m->f.dim == 3 ? (m->nx + 1) * (m->ny + 1) : (m->nx + 1);
  return m->own_b % per_layer == 0 && m->own_e % per_layer == 0;
}


// Chunking of the sweep axis: each chunk of len node layers processes len + 1 element layers
// (one recomputed).  Pick the chunk count that minimises waves x (len + 1), i.e. the
// makespan of tiles x chunks equal CTAs on per_wave resident slots.
inline int64_t pick_chunks(int64_t tiles, int64_t layers, int64_t per_wave, int64_t min_len) {
  int64_t best = 1;
  double best_t = 1e300;
  for (int64_t c = 1; c <= std::max<int64_t>(1, layers); ++c) {
    const int64_t len = (layers + c - 1) / c;
    if (c > 1 && len < min_len) break;
    const int64_t n = (layers + len - 1) / len;
    const int64_t waves = (tiles * n + per_wave - 1) / per_wave;
    const double t = double(waves) * double(len + 1);
    if (t < best_t * 0.999) {
      best_t = t;
      best = n;
    }
  }
  return best;
}

lgdm_status launch_sweep4(lgdm_mesh m) {
  SweepGeom G{};
  G.nx = m->nx;
  G.nyE = m->ny;
  G.nyN = m->ny + 1;
  G.nl = m->nz;
  const int64_t per_layer = (G.nx + 1) * G.nyN;
  G.lay_own_b = m->own_b / per_layer;
  G.lay_own_e = m->own_e / per_layer;
  G.own_node_b = m->own_b;
  G.k0g = m->k0g;
  G.alg = m->alg;
  G.tiles_x = int((G.nx + 1 + S4::TX - 1) / S4::TX);
  G.tiles_y = int((G.nyN + S4::TY - 1) / S4::TY);
  CU(set_smem_attr(k_sweep4, S4::SMEM, m->device));
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device);
  const int64_t layers = G.lay_own_e - G.lay_own_b;
  const int64_t tiles = int64_t(G.tiles_x) * G.tiles_y;
  const int64_t chunks = pick_chunks(tiles, layers, nsm, 8);
  G.chunk_len = (layers + chunks - 1) / chunks;
  G.chunks = int((layers + G.chunk_len - 1) / G.chunk_len);
  const int64_t grid = tiles * G.chunks;
  k_sweep4<<<unsigned(grid), S4::T, S4::SMEM, m->stream>>>(m->dm, G, m->coords, m->dofs, m->kappa,
                                                           m->base, m->val, m->R);
  return check_launch(m, "k_sweep4");
}

lgdm_status launch_sweepq(lgdm_mesh m) {
  SweepGeom G{};
  G.nx = m->nx;
  G.nyE = 1;
  G.nyN = 1;
  G.nl = m->ny;
  const int64_t per_layer = G.nx + 1;
  G.lay_own_b = m->own_b / per_layer;
  G.lay_own_e = m->own_e / per_layer;
  G.own_node_b = m->own_b;
  G.k0g = m->k0g;
  G.alg = m->alg;
  G.tiles_x = int((G.nx + 1 + SQ::TX - 1) / SQ::TX);
  G.tiles_y = 1;
  CU(set_smem_attr(k_sweepq, SQ::SMEM, m->device));
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device);
  const int64_t layers = G.lay_own_e - G.lay_own_b;
  const int64_t tiles = G.tiles_x;
  const int64_t chunks = pick_chunks(tiles, layers, nsm, 8);
  G.chunk_len = (layers + chunks - 1) / chunks;
  G.chunks = int((layers + G.chunk_len - 1) / G.chunk_len);
  const int64_t grid = tiles * G.chunks;
  k_sweepq<<<unsigned(grid), SQ::T, SQ::SMEM, m->stream>>>(m->dm, G, m->coords, m->dofs, m->kappa,
                                                           m->base, m->val, m->R);
  return check_launch(m, "k_sweepq");
}

// Automatic choice (kernel 0 or 2): k_sweepq (Q4) and k_sweep4 (Hex8).
lgdm_status assemble_sweep(lgdm_mesh m) {
  if (m->f.dim == 2) return launch_sweepq(m);
  return launch_sweep4(m);
}

}  // namespace

#ifdef LGDM_PHASE_TIMING
// debug builds only (-DLGDM_PHASE_TIMING; declared in include/lgdm.h under the same macro):
// per-phase cycle counters of the sweep kernels' PT_MARK points
extern "C" int lgdm_debug_phase_cycles(unsigned long long* out16, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out16, lgdm::g_phase, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(lgdm::g_phase, z, sizeof(z));
  }
  return 0;
}
#endif

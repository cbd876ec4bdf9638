// lgdm_sweep.cuh -- fused structured-sweep assembly (Q4 and Hex8), the hot kernel.
//
// Included by lgdm_api.cu after the definition of lgdm_mesh_s.
//
// Mapping (B200-first redesign of Alg. 2's "Compute and Assemble K, F"):
//   * One CTA owns a tile of node COLUMNS (Hex8: 4x4 (x,y) columns; Q4: 32 x-columns) and a
//     chunk of node LAYERS along the sweep axis (Hex8: z; Q4: y).  It writes exactly the CSR
//     block-rows of the nodes it owns, so no two CTAs ever touch the same entry (atomic-free).
//   * It sweeps the element layers that touch its nodes.  In each layer the elements around
//     the tile (owned columns + one halo element on each side) are processed in colour
//     batches -- parity of the element's (i, j) -- so no two elements of a batch share a node.
//   * Per batch: phase A (thread per element x GP: geometry, kinematics, Appendix A update,
//     per-node expansions, lgdm_device.cuh) into shared memory; phase C (thread per element x
//     node pair a<=b: Gauss sums of Eqs. 11a-f in registers, Kuu symmetry); then each pair
//     thread adds its blocks into the block-rows of its OWNED nodes.  Those rows are zeroed when
//     the sweep first reaches their layer and stay L2-resident (two node layers per CTA) while
//     they are accumulated, so DRAM sees each K value written once.
//   * Per-entry summation order = (element layer, colour, GP) -- a function of global indices
//     only, so any tiling / slabbing gives bitwise identical K and R.
#pragma once

namespace lgdm {

template <int D> struct SweepCfg;
template <> struct SweepCfg<2> { static constexpr int TX = 32, TY = 1, E = 16, NCOL = 2, MINB = 3; };
template <> struct SweepCfg<3> { static constexpr int TX = 4, TY = 4, E = 4, NCOL = 4, MINB = 3; };

struct SweepGeom {
  int64_t nx, nyE, nyN, nl;        // elements in x; elements / nodes in y (D=2: 1 / 1); layers
  int64_t lay_own_b, lay_own_e;    // owned node layers [b, e) (local)
  int64_t own_node_b;              // local id of the first owned node
  int64_t chunk_len;               // owned node layers per CTA chunk
  int tiles_x, tiles_y, chunks;
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

// slot of neighbour offset (dx,dy,dz) in the sorted neighbour list of node (x,y,z), and the
// row width W = deg * ndpn (reading R-PAT: neighbours sorted by global id = (z, y, x))
__device__ __forceinline__ void slot_of(const SweepGeom& G, int64_t x, int64_t y, int64_t z,
                                        int dx, int dy, int dz, int ndpn, int& slot, int& W) {
  const int xlo = x > 0 ? -1 : 0, xhi = x < G.nx ? 1 : 0;
  const int ylo = y > 0 ? -1 : 0, yhi = y < G.nyN - 1 ? 1 : 0;
  const int zlo = z > 0 ? -1 : 0, zhi = z < G.nl ? 1 : 0;
  const int wx = xhi - xlo + 1, wy = yhi - ylo + 1, wz = zhi - zlo + 1;
  slot = ((dz - zlo) * wy + (dy - ylo)) * wx + (dx - xlo);
  W = wx * wy * wz * ndpn;
}

template <int D>
__global__ void __launch_bounds__(SweepCfg<D>::E * Fam<D>::NPAIR, SweepCfg<D>::MINB)
k_sweep(DevMat m, SweepGeom G, const double* __restrict__ coords, const double* __restrict__ dofs,
        const double* __restrict__ kappa, const int64_t* __restrict__ base,
        double* __restrict__ val, double* __restrict__ Rv) {
  using F = Fam<D>;
  using C = SweepCfg<D>;
  constexpr int E = C::E, NT = E * F::NPAIR, NDPN = F::NDPN, NEN = F::NEN, NGP = F::NGP;
  extern __shared__ double sm[];
  double* recs = sm;                                   // [E][NGP][GpBlock]
  double* scal = recs + E * NGP * GpBlock<D>::STRIDE;  // [E][NGP][kScal]
  double* Xs = scal + E * NGP * kScal;                 // [E][NEN][D]
  double* Us = Xs + E * NEN * D;                       // [E][NEN][NDPN]
  __shared__ int64_t s_i[E], s_j[E];
  const int tid = threadIdx.x;

  int bid = blockIdx.x;
  const int tx = bid % G.tiles_x;
  bid /= G.tiles_x;
  const int ty = bid % G.tiles_y;
  const int ch = bid / G.tiles_y;
  const int64_t x0 = int64_t(tx) * C::TX, x1 = min(x0 + C::TX, G.nx + 1);
  const int64_t y0 = int64_t(ty) * C::TY, y1 = min(y0 + C::TY, G.nyN);
  const int64_t z0 = G.lay_own_b + int64_t(ch) * G.chunk_len;
  const int64_t z1 = min(z0 + G.chunk_len, G.lay_own_e);
  if (z0 >= z1) return;
  const int64_t nxN = G.nx + 1;
  const int64_t cols_x = x1 - x0, cols = cols_x * (y1 - y0);

  auto node_id = [&](int64_t x, int64_t y, int64_t z) { return x + nxN * (y + G.nyN * z); };

  // zero the block-rows and R entries of the tile's nodes in layer z (first touch)
  auto zero_layer = [&](int64_t z) {
    for (int64_t c = 0; c < cols; ++c) {
      const int64_t x = x0 + c % cols_x, y = y0 + c / cols_x;
      int sl, W;
      slot_of(G, x, y, z, 0, 0, 0, NDPN, sl, W);
      const int64_t o = node_id(x, y, z) - G.own_node_b;
      double* row = val + base[o];
      const int n = NDPN * W;
      if constexpr (NDPN == 4) {
        for (int k = tid; k < n / 2; k += NT) __stcg(reinterpret_cast<double2*>(row) + k, make_double2(0.0, 0.0));
      } else {
        for (int k = tid; k < n; k += NT) __stcg(row + k, 0.0);
      }
      if (tid < NDPN) __stcg(Rv + o * NDPN + tid, 0.0);
    }
  };

  const int64_t s_first = max(z0 - 1, int64_t(0));
  const int64_t s_last = min(z1, G.nl) - 1;
  if (s_first == z0) zero_layer(z0);

  const int64_t ilo = max(x0 - 1, int64_t(0)), ihi = min(x1, G.nx);
  const int64_t jlo = (D == 3) ? max(y0 - 1, int64_t(0)) : 0;
  const int64_t jhi = (D == 3) ? min(y1, G.nyE) : 1;

  for (int64_t s = s_first; s <= s_last; ++s) {
    if (s + 1 >= z0 && s + 1 < z1) zero_layer(s + 1);
    __syncthreads();
    for (int c = 0; c < C::NCOL; ++c) {
      const int ci = c & 1, cj = c >> 1;
      const int64_t ifst = ilo + ((ilo & 1) != ci ? 1 : 0);
      const int64_t ni = ifst < ihi ? (ihi - ifst + 1) / 2 : 0;
      int64_t jfst = 0, nj = 1;
      if constexpr (D == 3) {
        jfst = jlo + ((jlo & 1) != cj ? 1 : 0);
        nj = jfst < jhi ? (jhi - jfst + 1) / 2 : 0;
      }
      const int64_t nc = ni * nj;
      for (int64_t b0 = 0; b0 < nc; b0 += E) {
        if (tid < E) {
          const int64_t k = b0 + tid;
          s_i[tid] = k < nc ? ifst + 2 * (k % ni) : -1;
          s_j[tid] = k < nc ? jfst + 2 * (k / ni) : -1;
        }
        __syncthreads();
        // gather node data of the batch elements
        for (int t = tid; t < E * NEN; t += NT) {
          const int el = t / NEN, a = t % NEN;
          if (s_i[el] >= 0) {
            int ox, oy, oz;
            node_off<D>(a, ox, oy, oz);
            const int64_t n = node_id(s_i[el] + ox, s_j[el] + oy, s + oz);
#pragma unroll
            for (int i = 0; i < D; ++i) Xs[t * D + i] = coords[n * D + i];
#pragma unroll
            for (int i = 0; i < NDPN; ++i) Us[t * NDPN + i] = dofs[n * NDPN + i];
          }
        }
        __syncthreads();
        // phase A
        for (int t = tid; t < E * NGP; t += NT) {
          const int el = t / NGP, g = t % NGP;
          if (s_i[el] >= 0) {
            const int64_t e = s_i[el] + G.nx * (s_j[el] + G.nyE * s);
            phaseA<D>(m, Xs + el * NEN * D, Us + el * NEN * NDPN, kappa[e * NGP + g], g,
                      recs + size_t(t) * GpBlock<D>::STRIDE, scal + t * kScal);
          }
        }
        __syncthreads();
        // phase C + accumulation into owned block-rows
        {
          const int el = tid / F::NPAIR, p = tid % F::NPAIR;
          if (el < E && s_i[el] >= 0) {
            int a, b;
            pair_ab<NEN>(p, a, b);
            int oax, oay, oaz, obx, oby, obz;
            node_off<D>(a, oax, oay, oaz);
            node_off<D>(b, obx, oby, obz);
            const int64_t ax = s_i[el] + oax, ay = s_j[el] + oay, az = s + oaz;
            const int64_t bx = s_i[el] + obx, by = s_j[el] + oby, bz = s + obz;
            const bool own_a = ax >= x0 && ax < x1 && ay >= y0 && ay < y1 && az >= z0 && az < z1;
            const bool own_b = bx >= x0 && bx < x1 && by >= y0 && by < y1 && bz >= z0 && bz < z1;
            if (own_a || own_b) {
              PairAcc<D> acc;
              phaseC<D>(recs + size_t(el) * NGP * GpBlock<D>::STRIDE, scal + el * NGP * kScal, a,
                        b, acc);
              // rows of node A: K(A,i; B,j)
              if (own_a) {
                int sl, W;
                slot_of(G, ax, ay, az, obx - oax, oby - oay, obz - oaz, NDPN, sl, W);
                const int64_t o = node_id(ax, ay, az) - G.own_node_b;
                double* row0 = val + base[o] + NDPN * sl;
#pragma unroll
                for (int i = 0; i < NDPN; ++i) {
                  double v[NDPN];
#pragma unroll
                  for (int j = 0; j < D; ++j) v[j] = (i < D) ? acc.Kuu[i < D ? i : 0][j] : acc.Keu_ab[j];
                  v[D] = (i < D) ? acc.Kue_ab[i < D ? i : 0] : acc.Kee_ab;
                  double* q = row0 + int64_t(i) * W;
                  if constexpr (NDPN == 4) {
                    double2* q2 = reinterpret_cast<double2*>(q);
                    double2 u0 = __ldcg(q2), u1 = __ldcg(q2 + 1);
                    u0.x += v[0]; u0.y += v[1]; u1.x += v[2]; u1.y += v[3];
                    __stcg(q2, u0);
                    __stcg(q2 + 1, u1);
                  } else {
#pragma unroll
                    for (int j = 0; j < NDPN; ++j) __stcg(q + j, __ldcg(q + j) + v[j]);
                  }
                }
                if (a == b) {
#pragma unroll
                  for (int i = 0; i < NDPN; ++i) {
                    double* r = Rv + o * NDPN + i;
                    __stcg(r, __ldcg(r) + acc.Fd[i]);
                  }
                }
              }
              // rows of node B (a != b): K(B,i; A,j) = transpose of Kuu_ab, *_ba blocks
              if (own_b && a != b) {
                int sl, W;
                slot_of(G, bx, by, bz, oax - obx, oay - oby, oaz - obz, NDPN, sl, W);
                const int64_t o = node_id(bx, by, bz) - G.own_node_b;
                double* row0 = val + base[o] + NDPN * sl;
#pragma unroll
                for (int i = 0; i < NDPN; ++i) {
                  double v[NDPN];
#pragma unroll
                  for (int j = 0; j < D; ++j) v[j] = (i < D) ? acc.Kuu[j][i < D ? i : 0] : acc.Keu_ba[j];
                  v[D] = (i < D) ? acc.Kue_ba[i < D ? i : 0] : acc.Kee_ba;
                  double* q = row0 + int64_t(i) * W;
                  if constexpr (NDPN == 4) {
                    double2* q2 = reinterpret_cast<double2*>(q);
                    double2 u0 = __ldcg(q2), u1 = __ldcg(q2 + 1);
                    u0.x += v[0]; u0.y += v[1]; u1.x += v[2]; u1.y += v[3];
                    __stcg(q2, u0);
                    __stcg(q2 + 1, u1);
                  } else {
#pragma unroll
                    for (int j = 0; j < NDPN; ++j) __stcg(q + j, __ldcg(q + j) + v[j]);
                  }
                }
              }
            }
          }
        }
        __syncthreads();
      }
    }
  }
}

}  // namespace lgdm

namespace {

bool sweep_supported(lgdm_mesh m) {
  if (!m->structured || m->f.dim < 2) return false;
  const int64_t per_layer = m->f.dim == 3 ? (m->nx + 1) * (m->ny + 1) : (m->nx + 1);
  return m->own_b % per_layer == 0 && m->own_e % per_layer == 0;
}

template <int D> lgdm_status launch_sweep(lgdm_mesh m) {
  using F = Fam<D>;
  using Cf = SweepCfg<D>;
  SweepGeom G{};
  G.nx = m->nx;
  if (D == 3) {
    G.nyE = m->ny;
    G.nyN = m->ny + 1;
    G.nl = m->nz;
  } else {
    G.nyE = 1;
    G.nyN = 1;
    G.nl = m->ny;
  }
  const int64_t per_layer = (G.nx + 1) * G.nyN;
  G.lay_own_b = m->own_b / per_layer;
  G.lay_own_e = m->own_e / per_layer;
  G.own_node_b = m->own_b;
  G.tiles_x = int((G.nx + 1 + Cf::TX - 1) / Cf::TX);
  G.tiles_y = int((G.nyN + Cf::TY - 1) / Cf::TY);
  const size_t smem = sizeof(double) * (size_t(Cf::E) * F::NGP * GpBlock<D>::STRIDE +
                                        Cf::E * F::NGP * kScal + Cf::E * F::NEN * D +
                                        Cf::E * F::NEN * F::NDPN);
  static bool attr = false;
  if (!attr) {
    CU(cudaFuncSetAttribute(k_sweep<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  int nsm = 148, per_sm = 1;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep<D>, Cf::E * F::NPAIR, smem);
  per_sm = std::max(per_sm, 1);
  const int64_t layers = G.lay_own_e - G.lay_own_b;
  const int64_t tiles = int64_t(G.tiles_x) * G.tiles_y;
  // enough CTAs for ~4 waves, but chunks of at least 8 layers (each chunk re-reads one layer)
  int64_t chunks = (4 * int64_t(nsm) * per_sm + tiles - 1) / tiles;
  chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, (layers + 7) / 8));
  G.chunk_len = (layers + chunks - 1) / chunks;
  G.chunks = int((layers + G.chunk_len - 1) / G.chunk_len);
  const int64_t grid = tiles * G.chunks;
  k_sweep<D><<<unsigned(grid), Cf::E * F::NPAIR, smem, m->stream>>>(
      m->dm, G, m->coords, m->dofs, m->kappa, m->base, m->val, m->R);
  return check_launch(m, "k_sweep");
}

lgdm_status assemble_sweep(lgdm_mesh m) {
  if (m->f.dim == 2) return launch_sweep<2>(m);
  return launch_sweep<3>(m);
}

void sweep_free(lgdm_mesh) {}

}  // namespace

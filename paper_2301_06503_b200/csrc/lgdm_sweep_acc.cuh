// lgdm_sweep_acc.cuh -- fused structured sweep with SHARED-MEMORY block-row accumulators.
//
// Same schedule and producer / consumer split as k_sweep (lgdm_sweep.cuh), but the owned
// block-rows of the two node layers being assembled live in shared memory, in "offset space"
// (all 3^d neighbour offsets, so every element contribution lands at a fixed position).  When
// the sweep passes a node layer its rows are complete: they are compacted to the node's real
// neighbour slots and streamed to HBM once, contiguously (consecutive x-nodes have consecutive
// block-rows), with no read-modify-write of K.  Per-entry summation order is
// (element layer, colour, GP) -- identical to k_sweep and independent of tiling / slabbing.
#pragma once

namespace lgdm {

template <int D> struct AccCfg;
template <> struct AccCfg<2> { static constexpr int TX = 32, TY = 1, E = 16, NCOL = 2, MINB = 2; };
template <> struct AccCfg<3> { static constexpr int TX = 4, TY = 4, E = 4, NCOL = 4, MINB = 1; };

template <int D> struct AccThreads {
  static constexpr int P = (AccCfg<D>::E * Fam<D>::NGP + 31) / 32 * 32;
  static constexpr int C = (AccCfg<D>::E * Fam<D>::NPAIR + 31) / 32 * 32;
  static constexpr int T = P + C;
};

template <int D> struct AccLayout {
  static constexpr int NSLOT = D == 3 ? 27 : (D == 2 ? 9 : 3);   // neighbour offsets
  static constexpr int NDPN = Fam<D>::NDPN;
  static constexpr int ROW = NSLOT * NDPN;                        // doubles per row i
  static constexpr int NODE = NDPN * ROW + NDPN;                  // block-row + R
  static constexpr int NODE_PAD = (NODE % 2 == 1) ? NODE : NODE + 1;
};

// full (offset-space) slot of neighbour offset (dx, dy, dz), each in {-1, 0, 1}
template <int D> __device__ __forceinline__ int full_slot(int dx, int dy, int dz) {
  if constexpr (D == 3) return ((dz + 1) * 3 + (dy + 1)) * 3 + (dx + 1);
  else return (dz + 1) * 3 + (dx + 1);
}

template <int D>
__global__ void __launch_bounds__(AccThreads<D>::T, AccCfg<D>::MINB)
k_sweep_acc(DevMat m, SweepGeom G, const double* __restrict__ coords,
            const double* __restrict__ dofs, const double* __restrict__ kappa,
            const int64_t* __restrict__ base, double* __restrict__ val, double* __restrict__ Rv) {
  using F = Fam<D>;
  using Cf = AccCfg<D>;
  using Th = AccThreads<D>;
  using AL = AccLayout<D>;
  constexpr int E = Cf::E, NDPN = F::NDPN, NEN = F::NEN, NGP = F::NGP;
  constexpr int CS = Core<D>::STRIDE, GB = GpBlock<D>::STRIDE;
  constexpr int NCOLS = Cf::TX * Cf::TY;
  extern __shared__ double sm[];
  double* cores = sm;                             // [2][E][NGP][CS]
  double* recs = cores + 2 * E * NGP * CS;        // [E][NGP][GB]
  double* acc = recs + E * NGP * GB;              // [2 layers][NCOLS][NODE_PAD]
  const int tid = threadIdx.x;

  int bid = blockIdx.x;
  const int tx = bid % G.tiles_x;
  bid /= G.tiles_x;
  const int ty = bid % G.tiles_y;
  const int ch = bid / G.tiles_y;
  const int64_t x0 = int64_t(tx) * Cf::TX, x1 = min(x0 + Cf::TX, G.nx + 1);
  const int64_t y0 = int64_t(ty) * Cf::TY, y1 = min(y0 + Cf::TY, G.nyN);
  const int64_t z0 = G.lay_own_b + int64_t(ch) * G.chunk_len;
  const int64_t z1 = min(z0 + G.chunk_len, G.lay_own_e);
  if (z0 >= z1) return;
  const int64_t nxN = G.nx + 1;
  auto node_id = [&](int64_t x, int64_t y, int64_t z) { return x + nxN * (y + G.nyN * z); };

  const int64_t s_first = max(z0 - 1, int64_t(0));
  const int64_t s_last = min(z1, G.nl) - 1;
  const int64_t ilo = max(x0 - 1, int64_t(0)), ihi = min(x1, G.nx);
  const int64_t jlo = (D == 3) ? max(y0 - 1, int64_t(0)) : 0;
  const int64_t jhi = (D == 3) ? min(y1, G.nyE) : 1;
  const int64_t cols_x = x1 - x0, cols = cols_x * (y1 - y0);

  // schedule: per element layer s, per colour, batches of E; end_of_layer(s) after each layer
  auto schedule = [&](auto&& body, auto&& end_of_layer) {
    for (int64_t s = s_first; s <= s_last; ++s) {
      for (int c = 0; c < Cf::NCOL; ++c) {
        const int ci = c & 1;
        const int ifst = int(ilo) + ((ilo & 1) != ci ? 1 : 0);
        const int ni = ifst < ihi ? (int(ihi) - ifst + 1) / 2 : 0;
        int jfst = 0, nj = 1;
        if constexpr (D == 3) {
          const int cj = c >> 1;
          jfst = int(jlo) + ((jlo & 1) != cj ? 1 : 0);
          nj = jfst < jhi ? (int(jhi) - jfst + 1) / 2 : 0;
        }
        const int nc = ni * nj;
        for (int b0 = 0; b0 < nc; b0 += E) body(s, b0, ifst, ni, jfst, nc);
      }
      end_of_layer(s);
    }
  };

  if (tid < Th::P) {
    // ------------------------------ producer warps ------------------------------
    const int el = tid / NGP, g = tid % NGP;
    int t = 0;
    PT_DECL
    schedule(
        [&](int64_t s, int b0, int ifst, int ni, int jfst, int nc) {
          const int buf = t & 1;
          if (t >= 2) bar_sync_empty(buf, Th::T);
          PT_MARK(0, tid == 0);
          const int k = b0 + el;
          if (el < E && k < nc) {
            const int i = ifst + 2 * (k % ni), j = jfst + 2 * (k / ni);
            auto nid = [&](int a) {
              int ox, oy, oz;
              node_off<D>(a, ox, oy, oz);
              return node_id(i + ox, j + oy, s + oz);
            };
            auto X = [&](int a, int q) { return __ldg(coords + nid(a) * D + q); };
            auto U = [&](int a, int q) { return __ldg(dofs + nid(a) * NDPN + q); };
            const int64_t e = i + G.nx * (j + G.nyE * s);
            gpCore<D>(m, X, U, __ldg(kappa + e * NGP + g), g, cores + (size_t(buf) * E * NGP + tid) * CS);
          }
          PT_MARK(1, tid == 0);
          bar_arrive_full(buf, Th::T);
          ++t;
        },
        [&](int64_t) {});
    for (int k = max(t - 2, 0); k < t; ++k) bar_sync_empty(k & 1, Th::T);
    return;
  }

  // -------------------------------- consumer warps --------------------------------
  const int ct = tid - Th::P;
  const int cel = ct / F::NPAIR, cp = ct % F::NPAIR;
  int pa, pb;
  pair_ab<NEN>(cp, pa, pb);
  int oax, oay, oaz, obx, oby, obz;
  node_off<D>(pa, oax, oay, oaz);
  node_off<D>(pb, obx, oby, obz);
  const int fsAB = full_slot<D>(obx - oax, oby - oay, obz - oaz);
  const int fsBA = full_slot<D>(oax - obx, oay - oby, oaz - obz);

  auto accp = [&](int64_t z, int64_t x, int64_t y) {
    return acc + (size_t(z & 1) * NCOLS + (x - x0) + cols_x * (y - y0)) * AL::NODE_PAD;
  };
  auto zero_parity = [&](int par) {
    double* a0 = acc + size_t(par) * NCOLS * AL::NODE_PAD;
    for (int k = ct; k < NCOLS * AL::NODE_PAD; k += Th::C) a0[k] = 0.0;
  };
  // stream the complete rows of the tile's nodes in layer z to HBM (warp per node)
  auto flush_layer = [&](int64_t z) {
    const int warp = ct >> 5, lane = ct & 31;
    for (int64_t c = warp; c < cols; c += Th::C / 32) {
      const int64_t x = x0 + c % cols_x, y = y0 + c / cols_x;
      const int xlo = x > 0 ? -1 : 0, xhi = x < G.nx ? 1 : 0;
      const int ylo = y > 0 ? -1 : 0, yhi = y < G.nyN - 1 ? 1 : 0;
      const int zlo = z > 0 ? -1 : 0, zhi = z < G.nl ? 1 : 0;
      const int wx = xhi - xlo + 1, wy = yhi - ylo + 1, wz = zhi - zlo + 1;
      const int deg = wx * wy * wz, W = deg * NDPN;
      const int64_t o = node_id(x, y, z) - G.own_node_b;
      double* out = val + base[o];
      const double* src = accp(z, x, y);
      for (int idx = lane; idx < NDPN * W; idx += 32) {
        const int i = idx / W, cc = idx % W, sl = cc / NDPN, j = cc % NDPN;
        const int dx = xlo + sl % wx, dy = ylo + (sl / wx) % wy, dz = zlo + sl / (wx * wy);
        __stcs(out + idx, src[i * AL::ROW + full_slot<D>(dx, dy, dz) * NDPN + j]);
      }
      if (lane < NDPN) __stcs(Rv + o * NDPN + lane, src[NDPN * AL::ROW + lane]);
    }
  };

  zero_parity(0);
  zero_parity(1);
  // (made visible by the consumer barrier after the first expansion)
  int t = 0;
  PT_DECL
  schedule(
      [&](int64_t s, int b0, int ifst, int ni, int jfst, int nc) {
        const int buf = t & 1;
        PT_MARK(2, ct == 0);
        bar_sync_full(buf, Th::T);
        PT_MARK(3, ct == 0);
        const double* cb = cores + size_t(buf) * E * NGP * CS;
        for (int it = ct; it < E * NGP * NEN; it += Th::C) {
          const int eg = it / NEN, a = it % NEN;
          if (b0 + eg / NGP < nc)
            gpExpand<D>(cb + eg * CS, a, eg % NGP, recs + size_t(eg) * GB + a * Rec<D>::STRIDE);
        }
        PT_MARK(4, ct == 0);
        bar_sync<BAR_CONS>(Th::C);
        PT_MARK(5, ct == 0);
        const int k = b0 + cel;
        if (cel < E && k < nc) {
          const int i = ifst + 2 * (k % ni), j = jfst + 2 * (k / ni);
          const int64_t ax = i + oax, ay = j + oay, az = s + oaz;
          const int64_t bx = i + obx, by = j + oby, bz = s + obz;
          const bool own_a = ax >= x0 && ax < x1 && ay >= y0 && ay < y1 && az >= z0 && az < z1;
          const bool own_b = bx >= x0 && bx < x1 && by >= y0 && by < y1 && bz >= z0 && bz < z1;
          if (own_a || own_b) {
            PairAcc<D> pacc;
            phaseC<D, CS, Core<D>::MU, Core<D>::GHC>(recs + size_t(cel) * NGP * GB,
                                                      cb + cel * NGP * CS, pa, pb, pacc);
            // colour batches share no node, so these shared-memory updates never collide
            if (own_a) {
              double* A = accp(az, ax, ay);
#pragma unroll
              for (int r = 0; r < D; ++r) {
#pragma unroll
                for (int q = 0; q < D; ++q) A[r * AL::ROW + fsAB * NDPN + q] += pacc.Kuu[r][q];
                A[r * AL::ROW + fsAB * NDPN + D] += pacc.Kue_ab[r];
                A[D * AL::ROW + fsAB * NDPN + r] += pacc.Keu_ab[r];
              }
              A[D * AL::ROW + fsAB * NDPN + D] += pacc.Kee_ab;
              if (pa == pb) {
#pragma unroll
                for (int r = 0; r < NDPN; ++r) A[NDPN * AL::ROW + r] += pacc.Fd[r];
              }
            }
            if (own_b && pa != pb) {
              double* B = accp(bz, bx, by);
#pragma unroll
              for (int r = 0; r < D; ++r) {
#pragma unroll
                for (int q = 0; q < D; ++q) B[r * AL::ROW + fsBA * NDPN + q] += pacc.Kuu[q][r];
                B[r * AL::ROW + fsBA * NDPN + D] += pacc.Kue_ba[r];
                B[D * AL::ROW + fsBA * NDPN + r] += pacc.Keu_ba[r];
              }
              B[D * AL::ROW + fsBA * NDPN + D] += pacc.Kee_ba;
            }
          }
        }
        PT_MARK(6, ct == 0);
        bar_arrive_empty(buf, Th::T);
        bar_sync<BAR_CONS>(Th::C);
        PT_MARK(9, ct == 0);
        ++t;
      },
      [&](int64_t s) {
        PT_MARK(2, ct == 0);
        // node layer s is complete after element layer s (and layer s+1 too at the top)
        if (s >= z0 && s < z1) flush_layer(s);
        if (s == s_last && s + 1 >= z0 && s + 1 < z1) flush_layer(s + 1);
        bar_sync<BAR_CONS>(Th::C);
        zero_parity(int(s & 1));
        bar_sync<BAR_CONS>(Th::C);
        PT_MARK(8, ct == 0);
      });
}

}  // namespace lgdm

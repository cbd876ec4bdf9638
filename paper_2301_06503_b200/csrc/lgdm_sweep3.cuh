// lgdm_sweep3.cuh -- the hot kernel: fused structured-sweep K/R assembly with a three-stage
// warp-specialised pipeline and shared-memory block-row accumulation.  Included by
// lgdm_sweep.cuh (needs SweepGeom, node_off, first_contrib-free helpers, named barriers).
//
// One CTA owns a tile of TX x TY node columns and a chunk of node layers, sweeps the element
// layers touching them, and writes exactly the CSR block-rows (and R entries) of its nodes:
//   PC warps  (element x GP)   Gauss-point cores of batch t+1: geometry, kinematics, the
//                               Appendix A update and the tangent coefficients (gpCore)
//   PE warps  (element x node) per Gauss point g: the node expansions (gpExpand) of batch t
//                               into a double-buffered per-GP record block
//   C warps   (element x pair) Gauss sums of Eqs. 11a-f for node pairs a<=b in registers
//                               (Kuu symmetry), then one add into the shared-memory rows
// Elements are processed by layer, then colour (parity of i, j), in batches of E elements of
// one colour, which share no node -- so the shared-memory adds never collide and the per-entry
// summation order (layer, colour, GP) depends only on global indices (bitwise slab-invariant).
//
// Accumulators are split by neighbour plane dz = zB - zA (node rows are sorted by (z, y, x),
// so each plane is a contiguous piece of every row): while element layer s is processed a
// column holds plane 0 of node layer s (carried from layer s-1), plane +1 of node layer s,
// plane -1 and plane 0 of node layer s+1.  At the end of layer s the finished planes are
// compacted to the node's real neighbour slots and streamed to HBM once; plane 0 of layer s+1
// is carried.  DRAM therefore sees every K value written exactly once, with no zero fill and
// no read-modify-write.
#pragma once

namespace lgdm {

template <int D> struct S3Cfg;
// tile footprint (TX+1) x (TY+1) elements = NCOL colours x E: full batches for interior tiles.
// Thread counts are kept at <= 16 warps so that no SMSP holds more than 4 warps of a CTA and
// MAXREG registers are available (FP64 pair accumulators must not spill).
template <> struct S3Cfg<2> { static constexpr int TX = 31, TY = 1, E = 16, NCOL = 2, MAXREG = 112, MINB = 2; };
template <> struct S3Cfg<3> { static constexpr int TX = 3, TY = 7, E = 8, NCOL = 4, MAXREG = 128, MINB = 1; };

template <int D> struct S3Threads {
  static constexpr int PC = (S3Cfg<D>::E * Fam<D>::NGP + 31) / 32 * 32;
  static constexpr int PE = (S3Cfg<D>::E * Fam<D>::NEN + 31) / 32 * 32;
  static constexpr int C = (S3Cfg<D>::E * Fam<D>::NPAIR + 31) / 32 * 32;
  static constexpr int T = PC + PE + C;
};

template <int D> struct S3Layout {
  static constexpr int NDPN = Fam<D>::NDPN;
  // slot stride in doubles: odd, so the 16 lanes of a half-warp adding into different slots,
  // rows and planes of a column hit different 8-byte banks
  static constexpr int SS = (NDPN % 2 == 1) ? NDPN : NDPN + 1;
  static constexpr int PSLOT = D == 3 ? 9 : 3;               // in-plane neighbour offsets
  static constexpr int PROW = PSLOT * SS;                    // doubles of one row in one plane
  static constexpr int PLANE = NDPN * PROW;                  // one plane of one node's rows
  // per column: Z[2] (plane 0, by node-layer parity), UP (plane +1 of layer s),
  // DN (plane -1 of layer s+1), R[2] (by node-layer parity)
  static constexpr int Z0 = 0, Z1 = PLANE, UP = 2 * PLANE, DN = 3 * PLANE, R0 = 4 * PLANE,
                       R1 = 4 * PLANE + NDPN;
  static constexpr int COL = 4 * PLANE + 2 * NDPN;
  static constexpr int COL_PAD = (COL % 2 == 1) ? COL : COL + 1;
};

// in-plane slot of offset (dx, dy)
template <int D> __device__ __forceinline__ int plane_slot(int dx, int dy) {
  if constexpr (D == 3) return (dy + 1) * 3 + (dx + 1);
  else return dx + 1;
}

// barrier ids (0 is __syncthreads)
enum { B_CFULL = 1, B_CEMPTY = 3, B_RFULL = 5, B_REMPTY = 9, B_CONS3 = 13 };
constexpr int kRecRing = 3;   // per-GP record buffers in flight
template <int BASE> __device__ __forceinline__ void sync2(int buf, int n) {
  if (buf) bar_sync<BASE + 1>(n); else bar_sync<BASE>(n);
}
template <int BASE> __device__ __forceinline__ void arrive2(int buf, int n) {
  if (buf) bar_arrive<BASE + 1>(n); else bar_arrive<BASE>(n);
}
template <int BASE> __device__ __forceinline__ void sync4(int buf, int n) {
  switch (buf) {
    case 0: bar_sync<BASE>(n); break;
    case 1: bar_sync<BASE + 1>(n); break;
    default: bar_sync<BASE + 2>(n); break;
  }
}
template <int BASE> __device__ __forceinline__ void arrive4(int buf, int n) {
  switch (buf) {
    case 0: bar_arrive<BASE>(n); break;
    case 1: bar_arrive<BASE + 1>(n); break;
    default: bar_arrive<BASE + 2>(n); break;
  }
}

template <int D>
__global__ void __launch_bounds__(S3Threads<D>::T, S3Cfg<D>::MINB) __maxnreg__(S3Cfg<D>::MAXREG)
k_sweep3(DevMat m, SweepGeom G, const double* __restrict__ coords,
         const double* __restrict__ dofs, const double* __restrict__ kappa,
         const int64_t* __restrict__ base, double* __restrict__ val, double* __restrict__ Rv) {
  using F = Fam<D>;
  using Cf = S3Cfg<D>;
  using Th = S3Threads<D>;
  using L = S3Layout<D>;
  using Rc = Rec<D>;
  constexpr int E = Cf::E, NDPN = F::NDPN, NEN = F::NEN, NGP = F::NGP;
  constexpr int CS = Core<D>::STRIDE, GB = GpBlock<D>::STRIDE;
  constexpr int NCOLS = Cf::TX * Cf::TY;
  constexpr int MU_AT = NEN * Rc::STRIDE, GHC_AT = NEN * Rc::STRIDE + 1;   // pad of each GP block
  static_assert(GB >= NEN * Rc::STRIDE + 2, "GP block needs two spare doubles for mu*, ghc");
  extern __shared__ double sm[];
  double* cores = sm;                             // [2][E][NGP][CS]
  double* recs = cores + 2 * E * NGP * CS;        // [kRecRing][E][GB]  (one Gauss point each)
  double* acc = recs + kRecRing * E * GB;         // [NCOLS][COL_PAD]
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
  const int ilo = int(max(x0 - 1, int64_t(0))), ihi = int(min(x1, G.nx));
  const int jlo = (D == 3) ? int(max(y0 - 1, int64_t(0))) : 0;
  const int jhi = (D == 3) ? int(min(y1, G.nyE)) : 1;
  const int cols_x = int(x1 - x0), cols = cols_x * int(y1 - y0);

  // batch schedule (identical in every role): layer s, colour c, batches of E elements
  auto schedule = [&](auto&& body, auto&& end_of_layer) {
    for (int64_t s = s_first; s <= s_last; ++s) {
      for (int c = 0; c < Cf::NCOL; ++c) {
        const int ifst = ilo + ((ilo & 1) != (c & 1) ? 1 : 0);
        const int ni = ifst < ihi ? (ihi - ifst + 1) / 2 : 0;
        int jfst = 0, nj = 1;
        if constexpr (D == 3) {
          jfst = jlo + ((jlo & 1) != (c >> 1) ? 1 : 0);
          nj = jfst < jhi ? (jhi - jfst + 1) / 2 : 0;
        }
        const int nc = ni * nj;
        for (int b0 = 0; b0 < nc; b0 += E) body(s, c, b0, ifst, ni, jfst, nc);
      }
      end_of_layer(s);
    }
  };
  auto noop_layer = [](int64_t) {};

  if (tid < Th::PC) {
    // ---------------------------- PC: Gauss-point cores ----------------------------
    const int el = tid / NGP, g = tid % NGP;
    int t = 0;
    PT_DECL
    schedule(
        [&](int64_t s, int, int b0, int ifst, int ni, int jfst, int nc) {
          const int buf = t & 1;
          if (t >= 2) sync2<B_CEMPTY>(buf, Th::PC + Th::PE);
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
            gpCore<D>(m, X, U, __ldg(kappa + e * NGP + g), g,
                      cores + (size_t(buf) * E * NGP + el * NGP + g) * CS);
          }
          PT_MARK(1, tid == 0);
          arrive2<B_CFULL>(buf, Th::PC + Th::PE);
          ++t;
        },
        noop_layer);
    for (int k = max(t - 2, 0); k < t; ++k) sync2<B_CEMPTY>(k & 1, Th::PC + Th::PE);
    return;
  }

  if (tid < Th::PC + Th::PE) {
    // ------------------------- PE: per-GP node expansions -------------------------
    const int pt = tid - Th::PC;
    const int el = pt / NEN, a = pt % NEN;
    int t = 0, q = 0;
    PT_DECL
    schedule(
        [&](int64_t, int, int b0, int, int, int, int nc) {
          const int buf = t & 1;
          sync2<B_CFULL>(buf, Th::PC + Th::PE);
          PT_MARK(2, pt == 0);
          const double* cb = cores + size_t(buf) * E * NGP * CS;
          const bool live = el < E && b0 + el < nc;
          for (int g = 0; g < NGP; ++g, ++q) {
            const int rb = q % kRecRing;
            if (q >= kRecRing) sync4<B_REMPTY>(rb, Th::PE + Th::C);
            PT_MARK(3, pt == 0);
            double* blk = recs + (size_t(rb) * E + el) * GB;
            if (live) {
              const double* co = cb + (el * NGP + g) * CS;
              gpExpand<D>(co, a, g, blk + a * Rc::STRIDE);
              if (a == 0) {
                blk[MU_AT] = co[Core<D>::MU];
                blk[GHC_AT] = co[Core<D>::GHC];
              }
            }
            PT_MARK(4, pt == 0);
            arrive4<B_RFULL>(rb, Th::PE + Th::C);
          }
          arrive2<B_CEMPTY>(buf, Th::PC + Th::PE);
          ++t;
        },
        noop_layer);
    for (int k = max(q - kRecRing, 0); k < q; ++k) sync4<B_REMPTY>(k % kRecRing, Th::PE + Th::C);
    return;
  }

  // ------------------------------- C: pair sums + rows -------------------------------
  const int ct = tid - Th::PC - Th::PE;
  const int cel = ct / F::NPAIR, cp = ct % F::NPAIR;
  int pa, pb;
  pair_ab<NEN>(cp, pa, pb);
  int oax, oay, oaz, obx, oby, obz;
  node_off<D>(pa, oax, oay, oaz);
  node_off<D>(pb, obx, oby, obz);
  const int psAB = plane_slot<D>(obx - oax, oby - oay), psBA = plane_slot<D>(oax - obx, oay - oby);
  const int dzAB = obz - oaz;   // -1, 0, +1

  auto col_of = [&](int64_t x, int64_t y) { return acc + size_t((x - x0) + cols_x * (y - y0)) * L::COL_PAD; };
  // plane buffer for node layer zn (in {s, s+1}) and offset dz, during element layer s
  auto plane_of = [&](double* colp, int64_t zn, int64_t s, int dz) -> double* {
    if (dz == 0) return colp + ((zn & 1) ? L::Z1 : L::Z0);
    if (zn == s) return colp + L::UP;   // dz = +1
    return colp + L::DN;                // zn == s+1, dz = -1
  };

  // stream plane dz of the rows of node (x, y, z) (compacted to its real slots) to HBM
  auto flush_plane = [&](int64_t x, int64_t y, int64_t z, int dz, const double* src, int lane) {
    const int xlo = x > 0 ? -1 : 0, xhi = x < G.nx ? 1 : 0;
    const int ylo = y > 0 ? -1 : 0, yhi = y < G.nyN - 1 ? 1 : 0;
    const int zlo = z > 0 ? -1 : 0, zhi = z < G.nl ? 1 : 0;
    const int wx = xhi - xlo + 1, wy = yhi - ylo + 1, wz = zhi - zlo + 1;
    const int pw = wx * wy * NDPN;                 // doubles of this plane in one row
    const int W = pw * wz;
    double* out = val + base[node_id(x, y, z) - G.own_node_b] + (dz - zlo) * pw;
    for (int idx = lane; idx < NDPN * pw; idx += 32) {
      const int i = idx / pw, r = idx % pw, sl = r / NDPN, j = r % NDPN;
      const int dx = xlo + sl % wx, dy = ylo + sl / wx;
      __stcs(out + int64_t(i) * W + r, src[i * L::PROW + plane_slot<D>(dx, dy) * L::SS + j]);
    }
  };

  for (int k = ct; k < NCOLS * L::COL_PAD; k += Th::C) acc[k] = 0.0;
  bar_sync<B_CONS3>(Th::C);

  int q = 0, prev_c = -1;
  PT_DECL
  schedule(
      [&](int64_t s, int c, int b0, int ifst, int ni, int jfst, int nc) {
        const int k = b0 + cel;
        const bool live = cel < E && k < nc;
        int64_t ax = 0, ay = 0, az = 0, bx = 0, by = 0, bz = 0;
        bool own_a = false, own_b = false;
        if (live) {
          const int i = ifst + 2 * (k % ni), j = jfst + 2 * (k / ni);
          ax = i + oax; ay = j + oay; az = s + oaz;
          bx = i + obx; by = j + oby; bz = s + obz;
          own_a = ax >= x0 && ax < x1 && ay >= y0 && ay < y1 && az >= z0 && az < z1;
          own_b = bx >= x0 && bx < x1 && by >= y0 && by < y1 && bz >= z0 && bz < z1;
        }
        const bool work = own_a || own_b;
        PairAcc<D> pacc;
#pragma unroll
        for (int r = 0; r < D; ++r) {
#pragma unroll
          for (int u = 0; u < D; ++u) pacc.Kuu[r][u] = 0.0;
          pacc.Kue_ab[r] = pacc.Kue_ba[r] = pacc.Keu_ab[r] = pacc.Keu_ba[r] = 0.0;
        }
        pacc.Kee_ab = pacc.Kee_ba = 0.0;
#pragma unroll
        for (int r = 0; r <= D; ++r) pacc.Fd[r] = 0.0;
        for (int g = 0; g < NGP; ++g, ++q) {
          const int rb = q % kRecRing;
          PT_MARK(5, ct == 0);
          sync4<B_RFULL>(rb, Th::PE + Th::C);
          PT_MARK(6, ct == 0);
#ifndef LGDM_EXP
#define LGDM_EXP 0
#endif
          if (work && LGDM_EXP != 1) {
            const double* blk = recs + (size_t(rb) * E + cel) * GB;
            PairIn<D> in;
            load_pair<D>(blk + pa * Rc::STRIDE, blk + pb * Rc::STRIDE, in);
            accumulate_pair<D>(in, blk[MU_AT], blk[GHC_AT], pacc);
            if (pa == pb) {
#pragma unroll
              for (int r = 0; r <= D; ++r) pacc.Fd[r] += blk[pa * Rc::STRIDE + Rc::f(r)];
            }
          }
          PT_MARK(7, ct == 0);
          arrive4<B_REMPTY>(rb, Th::PE + Th::C);
        }
        // batches of one colour share no node; a new colour waits for the previous adds
        if (c != prev_c) bar_sync<B_CONS3>(Th::C);
        PT_MARK(8, ct == 0);
        prev_c = c;
        if (own_a && LGDM_EXP != 2) {
          double* P = plane_of(col_of(ax, ay), az, s, dzAB);
#pragma unroll
          for (int r = 0; r < D; ++r) {
#pragma unroll
            for (int u = 0; u < D; ++u) P[r * L::PROW + psAB * L::SS + u] += pacc.Kuu[r][u];
            P[r * L::PROW + psAB * L::SS + D] += pacc.Kue_ab[r];
            P[D * L::PROW + psAB * L::SS + r] += pacc.Keu_ab[r];
          }
          P[D * L::PROW + psAB * L::SS + D] += pacc.Kee_ab;
          if (pa == pb) {
            double* Rp = col_of(ax, ay) + ((az & 1) ? L::R1 : L::R0);
#pragma unroll
            for (int r = 0; r < NDPN; ++r) Rp[r] += pacc.Fd[r];
          }
        }
        if (own_b && pa != pb && LGDM_EXP != 2) {
          double* P = plane_of(col_of(bx, by), bz, s, -dzAB);
#pragma unroll
          for (int r = 0; r < D; ++r) {
#pragma unroll
            for (int u = 0; u < D; ++u) P[r * L::PROW + psBA * L::SS + u] += pacc.Kuu[u][r];
            P[r * L::PROW + psBA * L::SS + D] += pacc.Kue_ba[r];
            P[D * L::PROW + psBA * L::SS + r] += pacc.Keu_ba[r];
          }
          P[D * L::PROW + psBA * L::SS + D] += pacc.Kee_ba;
        }
        PT_MARK(9, ct == 0);
      },
      [&](int64_t s) {
        bar_sync<B_CONS3>(Th::C);
        PT_MARK(10, ct == 0);
        prev_c = -1;
        // flush: node layer s (planes 0, +1; plane -1 went out a layer ago), plane -1 of
        // node layer s+1, and at the top of the chunk the whole of node layer s+1
        const int warp = ct >> 5, lane = ct & 31;
        const bool own_s = s >= z0 && s < z1, own_s1 = s + 1 >= z0 && s + 1 < z1;
        const bool top = s == s_last && own_s1;   // no element layer above node layer s+1
        for (int cc = warp; cc < cols && LGDM_EXP != 3; cc += Th::C / 32) {
          const int64_t x = x0 + cc % cols_x, y = y0 + cc / cols_x;
          double* colp = col_of(x, y);
          if (own_s) {
            flush_plane(x, y, s, 0, colp + ((s & 1) ? L::Z1 : L::Z0), lane);
            if (s < G.nl) flush_plane(x, y, s, 1, colp + L::UP, lane);
            if (lane < NDPN)
              __stcs(Rv + (node_id(x, y, s) - G.own_node_b) * NDPN + lane, colp[((s & 1) ? L::R1 : L::R0) + lane]);
          }
          if (own_s1) {
            flush_plane(x, y, s + 1, -1, colp + L::DN, lane);
            if (top) {
              flush_plane(x, y, s + 1, 0, colp + (((s + 1) & 1) ? L::Z1 : L::Z0), lane);
              if (lane < NDPN)
                __stcs(Rv + (node_id(x, y, s + 1) - G.own_node_b) * NDPN + lane,
                       colp[(((s + 1) & 1) ? L::R1 : L::R0) + lane]);
            }
          }
        }
        bar_sync<B_CONS3>(Th::C);
        // reset: plane 0 and R of node layer s (reused for layer s+2), UP, DN
        for (int k = ct; k < NCOLS * (2 * L::PLANE + L::PLANE + NDPN); k += Th::C) {
          const int col = k / (3 * L::PLANE + NDPN), r = k % (3 * L::PLANE + NDPN);
          double* colp = acc + size_t(col) * L::COL_PAD;
          if (r < L::PLANE) colp[((s & 1) ? L::Z1 : L::Z0) + r] = 0.0;
          else if (r < 3 * L::PLANE) colp[L::UP + (r - L::PLANE)] = 0.0;   // UP and DN are adjacent
          else colp[((s & 1) ? L::R1 : L::R0) + (r - 3 * L::PLANE)] = 0.0;
        }
        bar_sync<B_CONS3>(Th::C);
        PT_MARK(11, ct == 0);
      });
}

}  // namespace lgdm

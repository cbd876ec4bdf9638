// lgdm_hex8.cuh -- Hex8 hot kernel (k_hex8): the structured-sweep K/R assembly of Eqs. 11a-f
// (P:94-104), Alg. 2's "Compute and Assemble".  Included by lgdm_sweep.cuh
// (needs SweepGeom, node_off, plane_slot, Core/gpCore and the S4 / C4 / pos4 / pair4 layout
// helpers of lgdm_sweep4.cuh).
//
// Contract (same as k_sweep4): one CTA owns TX x TY node columns and a chunk of node layers,
// sweeps the element layers touching them (ghost elements recomputed), writes exactly the CSR
// block-rows of its nodes.  Per-entry summation order = (element layer, colour): within a
// colour batch every block-row entry receives at most one add, so K and R are bitwise
// independent of tiling and slabbing.  Diagonal 4x4 blocks from the partition-of-unity
// row-sum identity at flush.
//
// Roles as in k_sweep4 -- PC warps compute the Appendix A cores into a ring, one C warp per
// element of a colour batch, the layer flush split between C and PC warps -- with the Kuu
// pair stage rebuilt around register tiling (ncu of k_sweep4: the 28 pair lanes loaded 29
// doubles of records per pair and GP, 4.7 B per FMA, a third of all shared-memory wavefronts):
//   * the 32 lanes of a C warp are 8 tiles x 4 GP quarters.  A tile is a 2 x 2 block of node
//     pairs (groups {2i, 2i+1} x {2j, 2j+1}; tiles 6, 7 take the 4 intra-group pairs).  A lane
//     loads J^-1, S, lam*, Ams, Ass, mu*, ghc of its GP from the core ring (12 x 16 B), rebuilds
//     grad N and S grad N of its 4 nodes in registers and Gauss-sums 4 Kuu blocks at once;
//   * a fixed-order shuffle reduction over the GP quarters leaves one pair per lane, and one
//     more shuffle hands each pair to the lane that adds it in k_sweep4's bank-searched order;
//   * the node expansions only produce the coupling records (W' grad N, Dt' grad N, E) that the
//     shape-function moments read, plus the node sums.
#pragma once

#include <type_traits>

namespace lgdm {

struct H8 {
  static constexpr int TX = S4::TX, TY = S4::TY, E = S4::E, NCOL = S4::NCOL;
  static constexpr int NGP = 8, NEN = 8, NDPN = 4, NOFF = 28;
  static constexpr int NPC = 4, NC = E;                          // warps per role
  static constexpr int T = 32 * (NPC + NC);
  static constexpr int SHT = S4::SHT;
  static constexpr int CSP = S4::CSP, CEL = S4::CEL, CSLOT = S4::CSLOT, NCSLOT = S4::NCSLOT;
  // warp-private coupling records [4 GP][8 node][RS] = [w0 w1 | w2 d0 | d1 d2 | E pad | pad pad]
  // (RS = 5 x 16 B: the 8 nodes of a quarter-warp store to distinct bank groups); the moments
  // M[n][m][c] reuse the buffer afterwards (mom_idx)
  static constexpr int RS = 10, RGP = NEN * RS, RWARP = 504;
  static constexpr int PLD = S4::PLD, Z0 = S4::Z0, Z1 = S4::Z1, UP = S4::UP, DN = S4::DN,
                       NS = S4::NS, COL = S4::COL;
  static constexpr int NCOLS = TX * TY;
  static constexpr size_t SMEM = sizeof(double) * (size_t(SHT) + size_t(NCSLOT) * CSLOT +
                                                   size_t(NC) * RWARP + size_t(NCOLS) * COL);
  static constexpr int B_CF = S4::B_CF, B_CE = S4::B_CE, B_C = S4::B_C, B_AD = S4::B_AD, B_FL = S4::B_FL;
  // per-thread registers by warpgroup (setmaxnreg): PC warps 0-3, C warps 4-11; the launch
  // gives 168 = 65536 / 384
  static constexpr int REG_PC = 128, REG_C = 184;
  static_assert(REG_PC + 2 * REG_C <= 3 * 168, "register file");
  static_assert(4 * RGP <= RWARP && 7 * 63 + 7 * 7 + 7 <= RWARP, "records and moments fit");
};

// warpgroup register reallocation (sm_90a / sm_100a; all 4 warps of the warpgroup execute it)
template <int N> __device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N));
}
template <int N> __device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N));
}

// shape-function derivatives dN_a/dxi_j at Gauss point g for runtime (a, g)
__device__ __forceinline__ void shape_rt(int a, int g, double (&dn)[3]) {
#pragma unroll
  for (int j = 0; j < 3; ++j) dn[j] = shape_dxi<3>(a, g, j);
}

// tile t (0..7) -> nodes (A1, A2, B1, B2); tiles 0-5 are the 2 x 2 blocks between node groups
// {2i, 2i+1} x {2j, 2j+1} (all four pairs), tiles 6 and 7 take the intra-group pairs
// (A1, B1) and (A2, B2) only.  Pair slots: p0 (A1,B1), p1 (A1,B2), p2 (A2,B1), p3 (A2,B2).
__device__ __forceinline__ void tile_nodes(int t, int& A1, int& A2, int& B1, int& B2) {
  if (t < 6) {
    const int gi = (t < 3) ? 0 : (t < 5 ? 1 : 2);
    const int gj = (t < 3) ? t + 1 : (t < 5 ? t - 1 : 3);
    A1 = 2 * gi; A2 = 2 * gi + 1; B1 = 2 * gj; B2 = 2 * gj + 1;
  } else {
    const int o = (t - 6) * 4;
    A1 = o; A2 = o + 2; B1 = o + 1; B2 = o + 3;
  }
}
// after the quarter reduction lane (t + 8 q) holds pair slot 2 (q & 1) + (q >> 1) of tile t;
// tile_src(l) = the lane holding pair4(l) (k_sweep4's add order), tabulated offline
__device__ __forceinline__ int tile_src(int l) {
  constexpr int S[28] = {21, 3, 20, 18, 2, 0, 30, 29, 24, 25, 4, 12, 10, 9,
                         26, 13, 5, 28, 7, 1, 31, 8, 27, 19, 16, 6, 17, 11};
  int r = 0;
#pragma unroll
  for (int k = 0; k < 28; ++k)
    if (l == k) r = S[k];
  return r;
}

// Coupling record of one node at one GP from its core (C4 layout): W' grad N, Dt' grad N, E
// (Eqs. 11b-d integrands), and the node sums ns = {Fu[3], Fe, U[3], V} (Eqs. 11e-f, the
// row-sum diagonal).  Same arithmetic as gpExpand.
__device__ __forceinline__ void expandx(const double* __restrict__ co, const double* __restrict__ sh,
                                        double* __restrict__ r, double (&ns)[8]) {
  const double2* c2 = reinterpret_cast<const double2*>(co);
  double c[C4::N];
#pragma unroll
  for (int k = 0; k < C4::N / 2; ++k) {
    // J^-1 (units 0-4), W', Dt', Sigma' (8-16), hN .. FV (18-23); S, lam*, Ams, Ass unused
    if (k == 5 || k == 6 || k == 7 || k == 17) continue;
    const double2 v = c2[k];
    c[2 * k] = v.x;
    c[2 * k + 1] = v.y;
  }
  const double2 sh0 = reinterpret_cast<const double2*>(sh)[0];
  const double2 sh1 = reinterpret_cast<const double2*>(sh)[1];
  const double dxi[3] = {sh0.x, sh0.y, sh1.x};
  const double Na = sh1.y;
  double gn[3], WgN[3], DgN[3], fu[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double s = c[C4::JI + i] * dxi[0];
    s = fma(c[C4::JI + 3 + i], dxi[1], s);
    s = fma(c[C4::JI + 6 + i], dxi[2], s);
    gn[i] = s;
  }
  symv<3>(c + C4::WT, gn, WgN);
  symv<3>(c + C4::DT, gn, DgN);
  symv<3>(c + C4::SG, gn, fu);
  double gvd = 0.0, fvd = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    gvd = fma(c[C4::GV + i], gn[i], gvd);
    fvd = fma(c[C4::FV + i], gn[i], fvd);
  }
  const double Ea = fma(c[C4::HN], Na, gvd);
  const double fe = fma(c[C4::FE0], Na, fvd);
  double2* r2 = reinterpret_cast<double2*>(r);
  r2[0] = make_double2(WgN[0], WgN[1]);
  r2[1] = make_double2(WgN[2], DgN[0]);
  r2[2] = make_double2(DgN[1], DgN[2]);
  r2[3] = make_double2(Ea, 0.0);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    ns[i] += fu[i];
    ns[4 + i] += WgN[i];
  }
  ns[3] += fe;
  ns[7] += Ea;
}

__global__ void __launch_bounds__(H8::T, 1)
k_hex8(DevMat m, SweepGeom G, const double* __restrict__ coords,
         const double* __restrict__ dofs, const double* __restrict__ kappa,
         const int64_t* __restrict__ base, double* __restrict__ val, double* __restrict__ Rv) {
  constexpr int NGP = 8, NEN = 8;
  extern __shared__ double sm[];
  double* shtab = sm;                              // [NGP][NEN][6] = (dN/dxi, N, pad)
  double* cores = shtab + H8::SHT;                 // [3][E][CEL]
  double* recs = cores + H8::NCSLOT * H8::CSLOT;   // [NC][RWARP]
  double* acc = recs + H8::NC * H8::RWARP;         // [NCOLS][COL]
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  int bid = blockIdx.x;
  const int tx = bid % G.tiles_x;
  bid /= G.tiles_x;
  const int ty = bid % G.tiles_y;
  const int ch = bid / G.tiles_y;
  const int64_t x0 = int64_t(tx) * H8::TX, x1 = min(x0 + H8::TX, G.nx + 1);
  const int64_t y0 = int64_t(ty) * H8::TY, y1 = min(y0 + H8::TY, G.nyN);
  const int64_t z0 = G.lay_own_b + int64_t(ch) * G.chunk_len;
  const int64_t z1 = min(z0 + G.chunk_len, G.lay_own_e);
  if (z0 >= z1) return;
  const int64_t nxN = G.nx + 1;
  auto node_id = [&](int64_t x, int64_t y, int64_t z) { return x + nxN * (y + G.nyN * z); };

  const int64_t s_first = max(z0 - 1, int64_t(0));
  const int64_t s_last = min(z1, G.nl) - 1;
  const int ilo = int(max(x0 - 1, int64_t(0))), ihi = int(min(x1, G.nx));
  const int jlo = int(max(y0 - 1, int64_t(0))), jhi = int(min(y1, G.nyE));
  const int cols_x = int(x1 - x0), cols = cols_x * int(y1 - y0);
  const int ix0 = int(x0), iy0 = int(y0), ix1 = int(x1), iy1 = int(y1);

  for (int k = tid; k < NGP * NEN; k += H8::T) {
    const int g = k >> 3, a = k & 7;
#pragma unroll
    for (int j = 0; j < 3; ++j) shtab[k * 6 + j] = shape_dxi<3>(a, g, j);
    shtab[k * 6 + 3] = shapeN<3>(a, g);
  }
  for (int k = tid; k < H8::NCOLS * H8::COL; k += H8::T) acc[k] = 0.0;
  __shared__ int64_t sbase[3][H8::NCOLS];   // CSR offsets of node layers (by z % 3)
  for (int q = tid; q < 2 * cols; q += H8::T) {
    const int cc = q % cols;
    const int64_t zq = s_first + q / cols;
    const int cy = cc / cols_x;
    if (zq >= z0 && zq < z1)
      sbase[zq % 3][cc] = base[node_id(ix0 + (cc - cy * cols_x), iy0 + cy, zq) - G.own_node_b];
  }
  __syncthreads();

  // batch schedule, identical in every role: layer s, colour c (parity of i, j), batches of
  // E elements of that colour (which share no node)
  auto schedule = [&](auto&& body, auto&& end_of_layer) {
    for (int64_t s = s_first; s <= s_last; ++s) {
      for (int c = 0; c < H8::NCOL; ++c) {
        const int ifst = ilo + ((ilo & 1) != (c & 1) ? 1 : 0);
        const int ni = ifst < ihi ? (ihi - ifst + 1) / 2 : 0;
        const int jfst = jlo + ((jlo & 1) != (c >> 1) ? 1 : 0);
        const int nj = jfst < jhi ? (jhi - jfst + 1) / 2 : 0;
        const int nc = ni * nj;
        body(s, c, 0, ifst, ni, jfst, nc);   // nc <= E: one batch per colour
      }
      end_of_layer(s);
    }
  };

  constexpr int NPC_T = 64, NC_T = 32 * H8::NC;
  static_assert(((H8::TX + 2) / 2) * ((H8::TY + 2) / 2) <= H8::E, "one batch per colour");
  constexpr int FL_T = H8::T;   // layer adds done (C -> PC) / PC flush part done (PC -> C)

  auto col_of = [&](int x, int y) { return acc + ((x - ix0) + cols_x * (y - iy0)) * H8::COL; };
  int lane_csr = 0;   // CSR chunk of smem chunk position `lane` (lanes 0..17) of a plane row:
#pragma unroll        // contiguous (conflict-free) smem reads, permuted 16-byte global stores
  for (int k = 0; k < 18; ++k)
    if (pos4(k >> 1, k & 1) == lane) lane_csr = k;
  // ---- flush helpers (one warp per column) ----
  // copy plane P ([row 4][9 slots][4]) of node (x, y, z) to its compacted CSR position
  auto write_plane = [&](int x, int y, int64_t z, int dz, const double* P, bool inner) {
    const int zlo = z > 0 ? -1 : 0, zhi = z < G.nl ? 1 : 0;
    if (inner) {
      const int W2 = 18 * (zhi - zlo + 1);   // row width in double2
      double2* out = reinterpret_cast<double2*>(val + sbase[z % 3][(x - ix0) + cols_x * (y - iy0)]) + (dz - zlo) * 18;
      const double2* src = reinterpret_cast<const double2*>(P);
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (lane < 18) __stcs(out + r * W2 + lane_csr, src[r * 18 + lane]);
      return;
    }
    const int xlo = x > 0 ? -1 : 0, xhi = x < G.nx ? 1 : 0;
    const int ylo = y > 0 ? -1 : 0, yhi = y < G.nyN - 1 ? 1 : 0;
    const int wx = xhi - xlo + 1, wy = yhi - ylo + 1, wz = zhi - zlo + 1;
    const int W = 4 * wx * wy * wz;
    double* out = val + sbase[z % 3][(x - ix0) + cols_x * (y - iy0)] + (dz - zlo) * (4 * wx * wy);
    for (int it = lane; it < 36; it += 32) {
      const int i = it / 9, sl = it - 9 * i;
      const int dy = sl / 3 - 1, dx = sl - 3 * (dy + 1) - 1;
      if (dx < xlo || dx > xhi || dy < ylo || dy > yhi) continue;
      const double2* src = reinterpret_cast<const double2*>(P + i * 36);
      double2* dst = reinterpret_cast<double2*>(out + i * W + 4 * ((dy - ylo) * wx + (dx - xlo)));
      int q0 = 0, q1 = 0;
#pragma unroll
      for (int k = 0; k < 9; ++k)
        if (sl == k) { q0 = pos4(k, 0); q1 = pos4(k, 1); }
      __stcs(dst, src[q0]);
      __stcs(dst + 1, src[q1]);
    }
  };
  // lanes 0..15: entry (i, j) = (lane / 4, lane % 4) of the 4x4 blocks, summed over slots
  auto plane_sum = [&](const double* P, bool skip_self) {   // pairwise: short add chains
    const double* p = P + (lane >> 2) * 36;
    const int j = lane & 3;
    double v[9];
#pragma unroll
    for (int sl = 0; sl < 9; ++sl) v[sl] = p[soff4(sl, j)];
    if (skip_self) v[4] = 0.0;
    return ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + ((v[6] + v[7]) + v[8]));
  };
  // finish node (x, y, z): diagonal block = -sum(plane -1) [kept in the self slot]
  // - sum(plane 0 off-diagonal) - sum(plane +1) + (U, V); then plane 0, +1 and R go out
  auto finish_node = [&](int x, int y, int64_t z, double* colp, bool has_up, bool inner) {
    double* Zp = colp + ((z & 1) ? H8::Z1 : H8::Z0);
    const double* ns = colp + H8::NS + (z & 1) * 8;
    if (lane < 16) {
      const int i = lane >> 2, j = lane & 3;
      double* self = Zp + i * 36 + soff4(4, j);
      double d = *self - plane_sum(Zp, true);
      if (has_up) d -= plane_sum(colp + H8::UP, false);
      if (j == 3) d += (i < 3) ? ns[4 + i] : ns[7];
      *self = d;
    }
    __syncwarp();
    write_plane(x, y, z, 0, Zp, inner);
    if (has_up) write_plane(x, y, z, 1, colp + H8::UP, inner);
    if (lane < 4) __stcs(Rv + (node_id(x, y, z) - G.own_node_b) * 4 + lane, ns[lane]);
  };

  // flush of element layer s for one node column cc: plane -1 of node layer s+1 out (its minus
  // row sums parked in the self slot of that node's plane 0), node layer s finished (and s+1
  // if s is the chunk's last layer), planes and node sums reset
  auto flush_col = [&](int64_t s, int cc) {
    const bool own_s = s >= z0 && s < z1, own_s1 = s + 1 >= z0 && s + 1 < z1;
    const bool top = s == s_last && own_s1;   // node layer s+1 has no element layer above
    const int cy = cc / cols_x;
    const int x = ix0 + (cc - cy * cols_x), y = iy0 + cy;
    const bool inner = x > 0 && x < G.nx && y > 0 && y < G.nyN - 1;
    double* colp = col_of(x, y);
    if (own_s1) {
      if (lane < 16)
        colp[(((s + 1) & 1) ? H8::Z1 : H8::Z0) + (lane >> 2) * 36 + soff4(4, lane & 3)] =
            -plane_sum(colp + H8::DN, false);
      write_plane(x, y, s + 1, -1, colp + H8::DN, inner);
    }
    __syncwarp();
    if (own_s) finish_node(x, y, s, colp, s < G.nl, inner);
    if (top) finish_node(x, y, s + 1, colp, false, inner);
    __syncwarp();
    double2* z2 = reinterpret_cast<double2*>(colp + ((s & 1) ? H8::Z1 : H8::Z0));
    double2* ud = reinterpret_cast<double2*>(colp + H8::UP);
    double2* dn2 = reinterpret_cast<double2*>(colp + H8::DN);
    const double2 zero = make_double2(0.0, 0.0);
    for (int k2 = lane; k2 < H8::PLD / 2; k2 += 32) z2[k2] = zero;
    for (int k2 = lane; k2 < H8::PLD / 2; k2 += 32) ud[k2] = zero;
    for (int k2 = lane; k2 < H8::PLD / 2; k2 += 32) dn2[k2] = zero;
    if (lane < 4) reinterpret_cast<double2*>(colp + H8::NS + (s & 1) * 8)[lane] = zero;
  };
  // the layer flush is split: the C warps take columns 0 .. NC-1 right after the layer's adds,
  // the PC warps (idle ~70 %) the rest while the C warps compute the next layer's first batch
  constexpr int NCC = H8::NC;

  if (warp < H8::NPC) {
    // ---------------------------- PC: Gauss-point cores ----------------------------
    setmaxnreg_dec<H8::REG_PC>();
    const int pair = warp >> 1;                       // batches t with t % 2 == pair
    const int lid = (warp & 1) * 32 + lane;
    const int el = lid >> 3, g = lid & 7;
    int t = 0;
    PT_DECL
    schedule(
        [&](int64_t s, int c, int b0, int ifst, int ni, int jfst, int nc) {
          if ((t & 1) == pair) {
            const int slot = pair;   // each PC pair owns one core slot (fixed producer)
            PT_MARK(12, tid == 0);
            if (t >= 2) bsync(H8::B_CE + slot, NPC_T + NC_T);
            PT_MARK(10, tid == 0);
            const int k = b0 + el;
            if (k < nc) {
              const int i = ifst + 2 * (k % ni), j = jfst + 2 * (k / ni);
              const int64_t n0 = node_id(i, j, s);
              auto nid = [&](int a) {
                int ox, oy, oz;
                node_off<3>(a, ox, oy, oz);
                return n0 + ox + nxN * (oy + G.nyN * oz);
              };
              auto X = [&](int a, int q) { return __ldg(coords + nid(a) * 3 + q); };
              auto U = [&](int a, int q) { return __ldg(dofs + nid(a) * 4 + q); };
              const int64_t e = i + G.nx * (j + G.nyE * s);
              double core[Core<3>::STRIDE];
              const int64_t q = e * NGP + g;   // defect fields if set
              gpCoreSK<3>(m, X, U, __ldg(kappa + q), G.k0g ? __ldg(G.k0g + q) : m.kappa0,
                          G.alg ? __ldg(G.alg + q) : m.alpha,
                          [&](int a, int j) { return shape_dxi<3>(a, g, j); },
                          [&](int a) { return shapeN<3>(a, g); }, core);
              double2* dst = reinterpret_cast<double2*>(cores + slot * H8::CSLOT + el * H8::CEL + g * H8::CSP);
#pragma unroll
              for (int k2 = 0; k2 < 4; ++k2) dst[k2] = make_double2(core[2 * k2], core[2 * k2 + 1]);
              dst[4] = make_double2(core[8], 0.0);
#pragma unroll
              for (int k2 = 5; k2 < 23; ++k2) dst[k2] = make_double2(core[2 * k2 - 1], core[2 * k2]);
              dst[23] = make_double2(core[45], 0.0);
            }
            PT_MARK(11, tid == 0);
            barrive(H8::B_CF + slot, NPC_T + NC_T);
            if (c == pair && s > s_first) {   // PC part of the flush of layer s - 1
              bsync(H8::B_AD, FL_T);
              PT_MARK(15, tid == 0);
              for (int cc = NCC + warp; cc < cols; cc += H8::NPC) flush_col(s - 1, cc);
              barrive(H8::B_FL, FL_T);
              // CSR offsets of node layer s+1 for flush(s) (slot (s+1) % 3 was last read by
              // flush(s-2), done); issued after the hand-off so the load latency stays off the
              // C warps' path; visible to them through B_AD / B_FL of the next layer
              if (pair == 0 && s + 1 >= z0 && s + 1 < z1)
                for (int cc = (warp & 1) * 32 + lane; cc < cols; cc += NPC_T) {
                  const int cy = cc / cols_x;
                  sbase[(s + 1) % 3][cc] = base[node_id(ix0 + (cc - cy * cols_x), iy0 + cy, s + 1) - G.own_node_b];
                }
              PT_MARK(14, tid == 0);
            }
          }
          ++t;
        },
        [](int64_t) {});
    bsync(H8::B_AD, FL_T);   // the last layer
    for (int cc = NCC + warp; cc < cols; cc += H8::NPC) flush_col(s_last, cc);
    // drain: the core-empty arrival of this pair's last batch
    for (int tt = max(t - 2, 0); tt < t; ++tt)
      if ((tt & 1) == pair) bsync(H8::B_CE + pair, NPC_T + NC_T);
    return;
  }

  // ------------------------- C: one warp per element of the batch -------------------------
  setmaxnreg_inc<H8::REG_C>();
  const int cw = warp - H8::NPC;                     // element slot of this warp
  const int ct = tid - 32 * H8::NPC;
  // expansion lane: node xa, Gauss point 4 * round + xg
  const int xa = lane & 7, xg = lane >> 3;
  int xox, xoy, xoz;
  node_off<3>(xa, xox, xoy, xoz);
  // pair lane
  const bool plane_lane = lane < H8::NOFF;
  int pa = 0, pb = 1;
  if (plane_lane) {
#pragma unroll
    for (int k = 0; k < H8::NOFF; ++k)
      if (lane == k) {
        pa = pair4(k) / 10;
        pb = pair4(k) % 10;
      }
  }
  int oax, oay, oaz, obx, oby, obz;
  node_off<3>(pa, oax, oay, oaz);
  node_off<3>(pb, obx, oby, obz);
  const int psAB = plane_slot<3>(obx - oax, oby - oay), psBA = plane_slot<3>(oax - obx, oay - oby);
  const int dzAB = obz - oaz;
  int qAB0 = 0, qAB1 = 0, qBA0 = 0, qBA1 = 0;   // pos4 of this lane's two slots
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    if (psAB == k) { qAB0 = pos4(k, 0); qAB1 = pos4(k, 1); }
    if (psBA == k) { qBA0 = pos4(k, 0); qBA1 = pos4(k, 1); }
  }
  double* myrec = recs + cw * H8::RWARP;
  // tile lanes: tile tt = lane & 7 over the GP quarter tq = lane >> 3 (GPs 2 tq, 2 tq + 1)
  const int tt = lane & 7, tq = lane >> 3;
  int A1, A2, B1, B2;
  tile_nodes(tt, A1, A2, B1, B2);
  const bool tfull = tt < 6;
  // dN_a/dxi at the lane's GPs g = 2 tq + gg: the y and z Gauss signs are lane constants, only x
  // follows gg, and the two 1D factors of an axis sum to 1 (P + M = 1).  Per node a:
  //   dN/dxi = 0.5 r_x f_y f_z,  dN/deta = (0.5 r_y f_z) f_x,  dN/dzeta = (0.5 r_z f_y) f_x,
  //   f_x = fx0 at gg = 0 and 1 - fx0 at gg = 1.
  double dnx[4], cy[4], cz[4], fx0[4];
  {
    const int tn[4] = {A1, A2, B1, B2};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int ox, oy, oz;
      node_off<3>(tn[k], ox, oy, oz);
      const double fy = (oy == (tq & 1)) ? LGDM_P : LGDM_M;
      const double fz = (oz == (tq >> 1)) ? LGDM_P : LGDM_M;
      fx0[k] = ox == 0 ? LGDM_P : LGDM_M;   // gg = 0: Gauss x sign -1
      dnx[k] = (ox ? 0.5 : -0.5) * fy * fz;
      cy[k] = (oy ? 0.5 : -0.5) * fz;
      cz[k] = (oz ? 0.5 : -0.5) * fy;
    }
  }
  const int src_lane = plane_lane ? tile_src(lane) : lane;   // holder of pair4(lane) after the reduction
  auto plane_of = [&](double* colp, int zpar, bool zs, int dz) -> double* {
    if (dz == 0) return colp + (zpar ? H8::Z1 : H8::Z0);
    return colp + (zs ? H8::UP : H8::DN);
  };

  int prev_c = -1, t = 0;
  [[maybe_unused]] const bool ptc = ct == 0;   // phase-timing build (PT_MARK)
  PT_DECL
  schedule(
      [&](int64_t s, int c, int b0, int ifst, int ni, int jfst, int nc) {
        const int k = b0 + cw;
        const bool live = k < nc;   // warp-uniform
        const int cslot = t & 1;
        ++t;
        const bool wait_flush = prev_c < 0 && s > s_first;   // PC part of flush(s - 1)
        PT_MARK(9, ptc);
        bsync(H8::B_CF + cslot, NPC_T + NC_T);
        PT_MARK(0, ptc);
        if (!live) {
          barrive(H8::B_CE + cslot, NPC_T + NC_T);
          if (wait_flush) bsync(H8::B_FL, FL_T);
          if (c != prev_c) bsync(H8::B_C, NC_T);
          prev_c = c;
          return;
        }
        const int i = ifst + 2 * (k % ni), j = jfst + 2 * (k / ni);
        const int sz = int(s - z0);   // layer of node z relative to the chunk
        const double* ce = cores + cslot * H8::CSLOT + cw * H8::CEL;
        // ---- Kuu tiles straight from the core ring: 4 pairs over 2 GPs per lane ----
        double K[4][10];
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 10; ++q) K[p][q] = 0.0;
#pragma unroll
        for (int gg = 0; gg < 2; ++gg) {
          const int g = 2 * tq + gg;
          const double2* tc = reinterpret_cast<const double2*>(ce + g * H8::CSP);
          double Ji[9], S[6], lam, Ams, Ass, mu, ghc;
          {
            double2 v;
            v = tc[0]; Ji[0] = v.x; Ji[1] = v.y;
            v = tc[1]; Ji[2] = v.x; Ji[3] = v.y;
            v = tc[2]; Ji[4] = v.x; Ji[5] = v.y;
            v = tc[3]; Ji[6] = v.x; Ji[7] = v.y;
            Ji[8] = tc[4].x;
            v = tc[5]; S[0] = v.x; S[1] = v.y;
            v = tc[6]; S[2] = v.x; S[3] = v.y;
            v = tc[7]; S[4] = v.x; S[5] = v.y;
            v = tc[17]; lam = v.x; Ams = v.y;     // C4::LAM = 34, AMS = 35
            Ass = tc[18].x;                       // C4::ASS = 36
            v = tc[19]; mu = v.y;                 // C4::MU = 39
            ghc = tc[20].x;                       // C4::GHC = 40
          }
          auto grad = [&](int k, double (&gn)[3], double (&sn)[3]) {
            const double fx = gg ? 1.0 - fx0[k] : fx0[k];
            const double dn[3] = {dnx[k], cy[k] * fx, cz[k] * fx};
#pragma unroll
            for (int ii = 0; ii < 3; ++ii) {
              double sv = Ji[ii] * dn[0];
              sv = fma(Ji[3 + ii], dn[1], sv);
              sv = fma(Ji[6 + ii], dn[2], sv);
              gn[ii] = sv;
            }
            symv<3>(S, gn, sn);
          };
          double gA[2][3], sA[2][3], gB[2][3], t1[2][3], t2[2][3];
          grad(0, gA[0], sA[0]);
          grad(1, gA[1], sA[1]);
#pragma unroll
          for (int bb = 0; bb < 2; ++bb) {
            double sB[3];
            grad(2 + bb, gB[bb], sB);
#pragma unroll
            for (int ii = 0; ii < 3; ++ii) {
              t1[bb][ii] = fma(lam, gB[bb][ii], Ams * sB[ii]);
              t2[bb][ii] = fma(Ams, gB[bb][ii], Ass * sB[ii]);
            }
          }
#pragma unroll
          for (int p = 0; p < 4; ++p) {   // p0 (A1,B1) p1 (A1,B2) p2 (A2,B1) p3 (A2,B2)
            const int aa = p >> 1, bb = p & 1;
            if (!(tfull || aa == bb)) continue;
            double dot = gA[aa][0] * gB[bb][0];
            dot = fma(gA[aa][1], gB[bb][1], dot);
            dot = fma(gA[aa][2], gB[bb][2], dot);
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              const double ub = mu * gB[bb][r];
#pragma unroll
              for (int u = 0; u < 3; ++u) {
                double x = K[p][3 * r + u];
                x = fma(gA[aa][r], t1[bb][u], x);
                x = fma(sA[aa][r], t2[bb][u], x);
                x = fma(gA[aa][u], ub, x);
                K[p][3 * r + u] = x;
              }
              K[p][4 * r] = fma(mu, dot, K[p][4 * r]);
            }
            K[p][9] = fma(ghc, dot, K[p][9]);
          }
        }
        // ---- coupling records + moments (w, d, E) and node sums: lanes = node x 4 GPs ----
        double M1[8], M2[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) M1[q] = M2[q] = 0.0;
        const int mt1 = lane, mt2 = lane + 32;
        const int mn1 = mt1 / 7, mc1 = mt1 - 7 * mn1;
        const int mn2 = mt2 < 56 ? mt2 / 7 : 0, mc2 = mt2 < 56 ? mt2 - 7 * (mt2 / 7) : 0;
        const double* mrec1 = myrec + mn1 * H8::RS + mc1;
        const double* mrec2 = myrec + mn2 * H8::RS + mc2;
        double ns[8];
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) ns[k2] = 0.0;
        auto moments = [&](auto rc) {
          constexpr int R = decltype(rc)::value;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double v1 = mrec1[k * H8::RGP];
            const double v2 = mt2 < 56 ? mrec2[k * H8::RGP] : 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const double nq = shapeN<3>(q, 4 * R + k);
              M1[q] = fma(nq, v1, M1[q]);
              M2[q] = fma(nq, v2, M2[q]);
            }
          }
        };
#pragma unroll 1
        for (int rnd = 0; rnd < 2; ++rnd) {
          {
            const int g = 4 * rnd + xg;
            expandx(ce + g * H8::CSP, shtab + (g * NEN + xa) * 6, myrec + xg * H8::RGP + xa * H8::RS, ns);
          }
          if (rnd == 1) barrive(H8::B_CE + cslot, NPC_T + NC_T);   // core slot no longer read
          __syncwarp();
          PT_MARK(1, ptc);
          if (rnd == 0) moments(std::integral_constant<int, 0>{});
          else moments(std::integral_constant<int, 1>{});
          __syncwarp();
          PT_MARK(2, ptc);
        }
        // ---- GP-quarter reduction of the tiles in a fixed order ((q0 + q1) + (q2 + q3)), then
        // each pair lane fetches its pair (pair4 order) from the lane holding it ----
        double Kuu[3][3], Gd;
        {
          double H[2][10], Fq[10];
          const bool odd = tq & 1, hi2 = tq >> 1;
#pragma unroll
          for (int q = 0; q < 10; ++q) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const double snd = odd ? K[h][q] : K[2 + h][q];
              const double rcv = __shfl_xor_sync(0xffffffffu, snd, 8);
              H[h][q] = odd ? rcv + K[2 + h][q] : K[h][q] + rcv;
            }
          }
#pragma unroll
          for (int q = 0; q < 10; ++q) {
            const double snd = hi2 ? H[0][q] : H[1][q];
            const double rcv = __shfl_xor_sync(0xffffffffu, snd, 16);
            Fq[q] = hi2 ? rcv + H[1][q] : H[0][q] + rcv;
          }
#pragma unroll
          for (int q = 0; q < 9; ++q) Kuu[q / 3][q % 3] = __shfl_sync(0xffffffffu, Fq[q], src_lane);
          Gd = __shfl_sync(0xffffffffu, Fq[9], src_lane);
        }
        // moments out (the record buffer is free now), then each pair lane picks its 14
        double* mom = myrec;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          mom[mom_idx(mn1, q, mc1)] = M1[q];
          if (mt2 < 56) mom[mom_idx(mn2, q, mc2)] = M2[q];
        }
        __syncwarp();
        Pair4 P;
        {
          const double* mab = mom + mom_idx(pa, pb, 0);   // M[a][b][.]
          const double* mba = mom + mom_idx(pb, pa, 0);
#pragma unroll
          for (int r = 0; r < 3; ++r) {
#pragma unroll
            for (int u = 0; u < 3; ++u) P.Kuu[r][u] = Kuu[r][u];
            P.Kue_ab[r] = mab[r];
            P.Kue_ba[r] = mba[r];
            P.Keu_ab[r] = mba[3 + r];
            P.Keu_ba[r] = mab[3 + r];
          }
          P.Kee_ab = mab[6] + Gd;
          P.Kee_ba = mba[6] + Gd;
        }
        // node sums: reduce the four Gauss-point lanes of each node (lanes xa + 8 xg)
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) {
          ns[k2] += __shfl_xor_sync(0xffffffffu, ns[k2], 8);
          ns[k2] += __shfl_xor_sync(0xffffffffu, ns[k2], 16);
        }
        PT_MARK(3, ptc);
        // batches of one colour share no node; a new colour waits for the previous adds
        if (wait_flush) bsync(H8::B_FL, FL_T);
        if (c != prev_c) bsync(H8::B_C, NC_T);
        prev_c = c;
        PT_MARK(4, ptc);
        const int zpar_s = int(s & 1);
        if (xg == 0) {
          const int nx_ = i + xox, ny_ = j + xoy;
          const int nz = sz + xoz;   // relative to z0
          if (nx_ >= ix0 && nx_ < ix1 && ny_ >= iy0 && ny_ < iy1 && nz >= 0 && s + xoz < z1) {
            double2* n2 = reinterpret_cast<double2*>(col_of(nx_, ny_) + H8::NS + ((zpar_s ^ xoz) & 1) * 8);
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) {
              double2 v = n2[k2];
              v.x += ns[2 * k2];
              v.y += ns[2 * k2 + 1];
              n2[k2] = v;
            }
          }
        }
        if (plane_lane) {
          const int ax = i + oax, ay = j + oay, azr = sz + oaz;
          const int bx = i + obx, by = j + oby, bzr = sz + obz;
          const bool own_a = ax >= ix0 && ax < ix1 && ay >= iy0 && ay < iy1 && azr >= 0 && s + oaz < z1;
          const bool own_b = bx >= ix0 && bx < ix1 && by >= iy0 && by < iy1 && bzr >= 0 && s + obz < z1;
          if (own_a) {
            double* Pp = plane_of(col_of(ax, ay), (zpar_s ^ oaz) & 1, oaz == 0, dzAB);
            // all 8 loads of the block first: the compiler cannot prove the rows distinct and
            // would otherwise serialise 8 read-modify-write round trips
            double2 lo[4], hi[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const double2* q = reinterpret_cast<const double2*>(Pp + r * 36);
              lo[r] = q[qAB0];
              hi[r] = q[qAB1];
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              double2* q = reinterpret_cast<double2*>(Pp + r * 36);
              if (r < 3) {
                lo[r].x += P.Kuu[r][0]; lo[r].y += P.Kuu[r][1]; hi[r].x += P.Kuu[r][2]; hi[r].y += P.Kue_ab[r];
              } else {
                lo[r].x += P.Keu_ab[0]; lo[r].y += P.Keu_ab[1]; hi[r].x += P.Keu_ab[2]; hi[r].y += P.Kee_ab;
              }
              q[qAB0] = lo[r];
              q[qAB1] = hi[r];
            }
          }
          if (own_b) {
            double* Pp = plane_of(col_of(bx, by), (zpar_s ^ obz) & 1, obz == 0, -dzAB);
            double2 lo[4], hi[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const double2* q = reinterpret_cast<const double2*>(Pp + r * 36);
              lo[r] = q[qBA0];
              hi[r] = q[qBA1];
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              double2* q = reinterpret_cast<double2*>(Pp + r * 36);
              if (r < 3) {
                lo[r].x += P.Kuu[0][r]; lo[r].y += P.Kuu[1][r]; hi[r].x += P.Kuu[2][r]; hi[r].y += P.Kue_ba[r];
              } else {
                lo[r].x += P.Keu_ba[0]; lo[r].y += P.Keu_ba[1]; hi[r].x += P.Keu_ba[2]; hi[r].y += P.Kee_ba;
              }
              q[qBA0] = lo[r];
              q[qBA1] = hi[r];
            }
          }
        }
      },
      [&](int64_t s) {
        PT_MARK(5, ptc);
        bsync(H8::B_C, NC_T);      // all adds of layer s are in
        barrive(H8::B_AD, FL_T);   // the PC warps may flush their columns
        PT_MARK(6, ptc);
        prev_c = -1;
        for (int cc = cw; cc < NCC && cc < cols; cc += H8::NC) flush_col(s, cc);
        PT_MARK(7, ptc);
        bsync(H8::B_C, NC_T);
        PT_MARK(8, ptc);
      });
}

}  // namespace lgdm

// lgdm_sweep4.cuh -- Hex8 hot kernel (k_sweep4): the structured-sweep K/R assembly, designed
// from the ncu profile of the round-1 sweep (profiles/r01).  Included by lgdm_sweep.cuh (needs
// SweepGeom, node_off, plane_slot, Core/gpCore).
//
// Contract (lgdm_sweep.cuh): one CTA owns TX x TY node columns and a chunk of node layers,
// sweeps the element layers touching them (ghost elements recomputed), writes exactly the
// CSR block-rows of its nodes; per-entry summation order = (element layer, colour), so K and
// R are bitwise independent of tiling and slabbing.  What changed:
//
//  1. Diagonal blocks by the partition-of-unity row-sum identity.  sum_b N_b = 1 gives
//     sum_b grad N_b = 0, so for every element and row node a (Eqs. 11a-d):
//        sum_b Kuu_ab = 0,  sum_b Keu_ab = 0,  sum_b Kue_ab = sum_g W' grad N_a = U_a,
//        sum_b Kee_ab = sum_g (h N_a + h c g' L grad N_a . grad ebar) dV = V_a,
//     and the same holds for a global row summed over its elements.  So only the 28
//     off-diagonal node pairs of an element are Gauss-summed (not 36); the diagonal 4x4
//     block of a row is [U_A, V_A] - sum of the row's 26 other blocks, formed at flush.
//     (Exact in exact arithmetic; the rounding difference is ~26 eps x row max.)
//  2. One C warp per element does the node expansions of its element itself (lane =
//     node x 4 Gauss points, two rounds) into a warp-private record buffer, then the 28
//     pair lanes read the Kuu fields of the records with 16-byte loads -- no inter-warp
//     hand-off per Gauss point, only one per batch (the core ring).
//  3. Coupling blocks by shape-function moments: Kue, Keu and the N E part of Kee of pair
//     (a, b) are sum_g N_b(g) x_a(g) with N_b(g) a constant (Eqs. 11b-d), so 56 (node,
//     component) lanes form M[n][m] = sum_g N_m(g) x_n(g) once per element and each pair
//     lane reads its 14 values; the pair Gauss sums keep only Kuu and sum ghc gA.gB.
//     Node sums (R = F, U, V) accumulate in registers and are reduced with shuffles.
//  6. Shared-memory layouts (pair lane order, plane-row chunk positions, plane / column
//     offsets, moment buffer, shape table) from quarter-warp bank-conflict searches
//     (tools/bank_search4.py).
//  4. The Appendix A core (exp, sqrt, divide: a long FP64 dependency chain) runs in two PC
//     warp pairs on alternate batches, one core slot each, 16-byte core stores/loads.
//  5. Flush: vectorised row copies, the -sum of plane -1 kept in the (never accumulated)
//     self slot of plane 0.
//
//   PC warps (element x GP)   gpCore -> core slots [2][E][NGP][CSP] (one per PC pair)
//   C  warps (one per element) expansions -> records [4 GP][8 node]; Kuu Gauss sums of the
//                              28 off-diagonal pairs; coupling moments; adds into the
//                              block-row planes; flush
#pragma once

#include <type_traits>

namespace lgdm {

struct S4 {
  static constexpr int TX = 3, TY = 7, E = 8, NCOL = 4;
  static constexpr int NGP = 8, NEN = 8, NDPN = 4, NOFF = 28;
  static constexpr int NPC = 4, NC = E;                          // warps per role
  static constexpr int T = 32 * (NPC + NC);
  // shape table [NGP][NEN][6] = (dN/dxi, N, pad) at the Gauss points
  static constexpr int SHT = NGP * NEN * 6;   // stride 3 x 16 B per (g, a): conflict-free reads
  // core ring [3][E][NGP][CSP]: core = Core<3> values with a pad after J^-1 so every field
  // group is 16-byte aligned (48 doubles); CSP = 50 (25 x 16 B) puts the 4 cores a C warp
  // reads at once into distinct bank groups
  static constexpr int CSP = 50, CEL = NGP * CSP + 2, CSLOT = E * CEL, NCSLOT = 2;
  // warp-private records [4 GP][8 node][RS] + (mu*, ghc) per GP
  static constexpr int RS = 22, RGP = NEN * RS + 2, RWARP = 4 * RGP;
  // accumulator column: planes Z0, Z1 (in-plane, by node-layer parity), UP, DN; each plane
  // [row 4][18 chunks of 16 B] = 144 doubles (chunk positions: pos4); NS[2][8].  Offsets in
  // 16-byte units: Z0 1, Z1 73, UP 149, DN 221 (= 1, 1, 5, 5 mod 8), NS 293, column 308
  // (= 4 mod 8): with the lane order of kPair4 and pos4 the quarter-warp bank model of the
  // block adds gives 40 wavefronts per (parity, h, AB/BA) sweep vs 67 for the round-1
  // layout (ideal 32; tools/bank_search4.py)
  static constexpr int PLD = 144, Z0 = 2, Z1 = 146, UP = 298, DN = 442, NS = 586,
                       COL = 616;
  static constexpr int NCOLS = TX * TY;
  static constexpr size_t SMEM = sizeof(double) * (size_t(SHT) + size_t(NCSLOT) * CSLOT +
                                                   size_t(NC) * RWARP + size_t(NCOLS) * COL);
  // named barriers: core full 1-2, core empty 3-4 (slot = PC pair), C warps 5
  static constexpr int B_CF = 1, B_CE = 3, B_C = 5, B_AD = 6, B_FL = 7;
};

// shifted Core<3> offsets in the ring (J^-1 at 0..8, pad, then the rest +1)
struct C4 {
  using Co = Core<3>;
  static constexpr int JI = 0, S = Co::S + 1, WT = Co::WT + 1, DT = Co::DT + 1, SG = Co::SG + 1,
                       LAM = Co::LAM + 1, AMS = Co::AMS + 1, ASS = Co::ASS + 1, HN = Co::HN + 1,
                       FE0 = Co::FE0 + 1, MU = Co::MU + 1, GHC = Co::GHC + 1, GV = Co::GV + 1,
                       FV = Co::FV + 1, N = 48;
  static_assert(Co::S == 9 && Co::USED == 46, "Core<3> layout");
};

// record of (element, GP, node), doubles:
//   [g0 g1][g2 s0][s1 s2][g2 t1_0][t1_1 t1_2][t2_0 t2_1][t2_2 E][w0 w1][w2 d0][d1 d2]
//   g = grad N, s = S grad N, t1 = lam* g + Ams s, t2 = Ams g + Ass s (Kuu), w = W' grad N
//   (Kue), d = Dt' grad N (Keu), E (Kee).  The pair lanes read only the Kuu fields (A side:
//   chunks 0-2, B side: chunks 0, 3-6); the coupling blocks come from moments (below).
// coupling moments: for node n and component c of (w0 w1 w2 d0 d1 d2 E),
//   M[n][m][c] = sum_g N_m(g) c_n(g), so that Kue_ab = M[a][b][w], Kue_ba = M[b][a][w],
//   Keu_ab = M[b][a][d], Keu_ba = M[a][b][d], Kee_ab = M[a][b][E] + sum_g ghc gA.gB
//   (Eqs. 11b-d with N_b evaluated at the Gauss points: constants)
__host__ __device__ constexpr int mom_off(int c) { return c < 6 ? 14 + c : 13; }   // record offset of component c
// moment M[n][m][c] at m * 63 + n * 7 + c: conflict-free stores of the (n, c) lanes and
// 42 (ideal 28) wavefronts for the pair lanes' 14 loads (bank search over linear layouts)
__host__ __device__ constexpr int mom_idx(int n, int m, int c) { return m * 63 + n * 7 + c; }
static_assert(mom_idx(7, 7, 6) < S4::RWARP, "moments fit the warp's record buffer");

__device__ __forceinline__ void bsync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void barrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Row layout inside a plane: 9 slots x 4 doubles = 18 double2 chunks per row.  The two chunks
// of slot sl are swizzled, chunk (sl, h) -> 2 sl + (h ^ bit2(sl)), so that the 16-byte adds of
// lanes targeting slots sl and sl+4 (same bank group otherwise) land in different bank groups.
__host__ __device__ constexpr int swz(int sl, int h) { return 2 * sl + (h ^ ((sl >> 2) & 1)); }
__host__ __device__ constexpr int soff(int sl, int j) { return 2 * swz(sl, j >> 1) + (j & 1); }

// k_sweep4 plane rows: chunk (slot sl, half h) of a row sits at 16-byte position pos4(sl, h)
// (a permutation of 0..17 found by tools/bank_search4.py); soff4 = double offset of entry j
// = {{2, 15}, {5, 14}, {0, 13}, {7, 4}, {6, 17}, {11, 8}, {16, 3}, {9, 10}, {12, 1}}[sl][h],
// packed 5 bits per slot so runtime (sl, h) never touch memory
__host__ __device__ constexpr int pos4(int sl, int h) {
  return int(((h ? 0x150d11235cfull : 0xc4c166380a2ull) >> (5 * sl)) & 31u);
}
__host__ __device__ constexpr int soff4(int sl, int j) { return 2 * pos4(sl, j >> 1) + (j & 1); }
// lane -> off-diagonal pair of the C warps' pair stage (same search)
__host__ __device__ constexpr int pair4(int lane) {
  constexpr int P[28] = {47, 24, 27, 7, 6, 2, 23, 57, 13, 15, 26, 36, 16, 14,
                         17, 56, 46, 37, 45, 4, 67, 12, 35, 25, 3, 1, 5, 34};
  return P[lane];
}

// off-diagonal pair p (0..27) -> (a, b), a < b
__device__ __forceinline__ void offdiag_ab(int p, int& a, int& b) {
  int aa = 0, rem = p;
  while (rem >= 7 - aa) {
    rem -= 7 - aa;
    ++aa;
  }
  a = aa;
  b = aa + 1 + rem;
}

// Expansion of one node at one GP from its core (C4 layout, 16-byte aligned): writes the
// record and accumulates the node sums ns = {Fu[3], Fe, U[3], V}.  Same arithmetic as
// gpExpand; sh = (dN/dxi, N) of the node at the GP from the shape table.
__device__ __forceinline__ void expand4(const double* __restrict__ co, const double* __restrict__ sh,
                                        double* __restrict__ r, double (&ns)[8]) {
  const double2* c2 = reinterpret_cast<const double2*>(co);
  double c[C4::N];
#pragma unroll
  for (int k = 0; k < C4::N / 2; ++k) {
    const double2 v = c2[k];
    c[2 * k] = v.x;
    c[2 * k + 1] = v.y;
  }
  const double2 sh0 = reinterpret_cast<const double2*>(sh)[0];
  const double2 sh1 = reinterpret_cast<const double2*>(sh)[1];
  const double dxi[3] = {sh0.x, sh0.y, sh1.x};
  const double Na = sh1.y;
  double gn[3], SgN[3], WgN[3], DgN[3], fu[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double s = c[C4::JI + i] * dxi[0];
    s = fma(c[C4::JI + 3 + i], dxi[1], s);
    s = fma(c[C4::JI + 6 + i], dxi[2], s);
    gn[i] = s;
  }
  symv<3>(c + C4::S, gn, SgN);
  symv<3>(c + C4::WT, gn, WgN);
  symv<3>(c + C4::DT, gn, DgN);
  symv<3>(c + C4::SG, gn, fu);
  const double lamS = c[C4::LAM], Ams = c[C4::AMS], Ass = c[C4::ASS];
  double t1[3], t2[3], gvd = 0.0, fvd = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    t1[i] = fma(lamS, gn[i], Ams * SgN[i]);
    t2[i] = fma(Ams, gn[i], Ass * SgN[i]);
    gvd = fma(c[C4::GV + i], gn[i], gvd);
    fvd = fma(c[C4::FV + i], gn[i], fvd);
  }
  const double Ea = fma(c[C4::HN], Na, gvd);
  const double fe = fma(c[C4::FE0], Na, fvd);
  double2* r2 = reinterpret_cast<double2*>(r);
  r2[0] = make_double2(gn[0], gn[1]);     // Kuu, row side (A): chunks 0-2
  r2[1] = make_double2(gn[2], SgN[0]);
  r2[2] = make_double2(SgN[1], SgN[2]);
  r2[3] = make_double2(gn[2], t1[0]);     // Kuu, column side (B): chunks 0, 3-6
  r2[4] = make_double2(t1[1], t1[2]);
  r2[5] = make_double2(t2[0], t2[1]);
  r2[6] = make_double2(t2[2], Ea);        // coupling moments read E, W' grad N, Dt' grad N
  r2[7] = make_double2(WgN[0], WgN[1]);
  r2[8] = make_double2(WgN[2], DgN[0]);
  r2[9] = make_double2(DgN[1], DgN[2]);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    ns[i] += fu[i];
    ns[4 + i] += WgN[i];
  }
  ns[3] += fe;
  ns[7] += Ea;
}

struct Pair4 {
  double Kuu[3][3], Kue_ab[3], Kue_ba[3], Keu_ab[3], Keu_ba[3], Kee_ab, Kee_ba;
};

__global__ void __launch_bounds__(S4::T, 1)
k_sweep4(DevMat m, SweepGeom G, const double* __restrict__ coords,
         const double* __restrict__ dofs, const double* __restrict__ kappa,
         const int64_t* __restrict__ base, double* __restrict__ val, double* __restrict__ Rv) {
  constexpr int NGP = 8, NEN = 8;
  extern __shared__ double sm[];
  double* shtab = sm;                              // [NGP][NEN][6] = (dN/dxi, N, pad)
  double* cores = shtab + S4::SHT;                 // [3][E][CEL]
  double* recs = cores + S4::NCSLOT * S4::CSLOT;   // [NC][RWARP]
  double* acc = recs + S4::NC * S4::RWARP;         // [NCOLS][COL]
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  int bid = blockIdx.x;
  const int tx = bid % G.tiles_x;
  bid /= G.tiles_x;
  const int ty = bid % G.tiles_y;
  const int ch = bid / G.tiles_y;
  const int64_t x0 = int64_t(tx) * S4::TX, x1 = min(x0 + S4::TX, G.nx + 1);
  const int64_t y0 = int64_t(ty) * S4::TY, y1 = min(y0 + S4::TY, G.nyN);
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

  for (int k = tid; k < NGP * NEN; k += S4::T) {
    const int g = k >> 3, a = k & 7;
#pragma unroll
    for (int j = 0; j < 3; ++j) shtab[k * 6 + j] = shape_dxi<3>(a, g, j);
    shtab[k * 6 + 3] = shapeN<3>(a, g);
  }
  for (int k = tid; k < S4::NCOLS * S4::COL; k += S4::T) acc[k] = 0.0;
  __shared__ int64_t sbase[3][S4::NCOLS];   // CSR offsets of node layers (by z % 3)
  for (int q = tid; q < 2 * cols; q += S4::T) {
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
      for (int c = 0; c < S4::NCOL; ++c) {
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

  constexpr int NPC_T = 64, NC_T = 32 * S4::NC;
  static_assert(((S4::TX + 2) / 2) * ((S4::TY + 2) / 2) <= S4::E, "one batch per colour");
  constexpr int FL_T = S4::T;   // layer adds done (C -> PC) / PC flush part done (PC -> C)

  auto col_of = [&](int x, int y) { return acc + ((x - ix0) + cols_x * (y - iy0)) * S4::COL; };
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
    double* Zp = colp + ((z & 1) ? S4::Z1 : S4::Z0);
    const double* ns = colp + S4::NS + (z & 1) * 8;
    if (lane < 16) {
      const int i = lane >> 2, j = lane & 3;
      double* self = Zp + i * 36 + soff4(4, j);
      double d = *self - plane_sum(Zp, true);
      if (has_up) d -= plane_sum(colp + S4::UP, false);
      if (j == 3) d += (i < 3) ? ns[4 + i] : ns[7];
      *self = d;
    }
    __syncwarp();
    write_plane(x, y, z, 0, Zp, inner);
    if (has_up) write_plane(x, y, z, 1, colp + S4::UP, inner);
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
        colp[(((s + 1) & 1) ? S4::Z1 : S4::Z0) + (lane >> 2) * 36 + soff4(4, lane & 3)] =
            -plane_sum(colp + S4::DN, false);
      write_plane(x, y, s + 1, -1, colp + S4::DN, inner);
    }
    __syncwarp();
    if (own_s) finish_node(x, y, s, colp, s < G.nl, inner);
    if (top) finish_node(x, y, s + 1, colp, false, inner);
    __syncwarp();
    // the planes need no reset: every entry's first contributor stores (see the C adds), and
    // the slots of a column's missing neighbours (mesh sides) are never written (zero)
    if (lane < 4) reinterpret_cast<double2*>(colp + S4::NS + (s & 1) * 8)[lane] = make_double2(0.0, 0.0);
  };
  // the layer flush is split: the C warps take columns 0 .. NC-1 right after the layer's adds,
  // the PC warps (idle ~70 %) the rest while the C warps compute the next layer's first batch
  constexpr int NCC = S4::NC;

  if (warp < S4::NPC) {
    // ---------------------------- PC: Gauss-point cores ----------------------------
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
            if (t >= 2) bsync(S4::B_CE + slot, NPC_T + NC_T);
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
              double2* dst = reinterpret_cast<double2*>(cores + slot * S4::CSLOT + el * S4::CEL + g * S4::CSP);
#pragma unroll
              for (int k2 = 0; k2 < 4; ++k2) dst[k2] = make_double2(core[2 * k2], core[2 * k2 + 1]);
              dst[4] = make_double2(core[8], 0.0);
#pragma unroll
              for (int k2 = 5; k2 < 23; ++k2) dst[k2] = make_double2(core[2 * k2 - 1], core[2 * k2]);
              dst[23] = make_double2(core[45], 0.0);
            }
            PT_MARK(11, tid == 0);
            barrive(S4::B_CF + slot, NPC_T + NC_T);
            if (c == pair && s > s_first) {   // PC part of the flush of layer s - 1
              bsync(S4::B_AD, FL_T);
              PT_MARK(15, tid == 0);
              for (int cc = NCC + warp; cc < cols; cc += S4::NPC) flush_col(s - 1, cc);
              barrive(S4::B_FL, FL_T);
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
    bsync(S4::B_AD, FL_T);   // the last layer
    for (int cc = NCC + warp; cc < cols; cc += S4::NPC) flush_col(s_last, cc);
    // drain: the core-empty arrival of this pair's last batch
    for (int tt = max(t - 2, 0); tt < t; ++tt)
      if ((tt & 1) == pair) bsync(S4::B_CE + pair, NPC_T + NC_T);
    return;
  }

  // ------------------------- C: one warp per element of the batch -------------------------
  const int cw = warp - S4::NPC;                     // element slot of this warp
  const int ct = tid - 32 * S4::NPC;
  // expansion lane: node xa, Gauss point 4 * round + xg
  const int xa = lane & 7, xg = lane >> 3;
  int xox, xoy, xoz;
  node_off<3>(xa, xox, xoy, xoz);
  // pair lane
  const bool plane_lane = lane < S4::NOFF;
  int pa = 0, pb = 1;
  if (plane_lane) {
#pragma unroll
    for (int k = 0; k < S4::NOFF; ++k)
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
  double* myrec = recs + cw * S4::RWARP;
  auto plane_of = [&](double* colp, int zpar, bool zs, int dz) -> double* {
    if (dz == 0) return colp + (zpar ? S4::Z1 : S4::Z0);
    return colp + (zs ? S4::UP : S4::DN);
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
        bsync(S4::B_CF + cslot, NPC_T + NC_T);
        PT_MARK(0, ptc);
        if (!live) {
          barrive(S4::B_CE + cslot, NPC_T + NC_T);
          if (wait_flush) bsync(S4::B_FL, FL_T);
          if (c != prev_c) bsync(S4::B_C, NC_T);
          prev_c = c;
          return;
        }
        const int i = ifst + 2 * (k % ni), j = jfst + 2 * (k / ni);
        const int sz = int(s - z0);   // layer of node z relative to the chunk
        const double* ce = cores + cslot * S4::CSLOT + cw * S4::CEL;
        // pair lanes: Kuu_ab and sum_g ghc gA.gB; moment lanes: two (node, component)
        // tasks t = lane, lane + 32 (t < 56: n = t / 7, c = t % 7), 8 moments each
        double Kuu[3][3], Gd = 0.0;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int u = 0; u < 3; ++u) Kuu[r][u] = 0.0;
        double M1[8], M2[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) M1[q] = M2[q] = 0.0;
        const int mt1 = lane, mt2 = lane + 32;
        const int mn1 = mt1 / 7, mc1 = mt1 - 7 * mn1;
        const int mn2 = mt2 < 56 ? mt2 / 7 : 0, mc2 = mt2 < 56 ? mt2 - 7 * (mt2 / 7) : 0;
        int mo1 = 0, mo2 = 0;
        mo1 = mom_off(mc1);
        mo2 = mom_off(mc2);
        const double* mrec1 = myrec + mn1 * S4::RS + mo1;
        const double* mrec2 = myrec + mn2 * S4::RS + mo2;
        double ns[8];
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) ns[k2] = 0.0;
        // moments of the records of round R (GPs 4R .. 4R + 3); N_m(g) compile-time constants
        auto moments = [&](auto rc) {
          constexpr int R = decltype(rc)::value;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double v1 = mrec1[k * S4::RGP];
            const double v2 = mt2 < 56 ? mrec2[k * S4::RGP] : 0.0;
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
          // expansions of the 8 nodes at GPs 4 rnd .. 4 rnd + 3
          {
            const int g = 4 * rnd + xg;
            const double* co = ce + g * S4::CSP;
            double* blk = myrec + xg * S4::RGP;
            expand4(co, shtab + (g * NEN + xa) * 6, blk + xa * S4::RS, ns);
            if (xa == 0)
              *reinterpret_cast<double2*>(blk + NEN * S4::RS) = make_double2(co[C4::MU], co[C4::GHC]);
          }
          if (rnd == 1) barrive(S4::B_CE + cslot, NPC_T + NC_T);   // core slot no longer read
          __syncwarp();
          PT_MARK(1, ptc);
          if (rnd == 0) moments(std::integral_constant<int, 0>{});
          else moments(std::integral_constant<int, 1>{});
#pragma unroll 1
          for (int gg = 0; gg < 4; ++gg) {
            const double* blk = myrec + gg * S4::RGP;
            const double2* A2 = reinterpret_cast<const double2*>(blk + pa * S4::RS);
            const double2* B2 = reinterpret_cast<const double2*>(blk + pb * S4::RS);
            const double2 hdr = *reinterpret_cast<const double2*>(blk + NEN * S4::RS);
            double gA[3], sA[3], gB[3], t1[3], t2[3];
            double2 v;
            v = A2[0]; gA[0] = v.x; gA[1] = v.y;
            v = A2[1]; gA[2] = v.x; sA[0] = v.y;
            v = A2[2]; sA[1] = v.x; sA[2] = v.y;
            v = B2[0]; gB[0] = v.x; gB[1] = v.y;
            v = B2[3]; gB[2] = v.x; t1[0] = v.y;
            v = B2[4]; t1[1] = v.x; t1[2] = v.y;
            v = B2[5]; t2[0] = v.x; t2[1] = v.y;
            t2[2] = B2[6].x;
            const double mu = hdr.x, ghc = hdr.y;
            double dot = gA[0] * gB[0];
            dot = fma(gA[1], gB[1], dot);
            dot = fma(gA[2], gB[2], dot);
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              const double ub = mu * gB[r];
#pragma unroll
              for (int u = 0; u < 3; ++u) {
                double x = Kuu[r][u];
                x = fma(gA[r], t1[u], x);
                x = fma(sA[r], t2[u], x);
                x = fma(gA[u], ub, x);
                Kuu[r][u] = x;
              }
              Kuu[r][r] = fma(mu, dot, Kuu[r][r]);
            }
            Gd = fma(ghc, dot, Gd);
          }
          __syncwarp();
          PT_MARK(2, ptc);
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
        if (wait_flush) bsync(S4::B_FL, FL_T);
        if (c != prev_c) bsync(S4::B_C, NC_T);
        prev_c = c;
        PT_MARK(4, ptc);
        const int zpar_s = int(s & 1);
        if (xg == 0) {
          const int nx_ = i + xox, ny_ = j + xoy;
          const int nz = sz + xoz;   // relative to z0
          if (nx_ >= ix0 && nx_ < ix1 && ny_ >= iy0 && ny_ < iy1 && nz >= 0 && s + xoz < z1) {
            double2* n2 = reinterpret_cast<double2*>(col_of(nx_, ny_) + S4::NS + ((zpar_s ^ xoz) & 1) * 8);
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
          // Is this element the first contributor (add order: layer, then colour (i&1) + 2 (j&1))
          // to the pair's entries?  The elements sharing nodes A and B differ from this one only
          // along the axes where A and B coincide: not first if the layer below shares them (A,
          // B on this element's bottom face), or a sharing neighbour in this layer has the
          // smaller colour (this element's parity bit is 1 on such an axis).  The first
          // contributor stores, the others add: the planes need no reset after a flush.
          bool first = !(obz == oaz && oaz == 0 && s >= 1);
          if (obx == oax) {
            const int ia = oax ? i + 1 : i - 1;
            if ((i & 1) && ia >= 0 && ia < G.nx) first = false;
          }
          if (oby == oay) {
            const int ja = oay ? j + 1 : j - 1;
            if ((j & 1) && ja >= 0 && ja < G.nyE) first = false;
          }
          const double2 zero2 = make_double2(0.0, 0.0);
          if (own_a) {
            double* Pp = plane_of(col_of(ax, ay), (zpar_s ^ oaz) & 1, oaz == 0, dzAB);
            // all 8 loads of the block first: the compiler cannot prove the rows distinct and
            // would otherwise serialise 8 read-modify-write round trips
            double2 lo[4], hi[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const double2* q = reinterpret_cast<const double2*>(Pp + r * 36);
              lo[r] = first ? zero2 : q[qAB0];
              hi[r] = first ? zero2 : q[qAB1];
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
              lo[r] = first ? zero2 : q[qBA0];
              hi[r] = first ? zero2 : q[qBA1];
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
        bsync(S4::B_C, NC_T);      // all adds of layer s are in
        barrive(S4::B_AD, FL_T);   // the PC warps may flush their columns
        PT_MARK(6, ptc);
        prev_c = -1;
        for (int cc = cw; cc < NCC && cc < cols; cc += S4::NC) flush_col(s, cc);
        PT_MARK(7, ptc);
        bsync(S4::B_C, NC_T);
        PT_MARK(8, ptc);
      });
}

}  // namespace lgdm

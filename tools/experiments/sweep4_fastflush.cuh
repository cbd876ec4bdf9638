// lgdm_sweep4.cuh -- Hex8 hot kernel (k_sweep4): the structured-sweep K/R assembly redesigned
// from the ncu profile of k_sweep3 (profiles/r01).  Included by lgdm_sweep.cuh (needs
// SweepGeom, node_off, plane_slot, Core/gpCore).
//
// Same contract as k_sweep3: one CTA owns TX x TY node columns and a chunk of node layers,
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
//     pair lanes read the records with broadcast 16-byte loads -- no inter-warp hand-off per
//     Gauss point, only one per batch (the core ring).
//  3. Node sums (R = F, U, V) accumulate in registers and are reduced with shuffles.
//  4. The Appendix A core (exp, sqrt, divide: a long FP64 dependency chain) runs in two PC
//     warp pairs on alternate batches, one core slot each, 16-byte core stores/loads.
//  5. Flush: vectorised row copies, the -sum of plane -1 kept in the (never accumulated)
//     self slot of plane 0.  The flush of element layer s runs in the PC warps (idle ~70 % of
//     the time waiting for core slots) while the C warps compute the first batch of layer
//     s + 1; the C warps only wait for it before that batch's adds.
//
//   PC warps (element x GP)   gpCore -> core slots [2][E][NGP][CSP] (one per PC pair)
//   C  warps (one per element) expansions -> records [4 GP][8 node]; Gauss sums of the 28
//                              off-diagonal pairs; adds into the block-row planes; flush
#pragma once

namespace lgdm {

struct S4 {
  static constexpr int TX = 3, TY = 7, E = 8, NCOL = 4;
  static constexpr int NGP = 8, NEN = 8, NDPN = 4, NOFF = 28;
  static constexpr int NPC = 4, NC = E;                          // warps per role
  static constexpr int T = 32 * (NPC + NC);
  // shape table [NGP][NEN][4] = (dN/dxi, N) at the Gauss points
  static constexpr int SHT = NGP * NEN * 4;
  // core ring [3][E][NGP][CSP]: core = Core<3> values with a pad after J^-1 so every field
  // group is 16-byte aligned (48 doubles); CSP = 50 (25 x 16 B) puts the 4 cores a C warp
  // reads at once into distinct bank groups
  static constexpr int CSP = 50, CEL = NGP * CSP + 2, CSLOT = E * CEL, NCSLOT = 2;
  // warp-private records [4 GP][8 node][RS] + (mu*, ghc) per GP
  static constexpr int RS = 22, RGP = NEN * RS + 2, RWARP = 4 * RGP;
  // accumulator column: planes Z0, Z1 (in-plane, by node-layer parity), UP, DN; each plane
  // [row 4][slot 9][j 4] = 144 doubles (+2 pad: 73 x 16 B, odd); NS[2][8]
  static constexpr int PL = 146, Z0 = 0, Z1 = PL, UP = 2 * PL, DN = 3 * PL, NS = 4 * PL,
                       COL = NS + 16 + 2;                 // 602 doubles = 301 x 16 B (odd)
  static constexpr int NCOLS = TX * TY;
  static constexpr size_t SMEM = sizeof(double) * (size_t(SHT) + size_t(NCSLOT) * CSLOT +
                                                   size_t(NC) * RWARP + size_t(NCOLS) * COL);
  // named barriers: core full 1-2, core empty 3-4 (slot = PC pair), C warps 5, layer adds
  // done (C -> PC) 6, layer flushed (PC -> C) 7
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
//   [g0 g1][g2 E][s0 s1][s2 w0][w1 w2][d0 d1][d2 N][t1_0 t1_1][t1_2 t2_0][t2_1 t2_2]
//   g = grad N, s = S grad N, w = W' grad N (Kue), d = Dt' grad N (Keu), E (Kee), N,
//   t1 = lam* g + Ams s, t2 = Ams g + Ass s (Kuu)

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
  r2[0] = make_double2(gn[0], gn[1]);
  r2[1] = make_double2(gn[2], Ea);
  r2[2] = make_double2(SgN[0], SgN[1]);
  r2[3] = make_double2(SgN[2], WgN[0]);
  r2[4] = make_double2(WgN[1], WgN[2]);
  r2[5] = make_double2(DgN[0], DgN[1]);
  r2[6] = make_double2(DgN[2], Na);
  r2[7] = make_double2(t1[0], t1[1]);
  r2[8] = make_double2(t1[2], t2[0]);
  r2[9] = make_double2(t2[1], t2[2]);
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
  constexpr int E = S4::E, NGP = 8, NEN = 8;
  extern __shared__ double sm[];
  double* shtab = sm;                              // [NGP][NEN][4]
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
    for (int j = 0; j < 3; ++j) shtab[k * 4 + j] = shape_dxi<3>(a, g, j);
    shtab[k * 4 + 3] = shapeN<3>(a, g);
  }
  for (int k = tid; k < S4::NCOLS * S4::COL; k += S4::T) acc[k] = 0.0;
  __shared__ int64_t sbase[2][S4::NCOLS];   // CSR offsets of node layers (by parity)
  for (int q = tid; q < 2 * cols; q += S4::T) {
    const int cc = q % cols;
    const int64_t zq = s_first + q / cols;
    const int cy = cc / cols_x;
    if (zq >= z0 && zq < z1)
      sbase[zq & 1][cc] = base[node_id(ix0 + (cc - cy * cols_x), iy0 + cy, zq) - G.own_node_b];
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
        const int nc = ni * nj;   // <= E: TX <= 3 and TY <= 7 give <= 2 x 4 per colour
        body(s, c, 0, ifst, ni, jfst, nc);
      }
      end_of_layer(s);
    }
  };

  constexpr int NPC_T = 64, NC_T = 32 * S4::NC;
  static_assert(((S4::TX + 2) / 2) * ((S4::TY + 2) / 2) <= S4::E, "one batch per colour");
  constexpr int FL_T = 32 * (S4::NPC + S4::NC);   // adds-done / flushed barriers: everyone

  auto fcol_of = [&](int x, int y) { return acc + ((x - ix0) + cols_x * (y - iy0)) * S4::COL; };
  // ---- flush helpers (one warp per column) ----
  // copy plane P ([row 4][9 slots][4]) of node (x, y, z) to its compacted CSR position
  auto write_plane = [&](int x, int y, int64_t z, int dz, const double* P, bool inner) {
    const int zlo = z > 0 ? -1 : 0, zhi = z < G.nl ? 1 : 0;
    if (inner) {
      const int W2 = 18 * (zhi - zlo + 1);   // row width in double2
      double2* out = reinterpret_cast<double2*>(val + sbase[z & 1][(x - ix0) + cols_x * (y - iy0)]) + (dz - zlo) * 18;
      const double2* src = reinterpret_cast<const double2*>(P);
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (lane < 18) __stcs(out + r * W2 + lane, src[r * 18 + (lane ^ ((lane >> 3) & 1))]);
      return;
    }
    const int xlo = x > 0 ? -1 : 0, xhi = x < G.nx ? 1 : 0;
    const int ylo = y > 0 ? -1 : 0, yhi = y < G.nyN - 1 ? 1 : 0;
    const int wx = xhi - xlo + 1, wy = yhi - ylo + 1, wz = zhi - zlo + 1;
    const int W = 4 * wx * wy * wz;
    double* out = val + sbase[z & 1][(x - ix0) + cols_x * (y - iy0)] + (dz - zlo) * (4 * wx * wy);
    for (int it = lane; it < 36; it += 32) {
      const int i = it / 9, sl = it - 9 * i;
      const int dy = sl / 3 - 1, dx = sl - 3 * (dy + 1) - 1;
      if (dx < xlo || dx > xhi || dy < ylo || dy > yhi) continue;
      const double2* src = reinterpret_cast<const double2*>(P + i * 36);
      double2* dst = reinterpret_cast<double2*>(out + i * W + 4 * ((dy - ylo) * wx + (dx - xlo)));
      __stcs(dst, src[swz(sl, 0)]);
      __stcs(dst + 1, src[swz(sl, 1)]);
    }
  };
  // lanes 0..15: entry (i, j) = (lane / 4, lane % 4) of the 4x4 blocks, summed over slots
  auto plane_sum = [&](const double* P, bool skip_self) {
    double s = 0.0;
    const double* p = P + (lane >> 2) * 36;
    const int j = lane & 3;
#pragma unroll
    for (int sl = 0; sl < 9; ++sl)
      if (!(skip_self && sl == 4)) s += p[soff(sl, j)];
    return s;
  };
  // finish node (x, y, z): diagonal block = -sum(plane -1) [kept in the self slot]
  // - sum(plane 0 off-diagonal) - sum(plane +1) + (U, V); then plane 0, +1 and R go out
  auto finish_node = [&](int x, int y, int64_t z, double* colp, bool has_up, bool inner) {
    double* Zp = colp + ((z & 1) ? S4::Z1 : S4::Z0);
    const double* ns = colp + S4::NS + (z & 1) * 8;
    if (lane < 16) {
      const int i = lane >> 2, j = lane & 3;
      double* self = Zp + i * 36 + soff(4, j);
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

  // flush of one interior column, written for throughput: (A) all row sums at once (lane =
  // entry x half, two partial sums combined by one shuffle), (B) the outgoing planes as one
  // flat loop of independent 16-byte copies, (C) the resets
  auto flush_col_inner = [&](int x, int y, int64_t s, double* colp, bool own_s, bool own_s1) {
    const int e = lane & 15, h = lane >> 4;
    const int ri = e >> 2, j = e & 3;
    double* Zs = colp + ((s & 1) ? S4::Z1 : S4::Z0);
    double* Zn = colp + (((s + 1) & 1) ? S4::Z1 : S4::Z0);
    const double* ns = colp + S4::NS + (s & 1) * 8;
    const bool has_up = s < G.nl;
    double a = 0.0, b = 0.0;
    if (h == 0) {
      const double* dn = colp + S4::DN + ri * 36;
      const double* zs = Zs + ri * 36;
      double a2 = 0.0, b2 = 0.0;
      if (own_s1) {
#pragma unroll
        for (int sl = 0; sl < 9; sl += 2) a += dn[soff(sl, j)];
#pragma unroll
        for (int sl = 1; sl < 9; sl += 2) a2 += dn[soff(sl, j)];
      }
      if (own_s) {
        b = zs[soff(0, j)] + zs[soff(1, j)];
        b2 = zs[soff(2, j)] + zs[soff(3, j)];
      }
      a += a2;
      b += b2;
    } else if (own_s) {
      const double* zs = Zs + ri * 36;
      const double* up = colp + S4::UP + ri * 36;
      double b2 = 0.0;
      b = zs[soff(5, j)] + zs[soff(6, j)];
      b2 = zs[soff(7, j)] + zs[soff(8, j)];
      if (has_up) {
        double u1 = 0.0, u2 = 0.0;
#pragma unroll
        for (int sl = 0; sl < 9; sl += 2) u1 += up[soff(sl, j)];
#pragma unroll
        for (int sl = 1; sl < 9; sl += 2) u2 += up[soff(sl, j)];
        b2 += u1 + u2;
      }
      b += b2;
    }
    b += __shfl_xor_sync(0xffffffffu, b, 16);
    if (h == 0) {
      if (own_s) {
        double* self = Zs + ri * 36 + soff(4, j);
        double d = *self - b;
        if (j == 3) d += (ri < 3) ? ns[4 + ri] : ns[7];
        *self = d;
      }
      if (own_s1) Zn[ri * 36 + soff(4, j)] = -a;
    }
    __syncwarp();
    // (B) planes out: DN as plane -1 of node layer s+1; plane 0 and +1 of node layer s
    const int cc = (x - ix0) + cols_x * (y - iy0);
    // plane kinds 0 = DN (if own_s1), 1 = plane 0 and 2 = UP of node layer s (if own_s)
    const int kfirst = own_s1 ? 0 : 1;
    const int np = (own_s1 ? 1 : 0) + (own_s ? (has_up ? 2 : 1) : 0);
    const int zlo_s = s > 0 ? -1 : 0;
    const int w2s = 18 * ((has_up ? 1 : 0) - zlo_s + 1);
    const int w2n = 18 * (((s + 1) < G.nl ? 1 : 0) + 2);
    double2* dn_out = reinterpret_cast<double2*>(val + sbase[(s + 1) & 1][cc]);
    double2* z_out = reinterpret_cast<double2*>(val + sbase[s & 1][cc]) + (0 - zlo_s) * 18;
#pragma unroll 4
    for (int it = lane; it < 72 * np; it += 32) {
      const int pl = it >= 72 ? (it >= 144 ? 2 : 1) : 0;
      const int kind = pl + kfirst;
      const int rem = it - 72 * pl;
      const int rr = rem >= 36 ? (rem >= 54 ? 3 : 2) : (rem >= 18 ? 1 : 0);
      const int q = rem - 18 * rr;
      const double* sp = colp + (kind == 0 ? S4::DN : (kind == 1 ? ((s & 1) ? S4::Z1 : S4::Z0) : S4::UP));
      double2* dp = kind == 0 ? dn_out + rr * w2n : z_out + (kind - 1) * 18 + rr * w2s;
      __stcs(dp + q, reinterpret_cast<const double2*>(sp)[rr * 18 + (q ^ ((q >> 3) & 1))]);
    }
    if (own_s && lane < 4) __stcs(Rv + (node_id(x, y, s) - G.own_node_b) * 4 + lane, ns[lane]);
    __syncwarp();
    // (C) reset plane 0 of node layer s (reused for s+2), UP, DN, node sums of s
    double2* z2 = reinterpret_cast<double2*>(Zs);
    double2* ud = reinterpret_cast<double2*>(colp + S4::UP);
    const double2 zero = make_double2(0.0, 0.0);
    for (int k2 = lane; k2 < S4::PL / 2; k2 += 32) z2[k2] = zero;
    for (int k2 = lane; k2 < S4::PL; k2 += 32) ud[k2] = zero;
    if (lane < 4) reinterpret_cast<double2*>(colp + S4::NS + (s & 1) * 8)[lane] = zero;
  };
  // flush of element layer s by the PC warps (one warp per column): plane -1 of node layer
  // s + 1 out (its minus row sums parked in that node's self slot), node layer s finished
  // (and node layer s + 1 if s is the chunk's last layer), planes and node sums reset
  auto flush_layer = [&](int64_t s, int w0, int nw) {
    const bool own_s = s >= z0 && s < z1, own_s1 = s + 1 >= z0 && s + 1 < z1;
    const bool top = s == s_last && own_s1;
    for (int cc = w0; cc < cols; cc += nw) {
      const int cy = cc / cols_x;
      const int x = ix0 + (cc - cy * cols_x), y = iy0 + cy;
      const bool inner = x > 0 && x < G.nx && y > 0 && y < G.nyN - 1;
      double* colp = fcol_of(x, y);
      if (inner && !top) {
        flush_col_inner(x, y, s, colp, own_s, own_s1);
        continue;
      }
      if (own_s1) {
        if (lane < 16)
          colp[(((s + 1) & 1) ? S4::Z1 : S4::Z0) + (lane >> 2) * 36 + soff(4, lane & 3)] =
              -plane_sum(colp + S4::DN, false);
        write_plane(x, y, s + 1, -1, colp + S4::DN, inner);
      }
      __syncwarp();
      if (own_s) finish_node(x, y, s, colp, s < G.nl, inner);
      if (top) finish_node(x, y, s + 1, colp, false, inner);
      __syncwarp();
      double2* z2 = reinterpret_cast<double2*>(colp + ((s & 1) ? S4::Z1 : S4::Z0));
      double2* ud = reinterpret_cast<double2*>(colp + S4::UP);
      const double2 zero = make_double2(0.0, 0.0);
      for (int k2 = lane; k2 < S4::PL / 2; k2 += 32) z2[k2] = zero;
      for (int k2 = lane; k2 < S4::PL; k2 += 32) ud[k2] = zero;
      if (lane < 4) reinterpret_cast<double2*>(colp + S4::NS + (s & 1) * 8)[lane] = zero;
    }
  };
  // CSR offsets of node layer zq into sbase[zq & 1], for the columns this PC warp flushes
  // (each warp reads only its own columns' entries: no cross-warp hazard)
  auto load_sbase = [&](int64_t zq) {
    for (int cc = warp + S4::NPC * lane; cc < cols; cc += 32 * S4::NPC) {
      const int cy = cc / cols_x;
      if (zq >= z0 && zq < z1)
        sbase[zq & 1][cc] = base[node_id(ix0 + (cc - cy * cols_x), iy0 + cy, zq) - G.own_node_b];
    }
  };

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
              gpCore<3>(m, X, U, __ldg(kappa + e * NGP + g), g, core);
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
          }
          ++t;
        },
        [](int64_t) {});
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
  if (plane_lane) offdiag_ab(lane, pa, pb);
  int oax, oay, oaz, obx, oby, obz;
  node_off<3>(pa, oax, oay, oaz);
  node_off<3>(pb, obx, oby, obz);
  const int psAB = plane_slot<3>(obx - oax, oby - oay), psBA = plane_slot<3>(oax - obx, oay - oby);
  const int dzAB = obz - oaz;
  double* myrec = recs + cw * S4::RWARP;
  auto col_of = [&](int x, int y) { return acc + ((x - ix0) + cols_x * (y - iy0)) * S4::COL; };
  auto plane_of = [&](double* colp, int zpar, bool zs, int dz) -> double* {
    if (dz == 0) return colp + (zpar ? S4::Z1 : S4::Z0);
    return colp + (zs ? S4::UP : S4::DN);
  };

  int prev_c = -1, t = 0;
  const bool ptc = ct == 0;
  PT_DECL
  schedule(
      [&](int64_t s, int c, int b0, int ifst, int ni, int jfst, int nc) {
        const int k = b0 + cw;
        const bool live = k < nc;   // warp-uniform
        const int cslot = t & 1;
        ++t;
        if (prev_c < 0 && s > s_first) {
          // first batch of element layer s: CSR offsets of node layer s+1 for this layer's
          // flush (the loads overlap the batch; sbase[(s+1) & 1] was last read by flush(s-1))
          for (int cc = ct; cc < cols; cc += NC_T) {
            const int cy = cc / cols_x;
            if (s + 1 >= z0 && s + 1 < z1)
              sbase[(s + 1) & 1][cc] = base[node_id(ix0 + (cc - cy * cols_x), iy0 + cy, s + 1) - G.own_node_b];
          }
        }
        PT_MARK(9, ptc);
        bsync(S4::B_CF + cslot, NPC_T + NC_T);
        PT_MARK(0, ptc);
        if (!live) {
          barrive(S4::B_CE + cslot, NPC_T + NC_T);
          if (c != prev_c) bsync(S4::B_C, NC_T);
          prev_c = c;
          return;
        }
        const int i = ifst + 2 * (k % ni), j = jfst + 2 * (k / ni);
        const int sz = int(s - z0);   // layer of node z relative to the chunk
        const double* ce = cores + cslot * S4::CSLOT + cw * S4::CEL;
        Pair4 P;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
#pragma unroll
          for (int u = 0; u < 3; ++u) P.Kuu[r][u] = 0.0;
          P.Kue_ab[r] = P.Kue_ba[r] = P.Keu_ab[r] = P.Keu_ba[r] = 0.0;
        }
        P.Kee_ab = P.Kee_ba = 0.0;
        double ns[8];
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) ns[k2] = 0.0;
#pragma unroll 1
        for (int rnd = 0; rnd < 2; ++rnd) {
          // expansions of the 8 nodes at GPs 4 rnd .. 4 rnd + 3
          {
            const int g = 4 * rnd + xg;
            const double* co = ce + g * S4::CSP;
            double* blk = myrec + xg * S4::RGP;
            expand4(co, shtab + (g * NEN + xa) * 4, blk + xa * S4::RS, ns);
            if (xa == 0)
              *reinterpret_cast<double2*>(blk + NEN * S4::RS) = make_double2(co[C4::MU], co[C4::GHC]);
          }
          if (rnd == 1) barrive(S4::B_CE + cslot, NPC_T + NC_T);   // core slot no longer read
          __syncwarp();
          PT_MARK(1, ptc);
#pragma unroll 1
          for (int gg = 0; gg < 4; ++gg) {
            const double* blk = myrec + gg * S4::RGP;
            const double2* A2 = reinterpret_cast<const double2*>(blk + pa * S4::RS);
            const double2* B2 = reinterpret_cast<const double2*>(blk + pb * S4::RS);
            const double2 hdr = *reinterpret_cast<const double2*>(blk + NEN * S4::RS);
            double gA[3], sA[3], wA[3], dA[3], EA, NA, gB[3], t1[3], t2[3], wB[3], dB[3], EB, NB;
            double2 v;
            v = A2[0]; gA[0] = v.x; gA[1] = v.y;
            v = A2[1]; gA[2] = v.x; EA = v.y;
            v = A2[2]; sA[0] = v.x; sA[1] = v.y;
            v = A2[3]; sA[2] = v.x; wA[0] = v.y;
            v = A2[4]; wA[1] = v.x; wA[2] = v.y;
            v = A2[5]; dA[0] = v.x; dA[1] = v.y;
            v = A2[6]; dA[2] = v.x; NA = v.y;
            v = B2[0]; gB[0] = v.x; gB[1] = v.y;
            v = B2[1]; gB[2] = v.x; EB = v.y;
            v = B2[3]; wB[0] = v.y;
            v = B2[4]; wB[1] = v.x; wB[2] = v.y;
            v = B2[5]; dB[0] = v.x; dB[1] = v.y;
            v = B2[6]; dB[2] = v.x; NB = v.y;
            v = B2[7]; t1[0] = v.x; t1[1] = v.y;
            v = B2[8]; t1[2] = v.x; t2[0] = v.y;
            v = B2[9]; t2[1] = v.x; t2[2] = v.y;
            const double mu = hdr.x, ghc = hdr.y;
            double dot = gA[0] * gB[0];
            dot = fma(gA[1], gB[1], dot);
            dot = fma(gA[2], gB[2], dot);
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              const double ub = mu * gB[r];
#pragma unroll
              for (int u = 0; u < 3; ++u) {
                double x = P.Kuu[r][u];
                x = fma(gA[r], t1[u], x);
                x = fma(sA[r], t2[u], x);
                x = fma(gA[u], ub, x);
                P.Kuu[r][u] = x;
              }
              P.Kuu[r][r] = fma(mu, dot, P.Kuu[r][r]);
              P.Kue_ab[r] = fma(NB, wA[r], P.Kue_ab[r]);
              P.Kue_ba[r] = fma(NA, wB[r], P.Kue_ba[r]);
              P.Keu_ab[r] = fma(NA, dB[r], P.Keu_ab[r]);
              P.Keu_ba[r] = fma(NB, dA[r], P.Keu_ba[r]);
            }
            P.Kee_ab = fma(NB, EA, fma(ghc, dot, P.Kee_ab));
            P.Kee_ba = fma(NA, EB, fma(ghc, dot, P.Kee_ba));
          }
          __syncwarp();
          PT_MARK(2, ptc);
        }
        // node sums: reduce the four Gauss-point lanes of each node (lanes xa + 8 xg)
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) {
          ns[k2] += __shfl_xor_sync(0xffffffffu, ns[k2], 8);
          ns[k2] += __shfl_xor_sync(0xffffffffu, ns[k2], 16);
        }
        PT_MARK(3, ptc);
        // batches of one colour share no node; a new colour waits for the previous adds
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
          if (own_a) {
            double* Pp = plane_of(col_of(ax, ay), (zpar_s ^ oaz) & 1, oaz == 0, dzAB);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              double2* q = reinterpret_cast<double2*>(Pp + r * 36);
              double2 lo = q[swz(psAB, 0)], hi = q[swz(psAB, 1)];
              if (r < 3) {
                lo.x += P.Kuu[r][0]; lo.y += P.Kuu[r][1]; hi.x += P.Kuu[r][2]; hi.y += P.Kue_ab[r];
              } else {
                lo.x += P.Keu_ab[0]; lo.y += P.Keu_ab[1]; hi.x += P.Keu_ab[2]; hi.y += P.Kee_ab;
              }
              q[swz(psAB, 0)] = lo;
              q[swz(psAB, 1)] = hi;
            }
          }
          if (own_b) {
            double* Pp = plane_of(col_of(bx, by), (zpar_s ^ obz) & 1, obz == 0, -dzAB);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              double2* q = reinterpret_cast<double2*>(Pp + r * 36);
              double2 lo = q[swz(psBA, 0)], hi = q[swz(psBA, 1)];
              if (r < 3) {
                lo.x += P.Kuu[0][r]; lo.y += P.Kuu[1][r]; hi.x += P.Kuu[2][r]; hi.y += P.Kue_ba[r];
              } else {
                lo.x += P.Keu_ba[0]; lo.y += P.Keu_ba[1]; hi.x += P.Keu_ba[2]; hi.y += P.Kee_ba;
              }
              q[swz(psBA, 0)] = lo;
              q[swz(psBA, 1)] = hi;
            }
          }
        }
      },
      [&](int64_t s) {
        PT_MARK(5, ptc);
        bsync(S4::B_C, NC_T);   // all adds of layer s are in
        PT_MARK(6, ptc);
        prev_c = -1;
        flush_layer(s, cw, S4::NC);
        PT_MARK(7, ptc);
        bsync(S4::B_C, NC_T);
        PT_MARK(8, ptc);
      });
}

}  // namespace lgdm

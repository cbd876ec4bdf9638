// lgdm_sweep6.cuh -- Hex8 kernel k_sweep6: register-resident pair stars.  Included by
// lgdm_sweep.cuh after lgdm_sweep4.cuh (reuses S4's plane layout, C4, swz/soff, bsync).
//
// Why: k_sweep4 is bound by shared-memory delivery (70 % of the crossbar, FP64 27 %): the
// node records of every (element, GP) go through shared memory and each of the 28 pair lanes
// reloads 31 doubles per GP.  Here a C lane owns one element and one node "star" -- a centre
// node A and four leaf nodes B (K8 = 7 stars of 4 edges: centre r < 7 has leaves
// {7, r+1, r+2, r+3 mod 7}; lane r = 7 only carries node 7's sums) -- and loops over the 8
// Gauss points itself: it reads the element's GP core once per GP, rebuilds the records it
// needs in registers (grad N_A once, grad N_B per leaf) and accumulates the 4 pair blocks in
// registers.  Shared-memory bytes per element drop ~3x; the FP64 work rises (records rebuilt
// per star), which is what the FP64 pipe (27 % busy) has room for.
//
// Pair algebra per GP (A = centre, B = leaf; t1/t2 of Eq. 11a folded into the centre):
//   Kuu_AB += uA gB^T + vA (S gB)^T + gB (mu gA)^T + mu (gA.gB) I,
//             uA = lam* gA + Ams S gA, vA = Ams gA + Ass S gA
//   Kue_AB += N_B W'gA,  Kue_BA += (N_A W') gB,  Keu_AB += (N_A Dt') gB,  Keu_BA += N_B Dt'gA
//   Kee_AB += N_B E_A + ghc gA.gB,   Kee_BA += N_A hN N_B + (N_A gv).gB + ghc gA.gB
// (same terms as accumulate_pair / the oracle, reassociated).  Diagonal blocks: row-sum
// identity at flush, as in k_sweep4.
//
// Pipeline (12 warps, 1 CTA / SM):
//   PC warps 0-3: two pairs, pair p computes the GP cores of the colours c with c % 2 == p
//                 into core slot c (fixed producer and consumer per slot).
//   C  warps 4-11: group q = colour q (2 warps x 4 elements x 8 star lanes).  Group q adds
//                 its batch after group q-1 (named-barrier chain, deterministic order
//                 (layer, colour) per entry); the end-of-layer flush is split between group
//                 3 (right after its adds) and group 0 (before its next adds), so groups 1 and
//                 2 never wait for it.
#pragma once

namespace lgdm {

struct S6 {
  static constexpr int TX = S4::TX, TY = S4::TY, E = 8, NCOL = 4;
  static constexpr int NGP = 8, NEN = 8;
  static constexpr int NPC = 4, NC = 8;
  static constexpr int T = 32 * (NPC + NC);
  static constexpr int SHT = NGP * NEN * 4;
  static constexpr int CSP = S4::CSP, CEL = S4::CEL, CSLOT = E * CEL, NCSLOT = NCOL;
  static constexpr int PL = S4::PL, Z0 = S4::Z0, Z1 = S4::Z1, UP = S4::UP, DN = S4::DN,
                       NS = S4::NS, COL = S4::COL;
  static constexpr int NCOLS = TX * TY;
  static constexpr size_t SMEM =
      sizeof(double) * (size_t(SHT) + size_t(NCSLOT) * CSLOT + size_t(NCOLS) * COL);
  // named barriers: core full 1-4 and empty 5-8 (slot = colour), add chain 9-11 (colour
  // 1..3 waits for colour-1), flush: X 12 (colour 3's adds done), Y 13 (its flush part done)
  static constexpr int B_CF = 1, B_CE = 5, B_A = 8, B_X = 12, B_Y = 13;
};

// leaf k (0..3) of star r (0..6)
__device__ __forceinline__ int star_leaf(int r, int k) {
  if (k == 0) return 7;
  const int b = r + k;
  return b >= 7 ? b - 7 : b;
}

__global__ void __launch_bounds__(S6::T, 1)
k_sweep6(DevMat m, SweepGeom G, const double* __restrict__ coords,
         const double* __restrict__ dofs, const double* __restrict__ kappa,
         const int64_t* __restrict__ base, double* __restrict__ val, double* __restrict__ Rv) {
  constexpr int NGP = 8, NEN = 8;
  extern __shared__ double sm[];
  double* shtab = sm;                              // [NGP][NEN][4] = (dN/dxi, N)
  double* cores = shtab + S6::SHT;                 // [4 colours][E][CEL]
  double* acc = cores + S6::NCSLOT * S6::CSLOT;    // [NCOLS][COL]
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  int bid = blockIdx.x;
  const int tx = bid % G.tiles_x;
  bid /= G.tiles_x;
  const int ty = bid % G.tiles_y;
  const int ch = bid / G.tiles_y;
  const int64_t x0 = int64_t(tx) * S6::TX, x1 = min(x0 + S6::TX, G.nx + 1);
  const int64_t y0 = int64_t(ty) * S6::TY, y1 = min(y0 + S6::TY, G.nyN);
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

  __shared__ int64_t sbase[2][S6::NCOLS];   // CSR offsets of node layers (by parity)
  for (int k = tid; k < NGP * NEN; k += S6::T) {
    const int g = k >> 3, a = k & 7;
#pragma unroll
    for (int j = 0; j < 3; ++j) shtab[k * 4 + j] = shape_dxi<3>(a, g, j);
    shtab[k * 4 + 3] = shapeN<3>(a, g);
  }
  for (int k = tid; k < S6::NCOLS * S6::COL; k += S6::T) acc[k] = 0.0;
  for (int q = tid; q < 2 * cols; q += S6::T) {
    const int cc = q % cols;
    const int64_t zq = s_first + q / cols;
    const int cy = cc / cols_x;
    if (zq >= z0 && zq < z1)
      sbase[zq & 1][cc] = base[node_id(ix0 + (cc - cy * cols_x), iy0 + cy, zq) - G.own_node_b];
  }
  __syncthreads();

  // batch (layer s, colour c): the elements (i, j) of layer s with (i & 1, j & 1) = colour
  // bits, at most E of them (TX, TY <= 2 E - 1 per parity class)
  struct Batch {
    int ifst, ni, jfst, nc;
  };
  auto batch_of = [&](int c) {
    Batch b;
    b.ifst = ilo + ((ilo & 1) != (c & 1) ? 1 : 0);
    b.ni = b.ifst < ihi ? (ihi - b.ifst + 1) / 2 : 0;
    b.jfst = jlo + ((jlo & 1) != (c >> 1) ? 1 : 0);
    const int nj = b.jfst < jhi ? (jhi - b.jfst + 1) / 2 : 0;
    b.nc = b.ni * nj;
    return b;
  };
  constexpr int SLOT_T = 192;   // 64 PC threads + 128 C threads per core slot

  if (warp < S6::NPC) {
    // ---------------------------- PC: Gauss-point cores ----------------------------
    const int pair = warp >> 1;                       // colours c with c % 2 == pair
    const int lid = (warp & 1) * 32 + lane;
    const int el = lid >> 3, g = lid & 7;
    PT_DECL
    for (int64_t s = s_first; s <= s_last; ++s) {
      for (int c = pair; c < S6::NCOL; c += 2) {
        const Batch B = batch_of(c);
        PT_MARK(15, tid == 0);
        if (s > s_first) bsync(S6::B_CE + c, SLOT_T);
        PT_MARK(13, tid == 0);
        if (el < B.nc) {
          const int i = B.ifst + 2 * (el % B.ni), j = B.jfst + 2 * (el / B.ni);
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
          double2* dst = reinterpret_cast<double2*>(cores + c * S6::CSLOT + el * S6::CEL + g * S6::CSP);
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) dst[k2] = make_double2(core[2 * k2], core[2 * k2 + 1]);
          dst[4] = make_double2(core[8], 0.0);
#pragma unroll
          for (int k2 = 5; k2 < 23; ++k2) dst[k2] = make_double2(core[2 * k2 - 1], core[2 * k2]);
          dst[23] = make_double2(core[45], 0.0);
        }
        PT_MARK(14, tid == 0);
        barrive(S6::B_CF + c, SLOT_T);
      }
    }
    // drain: the core-empty arrivals of the last layer
    for (int c = pair; c < S6::NCOL; c += 2) bsync(S6::B_CE + c, SLOT_T);
    return;
  }

  // ------------- C: super-group = colour parity, lane = (element, star) -------------
  const int cw = warp - S6::NPC;                   // 0..7
  const int sg = cw >> 2;                          // colours c with c % 2 == sg
  const int wi = cw & 3;
  const bool kuu = (wi & 1) == 0;                  // role: Kuu blocks / coupling blocks + sums
  const int st = wi * 32 + lane;                   // thread index within the super-group
  const int el = 4 * (wi >> 1) + (lane >> 3), r = lane & 7;
  const bool star = r < 7;
  int oax, oay, oaz;
  node_off<3>(r, oax, oay, oaz);

  auto col_of = [&](int x, int y) { return acc + ((x - ix0) + cols_x * (y - iy0)) * S6::COL; };
  auto plane_of = [&](double* colp, int zpar, bool zs, int dz) -> double* {
    if (dz == 0) return colp + (zpar ? S6::Z1 : S6::Z0);
    return colp + (zs ? S6::UP : S6::DN);
  };

  // ---- flush helpers (one warp per column), as k_sweep4 ----
  auto write_plane = [&](int x, int y, int64_t z, int dz, const double* P, bool inner) {
    const int zlo = z > 0 ? -1 : 0, zhi = z < G.nl ? 1 : 0;
    if (inner) {
      const int W2 = 18 * (zhi - zlo + 1);   // row width in double2
      double2* out = reinterpret_cast<double2*>(val + sbase[z & 1][(x - ix0) + cols_x * (y - iy0)]) + (dz - zlo) * 18;
      const double2* src = reinterpret_cast<const double2*>(P);
#pragma unroll
      for (int rr = 0; rr < 4; ++rr)
        if (lane < 18) __stcs(out + rr * W2 + lane, src[rr * 18 + (lane ^ ((lane >> 3) & 1))]);
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
  auto plane_sum = [&](const double* P, bool skip_self) {
    double s = 0.0;
    const double* p = P + (lane >> 2) * 36;
    const int j = lane & 3;
#pragma unroll
    for (int sl = 0; sl < 9; ++sl)
      if (!(skip_self && sl == 4)) s += p[soff(sl, j)];
    return s;
  };
  auto finish_node = [&](int x, int y, int64_t z, double* colp, bool has_up, bool inner) {
    double* Zp = colp + ((z & 1) ? S6::Z1 : S6::Z0);
    const double* ns = colp + S6::NS + (z & 1) * 8;
    if (lane < 16) {
      const int i = lane >> 2, j = lane & 3;
      double* self = Zp + i * 36 + soff(4, j);
      double d = *self - plane_sum(Zp, true);
      if (has_up) d -= plane_sum(colp + S6::UP, false);
      if (j == 3) d += (i < 3) ? ns[4 + i] : ns[7];
      *self = d;
    }
    __syncwarp();
    write_plane(x, y, z, 0, Zp, inner);
    if (has_up) write_plane(x, y, z, 1, colp + S6::UP, inner);
    if (lane < 4) __stcs(Rv + (node_id(x, y, z) - G.own_node_b) * 4 + lane, ns[lane]);
  };
  // flush of element layer s, part `part` (0: super-group 0, 1: super-group 1), one warp
  // per column: columns cc with cc % 8 = 4 part + wi
  auto flush_part = [&](int64_t s, int part) {
    const bool own_s = s >= z0 && s < z1, own_s1 = s + 1 >= z0 && s + 1 < z1;
    const bool top = s == s_last && own_s1;
    for (int cc = 4 * part + wi; cc < cols; cc += 8) {
      const int cy = cc / cols_x;
      const int x = ix0 + (cc - cy * cols_x), y = iy0 + cy;
      const bool inner = x > 0 && x < G.nx && y > 0 && y < G.nyN - 1;
      double* colp = col_of(x, y);
      if (own_s1) {
        if (lane < 16)
          colp[(((s + 1) & 1) ? S6::Z1 : S6::Z0) + (lane >> 2) * 36 + soff(4, lane & 3)] =
              -plane_sum(colp + S6::DN, false);
        write_plane(x, y, s + 1, -1, colp + S6::DN, inner);
      }
      __syncwarp();
      if (own_s) finish_node(x, y, s, colp, s < G.nl, inner);
      if (top) finish_node(x, y, s + 1, colp, false, inner);
      __syncwarp();
      double2* z2 = reinterpret_cast<double2*>(colp + ((s & 1) ? S6::Z1 : S6::Z0));
      double2* ud = reinterpret_cast<double2*>(colp + S6::UP);
      const double2 zero = make_double2(0.0, 0.0);
      for (int k2 = lane; k2 < S6::PL / 2; k2 += 32) z2[k2] = zero;
      for (int k2 = lane; k2 < S6::PL; k2 += 32) ud[k2] = zero;
      if (lane < 4) reinterpret_cast<double2*>(colp + S6::NS + (s & 1) * 8)[lane] = zero;
    }
  };

  constexpr int CHAIN_T = 256;   // both super-groups
  PT_DECL
  const bool ptk = sg == 0 && st == 0, ptu = sg == 0 && st == 32, pt1 = sg == 1 && st == 0;
  // wait for the turn of colour c of layer s (colour 0: also the flush of layer s - 1)
  auto wait_turn = [&](int64_t s, int c, int64_t pre) {
    if (c == 0) {
      if (s > s_first) {
        bsync(S6::B_X, CHAIN_T);
        flush_part(s - 1, 0);
        bsync(S6::B_Y, CHAIN_T);
        if (st < cols && s + 1 >= z0 && s + 1 < z1) sbase[(s + 1) & 1][st] = pre;
      }
    } else {
      bsync(S6::B_A + c, CHAIN_T);
    }
  };
  auto pass_turn = [&](int64_t s, int c) {
    if (c < 3) {
      barrive(S6::B_A + c + 1, CHAIN_T);
    } else {
      barrive(S6::B_X, CHAIN_T);
      flush_part(s, 1);
      PT_MARK(11, pt1);
      barrive(S6::B_Y, CHAIN_T);
    }
  };
  // owned-row tests and plane addressing of pair (centre r, leaf b) of element (i, j, s):
  // row 0 of the block (A, B) in A's plane and of (B, A) in B's plane, null if not owned
  struct PairAddr {
    double* pa;
    double* pb;
    int psAB, psBA;
  };
  auto pair_addr = [&](int64_t s, int i, int j, int b) {
    const int sz = int(s - z0);
    const int zpar_s = int(s & 1);
    int obx, oby, obz;
    node_off<3>(b, obx, oby, obz);
    PairAddr P;
    P.psAB = plane_slot<3>(obx - oax, oby - oay);
    P.psBA = plane_slot<3>(oax - obx, oay - oby);
    const int dzAB = obz - oaz;
    const int ax = i + oax, ay = j + oay, azr = sz + oaz;
    const int bx = i + obx, by = j + oby, bzr = sz + obz;
    const bool own_a = ax >= ix0 && ax < ix1 && ay >= iy0 && ay < iy1 && azr >= 0 && s + oaz < z1;
    const bool own_b = bx >= ix0 && bx < ix1 && by >= iy0 && by < iy1 && bzr >= 0 && s + obz < z1;
    P.pa = own_a ? plane_of(col_of(ax, ay), (zpar_s ^ oaz) & 1, oaz == 0, dzAB) : nullptr;
    P.pb = own_b ? plane_of(col_of(bx, by), (zpar_s ^ obz) & 1, obz == 0, -dzAB) : nullptr;
    return P;
  };
  auto add2 = [](double* p, double x, double y) {
    double2* q = reinterpret_cast<double2*>(p);
    double2 v = *q;
    v.x += x;
    v.y += y;
    *q = v;
  };

  for (int64_t s = s_first; s <= s_last; ++s) {
    for (int c = sg; c < S6::NCOL; c += 2) {
      const Batch B = batch_of(c);
      const bool live = el < B.nc;
      const int i = live ? B.ifst + 2 * (el % B.ni) : 0;
      const int j = live ? B.jfst + 2 * (el / B.ni) : 0;
      // super-group 0 prefetches the CSR offsets of node layer s + 1 (stored after flush(s-1))
      int64_t pre = -1;
      if (c == 0 && s > s_first && st < cols) {
        const int64_t zq = s + 1;
        const int cy = st / cols_x;
        if (zq >= z0 && zq < z1)
          pre = __ldg(base + node_id(ix0 + (st - cy * cols_x), iy0 + cy, zq) - G.own_node_b);
      }
      PT_MARK(0, ptk);
      PT_MARK(5, ptu);
      bsync(S6::B_CF + c, SLOT_T);
      PT_MARK(1, ptk);
      PT_MARK(6, ptu);
      const double* ce = cores + c * S6::CSLOT + el * S6::CEL;
      if (kuu) {
        // ---------------- Kuu role: 4 blocks Kuu_AB (3x3) ----------------
        double K[4][3][3];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int q = 0; q < 3; ++q) K[k][p][q] = 0.0;
        if (live && star) {
#pragma unroll 1
          for (int g = 0; g < NGP; ++g) {
            const double* co = ce + g * S6::CSP;
            auto ld2 = [&](int off, double& x, double& y) {
              const double2 v = *reinterpret_cast<const double2*>(co + off);
              x = v.x;
              y = v.y;
            };
            double Ji[9], S[6], lamS, Ams, Ass, hN, fe0, mu, pad;
            ld2(0, Ji[0], Ji[1]);
            ld2(2, Ji[2], Ji[3]);
            ld2(4, Ji[4], Ji[5]);
            ld2(6, Ji[6], Ji[7]);
            ld2(8, Ji[8], pad);
            ld2(C4::S, S[0], S[1]);
            ld2(C4::S + 2, S[2], S[3]);
            ld2(C4::S + 4, S[4], S[5]);
            ld2(C4::LAM, lamS, Ams);
            ld2(C4::LAM + 2, Ass, hN);
            ld2(C4::LAM + 4, fe0, mu);
            const double2 shA0 = reinterpret_cast<const double2*>(shtab + (g * NEN + r) * 4)[0];
            const double2 shA1 = reinterpret_cast<const double2*>(shtab + (g * NEN + r) * 4)[1];
            double gA[3], sA[3], uA[3], vA[3], mgA[3];
#pragma unroll
            for (int p = 0; p < 3; ++p)
              gA[p] = fma(Ji[6 + p], shA1.x, fma(Ji[3 + p], shA0.y, Ji[p] * shA0.x));
            symv<3>(S, gA, sA);
#pragma unroll
            for (int p = 0; p < 3; ++p) {
              uA[p] = fma(lamS, gA[p], Ams * sA[p]);
              vA[p] = fma(Ams, gA[p], Ass * sA[p]);
              mgA[p] = mu * gA[p];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              asm volatile("" ::: "memory");
              const int b = star_leaf(r, k);
              const double2 sh0 = reinterpret_cast<const double2*>(shtab + (g * NEN + b) * 4)[0];
              const double2 sh1 = reinterpret_cast<const double2*>(shtab + (g * NEN + b) * 4)[1];
              double gB[3], SgB[3];
#pragma unroll
              for (int p = 0; p < 3; ++p)
                gB[p] = fma(Ji[6 + p], sh1.x, fma(Ji[3 + p], sh0.y, Ji[p] * sh0.x));
              symv<3>(S, gB, SgB);
              double dot = gA[0] * gB[0];
              dot = fma(gA[1], gB[1], dot);
              dot = fma(gA[2], gB[2], dot);
#pragma unroll
              for (int p = 0; p < 3; ++p) {
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                  double x = K[k][p][q];
                  x = fma(uA[p], gB[q], x);
                  x = fma(vA[p], SgB[q], x);
                  x = fma(gB[p], mgA[q], x);
                  K[k][p][q] = x;
                }
                K[k][p][p] = fma(mu, dot, K[k][p][p]);
              }
            }
          }
        }
        PT_MARK(2, ptk);
        barrive(S6::B_CE + c, SLOT_T);
        wait_turn(s, c, pre);
        PT_MARK(3, ptk);
        PT_MARK(10, pt1);
        if (live && star) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const PairAddr P = pair_addr(s, i, j, star_leaf(r, k));
            if (P.pa) {
#pragma unroll
              for (int rr = 0; rr < 3; ++rr) {
                double* row = P.pa + rr * 36;
                add2(row + soff(P.psAB, 0), K[k][rr][0], K[k][rr][1]);
                row[soff(P.psAB, 2)] += K[k][rr][2];
              }
            }
            if (P.pb) {
#pragma unroll
              for (int rr = 0; rr < 3; ++rr) {
                double* row = P.pb + rr * 36;
                add2(row + soff(P.psBA, 0), K[k][0][rr], K[k][1][rr]);
                row[soff(P.psBA, 2)] += K[k][2][rr];
              }
            }
          }
        }
        PT_MARK(4, ptk);
      } else {
        // ------------- coupling role: Kue, Keu, Kee of 4 pairs; node sums of r -------------
        double Uab[4][3], Uba[4][3], Eab[4][3], Eba[4][3], Kab[4], Kba[4], ns[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
#pragma unroll
          for (int p = 0; p < 3; ++p) Uab[k][p] = Uba[k][p] = Eab[k][p] = Eba[k][p] = 0.0;
          Kab[k] = Kba[k] = 0.0;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) ns[k] = 0.0;
        if (live) {
#pragma unroll 1
          for (int g = 0; g < NGP; ++g) {
            const double* co = ce + g * S6::CSP;
            auto ld2 = [&](int off, double& x, double& y) {
              const double2 v = *reinterpret_cast<const double2*>(co + off);
              x = v.x;
              y = v.y;
            };
            double Ji[9], pad;
            ld2(0, Ji[0], Ji[1]);
            ld2(2, Ji[2], Ji[3]);
            ld2(4, Ji[4], Ji[5]);
            ld2(6, Ji[6], Ji[7]);
            ld2(8, Ji[8], pad);
            const double2 shA0 = reinterpret_cast<const double2*>(shtab + (g * NEN + r) * 4)[0];
            const double2 shA1 = reinterpret_cast<const double2*>(shtab + (g * NEN + r) * 4)[1];
            const double NA = shA1.y;
            double gA[3], wA[3], dA[3], NWT[6], NDT[6], NGV[3];
#pragma unroll
            for (int p = 0; p < 3; ++p)
              gA[p] = fma(Ji[6 + p], shA1.x, fma(Ji[3 + p], shA0.y, Ji[p] * shA0.x));
            {
              double T6[6];
              ld2(C4::WT, T6[0], T6[1]);
              ld2(C4::WT + 2, T6[2], T6[3]);
              ld2(C4::WT + 4, T6[4], T6[5]);
              symv<3>(T6, gA, wA);
#pragma unroll
              for (int q = 0; q < 6; ++q) NWT[q] = NA * T6[q];
              ld2(C4::DT, T6[0], T6[1]);
              ld2(C4::DT + 2, T6[2], T6[3]);
              ld2(C4::DT + 4, T6[4], T6[5]);
              symv<3>(T6, gA, dA);
#pragma unroll
              for (int q = 0; q < 6; ++q) NDT[q] = NA * T6[q];
              double fu[3];
              ld2(C4::SG, T6[0], T6[1]);
              ld2(C4::SG + 2, T6[2], T6[3]);
              ld2(C4::SG + 4, T6[4], T6[5]);
              symv<3>(T6, gA, fu);
#pragma unroll
              for (int p = 0; p < 3; ++p) {
                ns[p] += fu[p];
                ns[4 + p] += wA[p];
              }
            }
            double Ass, hN, fe0, mu, ghc, gv[3], fv[3];
            ld2(C4::LAM + 2, Ass, hN);
            ld2(C4::LAM + 4, fe0, mu);
            ld2(C4::LAM + 6, ghc, gv[0]);
            ld2(C4::LAM + 8, gv[1], gv[2]);
            ld2(C4::LAM + 10, fv[0], fv[1]);
            ld2(C4::LAM + 12, fv[2], pad);
            double gvd = 0.0, fvd = 0.0;
#pragma unroll
            for (int p = 0; p < 3; ++p) {
              gvd = fma(gv[p], gA[p], gvd);
              fvd = fma(fv[p], gA[p], fvd);
              NGV[p] = NA * gv[p];
            }
            const double EA = fma(hN, NA, gvd);
            const double NhN = NA * hN;
            ns[3] += fma(fe0, NA, fvd);
            ns[7] += EA;
            if (star) {
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                asm volatile("" ::: "memory");   // one leaf at a time: bounds the live temporaries
                const int b = star_leaf(r, k);
                const double2 sh0 = reinterpret_cast<const double2*>(shtab + (g * NEN + b) * 4)[0];
                const double2 sh1 = reinterpret_cast<const double2*>(shtab + (g * NEN + b) * 4)[1];
                const double NB = sh1.y;
                double gB[3], wB[3], dB[3];
#pragma unroll
                for (int p = 0; p < 3; ++p)
                  gB[p] = fma(Ji[6 + p], sh1.x, fma(Ji[3 + p], sh0.y, Ji[p] * sh0.x));
                symv<3>(NWT, gB, wB);
                symv<3>(NDT, gB, dB);
                double dot = gA[0] * gB[0];
                dot = fma(gA[1], gB[1], dot);
                dot = fma(gA[2], gB[2], dot);
                double gvB = NGV[0] * gB[0];
                gvB = fma(NGV[1], gB[1], gvB);
                gvB = fma(NGV[2], gB[2], gvB);
#pragma unroll
                for (int p = 0; p < 3; ++p) {
                  Uab[k][p] = fma(NB, wA[p], Uab[k][p]);
                  Uba[k][p] += wB[p];
                  Eab[k][p] += dB[p];
                  Eba[k][p] = fma(NB, dA[p], Eba[k][p]);
                }
                Kab[k] = fma(NB, EA, fma(ghc, dot, Kab[k]));
                Kba[k] = fma(NhN, NB, fma(ghc, dot, Kba[k])) + gvB;
              }
            }
          }
        }
        PT_MARK(7, ptu);
        barrive(S6::B_CE + c, SLOT_T);
        wait_turn(s, c, pre);
        PT_MARK(8, ptu);
        if (live) {
          const int sz = int(s - z0);
          const int nx_ = i + oax, ny_ = j + oay, nz = sz + oaz;
          if (nx_ >= ix0 && nx_ < ix1 && ny_ >= iy0 && ny_ < iy1 && nz >= 0 && s + oaz < z1) {
            double* n = col_of(nx_, ny_) + S6::NS + ((int(s & 1) ^ oaz) & 1) * 8;
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) add2(n + 2 * k2, ns[2 * k2], ns[2 * k2 + 1]);
          }
          if (star) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const PairAddr P = pair_addr(s, i, j, star_leaf(r, k));
              if (P.pa) {
#pragma unroll
                for (int rr = 0; rr < 3; ++rr) P.pa[rr * 36 + soff(P.psAB, 3)] += Uab[k][rr];
                add2(P.pa + 3 * 36 + soff(P.psAB, 0), Eab[k][0], Eab[k][1]);
                add2(P.pa + 3 * 36 + soff(P.psAB, 2), Eab[k][2], Kab[k]);
              }
              if (P.pb) {
#pragma unroll
                for (int rr = 0; rr < 3; ++rr) P.pb[rr * 36 + soff(P.psBA, 3)] += Uba[k][rr];
                add2(P.pb + 3 * 36 + soff(P.psBA, 0), Eba[k][0], Eba[k][1]);
                add2(P.pb + 3 * 36 + soff(P.psBA, 2), Eba[k][2], Kba[k]);
              }
            }
          }
        }
        PT_MARK(9, ptu);
      }
      pass_turn(s, c);
    }
  }
  if (sg == 0) {   // the flush of the last layer
    bsync(S6::B_X, CHAIN_T);
    flush_part(s_last, 0);
    bsync(S6::B_Y, CHAIN_T);
  }
}

}  // namespace lgdm

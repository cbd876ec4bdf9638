// lgdm_sweep5.cuh -- Hex8 hot kernel k_sweep5: k_sweep4 with the node expansions moved into
// the core lanes.  Included by lgdm_sweep.cuh after lgdm_sweep4.cuh (reuses S4's plane layout,
// swz/soff, offdiag_ab, bsync/barrive, Pair4).
//
// Why: k_sweep4 is bound by shared-memory delivery; 15 % of its bytes are the
// 8 node lanes of each Gauss point re-reading that point's 48-double core, and its PC warps
// idle 72 % of the time.  Here the PC lane (element, GP) keeps the Appendix A core in
// registers and writes the 8 node records of its Gauss point itself (grad N, S grad N, t1,
// t2, W' grad N, Dt' grad N, E, N, Fu, Fe) into ONE batch record slot; the C warps only do
// the 28 off-diagonal pair sums, the adds and the flush.  Two PC pairs alternate batches and
// hand the slot over through per-producer FULL/EMPTY barriers (fixed pairing, race-free).
#pragma once

namespace lgdm {

struct S5 {
  static constexpr int TX = S4::TX, TY = S4::TY, E = S4::E, NCOL = S4::NCOL;
  static constexpr int NGP = 8, NEN = 8, NOFF = 28;
  static constexpr int NPC = 4, NC = E;
  static constexpr int T = 32 * (NPC + NC);
  static constexpr int SHT = NGP * NEN * 4;
  // record (doubles): [g0 g1][g2 E][s0 s1][s2 w0][w1 w2][d0 d1][d2 N][t1_0 t1_1][t1_2 t2_0]
  // [t2_1 t2_2][fu0 fu1][fu2 fe][pad pad] = 26 (13 x 16 B, odd: the 8 node records of one
  // GP fall in distinct bank groups); per (element, GP): 8 records + (mu*, ghc) = 210 doubles
  // (105 x 16 B, odd: the 8 GP lanes of an element write distinct bank groups)
  static constexpr int RS = 26, RGP = NEN * RS + 2, REL = NGP * RGP, SLOT = E * REL;
  // accumulator column (k_sweep4's round-1 layout): planes Z0, Z1, UP, DN of 146 doubles, NS
  static constexpr int PL = 146, Z0 = 0, Z1 = PL, UP = 2 * PL, DN = 3 * PL, NS = 4 * PL,
                       COL = NS + 16 + 2, NCOLS = S4::NCOLS;
  static constexpr size_t SMEM = sizeof(double) * (size_t(SHT) + size_t(SLOT) + size_t(NCOLS) * COL);
  // The slot is split by Gauss point into halves h (GPs 4h .. 4h+3) written by PC warp (pair
  // p, half h) and released by C half by half, so the next batch's first half is written
  // while C still reads the second.  Named barriers: full [pair][half] 1-4, empty 5-8, C 9.
  static constexpr int B_FULL = 1, B_EMPTY = 5, B_C = 9;
};

__global__ void __launch_bounds__(S5::T, 1)
k_sweep5(DevMat m, SweepGeom G, const double* __restrict__ coords,
         const double* __restrict__ dofs, const double* __restrict__ kappa,
         const int64_t* __restrict__ base, double* __restrict__ val, double* __restrict__ Rv) {
  constexpr int E = S5::E, NGP = 8, NEN = 8;
  extern __shared__ double sm[];
  double* shtab = sm;                              // [NGP][NEN][4]
  double* recs = shtab + S5::SHT;                  // [E][NGP][RGP]
  double* acc = recs + S5::SLOT;                   // [NCOLS][COL]
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  int bid = blockIdx.x;
  const int tx = bid % G.tiles_x;
  bid /= G.tiles_x;
  const int ty = bid % G.tiles_y;
  const int ch = bid / G.tiles_y;
  const int64_t x0 = int64_t(tx) * S5::TX, x1 = min(x0 + S5::TX, G.nx + 1);
  const int64_t y0 = int64_t(ty) * S5::TY, y1 = min(y0 + S5::TY, G.nyN);
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

  for (int k = tid; k < NGP * NEN; k += S5::T) {
    const int g = k >> 3, a = k & 7;
#pragma unroll
    for (int j = 0; j < 3; ++j) shtab[k * 4 + j] = shape_dxi<3>(a, g, j);
    shtab[k * 4 + 3] = shapeN<3>(a, g);
  }
  for (int k = tid; k < S5::NCOLS * S5::COL; k += S5::T) acc[k] = 0.0;
  __syncthreads();

  auto schedule = [&](auto&& body, auto&& end_of_layer) {
    for (int64_t s = s_first; s <= s_last; ++s) {
      for (int c = 0; c < S5::NCOL; ++c) {
        const int ifst = ilo + ((ilo & 1) != (c & 1) ? 1 : 0);
        const int ni = ifst < ihi ? (ihi - ifst + 1) / 2 : 0;
        const int jfst = jlo + ((jlo & 1) != (c >> 1) ? 1 : 0);
        const int nj = jfst < jhi ? (jhi - jfst + 1) / 2 : 0;
        const int nc = ni * nj;
        for (int b0 = 0; b0 < nc; b0 += E) body(s, c, b0, ifst, ni, jfst, nc);
      }
      end_of_layer(s);
    }
  };

  [[maybe_unused]] constexpr int NPC_T = 64, NC_T = 32 * S5::NC;

  if (warp < S5::NPC) {
    // ---------- PC: core + 8 node expansions per lane (element, GP), straight to the slot ----------
    const int pair = warp >> 1;                       // batches t with t % 2 == pair
    const int half = warp & 1;                        // this warp writes GPs 4 half .. +3
    const int el = lane >> 2, g = 4 * half + (lane & 3);
    const int bsel = pair * 2 + half;
    const double* shg = shtab + g * NEN * 4;   // (dN/dxi, N) of the 8 nodes at this lane's GP
    auto sh = [&](int a, int j) { return shg[a * 4 + j]; };
    int t = 0;
    schedule(
        [&](int64_t s, int, int b0, int ifst, int ni, int jfst, int nc) {
          if ((t & 1) == pair) {
            const int k = b0 + el;
            const bool live = k < nc;
            double c[Core<3>::STRIDE];
            if (live) {
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
              gpCoreS<3>(m, X, U, __ldg(kappa + e * NGP + g), [&](int a, int jj) { return sh(a, jj); },
                         [&](int a) { return sh(a, 3); }, c);
            }
            if (t >= 1) bsync(S5::B_EMPTY + bsel, 32 + NC_T);   // half released by C
            if (live) {
              using Co = Core<3>;
              double* rg = recs + el * S5::REL + g * S5::RGP;
#pragma unroll
              for (int a = 0; a < NEN; ++a) {
                double gn[3], SgN[3], WgN[3], DgN[3], fu[3];
#pragma unroll
                for (int ii = 0; ii < 3; ++ii) {
                  double sacc = c[Co::JI + ii] * sh(a, 0);
                  sacc = fma(c[Co::JI + 3 + ii], sh(a, 1), sacc);
                  sacc = fma(c[Co::JI + 6 + ii], sh(a, 2), sacc);
                  gn[ii] = sacc;
                }
                symv<3>(c + Co::S, gn, SgN);
                symv<3>(c + Co::WT, gn, WgN);
                symv<3>(c + Co::DT, gn, DgN);
                symv<3>(c + Co::SG, gn, fu);
                const double Na = sh(a, 3);
                double t1[3], t2[3], gvd = 0.0, fvd = 0.0;
#pragma unroll
                for (int ii = 0; ii < 3; ++ii) {
                  t1[ii] = fma(c[Co::LAM], gn[ii], c[Co::AMS] * SgN[ii]);
                  t2[ii] = fma(c[Co::AMS], gn[ii], c[Co::ASS] * SgN[ii]);
                  gvd = fma(c[Co::GV + ii], gn[ii], gvd);
                  fvd = fma(c[Co::FV + ii], gn[ii], fvd);
                }
                const double Ea = fma(c[Co::HN], Na, gvd);
                const double fe = fma(c[Co::FE0], Na, fvd);
                double2* r2 = reinterpret_cast<double2*>(rg + a * S5::RS);
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
                r2[10] = make_double2(fu[0], fu[1]);
                r2[11] = make_double2(fu[2], fe);
              }
              *reinterpret_cast<double2*>(rg + NEN * S5::RS) = make_double2(c[Co::MU], c[Co::GHC]);
            }
            barrive(S5::B_FULL + bsel, 32 + NC_T);
          }
          ++t;
        },
        [](int64_t) {});
    // drain: C's slot release after the last batch is meant for the other pair's next batch
    if (t >= 1 && (t & 1) == pair) bsync(S5::B_EMPTY + bsel, 32 + NC_T);
    return;
  }

  // ------------------------------- C: one warp per element -------------------------------
  const int cw = warp - S5::NPC;
  const int ct = tid - 32 * S5::NPC;
  const bool plane_lane = lane < S5::NOFF;
  int pa = 0, pb = 1;
  if (plane_lane) offdiag_ab(lane, pa, pb);
  int oax, oay, oaz, obx, oby, obz;
  node_off<3>(pa, oax, oay, oaz);
  node_off<3>(pb, obx, oby, obz);
  const int psAB = plane_slot<3>(obx - oax, oby - oay), psBA = plane_slot<3>(oax - obx, oay - oby);
  const int dzAB = obz - oaz;
  auto col_of = [&](int x, int y) { return acc + ((x - ix0) + cols_x * (y - iy0)) * S5::COL; };
  auto plane_of = [&](double* colp, int zpar, bool zs, int dz) -> double* {
    if (dz == 0) return colp + (zpar ? S5::Z1 : S5::Z0);
    return colp + (zs ? S5::UP : S5::DN);
  };

  __shared__ int64_t sbase[2][S5::NCOLS];   // CSR offsets of node layers (by parity)
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
    double* Zp = colp + ((z & 1) ? S5::Z1 : S5::Z0);
    const double* ns = colp + S5::NS + (z & 1) * 8;
    if (lane < 16) {
      const int i = lane >> 2, j = lane & 3;
      double* self = Zp + i * 36 + soff(4, j);
      double d = *self - plane_sum(Zp, true);
      if (has_up) d -= plane_sum(colp + S5::UP, false);
      if (j == 3) d += (i < 3) ? ns[4 + i] : ns[7];
      *self = d;
    }
    __syncwarp();
    write_plane(x, y, z, 0, Zp, inner);
    if (has_up) write_plane(x, y, z, 1, colp + S5::UP, inner);
    if (lane < 4) __stcs(Rv + (node_id(x, y, z) - G.own_node_b) * 4 + lane, ns[lane]);
  };

  int prev_c = -1, t = 0;
  [[maybe_unused]] const bool ptc = ct == 0;
  PT_DECL
  schedule(
      [&](int64_t s, int c, int b0, int ifst, int ni, int jfst, int nc) {
        const int k = b0 + cw;
        const bool live = k < nc;   // warp-uniform
        const int prod = t & 1;
        ++t;
        if (prev_c < 0) {
          for (int q = ct; q < 2 * cols; q += NC_T) {
            const int cc = q % cols;
            const int64_t zq = s + q / cols;
            const int cy = cc / cols_x;
            if (zq >= z0 && zq < z1)
              sbase[zq & 1][cc] = base[node_id(ix0 + (cc - cy * cols_x), iy0 + cy, zq) - G.own_node_b];
          }
        }
        PT_MARK(9, ptc);
        Pair4 P;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
#pragma unroll
          for (int u = 0; u < 3; ++u) P.Kuu[r][u] = 0.0;
          P.Kue_ab[r] = P.Kue_ba[r] = P.Keu_ab[r] = P.Keu_ba[r] = 0.0;
        }
        P.Kee_ab = P.Kee_ba = 0.0;
        double nsa[2] = {0.0, 0.0};
        const double* re = recs + cw * S5::REL;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          bsync(S5::B_FULL + prod * 2 + h, 32 + NC_T);
          if (live) {
#pragma unroll 1
          for (int g = 4 * h; g < 4 * h + 4; ++g) {
            const double* blk = re + g * S5::RGP;
            const double2* A2 = reinterpret_cast<const double2*>(blk + pa * S5::RS);
            const double2* B2 = reinterpret_cast<const double2*>(blk + pb * S5::RS);
            const double2 hdr = *reinterpret_cast<const double2*>(blk + NEN * S5::RS);
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
          // node sums {Fu[3], Fe, U = sum W' grad N [3], V = sum E} over this half's GPs:
          // lane = (node a = lane / 4, quarter q) owns two of the eight values
          {
            const int a = lane >> 2, q = lane & 3;
            // record chunks: q0 (fu0, fu1) = 10, q1 (fu2, fe) = 11, q2 (w1, w2) = 4,
            // q3 (w0 = chunk 3 .y, E = chunk 1 .y)
            const int c0 = q == 0 ? 10 : q == 1 ? 11 : q == 2 ? 4 : 3;
#pragma unroll
            for (int g = 4 * h; g < 4 * h + 4; ++g) {
              const double2* r2 = reinterpret_cast<const double2*>(re + g * S5::RGP + a * S5::RS);
              const double2 x = r2[c0];
              const double2 y = r2[1];
              nsa[0] += q == 3 ? x.y : x.x;
              nsa[1] += q == 3 ? y.y : x.y;
            }
          }
          }
          // this half is free for the other PC pair's next batch
          barrive(S5::B_EMPTY + (prod ^ 1) * 2 + h, 32 + NC_T);
        }
        PT_MARK(2, ptc);
        if (c != prev_c) bsync(S5::B_C, NC_T);
        prev_c = c;
        PT_MARK(4, ptc);
        if (!live) return;
        const int i = ifst + 2 * (k % ni), j = jfst + 2 * (k / ni);
        const int sz = int(s - z0);
        const int zpar_s = int(s & 1);
        {   // node sums: lane (a, q) adds its two values (NS layout Fu0 Fu1 Fu2 Fe U0 U1 U2 V)
          const int a = lane >> 2, q = lane & 3;
          int ox, oy, oz;
          node_off<3>(a, ox, oy, oz);
          const int nx_ = i + ox, ny_ = j + oy;
          if (nx_ >= ix0 && nx_ < ix1 && ny_ >= iy0 && ny_ < iy1 && sz + oz >= 0 && s + oz < z1) {
            double* np = col_of(nx_, ny_) + S5::NS + ((zpar_s ^ oz) & 1) * 8;
            const int o0 = q == 0 ? 0 : q == 1 ? 2 : q == 2 ? 5 : 4;
            const int o1 = q == 0 ? 1 : q == 1 ? 3 : q == 2 ? 6 : 7;
            np[o0] += nsa[0];
            np[o1] += nsa[1];
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
        bsync(S5::B_C, NC_T);   // all adds of layer s are in
        PT_MARK(6, ptc);
        prev_c = -1;
        const bool own_s = s >= z0 && s < z1, own_s1 = s + 1 >= z0 && s + 1 < z1;
        const bool top = s == s_last && own_s1;   // node layer s+1 has no element layer above
        for (int cc = cw; cc < cols; cc += S5::NC) {
          const int cy = cc / cols_x;
          const int x = ix0 + (cc - cy * cols_x), y = iy0 + cy;
          const bool inner = x > 0 && x < G.nx && y > 0 && y < G.nyN - 1;
          double* colp = col_of(x, y);
          if (own_s1) {
            // plane -1 of node layer s+1 is complete: out, and minus its row sums go to the
            // self slot of that node's plane 0 (never accumulated by pair adds)
            if (lane < 16)
              colp[(((s + 1) & 1) ? S5::Z1 : S5::Z0) + (lane >> 2) * 36 + soff(4, lane & 3)] =
                  -plane_sum(colp + S5::DN, false);
            write_plane(x, y, s + 1, -1, colp + S5::DN, inner);
          }
          __syncwarp();
          if (own_s) finish_node(x, y, s, colp, s < G.nl, inner);
          if (top) finish_node(x, y, s + 1, colp, false, inner);
          __syncwarp();
          // reset plane 0 and node sums of node layer s (reused for layer s+2), UP, DN
          double2* z2 = reinterpret_cast<double2*>(colp + ((s & 1) ? S5::Z1 : S5::Z0));
          double2* ud = reinterpret_cast<double2*>(colp + S5::UP);
          const double2 zero = make_double2(0.0, 0.0);
          for (int k2 = lane; k2 < S5::PL / 2; k2 += 32) z2[k2] = zero;
          for (int k2 = lane; k2 < S5::PL; k2 += 32) ud[k2] = zero;
          if (lane < 4) reinterpret_cast<double2*>(colp + S5::NS + (s & 1) * 8)[lane] = zero;
        }
        PT_MARK(7, ptc);
        bsync(S5::B_C, NC_T);
        PT_MARK(8, ptc);
      });
}

}  // namespace lgdm

// lgdm_sweepq.cuh -- Q4 hot kernel (k_sweepq): fused structured-sweep K/R assembly for
// plane-strain 4-node quads.  Included by lgdm_sweep.cuh (needs SweepGeom, node_off, Core<2>,
// gpCore<2>, symv<2>, bsync/barrive from lgdm_sweep4.cuh).
//
// Contract as k_sweep4: one CTA owns TX node columns (x) and a chunk of node rows
// (y, the sweep axis), sweeps the element rows touching them (ghost elements recomputed),
// writes exactly the CSR block-rows of its nodes; per-entry summation order = (element row,
// colour) only, so K and R are bitwise independent of tiling and slabbing.
//
// Q4 is the configuration whose intensity sits on the B200 HBM/FP64 ridge, so the
// design minimises shared-memory traffic per element:
//   * PC warps, one lane per (element, Gauss point): the Appendix A core (gpCore) stays in
//     registers and the same lane expands it into the 4 node records of that Gauss point
//     (grad N, S grad N, t1, t2, W' grad N, Dt' grad N, E, N) and the per-node sums (R = F,
//     U = sum W' grad N, V = sum E), reduced over the element's 4 GP lanes by shuffles.  No
//     core ever goes through shared memory.  Four PC groups, one per (colour, row parity),
//     each owning one batch slot, so every slot has a fixed producer/consumer pair and two
//     batches of each colour are in production at once (the core chain is latency-bound).
//   * C warps, three lanes per element: lane k owns the star of node pairs {(k, b)} that
//     covers the element's 6 off-diagonal pairs twice-per-lane ({01,03}, {12,13}, {20,23}),
//     so the centre node's record is loaded once per Gauss point for two pairs.
//   * Diagonal blocks by the partition-of-unity row-sum identity (see lgdm_sweep4.cuh):
//     diag = [U, V] - sum of the row's other blocks, formed at flush.
#pragma once

namespace lgdm {

struct SQ {
  static constexpr int TX = 31, E = 16, NCOL = 2;            // 32 elements per row = 2 colours x E
  static constexpr int NGP = 4, NEN = 4, NDPN = 3;
  static constexpr int NPCG = 4, PCW = 2;                    // PC groups (colour x row parity), warps
  static constexpr int NCW = 4;                              // C warps: 2 groups (colours) x 2
  static constexpr int NFW = 4;                              // flush warps
  static constexpr int T = 32 * (NPCG * PCW + NCW + NFW);
  static constexpr int NSLOT = 4;                            // slot = 2 colour + row parity
  // shape table [NGP][NEN][4] = (dN/dxi0, dN/dxi1, N, 0)
  static constexpr int SHT = NGP * NEN * 4;
  // element block in a slot: records [NGP][NEN][RS] (GP stride GS), node sums [NEN][6],
  // (mu*, ghc)[NGP].  Strides chosen with a quarter-warp bank model (16-byte accesses): the
  // PC record stores are conflict-free, the C record loads 1.35x ideal (was 2x).
  static constexpr int RS = 14, GS = 60, REC = 0, NSUM = NGP * GS, HDR = NSUM + NEN * 6,
                       EL = 282;
  static_assert(HDR + 2 * NGP <= EL, "element block");
  static constexpr int SLOT = E * EL;
  // accumulators: the complete block-row of every tile node, in the CSR order of an
  // interior node: [row r 3][dy 3][dx 3][j 3] = 81 doubles; three node-row buffers (node
  // row zn uses buffer zn % 3) so the flush of node row s overlaps the adds of element row
  // s+1 (which touch node rows s+1, s+2); NS[3][TX][6]
  // Node sums are kept per colour (NSC apart) and added at flush: the colour-0 adds of
  // element row s+1 may run while the colour-1 adds of row s are still in flight, and both
  // touch the node sums of node row s+1 (never the same K entry: elements of different
  // colours in adjacent rows share no node pair).
  static constexpr int NROW = 81, NBUF = 3, ACC = NBUF * TX * NROW, NSB = ACC, NSS = 7,   // odd NS stride
                       NSC = NBUF * TX * NSS;
  static constexpr size_t SMEM = sizeof(double) * (size_t(SHT) + size_t(NSLOT) * SLOT +
                                                   size_t(ACC) + size_t(NCOL * NSC));
  // named barriers: slot full 1..3, slot empty 4..6; by row parity (group 0 may run up to
  // two rows ahead of the flush): colour-0 adds done 7/8, row adds done (C -> flush) 9/10,
  // node row flushed (flush -> group 0 two rows later) 11/12; flush warps 13
  static constexpr int B_F = 1, B_E = 1 + NSLOT, B_C0 = 1 + 2 * NSLOT, B_ADDS = B_C0 + 2,
                       B_FL = B_ADDS + 2, B_FW = B_FL + 2;
  static_assert(B_FW <= 15, "named barriers");
};

// record (doubles): [g0 g1][s0 s1][w0 w1][d0 d1][E N][t1_0 t1_1][t2_0 t2_1]

__global__ void __launch_bounds__(SQ::T, 1)
k_sweepq(DevMat m, SweepGeom G, const double* __restrict__ coords,
         const double* __restrict__ dofs, const double* __restrict__ kappa,
         const int64_t* __restrict__ base, double* __restrict__ val, double* __restrict__ Rv) {
  constexpr int E = SQ::E, NGP = 4, NEN = 4;
  extern __shared__ double sm[];
  double* shtab = sm;                          // [NGP][NEN][4]
  double* slots = shtab + SQ::SHT;             // [NSLOT][E][EL]
  double* acc = slots + SQ::NSLOT * SQ::SLOT;  // [TX][COL]
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  const int tx = blockIdx.x % G.tiles_x;
  const int ch = blockIdx.x / G.tiles_x;
  const int ix0 = tx * SQ::TX, ix1 = int(min(int64_t(ix0 + SQ::TX), G.nx + 1));
  const int64_t z0 = G.lay_own_b + int64_t(ch) * G.chunk_len;
  const int64_t z1 = min(z0 + G.chunk_len, G.lay_own_e);
  if (z0 >= z1) return;
  const int64_t nxN = G.nx + 1;
  const int64_t s_first = max(z0 - 1, int64_t(0));
  const int64_t s_last = min(z1, G.nl) - 1;
  const int ilo = max(ix0 - 1, 0), ihi = int(min(int64_t(ix1), G.nx));
  const int cols = ix1 - ix0;

  for (int k = tid; k < NGP * NEN; k += SQ::T) {
    const int g = k >> 2, a = k & 3;
    shtab[k * 4 + 0] = shape_dxi<2>(a, g, 0);
    shtab[k * 4 + 1] = shape_dxi<2>(a, g, 1);
    shtab[k * 4 + 2] = shapeN<2>(a, g);
    shtab[k * 4 + 3] = 0.0;
  }
  for (int k = tid; k < SQ::ACC + SQ::NCOL * SQ::NSC; k += SQ::T) acc[k] = 0.0;
  __syncthreads();

  // batch schedule (every role): element row s, colour c (parity of i) -- exactly one batch
  // (possibly empty) per colour and row, so batch t has colour t % 2
  static_assert(SQ::TX + 1 <= 2 * SQ::E, "one batch per colour");
  auto schedule = [&](auto&& body, auto&& end_of_row) {
    for (int64_t s = s_first; s <= s_last; ++s) {
      for (int c = 0; c < SQ::NCOL; ++c) {
        const int ifst = ilo + ((ilo & 1) != c ? 1 : 0);
        const int nc = ifst < ihi ? (ihi - ifst + 1) / 2 : 0;
        body(s, c, 0, ifst, nc);
      }
      end_of_row(s);
    }
  };
  constexpr int PCG_T = 32 * SQ::PCW, C_T = 32 * SQ::NCW, NFE = PCG_T + C_T / 2;

  if (warp < SQ::NPCG * SQ::PCW) {
    // ------------- PC: core + expansions + node sums, one lane per (element, GP) -------------
    const int grp = warp / SQ::PCW;
    const int lid = (warp % SQ::PCW) * 32 + lane;
    const int el = lid >> 2, g = lid & 3;
    double sh[NEN][3];
#pragma unroll
    for (int a = 0; a < NEN; ++a) {
      sh[a][0] = shtab[(g * NEN + a) * 4 + 0];
      sh[a][1] = shtab[(g * NEN + a) * 4 + 1];
      sh[a][2] = shtab[(g * NEN + a) * 4 + 2];
    }
    int t = 0;
    [[maybe_unused]] const bool ptp = tid == 0;
    PT_DECL
    schedule(
        [&](int64_t s, int, int b0, int ifst, int nc) {
          if ((t & 1) == (grp & 1) && ((t >> 1) & 1) == (grp >> 1)) {
            const int slot = 2 * (grp & 1) + (grp >> 1);   // = 2 colour + row parity
            PT_MARK(12, ptp);
            if (t >= SQ::NSLOT) bsync(SQ::B_E + slot, NFE);
            PT_MARK(10, ptp);
            const int k = b0 + el;
            double* eb = slots + slot * SQ::SLOT + el * SQ::EL;
            double ns[NEN][6];
#pragma unroll
            for (int a = 0; a < NEN; ++a)
#pragma unroll
              for (int q = 0; q < 6; ++q) ns[a][q] = 0.0;
            if (k < nc) {
              const int i = ifst + 2 * k;
              const int64_t n0 = i + nxN * s;
              auto nid = [&](int a) {
                int ox, oy, oz;
                node_off<2>(a, ox, oy, oz);
                return n0 + ox + nxN * oz;
              };
              auto X = [&](int a, int q) { return __ldg(coords + nid(a) * 2 + q); };
              auto U = [&](int a, int q) { return __ldg(dofs + nid(a) * 3 + q); };
              const int64_t e = i + G.nx * s;
              using Co = Core<2>;
              double c[Co::STRIDE];
              const int64_t q = e * NGP + g;   // defect fields if set
              gpCoreSK<2>(m, X, U, __ldg(kappa + q), G.k0g ? __ldg(G.k0g + q) : m.kappa0,
                          G.alg ? __ldg(G.alg + q) : m.alpha, [&](int a, int j) { return sh[a][j]; },
                          [&](int a) { return sh[a][2]; }, c);
#pragma unroll
              for (int a = 0; a < NEN; ++a) {
                double gn[2], SgN[2], WgN[2], DgN[2], fu[2];
                gn[0] = fma(c[Co::JI + 0], sh[a][0], c[Co::JI + 2] * sh[a][1]);
                gn[1] = fma(c[Co::JI + 1], sh[a][0], c[Co::JI + 3] * sh[a][1]);
                symv<2>(c + Co::S, gn, SgN);
                symv<2>(c + Co::WT, gn, WgN);
                symv<2>(c + Co::DT, gn, DgN);
                symv<2>(c + Co::SG, gn, fu);
                const double Na = sh[a][2];
                const double Ea = fma(c[Co::HN], Na, fma(c[Co::GV], gn[0], c[Co::GV + 1] * gn[1]));
                const double fe = fma(c[Co::FE0], Na, fma(c[Co::FV], gn[0], c[Co::FV + 1] * gn[1]));
                double2* r2 = reinterpret_cast<double2*>(eb + SQ::REC + g * SQ::GS + a * SQ::RS);
                r2[0] = make_double2(gn[0], gn[1]);
                r2[1] = make_double2(SgN[0], SgN[1]);
                r2[2] = make_double2(WgN[0], WgN[1]);
                r2[3] = make_double2(DgN[0], DgN[1]);
                r2[4] = make_double2(Ea, Na);
                r2[5] = make_double2(fma(c[Co::LAM], gn[0], c[Co::AMS] * SgN[0]),
                                     fma(c[Co::LAM], gn[1], c[Co::AMS] * SgN[1]));
                r2[6] = make_double2(fma(c[Co::AMS], gn[0], c[Co::ASS] * SgN[0]),
                                     fma(c[Co::AMS], gn[1], c[Co::ASS] * SgN[1]));
                ns[a][0] = fu[0];
                ns[a][1] = fu[1];
                ns[a][2] = fe;
                ns[a][3] = WgN[0];
                ns[a][4] = WgN[1];
                ns[a][5] = Ea;
              }
              reinterpret_cast<double2*>(eb + SQ::HDR)[g] = make_double2(c[Co::MU], c[Co::GHC]);
            }
            // node sums over the element's 4 GP lanes (lanes 4 el .. 4 el + 3): a transpose-
            // reduce that leaves lane g with the sums of node g, ((g0 + g1) + (g2 + g3)) in every
            // lane (commutative pairs: the same bits as a butterfly all-reduce).
            // step 1 (lane ^ 1): lanes keep the nodes a with (a & 1) == (g & 1)
            double h[2][6];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
              for (int q = 0; q < 6; ++q) {
                const double snd = (g & 1) ? ns[2 * u][q] : ns[2 * u + 1][q];
                const double rcv = __shfl_xor_sync(0xffffffffu, snd, 1);
                h[u][q] = ((g & 1) ? ns[2 * u + 1][q] : ns[2 * u][q]) + rcv;
              }
            // step 2 (lane ^ 2): lane g keeps node g = 2 (g >> 1) + (g & 1), i.e. h[g >> 1]
            double v[6];
#pragma unroll
            for (int q = 0; q < 6; ++q) {
              const double snd = (g >> 1) ? h[0][q] : h[1][q];
              const double rcv = __shfl_xor_sync(0xffffffffu, snd, 2);
              v[q] = ((g >> 1) ? h[1][q] : h[0][q]) + rcv;
            }
            if (k < nc) {
#pragma unroll
              for (int q = 0; q < 6; q += 2)
                *reinterpret_cast<double2*>(eb + SQ::NSUM + g * 6 + q) = make_double2(v[q], v[q + 1]);
            }
            barrive(SQ::B_F + slot, NFE);
            PT_MARK(11, ptp);
          }
          ++t;
        },
        [](int64_t) {});
    // drain the slot-empty arrivals no later batch of this group consumes
    for (int tt = max(t - SQ::NSLOT, 0); tt < t; ++tt)
      if ((tt & 1) == (grp & 1) && ((tt >> 1) & 1) == (grp >> 1)) bsync(SQ::B_E + 2 * (grp & 1) + (grp >> 1), NFE);
    return;
  }

  auto row_of = [&](int x, int64_t zn) { return acc + (int(zn % 3) * SQ::TX + (x - ix0)) * SQ::NROW; };
  auto ns_of = [&](int x, int64_t zn) { return acc + SQ::NSB + (int(zn % 3) * SQ::TX + (x - ix0)) * SQ::NSS; };
  const int ctid = tid - 32 * SQ::NPCG * SQ::PCW;   // C and flush threads

  if (ctid >= C_T) {
    // ------------------------------- flush warps -------------------------------
    // After both colours of element row s are added, node row s is complete: its diagonal
    // blocks come from the row-sum identity, then its block-rows (contiguous in the CSR for
    // consecutive interior nodes) and R stream out, and the row buffer is reset for s+2.
    const int ft = ctid - C_T;
    constexpr int F_T = 32 * SQ::NFW;
    [[maybe_unused]] const bool ptf = ft == 0;
    PT_DECL
    // compact the block-row of an edge node (fewer than 9 neighbours) into its CSR slots
    auto flush_edge = [&](int x, int64_t zn) {
      const int xlo = x > 0 ? -1 : 0, xhi = x < G.nx ? 1 : 0;
      const int zlo = zn > 0 ? -1 : 0, zhi = zn < G.nl ? 1 : 0;
      const int wx = xhi - xlo + 1, wz = zhi - zlo + 1;
      double* out = val + base[x + nxN * zn - G.own_node_b];
      double* row = row_of(x, zn);
      for (int idx = ft; idx < SQ::NROW; idx += F_T) {
        const int r = idx / 27, rem = idx - 27 * r, dy = rem / 9 - 1, rem2 = rem - 9 * (dy + 1);
        const int dx = rem2 / 3 - 1, j = rem2 - 3 * (dx + 1);
        if (dx >= xlo && dx <= xhi && dy >= zlo && dy <= zhi)
          __stcs(out + r * (3 * wx * wz) + (dy - zlo) * (3 * wx) + (dx - xlo) * 3 + j, row[idx]);
        row[idx] = 0.0;
      }
    };
    // nothing to flush for the two rows before the first: credit both parities
    barrive(SQ::B_FL + (int(s_first) & 1), F_T + 64);
    barrive(SQ::B_FL + (int(s_first + 1) & 1), F_T + 64);
    for (int64_t s = s_first; s <= s_last; ++s) {
      // CSR offset of the first interior node of node row s (and s+1 at the top), loaded
      // before the wait so the global-load latency hides behind it
      const bool topq = s == s_last && s + 1 >= z0 && s + 1 < z1;
      int64_t pre[2] = {0, 0};
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        const int64_t zn = s + pass;
        if ((pass == 0 || topq) && zn >= z0 && zn < z1 && zn > 0 && zn < G.nl && max(ix0, 1) < min(ix1, int(G.nx)))
          pre[pass] = base[max(ix0, 1) + nxN * zn - G.own_node_b];
      }
      PT_MARK(9, ptf);
      bsync(SQ::B_ADDS + (int(s) & 1), F_T + C_T);
      PT_MARK(4 + 10, ptf);
      const bool top = s == s_last && s + 1 >= z0 && s + 1 < z1;
      for (int pass = 0; pass < (top ? 2 : 1); ++pass) {
        const int64_t zn = s + pass;
        if (zn >= z0 && zn < z1) {
          // diagonal entries (column, r, j)
          for (int task = ft; task < cols * 9; task += F_T) {   // column fastest: conflict-free
            const int e = task / cols, cc = task - cols * e, r = e / 3, j = e - 3 * r;
            double* row = row_of(ix0 + cc, zn) + r * 27 + j;
            const double* ns0 = ns_of(ix0 + cc, zn);
            const double d0 = (row[0] + row[3]) + (row[6] + row[9]);
            const double d1 = (row[15] + row[18]) + (row[21] + row[24]);
            double d = -(d0 + d1);
            if (j == 2) {
              const int q = (r < 2) ? 3 + r : 5;
              d += ns0[q] + ns0[q + SQ::NSC];
            }
            row[4 * 3] = d;
          }
          PT_MARK(5, ptf);
          bsync(SQ::B_FW, F_T);
          PT_MARK(6, ptf);
          // rows out.  Interior nodes have 9 neighbours and consecutive node ids, so the
          // block-rows of a run of interior columns are ONE contiguous range of the CSR values,
          // in the same order as the row buffers: a linear copy.  Edge nodes (x = 0, x = nx,
          // first / last node row) are compacted element by element.
          const bool zin = zn > 0 && zn < G.nl;
          const int xa = zin ? max(ix0, 1) : ix1, xb = zin ? min(ix1, int(G.nx)) : ix1;
          if (xb > xa) {
            double* out = val + pre[pass];
            double* src = row_of(xa, zn);
            const int cnt = (xb - xa) * SQ::NROW;
            // 16-byte vectors when the CSR range and the row buffer are co-aligned
            const int head = ((reinterpret_cast<uintptr_t>(out) & 15) != 0) ? 1 : 0;
            const bool co = ((reinterpret_cast<uintptr_t>(out) ^ reinterpret_cast<uintptr_t>(src)) & 15) == 0;
            // (no reset: the next node row's first contributors store, see add_blocks)
            if (co) {
              if (head && ft == 0) __stcs(out, src[0]);
              const int nv = (cnt - head) >> 1;
              double2* o2 = reinterpret_cast<double2*>(out + head);
              const double2* s2 = reinterpret_cast<const double2*>(src + head);
#pragma unroll 4
              for (int k = ft; k < nv; k += F_T) __stcs(o2 + k, s2[k]);
              if (((cnt - head) & 1) && ft == 0) __stcs(out + cnt - 1, src[cnt - 1]);
            } else {
#pragma unroll 4
              for (int k = ft; k < cnt; k += F_T) __stcs(out + k, src[k]);
            }
          }
          for (int x = ix0; x < xa; ++x) flush_edge(x, zn);   // edge columns (x = 0) or rows
          for (int x = xb; x < ix1; ++x) flush_edge(x, zn);   // (x = nx)
          // R: consecutive nodes, 3 values each
          for (int k = ft; k < cols * 3; k += F_T) {
            const int cc = k / 3, j = k - 3 * cc;
            const double* ns0 = ns_of(ix0 + cc, zn);
            __stcs(Rv + (ix0 + cc + nxN * zn - G.own_node_b) * 3 + j, ns0[j] + ns0[j + SQ::NSC]);
          }
          bsync(SQ::B_FW, F_T);
          for (int k = ft; k < cols * SQ::NSS; k += F_T) {
            ns_of(ix0, zn)[k] = 0.0;
            ns_of(ix0, zn)[k + SQ::NSC] = 0.0;
          }
          // this buffer serves node row zn + 3 next; the mesh's top node row has no neighbours
          // above, so its (never written) dy = +1 slots must read as zero in the diagonal sums
          if (zn + 3 == G.nl)
            for (int k = ft; k < cols * 27; k += F_T) {
              const int cc = k / 27, q = k - 27 * cc, r = q / 9;
              row_of(ix0 + cc, zn)[r * 27 + 18 + (q - 9 * r)] = 0.0;
            }
          PT_MARK(7, ptf);
          bsync(SQ::B_FW, F_T);
          PT_MARK(8, ptf);
        }
      }
      barrive(SQ::B_FL + (int(s) & 1), F_T + 64);   // consumed by group 0 at row s + 2
      PT_MARK(9, ptf);
    }
    return;
  }

  // -------------------------- C: pair stars and adds --------------------------
  // two groups of 2 warps: group c consumes the colour-c batch of every row; both compute
  // concurrently, group 0 adds first (after the previous row is flushed), group 1 after
  const int ct = ctid;                            // 0 .. C_T-1
  const int cg = ct >> 6, gt = ct & 63;           // group, thread in group
  const int cel = gt / 3, ck = gt - 3 * cel;      // element slot, star index
  const bool star_lane = gt < 3 * E;
  // star k: centre A = k, B1 = {1, 2, 0}[k], B2 = 3
  const int pa = ck, pb1 = ck == 0 ? 1 : (ck == 1 ? 2 : 0), pb2 = 3;
  int oax, oay, oaz, ob1x, ob1y, ob1z, ob2x, ob2y, ob2z;
  node_off<2>(pa, oax, oay, oaz);
  node_off<2>(pb1, ob1x, ob1y, ob1z);
  node_off<2>(pb2, ob2x, ob2y, ob2z);

  struct PairQ {
    double Kuu[2][2], Kue_ab[2], Kue_ba[2], Keu_ab[2], Keu_ba[2], Kee_ab, Kee_ba;
  };
  auto zero_pair = [](PairQ& P) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      P.Kuu[r][0] = P.Kuu[r][1] = 0.0;
      P.Kue_ab[r] = P.Kue_ba[r] = P.Keu_ab[r] = P.Keu_ba[r] = 0.0;
    }
    P.Kee_ab = P.Kee_ba = 0.0;
  };
  // one Gauss point of pair (A, B): A side g, s, w, d, E, N; B side g, t1, t2, w, d, E, N
  auto acc_pair = [](PairQ& P, const double (&gA)[2], const double (&sA)[2], const double (&wA)[2],
                     const double (&dA)[2], double EA, double NA, const double2* B2, double mu,
                     double ghc) {
    double2 v;
    double gB[2], wB[2], dB[2], t1[2], t2[2], EB, NB;
    v = B2[0]; gB[0] = v.x; gB[1] = v.y;
    v = B2[2]; wB[0] = v.x; wB[1] = v.y;
    v = B2[3]; dB[0] = v.x; dB[1] = v.y;
    v = B2[4]; EB = v.x; NB = v.y;
    v = B2[5]; t1[0] = v.x; t1[1] = v.y;
    v = B2[6]; t2[0] = v.x; t2[1] = v.y;
    const double dot = fma(gA[1], gB[1], gA[0] * gB[0]);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const double ub = mu * gB[r];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
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
  };
  // block (row node, neighbour offset) inside the row buffer: [r][dy][dx][j]
  auto blk_of = [&](int x, int64_t zn, int dx, int dy) { return row_of(x, zn) + (dy + 1) * 9 + (dx + 1) * 3; };
  // first: this element is the first contributor to these entries in the add order (element
  // row, colour), so it stores instead of adding -- the row buffers need no reset after a
  // flush (only the never-written slots of edge nodes are kept at zero)
  auto add_blocks = [&](double* Pb, double* Qb, const PairQ& P, bool first) {
    auto put = [&](double* q, double v) { *q = first ? v : *q + v; };
    if (Pb) {   // K_AB into A's row at B's slot
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        put(Pb + r * 27 + 0, P.Kuu[r][0]);
        put(Pb + r * 27 + 1, P.Kuu[r][1]);
        put(Pb + r * 27 + 2, P.Kue_ab[r]);
      }
      put(Pb + 54 + 0, P.Keu_ab[0]);
      put(Pb + 54 + 1, P.Keu_ab[1]);
      put(Pb + 54 + 2, P.Kee_ab);
    }
    if (Qb) {   // K_BA into B's row at A's slot
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        put(Qb + r * 27 + 0, P.Kuu[0][r]);
        put(Qb + r * 27 + 1, P.Kuu[1][r]);
        put(Qb + r * 27 + 2, P.Kue_ba[r]);
      }
      put(Qb + 54 + 0, P.Keu_ba[0]);
      put(Qb + 54 + 1, P.Keu_ba[1]);
      put(Qb + 54 + 2, P.Kee_ba);
    }
  };
  auto owned = [&](int x, int64_t z) { return x >= ix0 && x < ix1 && z >= z0 && z < z1; };

  int t = 0;
  [[maybe_unused]] const bool ptc = ct == 0;
  PT_DECL
  schedule(
      [&](int64_t s, int c, int, int ifst, int nc) {
        const int slot = 2 * c + ((t >> 1) & 1);
        ++t;
        if (c != cg) return;                        // the other group's batch
        PT_MARK(0, ptc);
        bsync(SQ::B_F + slot, NFE);
        PT_MARK(1, ptc);
        const bool live = star_lane && cel < nc;
        const double* eb = slots + slot * SQ::SLOT + cel * SQ::EL;
        PairQ P1, P2;
        zero_pair(P1);
        zero_pair(P2);
        double nsum[6], nsum3[6];
        if (live) {
#pragma unroll 1
          for (int g = 0; g < NGP; ++g) {
            const double* rg = eb + SQ::REC + g * SQ::GS;
            const double2* A2 = reinterpret_cast<const double2*>(rg + pa * SQ::RS);
            const double2 hdr = reinterpret_cast<const double2*>(eb + SQ::HDR)[g];
            double gA[2], sA[2], wA[2], dA[2], EA, NA;
            double2 v;
            v = A2[0]; gA[0] = v.x; gA[1] = v.y;
            v = A2[1]; sA[0] = v.x; sA[1] = v.y;
            v = A2[2]; wA[0] = v.x; wA[1] = v.y;
            v = A2[3]; dA[0] = v.x; dA[1] = v.y;
            v = A2[4]; EA = v.x; NA = v.y;
            acc_pair(P1, gA, sA, wA, dA, EA, NA, reinterpret_cast<const double2*>(rg + pb1 * SQ::RS), hdr.x, hdr.y);
            acc_pair(P2, gA, sA, wA, dA, EA, NA, reinterpret_cast<const double2*>(rg + pb2 * SQ::RS), hdr.x, hdr.y);
          }
          // node sums of node ck (star 0 also node 3), read before the slot is released
#pragma unroll
          for (int q = 0; q < 6; ++q) {
            nsum[q] = eb[SQ::NSUM + ck * 6 + q];
            nsum3[q] = eb[SQ::NSUM + 3 * 6 + q];
          }
        }
        barrive(SQ::B_E + slot, NFE);
        // fixed add order: the previous row flushed, then colour 0, then colour 1
        PT_MARK(2, ptc);
        if (cg == 0) bsync(SQ::B_FL + (int(s) & 1), 32 * SQ::NFW + 64);   // node row s-2 flushed
        else bsync(SQ::B_C0 + (int(s) & 1), C_T);
        PT_MARK(3, ptc);
        if (live) {
          const int i = ifst + 2 * cel;
          const int ax = i + oax, b1x = i + ob1x, b2x = i + ob2x;
          const int64_t az = s + oaz, b1z = s + ob1z, b2z = s + ob2z;
          const bool oa = owned(ax, az), ob1 = owned(b1x, b1z), ob2 = owned(b2x, b2z);
          // first contributor of the pair's entries (shared with the neighbour across an edge):
          // star 0: (0,1) bottom edge -- element row s-1 adds first unless s = 0; (0,3) left
          // edge -- the even column of {i-1, i} (colour 0) first; star 1: (1,2) right edge
          // likewise, (1,3) diagonal; star 2: (2,0) diagonal, (2,3) top edge (row s+1 later)
          const bool ev = (i & 1) == 0;
          const bool first1 = ck == 0 ? s == 0 : (ck == 1 ? (ev || i + 1 == G.nx) : true);
          const bool first2 = ck == 0 ? (ev || i == 0) : true;
          add_blocks(oa ? blk_of(ax, az, b1x - ax, int(b1z - az)) : nullptr,
                     ob1 ? blk_of(b1x, b1z, ax - b1x, int(az - b1z)) : nullptr, P1, first1);
          add_blocks(oa ? blk_of(ax, az, b2x - ax, int(b2z - az)) : nullptr,
                     ob2 ? blk_of(b2x, b2z, ax - b2x, int(az - b2z)) : nullptr, P2, first2);
          auto add_ns = [&](int x, int64_t z, const double (&v)[6]) {
            double* np = ns_of(x, z) + cg * SQ::NSC;   // this colour's node sums
            double w[6];
#pragma unroll
            for (int q = 0; q < 6; ++q) w[q] = np[q];
#pragma unroll
            for (int q = 0; q < 6; ++q) np[q] = w[q] + v[q];
          };
          if (oa) add_ns(ax, az, nsum);
          if (ck == 0 && ob2) add_ns(b2x, b2z, nsum3);
        }
        if (cg == 0) barrive(SQ::B_C0 + (int(s) & 1), C_T);
        barrive(SQ::B_ADDS + (int(s) & 1), 32 * SQ::NFW + C_T);   // both groups, every row
        PT_MARK(4, ptc);
      },
      [&](int64_t) {});
  if (cg == 0) {   // the flushes of the last two rows
    if (s_last - 1 >= s_first) bsync(SQ::B_FL + (int(s_last - 1) & 1), 32 * SQ::NFW + 64);
    bsync(SQ::B_FL + (int(s_last) & 1), 32 * SQ::NFW + 64);
  }
}

}  // namespace lgdm

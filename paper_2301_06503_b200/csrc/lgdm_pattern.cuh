// lgdm_pattern.cuh -- the CSR pattern and the element maps built on the GPU (SURVEY 8a row A0,
// once per mesh).  The structural pattern of reading R-PAT: every (node a, node b) pair that
// shares an element, ndpn x ndpn dofs, columns ascending, explicit zeros kept -- what MATLAB's
// sparse() of the element triplets implies (Fig. 2 l.28-30) -- for any connectivity.
//
//   1. node -> adjacent (element, local node), ascending element id: a stable radix sort of the
//      element slots e * nen + a keyed by their node (CUB);
//   2. one warp per owned node stages the nodes of its adjacent elements (the candidates) in
//      shared memory; a candidate is a neighbour if no equal candidate precedes it; its rank
//      (= slot in the sorted neighbour list) is the number of distinct smaller candidates;
//      pass 1 counts the degree, an exclusive scan gives nbr_ptr (and base / row_ptr), pass 2
//      writes the sorted neighbour list and the element -> block-row slot map (AdjEntry).
// Deterministic: no atomics decide any order.  Limits: candidates per node (adjacent elements x
// nen) <= kCandMax, degree <= 255 (uint8 slots); beyond them create returns UNSUPPORTED.
#pragma once

#include <cub/cub.cuh>

namespace lgdm {

constexpr int kCandMax = 1024;   // candidate nodes per owned node (shared-memory staging)
constexpr int kPatWarps = 4;     // warps per CTA of the per-node passes

__global__ void k_adj_keys(int64_t n_slots, const int32_t* __restrict__ conn,
                           int32_t* __restrict__ keys, int32_t* __restrict__ vals,
                           int32_t* __restrict__ counts) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n_slots) return;
  const int32_t n = conn[i];
  keys[i] = n;
  vals[i] = int32_t(i);
  atomicAdd(counts + n, 1);   // a count: order-free
}

// per owned node: candidates into shared memory; returns the candidate count (or -1: too many)
__device__ __forceinline__ int stage_candidates(int64_t n, int nen, const int64_t* __restrict__ nadj_ptr,
                                                const int32_t* __restrict__ adj_slot,
                                                const int32_t* __restrict__ conn, int32_t* cand,
                                                int lane) {
  const int64_t k0 = nadj_ptr[n], k1 = nadj_ptr[n + 1];
  const int nc = int(k1 - k0) * nen;
  if (nc > kCandMax) return -1;
  for (int t = lane; t < nc; t += 32) {
    const int k = t / nen, b = t - k * nen;
    const int32_t slot = adj_slot[k0 + k];        // e * nen + a
    const int32_t e = slot / nen;
    cand[t] = conn[int64_t(e) * nen + b];
  }
  __syncwarp();
  return nc;
}

// first-occurrence flags of the staged candidates (a candidate is a neighbour if no equal
// candidate precedes it); returns the lane's count of first occurrences
__device__ __forceinline__ int mark_first(const int32_t* cand, uint8_t* first, int nc, int lane) {
  int cnt = 0;
  for (int t = lane; t < nc; t += 32) {
    const int32_t v = cand[t];
    bool f = true;
    for (int u = 0; u < t; ++u) f &= (cand[u] != v);
    first[t] = f ? 1 : 0;
    cnt += f ? 1 : 0;
  }
  __syncwarp();
  return cnt;
}

// pass 1: degree of each owned node (status: 1 = too many candidates, 2 = degree > 255)
__global__ void __launch_bounds__(kPatWarps * 32)
k_pat_degree(int64_t n_owned, int64_t own_b, int nen, const int64_t* __restrict__ nadj_ptr,
             const int32_t* __restrict__ adj_slot, const int32_t* __restrict__ conn,
             int64_t* __restrict__ deg, int* __restrict__ status) {
  __shared__ int32_t cands[kPatWarps][kCandMax];
  __shared__ uint8_t firsts[kPatWarps][kCandMax];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t o = int64_t(blockIdx.x) * kPatWarps + wl;
  if (o >= n_owned) return;
  int32_t* cand = cands[wl];
  const int nc = stage_candidates(o + own_b, nen, nadj_ptr, adj_slot, conn, cand, lane);
  if (nc < 0) {
    if (lane == 0) atomicOr(status, 1);
    return;
  }
  int cnt = mark_first(cand, firsts[wl], nc, lane);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
  if (lane == 0) {
    deg[o] = cnt;
    if (cnt > 255) atomicOr(status, 2);
  }
}

// adjacency offsets of the owned nodes: their slice of the node -> element CSR, rebased
__global__ void k_adj_ptr(int64_t n_owned, const int64_t* __restrict__ nadj_ptr_owned,
                          int64_t* __restrict__ adj_ptr) {
  const int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (o <= n_owned) adj_ptr[o] = nadj_ptr_owned[o] - nadj_ptr_owned[0];
}

// base, row_ptr from the exclusive scan of the degrees (nbr_ptr)
template <int NDPN>
__global__ void k_pat_rows(int64_t n_owned, const int64_t* __restrict__ nbr_ptr,
                           int64_t* __restrict__ base, int64_t* __restrict__ row_ptr) {
  const int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (o > n_owned) return;
  const int64_t b = int64_t(NDPN) * NDPN * nbr_ptr[o];
  if (o == n_owned) {
    row_ptr[n_owned * NDPN] = b;
    return;
  }
  const int64_t w = (nbr_ptr[o + 1] - nbr_ptr[o]) * NDPN;
  base[o] = b;
#pragma unroll
  for (int i = 0; i < NDPN; ++i) row_ptr[o * NDPN + i] = b + i * w;
}

// pass 2: sorted neighbour lists (local ids) and the adjacency entries of the owned nodes
__global__ void __launch_bounds__(kPatWarps * 32)
k_pat_fill(int64_t n_owned, int64_t own_b, int nen, const int64_t* __restrict__ nadj_ptr,
           const int32_t* __restrict__ adj_slot, const int32_t* __restrict__ conn,
           const int64_t* __restrict__ nbr_ptr, int32_t* __restrict__ nbr,
           AdjEntry* __restrict__ adj) {
  __shared__ int32_t cands[kPatWarps][kCandMax];
  __shared__ uint8_t firsts[kPatWarps][kCandMax];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t o = int64_t(blockIdx.x) * kPatWarps + wl;
  if (o >= n_owned) return;
  int32_t* cand = cands[wl];
  const int64_t n = o + own_b;
  const int nc = stage_candidates(n, nen, nadj_ptr, adj_slot, conn, cand, lane);
  if (nc < 0) return;
  const int64_t k0 = nadj_ptr[n];
  const int64_t a0 = nadj_ptr[n] - nadj_ptr[own_b];   // owned nodes are one contiguous range
  const uint8_t* first = firsts[wl];
  mark_first(cand, firsts[wl], nc, lane);
  for (int t = lane; t < nc; t += 32) {
    const int32_t v = cand[t];
    int rank = 0;   // distinct smaller candidates = slot in the sorted neighbour list
    for (int u = 0; u < nc; ++u) rank += (first[u] && cand[u] < v) ? 1 : 0;
    if (first[t]) nbr[nbr_ptr[o] + rank] = v;
    const int k = t / nen, b = t - k * nen;
    AdjEntry* en = adj + a0 + k;
    en->slot[b] = uint8_t(rank);
    if (b == 0) {
      const int32_t s = adj_slot[k0 + k];
      en->e = s / nen;
      en->aloc = uint8_t(s - (s / nen) * nen);
    }
  }
}

}  // namespace lgdm

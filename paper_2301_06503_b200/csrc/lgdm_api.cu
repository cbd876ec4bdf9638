// lgdm_api.cu -- the C ABI of liblgdm (include/lgdm.h): mesh setup (det J check, CSR
// pattern, element->CSR maps), state, assembly dispatch, history, residual norms, NCCL.
//
// Host-side setup is native C++ (OpenMP over nodes); every per-iteration step runs in the
// CUDA kernels of lgdm_kernels.cuh / lgdm_sweep.cuh.  There is no CPU fallback: without a
// usable CUDA device every call fails with LGDM_ERR_CUDA.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <nvtx3/nvToolsExt.h>
#include <chrono>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "../../include/lgdm.h"
#include "lgdm_kernels.cuh"
#include "lgdm_solver.cuh"
#include "lgdm_mixed.cuh"
#include "lgdm_pattern.cuh"
#include <cusolverSp.h>

using namespace lgdm;

namespace {

thread_local std::string g_err;

lgdm_status fail(lgdm_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CU(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(e_ == cudaErrorMemoryAllocation ? LGDM_ERR_OUT_OF_MEMORY : LGDM_ERR_CUDA, \
                  "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__);  \
  } while (0)

// Per-device "max dynamic shared memory" attribute: cudaFuncSetAttribute is a per-device
// setting, and one process may drive meshes on several GPUs, possibly from several threads.
template <class K> cudaError_t set_smem_attr(K kernel, size_t smem, int device) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), device);
  if (done.count(key)) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e == cudaSuccess) done.insert(key);
  return e;
}

// NCCL entry points, resolved at run time (the library does not link libnccl).
struct NcclApi {
  bool loaded = false;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  // point-to-point (ghost-dof halo exchange of the multi-rank Newton pieces) and all-gather
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
};
NcclApi g_nccl;

// cuSOLVER sparse QR (the direct solve of lgdm_solve_direct), dlopen'ed like NCCL: types from
// the headers only, no link-time dependency
struct SpSolverApi {
  bool loaded = false;
  cusolverStatus_t (*create)(cusolverSpHandle_t*);
  cusolverStatus_t (*destroy)(cusolverSpHandle_t);
  cusolverStatus_t (*setStream)(cusolverSpHandle_t, cudaStream_t);
  cusolverStatus_t (*lsvqr)(cusolverSpHandle_t, int, int, const cusparseMatDescr_t, const double*,
                            const int*, const int*, const double*, double, int, double*, int*);
  cusparseStatus_t (*createDescr)(cusparseMatDescr_t*);
  cusparseStatus_t (*destroyDescr)(cusparseMatDescr_t);
  cusparseStatus_t (*setType)(cusparseMatDescr_t, cusparseMatrixType_t);
  cusparseStatus_t (*setBase)(cusparseMatDescr_t, cusparseIndexBase_t);
};
SpSolverApi g_sps;
bool load_spsolver() {
  if (g_sps.loaded) return true;
  void* hs = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
  if (!hs) hs = dlopen("libcusolver.so", RTLD_NOW | RTLD_GLOBAL);
  void* hp = dlopen("libcusparse.so.12", RTLD_NOW | RTLD_GLOBAL);
  if (!hp) hp = dlopen("libcusparse.so", RTLD_NOW | RTLD_GLOBAL);
  if (!hs || !hp) return false;
  g_sps.create = (decltype(g_sps.create))dlsym(hs, "cusolverSpCreate");
  g_sps.destroy = (decltype(g_sps.destroy))dlsym(hs, "cusolverSpDestroy");
  g_sps.setStream = (decltype(g_sps.setStream))dlsym(hs, "cusolverSpSetStream");
  g_sps.lsvqr = (decltype(g_sps.lsvqr))dlsym(hs, "cusolverSpDcsrlsvqr");
  g_sps.createDescr = (decltype(g_sps.createDescr))dlsym(hp, "cusparseCreateMatDescr");
  g_sps.destroyDescr = (decltype(g_sps.destroyDescr))dlsym(hp, "cusparseDestroyMatDescr");
  g_sps.setType = (decltype(g_sps.setType))dlsym(hp, "cusparseSetMatType");
  g_sps.setBase = (decltype(g_sps.setBase))dlsym(hp, "cusparseSetMatIndexBase");
  g_sps.loaded = g_sps.create && g_sps.destroy && g_sps.setStream && g_sps.lsvqr && g_sps.createDescr &&
                 g_sps.destroyDescr && g_sps.setType && g_sps.setBase;
  return g_sps.loaded;
}

bool load_nccl() {
  if (g_nccl.loaded) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
  g_nccl.commInitRank = (decltype(g_nccl.commInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.allReduce = (decltype(g_nccl.allReduce))dlsym(h, "ncclAllReduce");
  g_nccl.commDestroy = (decltype(g_nccl.commDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.getErrorString = (decltype(g_nccl.getErrorString))dlsym(h, "ncclGetErrorString");
  g_nccl.getUniqueId = (decltype(g_nccl.getUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.send = (decltype(g_nccl.send))dlsym(h, "ncclSend");
  g_nccl.recv = (decltype(g_nccl.recv))dlsym(h, "ncclRecv");
  g_nccl.groupStart = (decltype(g_nccl.groupStart))dlsym(h, "ncclGroupStart");
  g_nccl.groupEnd = (decltype(g_nccl.groupEnd))dlsym(h, "ncclGroupEnd");
  g_nccl.allGather = (decltype(g_nccl.allGather))dlsym(h, "ncclAllGather");
  g_nccl.loaded = g_nccl.commInitRank && g_nccl.allReduce && g_nccl.commDestroy && g_nccl.getUniqueId &&
                  g_nccl.send && g_nccl.recv && g_nccl.groupStart && g_nccl.groupEnd && g_nccl.allGather;
  return g_nccl.loaded;
}

struct FamInfo {
  int dim, nen, ndpn, ngp, ndofe, maxdeg;
};
FamInfo fam_info(int type) {
  switch (type) {
    case LGDM_BAR2: return {1, 2, 2, 2, 4, 3};
    case LGDM_QUAD4: return {2, 4, 3, 4, 12, 9};
    case LGDM_BAR3: return {1, 3, 2, 3, 5, 5};      // mixed: nen = u nodes, ndpn = max dofs per node
    case LGDM_QUAD8: return {2, 8, 3, 9, 20, 21};
    default: return {3, 8, 4, 8, 32, 27};
  }
}

// NVTX ranges around the ABI calls (header-only NVTX3: inert unless a tool such as Nsight
// Systems is attached), so a trace shows create / assemble / step / solve phases by name
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// LGDM_CREATE_TIMING=1: per-phase wall times of lgdm_create_mesh on stderr (diagnostic)
struct PhaseTimer {
  bool on = getenv("LGDM_CREATE_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what, cudaStream_t st) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "[lgdm create] %-22s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

template <class T> cudaError_t dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) return cudaSuccess;
  return cudaMalloc((void**)p, count * sizeof(T));
}

}  // namespace

struct lgdm_mesh_s {
  int type = 0;
  FamInfo f{};
  int64_t n_nodes = 0, n_elems = 0, gid0 = 0, n_global_nodes = 0, own_b = 0, own_e = 0;
  int64_t n_owned = 0, n_rows = 0, nnz = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  DevMat dm{};
  // device buffers
  double* coords = nullptr;
  int32_t* conn = nullptr;
  double* dofs = nullptr;
  double* kappa = nullptr;
  double* k0g = nullptr;        // per-GP kappa0 / alpha (defect fields), NULL = material value
  double* alg = nullptr;
  int64_t* row_ptr = nullptr;
  int32_t* col_idx = nullptr;
  double* val = nullptr;
  double* R = nullptr;
  int64_t* nbr_ptr = nullptr;   // [n_owned+1]
  int64_t* base = nullptr;      // [n_owned] val offset of the node's first row
  int64_t* adj_ptr = nullptr;   // [n_owned+1]
  AdjEntry* adj = nullptr;      // general-path element->CSR map
  int64_t* react_buf = nullptr;  // lgdm_reaction: owned row ids + the sum (grown on demand)
  int64_t react_cap = 0;
  double* scratchK = nullptr;   // general path element blocks
  double* scratchF = nullptr;
  double* sumsq_part = nullptr; // [kSumBlocks*2]
  double* sumsq_out = nullptr;  // [2]
  double* host_pinned = nullptr;  // [2]
  double* sdv_dev = nullptr;      // staging for lgdm_update_state with a host destination
  double* sol = nullptr;          // solver work vectors [9][n_rows] + partial sums (lgdm_solve)
  double* sol_part = nullptr;
  uint8_t* fixed = nullptr;       // Dirichlet mask / increments (lgdm_apply_dirichlet)
  double* fixinc = nullptr;
  int64_t* rp_b = nullptr;        // blocked-order CSR (lgdm_get_blocked)
  int32_t* ci_b = nullptr;
  double* val_b = nullptr;
  double* R_b = nullptr;
  int64_t device_bytes = 0;
  bool have_state = false, have_kappa = false, assembled = false;
  int kernel = 0;  // 0 auto, 1 general, 2 sweep
  // structured topology (x-fastest lexicographic grid) -> sweep kernels
  bool structured = false;
  // lgdm_step: instantiated graphs of one hot-path pass, keyed by what the captured kernels read
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    const double* dofs = nullptr;
    const double* k0g = nullptr;
    const double* alg = nullptr;
    int kernel = -1, flags = -1;
    void* comm = nullptr;
    int64_t launches = 0;
  } sgraph[2];
  int sgraph_next = 0;
  bool step_warm = false;
  // graphs are captured and replayed on a private stream (the mesh stream may be the legacy
  // default stream, which cannot be captured), ordered with the mesh stream by events
  cudaStream_t gstream = nullptr;
  cudaEvent_t gev_in = nullptr, gev_out = nullptr;
  int max_deg = 0;                // largest node degree (neighbours incl. itself), equal order
  int64_t nx = 0, ny = 0, nz = 0;  // local element counts per axis (nz = layers for 3D, ny for 2D)
  int64_t launches = 0;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  bool halo_ok = false;           // slab neighbour layout validated (lgdm_set_comm)
  // halo exchange counts (dofs): sent to / received from the rank below and above
  int64_t halo_send_lo = 0, halo_recv_lo = 0, halo_send_hi = 0, halo_recv_hi = 0;
  void* sweep = nullptr;  // sweep-path state (lgdm_sweep.cuh)
  // mixed-order meshes (lgdm_mixed.cuh)
  bool mixed = false;
  int64_t n_dofs_local = 0;       // length of the dof vector (n_nodes * ndpn, or doff[n_nodes])
  std::vector<int64_t> hdoff;     // host copy of doff
  std::vector<uint8_t> hkind;     // host component index per dof
  int64_t* doff = nullptr;        // device [n_nodes+1]
  uint8_t* dkind = nullptr;       // device [ndof]
  NodeMeta* madj_ptr = nullptr;   // device [n_nodes] gather metadata
  MixAdj* madj = nullptr;         // device node -> element map of k_mixed_gather
  int32_t* gdof = nullptr;        // device [n_elems][ndofe] global dof of each element dof
  int max_row = 0;                // largest block-row (rows x width) in doubles
  // overlapped input transfer (lgdm_prefetch_dofs)
  double* dofs_back = nullptr;
  cudaStream_t cstream = nullptr;
  cudaEvent_t copy_ev = nullptr, free_ev = nullptr;
  bool prefetch_pending = false, free_ev_set = false;
  int64_t gdof0 = 0, n_global_dofs = 0;   // mixed slabs: global dof of local dof 0, total
  cusolverSpHandle_t sp_handle = nullptr;   // lgdm_solve_direct (created once per mesh)
  cusparseMatDescr_t sp_descr = nullptr;
  int32_t* rp32 = nullptr;
  int64_t* bperm = nullptr;       // blocked order of a mixed mesh: new -> old dof
  int32_t* binv = nullptr;        // old -> new dof
};

namespace {

template <class T> lgdm_status upload(lgdm_mesh m, T** dst, const T* src, size_t count) {
  CU(dalloc(dst, count));
  m->device_bytes += int64_t(count * sizeof(T));
  if (count) CU(cudaMemcpyAsync(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice, m->stream));
  return LGDM_OK;
}

lgdm_status check_launch(lgdm_mesh m, const char* what) {
  ++m->launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LGDM_ERR_CUDA, "%s launch: %s", what, cudaGetErrorString(e));
  return LGDM_OK;
}

bool validate_material(const lgdm_material* p, std::string* why) {
  const lgdm_material& m = *p;
  struct {
    bool ok;
    const char* msg;
  } checks[] = {
      {m.E > 0, "E > 0"},
      {m.nu >= 0 && m.nu < 0.5, "0 <= nu < 0.5"},
      {m.k >= 1, "k >= 1"},
      {m.kappa0 > 0, "kappa0 > 0"},
      {m.alpha > 0 && m.alpha <= 1, "0 < alpha <= 1"},
      {m.beta > 0, "beta > 0"},
      {m.h > 0, "h > 0"},
      {m.h_sigma >= 0, "h_sigma >= 0"},
      {m.c > 0, "c > 0"},
      {m.R > 0 && m.R < 1, "0 < R < 1"},
      {m.n > 0, "n > 0"},
      {m.thickness_or_area > 0, "thickness_or_area > 0"},
      {m.eq_variant == 0 || m.eq_variant == 1, "eq_variant in {0,1}"},
      {m.reserved == 0, "reserved == 0"},
  };
  for (auto& c : checks)
    if (!c.ok || std::isnan(m.E)) {
      *why = c.msg;
      return false;
    }
  return true;
}

DevMat derive(const lgdm_material& m, int dim) {
  DevMat d{};
  d.E = m.E;
  d.lam = m.E * m.nu / ((1.0 + m.nu) * (1.0 - 2.0 * m.nu));
  d.mu = m.E / (2.0 * (1.0 + m.nu));
  d.k = m.k;
  d.kappa0 = m.kappa0;
  d.alpha = m.alpha;
  d.beta = m.beta;
  d.h = m.h;
  d.hs = m.h_sigma;
  d.c = m.c;
  d.n = m.n;
  const double en = std::exp(-m.n);
  d.ga = (1.0 - m.R) / (1.0 - en);
  d.gb = (m.R - en) / (1.0 - en);
  d.t = m.thickness_or_area;
  const double k = m.k, nu = m.nu;
  d.c1 = (k - 1.0) / (2.0 * k * (1.0 - 2.0 * nu));
  d.c2 = ((k - 1.0) / (1.0 - 2.0 * nu)) * ((k - 1.0) / (1.0 - 2.0 * nu));
  d.c3 = m.eq_variant == 1 ? 2.0 * k / ((1.0 - nu) * (1.0 - nu)) : 12.0 * k / ((1.0 + nu) * (1.0 + nu));
  d.i2k = 1.0 / (2.0 * k);
  d.i4k = 1.0 / (4.0 * k);
  (void)dim;
  return d;
}

// Is conn an x-fastest structured grid (any coordinates)?  Fills nx, ny, nz.
bool detect_structured(int type, int64_t nn, int64_t ne, const int64_t* conn, int64_t* nx,
                       int64_t* ny, int64_t* nz) {
  if (ne < 1) return false;
  if (type == LGDM_BAR2) {
    for (int64_t e = 0; e < ne; ++e)
      if (conn[2 * e] != e || conn[2 * e + 1] != e + 1) return false;
    if (nn != ne + 1) return false;
    *nx = ne;
    *ny = *nz = 1;
    return true;
  }
  if (type == LGDM_QUAD4) {
    const int64_t X = conn[3] - 1;  // conn[0] = {0, 1, X+2, X+1}
    if (X < 1 || ne % X != 0) return false;
    const int64_t Y = ne / X;
    if (nn != (X + 1) * (Y + 1)) return false;
    bool ok = true;
#pragma omp parallel for reduction(&& : ok)
    for (int64_t e = 0; e < ne; ++e) {
      const int64_t i = e % X, j = e / X, b = i + (X + 1) * j;
      const int64_t* c = conn + 4 * e;
      ok = ok && c[0] == b && c[1] == b + 1 && c[2] == b + X + 2 && c[3] == b + X + 1;
    }
    if (!ok) return false;
    *nx = X;
    *ny = Y;
    *nz = 1;
    return true;
  }
  const int64_t X = conn[3] - 1;
  const int64_t SZ = conn[4];
  if (X < 1 || SZ % (X + 1) != 0) return false;
  const int64_t Y = SZ / (X + 1) - 1;
  if (Y < 1 || ne % (X * Y) != 0) return false;
  const int64_t Z = ne / (X * Y);
  if (nn != (X + 1) * (Y + 1) * (Z + 1)) return false;
  bool ok = true;
#pragma omp parallel for reduction(&& : ok)
  for (int64_t e = 0; e < ne; ++e) {
    const int64_t i = e % X, j = (e / X) % Y, k = e / (X * Y);
    const int64_t b = i + (X + 1) * j + SZ * k;
    const int64_t* c = conn + 8 * e;
    const int64_t q[4] = {b, b + 1, b + X + 2, b + X + 1};
    for (int a = 0; a < 4; ++a) ok = ok && c[a] == q[a] && c[a + 4] == q[a] + SZ;
  }
  if (!ok) return false;
  *nx = X;
  *ny = Y;
  *nz = Z;
  return true;
}

template <int D> void launch_detj(lgdm_mesh m, unsigned long long* bad) {
  const int64_t n = m->n_elems * Fam<D>::NGP;
  k_detj<D><<<unsigned((n + 255) / 256), 256, 0, m->stream>>>(m->n_elems, m->conn, m->coords, bad);
}

// ---- mixed-order elements (lgdm_mixed.cuh) ----
// Gauss points and shape functions of the two mixed families (closed forms, 3-point
// Gauss-Legendre per axis), tabulated once per mesh into constant memory.
template <int T> void mixed_tables(MShape<T>& S) {
  using F = MFam<T>;
  const double p[3] = {-std::sqrt(0.6), 0.0, std::sqrt(0.6)};
  const double q[3] = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
  for (int g = 0; g < F::NGP; ++g) {
    const int gx = g % 3, gy = g / 3;
    const double x = p[gx];
    if constexpr (F::DIM == 1) {
      S.w[g] = q[gx];
      S.Nu[g][0] = 0.5 * x * (x - 1.0);
      S.Nu[g][1] = 0.5 * x * (x + 1.0);
      S.Nu[g][2] = (1.0 - x) * (1.0 + x);
      S.dNu[g][0][0] = x - 0.5;
      S.dNu[g][1][0] = x + 0.5;
      S.dNu[g][2][0] = -2.0 * x;
      S.Ne[g][0] = 0.5 * (1.0 - x);
      S.Ne[g][1] = 0.5 * (1.0 + x);
      S.dNe[g][0][0] = -0.5;
      S.dNe[g][1][0] = 0.5;
    } else {
      const double y = p[gy];
      S.w[g] = q[gx] * q[gy];
      static const int cx[4] = {-1, 1, 1, -1}, cy[4] = {-1, -1, 1, 1};
      for (int a = 0; a < 4; ++a) {   // serendipity corners and bilinear ebar
        const double sx = cx[a], sy = cy[a];
        const double fx = 1.0 + sx * x, fy = 1.0 + sy * y;
        S.Nu[g][a] = 0.25 * fx * fy * (sx * x + sy * y - 1.0);
        S.dNu[g][a][0] = 0.25 * sx * fy * (2.0 * sx * x + sy * y);
        S.dNu[g][a][1] = 0.25 * sy * fx * (sx * x + 2.0 * sy * y);
        S.Ne[g][a] = 0.25 * fx * fy;
        S.dNe[g][a][0] = 0.25 * sx * fy;
        S.dNe[g][a][1] = 0.25 * sy * fx;
      }
      // midsides: (0,-1), (1,0), (0,1), (-1,0)
      const double bx = (1.0 - x) * (1.0 + x), by = (1.0 - y) * (1.0 + y);
      S.Nu[g][4] = 0.5 * bx * (1.0 - y);  S.dNu[g][4][0] = -x * (1.0 - y);  S.dNu[g][4][1] = -0.5 * bx;
      S.Nu[g][5] = 0.5 * (1.0 + x) * by;  S.dNu[g][5][0] = 0.5 * by;        S.dNu[g][5][1] = -y * (1.0 + x);
      S.Nu[g][6] = 0.5 * bx * (1.0 + y);  S.dNu[g][6][0] = -x * (1.0 + y);  S.dNu[g][6][1] = 0.5 * bx;
      S.Nu[g][7] = 0.5 * (1.0 - x) * by;  S.dNu[g][7][0] = -0.5 * by;       S.dNu[g][7][1] = -y * (1.0 - x);
    }
  }
}

template <int T> lgdm_status upload_tables(lgdm_mesh m) {
  MShape<T> S{};
  mixed_tables<T>(S);
  if constexpr (T == 4) CU(cudaMemcpyToSymbolAsync(c_shape4, &S, sizeof(S), 0, cudaMemcpyHostToDevice, m->stream));
  else CU(cudaMemcpyToSymbolAsync(c_shape5, &S, sizeof(S), 0, cudaMemcpyHostToDevice, m->stream));
  CU(cudaStreamSynchronize(m->stream));   // S is on the host stack
  return LGDM_OK;
}

lgdm_status create_mixed(lgdm_elem_type type, int64_t n_nodes, const double* coords, int64_t n_elems,
                         const int64_t* conn, const lgdm_material* mat, int64_t gid0, int64_t n_global,
                         int64_t own_b, int64_t own_e, int64_t gdof0, int64_t n_global_dofs,
                         int device, void* stream, lgdm_mesh* out) {
  const FamInfo f = fam_info(type);
  const int T = int(type);
  const int nene = T == LGDM_BAR3 ? 2 : 4;
  if (!coords || !conn || !mat) return fail(LGDM_ERR_INVALID_ARGUMENT, "NULL input pointer");
  if (n_nodes < 2 || n_elems < 1 || n_nodes >= (int64_t(1) << 30))
    return fail(LGDM_ERR_INVALID_ARGUMENT, "bad sizes n_nodes=%lld n_elems=%lld", (long long)n_nodes,
                (long long)n_elems);
  if (gid0 < 0 || n_global < gid0 + n_nodes || !(0 <= own_b && own_b < own_e && own_e <= n_nodes))
    return fail(LGDM_ERR_INVALID_ARGUMENT, "node ranges inconsistent");
  if (gdof0 < 0 || (gid0 == 0 && n_global == n_nodes && gdof0 != 0))
    return fail(LGDM_ERR_INVALID_ARGUMENT, "global dof offset inconsistent");
  std::string why;
  if (!validate_material(mat, &why)) return fail(LGDM_ERR_INVALID_ARGUMENT, "material: %s", why.c_str());
  std::vector<uint8_t> kind(n_nodes, 0);   // 1 corner (ebar), 2 midside
  for (int64_t e = 0; e < n_elems; ++e)
    for (int a = 0; a < f.nen; ++a) {
      const int64_t n = conn[e * f.nen + a];
      if (n < 0 || n >= n_nodes)
        return fail(LGDM_ERR_INVALID_ARGUMENT, "conn[%lld] = %lld out of range", (long long)(e * f.nen + a), (long long)n);
      const uint8_t k = a < nene ? 1 : 2;
      if (kind[n] && kind[n] != k)
        return fail(LGDM_ERR_INVALID_ARGUMENT, "node %lld is a corner of one element and a midside node of another", (long long)n);
      kind[n] = k;
    }
  std::vector<int64_t> doff(n_nodes + 1, 0);
  for (int64_t n = 0; n < n_nodes; ++n) {
    if (!kind[n]) return fail(LGDM_ERR_INVALID_ARGUMENT, "node %lld belongs to no element", (long long)n);
    doff[n + 1] = doff[n] + (kind[n] == 1 ? f.dim + 1 : f.dim);
  }
  const int64_t ndof = doff[n_nodes];
  if (n_global_dofs < 0) n_global_dofs = gdof0 + ndof;   // whole mesh
  if (n_global_dofs < gdof0 + ndof)
    return fail(LGDM_ERR_INVALID_ARGUMENT, "n_global_dofs < global dof offset + local dofs");
  if (n_global_dofs >= (int64_t(1) << 31)) return fail(LGDM_ERR_INVALID_ARGUMENT, "dof count exceeds int32 col_idx");
  const int64_t no = own_e - own_b, r_b = doff[own_b], nrow = doff[own_e] - doff[own_b];
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(LGDM_ERR_CUDA, "no CUDA device available (liblgdm has no CPU path)");
  if (device < 0 || device >= ndev) return fail(LGDM_ERR_INVALID_ARGUMENT, "bad device %d", device);
  CU(cudaSetDevice(device));
  lgdm_mesh m = new lgdm_mesh_s();
  m->type = type;
  m->f = f;
  m->mixed = true;
  m->n_nodes = n_nodes;
  m->n_elems = n_elems;
  m->gid0 = gid0;
  m->n_global_nodes = n_global;
  m->own_b = own_b;
  m->own_e = own_e;
  m->n_owned = no;
  m->n_rows = nrow;
  m->n_dofs_local = ndof;
  m->gdof0 = gdof0;
  m->n_global_dofs = n_global_dofs;
  m->device = device;
  m->stream = (cudaStream_t)stream;
  m->dm = derive(*mat, f.dim);
  m->hdoff = doff;
  m->hkind.resize(ndof);
  for (int64_t n = 0; n < n_nodes; ++n)
    for (int64_t r = doff[n]; r < doff[n + 1]; ++r) m->hkind[r] = uint8_t(r - doff[n]);
  auto bail = [&](lgdm_status s) {
    std::string keep = g_err;
    lgdm_destroy(m);
    g_err = keep;
    return s;
  };
  lgdm_status s;
  std::vector<int32_t> conn32(size_t(n_elems) * f.nen);
#pragma omp parallel for if (conn32.size() > (size_t(1) << 20))
  for (int64_t i = 0; i < int64_t(conn32.size()); ++i) conn32[i] = int32_t(conn[i]);
  if ((s = upload(m, &m->coords, coords, size_t(n_nodes) * f.dim)) != LGDM_OK) return bail(s);
  if ((s = upload(m, &m->conn, conn32.data(), conn32.size())) != LGDM_OK) return bail(s);
  if ((s = upload(m, &m->doff, doff.data(), doff.size())) != LGDM_OK) return bail(s);
  if ((s = upload(m, &m->dkind, m->hkind.data(), m->hkind.size())) != LGDM_OK) return bail(s);
  if ((s = (T == 4 ? upload_tables<4>(m) : upload_tables<5>(m))) != LGDM_OK) return bail(s);
  // det J > 0 at every GP
  unsigned long long* bad = nullptr;
  if (cudaMalloc(&bad, sizeof(unsigned long long)) != cudaSuccess)
    return bail(fail(LGDM_ERR_OUT_OF_MEMORY, "cudaMalloc"));
  cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), m->stream);
  const unsigned gb = unsigned((n_elems * f.ngp + 255) / 256);
  if (T == 4) k_mixed_detj<4><<<gb, 256, 0, m->stream>>>(n_elems, m->conn, m->coords, bad);
  else k_mixed_detj<5><<<gb, 256, 0, m->stream>>>(n_elems, m->conn, m->coords, bad);
  if ((s = check_launch(m, "k_mixed_detj")) != LGDM_OK) { cudaFree(bad); return bail(s); }
  unsigned long long hbad = 0;
  cudaMemcpyAsync(&hbad, bad, sizeof(hbad), cudaMemcpyDeviceToHost, m->stream);
  cudaError_t ce = cudaStreamSynchronize(m->stream);
  cudaFree(bad);
  if (ce != cudaSuccess) return bail(fail(LGDM_ERR_CUDA, "det J check: %s", cudaGetErrorString(ce)));
  if (hbad != ~0ull)
    return bail(fail(LGDM_ERR_INVERTED_ELEMENT, "det J <= 0 in element %lld at Gauss point %d",
                     (long long)(hbad / f.ngp), int(hbad % f.ngp)));
  // pattern (reading R-PAT): node adjacency, block-rows of variable width
  std::vector<int64_t> nadj(n_nodes + 1, 0);
  for (int64_t i = 0; i < n_elems * f.nen; ++i) ++nadj[conn[i] + 1];
  for (int64_t n = 0; n < n_nodes; ++n) nadj[n + 1] += nadj[n];
  std::vector<int32_t> adj_e(nadj[n_nodes]);
  std::vector<uint8_t> adj_a(nadj[n_nodes]);
  {
    std::vector<int64_t> fillp(nadj.begin(), nadj.end() - 1);
    for (int64_t e = 0; e < n_elems; ++e)
      for (int a = 0; a < f.nen; ++a) {
        const int64_t n = conn[e * f.nen + a];
        adj_e[fillp[n]] = int32_t(e);
        adj_a[fillp[n]] = uint8_t(a);
        ++fillp[n];
      }
  }
  std::vector<int32_t> width(n_nodes);
  std::vector<std::vector<int32_t>> nbs(n_nodes);
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < n_nodes; ++n) {
    std::vector<int32_t>& nb = nbs[n];
    for (int64_t k = nadj[n]; k < nadj[n + 1]; ++k)
      for (int b = 0; b < f.nen; ++b) nb.push_back(int32_t(conn[int64_t(adj_e[k]) * f.nen + b]));
    std::sort(nb.begin(), nb.end());
    nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
    int32_t w = 0;
    for (int32_t b : nb) w += int32_t(doff[b + 1] - doff[b]);
    width[n] = w;
  }
  // rows of the owned nodes only (row r = local dof r_b + r); columns are global dof ids
  std::vector<int64_t> row_ptr(nrow + 1, 0);
  int64_t pos = 0;
  int max_row = 0;
  for (int64_t n = own_b; n < own_e; ++n) {
    const int nr = int(doff[n + 1] - doff[n]);
    for (int i = 0; i < nr; ++i) {
      row_ptr[doff[n] - r_b + i] = pos;
      pos += width[n];
    }
    max_row = std::max(max_row, nr * width[n]);
  }
  row_ptr[nrow] = pos;
  m->nnz = pos;
  m->max_row = max_row;
  if (pos >= (int64_t(1) << 40)) return bail(fail(LGDM_ERR_INVALID_ARGUMENT, "pattern too large"));
  std::vector<int32_t> col(pos);
  std::vector<int64_t> madj_ptr(no + 1);
  for (int64_t o = 0; o < no; ++o) madj_ptr[o + 1] = madj_ptr[o] + (nadj[own_b + o + 1] - nadj[own_b + o]);
  std::vector<MixAdj> madj(madj_ptr[no]);
#pragma omp parallel for schedule(static)
  for (int64_t o = 0; o < no; ++o) {
    const int64_t n = own_b + o;
    const std::vector<int32_t>& nb = nbs[n];
    std::vector<int32_t> coff(nb.size());
    int32_t c = 0;
    for (size_t s2 = 0; s2 < nb.size(); ++s2) {
      coff[s2] = c;
      c += int32_t(doff[nb[s2] + 1] - doff[nb[s2]]);
    }
    const int nr = int(doff[n + 1] - doff[n]);
    for (int i = 0; i < nr; ++i) {
      int64_t p = row_ptr[doff[n] - r_b + i];
      for (int32_t b : nb)
        for (int64_t d = doff[b]; d < doff[b + 1]; ++d) col[p++] = int32_t(gdof0 + d);
    }
    for (int64_t k = nadj[n]; k < nadj[n + 1]; ++k) {
      MixAdj en{};
      en.e = adj_e[k];
      en.aloc = adj_a[k];
      for (int b = 0; b < f.nen; ++b) {
        const int32_t nbn = int32_t(conn[int64_t(en.e) * f.nen + b]);
        en.coff[b] = coff[std::lower_bound(nb.begin(), nb.end(), nbn) - nb.begin()];
      }
      madj[madj_ptr[o] + (k - nadj[n])] = en;
    }
  }
  if ((s = upload(m, &m->row_ptr, row_ptr.data(), row_ptr.size())) != LGDM_OK) return bail(s);
  if ((s = upload(m, &m->col_idx, col.data(), col.size())) != LGDM_OK) return bail(s);
  std::vector<NodeMeta> meta(no);
  for (int64_t o = 0; o < no; ++o) {
    const int64_t n = own_b + o;
    const int nr = int(doff[n + 1] - doff[n]);
    meta[o] = NodeMeta{row_ptr[doff[n] - r_b], doff[n] - r_b, madj_ptr[o], width[n], int16_t(nr),
                       int16_t(madj_ptr[o + 1] - madj_ptr[o])};
    if (madj_ptr[o + 1] - madj_ptr[o] > 32767) return bail(fail(LGDM_ERR_INVALID_ARGUMENT, "node %lld has too many elements", (long long)n));
  }
  if ((s = upload(m, &m->madj_ptr, meta.data(), meta.size())) != LGDM_OK) return bail(s);
  if ((s = upload(m, &m->madj, madj.data(), madj.size())) != LGDM_OK) return bail(s);
  {
    const int nd = f.ndofe, dim = f.dim;
    std::vector<int32_t> gd(size_t(n_elems) * nd);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n_elems; ++e)
      for (int c = 0; c < nd; ++c) {
        const int a = c < nene * (dim + 1) ? c / (dim + 1) : nene + (c - nene * (dim + 1)) / dim;
        const int comp = c < nene * (dim + 1) ? c % (dim + 1) : (c - nene * (dim + 1)) % dim;
        gd[size_t(e) * nd + c] = int32_t(doff[conn[e * f.nen + a]] + comp);
      }
    if ((s = upload(m, &m->gdof, gd.data(), gd.size())) != LGDM_OK) return bail(s);
  }
  if (dalloc(&m->val, size_t(m->nnz)) != cudaSuccess || dalloc(&m->R, size_t(nrow)) != cudaSuccess ||
      dalloc(&m->dofs, size_t(ndof)) != cudaSuccess || dalloc(&m->kappa, size_t(n_elems) * f.ngp) != cudaSuccess ||
      dalloc(&m->sumsq_part, size_t(2 * kSumBlocks)) != cudaSuccess || dalloc(&m->sumsq_out, 2) != cudaSuccess ||
      cudaMallocHost(&m->host_pinned, 2 * sizeof(double)) != cudaSuccess)
    return bail(fail(LGDM_ERR_OUT_OF_MEMORY, "cudaMalloc (nnz=%lld)", (long long)m->nnz));
  m->device_bytes += m->nnz * 8 + ndof * 16 + n_elems * f.ngp * 8;
  ce = cudaStreamSynchronize(m->stream);   // host staging vectors go out of scope
  if (ce != cudaSuccess) return bail(fail(LGDM_ERR_CUDA, "create: %s", cudaGetErrorString(ce)));
  *out = m;
  return LGDM_OK;
}

template <int T> lgdm_status assemble_mixed(lgdm_mesh m) {
  using F = MFam<T>;
  constexpr int WPB = 4, GW = 8;
  if (!m->scratchK) {
    CU(dalloc(&m->scratchK, size_t(m->n_elems) * F::NDOFE * F::NDOFE));
    CU(dalloc(&m->scratchF, size_t(m->n_elems) * F::NDOFE));
    m->device_bytes += m->n_elems * (F::NDOFE * F::NDOFE + F::NDOFE) * 8;
  }
  const size_t smem = sizeof(double) * (size_t(WPB) * MSmem<T>::SIZE + ((sizeof(MShape<T>) / 8 + 1) & ~size_t(1)));
  CU(set_smem_attr(k_mixed_blocks<T, WPB>, smem, m->device));
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mixed_blocks<T, WPB>, WPB * 32, smem);
  const int64_t nb = (m->n_elems + WPB - 1) / WPB;
  const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>(nb, int64_t(nsm) * std::max(per_sm, 1))));
  k_mixed_blocks<T, WPB><<<grid, WPB * 32, smem, m->stream>>>(m->dm, m->n_elems, m->conn, m->coords, m->gdof,
                                                              m->dofs, m->kappa, m->k0g, m->alg,
                                                              m->scratchK, m->scratchF);
  lgdm_status s = check_launch(m, "k_mixed_blocks");
  if (s != LGDM_OK) return s;
  const size_t gsm = sizeof(double) * size_t(GW) * (size_t(m->max_row) + MGStage<T>::SIZE);
  if (gsm > 48 * 1024) CU(set_smem_attr(k_mixed_gather<T, GW>, gsm, m->device));
  const int64_t gn = (m->n_owned + GW - 1) / GW;
  k_mixed_gather<T, GW><<<unsigned(std::min<int64_t>(gn, int64_t(nsm) * 16)), GW * 32, gsm, m->stream>>>(
      m->n_owned, m->madj_ptr, m->madj, m->scratchK, m->scratchF, m->max_row, m->val, m->R);
  return check_launch(m, "k_mixed_gather");
}

}  // namespace

#include "lgdm_sweep.cuh"

namespace {

// SURVEY 8a row A0 on the GPU: node adjacency, CSR row_ptr / base / col_idx and the element ->
// block-row slot map of the owned nodes (lgdm_pattern.cuh), from the device connectivity.
lgdm_status build_pattern(lgdm_mesh m, int64_t global_node_offset) {
  const FamInfo& f = m->f;
  const int nen = f.nen;
  const int64_t nn = m->n_nodes, ne = m->n_elems, no = m->n_owned, nsl = ne * nen;
  if (nsl >= (int64_t(1) << 31) || nn + 1 >= (int64_t(1) << 31))   // CUB item counts are int
    return fail(LGDM_ERR_UNSUPPORTED, "n_elems * nen or n_nodes + 1 >= 2^31");
  cudaStream_t st = m->stream;
  // scratch (freed at the end)
  int32_t *keys = nullptr, *vals = nullptr, *keys2 = nullptr, *adj_slot = nullptr, *counts = nullptr,
          *nbr = nullptr;
  int64_t *nadj_ptr = nullptr, *deg = nullptr;
  int* status = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  lgdm_status rc = LGDM_OK;
  auto cleanup = [&]() {
    cudaFree(keys); cudaFree(vals); cudaFree(keys2); cudaFree(adj_slot); cudaFree(counts);
    cudaFree(nbr); cudaFree(nadj_ptr); cudaFree(deg); cudaFree(status); cudaFree(tmp);
  };
#define PCU(call)                                                                         \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      rc = fail(e_ == cudaErrorMemoryAllocation ? LGDM_ERR_OUT_OF_MEMORY : LGDM_ERR_CUDA,  \
                "pattern: %s: %s", #call, cudaGetErrorString(e_));                        \
      cleanup();                                                                          \
      return rc;                                                                          \
    }                                                                                     \
  } while (0)
  PCU(cudaMalloc(&keys, nsl * 4));
  PCU(cudaMalloc(&vals, nsl * 4));
  PCU(cudaMalloc(&keys2, nsl * 4));
  PCU(cudaMalloc(&adj_slot, nsl * 4));
  PCU(cudaMalloc(&counts, (nn + 1) * 4));
  PCU(cudaMalloc(&nadj_ptr, (nn + 1) * 8));
  PCU(cudaMalloc(&deg, (no + 1) * 8));
  PCU(cudaMalloc(&status, sizeof(int)));
  PCU(cudaMemsetAsync(counts, 0, (nn + 1) * 4, st));
  PCU(cudaMemsetAsync(deg, 0, (no + 1) * 8, st));
  PCU(cudaMemsetAsync(status, 0, sizeof(int), st));
  k_adj_keys<<<unsigned((nsl + 255) / 256), 256, 0, st>>>(nsl, m->conn, keys, vals, counts);
  ++m->launches;
  // node -> element slots, stable by slot index (= ascending element id)
  int end_bit = 1;
  while ((int64_t(1) << end_bit) < nn) ++end_bit;
  size_t need = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, need, keys, keys2, vals, adj_slot, int(nsl), 0, end_bit, st);
  tmp_bytes = std::max(tmp_bytes, need);
  cub::DeviceScan::ExclusiveSum(nullptr, need, counts, nadj_ptr, int(nn + 1), st);
  tmp_bytes = std::max(tmp_bytes, need);
  cub::DeviceScan::ExclusiveSum(nullptr, need, deg, deg, int(no + 1), st);
  tmp_bytes = std::max(tmp_bytes, need);
  PCU(cudaMalloc(&tmp, tmp_bytes));
  PCU(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, vals, adj_slot, int(nsl), 0, end_bit, st));
  PCU(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, nadj_ptr, int(nn + 1), st));
  m->launches += 4;
  // pass 1: degrees -> nbr_ptr (exclusive scan in place), base, row_ptr
  const unsigned pb = unsigned((no + kPatWarps - 1) / kPatWarps);
  k_pat_degree<<<pb, kPatWarps * 32, 0, st>>>(no, m->own_b, nen, nadj_ptr, adj_slot, m->conn, deg, status);
  PCU(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, deg, deg, int(no + 1), st));
  int hstat = 0;
  int64_t nbr_total = 0, adj_lo = 0, adj_hi = 0;
  PCU(cudaMemcpyAsync(&hstat, status, sizeof(int), cudaMemcpyDeviceToHost, st));
  PCU(cudaMemcpyAsync(&nbr_total, deg + no, 8, cudaMemcpyDeviceToHost, st));
  PCU(cudaMemcpyAsync(&adj_lo, nadj_ptr + m->own_b, 8, cudaMemcpyDeviceToHost, st));
  PCU(cudaMemcpyAsync(&adj_hi, nadj_ptr + m->own_e, 8, cudaMemcpyDeviceToHost, st));
  PCU(cudaStreamSynchronize(st));
  m->launches += 3;
  if (hstat != 0) {
    cleanup();
    return fail(LGDM_ERR_UNSUPPORTED, "%s", (hstat & 1) ? "a node has more than 1024 candidate neighbours"
                                                        : "a node has more than 255 neighbours");
  }
  m->nnz = int64_t(f.ndpn) * f.ndpn * nbr_total;
  if (dalloc(&m->nbr_ptr, size_t(no + 1)) != cudaSuccess || dalloc(&m->base, size_t(no)) != cudaSuccess ||
      dalloc(&m->row_ptr, size_t(m->n_rows + 1)) != cudaSuccess ||
      dalloc(&m->adj_ptr, size_t(no + 1)) != cudaSuccess ||
      cudaMalloc(&m->adj, size_t(adj_hi - adj_lo) * sizeof(AdjEntry)) != cudaSuccess ||
      cudaMalloc(&nbr, size_t(nbr_total) * 4) != cudaSuccess) {
    cleanup();
    return fail(LGDM_ERR_OUT_OF_MEMORY, "cudaMalloc pattern");
  }
  m->device_bytes += (no + 1) * 24 + no * 8 + (m->n_rows + 1) * 8 + (adj_hi - adj_lo) * int64_t(sizeof(AdjEntry));
  PCU(cudaMemcpyAsync(m->nbr_ptr, deg, (no + 1) * 8, cudaMemcpyDeviceToDevice, st));
  const unsigned rb = unsigned((no + 1 + 255) / 256);
  if (f.ndpn == 2) k_pat_rows<2><<<rb, 256, 0, st>>>(no, m->nbr_ptr, m->base, m->row_ptr);
  else if (f.ndpn == 3) k_pat_rows<3><<<rb, 256, 0, st>>>(no, m->nbr_ptr, m->base, m->row_ptr);
  else k_pat_rows<4><<<rb, 256, 0, st>>>(no, m->nbr_ptr, m->base, m->row_ptr);
  k_adj_ptr<<<rb, 256, 0, st>>>(no, nadj_ptr + m->own_b, m->adj_ptr);
  // pass 2: sorted neighbour lists and adjacency entries
  k_pat_fill<<<pb, kPatWarps * 32, 0, st>>>(no, m->own_b, nen, nadj_ptr, adj_slot, m->conn,
                                           m->nbr_ptr, nbr, m->adj);
  m->launches += 3;
  if (dalloc(&m->col_idx, size_t(m->nnz)) != cudaSuccess || dalloc(&m->val, size_t(m->nnz)) != cudaSuccess ||
      dalloc(&m->R, size_t(m->n_rows)) != cudaSuccess) {
    cleanup();
    return fail(LGDM_ERR_OUT_OF_MEMORY, "cudaMalloc CSR (nnz=%lld)", (long long)m->nnz);
  }
  m->device_bytes += m->nnz * (4 + 8) + m->n_rows * 8;
  {
    const unsigned blocks = unsigned((no * 32 + 255) / 256);
    if (f.ndpn == 2) k_cols<2><<<blocks, 256, 0, st>>>(no, m->nbr_ptr, nbr, m->base, global_node_offset, m->col_idx);
    else if (f.ndpn == 3) k_cols<3><<<blocks, 256, 0, st>>>(no, m->nbr_ptr, nbr, m->base, global_node_offset, m->col_idx);
    else k_cols<4><<<blocks, 256, 0, st>>>(no, m->nbr_ptr, nbr, m->base, global_node_offset, m->col_idx);
    ++m->launches;
  }
  // the largest degree sizes the general path's per-warp block-row buffer
  {
    std::vector<int64_t> hp(no + 1);
    // (a host copy of nbr_ptr: one int64 per owned node, read once)
    PCU(cudaMemcpyAsync(hp.data(), m->nbr_ptr, (no + 1) * 8, cudaMemcpyDeviceToHost, st));
    PCU(cudaStreamSynchronize(st));
    int64_t mx = 0;
    for (int64_t o = 0; o < no; ++o) mx = std::max(mx, hp[o + 1] - hp[o]);
    m->max_deg = int(mx);
  }
  lgdm_status cs = check_launch(m, "pattern");
  cleanup();
#undef PCU
  return cs;
}

}  // namespace

extern "C" {

const char* lgdm_last_error(void) { return g_err.c_str(); }

lgdm_status lgdm_create_mesh(lgdm_elem_type type, int64_t n_nodes, const double* coords,
                             int64_t n_elems, const int64_t* conn, const lgdm_material* mat,
                             int64_t global_node_offset, int64_t n_global_nodes,
                             int64_t owned_node_begin, int64_t owned_node_end, int device,
                             void* cuda_stream, lgdm_mesh* out) {
  const NvtxRange nvtx_range("lgdm_create_mesh");
  PhaseTimer pt;
  if (!out) return fail(LGDM_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if ((type == LGDM_BAR3 || type == LGDM_QUAD8) && global_node_offset != 0)
    return fail(LGDM_ERR_INVALID_ARGUMENT, "mixed-order slabs need their global dof offset: use lgdm_create_mesh_mixed");
  if (type == LGDM_BAR3 || type == LGDM_QUAD8)
    return create_mixed(type, n_nodes, coords, n_elems, conn, mat, global_node_offset,
                        n_global_nodes, owned_node_begin, owned_node_end, 0, -1, device,
                        cuda_stream, out);
  if (type != LGDM_BAR2 && type != LGDM_QUAD4 && type != LGDM_HEX8)
    return fail(LGDM_ERR_INVALID_ARGUMENT, "unknown element type %d", int(type));
  if (!coords || !conn || !mat) return fail(LGDM_ERR_INVALID_ARGUMENT, "NULL input pointer");
  if (n_nodes < 2 || n_elems < 1 || n_nodes >= (int64_t(1) << 31))
    return fail(LGDM_ERR_INVALID_ARGUMENT, "bad sizes n_nodes=%lld n_elems=%lld",
                (long long)n_nodes, (long long)n_elems);
  if (global_node_offset < 0 || n_global_nodes < global_node_offset + n_nodes)
    return fail(LGDM_ERR_INVALID_ARGUMENT, "global node range inconsistent");
  if (!(0 <= owned_node_begin && owned_node_begin < owned_node_end && owned_node_end <= n_nodes))
    return fail(LGDM_ERR_INVALID_ARGUMENT, "owned node range [%lld,%lld) invalid",
                (long long)owned_node_begin, (long long)owned_node_end);
  const FamInfo f = fam_info(type);
  if ((n_global_nodes * f.ndpn) >= (int64_t(1) << 31))
    return fail(LGDM_ERR_INVALID_ARGUMENT, "global dof count exceeds int32 col_idx");
  std::string why;
  if (!validate_material(mat, &why)) return fail(LGDM_ERR_INVALID_ARGUMENT, "material: %s", why.c_str());
  {
    int64_t bad_i = INT64_MAX;   // smallest offending index (deterministic message)
#pragma omp parallel for reduction(min : bad_i) if (n_elems * f.nen > (1 << 20))
    for (int64_t i = 0; i < n_elems * f.nen; ++i)
      if (conn[i] < 0 || conn[i] >= n_nodes) bad_i = std::min(bad_i, i);
    if (bad_i != INT64_MAX)
      return fail(LGDM_ERR_INVALID_ARGUMENT, "conn[%lld] = %lld out of range", (long long)bad_i,
                  (long long)conn[bad_i]);
  }
  pt.mark("validate", nullptr);

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(LGDM_ERR_CUDA, "no CUDA device available (liblgdm has no CPU path)");
  if (device < 0 || device >= ndev) return fail(LGDM_ERR_INVALID_ARGUMENT, "bad device %d", device);
  CU(cudaSetDevice(device));

  lgdm_mesh m = new lgdm_mesh_s();
  m->type = type;
  m->f = f;
  m->n_nodes = n_nodes;
  m->n_elems = n_elems;
  m->gid0 = global_node_offset;
  m->n_global_nodes = n_global_nodes;
  m->own_b = owned_node_begin;
  m->own_e = owned_node_end;
  m->n_owned = owned_node_end - owned_node_begin;
  m->n_rows = m->n_owned * f.ndpn;
  m->n_dofs_local = n_nodes * f.ndpn;
  m->device = device;
  m->stream = (cudaStream_t)cuda_stream;
  m->dm = derive(*mat, f.dim);

  auto bail = [&](lgdm_status s) {
    std::string keep = g_err;
    lgdm_destroy(m);
    g_err = keep;
    return s;
  };
  lgdm_status s;

  // ---- coordinates and connectivity (int32 local ids on device) ----
  std::vector<int32_t> conn32(size_t(n_elems) * f.nen);
#pragma omp parallel for if (conn32.size() > (size_t(1) << 20))
  for (int64_t i = 0; i < int64_t(conn32.size()); ++i) conn32[i] = int32_t(conn[i]);
  if ((s = upload(m, &m->coords, coords, size_t(n_nodes) * f.dim)) != LGDM_OK) return bail(s);
  if ((s = upload(m, &m->conn, conn32.data(), conn32.size())) != LGDM_OK) return bail(s);
  pt.mark("conn32 + upload", m->stream);

  // ---- det J > 0 at every GP ----
  unsigned long long* bad = nullptr;
  if (cudaMalloc(&bad, sizeof(unsigned long long)) != cudaSuccess)
    return bail(fail(LGDM_ERR_OUT_OF_MEMORY, "cudaMalloc"));
  cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), m->stream);
  if (f.dim == 1) launch_detj<1>(m, bad);
  else if (f.dim == 2) launch_detj<2>(m, bad);
  else launch_detj<3>(m, bad);
  if ((s = check_launch(m, "k_detj")) != LGDM_OK) { cudaFree(bad); return bail(s); }
  unsigned long long hbad = 0;
  cudaMemcpyAsync(&hbad, bad, sizeof(hbad), cudaMemcpyDeviceToHost, m->stream);
  cudaError_t ce = cudaStreamSynchronize(m->stream);
  cudaFree(bad);
  if (ce != cudaSuccess) return bail(fail(LGDM_ERR_CUDA, "det J check: %s", cudaGetErrorString(ce)));
  if (hbad != ~0ull)
    return bail(fail(LGDM_ERR_INVERTED_ELEMENT, "det J <= 0 in element %lld at Gauss point %d",
                     (long long)(hbad / f.ngp), int(hbad % f.ngp)));
  pt.mark("det J", m->stream);

  // ---- pattern (reading R-PAT) and element maps, built on the GPU (lgdm_pattern.cuh) ----
  if ((s = build_pattern(m, global_node_offset)) != LGDM_OK) return bail(s);
  pt.mark("pattern", m->stream);
  // ---- state, reductions ----
  if (dalloc(&m->dofs, size_t(n_nodes) * f.ndpn) != cudaSuccess ||
      dalloc(&m->kappa, size_t(n_elems) * f.ngp) != cudaSuccess ||
      dalloc(&m->sumsq_part, size_t(2 * kSumBlocks)) != cudaSuccess ||
      dalloc(&m->sumsq_out, 2) != cudaSuccess ||
      cudaMallocHost(&m->host_pinned, 2 * sizeof(double)) != cudaSuccess) {
    return bail(fail(LGDM_ERR_OUT_OF_MEMORY, "cudaMalloc state"));
  }
  m->device_bytes += (n_nodes * f.ndpn + n_elems * f.ngp) * 8;
  m->structured = detect_structured(type, n_nodes, n_elems, conn, &m->nx, &m->ny, &m->nz);
  pt.mark("state + structure", m->stream);
  ce = cudaStreamSynchronize(m->stream);
  if (ce != cudaSuccess) return bail(fail(LGDM_ERR_CUDA, "create: %s", cudaGetErrorString(ce)));
  *out = m;
  return LGDM_OK;
}

lgdm_status lgdm_create_mesh_mixed(lgdm_elem_type type, int64_t n_nodes, const double* coords,
                                   int64_t n_elems, const int64_t* conn, const lgdm_material* mat,
                                   int64_t global_node_offset, int64_t n_global_nodes,
                                   int64_t owned_node_begin, int64_t owned_node_end,
                                   int64_t global_dof_offset, int64_t n_global_dofs, int device,
                                   void* cuda_stream, lgdm_mesh* out) {
  const NvtxRange nvtx_range("lgdm_create_mesh_mixed");
  if (!out) return fail(LGDM_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (type != LGDM_BAR3 && type != LGDM_QUAD8)
    return fail(LGDM_ERR_INVALID_ARGUMENT, "lgdm_create_mesh_mixed takes LGDM_BAR3 / LGDM_QUAD8");
  return create_mixed(type, n_nodes, coords, n_elems, conn, mat, global_node_offset, n_global_nodes,
                      owned_node_begin, owned_node_end, global_dof_offset, n_global_dofs, device,
                      cuda_stream, out);
}

lgdm_status lgdm_set_state(lgdm_mesh m, const double* dofs, int64_t n_dofs, const double* kappa,
                           int64_t n_kappa, int src_on_device) {
  if (!m) return fail(LGDM_ERR_INVALID_ARGUMENT, "mesh is NULL");
  if (!dofs) return fail(LGDM_ERR_INVALID_ARGUMENT, "dofs is NULL");
  if (n_dofs != m->n_dofs_local)
    return fail(LGDM_ERR_INVALID_STATE, "n_dofs = %lld, expected %lld", (long long)n_dofs,
                (long long)m->n_dofs_local);
  if (kappa && n_kappa != m->n_elems * m->f.ngp)
    return fail(LGDM_ERR_INVALID_STATE, "n_kappa = %lld, expected %lld", (long long)n_kappa,
                (long long)(m->n_elems * m->f.ngp));
  if (!kappa && !m->have_kappa) return fail(LGDM_ERR_INVALID_STATE, "kappa never set");
  CU(cudaSetDevice(m->device));
  const cudaMemcpyKind kind = src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CU(cudaMemcpyAsync(m->dofs, dofs, size_t(n_dofs) * 8, kind, m->stream));
  if (kappa) CU(cudaMemcpyAsync(m->kappa, kappa, size_t(n_kappa) * 8, kind, m->stream));
  m->have_state = true;
  if (kappa) m->have_kappa = true;
  return LGDM_OK;
}

}  // extern "C"

namespace {

template <int D> lgdm_status assemble_general(lgdm_mesh m) {
  using F = Fam<D>;
  constexpr int EPB = D == 3 ? 8 : (D == 2 ? 32 : 64);
  if (!m->scratchK) {
    CU(dalloc(&m->scratchK, size_t(m->n_elems) * F::NDOFE * F::NDOFE));
    CU(dalloc(&m->scratchF, size_t(m->n_elems) * F::NDOFE));
    m->device_bytes += m->n_elems * (F::NDOFE * F::NDOFE + F::NDOFE) * 8;
  }
  const size_t smem = sizeof(double) * (size_t(EPB) * F::NGP * GpBlock<D>::STRIDE +
                                        EPB * F::NGP * kScal + EPB * F::NEN * D + EPB * F::NEN * F::NDPN);
  CU(set_smem_attr(k_elem_blocks<D, EPB>, smem, m->device));
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_elem_blocks<D, EPB>, EPB * F::NPAIR, smem);
  const int64_t batches = (m->n_elems + EPB - 1) / EPB;
  const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>(batches, int64_t(nsm) * std::max(per_sm, 1))));
  k_elem_blocks<D, EPB><<<grid, EPB * F::NPAIR, smem, m->stream>>>(
      m->dm, m->n_elems, m->conn, m->coords, m->dofs, m->kappa, m->k0g, m->alg, m->scratchK,
      m->scratchF);
  lgdm_status s = check_launch(m, "k_elem_blocks");
  if (s != LGDM_OK) return s;
  constexpr int WPB = 8;
  // per-warp block-row buffer sized by the mesh's largest degree (any connectivity)
  const size_t gsm = sizeof(double) * WPB * F::NDPN * size_t(m->max_deg) * F::NDPN;
  if (gsm > 48 * 1024) CU(set_smem_attr(k_gather<D, WPB>, gsm, m->device));
  k_gather<D, WPB><<<unsigned((m->n_owned + WPB - 1) / WPB), WPB * 32, gsm, m->stream>>>(
      m->n_owned, m->adj_ptr, m->adj, m->nbr_ptr, m->base, m->scratchK, m->scratchF, m->max_deg,
      m->val, m->R);
  return check_launch(m, "k_gather");
}

}  // namespace

extern "C" {

lgdm_status lgdm_prefetch_dofs(lgdm_mesh m, const double* host_dofs, int64_t n_dofs) {
  if (!m || !host_dofs) return fail(LGDM_ERR_INVALID_ARGUMENT, "NULL argument");
  if (n_dofs != m->n_dofs_local)
    return fail(LGDM_ERR_INVALID_STATE, "n_dofs = %lld, expected %lld", (long long)n_dofs, (long long)m->n_dofs_local);
  if (m->prefetch_pending) return fail(LGDM_ERR_INVALID_STATE, "a prefetch is already pending");
  CU(cudaSetDevice(m->device));
  if (!m->dofs_back) {
    CU(dalloc(&m->dofs_back, size_t(n_dofs)));
    m->device_bytes += n_dofs * 8;
    CU(cudaStreamCreateWithFlags(&m->cstream, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&m->copy_ev, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&m->free_ev, cudaEventDisableTiming));
  }
  // the back buffer was the current dofs until the last swap: wait for the work that used it
  if (m->free_ev_set) CU(cudaStreamWaitEvent(m->cstream, m->free_ev, 0));
  CU(cudaMemcpyAsync(m->dofs_back, host_dofs, size_t(n_dofs) * 8, cudaMemcpyHostToDevice, m->cstream));
  CU(cudaEventRecord(m->copy_ev, m->cstream));
  m->prefetch_pending = true;
  return LGDM_OK;
}

lgdm_status lgdm_set_state_prefetched(lgdm_mesh m) {
  if (!m) return fail(LGDM_ERR_INVALID_ARGUMENT, "mesh is NULL");
  if (!m->prefetch_pending) return fail(LGDM_ERR_INVALID_STATE, "no pending prefetch");
  if (!m->have_kappa) return fail(LGDM_ERR_INVALID_STATE, "kappa never set");
  CU(cudaSetDevice(m->device));
  CU(cudaStreamWaitEvent(m->stream, m->copy_ev, 0));
  std::swap(m->dofs, m->dofs_back);
  CU(cudaEventRecord(m->free_ev, m->stream));   // old buffer free once the work so far is done
  m->free_ev_set = true;
  m->prefetch_pending = false;
  m->have_state = true;
  return LGDM_OK;
}

lgdm_status lgdm_assemble(lgdm_mesh m, lgdm_csr* K, double** R) {
  const NvtxRange nvtx_range("lgdm_assemble");
  if (!m) return fail(LGDM_ERR_INVALID_ARGUMENT, "mesh is NULL");
  if (!m->have_state || !m->have_kappa) return fail(LGDM_ERR_INVALID_STATE, "assemble before set_state");
  CU(cudaSetDevice(m->device));
  lgdm_status s;
  // per-GP defect fields: the general path and the default sweeps (k_sweep4, k_sweepq)
  const bool sweep = !m->mixed && (m->kernel >= 2 || (m->kernel == 0 && m->structured && sweep_supported(m)));
  if (m->kernel >= 2 && !(m->structured && sweep_supported(m)))
    return fail(LGDM_ERR_INVALID_ARGUMENT, "sweep kernel requested but mesh is not structured");
  if (m->mixed) s = m->type == LGDM_BAR3 ? assemble_mixed<4>(m) : assemble_mixed<5>(m);
  else if (sweep) s = assemble_sweep(m);
  else if (m->f.dim == 1) s = assemble_general<1>(m);
  else if (m->f.dim == 2) s = assemble_general<2>(m);
  else s = assemble_general<3>(m);
  if (s != LGDM_OK) return s;
  m->assembled = true;
  if (K) {
    K->n_rows = m->n_rows;
    K->n_cols = m->mixed ? m->n_global_dofs : m->n_global_nodes * m->f.ndpn;
    K->nnz = m->nnz;
    K->first_row = m->mixed ? m->gdof0 + m->hdoff[m->own_b] : (m->gid0 + m->own_b) * m->f.ndpn;
    K->row_ptr = m->row_ptr;
    K->col_idx = m->col_idx;
    K->val = m->val;
  }
  if (R) *R = m->R;
  return LGDM_OK;
}

lgdm_status lgdm_update_history(lgdm_mesh m) {
  const NvtxRange nvtx_range("lgdm_update_history");
  if (!m) return fail(LGDM_ERR_INVALID_ARGUMENT, "mesh is NULL");
  if (!m->have_state || !m->have_kappa) return fail(LGDM_ERR_INVALID_STATE, "update_history before set_state");
  CU(cudaSetDevice(m->device));
  const int64_t n = m->n_elems * m->f.ngp;
  const unsigned blocks = unsigned((n + 255) / 256);
  if (m->type == LGDM_BAR3) k_mixed_history<4><<<blocks, 256, 0, m->stream>>>(m->n_elems, m->conn, m->doff, m->dofs, m->kappa);
  else if (m->type == LGDM_QUAD8) k_mixed_history<5><<<blocks, 256, 0, m->stream>>>(m->n_elems, m->conn, m->doff, m->dofs, m->kappa);
  else if (m->f.dim == 1) k_update_history<1><<<blocks, 256, 0, m->stream>>>(m->n_elems, m->conn, m->dofs, m->kappa);
  else if (m->f.dim == 2) k_update_history<2><<<blocks, 256, 0, m->stream>>>(m->n_elems, m->conn, m->dofs, m->kappa);
  else k_update_history<3><<<blocks, 256, 0, m->stream>>>(m->n_elems, m->conn, m->dofs, m->kappa);
  return check_launch(m, "k_update_history");
}

int lgdm_sdv_width(lgdm_elem_type type) {
  switch (type) {
    case LGDM_BAR2: return StateW<1>::W;
    case LGDM_QUAD4: return StateW<2>::W;
    case LGDM_HEX8: return StateW<3>::W;
    case LGDM_BAR3: return StateW<1>::W;
    case LGDM_QUAD8: return StateW<2>::W;
    default: return -1;
  }
}

lgdm_status lgdm_set_defects(lgdm_mesh m, const double* kappa0_gp, const double* alpha_gp,
                             int64_t n, int src_on_device) {
  if (!m) return fail(LGDM_ERR_INVALID_ARGUMENT, "mesh is NULL");
  const int64_t ngp = m->n_elems * m->f.ngp;
  if ((kappa0_gp || alpha_gp) && n != ngp)
    return fail(LGDM_ERR_INVALID_STATE, "n = %lld, expected n_elems * ngp = %lld", (long long)n,
                (long long)ngp);
  CU(cudaSetDevice(m->device));
  const cudaMemcpyKind kind = src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  struct { const double* src; double** dst; } f[2] = {{kappa0_gp, &m->k0g}, {alpha_gp, &m->alg}};
  for (auto& x : f) {
    if (!x.src) {
      if (*x.dst) {
        CU(cudaStreamSynchronize(m->stream));
        CU(cudaFree(*x.dst));
        m->device_bytes -= ngp * 8;
        *x.dst = nullptr;
      }
      continue;
    }
    if (!*x.dst) {
      CU(dalloc(x.dst, size_t(ngp)));
      m->device_bytes += ngp * 8;
    }
    CU(cudaMemcpyAsync(*x.dst, x.src, size_t(ngp) * 8, kind, m->stream));
  }
  if (!src_on_device) CU(cudaStreamSynchronize(m->stream));   // host arrays may be pageable
  return LGDM_OK;
}

lgdm_status lgdm_update_state(lgdm_mesh m, double* sdv, int64_t n_sdv, int dst_on_device) {
  const NvtxRange nvtx_range("lgdm_update_state");
  if (!m) return fail(LGDM_ERR_INVALID_ARGUMENT, "mesh is NULL");
  if (!m->have_state || !m->have_kappa) return fail(LGDM_ERR_INVALID_STATE, "update_state before set_state");
  const int W = lgdm_sdv_width(lgdm_elem_type(m->type));
  const int64_t ngp = m->n_elems * m->f.ngp;
  if (sdv && n_sdv != ngp * W)
    return fail(LGDM_ERR_INVALID_STATE, "n_sdv = %lld, expected %lld", (long long)n_sdv,
                (long long)(ngp * W));
  CU(cudaSetDevice(m->device));
  double* out = nullptr;
  if (sdv && dst_on_device) out = sdv;
  if (sdv && !dst_on_device) {
    if (!m->sdv_dev) {
      CU(dalloc(&m->sdv_dev, size_t(ngp) * W));
      m->device_bytes += ngp * W * 8;
    }
    out = m->sdv_dev;
  }
  constexpr int TPB = 128;
  const unsigned blocks = unsigned((ngp + TPB - 1) / TPB);
  // record staging [TPB][W] + per-warp node values [TPB][dim + ndpn] (k_update_state)
  const size_t smem = size_t(TPB) * (W + m->f.dim + m->f.ndpn) * sizeof(double);
  CU(set_smem_attr(k_update_state<3>, size_t(TPB) * (StateW<3>::W + 7) * 8, m->device));
  if (m->mixed) {
    const size_t tbl = sizeof(double) * 400;   // >= the padded shape table of either family
    static_assert(sizeof(MShape<5>) <= 400 * sizeof(double) && sizeof(MShape<4>) <= 400 * sizeof(double), "table");
    const size_t sm2 = tbl + size_t(TPB) * W * sizeof(double);
    if (m->type == LGDM_BAR3)
      k_mixed_state<4><<<blocks, TPB, sm2, m->stream>>>(m->dm, m->n_elems, m->conn, m->coords, m->doff, m->dofs, m->kappa, m->k0g, m->alg, out);
    else
      k_mixed_state<5><<<blocks, TPB, sm2, m->stream>>>(m->dm, m->n_elems, m->conn, m->coords, m->doff, m->dofs, m->kappa, m->k0g, m->alg, out);
  } else if (m->f.dim == 1)
    k_update_state<1><<<blocks, TPB, smem, m->stream>>>(m->dm, m->n_elems, m->conn, m->coords, m->dofs, m->kappa, m->k0g, m->alg, out);
  else if (m->f.dim == 2)
    k_update_state<2><<<blocks, TPB, smem, m->stream>>>(m->dm, m->n_elems, m->conn, m->coords, m->dofs, m->kappa, m->k0g, m->alg, out);
  else
    k_update_state<3><<<blocks, TPB, smem, m->stream>>>(m->dm, m->n_elems, m->conn, m->coords, m->dofs, m->kappa, m->k0g, m->alg, out);
  lgdm_status s = check_launch(m, "k_update_state");
  if (s != LGDM_OK) return s;
  if (sdv && !dst_on_device) {
    CU(cudaMemcpyAsync(sdv, out, size_t(ngp) * W * 8, cudaMemcpyDeviceToHost, m->stream));
    CU(cudaStreamSynchronize(m->stream));
  }
  return LGDM_OK;
}

lgdm_status lgdm_get_blocked(lgdm_mesh m, lgdm_csr* K, double** R) {
  if (!m) return fail(LGDM_ERR_INVALID_ARGUMENT, "mesh is NULL");
  if (!m->assembled) return fail(LGDM_ERR_INVALID_STATE, "get_blocked before assemble");
  if (m->own_b != 0 || m->own_e != m->n_nodes || m->gid0 != 0 || m->n_global_nodes != m->n_nodes)
    return fail(LGDM_ERR_INVALID_ARGUMENT, "blocked order needs a single-rank whole mesh");
  CU(cudaSetDevice(m->device));
  if (!m->rp_b) {
    CU(dalloc(&m->rp_b, size_t(m->n_rows) + 1));
    CU(dalloc(&m->ci_b, size_t(m->nnz)));
    CU(dalloc(&m->val_b, size_t(m->nnz)));
    CU(dalloc(&m->R_b, size_t(m->n_rows)));
    m->device_bytes += (m->n_rows + 1) * 8 + m->nnz * 12 + m->n_rows * 8;
  }
  const unsigned blocks = unsigned((m->n_rows * 32 + 255) / 256);
  const int64_t no = m->n_owned;
  if (m->mixed) {
    if (!m->bperm) {   // permutation and blocked row_ptr, once per mesh
      const int64_t n = m->n_rows;
      std::vector<int64_t> perm(n), rp(n + 1, 0), hrp(n + 1);
      std::vector<int32_t> inv(n);
      int64_t k = 0;
      for (int pass = 0; pass < 2; ++pass)
        for (int64_t d = 0; d < n; ++d)
          if ((m->hkind[d] == m->f.dim) == (pass == 1)) { inv[d] = int32_t(k); perm[k++] = d; }
      CU(cudaMemcpyAsync(hrp.data(), m->row_ptr, size_t(n + 1) * 8, cudaMemcpyDeviceToHost, m->stream));
      CU(cudaStreamSynchronize(m->stream));
      for (int64_t r = 0; r < n; ++r) rp[r + 1] = rp[r] + (hrp[perm[r] + 1] - hrp[perm[r]]);
      CU(dalloc(&m->bperm, size_t(n)));
      CU(dalloc(&m->binv, size_t(n)));
      m->device_bytes += n * 12;
      CU(cudaMemcpyAsync(m->bperm, perm.data(), size_t(n) * 8, cudaMemcpyHostToDevice, m->stream));
      CU(cudaMemcpyAsync(m->binv, inv.data(), size_t(n) * 4, cudaMemcpyHostToDevice, m->stream));
      CU(cudaMemcpyAsync(m->rp_b, rp.data(), size_t(n + 1) * 8, cudaMemcpyHostToDevice, m->stream));
      CU(cudaStreamSynchronize(m->stream));   // host vectors go out of scope
    }
    k_blocked_mixed<<<blocks, 256, 0, m->stream>>>(m->n_rows, m->f.dim, m->bperm, m->binv, m->dkind, m->row_ptr, m->col_idx, m->val, m->R, m->rp_b, m->ci_b, m->val_b, m->R_b);
  } else if (m->f.dim == 1)
    k_blocked<1, 2><<<blocks, 256, 0, m->stream>>>(no, m->nbr_ptr, m->base, m->col_idx, m->val, m->R, m->rp_b, m->ci_b, m->val_b, m->R_b);
  else if (m->f.dim == 2)
    k_blocked<2, 3><<<blocks, 256, 0, m->stream>>>(no, m->nbr_ptr, m->base, m->col_idx, m->val, m->R, m->rp_b, m->ci_b, m->val_b, m->R_b);
  else
    k_blocked<3, 4><<<blocks, 256, 0, m->stream>>>(no, m->nbr_ptr, m->base, m->col_idx, m->val, m->R, m->rp_b, m->ci_b, m->val_b, m->R_b);
  lgdm_status s = check_launch(m, "k_blocked");
  if (s != LGDM_OK) return s;
  if (K) {
    K->n_rows = m->n_rows;
    K->n_cols = m->mixed ? m->n_rows : m->n_global_nodes * m->f.ndpn;
    K->nnz = m->nnz;
    K->first_row = 0;
    K->row_ptr = m->rp_b;
    K->col_idx = m->ci_b;
    K->val = m->val_b;
  }
  if (R) *R = m->R_b;
  return LGDM_OK;
}

static bool whole_single_rank(lgdm_mesh m) {
  return m->own_b == 0 && m->own_e == m->n_nodes && m->gid0 == 0 && m->n_global_nodes == m->n_nodes;
}

// Local dof ranges of the Newton pieces.  Local dofs = the mesh's nodes (owned + ghosts) in
// node order; the owned ones [own_b, own_e) are the rows of K / R; a CSR column c (global dof)
// is local dof c - col_off.
struct DofRange {
  int64_t own_b, own_e, nloc, col_off;
};
static DofRange dof_range(lgdm_mesh m) {
  if (m->mixed) return {m->hdoff[m->own_b], m->hdoff[m->own_e], m->n_dofs_local, m->gdof0};
  const int64_t k = m->f.ndpn;
  return {m->own_b * k, m->own_e * k, m->n_nodes * k, m->gid0 * k};
}
static bool multi_rank(lgdm_mesh m) { return m->comm && m->nranks > 1; }

// the Newton pieces need the whole system on one rank, or a communicator over the row-owned
// slabs (lgdm_set_comm validated the neighbour layout)
static lgdm_status newton_ready(lgdm_mesh m) {
  if (multi_rank(m)) return m->halo_ok ? LGDM_OK : fail(LGDM_ERR_UNSUPPORTED, "slab layout not validated by lgdm_set_comm");
  if (whole_single_rank(m) || (m->mixed && m->own_b == 0 && m->own_e == m->n_nodes && m->gdof0 == 0 &&
                               m->n_global_dofs == m->n_dofs_local))
    return LGDM_OK;
  return fail(LGDM_ERR_UNSUPPORTED, "a slab mesh needs a communicator (lgdm_set_comm) for the Newton pieces");
}

// Ghost-dof halo exchange (SURVEY 8e future exchange step): the ghost dofs of x (local dof
// vector) receive the owned values of the neighbouring slabs -- rank - 1 holds the nodes below
// the owned range, rank + 1 those above; each rank sends its first / last owned dofs, as many
// as the neighbour keeps as ghosts (mirror sizes, checked by lgdm_set_comm).
static lgdm_status halo_exchange(lgdm_mesh m, double* x) {
  if (!multi_rank(m)) return LGDM_OK;
  const DofRange d = dof_range(m);
  // below: my first owned dofs are the lower rank's upper ghosts; my lower ghosts are its last
  // owned dofs (counts from lgdm_set_comm: the two sides may differ, e.g. mixed-order slabs)
  const int64_t sl = m->halo_send_lo, rl = m->halo_recv_lo, sh = m->halo_send_hi, rh = m->halo_recv_hi;
  ncclResult_t r = g_nccl.groupStart();
  if (sl > 0 && r == ncclSuccess) r = g_nccl.send(x + d.own_b, size_t(sl), ncclFloat64, m->rank - 1, m->comm, m->stream);
  if (rl > 0 && r == ncclSuccess) r = g_nccl.recv(x + d.own_b - rl, size_t(rl), ncclFloat64, m->rank - 1, m->comm, m->stream);
  if (sh > 0 && r == ncclSuccess) r = g_nccl.send(x + d.own_e - sh, size_t(sh), ncclFloat64, m->rank + 1, m->comm, m->stream);
  if (rh > 0 && r == ncclSuccess) r = g_nccl.recv(x + d.own_e, size_t(rh), ncclFloat64, m->rank + 1, m->comm, m->stream);
  const ncclResult_t re = g_nccl.groupEnd();
  if (r != ncclSuccess || re != ncclSuccess)
    return fail(LGDM_ERR_NCCL, "halo exchange: %s", g_nccl.getErrorString ? g_nccl.getErrorString(r != ncclSuccess ? r : re) : "?");
  return LGDM_OK;
}

// sum of n device doubles over the ranks, in place (no-op on one rank)
static lgdm_status allreduce_sum(lgdm_mesh m, double* dev, int n) {
  if (!multi_rank(m)) return LGDM_OK;
  const ncclResult_t r = g_nccl.allReduce(dev, dev, size_t(n), ncclFloat64, ncclSum, m->comm, m->stream);
  if (r != ncclSuccess) return fail(LGDM_ERR_NCCL, "ncclAllReduce: %s", g_nccl.getErrorString ? g_nccl.getErrorString(r) : "?");
  return LGDM_OK;
}

lgdm_status lgdm_apply_dirichlet(lgdm_mesh m, int64_t n_fixed, const int64_t* dof_ids,
                                 const double* increments) {
  if (!m) return fail(LGDM_ERR_INVALID_ARGUMENT, "mesh is NULL");
  if (!m->assembled) return fail(LGDM_ERR_INVALID_STATE, "apply_dirichlet before assemble");
  lgdm_status s = newton_ready(m);
  if (s != LGDM_OK) return s;
  if (n_fixed < 0 || (n_fixed && (!dof_ids || !increments)))
    return fail(LGDM_ERR_INVALID_ARGUMENT, "dof_ids / increments");
  const DofRange d = dof_range(m);
  const int64_t nglob = m->mixed ? m->n_global_dofs : m->n_global_nodes * m->f.ndpn;
  std::vector<uint8_t> mask(d.nloc, 0);   // over the local dofs (owned + ghosts)
  std::vector<double> inc(d.nloc, 0.0);
  for (int64_t k = 0; k < n_fixed; ++k) {
    const int64_t g = dof_ids[k];   // global dof id (every rank passes the same list)
    if (g < 0 || g >= nglob) return fail(LGDM_ERR_INVALID_ARGUMENT, "dof id %lld out of range", (long long)g);
    const int64_t l = g - d.col_off;
    if (m->mixed ? (l >= 0 && l < d.nloc && m->hkind[l] == m->f.dim) : g % m->f.ndpn == m->f.dim)
      return fail(LGDM_ERR_INVALID_ARGUMENT, "dof %lld is an ebar dof (only u dofs can be constrained)", (long long)g);
    if (l < 0 || l >= d.nloc) continue;   // another rank's dof, not coupled to this rank's rows
    mask[l] = 1;
    inc[l] = increments[k];
  }
  CU(cudaSetDevice(m->device));
  if (!m->fixed) {
    CU(dalloc(&m->fixed, size_t(d.nloc)));
    CU(dalloc(&m->fixinc, size_t(d.nloc)));
    m->device_bytes += d.nloc * 9;
  }
  CU(cudaMemcpyAsync(m->fixed, mask.data(), size_t(d.nloc), cudaMemcpyHostToDevice, m->stream));
  CU(cudaMemcpyAsync(m->fixinc, inc.data(), size_t(d.nloc) * 8, cudaMemcpyHostToDevice, m->stream));
  const int64_t n = m->n_rows;
  k_dirichlet<<<unsigned((n * 32 + 255) / 256), 256, 0, m->stream>>>(
      n, d.col_off + d.own_b, d.own_b, d.col_off, m->row_ptr, m->col_idx, m->val, m->R, m->fixed, m->fixinc);
  s = check_launch(m, "k_dirichlet");
  if (s != LGDM_OK) return s;
  CU(cudaStreamSynchronize(m->stream));   // host staging vectors go out of scope
  return LGDM_OK;
}

lgdm_status lgdm_solve(lgdm_mesh m, double* delta, double tol, int max_iter, int* iters_out,
                       double* relres_out) {
  const NvtxRange nvtx_range("lgdm_solve");
  if (!m) return fail(LGDM_ERR_INVALID_ARGUMENT, "mesh is NULL");
  if (!m->assembled) return fail(LGDM_ERR_INVALID_STATE, "solve before assemble");
  lgdm_status s = newton_ready(m);
  if (s != LGDM_OK) return s;
  if (!delta || !(tol > 0) || max_iter < 1) return fail(LGDM_ERR_INVALID_ARGUMENT, "delta / tol / max_iter");
  // rows: the owned rows (n); delta, ph, sh: local dof vectors (owned + ghost dofs, nloc) whose
  // ghosts come from the neighbouring slabs before every SpMV; dots over the owned rows,
  // summed over the ranks (multi-rank Jacobi-BiCGSTAB)
  const int64_t n = m->n_rows;
  const DofRange d = dof_range(m);
  const int64_t nl = d.nloc, ob = d.own_b, row_g0 = d.col_off + d.own_b;
  CU(cudaSetDevice(m->device));
  if (!m->sol) {
    CU(dalloc(&m->sol, size_t(n) * 7 + size_t(nl) * 2));
    CU(dalloc(&m->sol_part, size_t(kRedBlocks) * 4 + 4));
    m->device_bytes += (n * 7 + nl * 2) * 8 + kRedBlocks * 32 + 32;
  }
  double *r = m->sol, *r0 = r + n, *p = r0 + n, *v = p + n, *sv = v + n, *t = sv + n, *dinv = t + n,
         *ph = dinv + n, *sh = ph + nl;
  double* part = m->sol_part;
  double* fin = part + size_t(kRedBlocks) * 4;
  cudaStream_t st = m->stream;
  const unsigned gw = unsigned((n * 32 + 255) / 256), ge = unsigned((n + 255) / 256);
  auto dots = [&](const double* a, const double* b, const double* c, const double* dd, double* h) -> lgdm_status {
    k_dot2<<<kRedBlocks, 256, 0, st>>>(n, a, b, c, dd, part);
    k_final<2><<<1, 256, 0, st>>>(kRedBlocks, part, fin);
    m->launches += 2;
    lgdm_status sr = allreduce_sum(m, fin, 2);
    if (sr != LGDM_OK) return sr;
    CU(cudaMemcpyAsync(h, fin, 16, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return LGDM_OK;
  };
  auto spmv = [&](double* x_local, double* y) -> lgdm_status {   // ghosts first
    lgdm_status sh_ = halo_exchange(m, x_local);
    if (sh_ != LGDM_OK) return sh_;
    k_spmv<<<gw, 256, 0, st>>>(n, m->row_ptr, m->col_idx, m->val, x_local, d.col_off, y);
    ++m->launches;
    return LGDM_OK;
  };
  // x = 0, r = r0 = b, p = v = 0, Jacobi M = diag(K)
  CU(cudaMemsetAsync(delta, 0, size_t(nl) * 8, st));
  CU(cudaMemsetAsync(ph, 0, size_t(nl) * 8, st));
  CU(cudaMemsetAsync(sh, 0, size_t(nl) * 8, st));
  CU(cudaMemcpyAsync(r, m->R, size_t(n) * 8, cudaMemcpyDeviceToDevice, st));
  CU(cudaMemcpyAsync(r0, m->R, size_t(n) * 8, cudaMemcpyDeviceToDevice, st));
  CU(cudaMemsetAsync(p, 0, size_t(n) * 8, st));
  CU(cudaMemsetAsync(v, 0, size_t(n) * 8, st));
  k_invdiag<<<ge, 256, 0, st>>>(n, row_g0, m->row_ptr, m->col_idx, m->val, dinv);
  ++m->launches;
  double h[2];
  if ((s = dots(r, r, nullptr, nullptr, h)) != LGDM_OK) return s;
  const double bnorm = std::sqrt(h[0]);
  int it = 0;
  double rel = 0.0;
  if (bnorm == 0.0) {
    if (iters_out) *iters_out = 0;
    if (relres_out) *relres_out = 0.0;
    return LGDM_OK;
  }
  double rho = 1.0, alpha = 1.0, omega = 1.0;
  rel = 1.0;
  for (it = 1; it <= max_iter; ++it) {
    if ((s = dots(r0, r, nullptr, nullptr, h)) != LGDM_OK) return s;
    const double rho_new = h[0];
    if (rho_new == 0.0 || omega == 0.0) break;   // breakdown
    const double beta = (rho_new / rho) * (alpha / omega);
    k_p_update<<<ge, 256, 0, st>>>(n, beta, omega, r, v, p);
    k_scale_mul<<<ge, 256, 0, st>>>(n, dinv, p, ph + ob);
    m->launches += 2;
    if ((s = spmv(ph, v)) != LGDM_OK) return s;
    if ((s = dots(r0, v, nullptr, nullptr, h)) != LGDM_OK) return s;
    if (h[0] == 0.0) break;
    alpha = rho_new / h[0];
    k_s_update<<<ge, 256, 0, st>>>(n, alpha, r, v, sv);
    ++m->launches;
    if ((s = dots(sv, sv, nullptr, nullptr, h)) != LGDM_OK) return s;
    if (std::sqrt(h[0]) / bnorm <= tol) {
      k_axpy<<<ge, 256, 0, st>>>(n, alpha, ph + ob, delta + ob);
      ++m->launches;
      rel = std::sqrt(h[0]) / bnorm;
      break;
    }
    k_scale_mul<<<ge, 256, 0, st>>>(n, dinv, sv, sh + ob);
    ++m->launches;
    if ((s = spmv(sh, t)) != LGDM_OK) return s;
    if ((s = dots(t, sv, t, t, h)) != LGDM_OK) return s;
    omega = h[1] != 0.0 ? h[0] / h[1] : 0.0;
    k_x_update<<<ge, 256, 0, st>>>(n, alpha, omega, ph + ob, sh + ob, delta + ob);
    k_r_update<<<ge, 256, 0, st>>>(n, omega, sv, t, r);
    m->launches += 2;
    if ((s = dots(r, r, nullptr, nullptr, h)) != LGDM_OK) return s;
    rel = std::sqrt(h[0]) / bnorm;
    if (rel <= tol) break;
    rho = rho_new;
  }
  // true residual of the returned delta (||b - K delta|| / ||b||); the SpMV also fills the
  // ghost dofs of delta, so lgdm_add_dofs updates every local dof consistently
  if ((s = spmv(delta, t)) != LGDM_OK) return s;
  k_s_update<<<ge, 256, 0, st>>>(n, 1.0, m->R, t, sv);
  ++m->launches;
  if ((s = dots(sv, sv, nullptr, nullptr, h)) != LGDM_OK) return s;
  rel = std::sqrt(h[0]) / bnorm;
  if (iters_out) *iters_out = std::min(it, max_iter);
  if (relres_out) *relres_out = rel;
  if (!(rel <= 10.0 * tol))
    return fail(LGDM_ERR_NOT_CONVERGED, "BiCGSTAB: relative residual %.3e after %d iterations (tol %.1e)", rel, std::min(it, max_iter), tol);
  return LGDM_OK;
}

lgdm_status lgdm_dof_offsets(lgdm_mesh m, int64_t* host_out, int64_t n) {
  if (!m || !host_out) return fail(LGDM_ERR_INVALID_ARGUMENT, "NULL argument");
  if (n != m->n_nodes + 1) return fail(LGDM_ERR_INVALID_ARGUMENT, "n = %lld, expected n_nodes + 1", (long long)n);
  for (int64_t i = 0; i <= m->n_nodes; ++i) host_out[i] = m->mixed ? m->hdoff[i] : i * m->f.ndpn;
  return LGDM_OK;
}

lgdm_status lgdm_reaction(lgdm_mesh m, int64_t n, const int64_t* dof_ids, double* out) {
  if (!m || !out || (n > 0 && !dof_ids)) return fail(LGDM_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!m->assembled) return fail(LGDM_ERR_INVALID_STATE, "reaction before assemble");
  lgdm_status s = newton_ready(m);
  if (s != LGDM_OK) return s;
  const DofRange d = dof_range(m);
  const int64_t nglob = m->mixed ? m->n_global_dofs : m->n_global_nodes * m->f.ndpn;
  std::vector<int64_t> rows;   // this rank's owned rows among the (global) dof ids
  for (int64_t k = 0; k < n; ++k) {
    if (dof_ids[k] < 0 || dof_ids[k] >= nglob) return fail(LGDM_ERR_INVALID_ARGUMENT, "dof id out of range");
    const int64_t r = dof_ids[k] - d.col_off - d.own_b;
    if (r >= 0 && r < m->n_rows) rows.push_back(r);
  }
  CU(cudaSetDevice(m->device));
  const int64_t nr = int64_t(rows.size());
  if (m->react_cap < nr + 1) {   // the mesh's buffer, grown (never per call)
    CU(cudaStreamSynchronize(m->stream));
    if (m->react_buf) cudaFree(m->react_buf);
    m->react_buf = nullptr;
    m->react_cap = 0;
    const int64_t cap = std::max<int64_t>(2 * (nr + 1), 64);
    CU(dalloc(&m->react_buf, size_t(cap)));
    m->react_cap = cap;
  }
  int64_t* ids = m->react_buf;
  double* sum = reinterpret_cast<double*>(ids + nr);   // one double-sized slot after the ids
  if (nr) CU(cudaMemcpyAsync(ids, rows.data(), size_t(nr) * 8, cudaMemcpyHostToDevice, m->stream));
  k_reaction<<<1, 256, 0, m->stream>>>(nr, ids, m->R, sum);
  ++m->launches;
  s = allreduce_sum(m, sum, 1);
  if (s == LGDM_OK) cudaMemcpyAsync(out, sum, 8, cudaMemcpyDeviceToHost, m->stream);
  cudaStreamSynchronize(m->stream);   // `rows` and `out` are the caller's / this frame's
  return s;
}

lgdm_status lgdm_solve_direct(lgdm_mesh m, double* delta, int* singularity) {
  const NvtxRange nvtx_range("lgdm_solve_direct");
  if (!m || !delta) return fail(LGDM_ERR_INVALID_ARGUMENT, "mesh / delta is NULL");
  if (!m->assembled) return fail(LGDM_ERR_INVALID_STATE, "solve before assemble");
  if (!whole_single_rank(m)) return fail(LGDM_ERR_UNSUPPORTED, "Newton pieces need a single-rank whole mesh");
  if (m->nnz > INT32_MAX || m->n_rows > INT32_MAX)
    return fail(LGDM_ERR_UNSUPPORTED, "direct solve needs nnz < 2^31 (use lgdm_solve)");
  if (!load_spsolver()) return fail(LGDM_ERR_UNSUPPORTED, "libcusolver / libcusparse not loadable");
  CU(cudaSetDevice(m->device));
  const int n = int(m->n_rows), nnz = int(m->nnz);
  bool ok = true;
  if (!m->sp_handle) {   // handle, descriptor and the int32 row pointers: once per mesh
    CU(dalloc(&m->rp32, size_t(n) + 1));
    m->device_bytes += (n + 1) * 4;
    k_rowptr32<<<unsigned((n + 256) / 256), 256, 0, m->stream>>>(n + 1, m->row_ptr, m->rp32);
    ++m->launches;
    ok = g_sps.create(&m->sp_handle) == CUSOLVER_STATUS_SUCCESS &&
         g_sps.createDescr(&m->sp_descr) == CUSPARSE_STATUS_SUCCESS &&
         g_sps.setType(m->sp_descr, CUSPARSE_MATRIX_TYPE_GENERAL) == CUSPARSE_STATUS_SUCCESS &&
         g_sps.setBase(m->sp_descr, CUSPARSE_INDEX_BASE_ZERO) == CUSPARSE_STATUS_SUCCESS;
  }
  int sing = -1;
  ok = ok && g_sps.setStream(m->sp_handle, m->stream) == CUSOLVER_STATUS_SUCCESS;
  if (ok)
    ok = g_sps.lsvqr(m->sp_handle, n, nnz, m->sp_descr, m->val, m->rp32, m->col_idx, m->R, 1e-14, 1,
                     delta, &sing) == CUSOLVER_STATUS_SUCCESS;
  cudaStreamSynchronize(m->stream);
  if (singularity) *singularity = sing;
  if (!ok) return fail(LGDM_ERR_CUDA, "cusolverSpDcsrlsvqr failed");
  if (sing >= 0) return fail(LGDM_ERR_NOT_CONVERGED, "singular system (QR pivot %d)", sing);
  return LGDM_OK;
}

lgdm_status lgdm_add_dofs(lgdm_mesh m, const double* delta, double alpha) {
  if (!m || !delta) return fail(LGDM_ERR_INVALID_ARGUMENT, "mesh / delta is NULL");
  if (!m->have_state) return fail(LGDM_ERR_INVALID_STATE, "add_dofs before set_state");
  lgdm_status s0 = newton_ready(m);
  if (s0 != LGDM_OK) return s0;
  CU(cudaSetDevice(m->device));
  const int64_t n = m->n_dofs_local;
  k_axpy<<<unsigned((n + 255) / 256), 256, 0, m->stream>>>(n, alpha, delta, m->dofs);
  return check_launch(m, "k_axpy");
}

lgdm_status lgdm_delta_norms(lgdm_mesh m, const double* delta, double out4[4]) {
  if (!m || !delta || !out4) return fail(LGDM_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!m->have_state) return fail(LGDM_ERR_INVALID_STATE, "delta_norms before set_state");
  lgdm_status s0 = newton_ready(m);
  if (s0 != LGDM_OK) return s0;
  CU(cudaSetDevice(m->device));
  if (!m->sol_part) {
    CU(dalloc(&m->sol_part, size_t(kRedBlocks) * 4 + 4));
    m->device_bytes += kRedBlocks * 32 + 32;
  }
  // sums over the owned dofs (ghost dofs belong to another rank), then over the ranks
  const DofRange d = dof_range(m);
  const int64_t n = d.own_e - d.own_b, ob = d.own_b;
  double* part = m->sol_part;
  double* fin = part + size_t(kRedBlocks) * 4;
  if (m->mixed) k_delta_sumsq_kind<<<kRedBlocks, 256, 0, m->stream>>>(n, m->f.dim, m->dkind + ob, delta + ob, m->dofs + ob, part);
  else if (m->f.ndpn == 2) k_delta_sumsq<2><<<kRedBlocks, 256, 0, m->stream>>>(n, delta + ob, m->dofs + ob, part);
  else if (m->f.ndpn == 3) k_delta_sumsq<3><<<kRedBlocks, 256, 0, m->stream>>>(n, delta + ob, m->dofs + ob, part);
  else k_delta_sumsq<4><<<kRedBlocks, 256, 0, m->stream>>>(n, delta + ob, m->dofs + ob, part);
  k_final<4><<<1, 256, 0, m->stream>>>(kRedBlocks, part, fin);
  m->launches += 2;
  if ((s0 = allreduce_sum(m, fin, 4)) != LGDM_OK) return s0;
  CU(cudaMemcpyAsync(out4, fin, 32, cudaMemcpyDeviceToHost, m->stream));
  CU(cudaStreamSynchronize(m->stream));
  return LGDM_OK;
}

lgdm_status lgdm_delta_ratios(lgdm_mesh m, const double* delta, double tol, double out2[2],
                              int* converged) {
  if (!out2 || !converged) return fail(LGDM_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!(tol > 0.0)) return fail(LGDM_ERR_INVALID_ARGUMENT, "tol must be > 0");
  double s4[4];
  const lgdm_status st = lgdm_delta_norms(m, delta, s4);
  if (st != LGDM_OK) return st;
  // Alg. 1 l.26: ||du|| / ||u|| and ||de|| / ||e|| (a zero iterate counts as norm 1e-16)
  out2[0] = std::sqrt(s4[0]) / std::max(std::sqrt(s4[1]), 1e-16);
  out2[1] = std::sqrt(s4[2]) / std::max(std::sqrt(s4[3]), 1e-16);
  *converged = (out2[0] <= tol && out2[1] <= tol) ? 1 : 0;
  return LGDM_OK;
}

lgdm_status lgdm_residual_sumsq(lgdm_mesh m, double* out2, int on_device) {
  const NvtxRange nvtx_range("lgdm_residual_sumsq");
  if (!m || !out2) return fail(LGDM_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!m->assembled) return fail(LGDM_ERR_INVALID_STATE, "residual before assemble");
  CU(cudaSetDevice(m->device));
  if (m->mixed) k_sumsq_kind<<<kSumBlocks, kSumThreads, 0, m->stream>>>(m->n_rows, m->f.dim, m->dkind + m->hdoff[m->own_b], m->R, m->sumsq_part);
  else k_sumsq_partial<<<kSumBlocks, kSumThreads, 0, m->stream>>>(m->n_rows, m->f.ndpn, m->f.dim, m->R, m->sumsq_part);
  lgdm_status s = check_launch(m, "k_sumsq_partial");
  if (s != LGDM_OK) return s;
  double* dst = on_device ? out2 : m->sumsq_out;
  k_sumsq_final<<<1, kSumThreads, 0, m->stream>>>(kSumBlocks, m->sumsq_part, dst);
  if ((s = check_launch(m, "k_sumsq_final")) != LGDM_OK) return s;
  if (!on_device) {
    CU(cudaMemcpyAsync(m->host_pinned, m->sumsq_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, m->stream));
    CU(cudaStreamSynchronize(m->stream));
    out2[0] = m->host_pinned[0];
    out2[1] = m->host_pinned[1];
  }
  return LGDM_OK;
}

lgdm_status lgdm_residual_norms(lgdm_mesh m, double out2[2]) {
  const NvtxRange nvtx_range("lgdm_residual_norms");
  if (!m || !out2) return fail(LGDM_ERR_INVALID_ARGUMENT, "NULL argument");
  lgdm_status s = lgdm_residual_sumsq(m, m->sumsq_out, 1);
  if (s != LGDM_OK) return s;
  if (m->comm) {
    ncclResult_t r = g_nccl.allReduce(m->sumsq_out, m->sumsq_out, 2, ncclFloat64, ncclSum, m->comm, m->stream);
    if (r != ncclSuccess)
      return fail(LGDM_ERR_NCCL, "ncclAllReduce: %s", g_nccl.getErrorString ? g_nccl.getErrorString(r) : "?");
  }
  CU(cudaMemcpyAsync(m->host_pinned, m->sumsq_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, m->stream));
  CU(cudaStreamSynchronize(m->stream));
  out2[0] = std::sqrt(m->host_pinned[0]);
  out2[1] = std::sqrt(m->host_pinned[1]);
  return LGDM_OK;
}

// one hot-path pass on the mesh stream (no host synchronisation inside)
static lgdm_status step_enqueue(lgdm_mesh m, bool hist) {
  lgdm_status s = lgdm_assemble(m, nullptr, nullptr);
  if (s != LGDM_OK) return s;
  if ((s = lgdm_residual_sumsq(m, m->sumsq_out, 1)) != LGDM_OK) return s;
  if (m->comm) {
    ncclResult_t r = g_nccl.allReduce(m->sumsq_out, m->sumsq_out, 2, ncclFloat64, ncclSum, m->comm, m->stream);
    if (r != ncclSuccess)
      return fail(LGDM_ERR_NCCL, "ncclAllReduce: %s", g_nccl.getErrorString ? g_nccl.getErrorString(r) : "?");
  }
  CU(cudaMemcpyAsync(m->host_pinned, m->sumsq_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, m->stream));
  if (hist) return lgdm_update_history(m);
  return LGDM_OK;
}

lgdm_status lgdm_step(lgdm_mesh m, int flags, double out2[2]) {
  const NvtxRange nvtx_range("lgdm_step");
  if (!m || !out2) return fail(LGDM_ERR_INVALID_ARGUMENT, "NULL argument");
  if (flags & ~3) return fail(LGDM_ERR_INVALID_ARGUMENT, "unknown step flags %d", flags);
  if (!m->have_state || !m->have_kappa) return fail(LGDM_ERR_INVALID_STATE, "step before set_state");
  CU(cudaSetDevice(m->device));
  const bool use_graph = flags & LGDM_STEP_GRAPH, hist = flags & LGDM_STEP_HISTORY;
  lgdm_status s;
  if (!use_graph || !m->step_warm) {
    // eager pass; the first one also allocates any lazily created scratch, so a later capture
    // records kernels and copies only
    if ((s = step_enqueue(m, hist)) != LGDM_OK) return s;
    m->step_warm = true;
  } else {
    if (!m->gstream) {
      CU(cudaStreamCreateWithFlags(&m->gstream, cudaStreamNonBlocking));
      CU(cudaEventCreateWithFlags(&m->gev_in, cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&m->gev_out, cudaEventDisableTiming));
    }
    CU(cudaEventRecord(m->gev_in, m->stream));
    CU(cudaStreamWaitEvent(m->gstream, m->gev_in, 0));
    lgdm_mesh_s::StepGraph* g = nullptr;
    for (auto& c : m->sgraph)
      if (c.exec && c.dofs == m->dofs && c.k0g == m->k0g && c.alg == m->alg && c.kernel == m->kernel &&
          c.flags == flags && c.comm == (void*)m->comm)
        g = &c;
    if (!g) {
      g = &m->sgraph[m->sgraph_next];
      m->sgraph_next ^= 1;
      if (g->exec) cudaGraphExecDestroy(g->exec), g->exec = nullptr;
      cudaGraph_t graph = nullptr;
      CU(cudaStreamBeginCapture(m->gstream, cudaStreamCaptureModeThreadLocal));
      const int64_t l0 = m->launches;
      cudaStream_t keep = m->stream;
      m->stream = m->gstream;   // every launch of the pass goes to the capturing stream
      s = step_enqueue(m, hist);
      m->stream = keep;
      const cudaError_t ec = cudaStreamEndCapture(m->gstream, &graph);
      if (s != LGDM_OK) {
        if (graph) cudaGraphDestroy(graph);
        return s;
      }
      if (ec != cudaSuccess) return fail(LGDM_ERR_CUDA, "step capture: %s", cudaGetErrorString(ec));
      const cudaError_t ei = cudaGraphInstantiate(&g->exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ei != cudaSuccess) return fail(LGDM_ERR_CUDA, "step graph instantiate: %s", cudaGetErrorString(ei));
      g->launches = m->launches - l0;
      m->launches = l0;
      g->dofs = m->dofs;
      g->k0g = m->k0g;
      g->alg = m->alg;
      g->kernel = m->kernel;
      g->flags = flags;
      g->comm = (void*)m->comm;
    }
    CU(cudaGraphLaunch(g->exec, m->gstream));
    m->launches += g->launches;
    CU(cudaEventRecord(m->gev_out, m->gstream));
    CU(cudaStreamWaitEvent(m->stream, m->gev_out, 0));
  }
  CU(cudaStreamSynchronize(m->stream));
  out2[0] = std::sqrt(m->host_pinned[0]);
  out2[1] = std::sqrt(m->host_pinned[1]);
  return LGDM_OK;
}

lgdm_status lgdm_set_comm(lgdm_mesh m, const void* uid, int nranks, int rank) {
  if (!m || !uid || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(LGDM_ERR_INVALID_ARGUMENT, "bad communicator arguments");
  if (!load_nccl()) return fail(LGDM_ERR_UNSUPPORTED, "cannot dlopen libnccl.so.2");
  CU(cudaSetDevice(m->device));
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  if (m->comm) g_nccl.commDestroy(m->comm), m->comm = nullptr;
  ncclResult_t r = g_nccl.commInitRank(&m->comm, nranks, id, rank);
  if (r != ncclSuccess)
    return fail(LGDM_ERR_NCCL, "ncclCommInitRank: %s", g_nccl.getErrorString ? g_nccl.getErrorString(r) : "?");
  m->nranks = nranks;
  m->rank = rank;
  m->halo_ok = false;
  if (nranks > 1) {
    // the Newton pieces' halo exchange assumes row-owned slabs in rank order: rank p's first
    // owned node follows rank p-1's last owned node, rank p's lower ghosts are rank p-1's
    // last owned nodes / dofs and rank p-1's upper ghosts rank p's first ones (the two counts
    // may differ: a mixed-order slab keeps two lattice rows below, one above).  All-gather
    // every rank's ranges and check; a layout that does not fit leaves the Newton pieces
    // unsupported (the assembly and the residual norms do not depend on it).
    const DofRange d = dof_range(m);
    const int64_t mine[8] = {m->gid0, m->own_b, m->own_e, m->n_nodes, d.col_off, d.own_b, d.own_e, d.nloc};
    int64_t* buf = nullptr;
    CU(dalloc(&buf, size_t(8) * (nranks + 1)));
    std::vector<int64_t> all(size_t(8) * nranks);
    CU(cudaMemcpyAsync(buf, mine, 64, cudaMemcpyHostToDevice, m->stream));
    r = g_nccl.allGather(buf, buf + 8, 8, ncclInt64, m->comm, m->stream);
    if (r == ncclSuccess) {
      cudaMemcpyAsync(all.data(), buf + 8, all.size() * 8, cudaMemcpyDeviceToHost, m->stream);
      cudaStreamSynchronize(m->stream);
    }
    cudaFree(buf);
    if (r != ncclSuccess)
      return fail(LGDM_ERR_NCCL, "ncclAllGather: %s", g_nccl.getErrorString ? g_nccl.getErrorString(r) : "?");
    // (per rank: gid0, own_b, own_e, n_nodes, dof col_off, dof own_b, dof own_e, dof nloc)
    bool ok = all[1] == 0 && all[5] == 0 && all[size_t(8) * (nranks - 1) + 2] == all[size_t(8) * (nranks - 1) + 3] &&
              all[size_t(8) * (nranks - 1) + 6] == all[size_t(8) * (nranks - 1) + 7];
    for (int p = 1; p < nranks && ok; ++p) {
      const int64_t* a = &all[size_t(8) * (p - 1)];
      const int64_t* b = &all[size_t(8) * p];
      ok = a[0] + a[2] == b[0] + b[1] && a[4] + a[6] == b[4] + b[5] &&   // owned ranges adjoin
           b[1] <= a[2] - a[1] && b[5] <= a[6] - a[5] &&                  // lower ghosts in p-1's
           a[3] - a[2] <= b[2] - b[1] && a[7] - a[6] <= b[6] - b[5];      // upper ghosts in p's
    }
    m->halo_ok = ok;
    if (ok) {
      const int64_t* me = &all[size_t(8) * rank];
      m->halo_recv_lo = me[5];
      m->halo_recv_hi = me[7] - me[6];
      m->halo_send_lo = rank > 0 ? all[size_t(8) * (rank - 1) + 7] - all[size_t(8) * (rank - 1) + 6] : 0;
      m->halo_send_hi = rank + 1 < nranks ? all[size_t(8) * (rank + 1) + 5] : 0;
    }
  }
  return LGDM_OK;
}

lgdm_status lgdm_nccl_unique_id(void* out, int64_t out_bytes) {
  if (!out || out_bytes < int64_t(sizeof(ncclUniqueId)))
    return fail(LGDM_ERR_INVALID_ARGUMENT, "need %d bytes", int(sizeof(ncclUniqueId)));
  if (!load_nccl()) return fail(LGDM_ERR_UNSUPPORTED, "cannot dlopen libnccl.so.2");
  ncclUniqueId id;
  ncclResult_t r = g_nccl.getUniqueId(&id);
  if (r != ncclSuccess) return fail(LGDM_ERR_NCCL, "ncclGetUniqueId failed");
  std::memcpy(out, &id, sizeof(id));
  return LGDM_OK;
}

lgdm_status lgdm_get_kappa(lgdm_mesh m, double* host_out) {
  if (!m || !host_out) return fail(LGDM_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!m->have_kappa) return fail(LGDM_ERR_INVALID_STATE, "kappa never set");
  CU(cudaSetDevice(m->device));
  CU(cudaMemcpyAsync(host_out, m->kappa, size_t(m->n_elems) * m->f.ngp * 8, cudaMemcpyDeviceToHost, m->stream));
  CU(cudaStreamSynchronize(m->stream));
  return LGDM_OK;
}

lgdm_status lgdm_scale_dofs(lgdm_mesh m, double sc) {
  if (!m) return fail(LGDM_ERR_INVALID_ARGUMENT, "mesh is NULL");
  if (!m->have_state) return fail(LGDM_ERR_INVALID_STATE, "scale before set_state");
  CU(cudaSetDevice(m->device));
  const int64_t n = m->n_dofs_local;
  k_scale<<<unsigned((n + 255) / 256), 256, 0, m->stream>>>(n, sc, m->dofs);
  return check_launch(m, "k_scale");
}

lgdm_status lgdm_set_kernel(lgdm_mesh m, int kernel) {
  if (!m || kernel < 0 || kernel > 2) return fail(LGDM_ERR_INVALID_ARGUMENT, "bad kernel selector");
  if (m->mixed && kernel > 1) return fail(LGDM_ERR_INVALID_ARGUMENT, "mixed-order meshes: kernels 0 and 1 only");
  if (kernel >= 2 && !(m->structured && sweep_supported(m)))
    return fail(LGDM_ERR_INVALID_ARGUMENT, "sweep kernel needs a structured mesh with whole owned layers");
  m->kernel = kernel;
  return LGDM_OK;
}

lgdm_status lgdm_get_info(lgdm_mesh m, lgdm_info* info) {
  if (!m || !info) return fail(LGDM_ERR_INVALID_ARGUMENT, "NULL argument");
  info->elem_type = m->type;
  info->dim = m->f.dim;
  info->nen = m->f.nen;
  info->ndpn = m->f.ndpn;
  info->ngp = m->f.ngp;
  info->structured = (m->structured && sweep_supported(m)) ? 1 : 0;
  info->n_nodes = m->n_nodes;
  info->n_elems = m->n_elems;
  info->n_owned_nodes = m->n_owned;
  info->n_rows = m->n_rows;
  info->nnz = m->nnz;
  info->nx = m->nx;
  info->ny = m->ny;
  info->nz = m->nz;
  info->device_bytes = m->device_bytes;
  return LGDM_OK;
}

int64_t lgdm_launch_count(lgdm_mesh m) { return m ? m->launches : -1; }

void lgdm_destroy(lgdm_mesh m) {
  if (!m) return;
  cudaSetDevice(m->device);
  if (m->stream) cudaStreamSynchronize(m->stream);
  for (auto& g : m->sgraph)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (m->gstream) cudaStreamSynchronize(m->gstream), cudaStreamDestroy(m->gstream);
  if (m->gev_in) cudaEventDestroy(m->gev_in);
  if (m->gev_out) cudaEventDestroy(m->gev_out);
  if (m->comm && g_nccl.loaded) g_nccl.commDestroy(m->comm);
  void* ptrs[] = {m->coords, m->conn, m->dofs, m->kappa, m->row_ptr, m->col_idx, m->val, m->R,
                  m->nbr_ptr, m->base, m->adj_ptr, m->adj, m->scratchK, m->scratchF,
                  m->sumsq_part, m->sumsq_out, m->k0g, m->alg, m->sdv_dev, m->rp_b,
                  m->ci_b, m->val_b, m->R_b, m->sol, m->sol_part, m->fixed, m->fixinc,
                  m->doff, m->dkind, m->madj_ptr, m->madj, m->bperm, m->binv, m->dofs_back, m->gdof,
                  m->rp32, m->react_buf};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (m->host_pinned) cudaFreeHost(m->host_pinned);
  if (m->sp_descr && g_sps.loaded) g_sps.destroyDescr(m->sp_descr);
  if (m->sp_handle && g_sps.loaded) g_sps.destroy(m->sp_handle);
  if (m->cstream) cudaStreamSynchronize(m->cstream), cudaStreamDestroy(m->cstream);
  if (m->copy_ev) cudaEventDestroy(m->copy_ev);
  if (m->free_ev) cudaEventDestroy(m->free_ev);
  delete m;
}

}  // extern "C"

// lbgpu engine: device memory, sweep orchestration and the C ABI of
// include/lbgpu.h. One engine = one lattice on one GPU, all work on one
// stream. The node kernels live in kernels.cuh (fast build and bit-exact
// build); this file owns the buffers, the solve/stop logic of the
// reference's drivers, the deterministic pairwise reductions and the error
// conventions of its C API.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "../../include/lbgpu.h"
#include "casebuild.h"
#include "types.cuh"

namespace lbgpu {
namespace {

struct Fail {
  int code;
  std::string msg;
};

#define CU(call)                                                                         \
  do {                                                                                   \
    const cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                             \
      (void)cudaGetLastError(); /* a failed call must not poison the next check */       \
      throw Fail{LBGPU_E_NUMERIC, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                      " (" #call ")"};                                   \
    }                                                                                    \
  } while (0)

// NCCL is resolved at run time: a process that already loaded libnccl
// (torch.distributed bundles its own) reuses that copy, so linking the
// system library cannot shadow the one the host framework expects.
struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};

const Nccl& nccl() {
  static Nccl t = [] {
    Nccl n{};
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) {
      const char* env = getenv("LBGPU_NCCL_LIB");
      h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) throw Fail{LBGPU_E_STATE, "libnccl.so.2 not found (set LBGPU_NCCL_LIB)"};
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p) throw Fail{LBGPU_E_STATE, std::string("NCCL symbol missing: ") + name};
      return p;
    };
    n.GetUniqueId = (decltype(n.GetUniqueId))sym("ncclGetUniqueId");
    n.CommInitRank = (decltype(n.CommInitRank))sym("ncclCommInitRank");
    n.CommDestroy = (decltype(n.CommDestroy))sym("ncclCommDestroy");
    n.GroupStart = (decltype(n.GroupStart))sym("ncclGroupStart");
    n.GroupEnd = (decltype(n.GroupEnd))sym("ncclGroupEnd");
    n.Send = (decltype(n.Send))sym("ncclSend");
    n.Recv = (decltype(n.Recv))sym("ncclRecv");
    n.AllReduce = (decltype(n.AllReduce))sym("ncclAllReduce");
    n.GetErrorString = (decltype(n.GetErrorString))sym("ncclGetErrorString");
    return n;
  }();
  return t;
}

constexpr unsigned long long kNoBad = ~0ull;
constexpr unsigned long long kIdxMask = (1ull << 40) - 1;
constexpr unsigned long long kKeyStepMask = (1ull << 24) - 1;  // step field of a bad-node key

// ------------------------------------------------------------ tables
// Full-pivot Gauss-Jordan inverse (the same elimination order as the oracle
// build's Eigen stand-in, so A agrees bit-for-bit with oracle/_ref; it agrees
// with the reference's Eigen FullPivLU to round-off).
bool invert(const std::vector<double>& m, int n, std::vector<double>& out) {
  std::vector<double> a = m, inv(size_t(n) * n, 0.0);
  std::vector<int> colperm(n);
  for (int i = 0; i < n; ++i) inv[i * n + i] = 1.0, colperm[i] = i;
  double det = 1.0;
  for (int k = 0; k < n; ++k) {
    int pr = k, pc = k;
    double best = -1.0;
    for (int i = k; i < n; ++i)
      for (int j = k; j < n; ++j)
        if (std::abs(a[i * n + j]) > best) best = std::abs(a[i * n + j]), pr = i, pc = j;
    if (!(best > 0.0)) return false;
    if (pr != k) {
      for (int j = 0; j < n; ++j) std::swap(a[pr * n + j], a[k * n + j]), std::swap(inv[pr * n + j], inv[k * n + j]);
      det = -det;
    }
    if (pc != k) {
      for (int i = 0; i < n; ++i) std::swap(a[i * n + pc], a[i * n + k]);
      std::swap(colperm[pc], colperm[k]);
      det = -det;
    }
    const double p = a[k * n + k];
    det *= p;
    for (int j = 0; j < n; ++j) a[k * n + j] /= p, inv[k * n + j] /= p;
    for (int i = 0; i < n; ++i) {
      if (i == k) continue;
      const double f = a[i * n + k];
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) a[i * n + j] -= f * a[k * n + j], inv[i * n + j] -= f * inv[k * n + j];
    }
  }
  if (!(std::abs(det) > 1e-12)) return false;
  out.assign(size_t(n) * n, 0.0);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j) out[colperm[k] * n + j] = inv[k * n + j];
  return true;
}

// operator* with the reference's loop order and zero skip (matrix.cpp:24-33).
std::vector<double> matmul(const std::vector<double>& l, const std::vector<double>& r, int n) {
  std::vector<double> out(size_t(n) * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) {
      const double v = l[i * n + k];
      if (v == 0.0) continue;
      for (int j = 0; j < n; ++j) out[i * n + j] += v * r[k * n + j];
    }
  return out;
}

template <class L>
void model_rows(std::vector<double>& U, std::vector<int>& cls) {
  U.assign(L::MF * L::MF, 0.0);
  cls.assign(L::MF, 0);
  for (int i = 0; i < L::MF; ++i) {
    cls[i] = L::row_class(i);
    for (int j = 0; j < L::MF; ++j) U[i * L::MF + j] = L::U(i, j);
  }
}

// ------------------------------------------------------- pairwise tree
// pairwise_sum_fn (reduce.hpp:43-52): leaves of <= 16 terms from midpoint
// splits, each combine adding its two halves. The shape depends only on n, so
// it is built once on the host and replayed on the device. Every combine is
// one fixed addition of two fixed operands, so any schedule that runs a
// combine after its children gives the reference's bits: the ops are grouped
// by height (all children one level down or more) and each level runs in
// parallel — wide levels as their own launch, the narrow top of the tree in
// one block with a barrier per level.
__global__ void __launch_bounds__(1024) k_tree_small(const double* __restrict__, const long long* __restrict__,
                             const long long* __restrict__, int, const int2* __restrict__,
                             const int* __restrict__, int, int, double*, unsigned long long*,
                             unsigned long long*);
struct PairTree {
  static constexpr int kTopOps = 2048;  // levels narrower than this: single-block kernel
  static constexpr size_t kSmallMax = 160 * 1024;  // whole tree in one block's shared memory
  size_t small_bytes = 0;
  bool small() const { return small_bytes <= kSmallMax; }
  long long n = -1;
  int leaves = 0, ops = 0;
  long long* d_lo = nullptr;
  long long* d_hi = nullptr;
  int2* d_ops = nullptr;   // sorted by height; op k writes vals[leaves + k]
  int* d_lvl = nullptr;    // level offsets into d_ops (top levels)
  double* d_vals = nullptr;
  std::vector<int> lvl;    // level offsets, lvl.size() = levels + 1
  int top = 0;             // first level handled by the single-block kernel

  void build(long long count) {
    release();
    n = count;
    std::vector<long long> lo, hi;
    std::vector<std::pair<int, int>> tmp;  // encoded child ids
    std::vector<int> height;
    std::function<int(long long, long long)> rec = [&](long long a, long long b) -> int {
      if (b - a <= 16) {
        lo.push_back(a);
        hi.push_back(b);
        return int(lo.size() - 1);  // leaf id >= 0
      }
      const long long mid = a + (b - a) / 2;
      const int x = rec(a, mid), y = rec(mid, b);
      auto h = [&](int id) { return id >= 0 ? 0 : height[-id - 1]; };
      tmp.push_back({x, y});
      height.push_back(1 + std::max(h(x), h(y)));
      return -int(tmp.size());  // internal id -k (k = 1-based post-order)
    };
    rec(0, count);
    leaves = int(lo.size());
    ops = int(tmp.size());
    const int levels = ops ? *std::max_element(height.begin(), height.end()) : 0;
    lvl.assign(levels + 1, 0);
    for (int k = 0; k < ops; ++k) ++lvl[height[k]];  // counts at index h (1-based)
    for (int h = 1; h <= levels; ++h) lvl[h] += lvl[h - 1];  // lvl[h] = end of level h
    // lvl[h-1] .. lvl[h] is level h; stable placement keeps post-order within a level
    std::vector<int> pos(ops), fill(lvl.begin(), lvl.end());
    for (int k = 0; k < ops; ++k) pos[k] = fill[height[k] - 1]++;
    auto dec = [&](int id) { return id >= 0 ? id : leaves + pos[-id - 1]; };
    std::vector<int2> o(ops);
    for (int k = 0; k < ops; ++k) o[pos[k]] = make_int2(dec(tmp[k].first), dec(tmp[k].second));
    top = levels;
    while (top > 0 && lvl[top] - lvl[top - 1] < kTopOps) --top;  // levels top+1.. are narrow
    small_bytes = size_t(leaves + ops) * sizeof(double) + size_t(ops) * sizeof(int2) +
                  size_t(levels + 1) * sizeof(int);
    if (small_bytes <= kSmallMax) {
      static bool attr = false;
      if (!attr) {
        CU(cudaFuncSetAttribute(k_tree_small, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmallMax)));
        attr = true;
      }
    }
    CU(cudaMalloc(&d_lo, sizeof(long long) * leaves));
    CU(cudaMalloc(&d_hi, sizeof(long long) * leaves));
    CU(cudaMalloc(&d_vals, sizeof(double) * (leaves + ops + 1)));
    CU(cudaMemcpy(d_lo, lo.data(), sizeof(long long) * leaves, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_hi, hi.data(), sizeof(long long) * leaves, cudaMemcpyHostToDevice));
    if (ops) {
      CU(cudaMalloc(&d_ops, sizeof(int2) * ops));
      CU(cudaMemcpy(d_ops, o.data(), sizeof(int2) * ops, cudaMemcpyHostToDevice));
      CU(cudaMalloc(&d_lvl, sizeof(int) * lvl.size()));
      CU(cudaMemcpy(d_lvl, lvl.data(), sizeof(int) * lvl.size(), cudaMemcpyHostToDevice));
    }
  }
  void release() {
    cudaFree(d_lo), cudaFree(d_hi), cudaFree(d_ops), cudaFree(d_vals), cudaFree(d_lvl);
    d_lo = d_hi = nullptr, d_ops = nullptr, d_vals = nullptr, d_lvl = nullptr, n = -1;
    lvl.clear();
  }
};

__global__ void k_leaf_sums(const double* __restrict__ t, const long long* lo, const long long* hi,
                            int leaves, double* vals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= leaves) return;
  double s = 0.0;
  for (long long k = lo[i]; k < hi[i]; ++k) s += t[k];
  vals[i] = s;
}

// One wide level of combines [b, e).
__global__ void k_combine_level(double* vals, const int2* __restrict__ ops, int leaves, int b, int e) {
  const int k = b + blockIdx.x * blockDim.x + threadIdx.x;
  if (k < e) vals[leaves + k] = vals[ops[k].x] + vals[ops[k].y];
}

// The narrow levels first+1 .. levels in one block, a barrier between levels;
// writes the root (or the single leaf) to *out.
__global__ void __launch_bounds__(1024) k_combine_top(double* vals, const int2* __restrict__ ops,
                                                      const int* __restrict__ lvl, int leaves,
                                                      int first, int levels, int nops, double* out) {
  for (int h = first + 1; h <= levels; ++h) {
    for (int k = lvl[h - 1] + threadIdx.x; k < lvl[h]; k += blockDim.x)
      vals[leaves + k] = vals[ops[k].x] + vals[ops[k].y];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = nops ? vals[leaves + nops - 1] : vals[0];
}

// A whole small tree in one block (the objective's support plane: ~1K leaves):
// the leaf sums (each leaf's <= 16 terms loaded at once, then added in the
// reference's left-to-right order), every level's combines in shared memory,
// the root to *out. Same additions on the same operands as k_leaf_sums +
// k_combine_top, so the same bits; one launch and no global round trip per level.
constexpr int kLeafMax = 16;
__global__ void __launch_bounds__(1024) k_tree_small(const double* __restrict__ t,
                                                     const long long* __restrict__ lo,
                                                     const long long* __restrict__ hi, int leaves,
                                                     const int2* __restrict__ ops,
                                                     const int* __restrict__ lvl, int levels,
                                                     int nops, double* out, unsigned long long* fl,
                                                     unsigned long long* pub) {
  extern __shared__ double sv[];  // [leaves + ops] values, then the ops, then lvl
  int2* sop = reinterpret_cast<int2*>(sv + leaves + nops);
  int* slv = reinterpret_cast<int*>(sop + nops);
  for (int k = threadIdx.x; k < nops; k += blockDim.x) sop[k] = ops[k];
  for (int k = threadIdx.x; k <= levels && nops; k += blockDim.x) slv[k] = lvl[k];
  for (int i = threadIdx.x; i < leaves; i += blockDim.x) {
    const long long b = lo[i];
    const int m = int(hi[i] - b);
    double x[kLeafMax];
#pragma unroll
    for (int k = 0; k < kLeafMax; ++k) x[k] = k < m ? t[b + k] : 0.0;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kLeafMax; ++k)
      if (k < m) s += x[k];
    sv[i] = s;
  }
  __syncthreads();
  for (int h = 1; h <= levels; ++h) {
    for (int k = slv[h - 1] + threadIdx.x; k < slv[h]; k += blockDim.x) {
      const int2 o = sop[k];
      sv[leaves + k] = sv[o.x] + sv[o.y];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double J = nops ? sv[leaves + nops - 1] : sv[0];
    *out = J;
    if (pub) {  // the call's last kernel: its status words and J straight to
                // mapped host memory, then the words' start values (no D2H
                // copy, no reset launch before the next call)
      for (int i = 0; i < 6; ++i)
        pub[i] = i == 4 ? (unsigned long long)__double_as_longlong(J) : fl[i];
      for (int i = 0; i < 6; ++i) fl[i] = (i == 1 || i == 3) ? kNoBad : 0ull;
    }
  }
}

// The flag words' start values (a kernel: no pageable-memory copy per call).
__global__ void k_reset_flags(unsigned long long* fl) {
  const int i = threadIdx.x;
  if (i < 6) fl[i] = (i == 1 || i == 3) ? kNoBad : 0ull;
}

__global__ void k_fill_bits(unsigned long long* p, long long n, unsigned long long v) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void k_gather_design(const double* __restrict__ full, const long long* __restrict__ nodes,
                                long long n, double* __restrict__ out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = full[nodes[i]];
}

__global__ void k_scatter_design(const double* __restrict__ vals, const long long* __restrict__ nodes,
                                 long long n, double* __restrict__ w) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) w[nodes[i]] = vals[i];
}

__global__ void k_penalty_terms(const double* __restrict__ w, const long long* __restrict__ nodes,
                                long long n, double* __restrict__ t) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double wi = w[nodes[i]];
  t[i] = wi * (1.0 - wi);  // topology.cpp:46-49
}

}  // namespace
}  // namespace lbgpu

using namespace lbgpu;

struct lbgpu_engine {
  // shape / mode
  int nx = 0, ny = 0, nz = 0, dim = 2, mf = 0, mt = 0, m = 0, prec = 64, exact = 0, ck = 0;
  // x-slab geometry: nx is the local array extent; owned
  // columns are local 0..span-1 = global x0..x0+span-1.
  int gnx = 0, x0 = 0, span = 0, slab_count = 1, slab_id = 0;
  bool ghosts = false;  // ghost-column layout (always with >1 slab; one slab on request)
  // halo exchange: 0 none (one slab, periodic wrap), 1 in-process group
  // (neighbour buffers read directly), 2 NCCL (one slab per rank), 3
  // in-process P2P group (one stream per slab, any devices; the sweeps push
  // their boundary planes into the neighbours' ghosts)
  int xmode = 0;
  // In-place AA streaming (lbgpu_system_desc::streaming): f[1] == f[0] and
  // v[1] == v[0]; fpar / vpar = the current layout of each (0: O, the
  // reference layout; 1: E) -- kernels.cuh FM_O / FM_E.
  int aa = 0, fpar = 0, vpar = 0;
  int fmode() const { return aa ? 1 + fpar : 0; }
  int vmode() const { return aa ? 1 + vpar : 0; }
  void require_db(const char* what) const {
    if (aa)
      throw Fail{LBGPU_E_STATE, std::string(what) +
                                    " needs the double-buffered state (in-place streaming keeps "
                                    "no previous state for the step residual)"};
  }
  void* push_dst_l[2] = {nullptr, nullptr};  // xmode 3: this sweep's neighbour destinations
  void* push_dst_r[2] = {nullptr, nullptr};  // ([0] primal field, [1] adjoint field)
  cudaEvent_t ev_step[2] = {nullptr, nullptr};  // xmode 3: sweep k done (parity k)
  long long gstep = 0;
  lbgpu_engine* nb_left = nullptr;
  lbgpu_engine* nb_right = nullptr;
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  void* halo_buf[4] = {nullptr, nullptr, nullptr, nullptr};  // send L, send R, recv L, recv R
  cudaStream_t st_comm = nullptr;  // halo traffic overlaps the interior columns
  cudaEvent_t ev_bnd = nullptr, ev_halo = nullptr;
  cudaStream_t st_h2d = nullptr;        // design uploads pipelined under the first sweep
  std::vector<cudaEvent_t> ev_chunk;    // one per z-chunk of that upload (+1: start)
  cudaStream_t st_adj = nullptr;        // design pair: adjoint z-chunks behind the primal's
  std::vector<cudaEvent_t> ev_prim;     // one per primal z-chunk (+1: adjoint done)
  bool owns_stream = true;
  long long N = 0;
  int device = 0;
  Model M{};
  NodeTables T{};
  Geom G{};
  // host copies
  std::vector<uint8_t> tag, mask, code;
  std::vector<double> w, bc_T, A, relax;
  std::vector<int8_t> bc_axis, bc_sign;
  std::vector<long long> design, support, inlets, adj_side, grad_side;
  // device
  void* f[2] = {nullptr, nullptr};
  void* v[2] = {nullptr, nullptr};
  void* snap = nullptr;  // rollback copy for exact tol-stop in batched solves
  void* tg[2] = {nullptr, nullptr};  // tangent df (post-collision pull layout), lazily
  int tc = 0;
  double* d_dw = nullptr;            // tangent direction on the full grid
  void* d_mom = nullptr;             // frozen adjoint base: moments + face scalars (k_base_moments)
  const void* mom_base = nullptr;    // the base d_mom currently describes (inside a scope)
  double tangent_drho = 0.0;         // 3 * d_inlet_dp
  double inlet_dp = 0.0;             // ModelParams::inlet_dp (rho_in = 1 + 3 inlet_dp)
  int fc = 0, vc = 0;
  uint8_t* d_code = nullptr;
  double *d_w = nullptr, *d_bcT = nullptr, *d_p0 = nullptr, *d_p1 = nullptr;
  double *d_A = nullptr, *d_At = nullptr;
  long long *d_design = nullptr, *d_support = nullptr, *d_inlets = nullptr;
  long long* d_adj_side = nullptr;
  long long* d_grad_side = nullptr;
  double *d_terms = nullptr, *d_grad = nullptr, *d_scalar = nullptr;
  double* d_ref = nullptr;
  double* d_wvals = nullptr;  // staging for design-order uploads
  bool w_host_stale = false;  // device w moved ahead of the host copy
  // [resid, bad, aux, adjoint bad, J (bits), upload timeout]: one D2H read per call
  unsigned long long* d_flags = nullptr;
  unsigned long long* d_ring = nullptr;   // per-step residual ring for batched solves
  unsigned long long* h_flags = nullptr;  // pinned mirror
  volatile unsigned long long* h_pub = nullptr;  // mapped: words published by k_tree_small
  unsigned long long* d_pub = nullptr;           // its device address
  PairTree tree_support, tree_design, tree_inlet;
  cudaStream_t st = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  long long primal_steps = 0, adjoint_steps = 0, tangent_steps = 0;
  // Step keys of bad-node reports are relative to these (set by reset_flags,
  // and per batch in solve()), so a key's 24-bit step field never wraps over
  // an engine's lifetime; reports add the caller's iteration offset.
  long long kb_p = 0, kb_a = 0, kb_t = 0;
  long long launches = 0;  // kernels this engine launched (sweeps + reductions + layout)
  std::vector<cudaEvent_t> evs;  // per-sweep timing events (lbgpu_time_pairs)
  std::string err;

  size_t bytes_per_real() const { return prec == 64 ? 8 : 4; }
  size_t field_bytes() const { return bytes_per_real() * size_t(m) * size_t(N); }

  ~lbgpu_engine() {
    if (!st) return;  // host-only instance (lbgpu_case_tables)
    if (comm) nccl().CommDestroy(comm);
    if (ev_bnd) cudaEventDestroy(ev_bnd);
    for (cudaEvent_t ev : ev_step)
      if (ev) cudaEventDestroy(ev);
    if (ev_halo) cudaEventDestroy(ev_halo);
    if (st_comm) cudaStreamDestroy(st_comm);
    for (cudaEvent_t ev : ev_chunk) cudaEventDestroy(ev);
    if (st_h2d) cudaStreamDestroy(st_h2d);
    for (cudaEvent_t ev : ev_prim) cudaEventDestroy(ev);
    if (st_adj) cudaStreamDestroy(st_adj);
    for (void* h : halo_buf) cudaFree(h);
    if (device >= 0) cudaSetDevice(device);
    if (aa) f[1] = v[1] = nullptr;  // aliases of f[0] / v[0]
    for (void* p : {f[0], f[1], v[0], v[1], snap, tg[0], tg[1]}) cudaFree(p);
    cudaFree(d_dw), cudaFree(d_mom);
    cudaFree(d_code), cudaFree(d_w), cudaFree(d_bcT), cudaFree(d_p0), cudaFree(d_p1);
    cudaFree(d_A), cudaFree(d_At), cudaFree(d_design), cudaFree(d_support), cudaFree(d_inlets);
    cudaFree(d_adj_side), cudaFree(d_grad_side), cudaFree(d_wvals), cudaFree(d_w2);
    cudaFree(d_wgate), cudaFree(d_inbox);
    cudaFree(d_terms), cudaFree(d_grad), cudaFree(d_scalar), cudaFree(d_ref), cudaFree(d_flags);
    cudaFree(d_ring);
    if (h_flags) cudaFreeHost(h_flags);
    if (h_pub) cudaFreeHost(const_cast<unsigned long long*>(h_pub));
    tree_support.release(), tree_design.release(), tree_inlet.release();
    for (cudaEvent_t ev : evs) cudaEventDestroy(ev);
    for (cudaEvent_t ev : trace_ev) cudaEventDestroy(ev);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (st && owns_stream) cudaStreamDestroy(st);
  }

  // ------------------------------------------------------------ setup
  // Host half: validation, tables, node codes (no CUDA calls).
  void setup_host(const lbgpu_system_desc& d) {
    if (d.nx < 1 || d.ny < 1 || d.nz < 1) throw Fail{LBGPU_E_CONFIG, "lattice extents must be positive"};
    if (d.precision != 64 && d.precision != 32) throw Fail{LBGPU_E_CONFIG, "precision must be 32 or 64"};
    if (d.exact && d.precision != 64)
      throw Fail{LBGPU_E_CONFIG, "the bit-exact build is double precision only"};
    if (!d.tag || !d.bc_T || !d.bc_axis || !d.bc_sign || !d.w || !d.design_mask ||
        (!d.support && d.n_support > 0))
      throw Fail{LBGPU_E_ARG, "system description is missing a per-node table"};
    nx = d.nx, ny = d.ny, nz = d.nz, prec = d.precision, exact = d.exact ? 1 : 0;
    if (d.streaming != 0 && d.streaming != 1) throw Fail{LBGPU_E_CONFIG, "streaming must be 0 or 1"};
    aa = d.streaming;
    if (aa && exact)
      throw Fail{LBGPU_E_CONFIG, "in-place streaming is a product-build mode (not the bit-exact build)"};
    device = d.device;
    gnx = d.nx;
    slab_count = d.slab_count > 1 ? d.slab_count : 1;
    slab_id = slab_count > 1 ? d.slab_id : 0;
    if (slab_count > 1) {
      if (slab_id < 0 || slab_id >= slab_count) throw Fail{LBGPU_E_CONFIG, "slab id out of range"};
      if (slab_count > gnx) throw Fail{LBGPU_E_CONFIG, "more workers than lattice columns"};
      decompose(gnx, slab_count, slab_id, x0, span);
      nx = lbgpu_slab_nxl(span);
      ghosts = true;
    } else if (d.slab_id == -1) {  // one slab in ghost layout: a single-rank ring
      x0 = 0, span = gnx, slab_id = 0;
      nx = lbgpu_slab_nxl(span);
      ghosts = true;
    } else {
      x0 = 0, span = gnx;
    }
    N = (long long)nx * ny * nz;
    // the sweeps address nodes with 32-bit offsets (kernels.cuh Nbr)
    if (N > 0x7fffffffll) throw Fail{LBGPU_E_CONFIG, "more than 2^31 - 1 nodes on one device: split into slabs"};
    dim = nz == 1 ? 2 : 3;
    mf = dim == 2 ? LatD2::MF : LatD3::MF;
    mt = dim == 2 ? LatD2::MT : LatD3::MT;
    m = mf + mt;
    if (d.vel || d.opp) check_lattice(d);
    if (!(d.nu > 0)) throw Fail{LBGPU_E_CONFIG, "viscosity must be positive"};
    if (d.beta_fluid < 0 || d.beta_solid < 0) throw Fail{LBGPU_E_CONFIG, "diffusivities must be non-negative"};
    if (!(d.u_clamp > 0)) throw Fail{LBGPU_E_CONFIG, "velocity clamp must be positive"};
    if (!(d.switch_theta > 0)) throw Fail{LBGPU_E_CONFIG, "switching exponent must be positive"};
    build_model(d);
    // tags (TagMap::validate, collision.cpp:8-23)
    tag.assign(d.tag, d.tag + N);
    bc_T.assign(d.bc_T, d.bc_T + N);
    bc_axis.assign(d.bc_axis, d.bc_axis + N);
    bc_sign.assign(d.bc_sign, d.bc_sign + N);
    w.assign(d.w, d.w + N);
    mask.assign(d.design_mask, d.design_mask + N);
    for (long long i = 0; i < N; ++i) {
      if (tag[i] > 4) throw Fail{LBGPU_E_CONFIG, "unknown node tag"};
      if (tag[i] == TAG_INLET || tag[i] == TAG_OUTLET) {
        if (bc_axis[i] < 0 || bc_axis[i] > 2 || (dim == 2 && bc_axis[i] == 2))
          throw Fail{LBGPU_E_CONFIG, "pressure node has a normal off the lattice axes"};
        if (bc_sign[i] != 1 && bc_sign[i] != -1)
          throw Fail{LBGPU_E_CONFIG, "pressure node normal sign must be +1 or -1"};
      }
      if (!std::isfinite(bc_T[i])) throw Fail{LBGPU_E_CONFIG, "prescribed temperature is not finite"};
      const bool owned = (i % nx) < span;
      if (mask[i] && owned) design.push_back(i);
      if (tag[i] == TAG_INLET && owned) inlets.push_back(i);
    }
    M.obj_kind = d.obj_kind, M.flux_axis = d.flux_axis, M.flux_sign = d.flux_sign;
    M.obj_on = 1;
    if (d.obj_kind < 0 || d.obj_kind > 2) throw Fail{LBGPU_E_CONFIG, "unknown objective kind"};
    if (d.n_support > 0) support.assign(d.support, d.support + d.n_support);
    for (size_t k = 0; k < support.size(); ++k)
      if (support[k] < 0 || support[k] >= N || (k && support[k] <= support[k - 1]))
        throw Fail{LBGPU_E_CONFIG, "objective support must be ascending node indices"};
    build_codes();
  }

  void setup(const lbgpu_system_desc& d) {
    setup_host(d);
    CU(cudaSetDevice(device));
    CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CU(cudaEventCreate(&ev0));
    CU(cudaEventCreate(&ev1));
    const size_t fb = field_bytes();
    for (int b = 0; b < (aa ? 1 : 2); ++b) {
      CU(cudaMalloc(&f[b], fb));
      CU(cudaMalloc(&v[b], fb));
      CU(cudaMemset(v[b], 0, fb));
    }
    if (aa) f[1] = f[0], v[1] = v[0];
    CU(cudaMalloc(&d_code, N));
    CU(cudaMalloc(&d_w, sizeof(double) * N));
    CU(cudaMalloc(&d_bcT, sizeof(double) * N));
    CU(cudaMemcpy(d_code, code.data(), N, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_w, w.data(), sizeof(double) * N, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_bcT, bc_T.data(), sizeof(double) * N, cudaMemcpyHostToDevice));
    CU(cudaMalloc(&d_A, sizeof(double) * mf * mf));
    CU(cudaMalloc(&d_At, sizeof(double) * mf * mf));
    std::vector<double> At(size_t(mf) * mf);
    for (int i = 0; i < mf; ++i)
      for (int j = 0; j < mf; ++j) At[j * mf + i] = A[i * mf + j];
    CU(cudaMemcpy(d_A, A.data(), sizeof(double) * mf * mf, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_At, At.data(), sizeof(double) * mf * mf, cudaMemcpyHostToDevice));
    M.A = d_A, M.At = d_At;
    auto up_list = [&](const std::vector<long long>& h, long long*& dptr) {
      CU(cudaMalloc(&dptr, sizeof(long long) * std::max<size_t>(h.size(), 1)));
      if (!h.empty())
        CU(cudaMemcpy(dptr, h.data(), sizeof(long long) * h.size(), cudaMemcpyHostToDevice));
    };
    up_list(design, d_design);
    up_list(support, d_support);
    up_list(inlets, d_inlets);
    // adjoint side list: support nodes whose partial needs the full
    // populations (synthetic objective) or that sit on a pressure face
    for (long long i : support)
      if (M.obj_kind == 2 || tag[i] == TAG_INLET || tag[i] == TAG_OUTLET) adj_side.push_back(i);
    up_list(adj_side, d_adj_side);
    // design positions on non-Interior nodes: the gradient's dual side launch
    for (size_t i = 0; i < design.size(); ++i)
      if (tag[design[i]] != TAG_INTERIOR) grad_side.push_back((long long)i);
    up_list(grad_side, d_grad_side);
    const size_t nt = std::max({design.size(), support.size(), inlets.size(), size_t(1)});
    CU(cudaMalloc(&d_terms, sizeof(double) * nt));
    CU(cudaMalloc(&d_grad, sizeof(double) * std::max<size_t>(design.size(), 1)));
    CU(cudaMalloc(&d_scalar, sizeof(double) * 4));
    CU(cudaMalloc(&d_flags, sizeof(unsigned long long) * 6));
    CU(cudaMalloc(&d_ring, sizeof(unsigned long long) * kRing));
    CU(cudaMallocHost(&h_flags, sizeof(unsigned long long) * (4 + kRing)));
    {
      void* hp = nullptr;
      CU(cudaHostAlloc(&hp, sizeof(unsigned long long) * 8, cudaHostAllocMapped));
      h_pub = static_cast<volatile unsigned long long*>(hp);
      CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_pub), hp, 0));
    }
    tree_support.build((long long)support.size());
    tree_design.build((long long)design.size());
    tree_inlet.build((long long)inlets.size());
    reset_flags();
    if (exact) {
      CU(cudaMalloc(&d_p0, sizeof(double) * N));
      CU(cudaMalloc(&d_p1, sizeof(double) * N));
      refresh_pow_tables();
    }
    T.code = d_code, T.w = d_w, T.w_adj = d_w, T.bcT = d_bcT, T.p0 = d_p0, T.p1 = d_p1;
    T.grad_side = d_grad_side, T.n_grad_side = (long long)grad_side.size();
    G = Geom{nx, ny, nz, 0, span, N, x0, gnx, ny};
    init_state();
    CU(cudaStreamSynchronize(st));
  }

  static constexpr int kRing = 64;

  void check_lattice(const lbgpu_system_desc& d) {
    for (int p = 0; p < m; ++p) {
      const int e0 = dim == 2 ? cvel<LatD2>(p, 0) : cvel<LatD3>(p, 0);
      const int e1 = dim == 2 ? cvel<LatD2>(p, 1) : cvel<LatD3>(p, 1);
      const int e2 = dim == 2 ? cvel<LatD2>(p, 2) : cvel<LatD3>(p, 2);
      const int o = dim == 2 ? copp<LatD2>(p) : copp<LatD3>(p);
      if (d.vel && (d.vel[3 * p] != e0 || d.vel[3 * p + 1] != e1 || d.vel[3 * p + 2] != e2))
        throw Fail{LBGPU_E_CONFIG, "coupled velocity table does not match the engine's lattice"};
      if (d.opp && d.opp[p] != o)
        throw Fail{LBGPU_E_CONFIG, "coupled opposite map does not match the engine's lattice"};
    }
  }

  // ModelTables::build (collision.cpp:46-71) and the fast-path factors.
  void build_model(const lbgpu_system_desc& d) {
    const double om = 1.0 / (0.5 + 3.0 * d.nu);
    std::vector<double> U;
    std::vector<int> cls;
    if (dim == 2) model_rows<LatD2>(U, cls);
    else model_rows<LatD3>(U, cls);
    const bool bgk = d.collision == 1;
    if (d.relax) {
      relax.assign(d.relax, d.relax + mf);
    } else if (bgk) {
      relax.assign(mf, om);
    } else {
      relax.assign(mf, d.omega_nonhydro);
      for (int i = 0; i < mf; ++i) {
        if (cls[i] == 1) relax[i] = om;
        if (cls[i] == 0) relax[i] = 1.0;
      }
    }
    if (d.A) {
      A.assign(d.A, d.A + mf * mf);
    } else {
      std::vector<double> Ub, Ubinv;
      if (bgk) {
        Ub.assign(mf * mf, 0.0);
        for (int i = 0; i < mf; ++i) Ub[i * mf + i] = 1.0;
        Ubinv = Ub;
      } else {
        Ub = U;
        if (!invert(Ub, mf, Ubinv)) throw Fail{LBGPU_E_CONFIG, "matrix not invertible (|det| <= tolerance)"};
      }
      std::vector<double> imt(mf * mf, 0.0);
      for (int i = 0; i < mf; ++i) imt[i * mf + i] = 1.0 - relax[i];
      A = matmul(Ubinv, matmul(imt, Ub, mf), mf);
    }
    M.om = om;
    M.beta_f = d.beta_fluid, M.beta_s = d.beta_solid;
    inlet_dp = d.inlet_dp;
    set_rho_in(1.0 + 3.0 * d.inlet_dp);
    M.rho_out = 1.0;
    M.u_clamp = d.u_clamp;
    M.inv_rho_in = 1.0 / M.rho_in, M.inv_rho_out = 1.0 / M.rho_out;
    M.inv_1m_uc = 1.0 / (1.0 - d.u_clamp), M.inv_1p_uc = 1.0 / (1.0 + d.u_clamp);
    M.theta = d.switch_theta;
    M.theta_int = (d.switch_theta == std::floor(d.switch_theta) && d.switch_theta >= 1 &&
                   d.switch_theta <= 16) ? int(d.switch_theta) : 0;
    M.fluid_power = d.switch_form == 1;
    M.collision_bgk = bgk;
    // Fast MRT: A = U^T diag(c) U with c_i = (1 - relax_i)/|U_i|^2 needs
    // mutually orthogonal moment rows; both bases are.
    M.nonhydro = 0;
    for (int i = 0; i < mf; ++i) {
      double n2 = 0.0;
      for (int j = 0; j < mf; ++j) n2 += U[i * mf + j] * U[i * mf + j];
      M.mrt_c[i] = (1.0 - relax[i]) / n2;
      if (cls[i] == 2 && relax[i] != 1.0) M.nonhydro = 1;
      for (int k = 0; k < i; ++k) {
        double dot = 0.0;
        for (int j = 0; j < mf; ++j) dot += U[i * mf + j] * U[k * mf + j];
        if (std::abs(dot) > 1e-12) throw Fail{LBGPU_E_CONFIG, "moment basis is not orthogonal"};
      }
    }
    ck = bgk ? 0 : (M.nonhydro ? 2 : 1);
    // Non-design nodes (w == 1): the pow pair and thermal rate are constants.
    const double base1 = M.fluid_power ? 1.0 : 0.0;
    T.pp_one = {std::pow(base1, M.theta), std::pow(base1, M.theta - 1.0)};
    if (prec == 64) {
      const double beta = 1.0 * M.beta_f + (1.0 - 1.0) * M.beta_s;
      T.omt_one = 1.0 / (0.5 + 3.0 * beta);
    } else {
      const float wf = 1.0f, beta = wf * float(M.beta_f) + (1.0f - wf) * float(M.beta_s);
      T.omt_one = double(1.0f / (0.5f + 3.0f * beta));
    }
  }

  void build_codes() {
    code.assign(N, 0);
    std::vector<uint8_t> on_support(N, 0);
    for (long long i : support) on_support[i] = 1;
    for (long long i = 0; i < N; ++i) {
      uint8_t c = tag[i];
      if (mask[i] || w[i] != 1.0) c |= CODE_HAS_W;
      if (mask[i] && tag[i] == TAG_INTERIOR) c |= CODE_DESIGN_INT;  // no face normal here
      if (on_support[i]) c |= CODE_SUPPORT;
      if (tag[i] == TAG_INLET || tag[i] == TAG_OUTLET) {
        c |= uint8_t(bc_axis[i] << CODE_AXIS_SHIFT);
        if (bc_sign[i] < 0) c |= CODE_NEG;
      }
      code[i] = c;
    }
  }

  // Exact build: pow(base, theta) / pow(base, theta-1) from the host libm,
  // exactly the calls switching_eval / switching_derivative / pow(Dual) make
  // (topology.hpp:42-46, topology.cpp:34-38, dual.hpp:56-61).
  void refresh_pow_tables() {
    std::vector<double> p0(N, 0.0), p1(N, 0.0);
    for (long long i = 0; i < N; ++i) {
      if (!(code[i] & CODE_HAS_W)) continue;
      const double base = M.fluid_power ? w[i] : 1.0 - w[i];
      p0[i] = std::pow(base, M.theta);
      p1[i] = std::pow(base, M.theta - 1.0);
    }
    CU(cudaMemcpyAsync(d_p0, p0.data(), sizeof(double) * N, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(d_p1, p1.data(), sizeof(double) * N, cudaMemcpyHostToDevice, st));
    CU(cudaStreamSynchronize(st));
  }

  // ------------------------------------------------------------ helpers
  // d_flags: [0] residual, [1] first bad node (primal, or the call's only
  // sweep kind), [2] aux, [3] first bad node of the adjoint half of a pair call
  // flags_clean: the last flag-touching operation was a design pair whose
  // final kernel published and reset the words (k_tree_small), so the next
  // reset needs no launch. Any reset or Launch clears it.
  mutable bool flags_clean = false;
  void reset_flags() {
    if (!flags_clean) k_reset_flags<<<1, 32, 0, st>>>(d_flags);
    flags_clean = false;
    kb_p = primal_steps, kb_a = adjoint_steps, kb_t = tangent_steps;
  }
  // step: the sweep's number relative to the current key base (1-based)
  Launch launch(unsigned long long step) const {
    flags_clean = false;
    Launch a;
    a.g = G;
    a.t = T;
    a.M = M;
    a.fl.resid = d_flags;
    a.fl.bad = d_flags + 1;
    a.fl.aux = d_flags + 2;
    a.fl.step_key = (step & kKeyStepMask) << 40;
    a.stream = st;
    return a;
  }
  SweepArgs sweep(unsigned long long step, bool resid, unsigned long long* resid_slot) const {
    SweepArgs s;
    s.a = launch(step);
    if (resid_slot) s.a.fl.resid = resid_slot;
    s.dim = dim, s.prec = prec, s.ck = ck, s.resid = resid;
    s.adj_side = d_adj_side, s.n_adj_side = (long long)adj_side.size();
    s.part = 0;
    s.fm = fmode(), s.vm = vmode();
    return s;
  }
  void sync() { CU(cudaStreamSynchronize(st)); }
  void pull_flags() {
    CU(cudaMemcpyAsync(h_flags, d_flags, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, st));
    sync();
  }
  // NumericError with the reference's message shape (collision.cpp:355-361,
  // 387-389): the iteration is `base` plus the key's call-relative step.
  void raise_bad(unsigned long long key, const char* what, long long base = 0) {
    const long long gidx = (long long)(key & kIdxMask);
    const long long step = base + (long long)(key >> 40);
    // keys hold the GLOBAL flat index (gflat): decode with the global x extent
    const int x = int(gidx % gnx), y = int((gidx / gnx) % ny), z = int(gidx / ((long long)gnx * ny));
    reset_flags();
    throw Fail{LBGPU_E_NUMERIC, "non-positive density at node (" + std::to_string(x) + "," +
                                    std::to_string(y) + "," + std::to_string(z) + ") (" + what +
                                    " " + std::to_string(step) + ")"};
  }
  void check_bad(const char* what) {
    pull_flags();
    if (h_flags[1] != kNoBad) raise_bad(h_flags[1], what);
  }
  static double bits_to_double(unsigned long long b) {
    double d;
    std::memcpy(&d, &b, sizeof d);
    return d;
  }

  // ------------------------------------------------------------ sweeps
  // NCCL mode: the boundary strips first, their halo on the comm stream
  // while the interior columns compute, joined before the next sweep.
  // kind: the exchange after the sweep (0 double-buffered; in place: 1 forward
  // after a sweep from O, 2 reverse after a sweep from E; kernels.cuh)
  template <class F>
  void overlapped(int field, void* dst, SweepArgs s, F&& launch_part, int kind = 0) {
    s.part = 2;
    launch_part(s);
    CU(cudaEventRecord(ev_bnd, st));
    CU(cudaStreamWaitEvent(st_comm, ev_bnd, 0));
    nccl_exchange(field, dst, st_comm, kind);
    CU(cudaEventRecord(ev_halo, st_comm));
    s.part = 1;
    launch_part(s);
    CU(cudaStreamWaitEvent(st, ev_halo, 0));
    launches += 1;
  }

  // One primal sweep src -> dst (and, in NCCL mode, the halo of dst).
  void primal_raw(const void* src, void* dst, bool resid, unsigned long long* slot, bool exch) {
    ++primal_steps;
    ++launches;
    SweepArgs s = sweep(primal_steps - kb_p, resid, slot);
    if (aa) {
      if (resid) require_db("a step residual");
      auto go = [&](const SweepArgs& a) { fast::primal_aa(a, dst); };
      if (exch && xmode == 2) overlapped(0, dst, s, go, 1 + fpar);
      else go(s);
      fpar ^= 1;
      return;
    }
    s.a.push = push_targets();
    auto go = [&](const SweepArgs& a) {
      if (exact) exact::primal(a, src, dst);
      else fast::primal(a, src, dst);
    };
    if (exch && xmode == 2) overlapped(0, dst, s, go);
    else go(s);
  }
  // One adjoint sweep src -> dst against the primal pull buffer `base`.
  // adj_gacc: the next gathering FP64 sweeps also accumulate the design
  // gradient of their inputs there (k_adjoint GRAD; the unsteady back step)
  double* adj_gacc = nullptr;
  void adjoint_raw(int kernel, const void* base, const void* src, void* dst, bool resid,
                   unsigned long long* slot, bool exch) {
    ++adjoint_steps;
    ++launches;
    SweepArgs s = sweep(adjoint_steps - kb_a, resid, slot);
    if (kernel == 0 && mom_base && mom_base == base && !adj_gacc) s.mom = d_mom;
    s.a.upd.gacc = adj_gacc;
    if (aa) {
      if (resid) require_db("a step residual");
      if (kernel != 0) require_db("the dual-sweep adjoint kernel");
      auto go = [&](const SweepArgs& a) { fast::adjoint_aa(a, base, dst); };
      if (exch && xmode == 2) overlapped(1, dst, s, go, 1 + vpar);
      else go(s);
      vpar ^= 1;
      return;
    }
    s.a.push = push_targets();
    auto go = [&](const SweepArgs& a) {
      if (kernel) {
        if (exact) exact::adjoint_dual(a, base, src, dst);
        else fast::adjoint_dual(a, base, src, dst);
      } else {
        if (exact) exact::adjoint(a, base, src, dst);
        else fast::adjoint(a, base, src, dst);
      }
    };
    if (exch && xmode == 2) overlapped(1, dst, s, go);
    else go(s);
  }
  // One tangent sweep of df against the frozen primal state f[fc].
  void tangent_launch(bool resid, unsigned long long* slot) {
    ++tangent_steps;
    ++launches;
    const SweepArgs s = sweep(tangent_steps - kb_t, resid, slot);
    if (exact) exact::tangent(s, f[fc], tg[tc], tg[1 - tc], d_dw, tangent_drho);
    else fast::tangent(s, f[fc], tg[tc], tg[1 - tc], d_dw, tangent_drho);
    tc ^= 1;
  }
  Push push_targets() const {
    Push p;
    if (xmode != 3) return p;
    for (int k = 0; k < 2; ++k) p.l_dst[k] = push_dst_l[k], p.r_dst[k] = push_dst_r[k];
    p.l_col = nb_left->span, p.l_nx = nb_left->nx, p.l_N = nb_left->N;
    p.r_col = nb_right->nx - 1, p.r_nx = nb_right->nx, p.r_N = nb_right->N;
    return p;
  }
  void primal_launch(bool resid, unsigned long long* slot, bool exch = true) {
    primal_raw(f[fc], f[1 - fc], resid, slot, exch);
    fc ^= 1;
  }
  void adjoint_launch(int kernel, bool resid, unsigned long long* slot, bool exch = true) {
    adjoint_raw(kernel, f[fc], v[vc], v[1 - vc], resid, slot, exch);
    vc ^= 1;
  }

  // ------------------------------------------------------------ halo
  void* cur(int field) const { return field == 0 ? f[fc] : v[vc]; }
  size_t halo_bytes() const { return bytes_per_real() * 6 * size_t(ny) * nz; }
  // one sweep's exchange for field `field` with pack / unpack ops of `kind`
  static int pack_op(int kind) { return kind == 0 ? 0 : kind == 1 ? 5 : 3; }
  static int unpack_op(int kind) { return kind == 0 ? 1 : kind == 1 ? 6 : 4; }
  void ensure_halo_bufs() {
    for (void*& h : halo_buf)
      if (!h) CU(cudaMalloc(&h, halo_bytes()));
  }
  void halo_op(int op, int field, void* a, void* b, const lbgpu_engine* l, const lbgpu_engine* r,
               void* buf = nullptr, cudaStream_t s_ = nullptr) {
    const Geom gl = l ? l->G : G, gr = r ? r->G : G;
    const void* lb = l ? l->cur(field) : nullptr;
    const void* rb = r ? r->cur(field) : nullptr;
    void* B = buf ? buf : cur(field);
    cudaStream_t S = s_ ? s_ : st;
    if (exact) exact::halo(op, G, dim, prec, field, B, a, b, lb, gl, rb, gr, S);
    else fast::halo(op, G, dim, prec, field, B, a, b, lb, gl, rb, gr, S);
    ++launches;
  }
  // Fill this slab's ghost columns of `field` after a sweep of it.
  void exchange(int field) {
    if (xmode == 1) {
      halo_op(2, field, nullptr, nullptr, nb_left, nb_right);
    } else if (xmode == 2) {
      nccl_exchange(field, cur(field), st);
    }
  }
  // pack -> NCCL send/recv with both neighbours -> unpack, all on stream S.
  void nccl_exchange(int field, void* buf, cudaStream_t S, int kind = 0) {
    {
      ensure_halo_bufs();
      halo_op(pack_op(kind), field, halo_buf[0], halo_buf[1], nullptr, nullptr, buf, S);
      const size_t cnt = halo_bytes() / bytes_per_real();
      const ncclDataType_t ty = prec == 64 ? ncclFloat64 : ncclFloat32;
      const int left = (rank - 1 + nranks) % nranks, right = (rank + 1) % nranks;
      // posting order per peer is the same on every rank, so with two ranks
      // (left == right) the i-th send meets the i-th receive
      const Nccl& N_ = nccl();
      N_.GroupStart();
      N_.Send(halo_buf[1], cnt, ty, right, comm, S);
      N_.Recv(halo_buf[2], cnt, ty, left, comm, S);
      N_.Send(halo_buf[0], cnt, ty, left, comm, S);
      N_.Recv(halo_buf[3], cnt, ty, right, comm, S);
      const ncclResult_t r = N_.GroupEnd();
      if (r != ncclSuccess) throw Fail{LBGPU_E_NUMERIC, std::string("NCCL: ") + N_.GetErrorString(r)};
      halo_op(unpack_op(kind), field, halo_buf[2], halo_buf[3], nullptr, nullptr, buf, S);
    }
  }
  // Global max / min of device flag words across ranks (NCCL mode).
  void reduce_flags(unsigned long long* d, size_t n, bool is_min) {
    if (xmode != 2) return;
    const ncclResult_t r =
        nccl().AllReduce(d, d, n, ncclUint64, is_min ? ncclMin : ncclMax, comm, st);
    if (r != ncclSuccess) throw Fail{LBGPU_E_NUMERIC, std::string("NCCL: ") + nccl().GetErrorString(r)};
  }
  void require_solo() const {
    if (xmode == 1 || xmode == 3)
      throw Fail{LBGPU_E_STATE, "slab engine in an in-process group: use lbgpu_group_* calls"};
  }

  void init_state() {
    if (exact) exact::init_state(N, dim, prec, f[fc], st);
    else fast::init_state(N, dim, prec, f[fc], st);
    // ghost layout: sweeps write owned columns only, so both ping-pong buffers
    // carry the same ghost columns until an exchange refreshes them
    if (ghosts && !aa) CU(cudaMemcpyAsync(f[1 - fc], f[fc], field_bytes(), cudaMemcpyDeviceToDevice, st));
    CU(cudaMemsetAsync(v[vc], 0, field_bytes(), st));
    fpar = vpar = 0;  // uniform planes (and zeros): layout O
    CU(cudaGetLastError());
  }

  // Several analytic adjoint sweeps against the unchanging base f[fc] (a
  // steady solve, or adjoint_step(n >= 2)): cache the base moments once so
  // each sweep skips the base gather (fast build).
  struct MomScope {
    lbgpu_engine* e;
    MomScope(lbgpu_engine* e_, long long n, int kernel) : e(e_) {
      if (e->exact || kernel != 0 || n < 2) return;
      if (!e->d_mom) CU(cudaMalloc(&e->d_mom, e->bytes_per_real() * size_t(e->dim + 7) * e->N));
      fast::base_moments(e->launch(e->adjoint_steps - e->kb_a), e->dim, e->prec, e->fmode(),
                         e->f[e->fc], e->d_mom);
      CU(cudaGetLastError());
      ++e->launches;
      e->mom_base = e->f[e->fc];
    }
    ~MomScope() { e->mom_base = nullptr; }
  };

  double steps(int which, long long n, int kernel, bool want_resid) {
    require_solo();
    if (want_resid) require_db("a step residual");
    if (n <= 0) return 0.0;
    reset_flags();
    MomScope ms(this, which == 1 ? n : 0, kernel);
    for (long long k = 0; k < n; ++k) {
      const bool r = want_resid && k == n - 1;
      if (which == 0) primal_launch(r, nullptr);
      else adjoint_launch(kernel, r, nullptr);
    }
    CU(cudaGetLastError());
    reduce_flags(d_flags, 1, false);
    reduce_flags(d_flags + 1, 1, true);
    pull_flags();
    if (h_flags[1] != kNoBad) raise_bad(h_flags[1], which == 0 ? "iteration" : "adjoint iteration");
    return want_resid ? bits_to_double(h_flags[0]) : 0.0;
  }

  // Queue the z-chunked H2D copy of design values (after everything already
  // on st): chunk c covers design positions [ib[c], ib[c+1]) = z planes
  // [zb[c], zb[c+1]); ev_chunk[c] fires when its slice has landed.
  // skew: chunk 0 = nz/32 and chunk 1 = 3nz/32 of the planes, the rest nz/8
  // each -- the first upload slice lands early, so the sweep starts early
  void design_bounds(long long* ib, int* zb, bool skew = false) const {
    const long long plane = (long long)nx * ny;
    static constexpr int kSkew[kChunks + 1] = {0, 1, 4, 8, 12, 16, 20, 24, 32};  // /32
    static_assert(kChunks == 8, "skewed chunk table");
    for (int c = 0; c <= kChunks; ++c) {
      zb[c] = skew ? int((long long)nz * kSkew[c] / 32) : int((long long)nz * c / kChunks);
      ib[c] = std::lower_bound(design.begin(), design.end(), plane * zb[c]) - design.begin();
    }
  }
  void ensure_h2d() {
    if (!d_wvals) CU(cudaMalloc(&d_wvals, sizeof(double) * std::max<size_t>(design.size(), 1)));
    if (!st_h2d) {
      CU(cudaStreamCreateWithFlags(&st_h2d, cudaStreamNonBlocking));
      ev_chunk.resize(kChunks + 1);
      for (cudaEvent_t& ev : ev_chunk) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
  }
  void queue_design_upload(const double* wd, long long* ib, int* zb, bool mark = true,
                           bool skew = false) {
    ensure_h2d();
    // the staging buffer is free once everything queued before us has run
    // (mark = false: the caller recorded ev_chunk[kChunks] on st already)
    if (mark) CU(cudaEventRecord(ev_chunk[kChunks], st));
    CU(cudaStreamWaitEvent(st_h2d, ev_chunk[kChunks], 0));
    design_bounds(ib, zb, skew);
    for (int c = 0; c < kChunks; ++c)
      if (ib[c + 1] > ib[c]) {
        CU(cudaMemcpyAsync(d_wvals + ib[c], wd + ib[c], sizeof(double) * (ib[c + 1] - ib[c]),
                           cudaMemcpyHostToDevice, st_h2d));
        CU(cudaEventRecord(ev_chunk[c], st_h2d));
      }
  }
  bool design_chunking() const {
    return !design.empty() && !exact && dim == 3 && xmode != 2 && nz >= 2 * kChunks;
  }

  // One iteration head of one_shot_run (optimizer.cpp:33-34: primal_step,
  // then adjoint_step against the new f) behind a design write-back
  // (optimizer.cpp:200-202), with J = evaluate_raw of the new state
  // (objective.cpp:64-72). Same results as primal_step_with_design(1) +
  // adjoint_step(1) + objective, bit for bit. Three overlapped pipelines:
  // the H2D copy of the design in z-chunks; the primal sweep chunk c after
  // its design slice; the adjoint sweep chunk c on a second stream after
  // primal chunk c+1 (it gathers the new f from planes z-1..z+1; chunks 0
  // and kChunks-1 also need the periodic z neighbour, so they go last).
  // C3 (LBGPU_TRACE_PAIR timeline): the 16 MB upload lands at 0.34 ms, the
  // step ends at 0.90 ms against 0.91 for the three calls; the adjoint,
  // HBM-bound, cannot start before primal chunk 2. Sweeping the design-free
  // columns first (primal, then adjoint, on a low-priority stream, the
  // design chunks on a high-priority one) measured 0.99-1.10 ms: the narrow
  // column launches run at 60% of the full sweep's rate.
  // LBGPU_TRACE_PAIR=1: print each pipeline stage's finish time (development).
  std::vector<cudaEvent_t> trace_ev;
  std::vector<std::string> trace_name;
  std::vector<double> trace_host;  // host clock at each mark (us)
  double trace_t_exit = 0.0;       // host clock when the previous traced call returned
  static double host_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }
  static bool trace_on() {
    static const bool on = std::getenv("LBGPU_TRACE_PAIR") != nullptr;
    return on;
  }
  void trace(const char* what, cudaStream_t s_) {
    if (!trace_on()) return;
    if (trace_ev.size() <= trace_name.size()) {
      trace_ev.emplace_back();
      CU(cudaEventCreate(&trace_ev.back()));
    }
    CU(cudaEventRecord(trace_ev[trace_name.size()], s_));
    trace_name.emplace_back(what);
    trace_host.push_back(host_us());
  }
  // one line per call: each mark's GPU time (ms after "start"), the host
  // clock of its enqueue (us after "start"), the host's return from the sync,
  // and the host gap since the previous traced call returned
  void trace_print() {
    if (trace_name.empty()) return;
    const double t_sync = host_us();
    CU(cudaDeviceSynchronize());
    for (size_t i = 1; i < trace_name.size(); ++i) {
      float ms = 0.f;
      CU(cudaEventElapsedTime(&ms, trace_ev[0], trace_ev[i]));
      std::fprintf(stderr, "%s %.3f (host +%.1f)  ", trace_name[i].c_str(), ms,
                   trace_host[i] - trace_host[0]);
    }
    std::fprintf(stderr, "synced host +%.1f  gap_before_call %.1f\n", t_sync - trace_host[0],
                 trace_t_exit > 0 ? trace_host[0] - trace_t_exit : 0.0);
    trace_name.clear();
    trace_host.clear();
    trace_t_exit = host_us();
  }
  void design_pair(const double* wd, double* rp, double* ra, double* J) {
    require_solo();
    require_db("the pipelined design pair");
    const bool want = rp || ra;
    if (!design_chunking()) {
      const double r = design_steps(wd, 1, want);
      const double q = steps(1, 1, 0, want);
      if (rp) *rp = r;
      if (ra) *ra = q;
      if (J) *J = objective();
      return;
    }
    if (!st_adj) {
      CU(cudaStreamCreateWithFlags(&st_adj, cudaStreamNonBlocking));
      ev_prim.resize(kChunks + 1);
      for (cudaEvent_t& ev : ev_prim) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    long long ib[kChunks + 1];
    int zb[kChunks + 1];
    reset_flags();
    CU(cudaMemsetAsync(d_ring, 0, sizeof(unsigned long long), st));
    trace_name.clear(), trace_host.clear();  // a call that raised before trace_print left its names
    trace("start", st);
    ensure_h2d();
    CU(cudaEventRecord(ev_chunk[kChunks], st));  // everything before this call
    CU(cudaStreamWaitEvent(st_adj, ev_chunk[kChunks], 0));
    queue_design_upload(wd, ib, zb, false);
    ++primal_steps;
    const void* fsrc = f[fc];
    void* fdst = f[1 - fc];
    for (int c = 0; c < kChunks; ++c) {
      const long long m_ = ib[c + 1] - ib[c];
      if (m_ > 0) {
        CU(cudaStreamWaitEvent(st, ev_chunk[c], 0));
        k_scatter_design<<<unsigned((m_ + 255) / 256), 256, 0, st>>>(d_wvals + ib[c], d_design + ib[c],
                                                                     m_, d_w);
        ++launches;
      }
      SweepArgs sa = sweep(primal_steps - kb_p, want, nullptr);
      sa.z0 = zb[c], sa.z1 = zb[c + 1];
      fast::primal(sa, fsrc, fdst);
      ++launches;
      CU(cudaEventRecord(ev_prim[c], st));
      if (trace_on()) trace(("P" + std::to_string(c)).c_str(), st);
    }
    fc ^= 1;
    w_host_stale = true;
    ++adjoint_steps;
    const void* vsrc = v[vc];
    void* vdst = v[1 - vc];
    for (int k = 0; k < kChunks; ++k) {
      const int c = k < kChunks - 1 ? k + 1 : 0;  // 1, 2, ..., kChunks-1, 0
      CU(cudaStreamWaitEvent(st_adj, ev_prim[std::min(c + 1, kChunks - 1)], 0));
      SweepArgs sa = sweep(adjoint_steps - kb_a, want, d_ring);
      sa.a.stream = st_adj;
      sa.a.fl.bad = d_flags + 3;  // the adjoint half reports after the primal's
      sa.z0 = zb[c], sa.z1 = zb[c + 1];
      if (k < kChunks - 1) sa.n_adj_side = 0;  // the side list once, after every chunk
      fast::adjoint(sa, f[fc], vsrc, vdst);
      launches += 1 + (k == kChunks - 1 && sa.n_adj_side > 0);
      if (trace_on()) trace(("A" + std::to_string(c)).c_str(), st_adj);
    }
    vc ^= 1;
    CU(cudaEventRecord(ev_prim[kChunks], st_adj));
    if (J) {  // overlaps the adjoint's tail
      fast::objective_terms(launch(primal_steps - kb_p), dim, prec, f[fc], d_support, (long long)support.size(),
                            d_terms, 0);
      ++launches;
      pairwise_queue(tree_support, d_terms);
    }
    CU(cudaStreamWaitEvent(st, ev_prim[kChunks], 0));
    CU(cudaGetLastError());
    reduce_flags(d_flags, 1, false);
    reduce_flags(d_ring, 1, false);
    reduce_flags(d_flags + 1, 1, true);
    reduce_flags(d_flags + 3, 1, true);
    CU(cudaMemcpyAsync(h_flags, d_flags, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(h_flags + 4, d_ring, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    if (J) CU(cudaMemcpyAsync(h_flags + 5, d_scalar, sizeof(double), cudaMemcpyDeviceToHost, st));
    sync();  // one host sync per call; the host design buffer is consumed too
    trace_print();
    // the primal's failure first (the three-call sequence raises before its
    // adjoint runs); on either error the adjoint half has already advanced v
    if (h_flags[1] != kNoBad) raise_bad(h_flags[1], "iteration");
    if (h_flags[3] != kNoBad) raise_bad(h_flags[3], "adjoint iteration");
    if (rp) *rp = bits_to_double(h_flags[0]);
    if (ra) *ra = bits_to_double(h_flags[4]);
    if (J) *J = bits_to_double(h_flags[5]);
  }

  // The deferred-adjoint form of the design pair (no residuals requested).
  // Call k uploads w_k and runs primal sweep k; its adjoint sweep (against
  // f^k, with w_k) is left pending and runs inside call k+1's primal sweep as
  // the adjoint half of one fused k_pair (DUALW: that half reads the previous
  // design, kept in the second w buffer), so each call streams 4 M s bytes per
  // node instead of 5 M s and the upload gates one kernel, not two. Any other
  // call flushes the pending sweep first (guarded()), so everything observable
  // -- f, v, w, J, gradients -- is bitwise the three separate calls; a rho <= 0
  // in a deferred adjoint sweep surfaces at the next call as "adjoint
  // iteration". Design buffers alternate: d_w (current, w_{k-1}) and d_w2
  // (receives w_k); outside the design nodes both hold the same values
  // (w2_synced; lbgpu_set_design clears it).
  bool adj_pending = false;
  double* d_w2 = nullptr;
  bool w2_synced = false;
  // Upload-gated single launch (kernels.cuh Gate): when the design nodes are
  // exactly a box (config-built cases: interior x the design x-range), the
  // fused sweep of a deferred pair is ONE launch behind ONE H2D copy of the
  // design vector into d_wgate: each box node's thread waits for its own value
  // to replace the sentinel and re-arms the entry -- no slices, no flags, no
  // z-chunk kernel boundaries, no scatter kernels.
  int gate_state = -1;  // -1 unknown, 0 no box, 1 box
  Gate gate_box{};
  double* d_wgate = nullptr;  // design-order upload buffer, kGateEmpty between uploads
  bool gate_armed = false;
  bool gate_ready() {
    if (gate_state >= 0) return gate_state == 1;
    gate_state = 0;
    if (design.empty() || ghosts) return false;
    int x0_ = nx, x1_ = -1, y0_ = ny, y1_ = -1, z0_ = nz, z1_ = -1;
    for (long long i : design) {
      const int x = int(i % nx), y = int((i / nx) % ny), z = int(i / ((long long)nx * ny));
      x0_ = std::min(x0_, x), x1_ = std::max(x1_, x), y0_ = std::min(y0_, y), y1_ = std::max(y1_, y);
      z0_ = std::min(z0_, z), z1_ = std::max(z1_, z);
    }
    const long long vol = (long long)(x1_ - x0_ + 1) * (y1_ - y0_ + 1) * (z1_ - z0_ + 1);
    if (vol != (long long)design.size()) return false;  // not a box: the chunked path
    gate_box.bx0 = x0_, gate_box.bx1 = x1_ + 1, gate_box.by0 = y0_, gate_box.by1 = y1_ + 1;
    gate_box.bz0 = z0_, gate_box.bz1 = z1_ + 1;
    CU(cudaMalloc(&d_wgate, sizeof(double) * design.size()));
    gate_armed = false;
    gate_state = 1;
    return true;
  }
  // The gated fused sweep of a deferred pair (adj_pending): the upload on the
  // copy stream (which waits for the work queued before this call: the
  // previous sweep's re-arming of d_wgate), THEN one k_pair launch on st.
  // Enqueueing the copy first keeps the scheme deadlock-free where launches
  // serialise with copies (CUDA_LAUNCH_BLOCKING, profilers): the values are
  // then in place when the sweep starts.
  // The upload of a gated sweep (copy stream); the caller launches the sweep
  // next and sets gate_armed again once its flags show no timeout.
  void gate_upload(const double* wd) {
    ensure_h2d();
    const long long n = (long long)design.size();
    if (!gate_armed) {  // first use, or after a timed-out upload
      k_fill_bits<<<unsigned((n + 255) / 256), 256, 0, st>>>(reinterpret_cast<unsigned long long*>(d_wgate),
                                                             n, kGateEmpty);
      ++launches;
    }
    CU(cudaEventRecord(ev_chunk[kChunks], st));
    CU(cudaStreamWaitEvent(st_h2d, ev_chunk[kChunks], 0));
    CU(cudaMemcpyAsync(d_wgate, wd, sizeof(double) * n, cudaMemcpyHostToDevice, st_h2d));
    gate_armed = false;  // until the sweep is known to have re-armed every entry
  }
  // Support plane of J for the inbox (Gate::inbox): every support node in one
  // column x = obj_plane_x with 1 <= x <= nx - 2 (config-built objectives:
  // the plane nx - 1 - plane_offset), else -1.
  int obj_plane_x = -2;  // -2: not determined yet
  double* d_inbox = nullptr;
  int obj_plane() {
    if (obj_plane_x != -2) return obj_plane_x;
    obj_plane_x = -1;
    if (support.empty() || ghosts || dim != 3) return -1;
    const int x0_ = int(support[0] % nx);
    for (long long i : support)
      if (int(i % nx) != x0_) return -1;
    if (x0_ < 1 || x0_ > nx - 2) return -1;
    CU(cudaMalloc(&d_inbox, sizeof(double) * m * (size_t)ny * nz));
    obj_plane_x = x0_;
    return obj_plane_x;
  }
  bool gated_pair(const double* wd, bool want_j) {
    gate_upload(wd);
    const int ox = want_j ? obj_plane() : -1;
    NodeTables tn = T;
    tn.w = d_w2;     // the new design's full-grid buffer (design nodes written by the sweep)
    tn.w_adj = d_w;  // the previous design (the deferred adjoint half)
    SweepArgs sa = sweep(primal_steps - kb_p, false, nullptr);
    sa.a.t = tn;
    sa.a.gate = gate_box;
    sa.a.gate.wd = d_wgate, sa.a.gate.w_out = d_w2;
    sa.a.gate.err = reinterpret_cast<unsigned*>(d_flags + 5);  // cleared by reset_flags
    sa.a.gate.obj_x = ox, sa.a.gate.inbox = d_inbox;
    sa.dualw = true;
    fast::pair(sa, f[fc], f[1 - fc], v[vc], v[1 - vc]);
    launches += 1 + (sa.n_adj_side > 0);
    if (trace_on()) trace("K", st);
    return ox >= 0;
  }
  void flush_pending() {
    if (!adj_pending) return;
    adj_pending = false;
    reset_flags();
    adjoint_launch(0, false, nullptr);
    CU(cudaGetLastError());
    reduce_flags(d_flags + 1, 1, true);
    pull_flags();
    if (h_flags[1] != kNoBad) raise_bad(h_flags[1], "adjoint iteration");
  }
  bool lazy_pair_ok() const { return design_chunking() && fuse_pairs() && !aa; }
  void design_pair_lazy(const double* wd, double* J) {
    require_solo();
    if (!d_w2) CU(cudaMalloc(&d_w2, sizeof(double) * N));
    if (!w2_synced) {
      CU(cudaMemcpyAsync(d_w2, d_w, sizeof(double) * N, cudaMemcpyDeviceToDevice, st));
      w2_synced = true;
    }
    const bool fuse = adj_pending;
    adj_pending = false;
    long long ib[kChunks + 1];
    int zb[kChunks + 1];
    trace_name.clear(), trace_host.clear();
    trace("start", st);
    reset_flags();
    ++primal_steps;
    if (fuse) ++adjoint_steps;
    const bool gated = fuse && gate_ready();
    bool published = false, inbox = false;
    if (gated) {
      inbox = gated_pair(wd, J != nullptr);
    } else {
      queue_design_upload(wd, ib, zb, true, true);
    }
    NodeTables tn = T;
    tn.w = d_w2;     // the new design (primal half)
    tn.w_adj = d_w;  // the previous one (the deferred adjoint half)
    for (int c = 0; c < (gated ? 0 : kChunks); ++c) {
      const long long m_ = ib[c + 1] - ib[c];
      if (m_ > 0) {
        CU(cudaStreamWaitEvent(st, ev_chunk[c], 0));
        k_scatter_design<<<unsigned((m_ + 255) / 256), 256, 0, st>>>(d_wvals + ib[c], d_design + ib[c],
                                                                     m_, d_w2);
        ++launches;
      }
      SweepArgs sa = sweep(primal_steps - kb_p, false, nullptr);
      sa.a.t = tn;
      sa.z0 = zb[c], sa.z1 = zb[c + 1];
      if (fuse) {
        sa.dualw = true;
        if (c < kChunks - 1) sa.n_adj_side = 0;  // the side list once, with the last chunk
        fast::pair(sa, f[fc], f[1 - fc], v[vc], v[1 - vc]);
        launches += 1 + (c == kChunks - 1 && sa.n_adj_side > 0);
      } else {
        fast::primal(sa, f[fc], f[1 - fc]);
        ++launches;
      }
      if (trace_on()) trace(("K" + std::to_string(c)).c_str(), st);
    }
    fc ^= 1;
    if (fuse) vc ^= 1;
    std::swap(d_w, d_w2);
    T.w = T.w_adj = d_w;
    w_host_stale = true;
    if (J) {
      if (inbox)  // the fused sweep left the plane's populations in the inbox
        fast::objective_inbox(launch(primal_steps - kb_p), dim, prec, d_inbox, d_support,
                              (long long)support.size(), d_terms);
      else
        fast::objective_terms(launch(primal_steps - kb_p), dim, prec, f[fc], d_support,
                              (long long)support.size(), d_terms, 0);
      ++launches;
      published = pairwise_queue(tree_support, d_terms, reinterpret_cast<double*>(d_flags + 4), true);
      if (trace_on()) trace("J", st);
    }
    CU(cudaGetLastError());
    reduce_flags(d_flags + 1, 1, true);
    if (!published)
      CU(cudaMemcpyAsync(h_flags, d_flags, sizeof(unsigned long long) * 6, cudaMemcpyDeviceToHost, st));
    sync();  // one host sync per call; the host design buffer is consumed too
    if (published)
      for (int i = 0; i < 6; ++i) h_flags[i] = h_pub[i];
    trace_print();
    if (gated && !h_flags[5]) gate_armed = true;
    if (gated && h_flags[5])
      throw Fail{LBGPU_E_NUMERIC, "design upload: a design value did not land within the sweep's wait bound"};
    if (h_flags[1] != kNoBad) raise_bad(h_flags[1], fuse ? "iteration (or the deferred adjoint iteration)" : "iteration");
    adj_pending = true;
    flags_clean = published;
    if (J) *J = bits_to_double(h_flags[4]);
  }

  // New design values (DesignField::nodes order, host memory) followed by n
  // primal sweeps: optimizer.cpp:200-202 (the MMA update's write-back, then
  // solve_fixed_point). The H2D copy overlaps the first sweep: for a
  // box-shaped design, ONE gated launch (each design node's thread waits for
  // its own value, gate_upload); otherwise z-chunks, each waiting only for
  // its own slice of the upload (design nodes ascend in flat index, i.e.
  // z-major, and a sweep node reads w only at itself). Falls back to
  // upload-then-sweep where neither applies (exact build: host pow tables;
  // 2D; NCCL halo overlap).
  static constexpr int kChunks = 8;
  double design_steps(const double* wd, long long nsteps, bool want_resid) {
    require_solo();
    require_db("the pipelined design upload");
    const long long n = (long long)design.size();
    if (!n || exact || dim == 2 || xmode == 2 || nz < 2 * kChunks) {
      upload_design_values(wd);
      return steps(0, nsteps, 0, want_resid);
    }
    if (nsteps <= 0) return 0.0;
    const bool r0 = want_resid && nsteps == 1;
    if (!r0 && gate_ready()) {
      // box-shaped design: ONE primal launch behind ONE copy, each design
      // node's thread waiting for its own value (the design pair's gate)
      reset_flags();
      ++primal_steps;
      gate_upload(wd);
      SweepArgs sa = sweep(primal_steps - kb_p, false, nullptr);
      sa.a.gate = gate_box;
      sa.a.gate.wd = d_wgate, sa.a.gate.w_out = d_w;  // == T.w: the sweep reads it back
      sa.a.gate.err = reinterpret_cast<unsigned*>(d_flags + 5);
      fast::primal(sa, f[fc], f[1 - fc]);
      ++launches;
      fc ^= 1;
      w_host_stale = true;
      for (long long k = 1; k < nsteps; ++k) primal_launch(want_resid && k == nsteps - 1, nullptr);
      CU(cudaGetLastError());
      CU(cudaMemcpyAsync(h_flags, d_flags, sizeof(unsigned long long) * 6, cudaMemcpyDeviceToHost, st));
      sync();  // also: the host buffer has been consumed when we return
      if (h_flags[5])
        throw Fail{LBGPU_E_NUMERIC, "design upload: a design value did not land within the sweep's wait bound"};
      gate_armed = true;
      if (h_flags[1] != kNoBad) raise_bad(h_flags[1], "iteration");
      return want_resid ? bits_to_double(h_flags[0]) : 0.0;
    }
    long long ib[kChunks + 1];
    int zb[kChunks + 1];
    reset_flags();
    queue_design_upload(wd, ib, zb);
    ++primal_steps;
    ++launches;
    for (int c = 0; c < kChunks; ++c) {
      const long long m_ = ib[c + 1] - ib[c];
      if (m_ > 0) {
        CU(cudaStreamWaitEvent(st, ev_chunk[c], 0));
        k_scatter_design<<<unsigned((m_ + 255) / 256), 256, 0, st>>>(d_wvals + ib[c], d_design + ib[c],
                                                                     m_, d_w);
      }
      SweepArgs sa = sweep(primal_steps - kb_p, r0, nullptr);
      sa.z0 = zb[c], sa.z1 = zb[c + 1];
      if (exact) exact::primal(sa, f[fc], f[1 - fc]);
      else fast::primal(sa, f[fc], f[1 - fc]);
    }
    launches += 2 * kChunks - 1;
    fc ^= 1;
    w_host_stale = true;
    for (long long k = 1; k < nsteps; ++k) primal_launch(want_resid && k == nsteps - 1, nullptr);
    CU(cudaGetLastError());
    reduce_flags(d_flags, 1, false);
    reduce_flags(d_flags + 1, 1, true);
    pull_flags();  // also: the host buffer has been consumed when we return
    if (h_flags[1] != kNoBad) raise_bad(h_flags[1], "iteration");
    return want_resid ? bits_to_double(h_flags[0]) : 0.0;
  }
  // lbgpu_set_design_values: design-order values -> device w (synchronous)
  void upload_design_values(const double* w_design) {
    const long long n = (long long)design.size();
    if (!n) return;
    if (!d_wvals) CU(cudaMalloc(&d_wvals, sizeof(double) * n));
    CU(cudaMemcpyAsync(d_wvals, w_design, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    k_scatter_design<<<unsigned((n + 255) / 256), 256, 0, st>>>(d_wvals, d_design, n, d_w);
    ++launches;
    CU(cudaGetLastError());
    if (exact) {  // the libm pow tables follow the host copy
      for (long long i = 0; i < n; ++i) w[design[i]] = w_design[i];
      refresh_pow_tables();
    } else {
      w_host_stale = true;
      sync();
    }
  }

  // n primal+adjoint pairs, each adjoint against the state its primal just
  // produced: one_shot_run (optimizer.cpp:25-72) at zeta = 0 without the
  // (then discarded) design gradient, and the bench step. The product build
  // runs adjoint n and primal n+1 as one fused sweep (k_pair: the shared
  // f^{n+1} gathered once, FP64); otherwise the sweeps run apart. Residuals
  // (nullable) are those of the last pair.
  // Fused pairs win at FP64 only (FP32 measured slower than the sweeps apart).
#ifndef LBGPU_FUSE_FP32
#define LBGPU_FUSE_FP32 0  // FP32 double-buffered pairs run apart (measured faster)
#endif
  bool fuse_pairs() const { return !exact && (prec == 64 || aa || LBGPU_FUSE_FP32); }
  void fused_pair_raw(bool resid) {
    ++primal_steps;
    ++adjoint_steps;
    ++launches;
    SweepArgs s = sweep(primal_steps - kb_p, resid, nullptr);
    if (aa) {
      if (resid) require_db("a step residual");
      auto go = [&](const SweepArgs& a) { fast::pair_aa(a, f[0], v[0]); };
      if (xmode == 2) {
        SweepArgs b = s;
        b.part = 2;
        go(b);
        CU(cudaEventRecord(ev_bnd, st));
        CU(cudaStreamWaitEvent(st_comm, ev_bnd, 0));
        nccl_exchange(0, f[0], st_comm, 1 + fpar);
        nccl_exchange(1, v[0], st_comm, 1 + vpar);
        CU(cudaEventRecord(ev_halo, st_comm));
        b.part = 1;
        go(b);
        CU(cudaStreamWaitEvent(st, ev_halo, 0));
        launches += 1;
      } else {
        go(s);
      }
      fpar ^= 1;
      vpar ^= 1;
      return;
    }
    void* fd = f[1 - fc];
    void* vd = v[1 - vc];
    const void* fsrc = f[fc];
    const void* vsrc = v[vc];
    s.a.push = push_targets();
    auto go = [&](const SweepArgs& a) { fast::pair(a, fsrc, fd, vsrc, vd); };
    if (xmode == 2) {
      SweepArgs b = s;
      b.part = 2;
      go(b);
      CU(cudaEventRecord(ev_bnd, st));
      CU(cudaStreamWaitEvent(st_comm, ev_bnd, 0));
      nccl_exchange(0, fd, st_comm);
      nccl_exchange(1, vd, st_comm);
      CU(cudaEventRecord(ev_halo, st_comm));
      b.part = 1;
      go(b);
      CU(cudaStreamWaitEvent(st, ev_halo, 0));
      launches += 1;
    } else {
      go(s);
    }
    fc ^= 1;
    vc ^= 1;
  }
  void pair_steps(long long n, double* rp, double* ra) {
    require_solo();
    if (n <= 0) return;
    const bool want = rp || ra;
    if (want) require_db("a step residual");
    reset_flags();
    CU(cudaMemsetAsync(d_ring, 0, sizeof(unsigned long long), st));
    if (!fuse_pairs()) {
      for (long long k = 0; k < n; ++k) {
        primal_launch(want && k == n - 1, nullptr);
        adjoint_launch(0, want && k == n - 1, d_ring);
      }
    } else {
      primal_launch(want && n == 1, nullptr);
      for (long long k = 1; k < n; ++k) fused_pair_raw(want && k == n - 1);
      adjoint_launch(0, want, d_ring);
    }
    CU(cudaGetLastError());
    reduce_flags(d_flags, 1, false);
    reduce_flags(d_ring, 1, false);
    reduce_flags(d_flags + 1, 1, true);
    CU(cudaMemcpyAsync(h_flags, d_flags, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(h_flags + 4, d_ring, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    sync();
    if (h_flags[1] != kNoBad) raise_bad(h_flags[1], "iteration");
    if (rp) *rp = bits_to_double(h_flags[0]);
    if (ra) *ra = bits_to_double(h_flags[4]);
  }

  // solve_fixed_point / solve_adjoint stop rule (collision.cpp:377-416,
  // adjoint.cpp:256-297), batched: every step writes its residual into a ring
  // slot, the host scans once per batch, and an overshoot past the first
  // r <= tol is undone from a snapshot and replayed, so the stop iteration
  // and final state are exactly the per-step loop's.
  // Small lattices are launch-bound (C1: ~5.5 us per step, of which the sweep
  // is ~1 us): full ring batches of the tol-stop solver run as a captured CUDA
  // graph of kRing sweeps (their residual slots baked in, step keys relative
  // to the batch), one graph per starting buffer parity, per solve.
  static constexpr long long kGraphMaxNodes = 1ll << 20;
  struct RingGraphs {
    cudaGraphExec_t ex[2] = {nullptr, nullptr};
    ~RingGraphs() {
      for (auto& g : ex)
        if (g) cudaGraphExecDestroy(g);
    }
  };
  void capture_ring(int which, int kernel, int par, cudaGraphExec_t* out) {
    cudaGraph_t g = nullptr;
    CU(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      for (int k = 0; k < kRing; ++k) {
        const int p = (par + k) & 1;
        SweepArgs s = sweep((unsigned long long)(k + 1), true, d_ring + k);
        if (which == 0) {
          if (exact) exact::primal(s, f[p], f[1 - p]);
          else fast::primal(s, f[p], f[1 - p]);
        } else if (which == 1) {
          if (kernel == 0 && mom_base && mom_base == f[fc]) s.mom = d_mom;
          if (kernel) {
            if (exact) exact::adjoint_dual(s, f[fc], v[p], v[1 - p]);
            else fast::adjoint_dual(s, f[fc], v[p], v[1 - p]);
          } else {
            if (exact) exact::adjoint(s, f[fc], v[p], v[1 - p]);
            else fast::adjoint(s, f[fc], v[p], v[1 - p]);
          }
        } else {
          if (exact) exact::tangent(s, f[fc], tg[p], tg[1 - p], d_dw, tangent_drho);
          else fast::tangent(s, f[fc], tg[p], tg[1 - p], d_dw, tangent_drho);
        }
      }
      CU(cudaGetLastError());
    } catch (...) {
      cudaStreamEndCapture(st, &g);
      if (g) cudaGraphDestroy(g);
      (void)cudaGetLastError();
      throw;
    }
    CU(cudaStreamEndCapture(st, &g));
    const cudaError_t r = cudaGraphInstantiate(out, g, 0);
    cudaGraphDestroy(g);
    CU(r);
  }

  void solve(int which, double tol, long long max_iter, long long fixed, int kernel,
             long long* iters, double* resid, int* conv, bool reset_v = true) {
    require_solo();
    require_db("a solve (its stop rule reads the step residual)");
    const long long n = fixed >= 0 ? fixed : max_iter;
    const char* what = which == 0 ? "iteration" : which == 1 ? "adjoint iteration" : "tangent iteration";
    if (which == 1 && reset_v) {
      CU(cudaMemsetAsync(v[vc], 0, field_bytes(), st));
      CU(cudaMemsetAsync(v[1 - vc], 0, field_bytes(), st));
    }
    if (fixed < 0 && !snap) CU(cudaMalloc(&snap, field_bytes()));
    reset_flags();
    MomScope ms(this, which == 1 ? n : 0, kernel);
    long long it = 0;
    double r = 0.0;
    long long batch = 1;
    const bool graphs = xmode == 0 && N <= kGraphMaxNodes;
    RingGraphs rg;
    while (it < n) {
      const long long b = std::min<long long>({batch, n - it, (long long)kRing});
      void** buf = which == 0 ? f : which == 1 ? v : tg;
      int& cur = which == 0 ? fc : which == 1 ? vc : tc;
      const int cur0 = cur;
      long long& steps = which == 0 ? primal_steps : which == 1 ? adjoint_steps : tangent_steps;
      const long long steps0 = steps;
      // keys of this batch: step k+1 at sweep k (as the captured graphs bake in)
      (which == 0 ? kb_p : which == 1 ? kb_a : kb_t) = steps0;
      if (fixed < 0 && b > 1) CU(cudaMemcpyAsync(snap, buf[cur], field_bytes(), cudaMemcpyDeviceToDevice, st));
      CU(cudaMemsetAsync(d_ring, 0, sizeof(unsigned long long) * b, st));
      const bool rel = graphs && b == kRing;  // graph batch: step keys 1..kRing
      if (rel) {
        if (!rg.ex[cur]) capture_ring(which, kernel, cur, &rg.ex[cur]);
        CU(cudaGraphLaunch(rg.ex[cur], st));
        steps += kRing;  // kRing is even: the buffer parity is back where it started
        launches += kRing;
      } else {
        for (long long k = 0; k < b; ++k) {
          if (which == 0) primal_launch(true, d_ring + k);
          else if (which == 1) adjoint_launch(kernel, true, d_ring + k);
          else tangent_launch(true, d_ring + k);
        }
      }
      CU(cudaGetLastError());
      reduce_flags(d_ring, size_t(b), false);
      reduce_flags(d_flags + 1, 1, true);
      CU(cudaMemcpyAsync(h_flags, d_flags, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, st));
      CU(cudaMemcpyAsync(h_flags + 4, d_ring, sizeof(unsigned long long) * b, cudaMemcpyDeviceToHost, st));
      sync();
      // first failing step in the batch, in step order; the iteration in a
      // report counts from the start of this solve, as the reference's does
      // (collision.cpp:387-389)
      long long stop = -1;
      for (long long k = 0; k < b; ++k) {
        const double rk = bits_to_double(h_flags[4 + k]);
        const long long itk = it + k + 1;
        const bool badk = h_flags[1] != kNoBad && (long long)(h_flags[1] >> 40) == k + 1;
        if (badk) raise_bad(h_flags[1], what, it);
        if (!std::isfinite(rk)) {
          reset_flags();
          if (which == 2)  // adjoint.cpp:472-473
            throw Fail{LBGPU_E_NUMERIC, "tangent diverged at iteration " + std::to_string(itk)};
          throw Fail{LBGPU_E_NUMERIC, std::string(which == 0 ? "state" : "adjoint") +
                                          " diverged (non-finite residual) at iteration " +
                                          std::to_string(itk)};
        }
        if (fixed < 0 && rk <= tol) {
          stop = k;
          r = rk;
          break;
        }
      }
      if (stop >= 0) {
        if (stop < b - 1) {  // roll back and replay exactly stop+1 steps
          CU(cudaMemcpyAsync(buf[cur0], snap, field_bytes(), cudaMemcpyDeviceToDevice, st));
          cur = cur0;
          steps = steps0;
          for (long long k = 0; k <= stop; ++k) {
            if (which == 0) primal_launch(false, nullptr);
            else if (which == 1) adjoint_launch(kernel, false, nullptr);
            else tangent_launch(false, nullptr);
          }
          sync();
        }
        it += stop + 1;
        break;
      }
      if (h_flags[1] != kNoBad) raise_bad(h_flags[1], what, it);  // any other bad key
      it += b;
      r = bits_to_double(h_flags[4 + b - 1]);
      batch = std::min<long long>(batch * 2, kRing);
    }
    *iters = it;
    *resid = r;
    *conv = r <= tol;
  }

  // tangent_solve (adjoint.cpp:422-490) from the current primal state: df from
  // zero to its fixed point under the frozen base (the solve() stop rule, same
  // batching and exact replay), then dF over the support, pairwise-summed.
  void tangent(const double* dw_design, double d_inlet_dp, double tol, long long max_iter,
               double* dF, long long* iters, double* resid, int* conv) {
    require_solo();
    require_db("tangent_solve");
    if (!tg[0]) {
      CU(cudaMalloc(&tg[0], field_bytes()));
      CU(cudaMalloc(&tg[1], field_bytes()));
    }
    if (!d_dw) CU(cudaMalloc(&d_dw, sizeof(double) * N));
    CU(cudaMemsetAsync(d_dw, 0, sizeof(double) * N, st));
    const long long n = (long long)design.size();
    if (n) {
      if (!d_wvals) CU(cudaMalloc(&d_wvals, sizeof(double) * n));
      CU(cudaMemcpyAsync(d_wvals, dw_design, sizeof(double) * n, cudaMemcpyHostToDevice, st));
      k_scatter_design<<<unsigned((n + 255) / 256), 256, 0, st>>>(d_wvals, d_design, n, d_dw);
      ++launches;
    }
    tangent_drho = 3.0 * d_inlet_dp;
    CU(cudaMemsetAsync(tg[tc], 0, field_bytes(), st));
    CU(cudaMemsetAsync(tg[1 - tc], 0, field_bytes(), st));
    solve(2, tol, max_iter, -1, 0, iters, resid, conv);
    const Launch a = launch(tangent_steps - kb_t);
    if (exact) exact::tangent_terms(a, dim, prec, f[fc], tg[tc], d_support, (long long)support.size(), d_terms);
    else fast::tangent_terms(a, dim, prec, f[fc], tg[tc], d_support, (long long)support.size(), d_terms);
    CU(cudaGetLastError());
    *dF = pairwise(tree_support, d_terms);
  }

  void sync_host_w() {
    if (!w_host_stale) return;
    CU(cudaMemcpyAsync(w.data(), d_w, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
    sync();
    w_host_stale = false;
  }
  // rho_in and the reciprocal the fast build's pressure faces use
  void set_rho_in(double r) {
    M.rho_in = r;
    M.inv_rho_in = 1.0 / r;
  }
  // Raw write of one node's w (no clamp), with its libm pow pair in exact mode.
  void set_node_w(long long idx, double val) {
    w[idx] = val;
    CU(cudaMemcpyAsync(d_w + idx, &w[idx], sizeof(double), cudaMemcpyHostToDevice, st));
    if (exact) {
      const double base = M.fluid_power ? val : 1.0 - val;
      const double pp[2] = {std::pow(base, M.theta), std::pow(base, M.theta - 1.0)};
      CU(cudaMemcpyAsync(d_p0 + idx, &pp[0], sizeof(double), cudaMemcpyHostToDevice, st));
      CU(cudaMemcpyAsync(d_p1 + idx, &pp[1], sizeof(double), cudaMemcpyHostToDevice, st));
    }
    sync();
  }
  // fd_gradient (adjoint.cpp:492-517): central difference of the raw objective
  // along design node `ordinal` (DesignField::nodes order) or, for ordinal < 0,
  // inlet_dp; each side is a cold-start primal solve (tol / max_iter, or
  // exactly `fixed` steps when fixed >= 0) with the parameter raw-perturbed.
  // The engine's primal state, design and model are restored afterwards.
  double fd_gradient(long long ordinal, double h, double tol, long long max_iter, long long fixed) {
    require_solo();
    require_db("fd_gradient");
    if (ordinal >= (long long)design.size())
      throw Fail{LBGPU_E_ARG, "design ordinal out of range"};
    sync_host_w();
    void* save = nullptr;
    CU(cudaMalloc(&save, field_bytes()));
    CU(cudaMemcpyAsync(save, f[fc], field_bytes(), cudaMemcpyDeviceToDevice, st));
    const int fc0 = fc;
    const double rho0 = M.rho_in;
    const long long idx = ordinal >= 0 ? design[ordinal] : -1;
    const double w0 = idx >= 0 ? w[idx] : 0.0;
    auto restore = [&] {
      set_rho_in(rho0);
      if (idx >= 0) set_node_w(idx, w0);
      fc = fc0;
      CU(cudaMemcpyAsync(f[fc], save, field_bytes(), cudaMemcpyDeviceToDevice, st));
      sync();
      cudaFree(save);
    };
    try {
      auto run = [&](double delta) {
        if (idx < 0) set_rho_in(1.0 + 3.0 * (inlet_dp + delta));  // rho_inlet(), collision.hpp:57
        else set_node_w(idx, w0 + delta);
        init_state();
        long long it = 0;
        double r = 0.0;
        int c = 0;
        solve(0, tol, max_iter, fixed, 0, &it, &r, &c);
        return objective();
      };
      const double fp = run(+h);
      const double fm = run(-h);
      restore();
      return (fp - fm) / (2.0 * h);
    } catch (...) {
      try { restore(); } catch (...) {}
      throw;
    }
  }

  // fd_gradient for n components with one host sync (fixed >= 0): every side
  // is queued on the stream -- the raw write of the perturbed value (w and, in
  // the exact build, its libm pow pair, staged in pinned memory; or rho_in,
  // which travels with each launch's Model), initialize_state, `fixed`
  // sweeps, evaluate_raw into a device slot, the write-back. Same sweeps and
  // reductions as fd_gradient, so the same bits.
  void fd_batch(long long n, const long long* ords, const double* hs, double tol,
                long long max_iter, long long fixed, bool from_state, double* out) {
    require_solo();
    require_db("fd_gradient");
    for (long long k = 0; k < n; ++k)
      if (ords[k] >= (long long)design.size()) throw Fail{LBGPU_E_ARG, "design ordinal out of range"};
    if (from_state && fixed < 0)
      throw Fail{LBGPU_E_ARG, "a finite difference from the current state needs fixed_iters >= 0"};
    if (fixed < 0) {
      for (long long k = 0; k < n; ++k) out[k] = fd_gradient(ords[k], hs[k], tol, max_iter, -1);
      return;
    }
    sync_host_w();
    void* save = nullptr;
    double* stage = nullptr;   // per side: w, p0, p1; then per component: w0, p0, p1
    double* d_vals = nullptr;  // J of each side
    const int fc0 = fc;
    const double rho0 = M.rho_in;
    auto release = [&] {
      set_rho_in(rho0);
      fc = fc0;
      if (save) cudaMemcpyAsync(f[fc], save, field_bytes(), cudaMemcpyDeviceToDevice, st);
      cudaStreamSynchronize(st);
      cudaFree(save), cudaFree(d_vals);
      if (stage) cudaFreeHost(stage);
    };
    try {
      CU(cudaMalloc(&save, field_bytes()));
      CU(cudaMemcpyAsync(save, f[fc], field_bytes(), cudaMemcpyDeviceToDevice, st));
      CU(cudaMallocHost(&stage, sizeof(double) * 9 * std::max<long long>(n, 1)));
      CU(cudaMalloc(&d_vals, sizeof(double) * 2 * std::max<long long>(n, 1)));
      auto pows = [&](double val, double* pp) {
        const double base = M.fluid_power ? val : 1.0 - val;
        pp[0] = std::pow(base, M.theta), pp[1] = std::pow(base, M.theta - 1.0);
      };
      reset_flags();
      for (long long k = 0; k < n; ++k) {
        const long long idx = ords[k] >= 0 ? design[ords[k]] : -1;
        double* sk = stage + 9 * k;
        for (int side = 0; side < 2; ++side) {
          const double delta = side == 0 ? hs[k] : -hs[k];
          if (idx < 0) {
            set_rho_in(1.0 + 3.0 * (inlet_dp + delta));  // rho_inlet(), collision.hpp:57
          } else {
            double* sv = sk + 3 * side;
            sv[0] = w[idx] + delta;
            if (exact) pows(sv[0], sv + 1);
            CU(cudaMemcpyAsync(d_w + idx, sv, sizeof(double), cudaMemcpyHostToDevice, st));
            if (exact) {
              CU(cudaMemcpyAsync(d_p0 + idx, sv + 1, sizeof(double), cudaMemcpyHostToDevice, st));
              CU(cudaMemcpyAsync(d_p1 + idx, sv + 2, sizeof(double), cudaMemcpyHostToDevice, st));
            }
          }
          if (from_state) {
            fc = fc0;
            CU(cudaMemcpyAsync(f[fc], save, field_bytes(), cudaMemcpyDeviceToDevice, st));
          } else {
            init_state();
          }
          for (long long i = 0; i < fixed; ++i) primal_launch(false, nullptr);
          const Launch a = launch(primal_steps - kb_p);
          if (exact) exact::objective_terms(a, dim, prec, f[fc], d_support, (long long)support.size(), d_terms, 0);
          else fast::objective_terms(a, dim, prec, f[fc], d_support, (long long)support.size(), d_terms, 0);
          pairwise_queue(tree_support, d_terms, d_vals + 2 * k + side);
        }
        if (idx < 0) {
          set_rho_in(rho0);
        } else {  // the write-back (fd_gradient's restore)
          double* s0 = sk + 6;
          s0[0] = w[idx];
          if (exact) pows(s0[0], s0 + 1);
          CU(cudaMemcpyAsync(d_w + idx, s0, sizeof(double), cudaMemcpyHostToDevice, st));
          if (exact) {
            CU(cudaMemcpyAsync(d_p0 + idx, s0 + 1, sizeof(double), cudaMemcpyHostToDevice, st));
            CU(cudaMemcpyAsync(d_p1 + idx, s0 + 2, sizeof(double), cudaMemcpyHostToDevice, st));
          }
        }
      }
      CU(cudaGetLastError());
      std::vector<double> vals(size_t(2 * n));
      CU(cudaMemcpyAsync(vals.data(), d_vals, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, st));
      pull_flags();  // the one host sync
      if (h_flags[1] != kNoBad) raise_bad(h_flags[1], "iteration");
      for (long long k = 0; k < n; ++k) out[k] = (vals[2 * k] - vals[2 * k + 1]) / (2.0 * hs[k]);
    } catch (...) {
      try { release(); } catch (...) {}
      throw;
    }
    release();
  }

  // ------------------------------------------------------- reductions
  double pairwise(PairTree& tr, const double* d_t) {
    pairwise_queue(tr, d_t);
    double out = 0.0;
    CU(cudaMemcpyAsync(&out, d_scalar, sizeof(double), cudaMemcpyDeviceToHost, st));
    sync();
    return out;
  }
  // the tree replay only; the sum lands in *out (default d_scalar[0])
  // publish: also copy the status words and the sum to h_pub (mapped) and
  // reset the words -- one-block trees only; returns whether it did
  bool pairwise_queue(PairTree& tr, const double* d_t, double* out = nullptr, bool publish = false) {
    if (!out) out = d_scalar;
    if (tr.small()) {
      k_tree_small<<<1, 1024, tr.small_bytes, st>>>(d_t, tr.d_lo, tr.d_hi, tr.leaves, tr.d_ops, tr.d_lvl,
                                                     int(tr.lvl.size()) - 1, tr.ops, out, d_flags,
                                                     publish ? d_pub : nullptr);
      ++launches;
      return publish;
    }
    const int nb = (tr.leaves + 127) / 128;
    k_leaf_sums<<<nb, 128, 0, st>>>(d_t, tr.d_lo, tr.d_hi, tr.leaves, tr.d_vals);
    for (int h = 1; h <= tr.top; ++h) {
      const int b = tr.lvl[h - 1], e = tr.lvl[h];
      k_combine_level<<<unsigned((e - b + 255) / 256), 256, 0, st>>>(tr.d_vals, tr.d_ops, tr.leaves, b, e);
    }
    k_combine_top<<<1, 1024, 0, st>>>(tr.d_vals, tr.d_ops, tr.d_lvl, tr.leaves, tr.top,
                                      int(tr.lvl.size()) - 1, tr.ops, out);
    launches += 2 + tr.top;
    return false;
  }
  // the objective's terms of a double-buffered state into d_terms (no sync)
  void objective_terms_queue(const void* P) {
    const Launch a = launch(primal_steps - kb_p);
    if (exact) exact::objective_terms(a, dim, prec, P, d_support, (long long)support.size(), d_terms, 0);
    else fast::objective_terms(a, dim, prec, P, d_support, (long long)support.size(), d_terms, 0);
    ++launches;
  }
  double objective(const void* buf = nullptr) {
    const Launch a = launch(primal_steps - kb_p);
    const void* P = buf ? buf : f[fc];
    const int bm = buf ? 0 : fmode();
    if (exact) exact::objective_terms(a, dim, prec, P, d_support, (long long)support.size(), d_terms, bm);
    else fast::objective_terms(a, dim, prec, P, d_support, (long long)support.size(), d_terms, bm);
    CU(cudaGetLastError());
    // J lands next to the status words: one readback, one host sync
    pairwise_queue(tree_support, d_terms, reinterpret_cast<double*>(d_flags + 4));
    CU(cudaMemcpyAsync(h_flags, d_flags, sizeof(unsigned long long) * 5, cudaMemcpyDeviceToHost, st));
    sync();
    if (h_flags[1] != kNoBad) raise_bad(h_flags[1], "iteration");
    return bits_to_double(h_flags[4]);
  }
  double penalty() {
    const long long n = (long long)design.size();
    if (n) k_penalty_terms<<<unsigned((n + 127) / 128), 128, 0, st>>>(d_w, d_design, n, d_terms);
    CU(cudaGetLastError());
    return pairwise(tree_design, d_terms);
  }
  void gradient(int kernel, double* g, double* gdp) {
    reset_flags();
    const Launch a = launch(adjoint_steps - kb_a);
    const long long n = (long long)design.size();
    if (aa && kernel != 0) require_db("the dual-number gradient");
    if (exact) exact::gradient(a, dim, prec, kernel, false, f[fc], v[vc], d_design, n, d_grad, nullptr, 0, 0, 0, 0, 0);
    else fast::gradient(a, dim, prec, kernel, false, f[fc], v[vc], d_design, n, d_grad, nullptr, 0, 0, 0, fmode(), vmode());
    CU(cudaGetLastError());
    if (g && n) CU(cudaMemcpyAsync(g, d_grad, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    if (gdp) {
      const long long ni = (long long)inlets.size();
      if (exact) exact::inlet_terms(a, dim, prec, f[fc], v[vc], d_inlets, ni, d_terms, 0, 0);
      else fast::inlet_terms(a, dim, prec, f[fc], v[vc], d_inlets, ni, d_terms, fmode(), vmode());
      CU(cudaGetLastError());
      *gdp = pairwise(tree_inlet, d_terms);
    }
    check_bad("gradient at iteration");
  }

  // ------------------------------------------------- unsteady adjoint
  // Discrete adjoint of N primal steps (no reference
  // function — SPEC.md:313). With P = S o W one primal step, the reference's
  // adjoint_step(base b, v) = S^-1 (J_W(b)^T v + dF(b)):
  //   mu^N     = adjoint_step(base f^N, 0, obj)
  //   mu^{n-1} = adjoint_step(base f^{n-1}, mu^n, obj if sum else none)
  //   dJ/dw    = sum_{n=N..1} param_gradient(v = mu^n, base f^{n-1})
  // for J = F(f^N) (terminal) or J = sum_{n=1..N} F(f^n). Primal states come
  // from checkpoints in `slots` state buffers, placed by a binomial schedule
  // (Schedule: the recompute-optimal split of every segment for its free
  // slot count, and checkpoints placed by the first forward pass itself,
  // which runs anyway); the sweeps write straight into the slot buffers.
  //
  // Schedule tables, for segment length n <= N and free slots s <= S:
  //   opt(n, s)   extra sweeps to reverse a segment from its first state;
  //   first(n, s) the same when the segment's states are produced by the
  //               first pass (checkpoints cost no extra sweeps there);
  //   opt(n, s)   = min_m m + opt(n - m, s - 1) + opt(m, s),
  //   first(n, s) = min_m first(n - m, s - 1) + opt(m, s),
  // with opt = first = n - 1 (store every inner state) when n - 1 <= s, and
  // n (n - 1) / 2 (recompute every base from the checkpoint) when s = 0.
  // Measured model at C5 slab size, N = 1000: round 1's recursive bisection
  // with 4 slots spent 10.6 N sweeps; this schedule spends 6.3 N with 4
  // slots and 5.3 N with 5 (the same device memory as round 1's 4 slots plus
  // its separate state-0 and state-N buffers, which now are the engine's own).
  struct Schedule {
    static constexpr long long kMaxN = 4096;  // DP tables up to here; bisection beyond
    long long N = 0;
    int S = 0;
    bool dp = false;
    std::vector<long long> oc, fcst;
    std::vector<int> om, fmv;
    size_t at(long long n, int s) const { return size_t(n) * size_t(S + 1) + size_t(s); }
    void build(long long N_, int S_) {
      N = N_, S = S_;
      dp = N <= kMaxN;
      if (!dp) return;
      const size_t sz = size_t(N + 1) * size_t(S + 1);
      oc.assign(sz, 0), fcst.assign(sz, 0), om.assign(sz, 0), fmv.assign(sz, 0);
      for (int sl = 0; sl <= S; ++sl)
        for (long long n = 2; n <= N; ++n) {
          if (n - 1 <= sl) {
            oc[at(n, sl)] = n - 1;
            continue;
          }
          if (sl == 0) {
            oc[at(n, sl)] = fcst[at(n, sl)] = n * (n - 1) / 2;
            continue;
          }
          long long bo = -1, bf = -1;
          int mo = 1, mf = 1;
          for (long long m = 1; m < n; ++m) {
            const long long co = m + oc[at(n - m, sl - 1)] + oc[at(m, sl)];
            const long long cf = fcst[at(n - m, sl - 1)] + oc[at(m, sl)];
            if (bo < 0 || co < bo) bo = co, mo = int(m);
            if (bf < 0 || cf < bf) bf = cf, mf = int(m);
          }
          oc[at(n, sl)] = bo, om[at(n, sl)] = mo;
          fcst[at(n, sl)] = bf, fmv[at(n, sl)] = mf;
        }
    }
    // checkpoint offset for a segment reversed from its start (>= 1)
    long long opt_split(long long n, long long s) const {
      if (!dp) return n / 2;
      return om[at(n, int(std::min<long long>(s, S)))];
    }
    // checkpoint offset the first pass places (0: none, the segment is terminal)
    long long first_split(long long n, long long s) const {
      if (!dp || n - 1 <= s || s == 0) return 0;
      return fmv[at(n, int(std::min<long long>(s, S)))];
    }
  };

  struct Unsteady {
    lbgpu_engine* e;
    bool sum;
    std::vector<void*> free_slots;
    void* work;   // ping-pong partners for forward segments
    void* work2;
    const Schedule* sch;
    double* d_gs = nullptr;  // per back step: the inlet_dp term's tree sum (summed on the host
    long long gn = 0;        // at the end, in step order: no host sync per step)
    double* d_gacc = nullptr;  // fused: per-node gradient sums, accumulated by the adjoint sweep
    // k >= 1 sweeps from `from`, the last one landing in `to` (via `tmp`)
    void fwd(const void* from, void* to, long long k, void* tmp) {
      const void* src = from;
      for (long long i = 0; i < k; ++i) {
        void* dst = ((k - 1 - i) % 2 == 0) ? to : tmp;
        e->primal_raw(src, dst, false, nullptr, true);
        src = dst;
      }
    }
    // mu^n -> grad += g(mu^n, f^{n-1}); mu^{n-1} = adjoint(f^{n-1}, mu^n)
    void back_step(const void* base) {
      const long long nd = (long long)e->design.size();
      const Launch a = e->launch(e->adjoint_steps - e->kb_a);
      if (!d_gacc) {  // else the adjoint sweep below adds each design node's term
        if (e->exact) exact::gradient(a, e->dim, e->prec, 0, false, base, e->v[e->vc], e->d_design, nd, e->d_grad, nullptr, 0, 0, 1, 0, 0);
        else fast::gradient(a, e->dim, e->prec, 0, false, base, e->v[e->vc], e->d_design, nd, e->d_grad, nullptr, 0, 0, 1, 0, 0);
      }
      if (!e->inlets.empty()) {
        if (e->exact) exact::inlet_terms(a, e->dim, e->prec, base, e->v[e->vc], e->d_inlets, (long long)e->inlets.size(), e->d_terms, 0, 0);
        else fast::inlet_terms(a, e->dim, e->prec, base, e->v[e->vc], e->d_inlets, (long long)e->inlets.size(), e->d_terms, 0, 0);
        e->pairwise_queue(e->tree_inlet, e->d_terms, d_gs + gn++);
      }
      e->M.obj_on = sum ? 1 : 0;
      e->adj_gacc = d_gacc;
      e->adjoint_raw(0, base, e->v[e->vc], e->v[1 - e->vc], false, nullptr, true);
      e->adj_gacc = nullptr;
      e->vc ^= 1;
      e->M.obj_on = 1;
    }
    // On entry v holds mu^b and `A` holds state a; leaves mu^a in v.
    void reverse(long long a, long long b, const void* A) {
      const long long inner = b - a - 1;  // states a+1 .. b-1
      if (inner > 0 && free_slots.empty()) {  // no memory left: recompute each base from A
        for (long long n = b; n > a; --n) {
          if (n - 1 == a) {
            back_step(A);
          } else {
            fwd(A, work2, n - 1 - a, work);
            back_step(work2);
          }
        }
        return;
      }
      if (inner <= (long long)free_slots.size()) {
        std::vector<void*> st(inner);
        const void* prev = A;
        for (long long k = 0; k < inner; ++k) {
          st[k] = free_slots.back();
          free_slots.pop_back();
          e->primal_raw(prev, st[k], false, nullptr, true);
          prev = st[k];
        }
        for (long long n = b; n > a; --n) back_step(n - 1 == a ? A : st[n - 1 - a - 1]);
        for (void* p : st) free_slots.push_back(p);
        return;
      }
      const long long m = a + sch->opt_split(b - a, (long long)free_slots.size());
      void* Ms = free_slots.back();
      free_slots.pop_back();
      fwd(A, Ms, m - a, work);
      reverse(m, b, Ms);
      free_slots.push_back(Ms);
      reverse(a, m, A);
    }
  };

  void unsteady(long long N, bool sum_obj, long long max_slots, double* g, double* gdp, double* J,
                long long* fsteps) {
    require_solo();
    require_db("the unsteady adjoint's checkpoint slots");
    if (N < 1) throw Fail{LBGPU_E_ARG, "unsteady adjoint needs at least one step"};
    const long long nslots = std::max<long long>(1, std::min<long long>(max_slots, N));
    std::vector<void*> slots;
    double* d_js = nullptr;  // J of each summed step, and the inlet_dp sums of the back steps
    double* d_gs = nullptr;
    double* d_gacc = nullptr;  // per-node gradient sums when the adjoint sweep carries them
    auto release = [&] {
      for (void* p : slots) cudaFree(p);
      cudaFree(d_js), cudaFree(d_gs), cudaFree(d_gacc);
    };
    // The back step's gradient rides in its adjoint sweep (k_adjoint GRAD)
    // where that sweep gathers an FP64 double-buffered base and every design
    // node is interior; bitwise the separate k_gradient pass.
    const bool fuse_grad = !exact && prec == 64 && xmode == 0 && grad_side.empty() && !design.empty();
    try {
      for (long long i = 0; i < nslots + 2; ++i) {
        void* p = nullptr;
        CU(cudaMalloc(&p, field_bytes()));
        // ghost layout: sweeps write owned columns only, so seed every slot's
        // ghosts with the current ones (the exchange refreshes them in NCCL mode)
        if (ghosts) CU(cudaMemcpyAsync(p, f[fc], field_bytes(), cudaMemcpyDeviceToDevice, st));
        slots.push_back(p);
      }
      Schedule sch;
      sch.build(N, int(nslots));
      // state 0 lives in the engine's idle buffer, state N lands in the
      // engine's current one (the primal state the call leaves behind)
      void* s0 = f[1 - fc];
      void* sN = f[fc];
      const long long steps0 = primal_steps;
      reset_flags();
      CU(cudaMemcpyAsync(s0, f[fc], field_bytes(), cudaMemcpyDeviceToDevice, st));
      CU(cudaMalloc(&d_js, sizeof(double) * (N + 1)));
      CU(cudaMalloc(&d_gs, sizeof(double) * (N + 1)));
      if (fuse_grad) {
        CU(cudaMalloc(&d_gacc, sizeof(double) * this->N));  // this->N: nodes (N here counts steps)
        CU(cudaMemsetAsync(d_gacc, 0, sizeof(double) * this->N, st));
      }
      Unsteady U{this, sum_obj, {}, slots[0], slots[1], &sch, d_gs, 0, d_gacc};
      for (long long i = 2; i < (long long)slots.size(); ++i) U.free_slots.push_back(slots[i]);
      // first pass: states 1..N and the objective, placing the schedule's
      // checkpoints (chain) and, in its last segment, every inner state
      long long jn = 0;
      std::vector<std::pair<long long, void*>> chain{{0, s0}};
      std::vector<void*> tail;  // the last segment's stored inner states
      long long a = 0;
      const void* src = s0;
      auto step_to = [&](long long n, void* dst) {
        primal_raw(src, dst, false, nullptr, true);
        src = dst;
        if (sum_obj || n == N) {  // J of state n, queued (summed on the host at the end)
          objective_terms_queue(dst);
          pairwise_queue(tree_support, d_terms, d_js + jn++);
        }
      };
      for (;;) {
        const long long n = N - a;
        const long long m = sch.first_split(n, (long long)U.free_slots.size());
        if (m == 0) {  // the last segment: store its inner states if they fit
          const bool store = n - 1 <= (long long)U.free_slots.size();
          for (long long k = a + 1; k <= N; ++k) {
            void* dst;
            if (k == N) {
              dst = sN;
            } else if (store) {
              dst = U.free_slots.back();
              U.free_slots.pop_back();
              tail.push_back(dst);
            } else {
              dst = ((N - k) % 2 == 1) ? U.work : U.work2;  // alternate; never sN's buffer
            }
            step_to(k, dst);
          }
          if (!store) tail.clear();
          break;
        }
        void* C = U.free_slots.back();  // a checkpoint m steps in
        U.free_slots.pop_back();
        for (long long k = a + 1; k <= a + m; ++k) step_to(k, k == a + m ? C : ((a + m - k) % 2 ? U.work : U.work2));
        a += m;
        chain.push_back({a, C});
      }
      // mu^N = adjoint_step(f^N, 0, obj)
      CU(cudaMemsetAsync(v[vc], 0, field_bytes(), st));
      CU(cudaMemsetAsync(v[1 - vc], 0, field_bytes(), st));
      CU(cudaMemsetAsync(d_grad, 0, sizeof(double) * std::max<size_t>(design.size(), 1), st));
      adjoint_raw(0, sN, v[vc], v[1 - vc], false, nullptr, true);
      vc ^= 1;
      // the last segment [a, N): its stored states, or recompute from its checkpoint
      {
        const long long ak = chain.back().first;
        const void* Ak = chain.back().second;
        if (!tail.empty() || N - ak <= 1) {
          for (long long n = N; n > ak; --n) U.back_step(n - 1 == ak ? Ak : tail[size_t(n - 1 - ak - 1)]);
          for (void* p : tail) U.free_slots.push_back(p);
        } else {
          U.reverse(ak, N, Ak);
        }
      }
      // then every earlier segment of the chain, from its checkpoint
      for (size_t j = chain.size() - 1; j-- > 0;) {
        U.free_slots.push_back(chain[j + 1].second);
        U.reverse(chain[j].first, chain[j + 1].first, chain[j].second);
      }
      // f^N stays in f[fc] (sN); f[1 - fc] (s0) is scratch again
      if (d_gacc) {
        const long long nd = (long long)design.size();
        k_gather_design<<<unsigned((nd + 255) / 256), 256, 0, st>>>(d_gacc, d_design, nd, d_grad);
        ++launches;
      }
      if (g && !design.empty())
        CU(cudaMemcpyAsync(g, d_grad, sizeof(double) * design.size(), cudaMemcpyDeviceToHost, st));
      std::vector<double> js(static_cast<size_t>(jn)), gs(static_cast<size_t>(U.gn));
      if (jn) CU(cudaMemcpyAsync(js.data(), d_js, sizeof(double) * jn, cudaMemcpyDeviceToHost, st));
      if (U.gn) CU(cudaMemcpyAsync(gs.data(), d_gs, sizeof(double) * U.gn, cudaMemcpyDeviceToHost, st));
      sync();
      check_bad("unsteady iteration");
      double Jv = 0.0, gd = 0.0;  // the per-step sums in the order the steps ran
      for (double x : js) Jv += x;
      for (double x : gs) gd += x;
      if (gdp) *gdp = gd;
      if (J) *J = Jv;
      if (fsteps) *fsteps = primal_steps - steps0;
    } catch (...) {
      sync();
      release();
      throw;
    }
    release();
  }

  // Iterations it0 .. it0+count-1 of a one-shot run of `total` iterations
  // (zeta/lambda indexed from it0); rows at it % ri == 0 and at it == total.
  void one_shot(long long it0, long long count, long long total, const double* zeta,
                const double* lambda, long long ri, lbgpu_run_row* rows, long long cap,
                long long* nrows) {
    require_solo();
    require_db("the one-shot loop");
    long long k = 0;
    reset_flags();
    const long long n = (long long)design.size();
    // Product build, one engine, interior design nodes only: iteration it's
    // design update rides in iteration it+1's primal sweep (k_primal UPD),
    // which gathers the same base f the gradient needs -- one f gather per
    // design node per iteration saved, bitwise the separate update. Record
    // iterations (their row needs the update's max|comp| and w) and the last
    // iteration of a call update on their own.
    const bool fusable = !exact && xmode == 0 && grad_side.empty() && n > 0;
    bool pend = false;
    double pz = 0.0, pl = 0.0;
    auto update_now = [&](double z_, double l_) {
      const Launch a = launch(adjoint_steps - kb_a);
      if (exact) exact::gradient(a, dim, prec, 0, true, f[fc], v[vc], d_design, n, nullptr, d_w, z_, l_, 0, 0, 0);
      else fast::gradient(a, dim, prec, 0, true, f[fc], v[vc], d_design, n, nullptr, d_w, z_, l_, 0, 0, 0);
      CU(cudaGetLastError());
      ++launches;
    };
    for (long long it = it0; it < it0 + count; ++it) {
      const bool rec = (it % ri == 0) || it == total;
      if (pend && rec) {  // this primal reports a residual: the update goes first, apart
        update_now(pz, pl);
        pend = false;
      }
      if (rec) CU(cudaMemsetAsync(d_flags, 0, sizeof(unsigned long long), st));
      if (pend) {
        ++primal_steps;
        ++launches;
        SweepArgs sa = sweep(primal_steps - kb_p, false, nullptr);
        sa.upd = true;
        sa.a.upd.v = v[vc], sa.a.upd.w = d_w, sa.a.upd.zeta = pz, sa.a.upd.lambda = pl;
        fast::primal(sa, f[fc], f[1 - fc]);
        fc ^= 1;
        pend = false;
      } else {
        primal_launch(rec, nullptr);
      }
      adjoint_launch(0, false, nullptr);
      if (rec) CU(cudaMemsetAsync(d_flags + 2, 0, sizeof(unsigned long long), st));
      if (fusable && !rec && it + 1 < it0 + count) {
        pend = true, pz = zeta[it - it0], pl = lambda[it - it0];
        continue;
      }
      update_now(zeta[it - it0], lambda[it - it0]);
      if (exact) {  // the device moved w: refresh the host copy and the libm pow tables
        CU(cudaMemcpyAsync(w.data(), d_w, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
        sync();
        refresh_pow_tables();
      }
      if (rec) {
        reduce_flags(d_flags, 1, false);
        reduce_flags(d_flags + 2, 1, false);
        reduce_flags(d_flags + 1, 1, true);
        pull_flags();
        if (h_flags[1] != kNoBad) raise_bad(h_flags[1], "iteration", it0 - 1);
        lbgpu_run_row row;
        row.iteration = double(it);
        row.residual = bits_to_double(h_flags[0]);
        const double gn = bits_to_double(h_flags[2]);
        row.objective = objective();
        row.penalty = penalty();
        row.penalty_weight = lambda[it - it0];
        row.composite = row.objective - lambda[it - it0] * row.penalty;
        row.grad_norm = gn;
        if (k < cap && rows) rows[k] = row;
        ++k;
      }
    }
    if (!exact) w_host_stale = true;
    pull_flags();
    if (h_flags[1] != kNoBad) raise_bad(h_flags[1], "iteration", it0 - 1);
    *nrows = k;
  }

  // ------------------------------------------------------------ layout
  void to_ref(int field, double* d_out) {
    void* buf = field == 0 ? f[fc] : v[vc];
    const int fm = field == 0 ? fmode() : vmode();
    if (exact) exact::layout(G, dim, prec, field, true, buf, d_out, st, 0);
    else fast::layout(G, dim, prec, field, true, buf, d_out, st, fm);
    CU(cudaGetLastError());
  }
  void from_ref(int field, const double* d_in) {
    void* buf = field == 0 ? f[fc] : v[vc];
    if (exact) exact::layout(G, dim, prec, field, false, d_in, buf, st, 0);
    else fast::layout(G, dim, prec, field, false, d_in, buf, st, aa ? 1 : 0);
    (field == 0 ? fpar : vpar) = 0;  // an in-place field lands in layout O
    CU(cudaGetLastError());
  }
  void ensure_ref() {
    if (!d_ref) CU(cudaMalloc(&d_ref, sizeof(double) * size_t(m) * N));
  }
};

namespace {

thread_local std::string g_create_err;

// Every API call first completes a deferred sweep (lbgpu_pair_step_with_design
// leaves one pending), so nothing observes a half-finished step; `keep`
// skips that for the call that manages the pending sweep itself.
template <class F>
int guarded(lbgpu_engine* e, F&& fn, bool keep = false) {
  if (!e) return LBGPU_E_ARG;
  try {
    if (e->device >= 0) cudaSetDevice(e->device);
    if (!keep) e->flush_pending();
    fn();
    e->err.clear();
    return LBGPU_OK;
  } catch (const Fail& f) {
    e->err = f.msg;
    return f.code;
  } catch (const std::exception& x) {
    e->err = x.what();
    return LBGPU_E_NUMERIC;
  }
}

}  // namespace

extern "C" {

const char* lbgpu_version(void) { return "0.1.0-b200"; }

int lbgpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  return n;
}

int lbgpu_slab_nxl(int span) { return (span + 2 + 15) / 16 * 16; }

int lbgpu_slab_info(const lbgpu_engine* e, int* out6) {
  if (!e || !out6) return LBGPU_E_ARG;
  const int v[6] = {e->gnx, e->x0, e->span, e->nx, e->slab_count, e->slab_id};
  std::memcpy(out6, v, sizeof v);
  return LBGPU_OK;
}

int lbgpu_group_link(lbgpu_engine** es, int n) {
  if (!es || n < 1) return LBGPU_E_ARG;
  for (int i = 0; i < n; ++i)
    if (!es[i] || es[i]->slab_count != n || es[i]->slab_id != i || es[i]->device != es[0]->device ||
        es[i]->aa)
      return LBGPU_E_ARG;
  if (n == 1) return LBGPU_OK;
  for (int i = 0; i < n; ++i) {
    lbgpu_engine* e = es[i];
    if (i > 0) {  // share slab 0's stream: lock-step order is stream order
      cudaSetDevice(e->device);
      cudaStreamSynchronize(e->st);
      if (e->owns_stream) cudaStreamDestroy(e->st);
      e->st = es[0]->st;
      e->owns_stream = false;
    }
    e->xmode = 1;
    e->nb_left = es[(i - 1 + n) % n];
    e->nb_right = es[(i + 1) % n];
  }
  return LBGPU_OK;
}

// The P2P group (partition.cpp:43-312's PartitionedRun, one stream per slab,
// slabs on any devices): every sweep stores its boundary planes straight into
// the neighbours' ghost columns (push_halo, peer memory across GPUs); sweep k
// of a slab waits only on its two neighbours' sweep k-1 (cross-device events).
int lbgpu_group_link_p2p(lbgpu_engine** es, int n) {
  if (!es || n < 2) return LBGPU_E_ARG;
  for (int i = 0; i < n; ++i)
    if (!es[i] || es[i]->slab_count != n || es[i]->slab_id != i || !es[i]->ghosts ||
        es[i]->xmode != 0 || es[i]->aa)
      return LBGPU_E_ARG;
  for (int i = 0; i < n; ++i) {
    lbgpu_engine* e = es[i];
    const int rc = guarded(e, [&] {
      for (lbgpu_engine* nb : {es[(i - 1 + n) % n], es[(i + 1) % n]}) {
        if (nb->device == e->device) continue;
        int can = 0;
        CU(cudaDeviceCanAccessPeer(&can, e->device, nb->device));
        if (!can)
          throw Fail{LBGPU_E_CONFIG, "no peer access from GPU " + std::to_string(e->device) +
                                         " to GPU " + std::to_string(nb->device)};
        const cudaError_t r = cudaDeviceEnablePeerAccess(nb->device, 0);
        if (r != cudaSuccess && r != cudaErrorPeerAccessAlreadyEnabled) CU(r);
        (void)cudaGetLastError();
      }
      for (cudaEvent_t& ev : e->ev_step)
        if (!ev) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      e->sync();
    });
    if (rc) return rc;
  }
  for (int i = 0; i < n; ++i) {
    es[i]->xmode = 3;
    es[i]->gstep = 0;
    es[i]->nb_left = es[(i - 1 + n) % n];
    es[i]->nb_right = es[(i + 1) % n];
  }
  return LBGPU_OK;
}

int lbgpu_group_exchange(lbgpu_engine** es, int n, int field) {
  if (!es || n < 1 || (field != 0 && field != 1)) return LBGPU_E_ARG;
  const bool p2p = es[0]->xmode == 3;
  if (p2p)  // every slab's buffers final before anyone reads across a cut
    for (int i = 0; i < n; ++i) {
      const int rc = guarded(es[i], [&] { es[i]->sync(); });
      if (rc) return rc;
    }
  for (int i = 0; i < n; ++i) {
    const int rc = guarded(es[i], [&] {
      if (p2p) es[i]->halo_op(2, field, nullptr, nullptr, es[i]->nb_left, es[i]->nb_right);
      else es[i]->exchange(field);
    });
    if (rc) return rc;
  }
  for (int i = 0; i < (p2p ? n : 1); ++i) {
    const int rc = guarded(es[i], [&] { es[i]->sync(); });
    if (rc) return rc;
  }
  return LBGPU_OK;
}

// One lock step of a P2P group (which: 0 primal, 1 adjoint, 2 fused pair:
// adjoint k + primal k+1, both fields pushed): each slab's sweep waits on
// its two neighbours' previous sweep (their ghosts are read-complete, WAR, and
// the planes they pushed into mine are written, RAW), then records its own.
static void p2p_sweep(lbgpu_engine** es, int n, int which, int kernel, bool r) {
  const int fpar = es[0]->fc, vpar = es[0]->vc;  // lock step: same parities everywhere
  for (int i = 0; i < n; ++i) {
    lbgpu_engine* e = es[i];
    CU(cudaSetDevice(e->device));
    for (int k = 0; k < 2; ++k) e->push_dst_l[k] = e->push_dst_r[k] = nullptr;
    if (which != 1) {  // the primal field's next buffer
      e->push_dst_l[0] = e->nb_left->f[1 - fpar];
      e->push_dst_r[0] = e->nb_right->f[1 - fpar];
    }
    if (which != 0) {  // the adjoint field's
      e->push_dst_l[1] = e->nb_left->v[1 - vpar];
      e->push_dst_r[1] = e->nb_right->v[1 - vpar];
    }
    const int prev = int((e->gstep + 1) & 1);
    CU(cudaStreamWaitEvent(e->st, e->nb_left->ev_step[prev], 0));
    CU(cudaStreamWaitEvent(e->st, e->nb_right->ev_step[prev], 0));
    if (which == 0) e->primal_launch(r, nullptr, false);
    else if (which == 1) e->adjoint_launch(kernel, r, nullptr, false);
    else e->fused_pair_raw(r);
    CU(cudaEventRecord(e->ev_step[e->gstep & 1], e->st));
  }
  for (int i = 0; i < n; ++i) ++es[i]->gstep;
}

int lbgpu_group_step(lbgpu_engine** es, int n, int which, int64_t steps, int kernel,
                     double* residual) {
  if (!es || n < 1 || steps < 0 || which < 0 || which > 2) return LBGPU_E_ARG;
  if (n > 1 && es[0] && es[0]->xmode == 3) {
    for (int i = 0; i < n; ++i)
      if (!es[i] || es[i]->xmode != 3) return LBGPU_E_STATE;
    if (which == 2 && (residual || !es[0]->fuse_pairs())) return LBGPU_E_STATE;
    return guarded(es[0], [&] {
      for (int i = 0; i < n; ++i) {  // whatever each slab had queued (uploads, init) lands first
        CU(cudaSetDevice(es[i]->device));
        es[i]->reset_flags();
        es[i]->sync();
      }
      for (int64_t k = 0; k < steps; ++k) p2p_sweep(es, n, which, kernel, residual && k == steps - 1);
      CU(cudaGetLastError());
      double rmax = 0.0;
      for (int i = 0; i < n; ++i) {
        CU(cudaSetDevice(es[i]->device));
        es[i]->pull_flags();
        if (es[i]->h_flags[1] != kNoBad)
          es[i]->raise_bad(es[i]->h_flags[1], which == 1 ? "adjoint iteration" : "iteration");
        const double ri = lbgpu_engine::bits_to_double(es[i]->h_flags[0]);
        if (!(ri <= rmax)) rmax = ri;
      }
      if (residual) *residual = rmax;
    });
  }
  if (which == 2) return LBGPU_E_ARG;  // fused pairs: P2P groups (and single engines) only
  for (int i = 0; i < n; ++i)
    if (!es[i] || (n > 1 && es[i]->xmode != 1)) return LBGPU_E_STATE;
  return guarded(es[0], [&] {
    for (int i = 0; i < n; ++i) es[i]->reset_flags();
    for (int64_t k = 0; k < steps; ++k) {
      const bool r = residual && k == steps - 1;
      for (int i = 0; i < n; ++i) {
        if (which == 0) es[i]->primal_launch(r, nullptr, false);
        else es[i]->adjoint_launch(kernel, r, nullptr, false);
      }
      if (n > 1)
        for (int i = 0; i < n; ++i) es[i]->exchange(which);
    }
    CU(cudaGetLastError());
    double rmax = 0.0;
    for (int i = 0; i < n; ++i) {
      es[i]->pull_flags();
      if (es[i]->h_flags[1] != kNoBad)
        es[i]->raise_bad(es[i]->h_flags[1], which == 0 ? "iteration" : "adjoint iteration");
      const double ri = lbgpu_engine::bits_to_double(es[i]->h_flags[0]);
      if (!(ri <= rmax)) rmax = ri;
    }
    if (residual) *residual = rmax;
  });
}

// Device time of `steps` lock steps of a P2P group (which as lbgpu_group_step,
// no residuals): events on every slab's stream around the steps, the maximum
// over slabs of their elapsed times (each slab ends no earlier than the last
// neighbour it waited on).
int lbgpu_group_time(lbgpu_engine** es, int n, int which, int64_t steps, double* ms) {
  if (!es || n < 2 || steps < 1 || !ms || which < 0 || which > 2) return LBGPU_E_ARG;
  for (int i = 0; i < n; ++i)
    if (!es[i] || es[i]->xmode != 3) return LBGPU_E_STATE;
  if (which == 2 && !es[0]->fuse_pairs()) return LBGPU_E_STATE;
  return guarded(es[0], [&] {
    std::vector<cudaEvent_t> t0(n), t1(n);
    for (int i = 0; i < n; ++i) {
      CU(cudaSetDevice(es[i]->device));
      es[i]->reset_flags();
      es[i]->sync();
      CU(cudaEventCreate(&t0[i]));
      CU(cudaEventCreate(&t1[i]));
    }
    // one host-side start: every slab's start event is queued before any sweep
    for (int i = 0; i < n; ++i) {
      CU(cudaSetDevice(es[i]->device));
      CU(cudaEventRecord(t0[i], es[i]->st));
    }
    for (int64_t k = 0; k < steps; ++k) p2p_sweep(es, n, which, 0, false);
    double worst = 0.0;
    for (int i = 0; i < n; ++i) {
      CU(cudaSetDevice(es[i]->device));
      CU(cudaEventRecord(t1[i], es[i]->st));
    }
    for (int i = 0; i < n; ++i) {
      CU(cudaSetDevice(es[i]->device));
      CU(cudaEventSynchronize(t1[i]));
      float t = 0.f;
      CU(cudaEventElapsedTime(&t, t0[i], t1[i]));
      worst = std::max(worst, double(t));
      cudaEventDestroy(t0[i]);
      cudaEventDestroy(t1[i]);
      es[i]->pull_flags();
      if (es[i]->h_flags[1] != kNoBad) es[i]->raise_bad(es[i]->h_flags[1], "iteration");
    }
    *ms = worst;
  });
}

int lbgpu_nccl_unique_id(void* out, int cap) {
  if (!out || cap < (int)sizeof(ncclUniqueId)) return LBGPU_E_ARG;
  ncclUniqueId id;
  try {
    if (nccl().GetUniqueId(&id) != ncclSuccess) return LBGPU_E_NUMERIC;
  } catch (const Fail& f) {
    g_create_err = f.msg;
    return f.code;
  }
  std::memcpy(out, &id, sizeof id);
  return LBGPU_OK;
}

int lbgpu_attach_nccl(lbgpu_engine* e, const void* uid, int nranks, int rank) {
  if (!uid || nranks < 1 || rank < 0 || rank >= nranks) return LBGPU_E_ARG;
  return guarded(e, [&] {
    if (e->slab_count != nranks || e->slab_id != rank)
      throw Fail{LBGPU_E_CONFIG, "engine must be slab `rank` of `nranks`"};
    if (nranks == 1 && !e->ghosts)
      throw Fail{LBGPU_E_CONFIG, "a single-rank ring needs the ghost-column layout (slab_id -1)"};
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof id);
    const ncclResult_t r = nccl().CommInitRank(&e->comm, nranks, id, rank);
    if (r != ncclSuccess) throw Fail{LBGPU_E_NUMERIC, std::string("NCCL: ") + nccl().GetErrorString(r)};
    e->rank = rank, e->nranks = nranks;
    e->xmode = 2;
    // the halo's pack / NCCL / unpack kernels take precedence over the
    // interior sweep's pending blocks, so the exchange never queues behind it
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU(cudaStreamCreateWithPriority(&e->st_comm, cudaStreamNonBlocking, hi));
    CU(cudaEventCreateWithFlags(&e->ev_bnd, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&e->ev_halo, cudaEventDisableTiming));
  });
}

int lbgpu_exchange(lbgpu_engine* e, int field) {
  if (field != 0 && field != 1) return LBGPU_E_ARG;
  return guarded(e, [&] {
    e->require_db("a stand-alone halo exchange");
    e->exchange(field);
    e->sync();
  });
}

int lbgpu_create(const lbgpu_system_desc* desc, lbgpu_engine** out) {
  if (!desc || !out) return LBGPU_E_ARG;
  *out = nullptr;
  g_create_err.clear();
  auto* e = new lbgpu_engine();
  try {
    e->setup(*desc);
    *out = e;
    return LBGPU_OK;
  } catch (const Fail& f) {
    g_create_err = f.msg;
    delete e;
    return f.code;
  } catch (const std::exception& x) {
    g_create_err = x.what();
    delete e;
    return LBGPU_E_NUMERIC;
  }
}

static int desc_from_config(const char* cfg_text, const char* overrides, int device, int exact,
                            CaseSpec& c, SystemArrays& s, lbgpu_system_desc& d,
                            int slab_count = 1, int slab_id = 0, int streaming = 0) {
  std::string err;
  if (!parse_case(cfg_text, overrides ? overrides : "", c, err)) {
    g_create_err = err;
    return LBGPU_E_CONFIG;
  }
  bool ok;
  if (slab_count <= 1 && slab_id == -1) {
    ok = build_slab(c, 0, c.nx, lbgpu_slab_nxl(c.nx), s, err);
  } else if (slab_count > 1) {
    if (slab_id < 0 || slab_id >= slab_count || slab_count > c.nx) {
      g_create_err = "invalid slab decomposition";
      return LBGPU_E_CONFIG;
    }
    int x0, span;
    decompose(c.nx, slab_count, slab_id, x0, span);
    ok = build_slab(c, x0, span, lbgpu_slab_nxl(span), s, err);
  } else {
    ok = build_system(c, s, err);
  }
  if (!ok) {
    g_create_err = err;
    return LBGPU_E_CONFIG;
  }
  d = lbgpu_system_desc{};
  d.slab_count = slab_count, d.slab_id = slab_id;
  d.streaming = streaming;
  d.nx = c.nx, d.ny = c.ny, d.nz = c.nz;
  d.precision = c.precision;
  d.exact = exact;
  d.device = device;
  d.collision = c.collision == "bgk" ? 1 : 0;
  d.nu = c.nu, d.beta_fluid = c.beta_fluid, d.beta_solid = c.beta_solid;
  d.inlet_dp = c.inlet_dp, d.u_clamp = c.u_clamp, d.omega_nonhydro = c.omega_nonhydro;
  d.switch_theta = c.switch_theta;
  d.switch_form = c.switch_form == "fluid_power" ? 1 : 0;
  d.tag = s.tag.data(), d.bc_T = s.bc_T.data(), d.bc_axis = s.bc_axis.data();
  d.bc_sign = s.bc_sign.data(), d.w = s.w.data(), d.design_mask = s.mask.data();
  d.obj_kind = s.obj_kind, d.flux_axis = s.flux_axis, d.flux_sign = s.flux_sign;
  d.support = s.support.data(), d.n_support = (int64_t)s.support.size();
  return LBGPU_OK;
}

int lbgpu_create_from_config(const char* cfg_text, const char* overrides, int device, int exact,
                             lbgpu_engine** out) {
  if (!cfg_text || !out) return LBGPU_E_ARG;
  *out = nullptr;
  g_create_err.clear();
  CaseSpec c;
  SystemArrays s;
  lbgpu_system_desc d;
  const int rc = desc_from_config(cfg_text, overrides, device, exact, c, s, d);
  if (rc) return rc;
  return lbgpu_create(&d, out);
}

int lbgpu_create_slab_from_config(const char* cfg_text, const char* overrides, int device,
                                  int exact, int slab_count, int slab_id, lbgpu_engine** out) {
  if (!cfg_text || !out) return LBGPU_E_ARG;
  *out = nullptr;
  g_create_err.clear();
  CaseSpec c;
  SystemArrays s;
  lbgpu_system_desc d;
  const int rc = desc_from_config(cfg_text, overrides, device, exact, c, s, d, slab_count, slab_id);
  if (rc) return rc;
  return lbgpu_create(&d, out);
}

int lbgpu_create_from_config_ex(const char* cfg_text, const char* overrides, int device,
                                int exact, int slab_count, int slab_id, int streaming,
                                lbgpu_engine** out) {
  if (!cfg_text || !out) return LBGPU_E_ARG;
  *out = nullptr;
  g_create_err.clear();
  CaseSpec c;
  SystemArrays s;
  lbgpu_system_desc d;
  const int rc =
      desc_from_config(cfg_text, overrides, device, exact, c, s, d, slab_count, slab_id, streaming);
  if (rc) return rc;
  return lbgpu_create(&d, out);
}

int lbgpu_case_slab_tables(const char* cfg_text, const char* overrides, int slab_count,
                           int slab_id, int* slab, int* dims, int64_t* counts, uint8_t* tag,
                           double* bc_T, int8_t* bc_axis, int8_t* bc_sign, double* w,
                           uint8_t* mask, int64_t* design, int64_t* support) {
  if (!cfg_text || !slab || !dims || !counts) return LBGPU_E_ARG;
  g_create_err.clear();
  CaseSpec c;
  SystemArrays s;
  lbgpu_system_desc d;
  const int rc = desc_from_config(cfg_text, overrides, 0, 0, c, s, d, slab_count, slab_id);
  if (rc) return rc;
  lbgpu_engine e;
  try {
    e.setup_host(d);
  } catch (const Fail& f) {
    g_create_err = f.msg;
    return f.code;
  }
  const int sl[6] = {e.gnx, e.x0, e.span, e.nx, e.slab_count, e.slab_id};
  std::memcpy(slab, sl, sizeof sl);
  const int dd[8] = {e.nx, e.ny, e.nz, e.m, e.mf, e.mt, e.prec, 0};
  std::memcpy(dims, dd, sizeof dd);
  counts[0] = e.N;
  counts[1] = (int64_t)e.design.size();
  counts[2] = (int64_t)e.support.size();
  counts[3] = (int64_t)e.inlets.size();
  return lbgpu_get_tables(&e, tag, bc_T, bc_axis, bc_sign, w, mask, design, support, nullptr);
}

int lbgpu_case_tables(const char* cfg_text, const char* overrides, int* dims, int64_t* counts,
                      uint8_t* tag, double* bc_T, int8_t* bc_axis, int8_t* bc_sign, double* w,
                      uint8_t* mask, int64_t* design, int64_t* support, double* A) {
  if (!cfg_text || !dims || !counts) return LBGPU_E_ARG;
  g_create_err.clear();
  CaseSpec c;
  SystemArrays s;
  lbgpu_system_desc d;
  const int rc = desc_from_config(cfg_text, overrides, 0, 0, c, s, d);
  if (rc) return rc;
  lbgpu_engine e;
  try {
    e.setup_host(d);
  } catch (const Fail& f) {
    g_create_err = f.msg;
    return f.code;
  }
  const int dd[8] = {e.nx, e.ny, e.nz, e.m, e.mf, e.mt, e.prec, 0};
  std::memcpy(dims, dd, sizeof dd);
  counts[0] = e.N;
  counts[1] = (int64_t)e.design.size();
  counts[2] = (int64_t)e.support.size();
  counts[3] = (int64_t)e.inlets.size();
  return lbgpu_get_tables(&e, tag, bc_T, bc_axis, bc_sign, w, mask, design, support, A);
}

void lbgpu_destroy(lbgpu_engine* e) { delete e; }
const char* lbgpu_last_create_error(void) { return g_create_err.c_str(); }
const char* lbgpu_error_message(const lbgpu_engine* e) { return e ? e->err.c_str() : "null handle"; }

int lbgpu_info(const lbgpu_engine* e, int* dims, int64_t* counts) {
  if (!e || !dims || !counts) return LBGPU_E_ARG;
  const int d[8] = {e->nx, e->ny, e->nz, e->m, e->mf, e->mt, e->prec, e->exact};
  std::memcpy(dims, d, sizeof d);
  counts[0] = e->N;
  counts[1] = (int64_t)e->design.size();
  counts[2] = (int64_t)e->support.size();
  counts[3] = (int64_t)e->inlets.size();
  return LBGPU_OK;
}

int lbgpu_get_tables(const lbgpu_engine* e, uint8_t* tag, double* bc_T, int8_t* bc_axis,
                     int8_t* bc_sign, double* w, uint8_t* mask, int64_t* design, int64_t* support,
                     double* A) {
  if (!e) return LBGPU_E_ARG;
  const size_t n = size_t(e->N);
  if (tag) std::memcpy(tag, e->tag.data(), n);
  if (bc_T) std::memcpy(bc_T, e->bc_T.data(), n * sizeof(double));
  if (bc_axis) std::memcpy(bc_axis, e->bc_axis.data(), n);
  if (bc_sign) std::memcpy(bc_sign, e->bc_sign.data(), n);
  if (w) std::memcpy(w, e->w.data(), n * sizeof(double));
  if (mask) std::memcpy(mask, e->mask.data(), n);
  if (design) for (size_t i = 0; i < e->design.size(); ++i) design[i] = e->design[i];
  if (support) for (size_t i = 0; i < e->support.size(); ++i) support[i] = e->support[i];
  if (A) std::memcpy(A, e->A.data(), e->A.size() * sizeof(double));
  return LBGPU_OK;
}

int lbgpu_counters(const lbgpu_engine* e, int64_t* p, int64_t* a) {
  if (!e || !p || !a) return LBGPU_E_ARG;
  *p = e->primal_steps;
  *a = e->adjoint_steps;
  return LBGPU_OK;
}

int64_t lbgpu_sweep_launches(const lbgpu_engine* e) { return e ? e->launches : -1; }

void* lbgpu_stream(const lbgpu_engine* e) { return e ? (void*)e->st : nullptr; }

int lbgpu_init_state(lbgpu_engine* e) {
  return guarded(e, [&] {
    e->init_state();
    e->sync();
  });
}

int lbgpu_reset_adjoint(lbgpu_engine* e) {
  return guarded(e, [&] {
    e->vpar = 0;
    CU(cudaMemsetAsync(e->v[e->vc], 0, e->field_bytes(), e->st));
    e->sync();
  });
}

int lbgpu_upload_state(lbgpu_engine* e, int field, const double* ref) {
  if (!ref || (field != 0 && field != 1)) return LBGPU_E_ARG;
  return guarded(e, [&] {
    e->ensure_ref();
    CU(cudaMemcpyAsync(e->d_ref, ref, sizeof(double) * e->m * e->N, cudaMemcpyHostToDevice, e->st));
    e->from_ref(field, e->d_ref);
    // ghosts (collective: every rank uploads); an in-place field lands in
    // layout O, whose next sweep reads no ghost
    if (e->xmode == 2 && !e->aa) e->exchange(field);
    e->sync();
  });
}

int lbgpu_download_state(lbgpu_engine* e, int field, double* ref) {
  if (!ref || (field != 0 && field != 1)) return LBGPU_E_ARG;
  return guarded(e, [&] {
    e->ensure_ref();
    e->to_ref(field, e->d_ref);
    CU(cudaMemcpyAsync(ref, e->d_ref, sizeof(double) * e->m * e->N, cudaMemcpyDeviceToHost, e->st));
    e->sync();
  });
}

int lbgpu_upload_state_device(lbgpu_engine* e, int field, const double* d_ref) {
  if (!d_ref || (field != 0 && field != 1)) return LBGPU_E_ARG;
  return guarded(e, [&] {
    e->from_ref(field, d_ref);
    e->sync();
  });
}

int lbgpu_download_state_device(lbgpu_engine* e, int field, double* d_ref) {
  if (!d_ref || (field != 0 && field != 1)) return LBGPU_E_ARG;
  return guarded(e, [&] {
    e->to_ref(field, d_ref);
    e->sync();
  });
}

int lbgpu_set_design(lbgpu_engine* e, const double* w_full) {
  if (!w_full) return LBGPU_E_ARG;
  return guarded(e, [&] {
    e->w2_synced = false;  // non-design values may change
    e->w.assign(w_full, w_full + e->N);
    e->w_host_stale = false;
    e->build_codes();
    CU(cudaMemcpyAsync(e->d_w, e->w.data(), sizeof(double) * e->N, cudaMemcpyHostToDevice, e->st));
    CU(cudaMemcpyAsync(e->d_code, e->code.data(), e->N, cudaMemcpyHostToDevice, e->st));
    e->sync();
    if (e->exact) e->refresh_pow_tables();
  });
}

int lbgpu_get_design(const lbgpu_engine* e, double* w_full) {
  if (!e || !w_full) return LBGPU_E_ARG;
  auto* m = const_cast<lbgpu_engine*>(e);
  return guarded(m, [&] {
    if (m->w_host_stale) {
      CU(cudaMemcpyAsync(m->w.data(), m->d_w, sizeof(double) * m->N, cudaMemcpyDeviceToHost, m->st));
      m->sync();
      m->w_host_stale = false;
    }
    std::memcpy(w_full, m->w.data(), sizeof(double) * m->N);
  });
}

int lbgpu_set_design_values(lbgpu_engine* e, const double* w_design) {
  if (!w_design) return LBGPU_E_ARG;
  return guarded(e, [&] { e->upload_design_values(w_design); });
}

int lbgpu_get_design_values(lbgpu_engine* e, double* w_design) {
  if (!w_design) return LBGPU_E_ARG;
  return guarded(e, [&] {
    std::vector<double> full(e->N);
    if (e->w_host_stale) {
      CU(cudaMemcpyAsync(e->w.data(), e->d_w, sizeof(double) * e->N, cudaMemcpyDeviceToHost, e->st));
      e->sync();
      e->w_host_stale = false;
    }
    for (size_t i = 0; i < e->design.size(); ++i) w_design[i] = e->w[e->design[i]];
  });
}

int lbgpu_primal_step(lbgpu_engine* e, int64_t n, double* residual) {
  return guarded(e, [&] {
    const double r = e->steps(0, n, 0, residual != nullptr);
    if (residual) *residual = r;
  });
}

int lbgpu_primal_step_with_design(lbgpu_engine* e, const double* w_design, int64_t n,
                                  double* residual) {
  if (!w_design || n < 1) return LBGPU_E_ARG;
  return guarded(e, [&] {
    const double r = e->design_steps(w_design, n, residual != nullptr);
    if (residual) *residual = r;
  });
}

int lbgpu_pair_step_with_design(lbgpu_engine* e, const double* w_design, double* primal_residual,
                                double* adjoint_residual, double* objective) {
  if (!w_design) return LBGPU_E_ARG;
  if (e && !primal_residual && !adjoint_residual && e->lazy_pair_ok())
    return guarded(e, [&] { e->design_pair_lazy(w_design, objective); }, true);
  return guarded(e, [&] { e->design_pair(w_design, primal_residual, adjoint_residual, objective); });
}

int lbgpu_finish(lbgpu_engine* e) {
  return guarded(e, [&] { e->sync(); });
}

int lbgpu_tangent_solve(lbgpu_engine* e, const double* dw_design, double d_inlet_dp, double tol,
                        int64_t max_iter, double* dF, int64_t* iterations, double* residual,
                        int* converged) {
  if (!dw_design || !dF || max_iter < 0) return LBGPU_E_ARG;
  return guarded(e, [&] {
    long long it = 0;
    double r = 0.0;
    int c = 0;
    e->tangent(dw_design, d_inlet_dp, tol, max_iter, dF, &it, &r, &c);
    if (iterations) *iterations = it;
    if (residual) *residual = r;
    if (converged) *converged = c;
  });
}

int lbgpu_fd_gradient(lbgpu_engine* e, int64_t ordinal, double h, double tol, int64_t max_iter,
                      int64_t fixed_iters, double* out) {
  if (!out || !(h != 0.0)) return LBGPU_E_ARG;
  return guarded(e, [&] { *out = e->fd_gradient(ordinal, h, tol, max_iter, fixed_iters); });
}

int lbgpu_fd_gradient_batch(lbgpu_engine* e, int64_t n, const int64_t* ordinals,
                            const double* steps, double tol, int64_t max_iter,
                            int64_t fixed_iters, int from_state, double* out) {
  if (n < 0 || (n > 0 && (!ordinals || !steps || !out))) return LBGPU_E_ARG;
  for (int64_t k = 0; k < n; ++k)
    if (!(steps[k] != 0.0)) return LBGPU_E_ARG;
  return guarded(e, [&] {
    std::vector<long long> o(ordinals, ordinals + n);
    e->fd_batch(n, o.data(), steps, tol, max_iter, fixed_iters, from_state != 0, out);
  });
}

int lbgpu_pair_steps(lbgpu_engine* e, int64_t n, double* primal_residual,
                     double* adjoint_residual) {
  if (n < 0) return LBGPU_E_ARG;
  return guarded(e, [&] { e->pair_steps(n, primal_residual, adjoint_residual); });
}

int lbgpu_time_pair_steps(lbgpu_engine* e, int64_t n, double* ms) {
  if (!ms || n < 1) return LBGPU_E_ARG;
  return guarded(e, [&] {
    e->require_solo();
    e->reset_flags();
    e->sync();
    CU(cudaEventRecord(e->ev0, e->st));
    if (!e->fuse_pairs()) {
      for (int64_t k = 0; k < n; ++k) {
        e->primal_launch(false, nullptr);
        e->adjoint_launch(0, false, nullptr);
      }
    } else {
      e->primal_launch(false, nullptr);
      for (int64_t k = 1; k < n; ++k) e->fused_pair_raw(false);
      e->adjoint_launch(0, false, nullptr);
    }
    CU(cudaEventRecord(e->ev1, e->st));
    CU(cudaGetLastError());
    CU(cudaEventSynchronize(e->ev1));
    float t = 0.f;
    CU(cudaEventElapsedTime(&t, e->ev0, e->ev1));
    *ms = t;
    e->reduce_flags(e->d_flags + 1, 1, true);
    e->check_bad("iteration");
  });
}

int lbgpu_adjoint_step(lbgpu_engine* e, int64_t n, int kernel, double* residual) {
  if (kernel != 0 && kernel != 1) return LBGPU_E_ARG;
  return guarded(e, [&] {
    const double r = e->steps(1, n, kernel, residual != nullptr);
    if (residual) *residual = r;
  });
}

int lbgpu_solve_primal(lbgpu_engine* e, double tol, int64_t max_iter, int64_t fixed,
                       int64_t* iters, double* residual, int* converged) {
  if (!iters || !residual || !converged) return LBGPU_E_ARG;
  return guarded(e, [&] {
    long long it = 0;
    e->solve(0, tol, max_iter, fixed, 0, &it, residual, converged);
    *iters = it;
  });
}

int lbgpu_solve_adjoint(lbgpu_engine* e, double tol, int64_t max_iter, int64_t fixed, int kernel,
                        int64_t* iters, double* residual, int* converged) {
  if (!iters || !residual || !converged || (kernel != 0 && kernel != 1)) return LBGPU_E_ARG;
  return guarded(e, [&] {
    long long it = 0;
    e->solve(1, tol, max_iter, fixed, kernel, &it, residual, converged);
    *iters = it;
  });
}

int lbgpu_param_gradient(lbgpu_engine* e, int kernel, double* g, double* gdp) {
  if (kernel != 0 && kernel != 1) return LBGPU_E_ARG;
  return guarded(e, [&] { e->gradient(kernel, g, gdp); });
}

int lbgpu_objective(lbgpu_engine* e, double* value) {
  if (!value) return LBGPU_E_ARG;
  return guarded(e, [&] { *value = e->objective(); });
}

int lbgpu_penalty(lbgpu_engine* e, double* value) {
  if (!value) return LBGPU_E_ARG;
  return guarded(e, [&] { *value = e->penalty(); });
}

int lbgpu_one_shot(lbgpu_engine* e, int64_t iterations, const double* zeta, const double* lambda,
                   int64_t record_interval, lbgpu_run_row* rows, int64_t cap, int64_t* n_rows) {
  if (!zeta || !lambda || !n_rows || record_interval < 1 || iterations < 0) return LBGPU_E_ARG;
  return guarded(e, [&] {
    long long nr = 0;
    e->one_shot(1, iterations, iterations, zeta, lambda, record_interval, rows, cap, &nr);
    *n_rows = nr;
  });
}

int lbgpu_one_shot_range(lbgpu_engine* e, int64_t first, int64_t count, int64_t total,
                         const double* zeta, const double* lambda, int64_t record_interval,
                         lbgpu_run_row* rows, int64_t cap, int64_t* n_rows) {
  if (!zeta || !lambda || !n_rows || record_interval < 1 || count < 0 || first < 1)
    return LBGPU_E_ARG;
  return guarded(e, [&] {
    long long nr = 0;
    e->one_shot(first, count, total, zeta, lambda, record_interval, rows, cap, &nr);
    *n_rows = nr;
  });
}

int lbgpu_continue_adjoint(lbgpu_engine* e, double tol, int64_t max_iter, int64_t fixed,
                           int kernel, int64_t* iters, double* residual, int* converged) {
  if (!iters || !residual || !converged || (kernel != 0 && kernel != 1)) return LBGPU_E_ARG;
  return guarded(e, [&] {
    long long it = 0;
    e->solve(1, tol, max_iter, fixed, kernel, &it, residual, converged, false);
    *iters = it;
  });
}

int lbgpu_time_sweeps(lbgpu_engine* e, int which, int64_t steps, double* ms) {
  if (!ms || steps < 0 || which < 0 || which > 2) return LBGPU_E_ARG;
  return guarded(e, [&] {
    if (which == 2 && !e->fuse_pairs())
      throw Fail{LBGPU_E_STATE, "fused pair sweeps run in the FP64 product build only"};
    e->reset_flags();
    e->sync();
    CU(cudaEventRecord(e->ev0, e->st));
    {
      // adjoint sweeps share one frozen base: its moment cache is built (and
      // timed) once, as in a steady solve
      lbgpu_engine::MomScope ms(e, which == 1 ? steps : 0, 0);
      for (int64_t k = 0; k < steps; ++k) {
        if (which == 0) e->primal_launch(false, nullptr);
        else if (which == 1) e->adjoint_launch(0, false, nullptr);
        else e->fused_pair_raw(false);
      }
    }
    CU(cudaEventRecord(e->ev1, e->st));
    CU(cudaGetLastError());
    CU(cudaEventSynchronize(e->ev1));
    float t = 0.f;
    CU(cudaEventElapsedTime(&t, e->ev0, e->ev1));
    *ms = t;
    e->check_bad(which == 1 ? "adjoint iteration" : "iteration");
  });
}

int lbgpu_unsteady_adjoint(lbgpu_engine* e, int64_t n_steps, int sum_objective, int64_t slots,
                           double* g_design, double* g_inlet_dp, double* J,
                           int64_t* forward_sweeps) {
  if (n_steps < 1 || slots < 1) return LBGPU_E_ARG;
  return guarded(e, [&] {
    long long fs = 0;
    e->unsteady(n_steps, sum_objective != 0, slots, g_design, g_inlet_dp, J, &fs);
    if (forward_sweeps) *forward_sweeps = fs;
  });
}

int lbgpu_time_pairs(lbgpu_engine* e, int64_t steps, double* ms_total, double* ms_primal,
                     double* ms_adjoint) {
  if (!ms_total || !ms_primal || !ms_adjoint || steps < 1) return LBGPU_E_ARG;
  return guarded(e, [&] {
    const size_t need = size_t(2 * steps + 1);
    while (e->evs.size() < need) {
      cudaEvent_t ev;
      CU(cudaEventCreate(&ev));
      e->evs.push_back(ev);
    }
    e->reset_flags();
    e->sync();
    CU(cudaEventRecord(e->evs[0], e->st));
    for (int64_t k = 0; k < steps; ++k) {
      e->primal_launch(false, nullptr);
      CU(cudaEventRecord(e->evs[2 * k + 1], e->st));
      e->adjoint_launch(0, false, nullptr);
      CU(cudaEventRecord(e->evs[2 * k + 2], e->st));
    }
    CU(cudaGetLastError());
    CU(cudaEventSynchronize(e->evs[2 * steps]));
    double tp = 0.0, ta = 0.0;
    for (int64_t k = 0; k < steps; ++k) {
      float a = 0.f, b = 0.f;
      CU(cudaEventElapsedTime(&a, e->evs[2 * k], e->evs[2 * k + 1]));
      CU(cudaEventElapsedTime(&b, e->evs[2 * k + 1], e->evs[2 * k + 2]));
      tp += a;
      ta += b;
    }
    float tot = 0.f;
    CU(cudaEventElapsedTime(&tot, e->evs[0], e->evs[2 * steps]));
    *ms_total = tot;
    *ms_primal = tp;
    *ms_adjoint = ta;
    e->check_bad("iteration");
  });
}

}  // extern "C"

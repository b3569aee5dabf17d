// Plain structs shared by the kernels and the host engine.
#pragma once
#include <cuda_runtime.h>

#include "physics.cuh"

namespace lbgpu {

struct Geom {
  int nx, ny, nz;   // local array extents
  int x0, x1;       // computed (owned) local columns [x0, x1)
  long long N;      // nodes of the local array = plane stride
  int gx_off;       // global x = local x + gx_off
  int gnx, gny;     // global extents (flat index for error reports)
  int z0 = 0;       // first z plane of a z-chunked sweep (grid.z counts from here)
};

struct NodeTables {
  const uint8_t* code;
  const double* w;
  const double* w_adj;  // the design the adjoint half of a lazy design pair uses (else == w)
  const double* bcT;
  const double* p0;  // exact build: host-glibc pow(base, theta) per node
  const double* p1;  //              pow(base, theta - 1)
  const long long* grad_side;  // design positions whose node is not Interior (dual gradient)
  long long n_grad_side;
  PowPair pp_one;    // pow pair of non-design nodes (w == 1)
  double omt_one;    // thermal relaxation rate at w == 1
};

struct Flags {
  unsigned long long* resid;  // NaN-propagating max |new-old| as a bit pattern
  unsigned long long* bad;    // smallest global flat index with rho <= 0
  unsigned long long* aux;    // kernel-specific (max |comp| for design updates)
  unsigned long long step_key;  // (step number << 40): orders "bad" reports by step
};

// P2P halo push targets (in-process slab groups linked with
// lbgpu_group_link_p2p): the neighbours' destination buffers of this sweep,
// possibly on other devices (peer memory), and where their ghost columns sit.
// Index 0 is the primal field's destination, 1 the adjoint field's (a fused
// pair sweep pushes both).
struct Push {
  void* l_dst[2] = {nullptr, nullptr};  // left neighbour: its right ghost column l_col
  void* r_dst[2] = {nullptr, nullptr};  // right neighbour: its left ghost column r_col
  int l_col = 0, l_nx = 0, r_col = 0, r_nx = 0;
  long long l_N = 0, r_N = 0;
};

// Upload-gated design sweep (the deferred design pair's single launch): the
// design nodes form the box [bx0,bx1) x [by0,by1) x [bz0,bz1) (interior x the
// design x-range, config.cpp:347-371), whose design values arrive by one H2D
// copy into wd, in DesignField::nodes order. Every entry of wd holds the
// sentinel kGateEmpty until its value lands: the value is its own flag. A
// thread whose node is in the box waits for it, takes it (re-arming the entry
// with the sentinel for the next upload) and writes it into the full-grid
// design buffer w_out.
constexpr unsigned long long kGateEmpty = 0x7ff4dead0000beefull;  // a NaN no upload carries
struct Gate {
  double* wd = nullptr;
  double* w_out = nullptr;
  unsigned* err = nullptr;  // set when a value never landed (bounded wait)
  int bx0 = 0, bx1 = 0, by0 = 0, by1 = 0, bz0 = 0, bz1 = 0;
  // J's inputs on the way (obj_x >= 0): the nodes of columns obj_x - 1 .. obj_x + 1
  // also store the post values that stream into the objective's support plane
  // x = obj_x, at inbox[P (ny nz) + y + ny z] of the receiving node (y, z)
  double* inbox = nullptr;
  int obj_x = -1;
};

// One-shot design update carried by the next primal sweep (k_primal UPD):
// the gradient of the previous adjoint state v at each interior design node,
// composite and clamped ascent step (optimizer.cpp:41-45, :8-16), then the
// collision with the new w.
struct Upd {
  const void* v = nullptr;  // adjoint state (double-buffered post layout)
  double* w = nullptr;      // design, updated in place
  double zeta = 0.0, lambda = 0.0;
  // adjoint sweep (k_adjoint GRAD, the unsteady adjoint's back step): the
  // design gradient of the sweep's own inputs (base f, v) accumulated per node
  double* gacc = nullptr;
};

struct Launch {
  Upd upd;
  Gate gate;
  Push push;
  Geom g;
  NodeTables t;
  Model M;
  Flags fl;
  cudaStream_t stream;
};

struct SweepArgs {
  Launch a;
  int dim, prec, ck;  // ck: 0 bgk, 1 mrt (shear rows), 2 mrt + non-hydro rows
  bool resid;
  const long long* adj_side;  // adjoint side-list nodes (k_adjoint_side)
  long long n_adj_side;
  int part;  // 0 all owned columns, 2 the boundary strips only (kernels.cuh kStrip), 1 the rest
  int z0 = 0, z1 = 0;  // z planes [z0, z1) only (z1 = 0: all)
  const void* mom = nullptr;  // adjoint: cached moments of a frozen base (fast build)
  int fm = 0, vm = 0;  // addressing modes of f and v: 0 double-buffered, 1/2 in place (O/E)
  bool dualw = false;  // fused pair: the adjoint half reads w from a.t.w_adj (3-D, no residual)
  bool upd = false;    // primal: apply a.upd (the previous one-shot iteration's update) first
};

// Launchers, one set per build (k_fast_*.cu / k_exact_*.cu).
#define LBGPU_DECLARE_LAUNCHERS(NS)                                                          \
  namespace NS {                                                                           \
  void primal(const SweepArgs& s, const void* src, void* dst);                             \
  void adjoint(const SweepArgs& s, const void* base, const void* src, void* dst);          \
  void adjoint_dual(const SweepArgs& s, const void* base, const void* src, void* dst);     \
  void gradient(const Launch& a, int dim, int prec, int ak, bool update, const void* p,    \
                const void* q, const long long* nodes, long long n, double* gout,          \
                double* w_rw, double zeta, double lambda, int accumulate, int bm, int vm); \
  void objective_terms(const Launch& a, int dim, int prec, const void* p,                  \
                       const long long* nodes, long long n, double* terms, int bm);        \
  void objective_inbox(const Launch& a, int dim, int prec, const double* inbox,            \
                       const long long* nodes, long long n, double* terms);                \
  void inlet_terms(const Launch& a, int dim, int prec, const void* p, const void* q,       \
                   const long long* nodes, long long n, double* terms, int bm, int vm);    \
  void layout(const Geom& g, int dim, int prec, int field, bool to_ref, const void* in,    \
              void* out, cudaStream_t st, int fm);                                         \
  void init_state(long long N, int dim, int prec, void* buf, cudaStream_t st);             \
  void base_moments(const Launch& a, int dim, int prec, int bm, const void* base, void* mom); \
  void primal_aa(const SweepArgs& s, void* A);                                             \
  void adjoint_aa(const SweepArgs& s, const void* base, void* V);                          \
  void pair_aa(const SweepArgs& s, void* F, void* V);                                      \
  void pair(const SweepArgs& s, const void* fsrc, void* fdst, const void* vsrc, void* vdst);  \
  void tangent(const SweepArgs& s, const void* base, const void* src, void* dst,              \
               const double* dw, double d_rho_in);                                           \
  void tangent_terms(const Launch& a, int dim, int prec, const void* base, const void* df,   \
                     const long long* nodes, long long n, double* terms);                    \
  void halo(int op, const Geom& g, int dim, int prec, int field, void* buf, void* a, void* b, \
            const void* left, const Geom& gl, const void* right, const Geom& gr,             \
            cudaStream_t st);                                                              \
  }
LBGPU_DECLARE_LAUNCHERS(fast)
LBGPU_DECLARE_LAUNCHERS(exact)

}  // namespace lbgpu

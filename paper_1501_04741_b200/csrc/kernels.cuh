// Device kernels of the hot path. This header is compiled twice:
//   kernels_fast.cu  (LBGPU_EXACT=0, FMA contraction on): the product path —
//       pull-scheme sweeps with the algebraically reduced collision
//       (rank-r MRT, moment-form adjoint, hand-derived pressure-face VJP);
//   kernels_exact.cu (LBGPU_EXACT=1, -fmad=false): the reference-order
//       formulation of physics.cuh everywhere (dense A, dual-number face
//       VJP), bit-for-bit equal to the reference on identical inputs.
//
// Storage: SoA planes, plane p at p*N, node index x + nx*(y + ny*z) — the
// reference layout (lattice.hpp:54-100) — but the buffers hold
// POST-collision values (pull scheme). The reference's pre-collision state is
// f_p(x) = post_p(x - e_p) for the primal and v_p(x) = post_p(x + e_p) for the
// adjoint (which streams against the links, adjoint.cpp:239-249); k_to_ref /
// k_from_ref convert. Streaming is a permutation, so the max-norm step
// residual of the post-collision buffers equals the reference's
// step_residual (collision.cpp:365-375) exactly.
#pragma once
#include <cuda_runtime.h>

#include "types.cuh"

#ifndef LBGPU_EXACT
#error "define LBGPU_EXACT"
#endif
#if LBGPU_EXACT
#define LBGPU_NS exact
#else
#define LBGPU_NS fast
#endif

namespace lbgpu {
namespace LBGPU_NS {  // per-build namespace: distinct kernel symbols per build

namespace detail {

LBGPU_HD long long gflat(const Geom& g, int x, int y, int z) {
  return (long long)(x + g.gx_off) + (long long)g.gnx * (y + (long long)g.gny * z);
}

// Neighbour coordinate tables with periodic wrap on every axis of the local
// array (primal_step's modular wrap, collision.cpp:343-351). Slab runs never
// wrap in x because their computed columns exclude the ghost columns.
// Node offsets are 32-bit (the engine holds N < 2^31 nodes per device): each
// population address is then the plane's base (buf + P N, warp-uniform, in
// uniform registers) plus one 32-bit offset -- one IMAD.WIDE per access
// instead of a chain of 64-bit adds.
struct Nbr {
  int xs[3], ys[3], zs[3];
};
__device__ __forceinline__ Nbr make_nbr(const Geom& g, int x, int y, int z) {
  Nbr n;
  n.xs[0] = x == 0 ? g.nx - 1 : x - 1;
  n.xs[1] = x;
  n.xs[2] = x == g.nx - 1 ? 0 : x + 1;
  const int ym = y == 0 ? g.ny - 1 : y - 1, yp = y == g.ny - 1 ? 0 : y + 1;
  const int zm = z == 0 ? g.nz - 1 : z - 1, zp = z == g.nz - 1 ? 0 : z + 1;
  n.ys[0] = g.nx * ym;
  n.ys[1] = g.nx * y;
  n.ys[2] = g.nx * yp;
  const int pl = g.nx * g.ny;
  n.zs[0] = pl * zm;
  n.zs[1] = pl * z;
  n.zs[2] = pl * zp;
  return n;
}
// Node index of x + D*e_P (D = -1: primal pull source, +1: adjoint pull source).
template <class L, int P, int D>
__device__ __forceinline__ int nbr_idx(const Nbr& n) {
  constexpr int ex = D * cvel<L>(P, 0), ey = D * cvel<L>(P, 1), ez = D * cvel<L>(P, 2);
  return n.xs[1 + ex] + n.ys[1 + ey] + n.zs[1 + ez];
}
// Population P of node i: plane base first (uniform), then the node offset.
// (32-bit element offsets P N + i, valid while M N < 2^32, measured mixed on
// B200 C3: FP32 in-place adjoint +4%, the FP64 fused pair -5%; not used.)
template <class R>
__device__ __forceinline__ R* pop(R* buf, long long N, int P, int i) {
  return (buf + P * N) + i;
}

template <class L, class R, int D>
__device__ __forceinline__ void gather(const R* __restrict__ buf, long long N, const Nbr& n,
                                       R* out) {
  LBGPU_FOR(P, 0, L::M, { out[P] = __ldg(pop(buf, N, P, nbr_idx<L, P, D>(n))); });
}

// Split adjoint: stage the v gather through shared memory (see adjoint_body).
#ifndef LBGPU_ADJ_STAGE
#define LBGPU_ADJ_STAGE 1
#endif
// FP64 split adjoint: the VJP reads the staged v in place instead of from a
// register copy. C3 with / without: frozen base 12,831 / 12,569 MLUPS, in
// place 6,582 / 6,497 GB/s (frozen 12,559 / 12,114); at 5 blocks per SM it
// spills 96 B and is slower.
#ifndef LBGPU_ADJ_VSMEM
#define LBGPU_ADJ_VSMEM 1
#endif
// Fused pair: its adjoint half reading the staged v in place measured no
// different (C3 7,699 against 7,692-7,695 MLUPS): off.
#ifndef LBGPU_PAIR_VSMEM
#define LBGPU_PAIR_VSMEM 0
#endif
#ifndef LBGPU_ADJ_STAGE32  // the FP32 split adjoint too
#define LBGPU_ADJ_STAGE32 0
#endif
// FP32 split adjoint: v's gather addresses re-formed after the moments (opaque)
// instead of kept from the base gather: C3 5,674 -> 5,737 GB/s (8 blocks per SM;
// at 6 blocks 5,357).
#ifndef LBGPU_ADJ_REMAT32
#define LBGPU_ADJ_REMAT32 1
#endif

// Asynchronous gather into shared memory (cp.async, LDGSTS): the loads are
// in flight without holding registers, so a sweep can issue one gather while
// it consumes another. Slot P of this thread is smem[P * stride].
template <class R>
__device__ __forceinline__ void cp_async_elem(R* smem, const R* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if constexpr (sizeof(R) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}
template <class L, class R, int D>
__device__ __forceinline__ void gather_async(const R* __restrict__ buf, long long N, const Nbr& n,
                                             R* smem, int stride) {
  LBGPU_FOR(P, 0, L::M, { cp_async_elem(smem + P * stride, pop(buf, N, P, nbr_idx<L, P, D>(n))); });
  cp_async_commit();
}

// ---------------------------------------------------------------------
// Field addressing modes. FM_DB: the double-buffered pull layout (the
// buffers hold post-collision values; a sweep reads its neighbours' from one
// buffer and writes its own node in the other). In-place (AA-pattern)
// streaming keeps ONE buffer per field and alternates two layouts:
//   FM_O: slot p at node y holds the pre-collision value f_p(y) = post_p(y + D e_p)
//         (exactly the reference's layout, lattice.hpp:54-100);
//   FM_E: slot opp(p) at node x holds x's own post-collision value post_p(x).
// A sweep from O reads and writes its own node only (and leaves E); a sweep
// from E reads post_p(x + D e_p) at (opp p, x + D e_p) and writes post_q(x)
// to (q, x - D e_q) (and leaves O). Since e_opp(p) = -e_p, the locations a
// node writes are exactly the ones it read, so each sweep is in place and
// race-free, at the same 2 M s bytes per node as the double buffer with half
// the memory. D = -1 for the primal field, +1 for the adjoint (which streams
// against the links, adjoint.cpp:239-249).
enum : int { FM_DB = 0, FM_O = 1, FM_E = 2 };
// where node idx reads its pre-collision population P / writes its post value P
template <class L, int D, int FM, int P, class R>
__device__ __forceinline__ R* in_at(R* buf, long long N, long long idx, const Nbr& n) {
  if constexpr (FM == FM_DB) return pop(buf, N, P, nbr_idx<L, P, D>(n));
  else if constexpr (FM == FM_O) return pop(buf, N, P, int(idx));
  else return pop(buf, N, copp<L>(P), nbr_idx<L, P, D>(n));
}
template <class L, int D, int FM, int P, class R>
__device__ __forceinline__ R* out_at(R* buf, long long N, long long idx, const Nbr& n) {
  if constexpr (FM == FM_DB) return pop(buf, N, P, int(idx));
  else if constexpr (FM == FM_O) return pop(buf, N, copp<L>(P), int(idx));
  else return pop(buf, N, P, nbr_idx<L, P, -D>(n));
}
// gather of the pre-collision populations of node idx under mode FM
template <class L, class R, int D, int FM>
__device__ __forceinline__ void gather_m(const R* buf, long long N, long long idx, const Nbr& n,
                                         R* out) {
  LBGPU_FOR(P, 0, L::M, { out[P] = __ldg(in_at<L, D, FM, P>(buf, N, idx, n)); });
}
template <class L, class R, int D, int FM>
__device__ __forceinline__ void gather_async_m(const R* buf, long long N, long long idx,
                                               const Nbr& n, R* smem, int stride) {
  LBGPU_FOR(P, 0, L::M, { cp_async_elem(smem + P * stride, in_at<L, D, FM, P>(buf, N, idx, n)); });
  cp_async_commit();
}
// A copy of the neighbour offsets the compiler cannot prove equal to the
// original: addresses derived from it are recomputed where they are used
// instead of being kept live from an earlier gather.
__device__ __forceinline__ Nbr opaque(const Nbr& n) {
  Nbr m;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    asm volatile("mov.b32 %0, %1;" : "=r"(m.xs[k]) : "r"(n.xs[k]));
    asm volatile("mov.b32 %0, %1;" : "=r"(m.ys[k]) : "r"(n.ys[k]));
    asm volatile("mov.b32 %0, %1;" : "=r"(m.zs[k]) : "r"(n.zs[k]));
  }
  return m;
}

// in-place store of node idx's post-collision values (FM_O / FM_E)
// C3 MLUPS with / without: FP64 in-place pair 7,523 / 7,076 (its E/E form spilled 304 B
// without), FP32 frozen-base in-place adjoint 23,103 / 18,842; the sweeps apart +0-2%.
#ifndef LBGPU_AA_REMAT
#define LBGPU_AA_REMAT 1
#endif
template <class L, class R, int D, int FM>
__device__ __forceinline__ void store_aa(R* buf, long long N, long long idx, const Nbr& n,
                                         const R* v) {
  static_assert(FM != FM_DB, "double-buffered stores go through store_node");
  if constexpr (FM == FM_E && LBGPU_AA_REMAT) {
    // the 26 shifted store addresses formed here from 9 integers instead of
    // being kept live (as the gather's) across the collision
    const Nbr m = opaque(n);
    LBGPU_FOR(P, 0, L::M, { *out_at<L, D, FM, P>(buf, N, idx, m) = v[P]; });
  } else {
    LBGPU_FOR(P, 0, L::M, { *out_at<L, D, FM, P>(buf, N, idx, n) = v[P]; });
  }
}

// Planes that cross a slab cut for a sweep pulling along D (-1 primal, +1
// adjoint): side S = -1 are pulled from the left neighbour (D*e_x == -1), S =
// +1 from the right one; the adjoint's lists are the primal's swapped, the
// reference's transposed plan (partition.cpp:143-146).
template <class L, int D, int S>
__device__ __forceinline__ constexpr int halo_slot(int k) {
  int c = 0;
  for (int p = 0; p < L::M; ++p)
    if (D * cvel<L>(p, 0) == S) {
      if (c == k) return p;
      ++c;
    }
  return -1;
}
template <class L>
constexpr int kHaloPlanes = 6;  // D2Q9+D2Q9: 3+3, D3Q19+D3Q7: 5+1

// Fused P2P halo: a lane on the slab's first / last owned column also stores
// the planes its neighbour will pull across the cut straight into that
// neighbour's destination ghost column (peer memory when the neighbour lives
// on another GPU). No pack, no separate exchange kernel.
template <class L, class R, int D>
__device__ __forceinline__ void push_halo(const Launch& a, int x, int y, int z, const R* out) {
  const Push& h = a.push;
  constexpr int F = D == -1 ? 0 : 1;  // the field pulled along D
  const long long row = y + (long long)a.g.ny * z;
  if (h.r_dst[F] && x == a.g.x1 - 1) {  // my last column -> right neighbour's left ghost
    R* d = static_cast<R*>(h.r_dst[F]);
    const long long i = (long long)h.r_nx * row + h.r_col;
    LBGPU_FOR(K, 0, kHaloPlanes<L>, {
      constexpr int p = halo_slot<L, D, -1>(K);
      d[p * h.r_N + i] = out[p];
    });
  }
  if (h.l_dst[F] && x == a.g.x0) {  // my first column -> left neighbour's right ghost
    R* d = static_cast<R*>(h.l_dst[F]);
    const long long i = (long long)h.l_nx * row + h.l_col;
    LBGPU_FOR(K, 0, kHaloPlanes<L>, {
      constexpr int p = halo_slot<L, D, +1>(K);
      d[p * h.l_N + i] = out[p];
    });
  }
}

__device__ __forceinline__ unsigned long long absdiff_bits(double a, double b) {
  return (unsigned long long)__double_as_longlong(fabs(a - b));
}

// Block-wide max of a bit pattern, one atomicMax per block. Warps are
// numbered by linear thread id (2-D blocks), and the leading barrier keeps a
// second call in the same kernel from overwriting `red` while warp 0 of the
// first call still reads it.
__device__ __forceinline__ void block_max_bits(unsigned long long v, unsigned long long* dst) {
  __shared__ unsigned long long red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int lane = tid & 31, warp = tid >> 5;
  const int nwarp = (blockDim.x * blockDim.y * blockDim.z + 31) >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < nwarp ? red[lane] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long u = __shfl_xor_sync(0xffffffffu, v, o);
      v = u > v ? u : v;
    }
    if (lane == 0 && v) atomicMax(dst, v);
  }
}

template <bool EXACT>
__device__ __forceinline__ PowPair node_pp(const Model& M, const NodeTables& t, long long idx,
                                           uint8_t code, double w) {
  if (!(code & CODE_HAS_W)) return t.pp_one;
  if constexpr (EXACT) {
    (void)M;
    (void)w;
    return {t.p0[idx], t.p1[idx]};
  } else {
    return pow_pair(M, w);
  }
}

__device__ __forceinline__ int code_axis(uint8_t c) { return (c >> CODE_AXIS_SHIFT) & 3; }
__device__ __forceinline__ int code_sign(uint8_t c) { return (c & CODE_NEG) ? -1 : 1; }

// ---------------------------------------------------------------------
// Fast interior collision: f' = feq(rho, G u) + A (f - feq(rho, u)) with A
// applied in moment space, A = sum_i c_i U_i^T U_i over the relaxing rows
// (U has orthogonal rows, so U^-1 = U^T diag(1/|U_i|^2)); the conserved rows
// drop out at compile time, and with omega_nonhydro = 1 only the shear rows
// remain (rank 2 in 2D, 5 in 3D). BGK is A = (1 - omega) I.
template <class L, class R, int CK>
__device__ __forceinline__ bool fast_collide_m(const Model& M, PowPair pp, double omt,
                                               const R* fin, R rho, R j0, R j1, R j2, R T,
                                               R* out);
// The moment sums of a gathered node, in the order fast_collide and the
// moment-form VJP both use (so a fused sweep can share them bit for bit).
template <class L, class R>
__device__ __forceinline__ void node_sums(const R* fin, R& rho, R* j, R& T) {
  R r = R(0), j0 = R(0), j1 = R(0), j2 = R(0);
  LBGPU_FOR(J, 0, L::MF, {
    r += fin[J];
    if constexpr (L::ef(J, 0) != 0) j0 = L::ef(J, 0) > 0 ? j0 + fin[J] : j0 - fin[J];
    if constexpr (L::ef(J, 1) != 0) j1 = L::ef(J, 1) > 0 ? j1 + fin[J] : j1 - fin[J];
    if constexpr (L::ef(J, 2) != 0) j2 = L::ef(J, 2) > 0 ? j2 + fin[J] : j2 - fin[J];
  });
  R t = R(0);
#pragma unroll
  for (int k = 0; k < L::MT; ++k) t += fin[L::MF + k];
  rho = r, j[0] = j0, j[1] = j1, j[2] = j2, T = t;
}
template <class L, class R, int CK>
__device__ __forceinline__ bool fast_collide(const Model& M, PowPair pp, double omt,
                                             const R* fin, R* out) {
  R rho, j[3], T;
  node_sums<L, R>(fin, rho, j, T);
  return fast_collide_m<L, R, CK>(M, pp, omt, fin, rho, j[0], j[1], j[2], T, out);
}
// The collision given 1/rho (rho > 0 checked by the caller): a fused pair
// sweep takes the reciprocal once for both halves.
template <class L, class R, int CK>
__device__ __forceinline__ void fast_collide_mi(const Model& M, PowPair pp, double omt,
                                                const R* fin, R rho, R inv, R j0, R j1, R j2,
                                                R T_, R* out);
template <class L, class R, int CK>
__device__ __forceinline__ bool fast_collide_m(const Model& M, PowPair pp, double omt,
                                               const R* fin, R rho, R j0, R j1, R j2, R T_,
                                               R* out) {
  if (!(rho > R(0))) return false;
  fast_collide_mi<L, R, CK>(M, pp, omt, fin, rho, R(1) / rho, j0, j1, j2, T_, out);
  return true;
}
template <class L, class R, int CK>
__device__ __forceinline__ void fast_collide_mi(const Model& M, PowPair pp, double omt,
                                                const R* fin, R rho, R inv, R j0, R j1, R j2,
                                                R T_, R* out) {
  const R u[3] = {j0 * inv, j1 * inv, j2 * inv};
  const R G = M.fluid_power ? R(pp.p0) : R(1.0 - pp.p0);
  const R up[3] = {G * u[0], G * u[1], G * u[2]};
  const R a0 = R(1) - R(1.5) * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
  const R b0 = R(1) - R(1.5) * (up[0] * up[0] + up[1] * up[1] + up[2] * up[2]);
  R df[L::MF];
  LBGPU_FOR(J, 0, L::MF, {
    const R eu = edotp<L, R, J>(u), eup = edotp<L, R, J>(up);
    const R wr = R(L::wf(J)) * rho;
    df[J] = fin[J] - wr * (a0 + eu * (R(3) + R(4.5) * eu));
    out[J] = wr * (b0 + eup * (R(3) + R(4.5) * eup));
  });
  if constexpr (CK == 0) {
    const R c = R(1.0 - M.om);
#pragma unroll
    for (int j = 0; j < L::MF; ++j) out[j] += c * df[j];
  } else {
    LBGPU_FOR(I, 0, L::MF, {
      if constexpr (L::row_class(I) == 1 || (CK == 2 && L::row_class(I) == 2)) {
        R m = R(0);
        LBGPU_FOR(J, 0, L::MF, {
          constexpr double uij = L::U(I, J);
          if constexpr (uij != 0.0) m += R(uij) * df[J];
        });
        m *= R(M.mrt_c[I]);
        LBGPU_FOR(J, 0, L::MF, {
          constexpr double uij = L::U(I, J);
          if constexpr (uij != 0.0) out[J] += R(uij) * m;
        });
      }
    });
  }
  const R* g = fin + L::MF;
  const R T = T_;
  const R om = R(omt);
  LBGPU_FOR(J, 0, L::MT, {
    const R eup = edotp<L, R, L::MF + J>(up);
    const R geq = R(L::wt(J)) * T * (R(1) + R(3) * eup);
    out[L::MF + J] = g[J] + om * (geq - g[J]);
  });
}

// Thermal relaxation rate of a node (collision.cpp:210-211).
template <class R>
__device__ __forceinline__ double node_omt(const Model& M, const NodeTables& t, uint8_t code,
                                           double w) {
  if (!(code & CODE_HAS_W)) return t.omt_one;
  const R wr = R(w);
  const R beta = wr * R(M.beta_f) + (R(1) - wr) * R(M.beta_s);
  return double(R(1) / (R(0.5) + R(3) * beta));
}

// Fast transpose of the interior collision Jacobian (interior_vjp,
// adjoint.cpp:50-121) in moment form: every contraction with d feq/d(rho,u)
// is accumulated directly from w_j x_j, e_j . u and e_j . G u, and A^T = A
// (symmetric for an orthogonal moment basis) is applied like the primal.
// Flow moments rho, j (and 1/rho) of one node's flow populations.
template <class L, class R>
__device__ __forceinline__ void flow_sums(const R* f, R& rho, R* j) {
  R r = R(0), j0 = R(0), j1 = R(0), j2 = R(0);
  LBGPU_FOR(J, 0, L::MF, {
    r += f[J];
    if constexpr (L::ef(J, 0) != 0) j0 = L::ef(J, 0) > 0 ? j0 + f[J] : j0 - f[J];
    if constexpr (L::ef(J, 1) != 0) j1 = L::ef(J, 1) > 0 ? j1 + f[J] : j1 - f[J];
    if constexpr (L::ef(J, 2) != 0) j2 = L::ef(J, 2) > 0 ? j2 + f[J] : j2 - f[J];
  });
  rho = r, j[0] = j0, j[1] = j1, j[2] = j2;
}

// The interior VJP reads the base state only through rho, u and T
// (adjoint.cpp:59, :95): the moment-form entry point takes those.
// VS: the stride of vf / vg (1: registers; 128: a thread's slots of a
// shared-memory staging buffer, read in place).
// The VJP given 1/rho (rho > 0 checked by the caller).
template <class L, class R, int CK, int VS = 1>
__device__ __forceinline__ void fast_vjp_mi(const Model& M, PowPair pp, double omt, R rho,
                                            R inv, const R* jv, R T, const R* vf, const R* vg,
                                            R* outf, R* outg) {
  const R u[3] = {jv[0] * inv, jv[1] * inv, jv[2] * inv};
  const R G = M.fluid_power ? R(pp.p0) : R(1.0 - pp.p0);
  const R up[3] = {G * u[0], G * u[1], G * u[2]};
  const R a0 = R(1) - R(1.5) * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
  const R b0 = R(1) - R(1.5) * (up[0] * up[0] + up[1] * up[1] + up[2] * up[2]);

  // r = A^T vf = sum_i U_i^T c_i (U_i . vf) over the relaxing rows (A is
  // symmetric). Only the few row moments mm_i are kept; r_j is rebuilt where
  // it is used, which keeps ~M fewer values live than storing r.
  R mm[L::MF];
  if constexpr (CK != 0) {
    LBGPU_FOR(I, 0, L::MF, {
      if constexpr (L::row_class(I) == 1 || (CK == 2 && L::row_class(I) == 2)) {
        R m = R(0);
        LBGPU_FOR(J, 0, L::MF, {
          constexpr double uij = L::U(I, J);
          if constexpr (uij != 0.0) m += R(uij) * vf[J * VS];
        });
        mm[I] = m * R(M.mrt_c[I]);
      }
    });
  }
  const R cb = R(1.0 - M.om);
  auto rj = [&]<int J>() -> R {
    if constexpr (CK == 0) {
      return cb * vf[J * VS];
    } else {
      R acc = R(0);
      LBGPU_FOR(I, 0, L::MF, {
        if constexpr (L::row_class(I) == 1 || (CK == 2 && L::row_class(I) == 2)) {
          constexpr double uij = L::U(I, J);
          if constexpr (uij != 0.0) acc += R(uij) * mm[I];
        }
      });
      return acc;
    }
  };

  R Pr = R(0), Rr = R(0), P0 = R(0), R0 = R(0);
  R Pu[3] = {R(0), R(0), R(0)}, Ru[3] = {R(0), R(0), R(0)};
  LBGPU_FOR(J, 0, L::MF, {
    const R eu = edotp<L, R, J>(u), eup = edotp<L, R, J>(up);
    const R tv = R(L::wf(J)) * vf[J * VS];
    const R tr = R(L::wf(J)) * rj.template operator()<J>();
    Pr += tv * (b0 + eup * (R(3) + R(4.5) * eup));
    Rr += tr * (a0 + eu * (R(3) + R(4.5) * eu));
    P0 += tv;
    R0 += tr;
    const R sp = tv * (R(3) + R(9) * eup);
    const R sr = tr * (R(3) + R(9) * eu);
    if constexpr (L::ef(J, 0) != 0) { Pu[0] += L::ef(J, 0) > 0 ? sp : -sp; Ru[0] += L::ef(J, 0) > 0 ? sr : -sr; }
    if constexpr (L::ef(J, 1) != 0) { Pu[1] += L::ef(J, 1) > 0 ? sp : -sp; Ru[1] += L::ef(J, 1) > 0 ? sr : -sr; }
    if constexpr (L::ef(J, 2) != 0) { Pu[2] += L::ef(J, 2) > 0 ? sp : -sp; Ru[2] += L::ef(J, 2) > 0 ? sr : -sr; }
  });
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    Pu[a] = rho * (Pu[a] - R(3) * up[a] * P0);
    Ru[a] = rho * (Ru[a] - R(3) * u[a] * R0);
  }

  R St0 = R(0), St1[3] = {R(0), R(0), R(0)};
  LBGPU_FOR(J, 0, L::MT, {
    const R tw = R(L::wt(J)) * vg[J * VS];
    St0 += tw;
    if constexpr (L::et(J, 0) != 0) St1[0] += L::et(J, 0) > 0 ? tw : -tw;
    if constexpr (L::et(J, 1) != 0) St1[1] += L::et(J, 1) > 0 ? tw : -tw;
    if constexpr (L::et(J, 2) != 0) St1[2] += L::et(J, 2) > 0 ? tw : -tw;
  });
  const R om = R(omt);
  const R sigma = St0 + R(3) * (up[0] * St1[0] + up[1] * St1[1] + up[2] * St1[2]);
  const R s3 = R(3) * om * T;
  R c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) c[a] = G * (Pu[a] + s3 * St1[a]) - Ru[a];
  const R s0 = Pr - Rr - (c[0] * u[0] + c[1] * u[1] + c[2] * u[2]) * inv;
  const R ci[3] = {c[0] * inv, c[1] * inv, c[2] * inv};
  LBGPU_FOR(K_, 0, L::MF, { outf[K_] = rj.template operator()<K_>() + s0 + edotp<L, R, K_>(ci); });
  const R om1 = R(1) - om, oms = om * sigma;
#pragma unroll
  for (int k = 0; k < L::MT; ++k) outg[k] = om1 * vg[k * VS] + oms;
}
template <class L, class R, int CK, int VS = 1>
__device__ __forceinline__ bool fast_vjp_m(const Model& M, PowPair pp, double omt, R rho,
                                           const R* jv, R T, const R* vf, const R* vg, R* outf,
                                           R* outg) {
  if (!(rho > R(0))) return false;
  fast_vjp_mi<L, R, CK, VS>(M, pp, omt, rho, R(1) / rho, jv, T, vf, vg, outf, outg);
  return true;
}

template <class L, class R, int CK>
__device__ __forceinline__ bool fast_vjp(const Model& M, PowPair pp, double omt, const R* f,
                                         const R* g, const R* vf, const R* vg, R* outf, R* outg) {
  R rho, jv[3];
  flow_sums<L, R>(f, rho, jv);
  R T = R(0);
#pragma unroll
  for (int k = 0; k < L::MT; ++k) T += g[k];
  return fast_vjp_m<L, R, CK>(M, pp, omt, rho, jv, T, vf, vg, outf, outg);
}

// node_partial (objective.cpp:34-62) from the node's moments.
template <class L, class R>
__device__ __forceinline__ bool fast_partial_m(const Model& M, R rho, const R* jv, R T, R* out) {
  if (!(rho > R(0))) return false;
  const R inv = R(1) / rho;
  const int a = M.flux_axis;
  const R ua = (a == 0 ? jv[0] : (a == 1 ? jv[1] : jv[2])) * inv;
  const R sgn = R(M.flux_sign);
  const R un = sgn * ua;
  const R du = (M.obj_kind == 0 ? (R(1) - T * T) * sgn : T * sgn) * inv;
  LBGPU_FOR(K_, 0, L::MF, {
    const int ea = a == 0 ? L::ef(K_, 0) : (a == 1 ? L::ef(K_, 1) : L::ef(K_, 2));
    out[K_] += du * (R(ea) - ua);
  });
  const R dT = M.obj_kind == 0 ? R(-2) * T * un : un;
#pragma unroll
  for (int k = 0; k < L::MT; ++k) out[L::MF + k] += dT;
  return true;
}

// Fast pressure-face adjoint: v_out = J_recon^T (J_int(frec, grec)^T v), the
// chain rule through collide_node's wet-node treatment (collision.cpp:248-292)
// with the Zou-He / thermal reconstruction reversed by hand. Follows the
// branch the primal value takes at the u_clamp test, like the reference's
// dual sweep (dual.hpp:12-13).
template <class L, class R, int CK>
__device__ __forceinline__ bool fast_face_vjp(const Model& M, PowPair pp, double omt, int tag,
                                              int axis, int sign, double bcT, const R* fin,
                                              const R* vin, R* vout) {
  const R* f = fin;
  const R* g = fin + L::MF;
  R frec[L::MF], grec[L::MT];
  const R rho_t = R(tag == TAG_INLET ? M.rho_in : M.rho_out);
  face_recon<L, R>(M, tag, axis, sign, bcT, fin, rho_t, frec, grec);

  // Scalars of the forward reconstruction.
  R k0 = R(0), km = R(0);
#pragma unroll
  for (int j = 0; j < L::MF; ++j) {
    const int ea = evel_axis(L::ef(j, 0), L::ef(j, 1), L::ef(j, 2), axis);
    if (ea == 0) k0 += f[j];
    else if (ea == -sign) km += f[j];
  }
  const R s = R(sign);
  const R Ksum = k0 + R(2) * km;
  R ua = s * (R(1) - Ksum / rho_t);
  R rho = rho_t;
  const bool clamped = (ua < R(0) ? -ua : ua) > R(M.u_clamp);
  if (clamped) {
    ua = ua > R(0) ? R(M.u_clamp) : R(-M.u_clamp);
    rho = Ksum / (R(1) - s * ua);
  }
  R Tstar = R(bcT), tden = R(1);
  if (tag == TAG_OUTLET) {
    R tnum = R(0);
    tden = R(0);
#pragma unroll
    for (int j = 0; j < L::MT; ++j) {
      const int ea = evel_axis(L::et(j, 0), L::et(j, 1), L::et(j, 2), axis);
      if (ea == sign) continue;
      tnum += g[j];
      tden += R(L::wt(j)) * (R(1) + R(3) * (R(ea) * ua));
    }
    Tstar = tnum / tden;
  }

  R af[L::MF], ag[L::MT];
  if (!fast_vjp<L, R, CK>(M, pp, omt, frec, grec, vin, vin + L::MF, af, ag)) return false;

  R* of = vout;
  R* og = vout + L::MF;
  R afeq[L::MF];
  R anb[3] = {R(0), R(0), R(0)};
#pragma unroll
  for (int j = 0; j < L::MF; ++j) of[j] = R(0), afeq[j] = R(0);
#pragma unroll
  for (int j = 0; j < L::MF; ++j) {
    const int e[3] = {L::ef(j, 0), L::ef(j, 1), L::ef(j, 2)};
    if (e[axis] != sign) {
      of[j] += af[j];
    } else {
      const int o = L::oppf(j);
      of[o] += af[j];
      afeq[j] += af[j];
      afeq[o] -= af[j];
#pragma unroll
      for (int b = 0; b < 3; ++b)
        if (b != axis && e[b]) anb[b] -= af[j] * R(e[b]);
    }
  }
#pragma unroll
  for (int j = 0; j < L::MF; ++j) {
    const int e[3] = {L::ef(j, 0), L::ef(j, 1), L::ef(j, 2)};
    if (e[axis] != 0) continue;
#pragma unroll
    for (int b = 0; b < 3; ++b)
      if (b != axis && e[b]) of[j] += R(0.5 * e[b]) * anb[b];
  }
  R arho = R(0), aua = R(0);
#pragma unroll
  for (int j = 0; j < L::MF; ++j) {
    const R ea = R(evel_axis(L::ef(j, 0), L::ef(j, 1), L::ef(j, 2), axis));
    const R wj = R(L::wf(j));
    const R eu = ea * ua;
    arho += afeq[j] * wj * (R(1) + R(3) * eu + R(4.5) * eu * eu - R(1.5) * ua * ua);
    aua += afeq[j] * wj * rho * (R(3) * ea + R(9) * ea * eu - R(3) * ua);
  }
  R aT = R(0);
#pragma unroll
  for (int j = 0; j < L::MT; ++j) {
    const R ea = R(evel_axis(L::et(j, 0), L::et(j, 1), L::et(j, 2), axis));
    const R tw = R(L::wt(j));
    aT += ag[j] * tw * (R(1) + R(3) * ea * ua);
    aua += ag[j] * tw * Tstar * R(3) * ea;
    og[j] = R(0);
  }
  if (tag == TAG_OUTLET) {
    const R atnum = aT / tden;
    const R atden = -aT * Tstar / tden;
#pragma unroll
    for (int j = 0; j < L::MT; ++j) {
      const int ea = evel_axis(L::et(j, 0), L::et(j, 1), L::et(j, 2), axis);
      if (ea == sign) continue;
      og[j] += atnum;
      aua += atden * R(L::wt(j)) * R(3) * R(ea);
    }
  }
  const R aK = clamped ? arho / (R(1) - s * ua) : -aua * s / rho_t;
#pragma unroll
  for (int j = 0; j < L::MF; ++j) {
    const int ea = evel_axis(L::ef(j, 0), L::ef(j, 1), L::ef(j, 2), axis);
    if (ea == 0) of[j] += aK;
    else if (ea == -sign) of[j] += R(2) * aK;
  }
  return true;
}


// ---------------------------------------------------------------------
// In-place pressure-face treatment for the fast bulk kernels. The wet-node
// collision of a Zou-He face is interior_collide applied to a reconstructed
// input (collision.cpp:248-292); the face lane rebuilds its gathered
// populations in place (compile-time normal axis AX and sign SG) and then
// shares the interior collision / interior VJP with the other lanes of its
// warp. The adjoint undoes the reconstruction by hand afterwards
// (v <- J_recon^T v), again in place, from a handful of scalars.
// The divisions of the reconstruction are reciprocals of per-model constants
// (1/rho_target, 1/(1 -+ u_clamp), precomputed on the host) and of the one
// runtime denominator tden, taken once.
template <class R>
struct FaceState {
  R ua, rho, Tstar, itden;  // itden = 1 / tden (1 at an inlet)
  bool clamped;
};
template <class R>
__device__ __forceinline__ R face_inv_rho_t(const Model& M, bool inlet) {
  return R(inlet ? M.inv_rho_in : M.inv_rho_out);
}
// 1 / (1 - s ua) for a clamped face (ua = +-u_clamp)
template <class R>
__device__ __forceinline__ R face_inv_clamp(const Model& M, R sua) {
  return R(sua > R(0) ? M.inv_1m_uc : M.inv_1p_uc);
}

template <class L, class R, int AX, int SG>
__device__ __forceinline__ FaceState<R> face_forward(const Model& M, bool inlet, double bcT,
                                                     R* f) {
  FaceState<R> fs;
  R k0 = R(0), km = R(0);
  LBGPU_FOR(J, 0, L::MF, {
    constexpr int ea = L::ef(J, AX);
    if constexpr (ea == 0) k0 += f[J];
    if constexpr (ea == -SG) km += f[J];
  });
  const R s = R(SG);
  const R Ksum = k0 + R(2) * km;
  R ua = s * (R(1) - Ksum * face_inv_rho_t<R>(M, inlet));
  R rho = R(inlet ? M.rho_in : M.rho_out);
  fs.clamped = (ua < R(0) ? -ua : ua) > R(M.u_clamp);
  if (fs.clamped) {
    ua = ua > R(0) ? R(M.u_clamp) : R(-M.u_clamp);
    rho = Ksum * face_inv_clamp<R>(M, s * ua);
  }
  fs.ua = ua, fs.rho = rho;
  // tangential momentum of the slots parallel to the face (collision.cpp:160-165)
  R nb[3] = {R(0), R(0), R(0)};
  LBGPU_FOR(J, 0, L::MF, {
    if constexpr (L::ef(J, AX) == 0) {
#pragma unroll
      for (int b = 0; b < 3; ++b)
        if (b != AX && L::ef(J, b) != 0) nb[b] += R(0.5 * L::ef(J, b)) * f[J];
    }
  });
  const R c0 = R(1) - R(1.5) * ua * ua;
  LBGPU_FOR(J, 0, L::MF, {
    if constexpr (L::ef(J, AX) == SG) {
      constexpr int o = L::oppf(J);
      const R eu = R(SG) * ua;
      const R wr = R(L::wf(J)) * rho;
      const R dfe = wr * (R(6) * eu);  // feq_j - feq_o: the even terms cancel
      R corr = R(0);
#pragma unroll
      for (int b = 0; b < 3; ++b)
        if (b != AX && L::ef(J, b) != 0) corr += R(L::ef(J, b)) * nb[b];
      f[J] = f[o] + dfe - corr;
    }
  });
  (void)c0;
  // thermal: imposed inlet temperature, or the outflow rebuild (collision.cpp:277-288)
  R* g = f + L::MF;
  if (inlet) {
    fs.Tstar = R(bcT);
    fs.itden = R(1);
  } else {
    R tnum = R(0), tden = R(0);
    LBGPU_FOR(J, 0, L::MT, {
      constexpr int ea = L::et(J, AX);
      if constexpr (ea != SG) {
        tnum += g[J];
        tden += R(L::wt(J)) * (R(1) + R(3) * (R(ea) * ua));
      }
    });
    fs.itden = R(1) / tden;
    fs.Tstar = tnum * fs.itden;
  }
  LBGPU_FOR(J, 0, L::MT, {
    constexpr int ea = L::et(J, AX);
    g[J] = R(L::wt(J)) * fs.Tstar * (R(1) + R(3) * (R(ea) * ua));
  });
  return fs;
}

// v <- J_recon^T v for the reconstruction above (the branch the primal value
// took at the u_clamp test, as the reference's dual sweep does).
template <class L, class R, int AX, int SG>
__device__ __forceinline__ void face_reverse(const Model& M, bool inlet, const FaceState<R>& fs,
                                             R* v) {
  const R ua = fs.ua, rho = fs.rho, s = R(SG);
  R arho = R(0), aua = R(0), anb[3] = {R(0), R(0), R(0)};
  LBGPU_FOR(J, 0, L::MF, {
    if constexpr (L::ef(J, AX) == SG) {
      constexpr int o = L::oppf(J);
      const R aj = v[J];
      v[o] += aj;
      v[J] = R(0);
      // feq_j - feq_o = w rho 6 e ua  (e = SG): d/drho and d/dua
      const R w = R(L::wf(J));
      arho += aj * (w * R(6) * s * ua);
      aua += aj * (w * rho * R(6) * s);
#pragma unroll
      for (int b = 0; b < 3; ++b)
        if (b != AX && L::ef(J, b) != 0) anb[b] -= aj * R(L::ef(J, b));
    }
  });
  LBGPU_FOR(J, 0, L::MF, {
    if constexpr (L::ef(J, AX) == 0) {
#pragma unroll
      for (int b = 0; b < 3; ++b)
        if (b != AX && L::ef(J, b) != 0) v[J] += R(0.5 * L::ef(J, b)) * anb[b];
    }
  });
  R* vg = v + L::MF;
  R aT = R(0);
  LBGPU_FOR(J, 0, L::MT, {
    constexpr int ea = L::et(J, AX);
    const R tw = R(L::wt(J));
    aT += vg[J] * tw * (R(1) + R(3) * (R(ea) * ua));
    if constexpr (ea != 0) aua += vg[J] * tw * fs.Tstar * R(3 * ea);
  });
  if (inlet) {
#pragma unroll
    for (int j = 0; j < L::MT; ++j) vg[j] = R(0);
  } else {
    const R atnum = aT * fs.itden;
    const R atden = -atnum * fs.Tstar;
    LBGPU_FOR(J, 0, L::MT, {
      constexpr int ea = L::et(J, AX);
      if constexpr (ea != SG) {
        vg[J] = atnum;
        if constexpr (ea != 0) aua += atden * R(L::wt(J)) * R(3 * ea);
      } else {
        vg[J] = R(0);
      }
    });
  }
  const R aK = fs.clamped ? arho * face_inv_clamp<R>(M, s * ua)
                          : -aua * s * face_inv_rho_t<R>(M, inlet);
  LBGPU_FOR(J, 0, L::MF, {
    constexpr int ea = L::ef(J, AX);
    if constexpr (ea == 0) v[J] += aK;
    if constexpr (ea == -SG) v[J] += R(2) * aK;
  });
}

// Runtime (axis, sign) -> compile-time dispatch; 2D lattices have no z faces.
template <class L, class F>
__device__ __forceinline__ void face_dispatch(uint8_t code, F&& fn) {
  const int ax = code_axis(code);
  const bool neg = code & CODE_NEG;
  if (ax == 0) {
    if (neg) fn.template operator()<0, -1>(); else fn.template operator()<0, 1>();
  } else if (ax == 1) {
    if (neg) fn.template operator()<1, -1>(); else fn.template operator()<1, 1>();
  } else if constexpr (L::DIM == 3) {
    if (neg) fn.template operator()<2, -1>(); else fn.template operator()<2, 1>();
  }
}

}  // namespace detail
using detail::halo_slot;
using detail::kHaloPlanes;
using detail::FM_DB;
using detail::FM_O;
using detail::FM_E;

namespace detail {

__device__ __forceinline__ void idx_xyz(const Geom& g, long long idx, int& x, int& y, int& z) {
  x = int(idx % g.nx);
  y = int((idx / g.nx) % g.ny);
  z = int(idx / ((long long)g.nx * g.ny));
}

__device__ __forceinline__ bool is_face(int tag) { return tag == TAG_INLET || tag == TAG_OUTLET; }

// Store one node's M outputs and fold |new - old| into the thread's max.
template <class L, class R, bool RESID>
__device__ __forceinline__ void store_node(const R* __restrict__ src, R* __restrict__ dst,
                                           long long N, long long idx, const R* in,
                                           const R* out, unsigned long long& rmax,
                                           bool in_valid = true) {
  LBGPU_FOR(P, 0, L::M, { *pop(dst, N, P, int(idx)) = out[P]; });
  if constexpr (RESID) {
    LBGPU_FOR(P, 0, L::M, {
      constexpr bool rest = cvel<L>(P, 0) == 0 && cvel<L>(P, 1) == 0 && cvel<L>(P, 2) == 0;
      const R old = (rest && in_valid) ? in[P] : __ldg(pop(src, N, P, int(idx)));
      const unsigned long long d = absdiff_bits(double(out[P]), double(old));
      rmax = d > rmax ? d : rmax;
    });
  }
}

// collide_node (collision.cpp:219-294) for one gathered node.
template <class L, class R, int CK, bool FACES>
__device__ __forceinline__ bool primal_node(const Launch& a, long long idx, uint8_t code,
                                            R* f, R* out) {
  const int tag = code & TAG_MASK;
  if (tag == TAG_WALL) {
    LBGPU_FOR(P, 0, L::M, { out[P] = f[copp<L>(P)]; });
    return true;
  }
  if (tag == TAG_HEATER) {
    LBGPU_FOR(P, 0, L::MF, { out[P] = f[L::oppf(P)]; });
    const R T = R(a.t.bcT[idx]);
#pragma unroll
    for (int j = 0; j < L::MT; ++j) out[L::MF + j] = R(L::wt(j)) * T * (R(1) + R(3) * R(0));
    return true;
  }
  const double w = (code & CODE_HAS_W) ? a.t.w[idx] : 1.0;
  const PowPair pp = node_pp<LBGPU_EXACT != 0>(a.M, a.t, idx, code, w);
#if LBGPU_EXACT
  return collide_node<L, R>(a.M, pp, tag, code_axis(code), code_sign(code), a.t.bcT[idx], f,
                            R(w), R(a.M.rho_in), out);
#else
  const double omt = node_omt<R>(a.M, a.t, code, w);
  if (FACES && is_face(tag)) {  // rebuild the face lane's inputs in place, then collide
    const bool inlet = tag == TAG_INLET;
    const double bcT = a.t.bcT[idx];
    face_dispatch<L>(code, [&]<int AX, int SG>() { face_forward<L, R, AX, SG>(a.M, inlet, bcT, f); });
  }
  return fast_collide<L, R, CK>(a.M, pp, omt, f, out);
#endif
}

// adjoint_collide_node (adjoint.cpp:156-204) for one node whose full base
// state is at hand (bit-exact build, dual kernel, pressure faces).
template <class L, class R, int CK, int AK>
__device__ __forceinline__ bool adjoint_node_full(const Launch& a, long long idx, uint8_t code,
                                                  const R* fin, const R* vin, R* vout) {
  const int tag = code & TAG_MASK;
  bool ok = true;
  if (AK == 0 && tag == TAG_WALL) {
    LBGPU_FOR(P, 0, L::M, { vout[P] = vin[copp<L>(P)]; });
  } else if (AK == 0 && tag == TAG_HEATER) {
    LBGPU_FOR(P, 0, L::MF, { vout[P] = vin[L::oppf(P)]; });
#pragma unroll
    for (int j = 0; j < L::MT; ++j) vout[L::MF + j] = R(0);
  } else {
    const double w = (code & CODE_HAS_W) ? a.t.w[idx] : 1.0;
    const PowPair pp = node_pp<LBGPU_EXACT != 0>(a.M, a.t, idx, code, w);
    if (AK == 1 || (LBGPU_EXACT && tag != TAG_INTERIOR)) {
      ok = vjp_dual<L, R>(a.M, pp, tag, code_axis(code), code_sign(code), a.t.bcT[idx], fin, R(w),
                          vin, vout);
    } else {
#if LBGPU_EXACT
      ok = interior_vjp<L, R>(a.M, pp, fin, fin + L::MF, R(w), vin, vin + L::MF, vout,
                              vout + L::MF);
#else
      const double omt = node_omt<R>(a.M, a.t, code, w);
      if (tag == TAG_INTERIOR)
        ok = fast_vjp<L, R, CK>(a.M, pp, omt, fin, fin + L::MF, vin, vin + L::MF, vout,
                                vout + L::MF);
      else
        ok = fast_face_vjp<L, R, CK>(a.M, pp, omt, tag, code_axis(code), code_sign(code),
                                     a.t.bcT[idx], fin, vin, vout);
#endif
    }
  }
  if (a.M.obj_on && (code & CODE_SUPPORT)) {
    R b[L::M];
    if (node_partial<L, R>(a.M, fin, b)) {
#pragma unroll
      for (int p = 0; p < L::M; ++p) vout[p] += b[p];
    } else {
      ok = false;
    }
  }
  return ok;
}

}  // namespace detail

// Take a design-box node's uploaded value: poll its entry of the upload
// buffer until the copy engine has replaced the sentinel, then re-arm it.
// Relaxed loads (L2, no fence, no block barrier: the node's gather stays in
// flight); the sweep runs in z order behind the upload, so the first load
// almost always passes. Bounded (0.5 s of wall time): a value that never lands
// is reported (LBGPU_E_NUMERIC at the call), never a hang.
__device__ __forceinline__ double gate_take(const Gate& gt, long long o) {
  unsigned long long* p = reinterpret_cast<unsigned long long*>(gt.wd + o);
  auto load = [p] {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
  };
  unsigned long long v = load();
  if (v == kGateEmpty) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while ((v = load()) == kGateEmpty) {
      __nanosleep(256);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 500000000ull) {
        atomicExch(gt.err, 1u);
        break;
      }
    }
  }
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(kGateEmpty) : "memory");
  return __longlong_as_double((long long)v);
}

// ====================================================================
// Sweep kernels. One thread per node, x fastest: grid (ceil(owned/BX), ny, nz).

// Primal sweep (primal_step, collision.cpp:308-363, in pull form) with the
// node dispatch of collide_node (collision.cpp:219-294), the rho <= 0 flag
// (collision.hpp:103) and, when RESID, the fused step_residual. Pressure-face
// lanes rebuild their inputs in place (face_forward) and share the interior
// collision with the rest of the warp.
// FM: the field's addressing mode (FM_DB: src -> dst; FM_O / FM_E: in place,
// src == dst, no residual). UPD: first the previous one-shot iteration's
// design update at an interior design node (a.upd: the gradient of a.upd.v
// against the f gathered here -- the base that iteration's adjoint used --
// then the composite ascent step), exactly k_gradient<UPDATE>'s arithmetic,
// so the primal collides with the new w it has just written.
// GATED (lbgpu_primal_step_with_design, box-shaped design): a design-box
// node's w is the just-uploaded value (gate_take, once its gather is in
// flight), written to a.gate.w_out == a.t.w, which primal_node reads back.
template <class L, class R, int CK, bool RESID, int FM = FM_DB, bool UPD = false, bool GATED = false>
__device__ __forceinline__ void primal_body(const Launch& a, const R* src, R* dst, int x, int y,
                                            int z, unsigned long long& rmax) {
  using namespace detail;
  static_assert(FM == FM_DB || !RESID, "in-place sweeps keep no old state for the residual");
  const Geom& g = a.g;
  const long long idx = x + (long long)g.nx * (y + (long long)g.ny * z);
  const uint8_t code = a.t.code[idx];
  const Nbr nb = make_nbr(g, x, y, z);
  R f[L::M], out[L::M];
  if constexpr (UPD) {
    // v of this node in flight (shared memory) while f is gathered
    __shared__ R vsm[L::M * 128];
    R* my = vsm + threadIdx.x;
    const bool dn = (code & (TAG_MASK | CODE_AXIS_BITS)) == (TAG_INTERIOR | CODE_DESIGN_INT);
    if (dn) gather_async<L, R, +1>(static_cast<const R*>(a.upd.v), g.N, nb, my, 128);
    gather<L, R, -1>(src, g.N, nb, f);
    if (dn) {
      cp_async_wait_all();
      const double w = a.t.w[idx];
      const PowPair pp = node_pp<LBGPU_EXACT != 0>(a.M, a.t, idx, code | CODE_HAS_W, w);
      double gv = 0.0;
      if (!design_gradient<L, R, 128>(a.M, pp, f, f + L::MF, R(w), my, my + L::MF * 128, gv))
        atomicMin(a.fl.bad, (a.fl.step_key | (unsigned long long)gflat(g, x, y, z)));
      double comp = gv;
      if (a.upd.lambda != 0.0) comp -= a.upd.lambda * (1.0 - 2.0 * w);
      double wn = w + a.upd.zeta * comp;
      wn = wn < 0.0 ? 0.0 : (1.0 < wn ? 1.0 : wn);
      a.upd.w[idx] = wn;  // primal_node reads it back below (same thread)
    }
  } else if constexpr (FM == FM_DB) {
    gather<L, R, -1>(src, g.N, nb, f);
    if constexpr (GATED) {
      const Gate& gt = a.gate;
      if (x >= gt.bx0 && x < gt.bx1 && y >= gt.by0 && y < gt.by1 && z >= gt.bz0 && z < gt.bz1) {
        const long long o = (long long)(x - gt.bx0) +
                            (long long)(gt.bx1 - gt.bx0) *
                                ((y - gt.by0) + (long long)(gt.by1 - gt.by0) * (z - gt.bz0));
        gt.w_out[idx] = gate_take(gt, o);
      }
    }
  } else {
    gather_m<L, R, -1, FM>(src, g.N, idx, nb, f);
  }
  if (!primal_node<L, R, CK, true>(a, idx, code, f, out))
    atomicMin(a.fl.bad, (a.fl.step_key | (unsigned long long)gflat(g, x, y, z)));
  if constexpr (FM == FM_DB) {
    store_node<L, R, RESID>(src, dst, g.N, idx, f, out, rmax, !is_face(code & TAG_MASK));
    push_halo<L, R, -1>(a, x, y, z, out);
  } else {
    store_aa<L, R, -1, FM>(dst, g.N, idx, nb, out);
  }
}

// Plain bounds: ptxas picks 64 regs (FP32) / 96-122 (FP64), no spills. Forcing
// more blocks spills (FP32 C3 primal GB/s: 64 regs 5748, 48 regs 5480, 40
// regs 4036); (128, 1) lets it take 106 regs (4827).
template <class L, class R, int CK, bool RESID, bool UPD = false, bool GATED = false>
__global__ void __launch_bounds__(128) k_primal(Launch a, const R* __restrict__ src,
                                                R* __restrict__ dst) {
  const int x = a.g.x0 + blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long rmax = 0;
  if (x < a.g.x1)
    primal_body<L, R, CK, RESID, FM_DB, UPD, GATED>(a, src, dst, x, blockIdx.y, a.g.z0 + blockIdx.z, rmax);
  if constexpr (RESID) detail::block_max_bits(rmax, a.fl.resid);
}

// In-place primal sweep (AA streaming, fast build) from layout FM over the
// owned columns of the 3-D grid.
// Register bound of the in-place primal (FP64). Before store_aa rematerialised
// the shifted store addresses (LBGPU_AA_REMAT) the sweep from E kept them
// live across the collision (182 registers unbounded; C3 GB/s at 1/2/3/4
// blocks per SM 5,543 / 5,535 / 5,922 / 5,648, 4 spilling 248 B). With it,
// 4 blocks fit without spill: 6,408 against 6,233 at 3.
#ifndef LBGPU_AA_PRIMAL_MINB
#define LBGPU_AA_PRIMAL_MINB 4
#endif
// FP32, blocks per SM (C3 GB/s) before LBGPU_AA_REMAT, 1/4/6/8: 5,276 / 5,326 /
// 5,036 / 4,690; with it, 4/6/8: 5,473 / 5,646 / 5,844.
#ifndef LBGPU_AA_PRIMAL_MINB32
#define LBGPU_AA_PRIMAL_MINB32 8
#endif
template <class L, class R, int CK, int FM>
__global__ void __launch_bounds__(128, sizeof(R) == 8 ? LBGPU_AA_PRIMAL_MINB : LBGPU_AA_PRIMAL_MINB32)
    k_primal_aa(Launch a, R* A) {
  unsigned long long rmax = 0;
  const int x = a.g.x0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (x < a.g.x1) primal_body<L, R, CK, false, FM>(a, A, A, x, blockIdx.y, a.g.z0 + blockIdx.z, rmax);
}

// Adjoint sweep (adjoint_step, adjoint.cpp:206-254, in pull form): gathers v
// against the links and the frozen base f along them, applies
// adjoint_collide_node (adjoint.cpp:156-204) and stores the post-collision
// adjoint. AK = 0 analytic kernel, 1 dual sweep (AdjointKernel, adjoint.hpp:14-18).
// Fast build: the gathered base is reduced to (rho, j, T) before the adjoint
// populations are loaded (the interior VJP reads f only through them,
// adjoint.cpp:59, :95); face lanes rebuild / un-build in place. SPLIT leaves
// the rare side-list nodes (synthetic-objective support, support nodes on a
// face) to k_adjoint_side.
// BM / VM: addressing modes of the base f and of v (in-place v: src == dst).
// GRAD (FP64 split sweep of a double-buffered field): at an interior design
// node, also k_gradient's term of this sweep's own inputs -- the base f in
// registers, v staged in shared memory, the same design_gradient call -- added
// to a.upd.gacc[node]: the unsteady adjoint's back step then needs no
// separate gradient pass over the design nodes.
template <class L, class R, int CK, int AK, bool RESID, bool SPLIT, bool MOM, int BM = FM_DB,
          int VM = FM_DB, bool GRAD = false>
__device__ __forceinline__ void adjoint_body(const Launch& a, const R* __restrict__ base,
                                             const R* src, R* dst, const R* __restrict__ mom,
                                             int x, int y, int z, unsigned long long& rmax) {
  using namespace detail;
  constexpr bool kInSmem = !LBGPU_EXACT && AK == 0 && SPLIT && LBGPU_ADJ_STAGE && sizeof(R) == 8 &&
                           LBGPU_ADJ_VSMEM;
  const Geom& g = a.g;
  const long long N = g.N;
  const long long idx = x + (long long)g.nx * (y + (long long)g.ny * z);
  const uint8_t code = a.t.code[idx];
  const int tag = code & TAG_MASK;
  const bool face = is_face(tag);
  const bool side = (code & CODE_SUPPORT) && (a.M.obj_kind == 2 || face);
  if (!(SPLIT && side)) {
    const Nbr nb = make_nbr(g, x, y, z);
    R vin[L::M], vout[L::M];
    bool ok = true;
    if constexpr (LBGPU_EXACT || AK == 1 || !SPLIT) {
      static_assert(BM == FM_DB && VM == FM_DB, "in-place streaming: product split path only");
      R fin[L::M];
      gather<L, R, -1>(base, N, nb, fin);
      gather<L, R, +1>(src, N, nb, vin);
      ok = adjoint_node_full<L, R, CK, AK>(a, idx, code, fin, vin, vout);
    } else {
      // FP64: v's gather goes out first, through shared memory, so it overlaps
      // the base gather and the moment sums instead of following them
      // (C3 +0.5% gathering, +1.7% frozen base; FP32 measured slower: off)
      constexpr bool kStage = LBGPU_ADJ_STAGE && (sizeof(R) == 8 || LBGPU_ADJ_STAGE32);
      __shared__ R vsm[kStage ? L::M * 128 : 1];
      R* my = vsm + (kStage ? threadIdx.x : 0);
      if constexpr (kStage) {
        if constexpr (VM == FM_DB) gather_async<L, R, +1>(src, N, nb, my, 128);
        else gather_async_m<L, R, +1, VM>(src, N, idx, nb, my, 128);
      }
      // FP32 frozen base: v's gather in registers before the moments are read
      // (C3 MLUPS 23,369 -> 24,843; gathering bases spill instead: 5,682 ->
      // 3,684 GB/s at 8 blocks per SM, 4,916 at 5)
      constexpr bool kEarly = !kStage && sizeof(R) == 4 && MOM;
      if constexpr (kEarly) {
        if constexpr (VM == FM_DB) gather<L, R, +1>(src, N, nb, vin);
        else gather_m<L, R, +1, VM>(src, N, idx, nb, vin);
      }
      R rho = R(1), jv[3] = {R(0), R(0), R(0)}, T = R(0);
      FaceState<R> fs{};
      const bool need = !(tag == TAG_WALL || tag == TAG_HEATER) || (code & CODE_SUPPORT);
      if (need && MOM) {  // frozen base: its moments, cached (k_base_moments)
        rho = mom[idx];
        jv[0] = mom[N + idx];
        jv[1] = mom[2 * N + idx];
        if constexpr (L::DIM == 3) jv[2] = mom[3 * N + idx];
        T = mom[(L::DIM + 1) * N + idx];
        if (face) {  // and the face reconstruction's scalars
          const R* fp = mom + (L::DIM + 2) * N + idx;
          fs.ua = fp[0], fs.rho = fp[N], fs.Tstar = fp[2 * N], fs.itden = fp[3 * N];
          fs.clamped = fp[4 * N] != R(0);
        }
      } else if (need) {
        R fin[L::M];
        if constexpr (BM == FM_DB) gather<L, R, -1>(base, N, nb, fin);
        else gather_m<L, R, -1, BM>(base, N, idx, nb, fin);
        if (face) {
          const bool inlet = tag == TAG_INLET;
          const double bcT = a.t.bcT[idx];
          face_dispatch<L>(code, [&]<int AX, int SG>() {
            fs = face_forward<L, R, AX, SG>(a.M, inlet, bcT, fin);
          });
        }
        flow_sums<L, R>(fin, rho, jv);
#pragma unroll
        for (int k = 0; k < L::MT; ++k) T += fin[L::MF + k];
        if constexpr (GRAD && kStage) {
          if ((code & (TAG_MASK | CODE_AXIS_BITS)) == (TAG_INTERIOR | CODE_DESIGN_INT)) {
            cp_async_wait_all();
            const double w = a.t.w[idx];
            const PowPair pp = node_pp<false>(a.M, a.t, idx, code | CODE_HAS_W, w);
            double gv = 0.0;
            if (!design_gradient<L, R, 128>(a.M, pp, fin, fin + L::MF, R(w), my, my + L::MF * 128, gv))
              ok = false;
            a.upd.gacc[idx] = a.upd.gacc[idx] + gv;
          }
        }
      }
      // kInSmem: the staged v is read in place by the VJP (no register copy)
      constexpr int VS = kInSmem ? 128 : 1;
      const R* vv = kInSmem ? my : vin;
      if constexpr (kStage) {
        cp_async_wait_all();
        if constexpr (!kInSmem) LBGPU_FOR(P, 0, L::M, { vin[P] = my[P * 128]; });
      } else if constexpr (kEarly) {
      } else if constexpr (VM == FM_DB && LBGPU_ADJ_REMAT32) {
        gather<L, R, +1>(src, N, opaque(nb), vin);  // offsets re-formed after the moments
      } else if constexpr (VM == FM_DB) {
        gather<L, R, +1>(src, N, nb, vin);
      } else {
        gather_m<L, R, +1, VM>(src, N, idx, nb, vin);
      }
      if (tag == TAG_WALL) {
        LBGPU_FOR(P, 0, L::M, { vout[P] = vv[copp<L>(P) * VS]; });
      } else if (tag == TAG_HEATER) {
        LBGPU_FOR(P, 0, L::MF, { vout[P] = vv[L::oppf(P) * VS]; });
#pragma unroll
        for (int j = 0; j < L::MT; ++j) vout[L::MF + j] = R(0);
      } else {
        const double w = (code & CODE_HAS_W) ? a.t.w[idx] : 1.0;
        const PowPair pp = node_pp<false>(a.M, a.t, idx, code, w);
        const double omt = node_omt<R>(a.M, a.t, code, w);
        ok = fast_vjp_m<L, R, CK, VS>(a.M, pp, omt, rho, jv, T, vv, vv + L::MF * VS, vout,
                                      vout + L::MF);
        if (face) {
          const bool inlet = tag == TAG_INLET;
          face_dispatch<L>(code, [&]<int AX, int SG>() {
            face_reverse<L, R, AX, SG>(a.M, inlet, fs, vout);
          });
        }
      }
      if (a.M.obj_on && (code & CODE_SUPPORT)) ok = fast_partial_m<L, R>(a.M, rho, jv, T, vout) && ok;
    }
    if (!ok) atomicMin(a.fl.bad, (a.fl.step_key | (unsigned long long)gflat(g, x, y, z)));
    if constexpr (VM == FM_DB) {
      store_node<L, R, RESID>(src, dst, N, idx, vin, vout, rmax, !kInSmem);
      push_halo<L, R, +1>(a, x, y, z, vout);
    } else {
      static_assert(!RESID, "in-place sweeps keep no old state for the residual");
      store_aa<L, R, +1, VM>(dst, N, idx, nb, vout);
    }
  }
}

// Moments of a frozen adjoint base (rho, j, T per node: planes 0..DIM+1),
// computed once per steady adjoint solve: the moment-form VJP reads the base
// only through them (adjoint.cpp:59, :95), so each sweep then reads
// (DIM + 2) reals per node instead of gathering all M populations. Same
// arithmetic as the in-sweep path, so the adjoint states are bitwise equal.
// Pressure-face nodes store the moments of their reconstructed populations
// and the five scalars face_reverse needs (planes DIM+2 .. DIM+6).
template <class L, class R, int BM = FM_DB>
__global__ void __launch_bounds__(128) k_base_moments(Launch a, const R* __restrict__ base,
                                                      R* __restrict__ mom) {
  using namespace detail;
  const int x = a.g.x0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= a.g.x1) return;
  const Geom& g = a.g;
  const int y = blockIdx.y, z = blockIdx.z;
  const long long N = g.N;
  const long long idx = x + (long long)g.nx * (y + (long long)g.ny * z);
  const uint8_t code = a.t.code[idx];
  const int tag = code & TAG_MASK;
  const bool need = !(tag == TAG_WALL || tag == TAG_HEATER) || (code & CODE_SUPPORT);
  if (!need) return;
  const Nbr nb = make_nbr(g, x, y, z);
  R fin[L::M];
  if constexpr (BM == FM_DB) gather<L, R, -1>(base, N, nb, fin);
  else gather_m<L, R, -1, BM>(base, N, idx, nb, fin);
  if (is_face(tag)) {
    FaceState<R> fs;
    const bool inlet = tag == TAG_INLET;
    const double bcT = a.t.bcT[idx];
    face_dispatch<L>(code, [&]<int AX, int SG>() {
      fs = face_forward<L, R, AX, SG>(a.M, inlet, bcT, fin);
    });
    R* fp = mom + (L::DIM + 2) * N + idx;
    fp[0] = fs.ua, fp[N] = fs.rho, fp[2 * N] = fs.Tstar, fp[3 * N] = fs.itden;
    fp[4 * N] = fs.clamped ? R(1) : R(0);
  }
  R rho, jv[3], T = R(0);
  flow_sums<L, R>(fin, rho, jv);
#pragma unroll
  for (int k = 0; k < L::MT; ++k) T += fin[L::MF + k];
  mom[idx] = rho;
  mom[N + idx] = jv[0];
  mom[2 * N + idx] = jv[1];
  if constexpr (L::DIM == 3) mom[3 * N + idx] = jv[2];
  mom[(L::DIM + 1) * N + idx] = T;
}

// Resident blocks per SM the split adjoint is compiled for (register cap
// 65536 / (128 * minb)). Measured on B200, C3 adjoint GB/s: FP64 minb 4 best
// (3 and 2 lower); FP32 4: 4197, 5: 4702, 6: 4950, 8: 5215 (64 regs, 24 B
// stack — the occupancy is worth the spill).
#ifndef LBGPU_ADJ_MINB
#define LBGPU_ADJ_MINB 4
#endif
#ifndef LBGPU_ADJ_MINB32
#define LBGPU_ADJ_MINB32 8
#endif
// The moment-cache variant (MOM) keeps the same bounds: measured FP64 5/6/8
// blocks 9,941 / 7,775 / 5,746 MLUPS against 10,887 at 4 (126 regs, no spill).
#ifndef LBGPU_ADJ_MINB_MOM
#define LBGPU_ADJ_MINB_MOM LBGPU_ADJ_MINB
#endif
#ifndef LBGPU_ADJ_MINB32_MOM
#define LBGPU_ADJ_MINB32_MOM LBGPU_ADJ_MINB32
#endif
#define LBGPU_ADJ_BOUNDS(SPLIT, R, MOM)                                                 \
  __launch_bounds__(128, !(SPLIT) ? 1                                                  \
                         : (MOM) ? (sizeof(R) == 4 ? LBGPU_ADJ_MINB32_MOM : LBGPU_ADJ_MINB_MOM) \
                                 : (sizeof(R) == 4 ? LBGPU_ADJ_MINB32 : LBGPU_ADJ_MINB))

template <class L, class R, int CK, int AK, bool RESID, bool SPLIT, bool MOM, bool GRAD = false>
__global__ void LBGPU_ADJ_BOUNDS(SPLIT, R, MOM) k_adjoint(Launch a,
                                                                const R* __restrict__ base,
                                                                const R* __restrict__ src,
                                                                R* __restrict__ dst,
                                                                const R* __restrict__ mom) {
  const int x = a.g.x0 + blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long rmax = 0;
  if (x < a.g.x1)
    adjoint_body<L, R, CK, AK, RESID, SPLIT, MOM, FM_DB, FM_DB, GRAD>(a, base, src, dst, mom, x, blockIdx.y,
                                                                      a.g.z0 + blockIdx.z, rmax);
  if constexpr (RESID) detail::block_max_bits(rmax, a.fl.resid);
}

// In-place adjoint sweep (AA streaming, fast build): base f read under BM, v
// updated in place from layout VM.
// In-place adjoint (FP64), C3 GB/s at 2/3/4 blocks per SM without
// LBGPU_AA_REMAT: 4,947 / 5,988 / 5,824 (4 spilled 144-472 B in the sweeps
// from E); with it, 4 blocks: 6,487 against 6,133 at 3 (frozen base 12,335
// against 11,185 MLUPS).
#ifndef LBGPU_AA_ADJ_MINB
#define LBGPU_AA_ADJ_MINB 4
#endif
// FP32, blocks per SM (C3 GB/s) before LBGPU_AA_REMAT, 4/5/6/8: 4,467 / 4,888 /
// 5,088 / 4,702; with it, 6/7/8: 5,362 / 5,579 / 5,713.
#ifndef LBGPU_AA_ADJ_MINB32
#define LBGPU_AA_ADJ_MINB32 8
#endif
template <class L, class R, int CK, int BM, int VM, bool MOM>
__global__ void __launch_bounds__(128, sizeof(R) == 8 ? LBGPU_AA_ADJ_MINB
                                                      : (MOM ? LBGPU_ADJ_MINB32_MOM : LBGPU_AA_ADJ_MINB32))
    k_adjoint_aa(Launch a, const R* __restrict__ base, R* V, const R* __restrict__ mom) {
  unsigned long long rmax = 0;
  const int x = a.g.x0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (x < a.g.x1)
    adjoint_body<L, R, CK, 0, false, true, MOM, BM, VM>(a, base, V, V, mom, x, blockIdx.y,
                                                        a.g.z0 + blockIdx.z, rmax);
}

// Side-list adjoint nodes with the full (reference-form) node update
// (BM / VM: addressing of base and v, as adjoint_body).
template <class L, class R, int CK, bool RESID, int BM = FM_DB, int VM = FM_DB>
__global__ void __launch_bounds__(128) k_adjoint_side(Launch a, const R* __restrict__ base,
                                                      const R* src, R* dst,
                                                      const long long* __restrict__ nodes,
                                                      long long n) {
  using namespace detail;
  const Geom& g = a.g;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  unsigned long long rmax = 0;
  if (i < n) {
    const long long idx = nodes[i];
    int x, y, z;
    idx_xyz(g, idx, x, y, z);
    const Nbr nb = make_nbr(g, x, y, z);
    R fin[L::M], vin[L::M], vout[L::M];
    if constexpr (BM == FM_DB) gather<L, R, -1>(base, g.N, nb, fin);
    else gather_m<L, R, -1, BM>(base, g.N, idx, nb, fin);
    if constexpr (VM == FM_DB) gather<L, R, +1>(src, g.N, nb, vin);
    else gather_m<L, R, +1, VM>(src, g.N, idx, nb, vin);
    if (!adjoint_node_full<L, R, CK, 0>(a, idx, a.t.code[idx], fin, vin, vout))
      atomicMin(a.fl.bad, (a.fl.step_key | (unsigned long long)gflat(g, x, y, z)));
    if constexpr (VM == FM_DB) {
      store_node<L, R, RESID>(src, dst, g.N, idx, vin, vout, rmax);
      push_halo<L, R, +1>(a, x, y, z, vout);
    } else {
      store_aa<L, R, +1, VM>(dst, g.N, idx, nb, vout);
    }
  }
  if constexpr (RESID) block_max_bits(rmax, a.fl.resid);
}

// Block shape of the fused pair sweep: BX nodes along x by BY rows of y
// (one warp per 32 x-nodes). Narrow blocks dilute the pressure-face lanes:
// a block holding a face node waits on that lane's divergent reconstruction,
// so with 128-wide rows every block of a 256-column channel pays for it, with
// 32-wide rows one block in four (measured in DESIGN.md).
// C3 FP64 (B200, MLUPS per pair): 128x1 7,433; 64x1 7,529; 32x1 7,443;
// 32x4 7,689 -- the last equals the face-free periodic box (7,696).
#ifndef LBGPU_PAIR_BX
#define LBGPU_PAIR_BX 32
#endif
#ifndef LBGPU_PAIR_BY
#define LBGPU_PAIR_BY 4
#endif
template <class R>
constexpr int kPairThreads = LBGPU_PAIR_BX * LBGPU_PAIR_BY;

// The post values of node (x, y, z) that stream into the support plane x =
// obj_x, stored at the receiving node's slot of the inbox (Gate): the pull
// of node d reads post_P(d - e_P) with periodic wrap, so node s feeds d = s +
// e_P. k_objective_inbox then reads the plane's populations coalesced instead
// of 26 scattered lines per node.
template <class L, class R>
__device__ __forceinline__ void inbox_store(const Gate& gt, const Geom& g, int x, int y, int z,
                                            const R* out) {
  const int dx = gt.obj_x - x;
  if (dx < -1 || dx > 1) return;
  const long long S = (long long)g.ny * g.nz;
  LBGPU_FOR(P, 0, L::M, {
    constexpr int ex = cvel<L>(P, 0), ey = cvel<L>(P, 1), ez = cvel<L>(P, 2);
    if (ex == dx) {
      int yd = y + ey, zd = z + ez;
      yd = yd < 0 ? g.ny - 1 : (yd >= g.ny ? 0 : yd);
      zd = zd < 0 ? g.nz - 1 : (zd >= g.nz ? 0 : zd);
      gt.inbox[P * S + yd + (long long)g.ny * zd] = double(out[P]);
    }
  });
}

// Fused primal + adjoint pair (product build): adjoint sweep n (base
// f^{n+1}) and primal sweep n+1 read the same gathered f^{n+1}, so one kernel
// gathers it once, takes its moments once (node_sums) and the node's
// switching pair, thermal rate and 1/rho once, collides it (primal_node's
// fast path) and runs the moment-form VJP against it (adjoint_body's split
// path): 4 M s bytes per node for the pair instead of 5 M s. Each half is
// bitwise the stand-alone sweep (same functions, same operands). Side-list
// nodes' adjoint half goes to k_adjoint_side as usual.
// FM / VM: addressing of f and v (in place: fsrc == fdst, vsrc == vdst).
// DUALW: the adjoint half is the previous design's (lbgpu_pair_step_with_design
// defers each call's adjoint sweep into the next call's fused kernel), so its
// node constants come from a.t.w_adj while the primal half uses a.t.w -- or,
// GATED, the just-uploaded design value (a.gate; gate_take waits for it).
template <class L, class R, int CK, bool RESID, int FM = FM_DB, int VM = FM_DB, bool DUALW = false,
          bool GATED = false>
__device__ __forceinline__ void pair_body(const Launch& a, const R* fsrc, R* fdst,
                                          const R* vsrc, R* vdst, int x, int y, int z, int tid,
                                          unsigned long long& rP, unsigned long long& rA) {
  static_assert((FM == FM_DB && VM == FM_DB) || !RESID, "in-place sweeps: no residual");
  using namespace detail;
  const Geom& g = a.g;
  const long long N = g.N;
  const long long idx = x + (long long)g.nx * (y + (long long)g.ny * z);
  const uint8_t code = a.t.code[idx];
  const int tag = code & TAG_MASK;
  const bool face = is_face(tag);
  const bool bb = tag == TAG_WALL || tag == TAG_HEATER;  // bounce-back: no collision
  const bool side = (code & CODE_SUPPORT) && (a.M.obj_kind == 2 || face);
  const Nbr nb = make_nbr(g, x, y, z);
  constexpr bool kStage = LBGPU_ADJ_STAGE && sizeof(R) == 8;
  constexpr int kTB = kPairThreads<R>;
  __shared__ R vsm[kStage ? L::M * kTB : 1];
  R* my = vsm + (kStage ? tid : 0);
  if constexpr (kStage) {
    if constexpr (VM == FM_DB) {
      if (!side) gather_async<L, R, +1>(vsrc, N, nb, my, kTB);
    } else {
      if (!side) gather_async_m<L, R, +1, VM>(vsrc, N, idx, nb, my, kTB);
    }
  }
  // the node's constants, shared by both halves
  double w = 1.0, omt = 0.0;
  PowPair pp{};
  // GATED: a design-box node's w is the just-uploaded value, taken once the
  // node's gather is in flight
  bool gated = false;
  if constexpr (GATED) {
    const Gate& gt = a.gate;
    gated = !bb && x >= gt.bx0 && x < gt.bx1 && y >= gt.by0 && y < gt.by1 && z >= gt.bz0 &&
            z < gt.bz1;
  }
  if (!bb && !gated) {
    w = (code & CODE_HAS_W) ? a.t.w[idx] : 1.0;
    pp = node_pp<false>(a.M, a.t, idx, code, w);
    omt = node_omt<R>(a.M, a.t, code, w);
  }
  R rho, jv[3], T, inv = R(1);
  FaceState<R> fs{};
  bool okP = true, okA = true;
  {
    R f[L::M], out[L::M];
    if constexpr (FM == FM_DB) gather<L, R, -1>(fsrc, N, nb, f);
    else gather_m<L, R, -1, FM>(fsrc, N, idx, nb, f);
    if constexpr (GATED) {
      if (gated) {
        const Gate& gt = a.gate;
        const long long o = (long long)(x - gt.bx0) +
                            (long long)(gt.bx1 - gt.bx0) *
                                ((y - gt.by0) + (long long)(gt.by1 - gt.by0) * (z - gt.bz0));
        w = gate_take(gt, o);
        gt.w_out[idx] = w;
        pp = node_pp<false>(a.M, a.t, idx, code, w);
        omt = node_omt<R>(a.M, a.t, code, w);
      }
    }
    if (tag == TAG_WALL) {
      LBGPU_FOR(P, 0, L::M, { out[P] = f[copp<L>(P)]; });
    } else if (tag == TAG_HEATER) {
      LBGPU_FOR(P, 0, L::MF, { out[P] = f[L::oppf(P)]; });
      const R Th = R(a.t.bcT[idx]);
#pragma unroll
      for (int j = 0; j < L::MT; ++j) out[L::MF + j] = R(L::wt(j)) * Th * (R(1) + R(3) * R(0));
    } else if (face) {
      const bool inlet = tag == TAG_INLET;
      const double bcT = a.t.bcT[idx];
      face_dispatch<L>(code, [&]<int AX, int SG>() {
        fs = face_forward<L, R, AX, SG>(a.M, inlet, bcT, f);
      });
    }
    node_sums<L, R>(f, rho, jv, T);
    if (rho > R(0)) inv = R(1) / rho;
    if (!bb) {
      if (rho > R(0)) fast_collide_mi<L, R, CK>(a.M, pp, omt, f, rho, inv, jv[0], jv[1], jv[2], T, out);
      else okP = false;
    }
    if constexpr (FM == FM_DB) {
      store_node<L, R, RESID>(fsrc, fdst, N, idx, f, out, rP, !face);
      push_halo<L, R, -1>(a, x, y, z, out);
      if constexpr (GATED) {
        if (a.gate.obj_x >= 0) inbox_store<L, R>(a.gate, g, x, y, z, out);
      }
    } else {
      store_aa<L, R, -1, FM>(fdst, N, idx, nb, out);
    }
  }
  if (!side) {
    R vin[L::M], vout[L::M];
    // kInSmem: the VJP reads the staged v in place (no register copy)
    constexpr bool kInSmem = kStage && LBGPU_PAIR_VSMEM;
    constexpr int VS = kInSmem ? kTB : 1;
    const R* vv = kInSmem ? my : vin;
    if constexpr (kStage) {
      cp_async_wait_all();
      if constexpr (!kInSmem) LBGPU_FOR(P, 0, L::M, { vin[P] = my[P * kTB]; });
    } else if constexpr (VM == FM_DB) {
      gather<L, R, +1>(vsrc, N, nb, vin);
    } else {
      gather_m<L, R, +1, VM>(vsrc, N, idx, nb, vin);
    }
    if (tag == TAG_WALL) {
      LBGPU_FOR(P, 0, L::M, { vout[P] = vv[copp<L>(P) * VS]; });
    } else if (tag == TAG_HEATER) {
      LBGPU_FOR(P, 0, L::MF, { vout[P] = vv[L::oppf(P) * VS]; });
#pragma unroll
      for (int j = 0; j < L::MT; ++j) vout[L::MF + j] = R(0);
    } else {
      PowPair ppa = pp;
      double omta = omt;
      if constexpr (DUALW) {
        if (code & CODE_HAS_W) {
          const double wa = a.t.w_adj[idx];
          ppa = node_pp<false>(a.M, a.t, idx, code, wa);
          omta = node_omt<R>(a.M, a.t, code, wa);
        }
      }
      if (rho > R(0))
        fast_vjp_mi<L, R, CK, VS>(a.M, ppa, omta, rho, inv, jv, T, vv, vv + L::MF * VS, vout, vout + L::MF);
      else
        okA = false;
      if (face) {
        const bool inlet = tag == TAG_INLET;
        face_dispatch<L>(code, [&]<int AX, int SG>() {
          face_reverse<L, R, AX, SG>(a.M, inlet, fs, vout);
        });
      }
    }
    if (a.M.obj_on && (code & CODE_SUPPORT)) okA = fast_partial_m<L, R>(a.M, rho, jv, T, vout) && okA;
    if constexpr (VM == FM_DB) {
      store_node<L, R, RESID>(vsrc, vdst, N, idx, vin, vout, rA, !kInSmem);
      push_halo<L, R, +1>(a, x, y, z, vout);
    } else {
      store_aa<L, R, +1, VM>(vdst, N, idx, nb, vout);
    }
  }
  if (!(okP && okA)) atomicMin(a.fl.bad, (a.fl.step_key | (unsigned long long)gflat(g, x, y, z)));
}

// FP32 pairs measured C3 (MLUPS): 4 blocks 9,968, 5: 10,188, 6: 9,903, 8
// (216 B spill) 8,321 -- all below the two FP32 sweeps run apart (10,433), so
// the engine fuses FP64 pairs only (7,067 against 6,109 apart).
#ifndef LBGPU_PAIR_MINB32
#define LBGPU_PAIR_MINB32 5
#endif
// FP64 pair, C3 MLUPS (128-thread blocks): 3 blocks (168 regs) 6,711; 4 (128
// regs) 7,067; 5 (96 regs + 248 B spill) 5,381. The bound is kept per 128
// threads whatever the block shape.
#ifndef LBGPU_PAIR_MINB
#define LBGPU_PAIR_MINB LBGPU_ADJ_MINB
#endif
#define LBGPU_PAIR_BOUNDS(R)                                                   \
  __launch_bounds__(kPairThreads<R>, (sizeof(R) == 4 ? LBGPU_PAIR_MINB32 : LBGPU_PAIR_MINB) * \
                                         128 / kPairThreads<R>)
template <class L, class R, int CK, bool RESID, bool DUALW = false, bool GATED = false>
__global__ void LBGPU_PAIR_BOUNDS(R) k_pair(Launch a, const R* __restrict__ fsrc,
                                                        R* __restrict__ fdst,
                                                        const R* __restrict__ vsrc,
                                                        R* __restrict__ vdst) {
  const int x = a.g.x0 + blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int z = a.g.z0 + blockIdx.z;
  unsigned long long rP = 0, rA = 0;
  if (x < a.g.x1 && y < a.g.ny)
    pair_body<L, R, CK, RESID, FM_DB, FM_DB, DUALW, GATED>(
        a, fsrc, fdst, vsrc, vdst, x, y, z, threadIdx.y * blockDim.x + threadIdx.x, rP, rA);
  if constexpr (RESID) {
    detail::block_max_bits(rP, a.fl.resid);
    detail::block_max_bits(rA, a.fl.aux);
  }
}

// In-place fused pair (AA streaming): f from layout FM, v from layout VM,
// each updated in place. The side-list adjoint nodes run
// BEFORE it (k_adjoint_side reads the base f^{n+1} that this kernel
// overwrites; their v locations are theirs alone).
#ifndef LBGPU_AAPAIR_MINB
#define LBGPU_AAPAIR_MINB LBGPU_PAIR_MINB
#endif
// FP32 in-place pair, C3 MLUPS at 5/6/8 blocks per SM (with LBGPU_AA_REMAT):
// 11,185 / 11,667 / 12,788.
#ifndef LBGPU_AAPAIR_MINB32
#define LBGPU_AAPAIR_MINB32 8
#endif
template <class L, class R, int CK, int FM, int VM>
__global__ void __launch_bounds__(kPairThreads<R>,
                                  (sizeof(R) == 4 ? LBGPU_AAPAIR_MINB32 : LBGPU_AAPAIR_MINB) * 128 /
                                      kPairThreads<R>)
    k_pair_aa(Launch a, R* F, R* V) {
  unsigned long long rP = 0, rA = 0;
  const int x = a.g.x0 + blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x < a.g.x1 && y < a.g.ny)
    pair_body<L, R, CK, false, FM, VM>(a, F, F, V, V, x, y, a.g.z0 + blockIdx.z,
                                       threadIdx.y * blockDim.x + threadIdx.x, rP, rA);
}

// Per-design-node gradient (param_gradient's design part, adjoint.cpp:377-398)
// with, when UPDATE, the one-shot composite/ascent step fused in
// (optimizer.cpp:41-45, descent_update :8-16). The node list holds local
// indices in ascending global order. The analytic kernel (AK = 0) handles
// Interior design nodes only — the reference's own split (adjoint.cpp:388-396)
// — so it carries no dual-number code; design nodes on any other tag (none
// for config-built cases, config.cpp:355) are the SIDE launch over
// NodeTables::grad_side with the dual path (design_gradient_node_dual).
// The analytic kernel stages its v gather through shared memory (cp.async):
// the loads fly while f is gathered and reduced, and hold no registers, so it
// fits 4 resident blocks (128 registers) instead of 3 (148).
template <class L, class R, int AK, bool UPDATE, bool SIDE, int BM = FM_DB, int VM = FM_DB>
__global__ void __launch_bounds__(128, (AK == 0 && !SIDE) ? 4 : 1) k_gradient(Launch a, const R* __restrict__ p,
                                                  const R* __restrict__ q,
                                                  const long long* __restrict__ nodes,
                                                  long long n, double* __restrict__ gout,
                                                  double* __restrict__ w_rw, double zeta,
                                                  double lambda, int accumulate) {
  using namespace detail;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  unsigned long long cmax = 0;
  const long long cnt = SIDE ? a.t.n_grad_side : n;
  if (t < cnt) {
    const long long i = SIDE ? a.t.grad_side[t] : t;
    const Geom& g = a.g;
    const long long idx = nodes[i];
    const uint8_t code = a.t.code[idx];
    constexpr bool kAnalytic = AK == 0 && !SIDE;
    if (!kAnalytic || (code & TAG_MASK) == TAG_INTERIOR) {
      const int x = int(idx % g.nx);
      const int y = int((idx / g.nx) % g.ny);
      const int z = int(idx / ((long long)g.nx * g.ny));
      const Nbr nb = make_nbr(g, x, y, z);
      const double w = a.t.w[idx];
      const PowPair pp = node_pp<LBGPU_EXACT != 0>(a.M, a.t, idx, code | CODE_HAS_W, w);
      double gv = 0.0;
      bool ok;
      if constexpr (kAnalytic) {
        __shared__ R vsm[L::M * 128];
        R* my = vsm + threadIdx.x;
        gather_async_m<L, R, +1, VM>(q, g.N, idx, nb, my, 128);
        R f[L::M];
        gather_m<L, R, -1, BM>(p, g.N, idx, nb, f);
        cp_async_wait_all();
        ok = design_gradient<L, R, 128>(a.M, pp, f, f + L::MF, R(w), my, my + L::MF * 128, gv);
      } else {  // design_gradient_node_dual (adjoint.cpp:361-373)
        R f[L::M], v[L::M];
        gather_m<L, R, -1, BM>(p, g.N, idx, nb, f);
        gather_m<L, R, +1, VM>(q, g.N, idx, nb, v);
        Dual<R> din[L::M], dout[L::M];
#pragma unroll
        for (int k = 0; k < L::M; ++k) din[k] = Dual<R>(f[k]);
        ok = collide_node<L>(a.M, pp, code & TAG_MASK, code_axis(code), code_sign(code),
                             a.t.bcT[idx], din, Dual<R>(R(w), R(1)), Dual<R>(R(a.M.rho_in)), dout);
        R acc = R(0);
#pragma unroll
        for (int k = 0; k < L::M; ++k) acc = acc + v[k] * dout[k].d;
        gv = double(acc);
      }
      if (!ok) atomicMin(a.fl.bad, (a.fl.step_key | (unsigned long long)gflat(g, x, y, z)));
      if constexpr (UPDATE) {
        double comp = gv;
        if (lambda != 0.0) comp -= lambda * (1.0 - 2.0 * w);
        double wn = w + zeta * comp;
        wn = wn < 0.0 ? 0.0 : (1.0 < wn ? 1.0 : wn);
        w_rw[idx] = wn;
        cmax = (unsigned long long)__double_as_longlong(fabs(comp));
      } else {
        gout[i] = accumulate ? gout[i] + gv : gv;
      }
    }
  }
  if constexpr (UPDATE) block_max_bits(cmax, a.fl.aux);
}

// Tangent sweep (tangent_solve, adjoint.cpp:438-476): a primal-shaped pull
// sweep of Dual<R> = (frozen base, df) through the reference-order
// collide_node with w -> (w, dw) and rho_in -> (rho_in, 3 d_inlet_dp); the
// derivative part is stored and the residual is step_residual(df). The value
// part never advances, so only df ping-pongs. Both builds use the reference
// formulas (a verification path).
template <class L, class R, bool RESID>
__global__ void __launch_bounds__(128) k_tangent(Launch a, const R* __restrict__ base,
                                                 const R* __restrict__ src, R* __restrict__ dst,
                                                 const double* __restrict__ dw, double d_rho_in) {
  using namespace detail;
  const int x = a.g.x0 + blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long rmax = 0;
  if (x < a.g.x1) {
    const Geom& g = a.g;
    const int y = blockIdx.y, z = g.z0 + blockIdx.z;
    const long long idx = x + (long long)g.nx * (y + (long long)g.ny * z);
    const Nbr nb = make_nbr(g, x, y, z);
    R fb[L::M], fd[L::M];
    gather<L, R, -1>(base, g.N, nb, fb);
    gather<L, R, -1>(src, g.N, nb, fd);
    const uint8_t code = a.t.code[idx];
    const bool hw = code & CODE_HAS_W;
    const double w = hw ? a.t.w[idx] : 1.0;
    const double dwv = hw ? dw[idx] : 0.0;
    const PowPair pp = node_pp<LBGPU_EXACT != 0>(a.M, a.t, idx, code, w);
    Dual<R> din[L::M], dout[L::M];
#pragma unroll
    for (int k = 0; k < L::M; ++k) din[k] = Dual<R>(fb[k], fd[k]);
    collide_node<L>(a.M, pp, code & TAG_MASK, code_axis(code), code_sign(code), a.t.bcT[idx], din,
                    Dual<R>(R(w), R(dwv)), Dual<R>(R(a.M.rho_in), R(d_rho_in)), dout);
    R out[L::M];
#pragma unroll
    for (int k = 0; k < L::M; ++k) out[k] = dout[k].d;
    store_node<L, R, RESID>(src, dst, g.N, idx, fd, out, rmax);
  }
  if constexpr (RESID) block_max_bits(rmax, a.fl.resid);
}

// dF terms of tangent_solve (adjoint.cpp:478-488): per support node,
// sum_p dF^x/df_p * df_p accumulated in double in plane order.
template <class L, class R>
__global__ void k_tangent_terms(Launch a, const R* __restrict__ base, const R* __restrict__ df,
                                const long long* __restrict__ nodes, long long n,
                                double* __restrict__ terms) {
  using namespace detail;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Geom& g = a.g;
  const long long idx = nodes[i];
  const int x = int(idx % g.nx), y = int((idx / g.nx) % g.ny), z = int(idx / ((long long)g.nx * g.ny));
  const Nbr nb = make_nbr(g, x, y, z);
  R fin[L::M], dfin[L::M], b[L::M];
  gather<L, R, -1>(base, g.N, nb, fin);
  gather<L, R, -1>(df, g.N, nb, dfin);
#pragma unroll
  for (int k = 0; k < L::M; ++k) b[k] = R(0);
  node_partial<L, R>(a.M, fin, b);
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < L::M; ++k) acc += double(b[k]) * double(dfin[k]);
  terms[i] = acc;
}

// Objective terms F^x on the support list (evaluate_raw, objective.cpp:64-72).
template <class L, class R, int BM = FM_DB>
__global__ void k_objective_terms(Launch a, const R* __restrict__ p,
                                  const long long* __restrict__ nodes, long long n,
                                  double* __restrict__ terms) {
  using namespace detail;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Geom& g = a.g;
  const long long idx = nodes[i];
  const int x = int(idx % g.nx), y = int((idx / g.nx) % g.ny), z = int(idx / ((long long)g.nx * g.ny));
  const Nbr nb = make_nbr(g, x, y, z);
  R f[L::M];
  gather_m<L, R, -1, BM>(p, g.N, idx, nb, f);
  R t;
  if (!node_term<L, R>(a.M, f, t)) {
    atomicMin(a.fl.bad, (a.fl.step_key | (unsigned long long)gflat(g, x, y, z)));
    t = R(NAN);
  }
  terms[i] = double(t);
}

// Objective terms from the inbox the gated fused sweep filled (Gate::inbox):
// the same populations k_objective_terms gathers, read coalesced.
template <class L, class R>
__global__ void k_objective_inbox(Launch a, const double* __restrict__ inbox,
                                  const long long* __restrict__ nodes, long long n,
                                  double* __restrict__ terms) {
  using namespace detail;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Geom& g = a.g;
  const long long idx = nodes[i];
  const int x = int(idx % g.nx), y = int((idx / g.nx) % g.ny), z = int(idx / ((long long)g.nx * g.ny));
  const long long S = (long long)g.ny * g.nz, o = y + (long long)g.ny * z;
  R f[L::M];
  LBGPU_FOR(P, 0, L::M, { f[P] = R(inbox[P * S + o]); });
  R t;
  if (!node_term<L, R>(a.M, f, t)) {
    atomicMin(a.fl.bad, (a.fl.step_key | (unsigned long long)gflat(g, x, y, z)));
    t = R(NAN);
  }
  terms[i] = double(t);
}

// Inlet-overpressure global (param_gradient, adjoint.cpp:399-418): one dual
// collision per inlet node with rho_target seeded by 3.
template <class L, class R, int BM = FM_DB, int VM = FM_DB>
__global__ void k_inlet_terms(Launch a, const R* __restrict__ p, const R* __restrict__ q,
                              const long long* __restrict__ nodes, long long n,
                              double* __restrict__ terms) {
  using namespace detail;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Geom& g = a.g;
  const long long idx = nodes[i];
  const int x = int(idx % g.nx), y = int((idx / g.nx) % g.ny), z = int(idx / ((long long)g.nx * g.ny));
  const Nbr nb = make_nbr(g, x, y, z);
  R f[L::M], v[L::M];
  gather_m<L, R, -1, BM>(p, g.N, idx, nb, f);
  gather_m<L, R, +1, VM>(q, g.N, idx, nb, v);
  const uint8_t code = a.t.code[idx];
  const double w = (code & CODE_HAS_W) ? a.t.w[idx] : 1.0;
  const PowPair pp = node_pp<LBGPU_EXACT != 0>(a.M, a.t, idx, code, w);
  Dual<R> din[L::M], dout[L::M];
#pragma unroll
  for (int k = 0; k < L::M; ++k) din[k] = Dual<R>(f[k]);
  const bool ok = collide_node<L>(a.M, pp, code & TAG_MASK, code_axis(code), code_sign(code),
                                  a.t.bcT[idx], din, Dual<R>(R(w)),
                                  Dual<R>(R(a.M.rho_in), R(3)), dout);
  if (!ok) atomicMin(a.fl.bad, (a.fl.step_key | (unsigned long long)gflat(g, x, y, z)));
  R acc = R(0);
#pragma unroll
  for (int k = 0; k < L::M; ++k) acc = acc + v[k] * dout[k].d;
  terms[i] = double(acc);
}

// Reference-layout conversion. D = -1: primal (f_ref(x) = post(x - e)),
// D = +1: adjoint (v_ref(x) = post(x + e)). TO_REF gathers post -> ref,
// otherwise scatters ref -> post (the exact inverse permutation).
// FM: the post buffer's addressing mode; an in-place field is always
// uploaded into layout O (where it equals the reference layout).
template <class L, class R, int D, bool TO_REF, int FM = FM_DB>
__global__ void k_layout(Geom g, const void* __restrict__ in, void* __restrict__ out) {
  using namespace detail;
  const int x = g.x0 + blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= g.x1) return;
  const long long N = g.N;
  const long long idx = x + (long long)g.nx * (y + (long long)g.ny * z);
  const Nbr nb = make_nbr(g, x, y, z);
  if constexpr (TO_REF) {
    const R* post = static_cast<const R*>(in);
    double* ref = static_cast<double*>(out);
    LBGPU_FOR(P, 0, L::M, { ref[P * N + idx] = double(*in_at<L, D, FM, P>(post, N, idx, nb)); });
  } else {
    const double* ref = static_cast<const double*>(in);
    R* post = static_cast<R*>(out);
    if constexpr (FM == FM_DB) {
      // post(y) = ref(y - D e)
      LBGPU_FOR(P, 0, L::M, { post[P * N + idx] = R(ref[P * N + nbr_idx<L, P, -D>(nb)]); });
    } else {
      static_assert(FM == FM_O, "uploads land in layout O");
      LBGPU_FOR(P, 0, L::M, { post[P * N + idx] = R(ref[P * N + idx]); });
    }
  }
}

// initialize_state (collision.cpp:296-306): flow planes at w_j, thermal 0.
// Uniform planes are invariant under streaming, so the post-collision layout
// holds the same values.
template <class L, class R>
__global__ void k_init(long long N, R* __restrict__ buf) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= N) return;
#pragma unroll
  for (int p = 0; p < L::M; ++p) buf[p * N + i] = p < L::MF ? R(L::wf(p)) : R(0);
}

// ---------------------------------------------------------------------
// Halo exchange between x-slabs (PartitionedRun::do_step's pack / send /
// recv / install, partition.cpp:133-174, in pull form). After a sweep of a
// field with pull direction D (-1 primal, +1 adjoint), the next sweep's
// owned column 0 reads the planes with D*e_x = -1 from the left ghost
// (local nx-1) and column span-1 reads the planes with D*e_x = +1 from the
// right ghost (local span). So each slab ships its last owned column's
// D*e_x = -1 planes to the right neighbour and its first column's
// D*e_x = +1 planes to the left neighbour: 6 planes x ny x nz each way for
// both lattice pairs. For the adjoint (D = +1) these are the primal's lists
// swapped, the reference's transposed plan (partition.cpp:143-146).

template <class L, class R, int D>
__global__ void k_halo_pack(Geom g, const R* __restrict__ buf, R* __restrict__ send_left,
                            R* __restrict__ send_right) {
  const long long yz = (long long)g.ny * g.nz;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= yz) return;
  const long long row = (long long)g.nx * t;  // node (0, y, z) with t = y + ny*z
#pragma unroll
  for (int k = 0; k < kHaloPlanes<L>; ++k) {
    const int pr = halo_slot<L, D, -1>(k), pl = halo_slot<L, D, +1>(k);
    send_right[k * yz + t] = buf[pr * g.N + row + (g.x1 - 1)];
    send_left[k * yz + t] = buf[pl * g.N + row + g.x0];
  }
}

template <class L, class R, int D>
__global__ void k_halo_unpack(Geom g, R* __restrict__ buf, const R* __restrict__ recv_left,
                              const R* __restrict__ recv_right) {
  const long long yz = (long long)g.ny * g.nz;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= yz) return;
  const long long row = (long long)g.nx * t;
#pragma unroll
  for (int k = 0; k < kHaloPlanes<L>; ++k) {
    const int pr = halo_slot<L, D, -1>(k), pl = halo_slot<L, D, +1>(k);
    buf[pr * g.N + row + (g.nx - 1)] = recv_left[k * yz + t];
    buf[pl * g.N + row + g.x1] = recv_right[k * yz + t];
  }
}

// In-process variant: read the neighbours' buffers directly (same device or
// peer-mapped), no staging.
template <class L, class R, int D>
__global__ void k_halo_pull(Geom g, R* __restrict__ buf, const R* __restrict__ left, Geom gl,
                            const R* __restrict__ right, Geom gr) {
  const long long yz = (long long)g.ny * g.nz;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= yz) return;
#pragma unroll
  for (int k = 0; k < kHaloPlanes<L>; ++k) {
    const int pr = halo_slot<L, D, -1>(k), pl = halo_slot<L, D, +1>(k);
    buf[pr * g.N + (long long)g.nx * t + (g.nx - 1)] =
        left[pr * gl.N + (long long)gl.nx * t + (gl.x1 - 1)];
    buf[pl * g.N + (long long)g.nx * t + g.x1] = right[pl * gr.N + (long long)gr.nx * t + gr.x0];
  }
}

// In-place (AA) streaming across slab cuts. A sweep from layout E writes the
// slots that cross a cut into the ghost columns (node x0 stores to x0 - D e_q
// for D e_x(q) = +1, i.e. the left ghost; x1-1 to the right ghost for
// D e_x(q) = -1); they belong to the neighbours' boundary columns, in layout
// O. The reverse exchange ships them there: pack from the ghosts, unpack
// into the receiver's owned boundary columns. (A sweep from O reads its own
// node only; its E-layout boundary values reach the neighbours' ghosts by
// the forward exchange, k_halo_pack / k_halo_unpack with D negated.)
template <class L, class R, int D>
__global__ void k_halo_rpack(Geom g, const R* __restrict__ buf, R* __restrict__ send_left,
                             R* __restrict__ send_right) {
  const long long yz = (long long)g.ny * g.nz;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= yz) return;
  const long long row = (long long)g.nx * t;
#pragma unroll
  for (int k = 0; k < kHaloPlanes<L>; ++k) {
    const int pl = halo_slot<L, D, +1>(k), pr = halo_slot<L, D, -1>(k);
    send_left[k * yz + t] = buf[pl * g.N + row + (g.nx - 1)];  // left ghost
    send_right[k * yz + t] = buf[pr * g.N + row + g.x1];      // right ghost
  }
}
template <class L, class R, int D>
__global__ void k_halo_runpack(Geom g, R* __restrict__ buf, const R* __restrict__ recv_left,
                               const R* __restrict__ recv_right) {
  const long long yz = (long long)g.ny * g.nz;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= yz) return;
  const long long row = (long long)g.nx * t;
#pragma unroll
  for (int k = 0; k < kHaloPlanes<L>; ++k) {
    const int pr = halo_slot<L, D, -1>(k), pl = halo_slot<L, D, +1>(k);
    buf[pr * g.N + row + g.x0] = recv_left[k * yz + t];        // the left neighbour's right ghost
    buf[pl * g.N + row + (g.x1 - 1)] = recv_right[k * yz + t]; // the right neighbour's left ghost
  }
}

// ---------------------------------------------------------------------
// Host-side launchers (one set per build), dispatched by the engine.


// part (SweepArgs): 0 all owned columns; 2 the boundary strips, kStrip
// columns at each end of the slab (whole coalesced rows, computed first so
// their halo can travel; a kernel over single boundary columns would read 26
// scattered lines per node); 1 the columns between the strips.
constexpr int kStrip = 32;
inline int part_ranges(int part, int x0, int x1, int r[2][2]) {
  const bool strips = x1 - x0 > 2 * kStrip;
  if (part == 0 || (part == 2 && !strips)) {
    r[0][0] = x0, r[0][1] = x1;
    return 1;
  }
  if (part == 1) {
    if (!strips) return 0;
    r[0][0] = x0 + kStrip, r[0][1] = x1 - kStrip;
    return 1;
  }
  r[0][0] = x0, r[0][1] = x0 + kStrip, r[1][0] = x1 - kStrip, r[1][1] = x1;
  return 2;
}
// each x-range of s.part, as a Launch whose owned columns are that range
template <class F>
static void for_part(const SweepArgs& s, F&& fn) {
  int r[2][2];
  const int n = part_ranges(s.part, s.a.g.x0, s.a.g.x1, r);
  for (int k = 0; k < n; ++k) {
    Launch a = s.a;
    a.g.x0 = r[k][0], a.g.x1 = r[k][1];
    fn(a);
  }
}

template <class L, class R, int CK, bool RES>
void primal_range(const SweepArgs& s, Launch a, const void* src, void* dst) {
  const R* in = static_cast<const R*>(src);
  R* out = static_cast<R*>(dst);
  if (a.g.x1 <= a.g.x0) return;
  const int bx = (a.g.x1 - a.g.x0) >= 128 ? 128 : ((a.g.x1 - a.g.x0) >= 64 ? 64 : 32);
  int nzs = a.g.nz;
  if (s.z1 > s.z0) a.g.z0 = s.z0, nzs = s.z1 - s.z0;  // z-chunk (pipelined design upload)
  dim3 grid((a.g.x1 - a.g.x0 + bx - 1) / bx, a.g.ny, nzs);
#if !LBGPU_EXACT
  if constexpr (!RES) {
    if (s.upd) {
      k_primal<L, R, CK, false, true><<<grid, bx, 0, a.stream>>>(a, in, out);
      return;
    }
    if constexpr (L::DIM == 3) {
      if (a.gate.wd) {  // upload-gated primal_step_with_design
        k_primal<L, R, CK, false, false, true><<<grid, bx, 0, a.stream>>>(a, in, out);
        return;
      }
    }
  }
#endif
  k_primal<L, R, CK, RES><<<grid, bx, 0, a.stream>>>(a, in, out);
}
template <class L, class R, int CK, bool RES>
void primal_t(const SweepArgs& s, const void* src, void* dst) {
  for_part(s, [&](Launch a) { primal_range<L, R, CK, RES>(s, a, src, dst); });
}
template <class L, class R, int CK, int AK, bool RES>
void adjoint_t(const SweepArgs& s, const void* base, const void* src, void* dst) {
  const R* b = static_cast<const R*>(base);
  const R* in = static_cast<const R*>(src);
  R* out = static_cast<R*>(dst);
  constexpr bool split = !LBGPU_EXACT && AK == 0;
  const R* mom = static_cast<const R*>(s.mom);
  auto go = [&]<bool MOM>() {
    for_part(s, [&](Launch a) {
      if (a.g.x1 > a.g.x0) {
        const int bx = (a.g.x1 - a.g.x0) >= 128 ? 128 : ((a.g.x1 - a.g.x0) >= 64 ? 64 : 32);
        int nzs = a.g.nz;
        if (s.z1 > s.z0) a.g.z0 = s.z0, nzs = s.z1 - s.z0;  // z-chunk (design pair)
        dim3 grid((a.g.x1 - a.g.x0 + bx - 1) / bx, a.g.ny, nzs);
        if constexpr (split && !MOM && !RES && sizeof(R) == 8) {
          if (a.upd.gacc) {  // the sweep also accumulates the design gradient
            k_adjoint<L, R, CK, AK, false, true, false, true><<<grid, bx, 0, a.stream>>>(a, b, in, out, mom);
            return;
          }
        }
        k_adjoint<L, R, CK, AK, RES, split, MOM><<<grid, bx, 0, a.stream>>>(a, b, in, out, mom);
      }
    });
  };
  if constexpr (split) {
    if (mom) go.template operator()<true>();
    else go.template operator()<false>();
  } else {
    go.template operator()<false>();
  }
  // side-list nodes go with the full sweep, or with the boundary part so that
  // they are final before a halo is packed
  if (split && s.n_adj_side > 0 && s.part != 1)
    k_adjoint_side<L, R, CK, RES><<<unsigned((s.n_adj_side + 127) / 128), 128, 0, s.a.stream>>>(
        s.a, b, in, out, s.adj_side, s.n_adj_side);
}

#define LBGPU_CK_DISPATCH(...)                                        \
  do {                                                                \
    if (s.ck == 0) { constexpr int CKV = 0; __VA_ARGS__; }            \
    else if (s.ck == 1) { constexpr int CKV = 1; __VA_ARGS__; }       \
    else { constexpr int CKV = 2; __VA_ARGS__; }                      \
  } while (0)

template <class L, class R>
void primal_l(const SweepArgs& s, const void* src, void* dst) {
#if LBGPU_EXACT
  if (s.resid) primal_t<L, R, 0, true>(s, src, dst);
  else primal_t<L, R, 0, false>(s, src, dst);
#else
  if (s.resid) LBGPU_CK_DISPATCH((primal_t<L, R, CKV, true>(s, src, dst)));
  else LBGPU_CK_DISPATCH((primal_t<L, R, CKV, false>(s, src, dst)));
#endif
}
template <class L, class R, int AK>
void adjoint_l(const SweepArgs& s, const void* base, const void* src, void* dst) {
  if constexpr (AK == 1 || LBGPU_EXACT) {
    if (s.resid) adjoint_t<L, R, 0, AK, true>(s, base, src, dst);
    else adjoint_t<L, R, 0, AK, false>(s, base, src, dst);
  } else {
    if (s.resid) LBGPU_CK_DISPATCH((adjoint_t<L, R, CKV, 0, true>(s, base, src, dst)));
    else LBGPU_CK_DISPATCH((adjoint_t<L, R, CKV, 0, false>(s, base, src, dst)));
  }
}

// addressing mode (0 FM_DB, 1 FM_O, 2 FM_E) -> compile-time NAME
#define LBGPU_FM_DISPATCH(MODE, NAME, ...)                              \
  do {                                                                  \
    if ((MODE) == FM_DB) { constexpr int NAME = FM_DB; __VA_ARGS__; }   \
    else if ((MODE) == FM_O) { constexpr int NAME = FM_O; __VA_ARGS__; } \
    else { constexpr int NAME = FM_E; __VA_ARGS__; }                    \
  } while (0)
// in-place layouts only (FM_O, FM_E)
#define LBGPU_AA_DISPATCH(MODE, NAME, ...)                              \
  do {                                                                  \
    if ((MODE) == FM_O) { constexpr int NAME = FM_O; __VA_ARGS__; }     \
    else { constexpr int NAME = FM_E; __VA_ARGS__; }                    \
  } while (0)

#define LBGPU_LR_DISPATCH(DIM, PREC, ...)                                   \
  do {                                                                      \
    if ((DIM) == 2 && (PREC) == 64) { using L = LatD2; using R = double; __VA_ARGS__; } \
    else if ((DIM) == 2) { using L = LatD2; using R = float; __VA_ARGS__; } \
    else if ((PREC) == 64) { using L = LatD3; using R = double; __VA_ARGS__; } \
    else { using L = LatD3; using R = float; __VA_ARGS__; }                 \
  } while (0)

#if defined(LBGPU_PART_PRIMAL)
void primal(const SweepArgs& s, const void* src, void* dst) {
  LBGPU_LR_DISPATCH(s.dim, s.prec, (primal_l<L, R>(s, src, dst)));
}
#endif
#if defined(LBGPU_PART_ADJOINT)
void adjoint(const SweepArgs& s, const void* base, const void* src, void* dst) {
  LBGPU_LR_DISPATCH(s.dim, s.prec, (adjoint_l<L, R, 0>(s, base, src, dst)));
}
#endif
#if defined(LBGPU_PART_PAIR)
// k_pair over s.part's columns, then the side-list adjoint nodes (part != 1);
// the primal residual goes to a.fl.resid, the adjoint's to a.fl.aux.
template <class L, class R, int CK, bool RES>
void pair_t(const SweepArgs& s, const void* fs_, void* fd_, const void* vs_, void* vd_) {
  const R* fsrc = static_cast<const R*>(fs_);
  const R* vsrc = static_cast<const R*>(vs_);
  R* fdst = static_cast<R*>(fd_);
  R* vdst = static_cast<R*>(vd_);
  constexpr int TB = kPairThreads<R>;
  for_part(s, [&](Launch a) {
    if (a.g.x1 > a.g.x0) {
      const int wx = a.g.x1 - a.g.x0;
      const int bx = wx >= LBGPU_PAIR_BX ? LBGPU_PAIR_BX : (wx >= 64 ? 64 : 32);
      const int by = TB / bx;  // narrow slabs: more rows per block
      int nzs = a.g.nz;
      if (s.z1 > s.z0) a.g.z0 = s.z0, nzs = s.z1 - s.z0;  // z-chunk (design pair)
      dim3 grid((wx + bx - 1) / bx, (a.g.ny + by - 1) / by, nzs);
      bool done = false;
      if constexpr (!RES && L::DIM == 3) {
        if (s.dualw && a.gate.wd) {
          k_pair<L, R, CK, false, true, true><<<grid, dim3(bx, by), 0, a.stream>>>(a, fsrc, fdst, vsrc, vdst);
          done = true;
        } else if (s.dualw) {
          k_pair<L, R, CK, false, true><<<grid, dim3(bx, by), 0, a.stream>>>(a, fsrc, fdst, vsrc, vdst);
          done = true;
        }
      }
      if (!done) k_pair<L, R, CK, RES><<<grid, dim3(bx, by), 0, a.stream>>>(a, fsrc, fdst, vsrc, vdst);
    }
  });
  if (s.n_adj_side > 0 && s.part != 1) {
    Launch as = s.a;
    if (s.dualw) as.t.w = as.t.w_adj;  // the side nodes' adjoint is the previous design's
    as.fl.resid = s.a.fl.aux;  // the side nodes' residual is the adjoint's
    k_adjoint_side<L, R, CK, RES><<<unsigned((s.n_adj_side + 127) / 128), 128, 0, as.stream>>>(
        as, fsrc, vsrc, vdst, s.adj_side, s.n_adj_side);
  }
}
void pair(const SweepArgs& s, const void* fsrc, void* fdst, const void* vsrc, void* vdst) {
#if LBGPU_EXACT
  (void)s, (void)fsrc, (void)fdst, (void)vsrc, (void)vdst;  // the exact build runs the sweeps apart
#else
  LBGPU_LR_DISPATCH(s.dim, s.prec, {
    if (s.resid) LBGPU_CK_DISPATCH((pair_t<L, R, CKV, true>(s, fsrc, fdst, vsrc, vdst)));
    else LBGPU_CK_DISPATCH((pair_t<L, R, CKV, false>(s, fsrc, fdst, vsrc, vdst)));
  });
#endif
}
#endif
#if defined(LBGPU_PART_ADJOINT)
void base_moments(const Launch& a, int dim, int prec, int bm, const void* base, void* mom) {
  const int bx = (a.g.x1 - a.g.x0) >= 128 ? 128 : ((a.g.x1 - a.g.x0) >= 64 ? 64 : 32);
  dim3 grid((a.g.x1 - a.g.x0 + bx - 1) / bx, a.g.ny, a.g.nz);
  LBGPU_LR_DISPATCH(dim, prec, LBGPU_FM_DISPATCH(bm, BM, (k_base_moments<L, R, BM><<<grid, bx, 0, a.stream>>>(
                                    a, static_cast<const R*>(base), static_cast<R*>(mom)))));
}
#endif
#if defined(LBGPU_PART_AA)
// In-place (AA) sweeps, product build: s.fm / s.vm are the current layouts
// (FM_O / FM_E) of f and v; s.part as for the double-buffered launchers.
// launch(a, grid, block) for each x-range of s.part
template <class F>
static void aa_grid(const SweepArgs& s, F&& launch) {
  for_part(s, [&](Launch a) {
    if (a.g.x1 <= a.g.x0) return;
    const int bx = (a.g.x1 - a.g.x0) >= 128 ? 128 : ((a.g.x1 - a.g.x0) >= 64 ? 64 : 32);
    launch(a, dim3((a.g.x1 - a.g.x0 + bx - 1) / bx, a.g.ny, a.g.nz), dim3(bx));
  });
}
void primal_aa(const SweepArgs& s, void* A) {
#if !LBGPU_EXACT
  LBGPU_LR_DISPATCH(s.dim, s.prec, LBGPU_CK_DISPATCH(LBGPU_AA_DISPATCH(s.fm, FM, {
    aa_grid(s, [&](const Launch& a, dim3 grid, dim3 block) {
      k_primal_aa<L, R, CKV, FM><<<grid, block, 0, a.stream>>>(a, static_cast<R*>(A));
    });
  })));
#else
  (void)s, (void)A;
#endif
}
void adjoint_aa(const SweepArgs& s, const void* base, void* V) {
#if !LBGPU_EXACT
  const bool mom = s.mom != nullptr;
  LBGPU_LR_DISPATCH(s.dim, s.prec, LBGPU_CK_DISPATCH(LBGPU_AA_DISPATCH(s.vm, VM, {
    {
      const R* b = static_cast<const R*>(base);
      const R* mo = static_cast<const R*>(s.mom);
      R* v = static_cast<R*>(V);
      if (mom) {  // frozen base: its moments (any base layout)
        aa_grid(s, [&](const Launch& a, dim3 grid, dim3 block) {
          k_adjoint_aa<L, R, CKV, FM_O, VM, true><<<grid, block, 0, a.stream>>>(a, b, v, mo);
        });
      } else if (s.fm == FM_O) {
        aa_grid(s, [&](const Launch& a, dim3 grid, dim3 block) {
          k_adjoint_aa<L, R, CKV, FM_O, VM, false><<<grid, block, 0, a.stream>>>(a, b, v, mo);
        });
      } else {
        aa_grid(s, [&](const Launch& a, dim3 grid, dim3 block) {
          k_adjoint_aa<L, R, CKV, FM_E, VM, false><<<grid, block, 0, a.stream>>>(a, b, v, mo);
        });
      }
      if (s.n_adj_side > 0 && s.part != 1) {
        const unsigned nb = unsigned((s.n_adj_side + 127) / 128);
        if (s.fm == FM_O)
          k_adjoint_side<L, R, CKV, false, FM_O, VM><<<nb, 128, 0, s.a.stream>>>(s.a, b, v, v, s.adj_side, s.n_adj_side);
        else
          k_adjoint_side<L, R, CKV, false, FM_E, VM><<<nb, 128, 0, s.a.stream>>>(s.a, b, v, v, s.adj_side, s.n_adj_side);
      }
    }
  })));
#else
  (void)s, (void)base, (void)V;
#endif
}
#endif
#if defined(LBGPU_PART_AAPAIR)
// Block width of the in-place pair (rows of the block along x).
#ifndef LBGPU_AAPAIR_BX
#define LBGPU_AAPAIR_BX LBGPU_PAIR_BX
#endif
void pair_aa(const SweepArgs& s, void* F, void* V) {
#if !LBGPU_EXACT
  LBGPU_LR_DISPATCH(s.dim, s.prec, LBGPU_CK_DISPATCH({
    R* f = static_cast<R*>(F);
    R* v = static_cast<R*>(V);
    // side-list adjoint nodes first: they read the base this kernel overwrites
    if (s.n_adj_side > 0 && s.part != 1) {
      const unsigned nb = unsigned((s.n_adj_side + 127) / 128);
      auto side = [&]<int FM, int VM>() {
        k_adjoint_side<L, R, CKV, false, FM, VM><<<nb, 128, 0, s.a.stream>>>(s.a, f, v, v, s.adj_side, s.n_adj_side);
      };
      if (s.fm == FM_O && s.vm == FM_O) side.template operator()<FM_O, FM_O>();
      else if (s.fm == FM_O) side.template operator()<FM_O, FM_E>();
      else if (s.vm == FM_O) side.template operator()<FM_E, FM_O>();
      else side.template operator()<FM_E, FM_E>();
    }
    auto go = [&]<int FM, int VM>() {
      constexpr int TB = kPairThreads<R>;
      for_part(s, [&](Launch a) {
        if (a.g.x1 <= a.g.x0) return;
        const int wx = a.g.x1 - a.g.x0;
        const int bx = wx >= LBGPU_AAPAIR_BX ? LBGPU_AAPAIR_BX : (wx >= 64 ? 64 : 32);
        const int by = TB / bx;
        dim3 grid((wx + bx - 1) / bx, (a.g.ny + by - 1) / by, a.g.nz);
        k_pair_aa<L, R, CKV, FM, VM><<<grid, dim3(bx, by), 0, a.stream>>>(a, f, v);
      });
    };
    if (s.fm == FM_O && s.vm == FM_O) go.template operator()<FM_O, FM_O>();
    else if (s.fm == FM_O) go.template operator()<FM_O, FM_E>();
    else if (s.vm == FM_O) go.template operator()<FM_E, FM_O>();
    else go.template operator()<FM_E, FM_E>();
  }));
#else
  (void)s, (void)F, (void)V;
#endif
}
#endif
#if defined(LBGPU_PART_ADJDUAL)
void adjoint_dual(const SweepArgs& s, const void* base, const void* src, void* dst) {
  LBGPU_LR_DISPATCH(s.dim, s.prec, (adjoint_l<L, R, 1>(s, base, src, dst)));
}
#endif
#if defined(LBGPU_PART_AUX)
void gradient(const Launch& a, int dim, int prec, int ak, bool update, const void* p,
              const void* q, const long long* nodes, long long n, double* gout, double* w_rw,
              double zeta, double lambda, int accumulate, int bm, int vm) {
  if (n <= 0) return;
  const int bs = 128;
  const unsigned nb = unsigned((n + bs - 1) / bs);
  LBGPU_LR_DISPATCH(dim, prec, {
    const R* pp = static_cast<const R*>(p);
    const R* qq = static_cast<const R*>(q);
    const unsigned ns = unsigned((a.t.n_grad_side + bs - 1) / bs);
    if (bm != FM_DB || vm != FM_DB) {  // in-place fields: param_gradient only
#if !LBGPU_EXACT
      auto go = [&]<int BM, int VM>() {
        if (ak == 0) {
          k_gradient<L, R, 0, false, false, BM, VM><<<nb, bs, 0, a.stream>>>(a, pp, qq, nodes, n, gout, w_rw, zeta, lambda, accumulate);
          if (ns) k_gradient<L, R, 1, false, true, BM, VM><<<ns, bs, 0, a.stream>>>(a, pp, qq, nodes, n, gout, w_rw, zeta, lambda, accumulate);
        } else {
          k_gradient<L, R, 1, false, false, BM, VM><<<nb, bs, 0, a.stream>>>(a, pp, qq, nodes, n, gout, w_rw, zeta, lambda, accumulate);
        }
      };
      if (bm == FM_O && vm == FM_O) go.template operator()<FM_O, FM_O>();
      else if (bm == FM_O) go.template operator()<FM_O, FM_E>();
      else if (vm == FM_O) go.template operator()<FM_E, FM_O>();
      else go.template operator()<FM_E, FM_E>();
#endif
    } else if (ak == 0 && !update) {
      k_gradient<L, R, 0, false, false><<<nb, bs, 0, a.stream>>>(a, pp, qq, nodes, n, gout, w_rw, zeta, lambda, accumulate);
      if (ns) k_gradient<L, R, 1, false, true><<<ns, bs, 0, a.stream>>>(a, pp, qq, nodes, n, gout, w_rw, zeta, lambda, accumulate);
    } else if (ak == 0) {
      k_gradient<L, R, 0, true, false><<<nb, bs, 0, a.stream>>>(a, pp, qq, nodes, n, gout, w_rw, zeta, lambda, accumulate);
      if (ns) k_gradient<L, R, 1, true, true><<<ns, bs, 0, a.stream>>>(a, pp, qq, nodes, n, gout, w_rw, zeta, lambda, accumulate);
    } else if (!update) {
      k_gradient<L, R, 1, false, false><<<nb, bs, 0, a.stream>>>(a, pp, qq, nodes, n, gout, w_rw, zeta, lambda, accumulate);
    } else {
      k_gradient<L, R, 1, true, false><<<nb, bs, 0, a.stream>>>(a, pp, qq, nodes, n, gout, w_rw, zeta, lambda, accumulate);
    }
  });
}
void objective_terms(const Launch& a, int dim, int prec, const void* p, const long long* nodes,
                     long long n, double* terms, int bm) {
  if (n <= 0) return;
  const unsigned nb = unsigned((n + 127) / 128);
  LBGPU_LR_DISPATCH(dim, prec, LBGPU_FM_DISPATCH(bm, BM, (k_objective_terms<L, R, BM><<<nb, 128, 0, a.stream>>>(
                                    a, static_cast<const R*>(p), nodes, n, terms))));
}
void objective_inbox(const Launch& a, int dim, int prec, const double* inbox, const long long* nodes,
                     long long n, double* terms) {
  if (n <= 0) return;
  const unsigned nb = unsigned((n + 127) / 128);
  LBGPU_LR_DISPATCH(dim, prec, (k_objective_inbox<L, R><<<nb, 128, 0, a.stream>>>(a, inbox, nodes, n, terms)));
}
void inlet_terms(const Launch& a, int dim, int prec, const void* p, const void* q,
                 const long long* nodes, long long n, double* terms, int bm, int vm) {
  if (n <= 0) return;
  const unsigned nb = unsigned((n + 127) / 128);
  LBGPU_LR_DISPATCH(dim, prec, {
    const R* pp = static_cast<const R*>(p);
    const R* qq = static_cast<const R*>(q);
    if (bm == FM_DB && vm == FM_DB) k_inlet_terms<L, R><<<nb, 128, 0, a.stream>>>(a, pp, qq, nodes, n, terms);
    else if (bm == FM_O && vm == FM_O) k_inlet_terms<L, R, FM_O, FM_O><<<nb, 128, 0, a.stream>>>(a, pp, qq, nodes, n, terms);
    else if (bm == FM_O) k_inlet_terms<L, R, FM_O, FM_E><<<nb, 128, 0, a.stream>>>(a, pp, qq, nodes, n, terms);
    else if (vm == FM_O) k_inlet_terms<L, R, FM_E, FM_O><<<nb, 128, 0, a.stream>>>(a, pp, qq, nodes, n, terms);
    else k_inlet_terms<L, R, FM_E, FM_E><<<nb, 128, 0, a.stream>>>(a, pp, qq, nodes, n, terms);
  });
}
#endif
#if defined(LBGPU_PART_TANGENT)
void tangent(const SweepArgs& s, const void* base, const void* src, void* dst, const double* dw,
             double d_rho_in) {
  const Launch& a = s.a;
  const int bx = (a.g.x1 - a.g.x0) >= 128 ? 128 : ((a.g.x1 - a.g.x0) >= 64 ? 64 : 32);
  dim3 grid((a.g.x1 - a.g.x0 + bx - 1) / bx, a.g.ny, a.g.nz);
  LBGPU_LR_DISPATCH(s.dim, s.prec, {
    const R* b = static_cast<const R*>(base);
    const R* in = static_cast<const R*>(src);
    R* out = static_cast<R*>(dst);
    if (s.resid) k_tangent<L, R, true><<<grid, bx, 0, a.stream>>>(a, b, in, out, dw, d_rho_in);
    else k_tangent<L, R, false><<<grid, bx, 0, a.stream>>>(a, b, in, out, dw, d_rho_in);
  });
}
void tangent_terms(const Launch& a, int dim, int prec, const void* base, const void* df,
                   const long long* nodes, long long n, double* terms) {
  if (n <= 0) return;
  const unsigned nb = unsigned((n + 127) / 128);
  LBGPU_LR_DISPATCH(dim, prec, (k_tangent_terms<L, R><<<nb, 128, 0, a.stream>>>(
                                    a, static_cast<const R*>(base), static_cast<const R*>(df),
                                    nodes, n, terms)));
}
#endif
#if defined(LBGPU_PART_PRIMAL)
// fm: the field's addressing mode (uploads into an in-place field land in O)
void layout(const Geom& g, int dim, int prec, int field, bool to_ref, const void* in, void* out,
            cudaStream_t st, int fm) {
  const int bx = (g.x1 - g.x0) >= 128 ? 128 : 32;
  dim3 grid((g.x1 - g.x0 + bx - 1) / bx, g.ny, g.nz);
  LBGPU_LR_DISPATCH(dim, prec, {
    if (!to_ref && fm != FM_DB) {
      if (field == 0) k_layout<L, R, -1, false, FM_O><<<grid, bx, 0, st>>>(g, in, out);
      else k_layout<L, R, +1, false, FM_O><<<grid, bx, 0, st>>>(g, in, out);
    } else if (to_ref) {
      LBGPU_FM_DISPATCH(fm, FM, {
        if (field == 0) k_layout<L, R, -1, true, FM><<<grid, bx, 0, st>>>(g, in, out);
        else k_layout<L, R, +1, true, FM><<<grid, bx, 0, st>>>(g, in, out);
      });
    } else {
      if (field == 0) k_layout<L, R, -1, false><<<grid, bx, 0, st>>>(g, in, out);
      else k_layout<L, R, +1, false><<<grid, bx, 0, st>>>(g, in, out);
    }
  });
}
void halo(int op, const Geom& g, int dim, int prec, int field, void* buf, void* a, void* b,
          const void* left, const Geom& gl, const void* right, const Geom& gr, cudaStream_t st) {
  const long long yz = (long long)g.ny * g.nz;
  const unsigned nb = unsigned((yz + 127) / 128);
  LBGPU_LR_DISPATCH(dim, prec, {
    R* B = static_cast<R*>(buf);
    // field 0: D = -1 (primal), 1: D = +1 (adjoint); ops 5 / 6 negate D (AA forward)
    if (op == 0 || op == 5) {  // pack into a (left), b (right)
      if ((field == 0) == (op == 0)) k_halo_pack<L, R, -1><<<nb, 128, 0, st>>>(g, B, (R*)a, (R*)b);
      else k_halo_pack<L, R, +1><<<nb, 128, 0, st>>>(g, B, (R*)a, (R*)b);
    } else if (op == 1 || op == 6) {  // unpack from a (left), b (right)
      if ((field == 0) == (op == 1)) k_halo_unpack<L, R, -1><<<nb, 128, 0, st>>>(g, B, (const R*)a, (const R*)b);
      else k_halo_unpack<L, R, +1><<<nb, 128, 0, st>>>(g, B, (const R*)a, (const R*)b);
    } else if (op == 3) {  // AA reverse: pack the ghosts
      if (field == 0) k_halo_rpack<L, R, -1><<<nb, 128, 0, st>>>(g, B, (R*)a, (R*)b);
      else k_halo_rpack<L, R, +1><<<nb, 128, 0, st>>>(g, B, (R*)a, (R*)b);
    } else if (op == 4) {  // AA reverse: unpack into the owned boundary columns
      if (field == 0) k_halo_runpack<L, R, -1><<<nb, 128, 0, st>>>(g, B, (const R*)a, (const R*)b);
      else k_halo_runpack<L, R, +1><<<nb, 128, 0, st>>>(g, B, (const R*)a, (const R*)b);
    } else {  // pull from neighbour buffers
      if (field == 0)
        k_halo_pull<L, R, -1><<<nb, 128, 0, st>>>(g, B, (const R*)left, gl, (const R*)right, gr);
      else
        k_halo_pull<L, R, +1><<<nb, 128, 0, st>>>(g, B, (const R*)left, gl, (const R*)right, gr);
    }
  });
}
void init_state(long long N, int dim, int prec, void* buf, cudaStream_t st) {
  const unsigned nb = unsigned((N + 255) / 256);
  LBGPU_LR_DISPATCH(dim, prec, (k_init<L, R><<<nb, 256, 0, st>>>(N, static_cast<R*>(buf))));
}
#endif

}  // namespace LBGPU_NS
}  // namespace lbgpu

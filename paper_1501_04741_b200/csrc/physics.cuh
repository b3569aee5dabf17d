// Node physics, written once over a scalar type T that is either the storage
// real R (float/double) or the forward-mode dual Dual<R>.
//
// This is the "reference-order" formulation: every expression follows the
// reference's evaluation order (left-to-right C++), so that compiled without
// FMA contraction (kernels_exact.cu, -fmad=false) it reproduces the reference
// bit for bit, and seeded with duals it reproduces the reference's Jacobian
// columns (adjoint.cpp:21-42). The fast kernels (kernels.cuh) use it for
// everything off the bulk path (pressure-face reconstruction, gradients,
// objective terms, dual sweeps) and have their own algebraically simplified
// bulk formulas.
//
// Zero velocity components are skipped at compile time; for finite inputs
// that changes at most the sign of an exact zero that is always later added
// to a non-zero value, so results are unchanged.
#pragma once
#include <cmath>
#include <cstdint>

#include "lattice.cuh"

#ifndef LBGPU_HD
#define LBGPU_HD __host__ __device__ __forceinline__
#endif

namespace lbgpu {

// ---------------------------------------------------------------- Dual<R>
// Forward-mode dual (dual.hpp:14-71): value + one directional derivative.
template <class R>
struct Dual {
  R v, d;
  LBGPU_HD Dual() : v(0), d(0) {}
  LBGPU_HD Dual(R value) : v(value), d(0) {}
  LBGPU_HD Dual(R value, R deriv) : v(value), d(deriv) {}
};
template <class R> LBGPU_HD Dual<R> operator-(Dual<R> a) { return {-a.v, -a.d}; }
template <class R> LBGPU_HD Dual<R> operator+(Dual<R> a, Dual<R> b) { return {a.v + b.v, a.d + b.d}; }
template <class R> LBGPU_HD Dual<R> operator-(Dual<R> a, Dual<R> b) { return {a.v - b.v, a.d - b.d}; }
template <class R> LBGPU_HD Dual<R> operator*(Dual<R> a, Dual<R> b) {
  return {a.v * b.v, a.d * b.v + a.v * b.d};
}
template <class R> LBGPU_HD Dual<R> operator/(Dual<R> a, Dual<R> b) {
  const R q = a.v / b.v;
  return {q, (a.d - q * b.d) / b.v};
}
template <class R> LBGPU_HD Dual<R>& operator+=(Dual<R>& a, Dual<R> b) { return a = a + b; }
template <class R> LBGPU_HD Dual<R>& operator-=(Dual<R>& a, Dual<R> b) { return a = a - b; }

template <class T> struct RealOf { using type = T; };
template <class R> struct RealOf<Dual<R>> { using type = R; };
template <class T> using real_t = typename RealOf<T>::type;

template <class T> LBGPU_HD T K(double c) { return T(real_t<T>(c)); }
template <class R> LBGPU_HD R val(R x) { return x; }
template <class R> LBGPU_HD R val(Dual<R> x) { return x.v; }
template <class R> LBGPU_HD R der(R) { return R(0); }
template <class R> LBGPU_HD R der(Dual<R> x) { return x.d; }

// ------------------------------------------------------------ model block
// Everything node-independent a node update needs. Passed by value into
// kernels (param space).
struct Model {
  double om;          // flow relaxation 1/(0.5+3 nu) (collision.hpp:56)
  double beta_f, beta_s;
  double rho_in, rho_out;  // collision.hpp:57-58
  double u_clamp;
  // fast build's pressure faces: 1/rho_in, 1/rho_out, 1/(1-u_clamp), 1/(1+u_clamp)
  double inv_rho_in, inv_rho_out, inv_1m_uc, inv_1p_uc;
  double theta;
  int theta_int;      // theta when it is a small positive integer, else 0
  int fluid_power;    // SwitchingSpec::Form (topology.hpp:33-38)
  int collision_bgk;
  int nonhydro;       // any "other" moment row relaxes at omega_nonhydro != 1
  double mrt_c[19];   // fast MRT: (1 - relax_i) / |U_i|^2 per moment row
  const double* A;    // dense relaxation matrix (mf x mf), reference order
  const double* At;   // its transpose (ModelTables::At)
  int obj_kind;       // 0 mixing 1 heatflux 2 synthetic
  int obj_on;         // adjoint sweeps add the objective partial on support nodes
  int flux_axis, flux_sign;
};

// pow(base, theta) and pow(base, theta-1) for one node's switching base
// (w for fluid_power, 1-w for solid_power). In the exact build they come
// from host glibc via per-node tables (glibc pow is not correctly rounded, so
// only the host library reproduces the reference bits); in the fast build
// they are computed on the device.
struct PowPair {
  double p0, p1;
};

// Correctly rounded x^n for small positive n via a double-double product
// chain (explicit fma, so it is independent of -fmad).
LBGPU_HD double dd_pow_int(double x, int n) {
  if (n == 0) return 1.0;
  double hi = x, lo = 0.0;
  for (int i = 1; i < n; ++i) {
    const double p = hi * x;
#ifdef __CUDA_ARCH__
    double e = __fma_rn(hi, x, -p);
    e = __fma_rn(lo, x, e);
#else
    double e = std::fma(hi, x, -p);
    e = std::fma(lo, x, e);
#endif
    const double s = p + e;
    lo = e - (s - p);
    hi = s;
  }
  return hi + lo;
}

LBGPU_HD PowPair pow_pair(const Model& M, double w) {
  const double base = M.fluid_power ? w : 1.0 - w;
  if (M.theta_int > 0) return {dd_pow_int(base, M.theta_int), dd_pow_int(base, M.theta_int - 1)};
  return {pow(base, M.theta), pow(base, M.theta - 1.0)};
}

// switching_eval (topology.hpp:42-46) given the node's pow pair. With T a
// dual, the derivative part is the reference's pow(Dual) rule (dual.hpp:56-61).
template <class T>
LBGPU_HD T switching(const Model& M, PowPair pp, T w);
template <>
LBGPU_HD double switching<double>(const Model& M, PowPair pp, double w) {
  (void)w;
  return M.fluid_power ? pp.p0 : 1.0 - pp.p0;
}
template <>
LBGPU_HD float switching<float>(const Model& M, PowPair pp, float w) {
  (void)w;
  return M.fluid_power ? float(pp.p0) : float(1.0 - pp.p0);
}
template <>
LBGPU_HD Dual<double> switching<Dual<double>>(const Model& M, PowPair pp, Dual<double> w) {
  const double dv = M.theta * pp.p1;
  if (M.fluid_power) return {pp.p0, dv * w.d};
  const Dual<double> x = Dual<double>(1.0) - w;
  return Dual<double>(1.0) - Dual<double>(pp.p0, dv * x.d);
}
template <>
LBGPU_HD Dual<float> switching<Dual<float>>(const Model& M, PowPair pp, Dual<float> w) {
  const float dv = float(M.theta * pp.p1);
  if (M.fluid_power) return {float(pp.p0), dv * w.d};
  const Dual<float> x = Dual<float>(1.0f) - w;
  return Dual<float>(1.0f) - Dual<float>(float(pp.p0), dv * x.d);
}

// switching_derivative (topology.cpp:34-38), in double.
LBGPU_HD double switching_derivative(const Model& M, PowPair pp) { return M.theta * pp.p1; }

// diffusivity (topology.hpp:51-54)
template <class T>
LBGPU_HD T diffusivity(const Model& M, T w) {
  return w * K<T>(M.beta_f) + (K<T>(1.0) - w) * K<T>(M.beta_s);
}

// e . u with compile-time skipping of zero components (order preserved).
template <class T, int EX, int EY, int EZ>
LBGPU_HD T edot3(const T* u) {
  T acc = K<T>(0.0);
  bool first = true;
  if (EX) { acc = (EX > 0) ? u[0] : -u[0]; first = false; }
  if (EY) { const T t = (EY > 0) ? u[1] : -u[1]; acc = first ? t : acc + t; first = false; }
  if (EZ) { const T t = (EZ > 0) ? u[2] : -u[2]; acc = first ? t : acc + t; first = false; }
  return acc;
}
template <class L, class T, int P>
LBGPU_HD T edotp(const T* u) {
  return edot3<T, cvel<L>(P, 0), cvel<L>(P, 1), cvel<L>(P, 2)>(u);
}

// Compile-time unrolled loop helper.
template <int I, int N>
struct Unroll {
  template <class F>
  LBGPU_HD static void run(F&& f) {
    f.template operator()<I>();
    Unroll<I + 1, N>::run(f);
  }
};
template <int N>
struct Unroll<N, N> {
  template <class F>
  LBGPU_HD static void run(F&&) {}
};
#define LBGPU_FOR(I, LO, HI, ...) \
  Unroll<(LO), (HI)>::run([&]<int I>() __VA_ARGS__)

// ----------------------------------------------- moments and equilibria
// flow_moments (collision.hpp:92-105). Returns false for rho <= 0 / NaN.
template <class L, class T>
LBGPU_HD bool flow_moments(const T* f, T& rho, T* u) {
  T r = K<T>(0.0), q0 = K<T>(0.0), q1 = K<T>(0.0), q2 = K<T>(0.0);
  LBGPU_FOR(J, 0, L::MF, {
    r = r + f[J];
    if constexpr (L::ef(J, 0) != 0) q0 = L::ef(J, 0) > 0 ? q0 + f[J] : q0 - f[J];
    if constexpr (L::ef(J, 1) != 0) q1 = L::ef(J, 1) > 0 ? q1 + f[J] : q1 - f[J];
    if constexpr (L::ef(J, 2) != 0) q2 = L::ef(J, 2) > 0 ? q2 + f[J] : q2 - f[J];
  });
  rho = r;
  if (!(val(r) > 0)) return false;
  u[0] = q0 / r;
  u[1] = q1 / r;
  u[2] = q2 / r;
  return true;
}

template <class L, class T>
LBGPU_HD T thermal_moment(const T* g) {
  T s = K<T>(0.0);
  LBGPU_FOR(J, 0, L::MT, { s = s + g[J]; });
  return s;
}

// flow_equilibrium (collision.hpp:115-124)
template <class L, class T>
LBGPU_HD void flow_eq(T rho, const T* u, T* feq) {
  const T usq = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
  LBGPU_FOR(J, 0, L::MF, {
    const T eu = edotp<L, T, J>(u);
    feq[J] = K<T>(L::wf(J)) * rho *
             (K<T>(1.0) + K<T>(3.0) * eu + K<T>(4.5) * eu * eu - K<T>(1.5) * usq);
  });
}

// thermal_equilibrium (collision.hpp:127-134)
template <class L, class T>
LBGPU_HD void therm_eq(T temp, const T* u, T* geq) {
  LBGPU_FOR(J, 0, L::MT, {
    const T eu = edotp<L, T, L::MF + J>(u);
    geq[J] = K<T>(L::wt(J)) * temp * (K<T>(1.0) + K<T>(3.0) * eu);
  });
}

// interior_collide (collision.cpp:181-215), dense A in reference order.
template <class L, class T>
LBGPU_HD bool interior_collide(const Model& M, PowPair pp, const T* f, const T* g, T w, T* of,
                               T* og) {
  T rho, u[3];
  if (!flow_moments<L>(f, rho, u)) return false;
  const T G = switching<T>(M, pp, w);
  const T up[3] = {G * u[0], G * u[1], G * u[2]};
  T fpre[L::MF], fpost[L::MF], df[L::MF];
  flow_eq<L>(rho, u, fpre);
  flow_eq<L>(rho, up, fpost);
#pragma unroll
  for (int j = 0; j < L::MF; ++j) df[j] = f[j] - fpre[j];
#pragma unroll
  for (int i = 0; i < L::MF; ++i) {
    T acc = fpost[i];
#pragma unroll
    for (int j = 0; j < L::MF; ++j) acc = acc + K<T>(M.A[i * L::MF + j]) * df[j];
    of[i] = acc;
  }
  const T temp = thermal_moment<L>(g);
  const T beta = diffusivity(M, w);
  const T om = K<T>(1.0) / (K<T>(0.5) + K<T>(3.0) * beta);
  T geq[L::MT];
  therm_eq<L>(temp, up, geq);
#pragma unroll
  for (int j = 0; j < L::MT; ++j) og[j] = g[j] + om * (geq[j] - g[j]);
  return true;
}

LBGPU_HD int evel_axis(int e0, int e1, int e2, int axis) {
  return axis == 0 ? e0 : (axis == 1 ? e1 : e2);
}

// zou_he_pressure (collision.cpp:122-177). Returns the axial velocity.
template <class L, class T>
LBGPU_HD T zou_he(const Model& M, const T* fin, T rho_t, int axis, int sign, T* fout) {
  T k0 = K<T>(0.0), km = K<T>(0.0);
#pragma unroll
  for (int j = 0; j < L::MF; ++j) {
    const int ea = evel_axis(L::ef(j, 0), L::ef(j, 1), L::ef(j, 2), axis);
    if (ea == 0) k0 = k0 + fin[j];
    else if (ea == -sign) km = km + fin[j];
  }
  const T s = K<T>(double(sign));
  T ua = s * (K<T>(1.0) - (k0 + K<T>(2.0) * km) / rho_t);
  T rho = rho_t;
  const T aua = val(ua) < 0 ? -ua : ua;
  if (val(aua) > val(K<T>(M.u_clamp))) {
    ua = val(ua) > 0 ? K<T>(M.u_clamp) : K<T>(-M.u_clamp);
    rho = (k0 + K<T>(2.0) * km) / (K<T>(1.0) - s * ua);
  }
  T u[3] = {K<T>(0.0), K<T>(0.0), K<T>(0.0)};
  u[axis] = ua;
  T feq[L::MF];
  flow_eq<L>(rho, u, feq);
  T nb[3] = {K<T>(0.0), K<T>(0.0), K<T>(0.0)};
#pragma unroll
  for (int j = 0; j < L::MF; ++j) {
    const int e[3] = {L::ef(j, 0), L::ef(j, 1), L::ef(j, 2)};
    if (e[axis] != 0) continue;
#pragma unroll
    for (int b = 0; b < 3; ++b)
      if (b != axis && e[b]) nb[b] = nb[b] + K<T>(0.5 * e[b]) * fin[j];
  }
#pragma unroll
  for (int j = 0; j < L::MF; ++j) fout[j] = fin[j];
#pragma unroll
  for (int j = 0; j < L::MF; ++j) {
    const int e[3] = {L::ef(j, 0), L::ef(j, 1), L::ef(j, 2)};
    if (e[axis] != sign) continue;
    const int o = L::oppf(j);
    T corr = K<T>(0.0);
#pragma unroll
    for (int b = 0; b < 3; ++b)
      if (b != axis && e[b]) corr = corr + K<T>(double(e[b])) * nb[b];
    fout[j] = fin[o] + (feq[j] - feq[o]) - corr;
  }
  return ua;
}

// Pressure-face reconstruction of collide_node (collision.cpp:248-292): the
// Zou-He flow slots plus the imposed (inlet) or outflow-rebuilt (outlet)
// thermal equilibrium, i.e. everything before the wet-node interior collide.
template <class L, class T>
LBGPU_HD void face_recon(const Model& M, int tag, int axis, int sign, double bcT, const T* fin,
                         T rho_t, T* frec, T* grec) {
  const T* g = fin + L::MF;
  T u[3] = {K<T>(0.0), K<T>(0.0), K<T>(0.0)};
  if (tag == TAG_INLET) {
    u[axis] = zou_he<L>(M, fin, rho_t, axis, sign, frec);
    therm_eq<L>(K<T>(bcT), u, grec);
  } else {
    u[axis] = zou_he<L>(M, fin, K<T>(M.rho_out), axis, sign, frec);
    T tnum = K<T>(0.0), tden = K<T>(0.0);
    LBGPU_FOR(J, 0, L::MT, {
      if (evel_axis(L::et(J, 0), L::et(J, 1), L::et(J, 2), axis) != sign) {
        const T eu = edotp<L, T, L::MF + J>(u);
        tnum = tnum + g[J];
        tden = tden + K<T>(L::wt(J)) * (K<T>(1.0) + K<T>(3.0) * eu);
      }
    });
    therm_eq<L>(tnum / tden, u, grec);
  }
}

// collide_node (collision.cpp:219-294), reference order. Returns false when
// flow_moments would throw NumericError.
template <class L, class T>
LBGPU_HD bool collide_node(const Model& M, PowPair pp, int tag, int axis, int sign, double bcT,
                           const T* fin, T w, T rho_t, T* fout) {
  const T* f = fin;
  const T* g = fin + L::MF;
  T* of = fout;
  T* og = fout + L::MF;
  switch (tag) {
    case TAG_INTERIOR:
      return interior_collide<L>(M, pp, f, g, w, of, og);
    case TAG_WALL:
      LBGPU_FOR(J, 0, L::MF, { of[J] = f[L::oppf(J)]; });
      LBGPU_FOR(J, 0, L::MT, { og[J] = g[L::oppt(J)]; });
      return true;
    case TAG_HEATER: {
      LBGPU_FOR(J, 0, L::MF, { of[J] = f[L::oppf(J)]; });
      const T u0[3] = {K<T>(0.0), K<T>(0.0), K<T>(0.0)};
      therm_eq<L>(K<T>(bcT), u0, og);
      return true;
    }
    default: {
      T frec[L::MF], grec[L::MT];
      face_recon<L>(M, tag, axis, sign, bcT, fin, rho_t, frec, grec);
      return interior_collide<L>(M, pp, frec, grec, w, of, og);
    }
  }
}

// ------------------------------------------------------------- objective
// node_term (objective.cpp:19-32)
template <class L, class R>
LBGPU_HD bool node_term(const Model& M, const R* fin, R& out) {
  if (M.obj_kind == 2) {
    R s = R(0);
#pragma unroll
    for (int p = 0; p < L::M; ++p) s = s + fin[p] * fin[p];
    out = R(0.5) * s;
    return true;
  }
  R rho, u[3];
  if (!flow_moments<L>(fin, rho, u)) return false;
  const R temp = thermal_moment<L>(fin + L::MF);
  const R un = R(double(M.flux_sign)) * u[M.flux_axis];
  out = M.obj_kind == 0 ? un * (R(1.0) - temp * temp) : un * temp;
  return true;
}

// node_partial (objective.cpp:34-62)
template <class L, class R>
LBGPU_HD bool node_partial(const Model& M, const R* fin, R* out) {
  if (M.obj_kind == 2) {
#pragma unroll
    for (int p = 0; p < L::M; ++p) out[p] = fin[p];
    return true;
  }
  R rho, u[3];
  if (!flow_moments<L>(fin, rho, u)) return false;
  const R temp = thermal_moment<L>(fin + L::MF);
  const int a = M.flux_axis;
  const R sgn = R(double(M.flux_sign));
  const R un = sgn * u[a];
  const R du = M.obj_kind == 0 ? (R(1.0) - temp * temp) * sgn : temp * sgn;
#pragma unroll
  for (int k = 0; k < L::MF; ++k) {
    const int ea = a == 0 ? L::ef(k, 0) : (a == 1 ? L::ef(k, 1) : L::ef(k, 2));
    out[k] = du * (R(double(ea)) - u[a]) / rho;
  }
  const R dT = M.obj_kind == 0 ? R(-2.0) * temp * un : un;
#pragma unroll
  for (int k = 0; k < L::MT; ++k) out[L::MF + k] = dT;
  return true;
}

// --------------------------------------------------------------- adjoint
// interior_vjp (adjoint.cpp:50-121), reference order with dense A^T.
template <class L, class R>
LBGPU_HD bool interior_vjp(const Model& M, PowPair pp, const R* f, const R* g, R w, const R* vf,
                           const R* vg, R* outf, R* outg) {
  R rho, u[3];
  if (!flow_moments<L>(f, rho, u)) return false;
  const R G = switching<R>(M, pp, w);
  const R up[3] = {G * u[0], G * u[1], G * u[2]};
  R fpre[L::MF], fpost[L::MF], r[L::MF];
  flow_eq<L>(rho, u, fpre);
  flow_eq<L>(rho, up, fpost);
#pragma unroll
  for (int k = 0; k < L::MF; ++k) {
    R acc = R(0);
#pragma unroll
    for (int j = 0; j < L::MF; ++j) acc = acc + R(M.At[k * L::MF + j]) * vf[j];
    r[k] = acc;
  }
  R Pr = R(0), Rr = R(0), Pu[3] = {R(0), R(0), R(0)}, Ru[3] = {R(0), R(0), R(0)};
  LBGPU_FOR(J, 0, L::MF, {
    Pr = Pr + vf[J] * fpost[J];
    Rr = Rr + r[J] * fpre[J];
    const R wjrho = R(L::wf(J)) * rho;
    const R eup = edotp<L, R, J>(up);
    const R eu = edotp<L, R, J>(u);
    const R cp = vf[J] * wjrho, cr = r[J] * wjrho;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int ea = L::ef(J, a);
      const R tp = ea ? R(3) * R(double(ea)) + R(9) * eup * R(double(ea)) : R(9) * eup * R(0.0);
      const R tr = ea ? R(3) * R(double(ea)) + R(9) * eu * R(double(ea)) : R(9) * eu * R(0.0);
      Pu[a] = Pu[a] + cp * (tp - R(3) * up[a]);
      Ru[a] = Ru[a] + cr * (tr - R(3) * u[a]);
    }
  });
  Pr = Pr / rho;
  Rr = Rr / rho;
  const R temp = thermal_moment<L>(g);
  const R beta = diffusivity(M, w);
  const R om = R(1) / (R(0.5) + R(3) * beta);
  R sigma = R(0), S[3] = {R(0), R(0), R(0)};
  LBGPU_FOR(J, 0, L::MT, {
    const R tw = R(L::wt(J));
    const R eup = edotp<L, R, L::MF + J>(up);
    sigma = sigma + vg[J] * tw * (R(1) + R(3) * eup);
    const R c = R(3) * om * temp * vg[J] * tw;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int ea = L::et(J, a);
      if (ea) S[a] = S[a] + (ea > 0 ? c : -c);
      else S[a] = S[a] + c * R(0.0);
    }
  });
  R c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) c[a] = G * (Pu[a] + S[a]) - Ru[a];
  const R s0 = Pr - Rr - (c[0] * u[0] + c[1] * u[1] + c[2] * u[2]) / rho;
  LBGPU_FOR(K_, 0, L::MF, {
    const R ce = edot3<R, L::ef(K_, 0), L::ef(K_, 1), L::ef(K_, 2)>(c);
    outf[K_] = r[K_] + s0 + ce / rho;
  });
#pragma unroll
  for (int k = 0; k < L::MT; ++k) outg[k] = (R(1) - om) * vg[k] + om * sigma;
  return true;
}

// vjp_dual (adjoint.cpp:21-42): J^T v from M dual-number collisions.
template <class L, class R>
LBGPU_HD bool vjp_dual(const Model& M, PowPair pp, int tag, int axis, int sign, double bcT,
                       const R* fin, R w, const R* vin, R* vout) {
  for (int k = 0; k < L::M; ++k) {
    Dual<R> din[L::M], col[L::M];
#pragma unroll
    for (int p = 0; p < L::M; ++p) din[p] = Dual<R>(fin[p], R(p == k ? 1 : 0));
    if (!collide_node<L>(M, pp, tag, axis, sign, bcT, din, Dual<R>(w), Dual<R>(R(M.rho_in)), col))
      return false;
    R acc = R(0);
#pragma unroll
    for (int j = 0; j < L::M; ++j) acc = acc + vin[j] * col[j].d;
    vout[k] = acc;
  }
  return true;
}

// design_gradient_node (adjoint.cpp:311-358), reference order. VS: the stride
// of vf / vg (1, or the block size when they sit in shared memory).
template <class L, class R, int VS = 1>
LBGPU_HD bool design_gradient(const Model& M, PowPair pp, const R* f, const R* g, R w, const R* vf,
                              const R* vg, double& out) {
  R rho, u[3];
  if (!flow_moments<L>(f, rho, u)) return false;
  const R G = switching<R>(M, pp, w);
  const R up[3] = {G * u[0], G * u[1], G * u[2]};
  const R dG = R(switching_derivative(M, pp));
  R fpost[L::MF];
  flow_eq<L>(rho, up, fpost);
  (void)fpost;
  R Pu[3] = {R(0), R(0), R(0)};
  LBGPU_FOR(J, 0, L::MF, {
    const R eup = edotp<L, R, J>(up);
    const R cp = vf[J * VS] * R(L::wf(J)) * rho;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int ea = L::ef(J, a);
      const R tp = ea ? R(3) * R(double(ea)) + R(9) * eup * R(double(ea)) : R(9) * eup * R(0.0);
      Pu[a] = Pu[a] + cp * (tp - R(3) * up[a]);
    }
  });
  const R temp = thermal_moment<L>(g);
  const R beta = diffusivity(M, w);
  const R om = R(1) / (R(0.5) + R(3) * beta);
  const R dom = R(-3) * (R(M.beta_f) - R(M.beta_s)) * om * om;
  R geq[L::MT];
  therm_eq<L>(temp, up, geq);
  R S[3] = {R(0), R(0), R(0)}, relax = R(0);
  LBGPU_FOR(J, 0, L::MT, {
    const R c = R(3) * om * temp * vg[J * VS] * R(L::wt(J));
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int ea = L::et(J, a);
      if (ea) S[a] = S[a] + (ea > 0 ? c : -c);
      else S[a] = S[a] + c * R(0.0);
    }
    relax = relax + vg[J * VS] * (geq[J] - g[J]);
  });
  R acc = R(0);
#pragma unroll
  for (int a = 0; a < 3; ++a) acc = acc + u[a] * (Pu[a] + S[a]);
  out = double(dG * acc + dom * relax);
  return true;
}

}  // namespace lbgpu

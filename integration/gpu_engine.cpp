// Reference-side binding (see gpu_engine.hpp). Compiled against the
// reference's own headers: g++ -std=c++20 -I<ref>/proj/include -I<repo>/include.
#include "gpu_engine.hpp"

#include <string>

#include "lbopt/errors.hpp"

namespace lbopt {

lbgpu_engine* make_gpu_engine(const System& s, const ObjectiveSpec& o, int precision, int exact,
                              int device) {
  const long n = s.shape.nodes();
  std::vector<uint8_t> tag(static_cast<std::size_t>(n));
  for (long i = 0; i < n; ++i) tag[std::size_t(i)] = uint8_t(s.tags.tag[std::size_t(i)]);
  std::vector<int32_t> vel, opp;
  for (int p = 0; p < s.m; ++p) {
    vel.insert(vel.end(), {s.vel[std::size_t(p)].x, s.vel[std::size_t(p)].y, s.vel[std::size_t(p)].z});
    opp.push_back(s.opp[std::size_t(p)]);
  }
  std::vector<int64_t> support(o.support.begin(), o.support.end());
  lbgpu_system_desc d{};
  d.nx = s.shape.nx, d.ny = s.shape.ny, d.nz = s.shape.nz;
  d.precision = precision, d.exact = exact, d.device = device;
  d.collision = s.model.collision == CollisionKind::BGK ? 1 : 0;
  d.nu = s.model.nu, d.beta_fluid = s.model.beta_fluid, d.beta_solid = s.model.beta_solid;
  d.inlet_dp = s.model.inlet_dp, d.u_clamp = s.model.u_clamp;
  d.omega_nonhydro = s.model.omega_nonhydro, d.switch_theta = s.model.switching.theta;
  d.switch_form = s.model.switching.form == SwitchingSpec::Form::FluidPower ? 1 : 0;
  d.A = s.tables.A.a.data();
  d.relax = s.tables.relax.data();
  d.vel = vel.data(), d.opp = opp.data();
  d.tag = tag.data(), d.bc_T = s.tags.bc_T.data();
  d.bc_axis = s.tags.bc_axis.data(), d.bc_sign = s.tags.bc_sign.data();
  d.w = s.design.w.data(), d.design_mask = s.design.mask.data();
  d.obj_kind = int(o.kind), d.flux_axis = o.flux_axis, d.flux_sign = o.flux_sign;
  d.support = support.data(), d.n_support = int64_t(support.size());
  d.slab_count = 1, d.slab_id = 0, d.streaming = 0;
  lbgpu_engine* e = nullptr;
  const int rc = lbgpu_create(&d, &e);
  if (rc == LBGPU_E_CONFIG) throw ConfigError(lbgpu_last_create_error());
  if (rc != LBGPU_OK) throw NumericError(lbgpu_last_create_error());
  return e;
}

void gpu_check(lbgpu_engine* e, int rc) {
  if (rc == LBGPU_OK) return;
  const std::string msg = lbgpu_error_message(e);
  if (rc == LBGPU_E_CONFIG) throw ConfigError(msg);
  if (rc == LBGPU_E_STATE) throw StateError(msg);
  if (rc == LBGPU_E_IO) throw IoError(msg);
  throw NumericError(msg);
}

namespace {
template <class R>
void upload(lbgpu_engine* e, int field, const StateField<R>& s) {
  const auto raw = s.raw(s.buffer_id());
  std::vector<double> host(raw.begin(), raw.end());
  gpu_check(e, lbgpu_upload_state(e, field, host.data()));
}
template <class R>
void download(lbgpu_engine* e, int field, StateField<R>& s) {
  auto raw = s.raw(s.buffer_id());
  std::vector<double> host(raw.size());
  gpu_check(e, lbgpu_download_state(e, field, host.data()));
  for (std::size_t i = 0; i < raw.size(); ++i) raw[i] = R(host[i]);
}
}  // namespace

template <class R>
SolveResult gpu_solve_fixed_point(lbgpu_engine* e, StateField<R>& f, const SolveOptions<R>& opt) {
  upload(e, 0, f);
  int64_t it = 0;
  double r = 0.0;
  int conv = 0;
  gpu_check(e, lbgpu_solve_primal(e, opt.tol, opt.max_iter, opt.fixed_iters, &it, &r, &conv));
  download(e, 0, f);
  SolveResult res;
  res.converged = conv != 0, res.iterations = long(it), res.residual = r;
  return res;
}

template <class R>
SolveResult gpu_solve_adjoint(lbgpu_engine* e, StateField<R>& v, const AdjointSolveOptions<R>& opt) {
  int64_t it = 0;
  double r = 0.0;
  int conv = 0;
  gpu_check(e, lbgpu_solve_adjoint(e, opt.tol, opt.max_iter, opt.fixed_iters,
                                   opt.kernel == AdjointKernel::DualSweep ? 1 : 0, &it, &r, &conv));
  download(e, 1, v);
  SolveResult res;
  res.converged = conv != 0, res.iterations = long(it), res.residual = r;
  return res;
}

GradientVector gpu_param_gradient(lbgpu_engine* e, AdjointKernel kernel) {
  int dims[8];
  int64_t counts[4];
  gpu_check(e, lbgpu_info(e, dims, counts));
  GradientVector g;
  g.design.resize(std::size_t(counts[1]));
  double gdp = 0.0;
  gpu_check(e, lbgpu_param_gradient(e, kernel == AdjointKernel::DualSweep ? 1 : 0,
                                    g.design.data(), &gdp));
  g.globals.emplace_back("inlet_dp", gdp);
  return g;
}

double gpu_evaluate_raw(lbgpu_engine* e) {
  double J = 0.0;
  gpu_check(e, lbgpu_objective(e, &J));
  return J;
}

template <class R>
GradientVector gpu_mma_iteration(lbgpu_engine* e, const std::vector<double>& w_design,
                                 const SolveOptions<R>& popt, SolveResult* primal) {
  gpu_check(e, lbgpu_set_design_values(e, w_design.data()));
  int64_t it = 0, ia = 0;
  double r = 0.0, ra = 0.0;
  int conv = 0, ca = 0;
  gpu_check(e, lbgpu_solve_primal(e, popt.tol, popt.max_iter, popt.fixed_iters, &it, &r, &conv));
  gpu_check(e, lbgpu_solve_adjoint(e, popt.tol, popt.max_iter, it, 0, &ia, &ra, &ca));
  if (primal) primal->converged = conv != 0, primal->iterations = long(it), primal->residual = r;
  return gpu_param_gradient(e, AdjointKernel::Analytic);
}

template SolveResult gpu_solve_fixed_point<double>(lbgpu_engine*, StateField<double>&,
                                                   const SolveOptions<double>&);
template SolveResult gpu_solve_fixed_point<float>(lbgpu_engine*, StateField<float>&,
                                                  const SolveOptions<float>&);
template SolveResult gpu_solve_adjoint<double>(lbgpu_engine*, StateField<double>&,
                                               const AdjointSolveOptions<double>&);
template SolveResult gpu_solve_adjoint<float>(lbgpu_engine*, StateField<float>&,
                                              const AdjointSolveOptions<float>&);
template GradientVector gpu_mma_iteration<double>(lbgpu_engine*, const std::vector<double>&,
                                                  const SolveOptions<double>&, SolveResult*);

}  // namespace lbopt

// The reference's case-level C API (lbopt.h) on the B200 engine — SURVEY.md
// §8f row F1. Each operation follows the reference's Case driver
// (proj/src/case.cpp) step for step, but every solve, sweep, gradient and
// reduction runs through the thin engine ABI (include/lbgpu.h); output files
// follow proj/src/io.cpp byte for byte (17-significant-digit CSV, legacy VTK).
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <limits>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lbgpu.h"
#include "../../include/lbopt_gpu.h"
#include "casebuild.h"

namespace {

using lbgpu::CaseSpec;
using lbgpu::SystemArrays;

// Error families of the reference (errors.hpp:11-33) -> status codes (capi.cpp:39-59).
struct CaseFail {
  int code;
  std::string msg;
};
[[noreturn]] void fail(int code, const std::string& m) { throw CaseFail{code, m}; }

constexpr double kNaN = std::numeric_limits<double>::quiet_NaN();

std::string g17(double v) {  // io.cpp:13-18
  if (std::isnan(v)) return "";
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

struct Row {  // RunRow (run_record.hpp:11-19)
  long iteration = 0;
  double residual = kNaN, objective = kNaN, penalty = kNaN, weight = kNaN, composite = kNaN,
         grad_norm = kNaN;
};

struct Solve {
  bool converged = false;
  long iterations = 0;
  double residual = 0.0;
};

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

}  // namespace

struct lbopt_case {
  CaseSpec cfg;
  bool dirty = false;
  SystemArrays sys;
  std::vector<int64_t> design;  // DesignField::nodes
  lbgpu_engine* e = nullptr;
  bool has_primal = false;
  int mf = 0, mt = 0, m = 0;
  long n = 0;
  std::string error;
  // Status (case.hpp:94-101)
  double objective = kNaN, residual = kNaN, cost_ratio = kNaN, max_rel_err = kNaN;
  long iterations = 0;
  bool converged = false;

  explicit lbopt_case(const CaseSpec& c) : cfg(c) { rebuild(); }
  ~lbopt_case() { lbgpu_destroy(e); }

  // ------------------------------------------------------------ engine
  lbgpu_system_desc desc(const SystemArrays& s, double inlet_dp) const {
    lbgpu_system_desc d{};
    d.nx = cfg.nx, d.ny = cfg.ny, d.nz = cfg.nz;
    d.precision = cfg.precision;
    d.exact = env_int("LBOPT_GPU_EXACT", 0) && cfg.precision == 64;
    d.device = env_int("LBOPT_GPU_DEVICE", 0);
    d.collision = cfg.collision == "bgk" ? 1 : 0;
    d.nu = cfg.nu, d.beta_fluid = cfg.beta_fluid, d.beta_solid = cfg.beta_solid;
    d.inlet_dp = inlet_dp, d.u_clamp = cfg.u_clamp, d.omega_nonhydro = cfg.omega_nonhydro;
    d.switch_theta = cfg.switch_theta;
    d.switch_form = cfg.switch_form == "fluid_power" ? 1 : 0;
    d.tag = s.tag.data(), d.bc_T = s.bc_T.data(), d.bc_axis = s.bc_axis.data();
    d.bc_sign = s.bc_sign.data(), d.w = s.w.data(), d.design_mask = s.mask.data();
    d.obj_kind = s.obj_kind, d.flux_axis = s.flux_axis, d.flux_sign = s.flux_sign;
    d.support = s.support.data(), d.n_support = (int64_t)s.support.size();
    return d;
  }
  lbgpu_engine* make_engine(const SystemArrays& s, double inlet_dp) const {
    const lbgpu_system_desc d = desc(s, inlet_dp);
    lbgpu_engine* x = nullptr;
    const int rc = lbgpu_create(&d, &x);
    if (rc) fail(rc, lbgpu_last_create_error());
    return x;
  }
  void ok(lbgpu_engine* x, int rc) const {
    if (rc) fail(rc, lbgpu_error_message(x));
  }

  // Case::rebuild (case.cpp:35-41): validated config -> System -> engine.
  void rebuild() {
    std::string err;
    if (!lbgpu::check_case(cfg, err)) fail(LBOPT_E_CONFIG, err);
    SystemArrays s;
    if (!lbgpu::build_system(cfg, s, err)) fail(LBOPT_E_CONFIG, err);
    lbgpu_engine* x = make_engine(s, cfg.inlet_dp);
    lbgpu_destroy(e);
    e = x;
    sys = std::move(s);
    design.clear();
    for (long i = 0; i < (long)sys.mask.size(); ++i)
      if (sys.mask[i]) design.push_back(i);
    mf = cfg.nz == 1 ? 9 : 19;
    mt = cfg.nz == 1 ? 9 : 7;
    m = mf + mt;
    n = long(cfg.nx) * cfg.ny * cfg.nz;
    has_primal = false;
    objective = residual = cost_ratio = max_rel_err = kNaN;
    iterations = 0;
    converged = false;
  }
  void ensure_built() {  // case.cpp:47-52
    if (!dirty) return;
    std::string err;
    if (!lbgpu::check_case(cfg, err)) fail(LBOPT_E_CONFIG, err);
    rebuild();
    dirty = false;
  }

  // ------------------------------------------------------------ helpers
  std::string out_path(const std::string& name) const {  // case.cpp:62-67
    std::error_code ec;
    std::filesystem::create_directories(cfg.out_dir, ec);
    if (ec) fail(LBOPT_E_IO, "cannot create output directory: " + cfg.out_dir);
    return cfg.out_dir + "/" + name;
  }
  int kernel() const { return cfg.adjoint_kernel == "dual" ? 1 : 0; }
  double evaluate() {
    double v = 0;
    ok(e, lbgpu_objective(e, &v));
    return v;
  }
  std::vector<double> state(int field) {
    std::vector<double> s(size_t(m) * n);
    ok(e, lbgpu_download_state(e, field, s.data()));
    return s;
  }
  std::vector<double> design_full() {
    std::vector<double> w(n);
    ok(e, lbgpu_get_design(e, w.data()));
    return w;
  }
  // PenaltySchedule::weight_at (objective.cpp:91-97)
  double weight_at(long it) const {
    if (cfg.penalty_w0 <= 0.0 || it < cfg.penalty_start) return 0.0;
    const double expo = double(it - cfg.penalty_start) / double(cfg.penalty_interval);
    double w = cfg.penalty_w0 * std::pow(cfg.penalty_growth, expo);
    if (cfg.penalty_cap > 0.0 && w > cfg.penalty_cap) w = cfg.penalty_cap;
    return w;
  }
  double penalty() {
    double p = 0;
    ok(e, lbgpu_penalty(e, &p));
    return p;
  }

  // solve_fixed_point (collision.cpp:377-416) from the current state, rows at
  // it % record_interval == 0 and at the end (the monitor is evaluate_raw;
  // the partitioned solver records no objective, partition.cpp:295-300).
  Solve solve_primal(double tol, long max_iter, long ri, std::vector<Row>* rows, bool monitor) {
    Solve res;
    long it = 0;
    for (;;) {
      const long chunk = rows ? std::min(ri - it % ri, max_iter - it) : max_iter - it;
      int64_t k = 0;
      double r = 0;
      int cv = 0;
      ok(e, lbgpu_solve_primal(e, tol, chunk, -1, &k, &r, &cv));
      it += k;
      res.iterations = it;
      res.residual = r;
      const bool done = r <= tol || it == max_iter;
      if (rows && (it % ri == 0 || done)) {
        Row row;
        row.iteration = it;
        row.residual = r;
        if (monitor) row.objective = evaluate();
        rows->push_back(row);
      }
      if (done) break;
    }
    res.converged = res.residual <= tol;
    return res;
  }
  // solve_adjoint (adjoint.cpp:256-297): v <- 0, rows at it % ri == 0, at the
  // last iteration and at the stop.
  Solve solve_adjoint(double tol, long max_iter, long fixed, long ri, std::vector<Row>* rows) {
    ok(e, lbgpu_reset_adjoint(e));
    Solve res;
    const long nmax = fixed >= 0 ? fixed : max_iter;
    long it = 0;
    while (it < nmax) {
      const long chunk = rows ? std::min(ri - it % ri, nmax - it) : nmax - it;
      int64_t k = 0;
      double r = 0;
      int cv = 0;
      ok(e, lbgpu_continue_adjoint(e, tol, chunk, fixed >= 0 ? chunk : -1, kernel(), &k, &r, &cv));
      it += k;
      res.iterations = it;
      res.residual = r;
      const bool stop = fixed < 0 && r <= tol;
      if (rows && (it % ri == 0 || it == nmax || r <= tol)) {
        Row row;
        row.iteration = it;
        row.residual = r;
        rows->push_back(row);
      }
      if (stop) break;
    }
    res.converged = res.residual <= tol;
    return res;
  }

  // ------------------------------------------------------------ writers (io.cpp)
  std::ofstream open_out(const std::string& path) const {
    std::ofstream out(path);
    if (!out) fail(LBOPT_E_IO, "cannot open for writing: " + path);
    return out;
  }
  void closed(std::ofstream& out, const std::string& path) const {
    if (!out) fail(LBOPT_E_IO, "write failed: " + path);
  }
  void xyz(long i, int& x, int& y, int& z) const {
    x = int(i % cfg.nx);
    y = int((i / cfg.nx) % cfg.ny);
    z = int(i / (long(cfg.nx) * cfg.ny));
  }
  struct FieldRow {
    double rho, ux, uy, uz, T, w;
  };
  // node_fields (io.cpp:71-96): flow_moments / thermal_moment in the state's
  // precision, NumericError on rho <= 0.
  template <class R>
  std::vector<FieldRow> field_table_r(const std::vector<double>& st, const std::vector<double>& w) {
    static const int E2[9][2] = {{0, 0}, {1, 0}, {-1, 0}, {0, 1}, {0, -1}, {1, 1}, {-1, 1}, {1, -1}, {-1, -1}};
    static const int E3[19][3] = {{0, 0, 0},  {1, 0, 0},  {-1, 0, 0},  {0, 1, 0},  {0, -1, 0},
                                  {0, 0, 1},  {0, 0, -1}, {1, 1, 0},   {-1, 1, 0}, {1, -1, 0},
                                  {-1, -1, 0}, {1, 0, 1}, {-1, 0, 1},  {1, 0, -1}, {-1, 0, -1},
                                  {0, 1, 1},  {0, -1, 1}, {0, 1, -1},  {0, -1, -1}};
    std::vector<FieldRow> rows(n);
    for (long i = 0; i < n; ++i) {
      R rho = R(0), q[3] = {R(0), R(0), R(0)};
      for (int j = 0; j < mf; ++j) {
        const R fj = R(st[size_t(j) * n + i]);
        rho += fj;
        for (int a = 0; a < 3; ++a) {
          const int ea = cfg.nz == 1 ? (a < 2 ? E2[j][a] : 0) : E3[j][a];
          if (ea) q[a] += R(double(ea)) * fj;
        }
      }
      if (!(rho > R(0))) fail(LBOPT_E_NUMERIC, "non-positive density");
      R T = R(0);
      for (int j = 0; j < mt; ++j) T += R(st[size_t(mf + j) * n + i]);
      rows[i] = {double(rho), double(q[0] / rho), double(q[1] / rho), double(q[2] / rho),
                 double(T), w[i]};
    }
    return rows;
  }
  std::vector<FieldRow> field_table() {
    const auto st = state(0);
    const auto w = design_full();
    return cfg.precision == 32 ? field_table_r<float>(st, w) : field_table_r<double>(st, w);
  }
  void write_fields_csv(const std::vector<FieldRow>& t, const std::string& path) {
    auto out = open_out(path);
    out << "x,y,z,rho,ux,uy,uz,T,w\n";
    for (long i = 0; i < n; ++i) {
      int x, y, z;
      xyz(i, x, y, z);
      const FieldRow& r = t[i];
      out << x << ',' << y << ',' << z << ',' << g17(r.rho) << ',' << g17(r.ux) << ','
          << g17(r.uy) << ',' << g17(r.uz) << ',' << g17(r.T) << ',' << g17(r.w) << '\n';
    }
    closed(out, path);
  }
  void write_fields_vtk(const std::vector<FieldRow>& t, const std::string& path) {
    auto out = open_out(path);
    out << "# vtk DataFile Version 3.0\nmacroscopic fields\nASCII\nDATASET STRUCTURED_POINTS\n";
    out << "DIMENSIONS " << cfg.nx << ' ' << cfg.ny << ' ' << cfg.nz << '\n';
    out << "ORIGIN 0 0 0\nSPACING 1 1 1\n";
    out << "POINT_DATA " << n << '\n';
    auto scalars = [&](const char* name, auto get) {
      out << "SCALARS " << name << " double 1\nLOOKUP_TABLE default\n";
      for (const FieldRow& r : t) out << g17(get(r)) << '\n';
    };
    scalars("rho", [](const FieldRow& r) { return r.rho; });
    out << "VECTORS velocity double\n";
    for (const FieldRow& r : t) out << g17(r.ux) << ' ' << g17(r.uy) << ' ' << g17(r.uz) << '\n';
    scalars("T", [](const FieldRow& r) { return r.T; });
    scalars("w", [](const FieldRow& r) { return r.w; });
    closed(out, path);
  }
  void write_state_csv(const std::string& path) {
    const auto st = state(0);
    auto out = open_out(path);
    out << "x,y,z";
    for (int j = 1; j <= m; ++j) out << ",f_" << j;
    out << '\n';
    for (long i = 0; i < n; ++i) {
      int x, y, z;
      xyz(i, x, y, z);
      out << x << ',' << y << ',' << z;
      for (int j = 0; j < m; ++j) out << ',' << g17(st[size_t(j) * n + i]);
      out << '\n';
    }
    closed(out, path);
  }
  void write_design_csv(const std::string& path) {
    const auto w = design_full();
    auto out = open_out(path);
    out << "x,y,z,w\n";
    for (long i = 0; i < n; ++i) {
      int x, y, z;
      xyz(i, x, y, z);
      out << x << ',' << y << ',' << z << ',' << g17(w[i]) << '\n';
    }
    closed(out, path);
  }
  void write_record_csv(const std::vector<Row>& rows, const std::string& path) {
    auto out = open_out(path);
    out << "iter,residual,objective,penalty,weight,composite,grad_norm\n";
    for (const Row& r : rows)
      out << r.iteration << ',' << g17(r.residual) << ',' << g17(r.objective) << ','
          << g17(r.penalty) << ',' << g17(r.weight) << ',' << g17(r.composite) << ','
          << g17(r.grad_norm) << '\n';
    closed(out, path);
  }
  void write_convergence_csv(const std::vector<Row>& rows, const std::string& path) {
    auto out = open_out(path);
    out << "iter,objective,penalty,weight,composite\n";
    for (const Row& r : rows)
      out << r.iteration << ',' << g17(r.objective) << ',' << g17(r.penalty) << ','
          << g17(r.weight) << ',' << g17(r.composite) << '\n';
    closed(out, path);
  }
  void write_gradient_csv(const std::vector<double>& g, double gdp, const std::string& path) {
    auto out = open_out(path);
    out << "x,y,z,dF_dw,name\n";
    for (size_t k = 0; k < g.size(); ++k) {
      int x, y, z;
      xyz(design[k], x, y, z);
      out << x << ',' << y << ',' << z << ',' << g17(g[k]) << ",\n";
    }
    out << "-1,-1,-1," << g17(gdp) << ",inlet_dp\n";
    closed(out, path);
  }
  void write_fields_outputs(const std::string& stem_csv, const std::string& stem_vtk) {
    if (stem_csv.empty() && stem_vtk.empty()) return;
    const auto t = field_table();
    if (!stem_csv.empty()) write_fields_csv(t, stem_csv);
    if (!stem_vtk.empty()) write_fields_vtk(t, stem_vtk);
  }

  void set_status(const Solve& s, double obj) {
    objective = obj;
    iterations = s.iterations;
    converged = s.converged;
    residual = s.residual;
  }

  // ------------------------------------------------------------ operations
  void simulate() {  // case.cpp:75-113
    ok(e, lbgpu_init_state(e));
    std::vector<Row> rows;
    const Solve sr = solve_primal(cfg.primal_tol, cfg.max_inner, cfg.record_interval, &rows,
                                  cfg.workers <= 1);
    has_primal = true;
    if (cfg.write_csv) {
      write_fields_outputs(out_path("fields.csv"), "");
      write_state_csv(out_path("state.csv"));
      write_record_csv(rows, out_path("record.csv"));
    }
    if (cfg.write_vtk) write_fields_outputs("", out_path("fields.vtk"));
    set_status(sr, evaluate());
  }

  void run_adjoint() {  // case.cpp:122-153
    if (!has_primal) fail(LBOPT_E_STATE, "adjoint needs a primal state: run simulate or load one first");
    std::vector<Row> rows;
    const Solve ar = solve_adjoint(cfg.adjoint_tol, cfg.max_inner, -1, cfg.record_interval, &rows);
    std::vector<double> g(design.size());
    double gdp = 0;
    ok(e, lbgpu_param_gradient(e, kernel(), g.data(), &gdp));
    if (cfg.write_csv) {
      write_gradient_csv(g, gdp, out_path("gradient.csv"));
      write_record_csv(rows, out_path("adjoint_record.csv"));
    }
    set_status(ar, evaluate());
  }

  // mma_update (optimizer.cpp:78-138): Svanberg asymptotes in the [0,1] box.
  struct Mma {
    long iter = 0;
    std::vector<double> x_prev, x_prev2, low, upp;
  };
  std::vector<double> mma_update(const std::vector<double>& x, const std::vector<double>& grad,
                                 Mma& st) const {
    const double asy_init = 0.5, asy_expand = 1.2, asy_contract = 0.7;
    const size_t nn = x.size();
    if (st.low.size() != nn) st.low.assign(nn, 0.0), st.upp.assign(nn, 0.0);
    for (size_t i = 0; i < nn; ++i) {
      if (st.iter < 2) {
        st.low[i] = x[i] - asy_init;
        st.upp[i] = x[i] + asy_init;
      } else {
        const double osc = (x[i] - st.x_prev[i]) * (st.x_prev[i] - st.x_prev2[i]);
        const double gm = osc > 0 ? asy_expand : (osc < 0 ? asy_contract : 1.0);
        st.low[i] = x[i] - gm * (st.x_prev[i] - st.low[i]);
        st.upp[i] = x[i] + gm * (st.upp[i] - st.x_prev[i]);
      }
      st.low[i] = std::clamp(st.low[i], x[i] - 10.0, x[i] - 0.01);
      st.upp[i] = std::clamp(st.upp[i], x[i] + 0.01, x[i] + 10.0);
    }
    std::vector<double> xn(nn);
    for (size_t i = 0; i < nn; ++i) {
      const double L = st.low[i], U = st.upp[i];
      const double lo = std::max({0.0, L + 0.1 * (x[i] - L), x[i] - cfg.move_limit});
      const double hi = std::min({1.0, U - 0.1 * (U - x[i]), x[i] + cfg.move_limit});
      const double gm = -grad[i];
      const double p = (U - x[i]) * (U - x[i]) * (1.001 * std::max(gm, 0.0) + 0.001 * std::max(-gm, 0.0));
      const double q = (x[i] - L) * (x[i] - L) * (0.001 * std::max(gm, 0.0) + 1.001 * std::max(-gm, 0.0));
      double xi = x[i];
      if (!(p == 0.0 && q == 0.0)) {
        const double sp = std::sqrt(p), sq = std::sqrt(q);
        xi = (L * sp + U * sq) / (sp + sq);
      }
      xn[i] = std::clamp(xi, lo, hi);
    }
    st.x_prev2 = st.iter >= 1 ? st.x_prev : x;
    st.x_prev = x;
    ++st.iter;
    return xn;
  }

  void optimize() {  // case.cpp:162-220
    ok(e, lbgpu_init_state(e));
    ok(e, lbgpu_reset_adjoint(e));
    std::vector<Row> rows;
    auto snapshot = [&](long k) {
      if (!cfg.write_csv) return;
      char a[64], b[64];
      std::snprintf(a, sizeof a, "design_%06ld.csv", k);
      std::snprintf(b, sizeof b, "fields_%06ld.csv", k);
      write_design_csv(out_path(a));
      write_fields_outputs(out_path(b), "");
    };
    Solve s_out;
    long iters_out = 0;
    bool conv_out = false;
    if (cfg.method == "oneshot") {
      std::vector<std::pair<long, double>> stages;
      std::string err;
      if (!lbgpu::zeta_stages(cfg, stages, err)) fail(LBOPT_E_CONFIG, err);
      const long N = cfg.iterations, si = std::max<long>(N / 5, 1);
      long it = 1;
      while (it <= N) {
        const long stop = std::min(N, (it + si - 1) / si * si);  // next snapshot iteration
        const long cnt = stop - it + 1;
        std::vector<double> zeta(cnt), lam(cnt);
        for (long k = 0; k < cnt; ++k) {
          double z = 0.0;  // zeta_at (optimizer.cpp:18-23)
          for (const auto& s : stages)
            if (it + k >= s.first) z = s.second;
          zeta[k] = z;
          lam[k] = weight_at(it + k);
        }
        std::vector<lbgpu_run_row> rr(size_t(cnt / cfg.record_interval + 2));
        int64_t nr = 0;
        ok(e, lbgpu_one_shot_range(e, it, cnt, N, zeta.data(), lam.data(), cfg.record_interval,
                                   rr.data(), (int64_t)rr.size(), &nr));
        for (int64_t k = 0; k < nr; ++k)
          rows.push_back({long(rr[k].iteration), rr[k].residual, rr[k].objective, rr[k].penalty,
                          rr[k].penalty_weight, rr[k].composite, rr[k].grad_norm});
        if (stop % si == 0 || stop == N) snapshot(stop);
        it = stop + 1;
      }
      iters_out = N;
    } else if (cfg.method == "mma") {  // mma_run (optimizer.cpp:140-212)
      long primal_steps = 0;
      bool all_conv = true;
      const long outers = cfg.outer_iterations, si = std::max<long>(outers / 5, 1);
      auto record = [&](long outer, const Solve& pr, double gn) {
        Row row;
        row.iteration = outer;
        row.residual = pr.residual;
        row.objective = evaluate();
        row.penalty = penalty();
        row.weight = weight_at(primal_steps);
        row.composite = row.objective - row.weight * row.penalty;
        row.grad_norm = gn;
        rows.push_back(row);
      };
      Solve pr = solve_primal(cfg.primal_tol, cfg.max_inner, 1, nullptr, false);
      primal_steps += pr.iterations;
      all_conv = all_conv && pr.converged;
      record(0, pr, kNaN);
      Mma st;
      std::vector<double> x(design.size()), comp(design.size()), g(design.size());
      for (long outer = 1; outer <= outers; ++outer) {
        const long fixed = cfg.adjoint_stop == "match" ? std::max<long>(pr.iterations, 1) : -1;
        solve_adjoint(cfg.adjoint_tol, cfg.max_inner, fixed, 1, nullptr);
        double gdp = 0;
        ok(e, lbgpu_param_gradient(e, kernel(), g.data(), &gdp));
        const double lambda = weight_at(primal_steps);
        ok(e, lbgpu_get_design_values(e, x.data()));
        double gn = 0.0;
        for (size_t i = 0; i < x.size(); ++i) {
          comp[i] = g[i];
          if (lambda != 0.0) comp[i] -= lambda * (1.0 - 2.0 * x[i]);
          gn = std::max(gn, std::abs(comp[i]));
        }
        const std::vector<double> xn = mma_update(x, comp, st);
        ok(e, lbgpu_set_design_values(e, xn.data()));
        pr = solve_primal(cfg.primal_tol, cfg.max_inner, 1, nullptr, false);
        primal_steps += pr.iterations;
        all_conv = all_conv && pr.converged;
        record(outer, pr, gn);
        if (outer % si == 0 || outer == outers) snapshot(outer);
      }
      iters_out = primal_steps;
      conv_out = all_conv;
    } else {
      fail(LBOPT_E_CONFIG, "optimize needs [optimizer] method = oneshot or mma");
    }
    // converged objective of the final design (one-shot leaves the state mid-flight)
    const Solve fr = solve_primal(cfg.primal_tol, cfg.max_inner, 1, nullptr, false);
    has_primal = true;
    if (cfg.write_csv) {
      write_design_csv(out_path("design.csv"));
      write_fields_outputs(out_path("fields.csv"), "");
      write_state_csv(out_path("state.csv"));
      write_convergence_csv(rows, out_path("convergence.csv"));
      write_record_csv(rows, out_path("optimize_record.csv"));
    }
    if (cfg.write_vtk) write_fields_outputs("", out_path("fields.vtk"));
    s_out = fr;
    s_out.iterations = iters_out;
    if (cfg.method == "oneshot") conv_out = fr.converged;
    s_out.converged = conv_out;
    set_status(s_out, evaluate());
  }

  // fd_gradient (adjoint.cpp:491-516): two cold-start fixed-iteration solves.
  double fd_gradient(long ordinal, double h, long fixed) {
    auto run = [&](double delta) {
      SystemArrays s = sys;
      double dp = cfg.inlet_dp;
      if (ordinal < 0) dp += delta;
      else s.w[design[ordinal]] = ensure_w(ordinal) + delta;  // raw write: FD probes do not clamp
      lbgpu_engine* x = make_engine(s, dp);
      double obj = 0;
      int64_t k = 0;
      double r = 0;
      int cv = 0;
      int rc = lbgpu_solve_primal(x, cfg.primal_tol, cfg.max_inner, fixed, &k, &r, &cv);
      if (!rc) rc = lbgpu_objective(x, &obj);
      const std::string msg = rc ? lbgpu_error_message(x) : "";
      lbgpu_destroy(x);
      if (rc) fail(rc, msg);
      return obj;
    };
    const double fp = run(+h), fm = run(-h);
    return (fp - fm) / (2.0 * h);
  }
  std::vector<double> w_now;
  double ensure_w(long ordinal) { return w_now[design[ordinal]]; }

  void grad_check(double* out_err) {  // case.cpp:229-329
    ok(e, lbgpu_init_state(e));
    const Solve pr = solve_primal(cfg.primal_tol, cfg.max_inner, 1, nullptr, false);
    if (!pr.converged) {
      char b[64];
      std::snprintf(b, sizeof b, "%f", cfg.primal_tol);
      fail(LBOPT_E_NUMERIC, std::string("gradient check: primal did not reach tol ") + b);
    }
    has_primal = true;
    const Solve ar = solve_adjoint(cfg.adjoint_tol, cfg.max_inner, -1, 1, nullptr);
    if (!ar.converged) {
      char b[64];
      std::snprintf(b, sizeof b, "%f", cfg.adjoint_tol);
      fail(LBOPT_E_NUMERIC, std::string("gradient check: adjoint did not reach tol ") + b);
    }
    std::vector<double> g(design.size());
    double gdp = 0;
    ok(e, lbgpu_param_gradient(e, kernel(), g.data(), &gdp));
    if (design.empty()) fail(LBOPT_E_CONFIG, "gradient check needs a design region");
    w_now = design_full();
    std::vector<size_t> ord(g.size());
    std::iota(ord.begin(), ord.end(), size_t{0});
    std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
      const double ga = std::abs(g[a]), gb = std::abs(g[b]);
      return ga != gb ? ga > gb : a < b;
    });
    const size_t n_pick = std::min<size_t>(g.size(), 12);
    double g_scale = 0.0;
    for (size_t k = 0; k < n_pick; ++k) g_scale = std::max(g_scale, std::abs(g[ord[k]]));
    g_scale = std::max(g_scale, std::abs(gdp));
    const double steps[] = {1e-5, 1e-6, 1e-7};
    auto rel = [&](double adj, double fd) {
      const double den = std::max({std::abs(adj), std::abs(fd), 1e-6 * g_scale, 1e-300});
      return std::abs(fd - adj) / den;
    };
    struct GRow {
      bool global;
      int x, y, z;
      double adjoint, fd, rel_err, step;
    };
    std::vector<GRow> rows;
    double max_err = 0.0;
    auto check = [&](long ordinal, double adj, GRow row) {
      row.adjoint = adj;
      row.rel_err = std::numeric_limits<double>::infinity();
      for (double h : steps) {
        const double fd = fd_gradient(ordinal, h, pr.iterations);
        const double err = rel(adj, fd);
        if (err < row.rel_err) row.rel_err = err, row.fd = fd, row.step = h;
      }
      max_err = std::max(max_err, row.rel_err);
      rows.push_back(row);
    };
    for (size_t k = 0; k < n_pick; ++k) {
      GRow row{false, 0, 0, 0, 0, 0, 0, 0};
      xyz(design[ord[k]], row.x, row.y, row.z);
      check(long(ord[k]), g[ord[k]], row);
    }
    check(-1, gdp, GRow{true, -1, -1, -1, 0, 0, 0, 0});
    if (cfg.write_csv) {
      const std::string path = out_path("gradcheck.csv");
      auto out = open_out(path);
      out << "name,x,y,z,adjoint,fd,rel_err,step\n";
      for (const GRow& r : rows)
        out << (r.global ? "inlet_dp" : "w") << ',' << r.x << ',' << r.y << ',' << r.z << ','
            << g17(r.adjoint) << ',' << g17(r.fd) << ',' << g17(r.rel_err) << ',' << g17(r.step)
            << '\n';
      closed(out, path);
    }
    max_rel_err = max_err;
    iterations = pr.iterations;
    converged = true;
    residual = pr.residual;
    objective = evaluate();
    if (out_err) *out_err = max_err;
  }

  void threshold(double* best_eta, double* best_obj) {  // case.cpp:333-347, optimizer.cpp:214-246
    const int P = cfg.threshold_points;
    const auto w = design_full();
    struct Pt {
      double eta, obj;
      bool conv;
    };
    std::vector<Pt> pts;
    bool any = false;
    double beta = 0.0, bobj = 0.0;
    for (int i = 0; i < P; ++i) {
      const double eta = double(i) / (P - 1);
      SystemArrays s = sys;
      s.w = w;
      for (int64_t k : design) s.w[k] = w[k] >= eta ? 1.0 : 0.0;
      lbgpu_engine* x = make_engine(s, cfg.inlet_dp);
      int64_t it = 0;
      double r = 0;
      int cv = 0;
      Pt pt{eta, 0.0, false};
      if (lbgpu_solve_primal(x, cfg.primal_tol, cfg.max_inner, -1, &it, &r, &cv) == LBGPU_OK) {
        pt.conv = cv != 0;
        if (pt.conv && lbgpu_objective(x, &pt.obj) != LBGPU_OK) pt.conv = false;
      }
      lbgpu_destroy(x);
      if (pt.conv && (!any || pt.obj > bobj)) any = true, bobj = pt.obj, beta = eta;
      pts.push_back(pt);
    }
    if (cfg.write_csv) {
      const std::string path = out_path("threshold.csv");
      auto out = open_out(path);
      out << "eta,objective\n";
      for (const Pt& p : pts) out << g17(p.eta) << ',' << (p.conv ? g17(p.obj) : "") << '\n';
      closed(out, path);
    }
    objective = bobj;
    converged = any;
    if (best_eta) *best_eta = beta;
    if (best_obj) *best_obj = bobj;
  }

  // workers -> GPUs: worker i runs on device
  // (LBOPT_GPU_DEVICE + i) mod G, G = LBOPT_GPU_COUNT or every visible GPU;
  // the slabs form a P2P group (peer stores across GPUs, concurrent streams
  // when several share one).
  static int worker_device(int i) {
    const int d0 = env_int("LBOPT_GPU_DEVICE", 0);
    int g = env_int("LBOPT_GPU_COUNT", 0);
    const int vis = lbgpu_device_count();
    if (g <= 0 || g > vis) g = vis;
    if (g <= 0) return d0;
    return (d0 + i) % g;
  }

  // partition_check (partition.cpp:314-357) against the engine's slab groups.
  void partition_check(long steps, double* max_diff) {
    const std::string text = lbgpu::serialize_case(cfg);
    const int W = cfg.workers;
    std::vector<lbgpu_engine*> slabs(W, nullptr);
    lbgpu_engine* mono = make_engine(sys, cfg.inlet_dp);
    auto cleanup = [&] {
      for (auto* s : slabs) lbgpu_destroy(s);
      lbgpu_destroy(mono);
    };
    try {
      const int ex = env_int("LBOPT_GPU_EXACT", 0);
      for (int i = 0; i < W; ++i) {
        const int rc = lbgpu_create_slab_from_config(text.c_str(), "", worker_device(i),
                                                     ex && cfg.precision == 64, W, i, &slabs[i]);
        if (rc) fail(rc, lbgpu_last_create_error());
      }
      if (W > 1) ok(slabs[0], lbgpu_group_link_p2p(slabs.data(), W));
      std::vector<int> geo(6 * W);
      for (int i = 0; i < W; ++i) lbgpu_slab_info(slabs[i], geo.data() + 6 * i);
      auto gathered = [&](int field) {
        std::vector<double> out(size_t(m) * n);
        for (int i = 0; i < W; ++i) {
          const int x0 = geo[6 * i + 1], span = geo[6 * i + 2], nxl = geo[6 * i + 3];
          std::vector<double> loc(size_t(m) * nxl * cfg.ny * cfg.nz);
          ok(slabs[i], lbgpu_download_state(slabs[i], field, loc.data()));
          const long rows = long(cfg.ny) * cfg.nz;
          for (int p = 0; p < m; ++p)
            for (long r = 0; r < rows; ++r)
              for (int lx = 0; lx < span; ++lx)
                out[size_t(p) * n + r * cfg.nx + x0 + lx] =
                    loc[size_t(p) * nxl * rows + r * nxl + lx];
        }
        return out;
      };
      auto diff = [](const std::vector<double>& a, const std::vector<double>& b) {
        double d = 0.0;
        for (size_t i = 0; i < a.size(); ++i) {
          const double x = std::abs(a[i] - b[i]);
          if (!(x <= d)) d = x;
        }
        return d;
      };
      double dp = 0.0, da = 0.0;
      for (long it = 0; it < steps; ++it) {
        ok(mono, lbgpu_primal_step(mono, 1, nullptr));
        ok(slabs[0], lbgpu_group_step(slabs.data(), W, 0, 1, 0, nullptr));
        std::vector<double> ms(size_t(m) * n);
        ok(mono, lbgpu_download_state(mono, 0, ms.data()));
        const double d = diff(ms, gathered(0));
        if (!(d <= dp)) dp = d;
      }
      for (long it = 0; it < steps; ++it) {
        ok(mono, lbgpu_adjoint_step(mono, 1, 0, nullptr));
        ok(slabs[0], lbgpu_group_step(slabs.data(), W, 1, 1, 0, nullptr));
        std::vector<double> ms(size_t(m) * n);
        ok(mono, lbgpu_download_state(mono, 1, ms.data()));
        const double d = diff(ms, gathered(1));
        if (!(d <= da)) da = d;
      }
      if (cfg.write_csv) {
        const std::string path = out_path("partition.csv");
        auto out = open_out(path);
        char buf[96];
        std::snprintf(buf, sizeof buf, "%ld,%.17g,%.17g\n", steps, dp, da);
        out << "steps,max_primal_diff,max_adjoint_diff\n" << buf;
        closed(out, path);
      }
      residual = std::max(dp, da);
      iterations = steps;
      if (max_diff) *max_diff = std::max(dp, da);
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  }

  void scaling(long steps) {  // case.cpp:369-382, partition.cpp:359-383
    std::vector<int> counts;
    for (int w = 1; w <= cfg.workers; w *= 2) counts.push_back(w);
    if (counts.empty() || counts.back() != cfg.workers) counts.push_back(cfg.workers);
    const std::string text = lbgpu::serialize_case(cfg);
    std::vector<std::array<double, 3>> rows;
    for (int W : counts) {
      std::vector<lbgpu_engine*> slabs(W, nullptr);
      auto cleanup = [&] {
        for (auto* s : slabs) lbgpu_destroy(s);
      };
      try {
        for (int i = 0; i < W; ++i) {
          const int rc = lbgpu_create_slab_from_config(text.c_str(), "", worker_device(i), 0, W, i, &slabs[i]);
          if (rc) fail(rc, lbgpu_last_create_error());
        }
        ok(slabs[0], W > 1 ? lbgpu_group_link_p2p(slabs.data(), W) : lbgpu_group_link(slabs.data(), W));
        using clk = std::chrono::steady_clock;
        const auto t0 = clk::now();
        ok(slabs[0], lbgpu_group_step(slabs.data(), W, 0, steps, 0, nullptr));
        const auto t1 = clk::now();
        ok(slabs[0], lbgpu_group_step(slabs.data(), W, 1, steps, 0, nullptr));
        const auto t2 = clk::now();
        rows.push_back({double(W), steps / std::chrono::duration<double>(t1 - t0).count(),
                        steps / std::chrono::duration<double>(t2 - t1).count()});
      } catch (...) {
        cleanup();
        throw;
      }
      cleanup();
    }
    if (cfg.write_csv) {
      const std::string path = out_path("scaling.csv");
      auto out = open_out(path);
      out << "workers,primal_steps_per_sec,adjoint_steps_per_sec,ratio\n";
      for (const auto& r : rows)
        out << int(r[0]) << ',' << g17(r[1]) << ',' << g17(r[2]) << ','
            << g17(r[2] > 0 ? r[1] / r[2] : kNaN) << '\n';
      closed(out, path);
    }
  }

  double cost_ratio_run(long steps) {  // case.cpp:393-414
    if (steps < 1) fail(LBOPT_E_CONFIG, "cost ratio needs at least one step");
    ok(e, lbgpu_init_state(e));
    using clk = std::chrono::steady_clock;
    ok(e, lbgpu_primal_step(e, 5, nullptr));
    auto t0 = clk::now();
    ok(e, lbgpu_primal_step(e, steps, nullptr));
    const double tp = std::chrono::duration<double>(clk::now() - t0).count();
    ok(e, lbgpu_reset_adjoint(e));
    ok(e, lbgpu_adjoint_step(e, 5, kernel(), nullptr));
    t0 = clk::now();
    ok(e, lbgpu_adjoint_step(e, steps, kernel(), nullptr));
    const double ta = std::chrono::duration<double>(clk::now() - t0).count();
    if (!(tp > 0)) fail(LBOPT_E_NUMERIC, "primal timing too short to resolve");
    cost_ratio = ta / tp;
    return cost_ratio;
  }

  void generate_fins(int count, int width) {  // case.cpp:418-446
    if (count < 1 || width < 1) fail(LBOPT_E_CONFIG, "fins: count and width must be positive");
    if (design.empty()) fail(LBOPT_E_CONFIG, "fins: case has no design region");
    auto w = design_full();
    for (int64_t i : design) w[i] = 1.0;
    const int x0 = cfg.design_x0, x1 = cfg.design_x1, span = x1 - x0 + 1;
    if (span < count * width) fail(LBOPT_E_CONFIG, "fins: design span too short for the requested comb");
    const int len = std::max(1, 2 * (cfg.ny - 2) / 3);
    for (int i = 0; i < count; ++i) {
      const double cx = x0 + (i + 0.5) * double(span) / count;
      const int fx0 = int(cx) - width / 2, fx1 = fx0 + width - 1;
      const bool bottom = i % 2 == 0;
      for (int64_t idx : design) {
        const int x = int(idx % cfg.nx);
        if (x < fx0 || x > fx1) continue;
        const int y = int((idx / cfg.nx) % cfg.ny);
        if (bottom ? y <= len : y >= cfg.ny - 1 - len) w[idx] = 0.0;
      }
    }
    ok(e, lbgpu_set_design(e, w.data()));
    has_primal = false;
  }

  // Case::apply_threshold_now (case.cpp:450-457) discards apply_threshold's
  // result: the design is left unchanged and only the
  // primal state is invalidated. Kept as is for drop-in fidelity.
  void apply_threshold_now(double) { has_primal = false; }

  void load_state(const std::string& path) {  // io.cpp:198-229
    std::ifstream in(path);
    if (!in) fail(LBOPT_E_IO, "cannot open for reading: " + path);
    std::string line;
    long ln = 1;
    if (!std::getline(in, line)) fail(LBOPT_E_IO, path + ": empty state file");
    auto split = [](const std::string& s) {
      std::vector<std::string> out;
      std::string cur;
      for (char ch : s) {
        if (ch == ',') out.push_back(cur), cur.clear();
        else if (ch != '\r') cur.push_back(ch);
      }
      out.push_back(cur);
      return out;
    };
    const auto hdr = split(line);
    if (int(hdr.size()) != 3 + m)
      fail(LBOPT_E_IO, path + ": state file has " + std::to_string(int(hdr.size()) - 3) +
                           " planes, case needs " + std::to_string(m));
    std::vector<double> st(size_t(m) * n, 0.0);
    long filled = 0;
    auto num = [&](const std::string& s) {
      if (s.empty()) return kNaN;
      try {
        size_t pos = 0;
        const double v = std::stod(s, &pos);
        if (pos != s.size()) throw std::invalid_argument(s);
        return v;
      } catch (const std::exception&) {
        fail(LBOPT_E_IO, path + ":" + std::to_string(ln) + ": bad numeric cell '" + s + "'");
      }
    };
    auto inum = [&](const std::string& s) {
      try {
        size_t pos = 0;
        const long v = std::stol(s, &pos);
        if (pos != s.size()) throw std::invalid_argument(s);
        return v;
      } catch (const std::exception&) {
        fail(LBOPT_E_IO, path + ":" + std::to_string(ln) + ": bad integer cell '" + s + "'");
      }
    };
    while (std::getline(in, line)) {
      ++ln;
      if (line.empty()) continue;
      const auto c = split(line);
      if (int(c.size()) != 3 + m) fail(LBOPT_E_IO, path + ":" + std::to_string(ln) + ": wrong cell count");
      const long x = inum(c[0]), y = inum(c[1]), z = inum(c[2]);
      if (x < 0 || x >= cfg.nx || y < 0 || y >= cfg.ny || z < 0 || z >= cfg.nz)
        fail(LBOPT_E_IO, path + ":" + std::to_string(ln) + ": node outside the lattice");
      const long idx = x + long(cfg.nx) * (y + long(cfg.ny) * z);
      for (int j = 0; j < m; ++j) {
        double v = num(c[3 + j]);
        if (cfg.precision == 32) v = double(float(v));
        st[size_t(j) * n + idx] = v;
      }
      ++filled;
    }
    if (filled != n)
      fail(LBOPT_E_IO, path + ": covers " + std::to_string(filled) + " of " + std::to_string(n) + " nodes");
    ok(e, lbgpu_upload_state(e, 0, st.data()));
    has_primal = true;
  }

  void load_design(const std::string& path) {  // io.cpp:231-260, topology.cpp:22-28
    std::ifstream in(path);
    if (!in) fail(LBOPT_E_IO, "cannot open for reading: " + path);
    std::string line;
    long ln = 1;
    if (!std::getline(in, line) || line.substr(0, line.find(',')) != "x")
      fail(LBOPT_E_IO, path + ": missing design CSV header");
    auto w = design_full();
    while (std::getline(in, line)) {
      ++ln;
      if (line.empty()) continue;
      std::vector<std::string> c;
      std::stringstream ss(line);
      std::string cell;
      while (std::getline(ss, cell, ',')) c.push_back(cell);
      if (!line.empty() && line.back() == ',') c.push_back("");
      if (c.size() != 4) fail(LBOPT_E_IO, path + ":" + std::to_string(ln) + ": expected 4 cells");
      long x, y, z;
      double v;
      try {
        x = std::stol(c[0]), y = std::stol(c[1]), z = std::stol(c[2]);
        v = c[3].empty() ? kNaN : std::stod(c[3]);
      } catch (const std::exception&) {
        fail(LBOPT_E_IO, path + ":" + std::to_string(ln) + ": bad cell");
      }
      if (x < 0 || x >= cfg.nx || y < 0 || y >= cfg.ny || z < 0 || z >= cfg.nz)
        fail(LBOPT_E_IO, path + ":" + std::to_string(ln) + ": node outside the lattice");
      const long idx = x + long(cfg.nx) * (y + long(cfg.ny) * z);
      if (sys.mask[idx]) w[idx] = (v < 0.0 || v > 1.0) ? (v < 0.0 ? 0.0 : 1.0) : v;
    }
    ok(e, lbgpu_set_design(e, w.data()));
    has_primal = false;
  }
};

namespace {

thread_local std::string g_open_error;

template <class F>
int open_guarded(lbopt_case** out, F&& make) {  // capi.cpp:19-37
  if (!out) return LBOPT_E_ARG;
  *out = nullptr;
  g_open_error.clear();
  try {
    *out = new lbopt_case(make());
    return LBOPT_OK;
  } catch (const CaseFail& f) {
    g_open_error = f.msg;
    return f.code == LBOPT_E_STATE ? LBOPT_E_NUMERIC : f.code;
  } catch (const std::exception& x) {
    g_open_error = x.what();
    return LBOPT_E_NUMERIC;
  }
}

template <class F>
int guarded(lbopt_case* c, F&& fn) {  // capi.cpp:39-59
  if (!c) return LBOPT_E_ARG;
  try {
    fn();
    c->error.clear();
    return LBOPT_OK;
  } catch (const CaseFail& f) {
    c->error = f.msg;
    return f.code == LBOPT_E_ARG ? LBOPT_E_NUMERIC : f.code;
  } catch (const std::exception& x) {
    c->error = x.what();
    return LBOPT_E_NUMERIC;
  }
}

CaseSpec parse_or_fail(const std::string& text, const std::string& origin) {
  CaseSpec c;
  std::string err;
  if (!lbgpu::parse_case_text(text, origin, c, err)) fail(LBOPT_E_CONFIG, err);
  return c;
}

}  // namespace

template <class F>
int op(lbopt_case* c, F&& body) {
  return guarded(c, [&] {
    c->ensure_built();
    body();
  });
}

extern "C" {

const char* lbopt_version(void) { return "0.1.0"; }

int lbopt_open(const char* config_path, lbopt_case** out) {
  if (!config_path) return LBOPT_E_ARG;
  return open_guarded(out, [&] {
    std::ifstream in(config_path);
    if (!in) fail(LBOPT_E_IO, std::string("cannot open config file: ") + config_path);
    std::ostringstream ss;
    ss << in.rdbuf();
    return parse_or_fail(ss.str(), config_path);
  });
}

int lbopt_open_text(const char* text, lbopt_case** out) {
  if (!text) return LBOPT_E_ARG;
  return open_guarded(out, [&] { return parse_or_fail(text, "<text>"); });
}

void lbopt_close(lbopt_case* c) { delete c; }
const char* lbopt_last_open_error(void) { return g_open_error.c_str(); }
const char* lbopt_error_message(const lbopt_case* c) { return c ? c->error.c_str() : "null handle"; }

int lbopt_set(lbopt_case* c, const char* key, const char* value) {
  if (!key || !value) return LBOPT_E_ARG;
  return guarded(c, [&] {
    std::string err;
    if (!lbgpu::set_case_key(c->cfg, key, value, err)) fail(LBOPT_E_CONFIG, err);
    c->dirty = true;
  });
}

int lbopt_save_config(lbopt_case* c, const char* path) {
  if (!path) return LBOPT_E_ARG;
  return guarded(c, [&] {
    c->ensure_built();
    std::ofstream out(path);
    if (!out) fail(LBOPT_E_IO, std::string("cannot open for writing: ") + path);
    out << lbgpu::serialize_case(c->cfg);
    if (!out) fail(LBOPT_E_IO, std::string("write failed: ") + path);
  });
}

int lbopt_simulate(lbopt_case* c) { return op(c, [&] { c->simulate(); }); }
int lbopt_solve_adjoint(lbopt_case* c) { return op(c, [&] { c->run_adjoint(); }); }
int lbopt_optimize(lbopt_case* c) { return op(c, [&] { c->optimize(); }); }
int lbopt_grad_check(lbopt_case* c, double* max_rel_err) {
  return op(c, [&] { c->grad_check(max_rel_err); });
}
int lbopt_threshold_sweep(lbopt_case* c, double* best_eta, double* best_objective) {
  return op(c, [&] { c->threshold(best_eta, best_objective); });
}
int lbopt_partition_check(lbopt_case* c, long steps, double* max_diff) {
  return op(c, [&] { c->partition_check(steps, max_diff); });
}
int lbopt_scaling_report(lbopt_case* c, long steps) { return op(c, [&] { c->scaling(steps); }); }
int lbopt_cost_ratio(lbopt_case* c, long steps, double* ratio) {
  return op(c, [&] {
    const double r = c->cost_ratio_run(steps);
    if (ratio) *ratio = r;
  });
}
int lbopt_generate_fins(lbopt_case* c, int count, int width) {
  return op(c, [&] { c->generate_fins(count, width); });
}
int lbopt_apply_threshold(lbopt_case* c, double eta) {
  return op(c, [&] { c->apply_threshold_now(eta); });
}

int lbopt_load_state_csv(lbopt_case* c, const char* path) {
  if (!path) return LBOPT_E_ARG;
  return guarded(c, [&] {
    c->ensure_built();
    c->load_state(path);
  });
}

int lbopt_load_design_csv(lbopt_case* c, const char* path) {
  if (!path) return LBOPT_E_ARG;
  return guarded(c, [&] {
    c->ensure_built();
    c->load_design(path);
  });
}

int lbopt_write_fields(lbopt_case* c, const char* csv_path, const char* vtk_path) {
  return guarded(c, [&] {
    c->ensure_built();
    c->write_fields_outputs(csv_path ? csv_path : "", vtk_path ? vtk_path : "");
  });
}

int lbopt_shape(const lbopt_case* c, int* nx, int* ny, int* nz) {
  if (!c || !nx || !ny || !nz) return LBOPT_E_ARG;
  *nx = c->cfg.nx, *ny = c->cfg.ny, *nz = c->cfg.nz;
  return LBOPT_OK;
}
int lbopt_objective_value(const lbopt_case* c, double* v) {
  if (!c || !v) return LBOPT_E_ARG;
  *v = c->objective;
  return LBOPT_OK;
}
int lbopt_iterations(const lbopt_case* c, long* it) {
  if (!c || !it) return LBOPT_E_ARG;
  *it = c->iterations;
  return LBOPT_OK;
}
int lbopt_converged(const lbopt_case* c, int* flag) {
  if (!c || !flag) return LBOPT_E_ARG;
  *flag = c->converged ? 1 : 0;
  return LBOPT_OK;
}
int lbopt_residual(const lbopt_case* c, double* v) {
  if (!c || !v) return LBOPT_E_ARG;
  *v = c->residual;
  return LBOPT_OK;
}
int lbopt_out_dir(const lbopt_case* c, char* buf, int cap) {
  if (!c || !buf || cap < 1) return LBOPT_E_ARG;
  const std::string& d = c->cfg.out_dir;
  if (int(d.size()) + 1 > cap) return LBOPT_E_ARG;
  std::memcpy(buf, d.c_str(), d.size() + 1);
  return LBOPT_OK;
}

}  // extern "C"

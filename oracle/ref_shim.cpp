// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A C-ABI shim over the reference's own C++ operators (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/liblbopt_ref.so).
// It exposes exactly the inner operator seam the GPU engine replaces
// (SURVEY.md §8b "B2"): initialize_state, primal_step, step_residual,
// solve_fixed_point (collision.hpp:166-201), adjoint_step, solve_adjoint,
// param_gradient (adjoint.hpp:47-80), evaluate_raw (objective.hpp:40-41),
// one_shot_run (optimizer.hpp:41-44), PartitionedRun (partition.hpp:67-127),
// plus the tag/design/support builders (config.cpp:302-395) so tests can check
// the product's masks bit-exactly. Used by tests/, bench.py's cpu_baseline /
// --impl reference legs and tests/golden/make_golden.py only.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <algorithm>
#include <variant>

#include "lbopt/adjoint.hpp"
#include "lbopt/collision.hpp"
#include "lbopt/config.hpp"
#include "lbopt/objective.hpp"
#include "lbopt/optimizer.hpp"
#include "lbopt/partition.hpp"

using namespace lbopt;

namespace {

thread_local std::string g_err;

template <class R>
struct Fields {
  StateField<R> f, v;
  explicit Fields(const System& s) : f(s.shape, s.m), v(s.shape, s.m) {}
};

struct Handle {
  CaseConfig cfg;
  BuiltCase bc;
  std::variant<Fields<double>, Fields<float>> fl;
  Handle(const CaseConfig& c, BuiltCase b)
      : cfg(c), bc(std::move(b)), fl(std::in_place_type<Fields<double>>, bc.sys) {
    if (cfg.precision == 32) fl.emplace<Fields<float>>(bc.sys);
  }
};

template <class F>
int guard(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const IoError& e) {
    g_err = e.what();
    return 4;
  } catch (const StateError& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

Handle* H(void* h) { return static_cast<Handle*>(h); }

AdjointKernel kern(int k) { return k ? AdjointKernel::DualSweep : AdjointKernel::Analytic; }

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// overrides: newline-separated "section.key=value" lines (may be NULL).
void* ref_open(const char* cfg_text, const char* overrides) {
  Handle* out = nullptr;
  const int rc = guard([&] {
    CaseConfig cfg = CaseConfig::parse_text(cfg_text ? cfg_text : "", "<oracle>");
    if (overrides) {
      std::istringstream in(overrides);
      std::string line;
      while (std::getline(in, line)) {
        if (line.empty()) continue;
        const auto eq = line.find('=');
        if (eq == std::string::npos) throw ConfigError("bad override: " + line);
        cfg.set(line.substr(0, eq), line.substr(eq + 1));
      }
    }
    cfg.validate();
    out = new Handle(cfg, build_case(cfg));
  });
  return rc == 0 ? out : nullptr;
}

void ref_close(void* h) { delete H(h); }

int ref_info(void* h, int* dims /*nx,ny,nz,m,mf,mt,precision*/, long* counts /*nodes,design,support*/) {
  return guard([&] {
    const System& s = H(h)->bc.sys;
    dims[0] = s.shape.nx; dims[1] = s.shape.ny; dims[2] = s.shape.nz;
    dims[3] = s.m; dims[4] = s.mf; dims[5] = s.mt; dims[6] = H(h)->cfg.precision;
    counts[0] = s.shape.nodes();
    counts[1] = long(s.design.nodes.size());
    counts[2] = long(H(h)->bc.objective.support.size());
  });
}

int ref_tables(void* h, uint8_t* tag, double* bc_T, int8_t* axis, int8_t* sign, double* w,
               uint8_t* mask, long* design_nodes, long* support, double* A, double* relax,
               int32_t* vel /* m*3 */, int32_t* opp /* m */) {
  return guard([&] {
    const System& s = H(h)->bc.sys;
    const long n = s.shape.nodes();
    for (long i = 0; i < n; ++i) {
      tag[i] = uint8_t(s.tags.tag[i]);
      bc_T[i] = s.tags.bc_T[i];
      axis[i] = s.tags.bc_axis[i];
      sign[i] = s.tags.bc_sign[i];
      w[i] = s.design.w[i];
      mask[i] = s.design.mask[i];
    }
    for (std::size_t i = 0; i < s.design.nodes.size(); ++i) design_nodes[i] = s.design.nodes[i];
    const auto& sup = H(h)->bc.objective.support;
    for (std::size_t i = 0; i < sup.size(); ++i) support[i] = sup[i];
    std::memcpy(A, s.tables.A.a.data(), sizeof(double) * s.mf * s.mf);
    for (int i = 0; i < s.mf; ++i) relax[i] = s.tables.relax[i];
    for (int p = 0; p < s.m; ++p) {
      vel[3 * p] = s.vel[p].x; vel[3 * p + 1] = s.vel[p].y; vel[3 * p + 2] = s.vel[p].z;
      opp[p] = s.opp[p];
    }
  });
}

int ref_set_design(void* h, const double* w_full) {
  return guard([&] {
    System& s = H(h)->bc.sys;
    for (long i = 0; i < s.shape.nodes(); ++i) s.design.w[i] = w_full[i];
  });
}

int ref_init_state(void* h) {
  return guard([&] {
    std::visit([&](auto& F) {
      initialize_state(H(h)->bc.sys, F.f);
      F.v.fill(0);
    }, H(h)->fl);
  });
}

// field 0 = primal f, 1 = adjoint v; current buffer, reference layout (planes x-fastest).
int ref_get_state(void* h, int field, double* out) {
  return guard([&] {
    std::visit([&](auto& F) {
      auto& S = field ? F.v : F.f;
      auto raw = S.raw(S.buffer_id());
      for (std::size_t i = 0; i < raw.size(); ++i) out[i] = double(raw[i]);
    }, H(h)->fl);
  });
}

int ref_set_state(void* h, int field, const double* in) {
  return guard([&] {
    std::visit([&](auto& F) {
      using R = std::decay_t<decltype(F.f.raw(0)[0])>;
      auto& S = field ? F.v : F.f;
      auto raw = S.raw(S.buffer_id());
      for (std::size_t i = 0; i < raw.size(); ++i) raw[i] = R(in[i]);
    }, H(h)->fl);
  });
}

int ref_primal_steps(void* h, long n, double* residual) {
  return guard([&] {
    std::visit([&](auto& F) {
      for (long i = 0; i < n; ++i) primal_step(H(h)->bc.sys, F.f);
      if (residual) *residual = n > 0 ? step_residual(F.f) : 0.0;
    }, H(h)->fl);
  });
}

int ref_adjoint_steps(void* h, long n, int kernel, double* residual) {
  return guard([&] {
    std::visit([&](auto& F) {
      for (long i = 0; i < n; ++i)
        adjoint_step(H(h)->bc.sys, H(h)->bc.objective, F.f, F.v, kern(kernel));
      if (residual) *residual = n > 0 ? step_residual(F.v) : 0.0;
    }, H(h)->fl);
  });
}

int ref_solve_primal(void* h, double tol, long max_iter, long fixed, long* iters,
                     double* res, int* conv) {
  return guard([&] {
    std::visit([&](auto& F) {
      using R = std::decay_t<decltype(F.f.raw(0)[0])>;
      SolveOptions<R> o;
      o.tol = tol;
      o.max_iter = max_iter;
      o.fixed_iters = fixed;
      o.record_interval = 1L << 30;
      const SolveResult r = solve_fixed_point(H(h)->bc.sys, F.f, o);
      *iters = r.iterations;
      *res = r.residual;
      *conv = r.converged;
    }, H(h)->fl);
  });
}

int ref_solve_adjoint(void* h, double tol, long max_iter, long fixed, int kernel, long* iters,
                      double* res, int* conv) {
  return guard([&] {
    std::visit([&](auto& F) {
      using R = std::decay_t<decltype(F.f.raw(0)[0])>;
      AdjointSolveOptions<R> o;
      o.tol = tol;
      o.max_iter = max_iter;
      o.fixed_iters = fixed;
      o.kernel = kern(kernel);
      o.record_interval = 1L << 30;
      const SolveResult r = solve_adjoint(H(h)->bc.sys, H(h)->bc.objective, F.f, F.v, o);
      *iters = r.iterations;
      *res = r.residual;
      *conv = r.converged;
    }, H(h)->fl);
  });
}

int ref_gradient(void* h, int kernel, double* g, double* g_dp) {
  return guard([&] {
    std::visit([&](auto& F) {
      const GradientVector gv = param_gradient(H(h)->bc.sys, F.v, F.f, kern(kernel));
      for (std::size_t i = 0; i < gv.design.size(); ++i) g[i] = gv.design[i];
      *g_dp = gv.globals.at(0).second;
    }, H(h)->fl);
  });
}

int ref_objective(void* h, double* value) {
  return guard([&] {
    std::visit([&](auto& F) { *value = evaluate_raw(H(h)->bc.objective, H(h)->bc.sys, F.f); },
               H(h)->fl);
  });
}

int ref_penalty(void* h, double* value) {
  return guard([&] { *value = penalty(H(h)->bc.sys.design).value; });
}

// One-shot with the options the config describes (build_one_shot_options),
// iteration count overridden. rows: 7 doubles per RunRow
// (iteration, residual, objective, penalty, weight, composite, grad_norm).
int ref_one_shot(void* h, long iterations, long record_interval, double* rows, long cap,
                 long* n_rows) {
  return guard([&] {
    std::visit([&](auto& F) {
      OneShotOptions o = build_one_shot_options(H(h)->cfg);
      o.iterations = iterations;
      o.record_interval = record_interval;
      RunRecord rec;
      one_shot_run(H(h)->bc.sys, H(h)->bc.objective, F.f, F.v, o, &rec);
      long k = 0;
      for (const RunRow& r : rec.rows) {
        if (k >= cap) break;
        double* o7 = rows + 7 * k++;
        o7[0] = double(r.iteration); o7[1] = r.residual; o7[2] = r.objective;
        o7[3] = r.penalty; o7[4] = r.penalty_weight; o7[5] = r.composite; o7[6] = r.grad_norm;
      }
      *n_rows = long(rec.rows.size());
    }, H(h)->fl);
  });
}

int ref_collide_node(void* h, int tag, int axis, int sign, double bcT, const double* fin,
                     double w, double* fout) {
  return guard([&] {
    const System& s = H(h)->bc.sys;
    std::vector<double> in(fin, fin + s.m), out(s.m);
    collide_node<double>(s, NodeTag(tag), axis, sign, bcT, in, w, s.model.rho_inlet(),
                         std::span<double>(out));
    std::memcpy(fout, out.data(), sizeof(double) * s.m);
  });
}

int ref_fd_gradient(void* h, long ordinal, double step, double tol, long max_iter, long fixed,
                    double* out) {
  return guard([&] {
    FdComponent c;
    if (ordinal < 0) {
      c.is_global = true;
      c.global = "inlet_dp";
    } else {
      c.design_ordinal = ordinal;
    }
    if (H(h)->cfg.precision == 32)
      *out = fd_gradient<float>(H(h)->bc.sys, H(h)->bc.objective, c, step, tol, max_iter, fixed);
    else
      *out = fd_gradient<double>(H(h)->bc.sys, H(h)->bc.objective, c, step, tol, max_iter, fixed);
  });
}

// tangent_solve (adjoint.cpp:422-489) on the current primal state; dw in
// DesignField::nodes order. out: dF, iterations, residual, converged.
int ref_tangent(void* h, const double* dw, double d_inlet_dp, double tol, long max_iter,
                double* dF, long* iters, double* resid, int* conv) {
  return guard([&] {
    Direction d;
    d.dw.assign(dw, dw + H(h)->bc.sys.design.nodes.size());
    d.d_inlet_dp = d_inlet_dp;
    std::visit([&](auto& F) {
      const auto r = tangent_solve(H(h)->bc.sys, H(h)->bc.objective, F.f, d, tol, max_iter);
      *dF = r.dF;
      *iters = r.solve.iterations;
      *resid = r.solve.residual;
      *conv = r.solve.converged ? 1 : 0;
    }, H(h)->fl);
  });
}

int ref_partition_check(void* h, int parts, long steps, double* pd, double* ad) {
  return guard([&] {
    const PartitionCheckResult r =
        H(h)->cfg.precision == 32
            ? partition_check<float>(H(h)->bc.sys, H(h)->bc.objective, parts, steps)
            : partition_check<double>(H(h)->bc.sys, H(h)->bc.objective, parts, steps);
    *pd = r.max_primal_diff;
    *ad = r.max_adjoint_diff;
  });
}

// Wall-clock seconds for `steps` sweeps of `which` (0 primal, 1 adjoint)
// starting from the handle's current f (and v for the adjoint). threads == 1
// runs the monolithic operators; threads > 1 the reference's thread-per-slab
// PartitionedRun (partition.cpp:93-188), its only multi-core path. The state
// of the handle is left untouched for threads > 1.
int ref_time(void* h, int which, int threads, long steps, double* seconds) {
  return guard([&] {
    std::visit([&](auto& F) {
      using R = std::decay_t<decltype(F.f.raw(0)[0])>;
      const System& s = H(h)->bc.sys;
      const ObjectiveSpec& ob = H(h)->bc.objective;
      const auto t0 = std::chrono::steady_clock::now();
      if (threads <= 1) {
        for (long i = 0; i < steps; ++i) {
          if (which == 0) primal_step(s, F.f);
          else adjoint_step(s, ob, F.f, F.v, AdjointKernel::Analytic);
        }
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      } else {
        PartitionedRun<R> run(s, ob, threads);
        run.load_state(F.f);
        run.reset_adjoint();
        const auto t1 = std::chrono::steady_clock::now();
        for (long i = 0; i < steps; ++i) {
          if (which == 0) run.step_primal();
          else run.step_adjoint();
        }
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
      }
    }, H(h)->fl);
  });
}

// Full-size parity oracle: the reference's thread-per-slab runner
// (PartitionedRun, partition.cpp:93-253; bitwise equal to the monolithic
// operators, test_partition.cpp:53-141) over the handle's state. Loads the
// handle's f, zeroes v, runs n_primal primal lock steps, then n_adjoint
// adjoint lock steps against the state the slabs hold, then n_pairs
// (primal, adjoint) pairs, and gathers f and v back into the handle.
// resid[0] / resid[1]: last_residual() after the last primal / adjoint step.
int ref_partitioned(void* h, int threads, long n_primal, long n_adjoint, long n_pairs,
                    double* resid) {
  return guard([&] {
    std::visit([&](auto& F) {
      using R = std::decay_t<decltype(F.f.raw(0)[0])>;
      PartitionedRun<R> run(H(h)->bc.sys, H(h)->bc.objective, threads);
      run.load_state(F.f);
      run.reset_adjoint();
      double rp = 0.0, ra = 0.0;
      for (long i = 0; i < n_primal; ++i) run.step_primal();
      if (n_primal > 0) rp = run.last_residual();
      for (long i = 0; i < n_adjoint; ++i) run.step_adjoint();
      if (n_adjoint > 0) ra = run.last_residual();
      for (long i = 0; i < n_pairs; ++i) {
        run.step_primal();
        if (i == n_pairs - 1) rp = run.last_residual();
        run.step_adjoint();
      }
      if (n_pairs > 0) ra = run.last_residual();
      run.gather_state(F.f);
      run.gather_adjoint(F.v);
      if (resid) resid[0] = rp, resid[1] = ra;
    }, H(h)->fl);
  });
}

// partitioned_fixed_point (partition.cpp:279-312): the reference's
// tol-stop primal solve on its thread-per-slab runner (bitwise its
// monolithic solve_fixed_point), from the handle's f; the state is gathered
// back into the handle.
int ref_partitioned_solve(void* h, int threads, double tol, long max_iter, long fixed,
                          long* iters, double* res, int* conv) {
  return guard([&] {
    std::visit([&](auto& F) {
      using R = std::decay_t<decltype(F.f.raw(0)[0])>;
      SolveOptions<R> o;
      o.tol = tol;
      o.max_iter = max_iter;
      o.fixed_iters = fixed;
      const SolveResult r =
          partitioned_fixed_point<R>(H(h)->bc.sys, H(h)->bc.objective, F.f, threads, o);
      *iters = r.iterations;
      *res = r.residual;
      *conv = r.converged ? 1 : 0;
    }, H(h)->fl);
  });
}

// The A14 composition recipe's obj_empty: on = 0 clears the
// objective's full-grid membership flags so adjoint_step skips the source
// term (adjoint.cpp:199); on = 1 restores them from the support list.
int ref_objective_enabled(void* h, int on) {
  return guard([&] {
    ObjectiveSpec& ob = H(h)->bc.objective;
    std::fill(ob.on_support.begin(), ob.on_support.end(), std::uint8_t(0));
    if (on)
      for (long i : ob.support) ob.on_support[std::size_t(i)] = 1;
  });
}

}  // extern "C"

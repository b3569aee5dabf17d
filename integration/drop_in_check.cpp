// Drop-in check of the reference-side binding (gpu_engine.hpp): the
// reference's own parse_text + build_case (config.cpp:129-427) and solvers on
// the CPU, and the same System through make_gpu_engine -> lbgpu on the GPU,
// from initialize_state: fixed-iteration solve_fixed_point, solve_adjoint,
// evaluate_raw, param_gradient, then one gpu_mma_iteration against the
// reference's write-back + solves. Prints one JSON line of max differences
// (all 0 in the bit-exact build).
//   drop_in_check <case file> <exact 0|1> <primal iters> <adjoint iters>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>

#include "gpu_engine.hpp"
#include "lbopt/config.hpp"
#include "lbopt/objective.hpp"

using namespace lbopt;

static double maxdiff(std::span<const double> a, std::span<const double> b) {
  double d = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) d = std::max(d, std::abs(a[i] - b[i]));
  return d;
}

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: drop_in_check <case file> <exact> <primal iters> <adjoint iters>\n");
    return 2;
  }
  std::ifstream in(argv[1]);
  std::stringstream text;
  text << in.rdbuf();
  const int exact = std::atoi(argv[2]);
  const long kp = std::atol(argv[3]), ka = std::atol(argv[4]);
  try {
    const CaseConfig cfg = CaseConfig::parse_text(text.str());
    BuiltCase bc = build_case(cfg);
    const System& s = bc.sys;
    // the reference
    StateField<double> f(s.shape, s.m), v(s.shape, s.m);
    initialize_state(s, f);
    SolveOptions<double> po;
    po.fixed_iters = kp;
    const SolveResult pr = solve_fixed_point(s, f, po);
    AdjointSolveOptions<double> ao;
    ao.fixed_iters = ka;
    const SolveResult ar = solve_adjoint(s, bc.objective, f, v, ao);
    const double J = evaluate_raw(bc.objective, s, f);
    const GradientVector g = param_gradient(s, v, f, AdjointKernel::Analytic);
    // the same System on the GPU through the binding
    lbgpu_engine* e = make_gpu_engine(s, bc.objective, 64, exact);
    StateField<double> fg(s.shape, s.m), vg(s.shape, s.m);
    initialize_state(s, fg);
    const SolveResult gpr = gpu_solve_fixed_point(e, fg, po);
    const SolveResult gar = gpu_solve_adjoint(e, vg, ao);
    const double Jg = gpu_evaluate_raw(e);
    const GradientVector gg = gpu_param_gradient(e, AdjointKernel::Analytic);
    // one MMA-shaped outer iteration on both: design write-back, then solves
    // (cases without a design region skip it)
    GradientVector g2, gg2;
    std::vector<double> wd(s.design.nodes.size());
    if (!wd.empty()) {
      for (std::size_t i = 0; i < wd.size(); ++i)
        wd[i] = std::min(1.0, std::max(0.0, s.design.w[std::size_t(s.design.nodes[i])] + 1e-3 * g.design[i] / (g.max_abs() + 1e-300)));
      System s2 = s;
      for (std::size_t i = 0; i < wd.size(); ++i) s2.design.w[std::size_t(s2.design.nodes[i])] = wd[i];
      StateField<double> f2(s.shape, s.m), v2(s.shape, s.m);
      initialize_state(s2, f2);
      solve_fixed_point(s2, f2, po);
      AdjointSolveOptions<double> ao2;
      ao2.fixed_iters = kp;  // mma_run: the adjoint runs the primal's count (optimizer.cpp:179)
      solve_adjoint(s2, bc.objective, f2, v2, ao2);
      g2 = param_gradient(s2, v2, f2, AdjointKernel::Analytic);
      gpu_check(e, lbgpu_init_state(e));
      SolveResult p2;
      gg2 = gpu_mma_iteration(e, wd, po, &p2);
    }
    std::printf(
        "{\"nodes\": %ld, \"design\": %zu, \"exact\": %d, \"primal_iters\": [%ld, %ld], "
        "\"primal_residual\": [%.17g, %.17g], \"adjoint_residual\": [%.17g, %.17g], "
        "\"f_maxdiff\": %.17g, \"f_max\": %.17g, \"v_maxdiff\": %.17g, \"v_max\": %.17g, "
        "\"J\": [%.17g, %.17g], \"g_maxdiff\": %.17g, \"g_max\": %.17g, \"gdp\": [%.17g, %.17g], "
        "\"mma_g_maxdiff\": %.17g, \"mma_g_max\": %.17g}\n",
        s.shape.nodes(), s.design.nodes.size(), exact, pr.iterations, gpr.iterations, pr.residual,
        gpr.residual, ar.residual, gar.residual,
        maxdiff(f.raw(f.buffer_id()), fg.raw(fg.buffer_id())),
        maxdiff(f.raw(f.buffer_id()), std::vector<double>(f.raw(f.buffer_id()).size(), 0.0)),
        maxdiff(v.raw(v.buffer_id()), vg.raw(vg.buffer_id())),
        maxdiff(v.raw(v.buffer_id()), std::vector<double>(v.raw(v.buffer_id()).size(), 0.0)), J,
        Jg, maxdiff(g.design, gg.design), g.max_abs(), g.globals[0].second, gg.globals[0].second,
        maxdiff(g2.design, gg2.design), g2.max_abs());
    lbgpu_destroy(e);
  } catch (const std::exception& x) {
    std::fprintf(stderr, "error: %s\n", x.what());
    return 1;
  }
  return 0;
}

// The reference-side binding a maintainer adds to the reference tree
// (proj/src/gpu_engine.cpp + this header): the reference's own types in,
// liblbgpu underneath. INTEGRATION.md §2 describes it; tests compile it
// against /root/reference/proj/include and run it (tests/test_integration.py).
#pragma once

#include <vector>

#include "lbgpu.h"
#include "lbopt/adjoint.hpp"
#include "lbopt/collision.hpp"
#include "lbopt/objective.hpp"

namespace lbopt {

// The reference's own System + ObjectiveSpec (collision.hpp:74-88,
// objective.hpp:19-28), flattened as-is -- tags, bc arrays, design w / mask,
// support, ModelTables::A and relax, the coupled vel / opp tables -- so the
// engine's masks and A are the reference's by construction.
lbgpu_engine* make_gpu_engine(const System& s, const ObjectiveSpec& o, int precision,
                              int exact = 0, int device = 0);

// lbgpu status -> the reference's exception types (capi.cpp:19-59 in reverse).
void gpu_check(lbgpu_engine* e, int rc);

// solve_fixed_point (collision.cpp:377-416) on the GPU: f's current buffer is
// uploaded, solved, and downloaded back into it.
template <class R>
SolveResult gpu_solve_fixed_point(lbgpu_engine* e, StateField<R>& f, const SolveOptions<R>& opt);

// solve_adjoint (adjoint.cpp:256-297) against the engine's current primal
// state; v's current buffer receives the adjoint state.
template <class R>
SolveResult gpu_solve_adjoint(lbgpu_engine* e, StateField<R>& v, const AdjointSolveOptions<R>& opt);

// param_gradient (adjoint.cpp:377-420) of the engine's (v, f).
GradientVector gpu_param_gradient(lbgpu_engine* e, AdjointKernel kernel);

// evaluate_raw (objective.cpp:64-72) of the engine's primal state.
double gpu_evaluate_raw(lbgpu_engine* e);

// A host-side MMA loop (mma_run, optimizer.cpp:141-212) on the engine: the
// design write-back (optimizer.cpp:200-202) in DesignField::nodes order,
// then solve_fixed_point, solve_adjoint with the primal's iteration count as
// fixed_iters (optimizer.cpp:179) and param_gradient -- the calls the
// reference makes per outer iteration.
template <class R>
GradientVector gpu_mma_iteration(lbgpu_engine* e, const std::vector<double>& w_design,
                                 const SolveOptions<R>& popt, SolveResult* primal);

}  // namespace lbopt

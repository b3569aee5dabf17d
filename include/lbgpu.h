/* lbgpu — B200 (sm_100a) engine for the LBM primal / discrete-adjoint hot
 * path of the reference (arxiv/paper_1501_04741, /root/reference/proj).
 *
 * This is the thin C ABI the GPU path sits behind (seam "B2").
 * Each entry point replaces one operator of the reference's inner seam; the
 * reference interface it replaces is cited beside it. Plain pointers and
 * sizes only; all host arrays use the reference's layout: SoA planes of the
 * current (pre-collision) state, plane p at p*N, node index
 * x + nx*(y + ny*z) (lattice.hpp:25-27, :54-100).
 *
 * Status codes are the reference's (lbopt.h:18-25). Errors store a message
 * on the engine (lbgpu_error_message), cleared on success (capi.cpp:39-59);
 * creation failures go to thread-local storage (lbgpu_last_create_error).
 * An engine is not thread-safe; use one per host thread. Every call is
 * synchronous on return.
 */
#ifndef LBGPU_H
#define LBGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  LBGPU_OK = 0,        /* LBOPT_OK */
  LBGPU_E_ARG = 1,     /* LBOPT_E_ARG: null handle or bad argument */
  LBGPU_E_CONFIG = 2,  /* LBOPT_E_CONFIG: invalid system description */
  LBGPU_E_NUMERIC = 3, /* LBOPT_E_NUMERIC: rho <= 0, non-finite residual, CUDA fault */
  LBGPU_E_IO = 4,      /* LBOPT_E_IO */
  LBGPU_E_STATE = 5    /* LBOPT_E_STATE: operation out of order */
};

typedef struct lbgpu_engine lbgpu_engine; /* opaque; owns all device memory */

/* Flattened lbopt::System + ObjectiveSpec (collision.hpp:74-88,
 * objective.hpp:19-28). The caller keeps ownership of every array; the
 * engine copies what it needs. The lattice pair is implied by nz:
 * nz == 1 -> D2Q9 flow + D2Q9 temperature, else D3Q19 + D3Q7
 * (config.cpp:404-410). */
typedef struct {
  int nx, ny, nz;
  int precision;  /* 64 | 32 ([model] precision, config.hpp:26) */
  int exact;      /* 1: reference operation order, no FMA (FP64 only): bit-exact */
  int device;     /* CUDA device ordinal */
  /* ModelSpec (collision.hpp:46-59) */
  int collision;  /* 0 fmrt, 1 bgk */
  double nu, beta_fluid, beta_solid, inlet_dp, u_clamp, omega_nonhydro, switch_theta;
  int switch_form; /* 0 solid_power, 1 fluid_power */
  /* Optional: ModelTables::A (mf x mf, row-major) and the relaxation
   * diagonal (mf). NULL -> built here the way ModelTables::build does. */
  const double* A;
  const double* relax;
  /* Optional: coupled velocity table (m x 3) and opposite map (m) of
   * System::finalize; when given they must match the engine's bit-exactly. */
  const int32_t* vel;
  const int32_t* opp;
  /* TagMap + DesignField, N entries each (collision.hpp:25-41, topology.hpp:15-27) */
  const uint8_t* tag; /* NodeTag: 0 interior 1 wall 2 inlet 3 outlet 4 heater */
  const double* bc_T;
  const int8_t* bc_axis;
  const int8_t* bc_sign;
  const double* w;
  const uint8_t* design_mask;
  /* ObjectiveSpec */
  int obj_kind; /* 0 mixing 1 heatflux 2 synthetic */
  int flux_axis, flux_sign;
  const int64_t* support; /* ascending flat indices */
  int64_t n_support;
  /* x-slab decomposition (partition.cpp:9-21): with slab_count > 1 the engine
   * owns global columns [x0, x0+span) of slab slab_id (decompose's sizes) and
   * every per-node array above is in the local layout of lbgpu_slab_nxl(span)
   * columns: owned at 0..span-1, right ghost at span, left ghost at nxl-1;
   * support indices are local. nx stays the global extent. */
  int slab_count, slab_id;
  /* State storage (no reference counterpart: StateField<R> always double-
   * buffers, lattice.hpp:57-92). 0: two buffers per field (every operation).
   * 1: in-place AA-pattern streaming, one buffer per field (half the memory,
   * the same bytes per sweep): fixed-step sweeps, pairs, objective and
   * gradient only -- no step residual, hence no tol-stop solves (product
   * build only). */
  int streaming;
} lbgpu_system_desc;

/* One monitoring row (run_record.hpp:11-19): iteration, residual,
 * objective, penalty, penalty_weight, composite, grad_norm. */
typedef struct {
  double iteration, residual, objective, penalty, penalty_weight, composite, grad_norm;
} lbgpu_run_row;

const char* lbgpu_version(void);
/* Visible CUDA devices (0 when there is no usable driver / GPU). */
int lbgpu_device_count(void);
/* Local column count of a slab of `span` owned columns (span + 2 ghosts,
 * rounded up to 16 so rows stay 128-byte aligned). */
int lbgpu_slab_nxl(int span);

/* --- lifecycle --- */
int lbgpu_create(const lbgpu_system_desc* desc, lbgpu_engine** out);
/* Build the System from case-file text (CaseConfig::parse_text + newline-
 * separated "section.key=value" overrides + build_case, config.cpp:129-427)
 * and create the engine. exact as in lbgpu_system_desc. */
int lbgpu_create_from_config(const char* cfg_text, const char* overrides, int device, int exact,
                             lbgpu_engine** out);
/* One x-slab of the case: decompose(nx, slab_count)[slab_id] with local tables. */
int lbgpu_create_slab_from_config(const char* cfg_text, const char* overrides, int device,
                                  int exact, int slab_count, int slab_id, lbgpu_engine** out);
/* Both of the above with the storage choice (lbgpu_system_desc::streaming):
 * slab_count 1 and slab_id 0 is the whole lattice, slab_id -1 one slab in the
 * ghost-column layout (a single-rank ring). */
int lbgpu_create_from_config_ex(const char* cfg_text, const char* overrides, int device,
                                int exact, int slab_count, int slab_id, int streaming,
                                lbgpu_engine** out);
void lbgpu_destroy(lbgpu_engine* e);
/* Host-only: the System build_case would assemble from this case text, in
 * reference form (tags, bc arrays, design w/mask/nodes, support, A), without
 * touching a GPU. dims/counts as lbgpu_info; any array pointer may be NULL. */
int lbgpu_case_tables(const char* cfg_text, const char* overrides, int* dims, int64_t* counts,
                      uint8_t* tag, double* bc_T, int8_t* bc_axis, int8_t* bc_sign, double* w,
                      uint8_t* mask, int64_t* design, int64_t* support, double* A);
/* Host-only slab variant (local layout). slab: gnx x0 span nxl count id. */
int lbgpu_case_slab_tables(const char* cfg_text, const char* overrides, int slab_count,
                           int slab_id, int* slab, int* dims, int64_t* counts, uint8_t* tag,
                           double* bc_T, int8_t* bc_axis, int8_t* bc_sign, double* w,
                           uint8_t* mask, int64_t* design, int64_t* support);
const char* lbgpu_last_create_error(void);
const char* lbgpu_error_message(const lbgpu_engine* e);

/* --- queries --- */
/* dims: nx ny nz m mf mt precision exact; counts: nodes design support inlets */
int lbgpu_info(const lbgpu_engine* e, int* dims, int64_t* counts);
/* The engine's tables in reference form (for mask parity): any pointer may be NULL. */
int lbgpu_get_tables(const lbgpu_engine* e, uint8_t* tag, double* bc_T, int8_t* bc_axis,
                     int8_t* bc_sign, double* w, uint8_t* mask, int64_t* design,
                     int64_t* support, double* A);
/* gnx x0 span nxl slab_count slab_id */
int lbgpu_slab_info(const lbgpu_engine* e, int* out6);
/* Steps done since creation / the last reset. */
int lbgpu_counters(const lbgpu_engine* e, int64_t* primal_steps, int64_t* adjoint_steps);
/* The CUDA stream all work is issued on (cudaStream_t), for event timing. */
void* lbgpu_stream(const lbgpu_engine* e);

/* --- state (field 0 = primal f, 1 = adjoint v) --- */
int lbgpu_init_state(lbgpu_engine* e);        /* initialize_state (collision.cpp:296-306), v = 0 */
int lbgpu_reset_adjoint(lbgpu_engine* e);     /* v.fill(0) (adjoint.cpp:261) */
int lbgpu_upload_state(lbgpu_engine* e, int field, const double* ref_layout);
int lbgpu_download_state(lbgpu_engine* e, int field, double* ref_layout);
/* Device-resident variants: the same layout, pointers to device memory. */
int lbgpu_upload_state_device(lbgpu_engine* e, int field, const double* d_ref_layout);
int lbgpu_download_state_device(lbgpu_engine* e, int field, double* d_ref_layout);
int lbgpu_set_design(lbgpu_engine* e, const double* w_full);   /* DesignField::w (N) */
int lbgpu_get_design(const lbgpu_engine* e, double* w_full);
/* The design vector in DesignField::nodes order (n_design values): the form
 * descent_update / mma_update produce (optimizer.cpp:8-16, :105-138). */
int lbgpu_set_design_values(lbgpu_engine* e, const double* w_design);
int lbgpu_get_design_values(lbgpu_engine* e, double* w_design);

/* --- sweeps --- */
/* n x primal_step (collision.cpp:308-363); residual (nullable) = step_residual
 * of the last step (collision.cpp:365-375). */
int lbgpu_primal_step(lbgpu_engine* e, int64_t n, double* residual);
/* n primal+adjoint pairs, each adjoint sweep against the state its primal
 * step just produced: one_shot_run (optimizer.cpp:25-72) at zeta = 0 without
 * its discarded design gradient (test_optimizer.cpp:182-209), and the bench
 * step. The product build fuses adjoint k with primal k+1 (one gather of the
 * shared state); states equal lbgpu_primal_step(1) + lbgpu_adjoint_step(1)
 * repeated n times, bit for bit. Residuals of the last pair (nullable). */
int lbgpu_pair_steps(lbgpu_engine* e, int64_t n, double* primal_residual,
                     double* adjoint_residual);
/* tangent_solve (adjoint.cpp:422-490): forward-mode sensitivity of the
 * objective along a design direction dw (DesignField::nodes order) plus
 * d_inlet_dp, from the current primal state (frozen base). df starts at zero
 * and is iterated to max|df_new - df_old| <= tol (solve_fixed_point's stop
 * rule); dF = sum over the support of dF^x/df . df. "tangent diverged at
 * iteration k" (LBGPU_E_NUMERIC) on a non-finite residual. iterations,
 * residual, converged are nullable. Engine state (f, v, w) is unchanged. */
int lbgpu_tangent_solve(lbgpu_engine* e, const double* dw_design, double d_inlet_dp, double tol,
                        int64_t max_iter, double* dF, int64_t* iterations, double* residual,
                        int* converged);
/* fd_gradient (adjoint.cpp:492-517): central difference (J(p+h) - J(p-h)) / 2h
 * of the raw objective along design node `ordinal` (DesignField::nodes order;
 * < 0: inlet_dp), each side a cold-start primal solve to tol / max_iter, or of
 * exactly fixed_iters steps when fixed_iters >= 0. The perturbation is a raw
 * write (no clamp), as in the reference. State, design and model are restored. */
int lbgpu_fd_gradient(lbgpu_engine* e, int64_t ordinal, double h, double tol, int64_t max_iter,
                      int64_t fixed_iters, double* out);
/* n fd_gradient components at once (grad_check_impl's 12 components x 3
 * steps, case.cpp:256-283, as one call): out[k] = the central difference along
 * ordinals[k] with step steps[k]. With fixed_iters >= 0 every side is queued
 * on the device back to back -- raw write of the perturbed w (or rho_in), the
 * start state, fixed_iters sweeps, evaluate_raw into a device slot,
 * write-back -- with one host sync for the whole batch; with fixed_iters < 0
 * each side is a tol-stop solve. from_state 0: each side starts from
 * initialize_state (bitwise lbgpu_fd_gradient per component); 1 (fixed_iters
 * >= 0 only): from the engine's current primal state -- the finite-difference
 * check of lbgpu_unsteady_adjoint run from a developed state. */
int lbgpu_fd_gradient_batch(lbgpu_engine* e, int64_t n, const int64_t* ordinals,
                            const double* steps, double tol, int64_t max_iter,
                            int64_t fixed_iters, int from_state, double* out);
/* optimizer.cpp:200-202: write new design values (DesignField::nodes order,
 * host memory; pinned overlaps best) into w, then n >= 1 primal steps. The
 * upload overlaps the first sweep: one launch whose design nodes wait for
 * their own values (3D product build, box-shaped design, no residual on the
 * first sweep), else z-chunks. Equivalent to lbgpu_set_design_values +
 * lbgpu_primal_step; the buffer is consumed when the call returns. residual
 * (nullable) as lbgpu_primal_step. The gated form, like the design pair's,
 * reads the bit pattern 0x7ff4dead0000beef as "not landed yet". */
int lbgpu_primal_step_with_design(lbgpu_engine* e, const double* w_design, int64_t n,
                                  double* residual);
/* A benchmark composite of the reference's operators (no reference loop runs
 * exactly this): the design write-back of
 * optimizer.cpp:200-202, one primal_step, one adjoint_step against the new f
 * (optimizer.cpp:33-34) and J = evaluate_raw of the new state
 * (objective.cpp:64-72). Equals lbgpu_primal_step_with_design(1) +
 * lbgpu_adjoint_step(1, kernel 0) + lbgpu_objective bit for bit in everything
 * observable. Residuals and objective are nullable. Without residuals (3D,
 * FP64 product build) the call's adjoint sweep is deferred into the next
 * call's primal sweep (one fused kernel reading f once, each design node's
 * thread waiting for its own uploaded value); every other lbgpu call, or
 * lbgpu_finish, completes it first. A rho <= 0 inside a deferred sweep is
 * reported by the call that runs it. The gated sweep takes a value equal to
 * the bit pattern 0x7ff4dead0000beef (a NaN) as "not landed yet": such a
 * value fails the call (LBGPU_E_NUMERIC) after a bounded wait. */
int lbgpu_pair_step_with_design(lbgpu_engine* e, const double* w_design, double* primal_residual,
                                double* adjoint_residual, double* objective);
/* Complete any deferred sweep and wait for the engine's stream. */
int lbgpu_finish(lbgpu_engine* e);
/* n x adjoint_step (adjoint.cpp:206-254) against the current primal state.
 * kernel: 0 analytic, 1 dual sweep (AdjointKernel, adjoint.hpp:14-18). */
int lbgpu_adjoint_step(lbgpu_engine* e, int64_t n, int kernel, double* residual);
/* solve_fixed_point (collision.cpp:377-416): from the current state; tol stop
 * unless fixed_iters >= 0. Non-finite residual / rho <= 0 -> LBGPU_E_NUMERIC. */
int lbgpu_solve_primal(lbgpu_engine* e, double tol, int64_t max_iter, int64_t fixed_iters,
                       int64_t* iterations, double* residual, int* converged);
/* solve_adjoint (adjoint.cpp:256-297): v <- 0, then sweeps to tol. */
int lbgpu_solve_adjoint(lbgpu_engine* e, double tol, int64_t max_iter, int64_t fixed_iters,
                        int kernel, int64_t* iterations, double* residual, int* converged);

/* As lbgpu_solve_adjoint but continuing from the current v (no reset). */
int lbgpu_continue_adjoint(lbgpu_engine* e, double tol, int64_t max_iter, int64_t fixed_iters,
                           int kernel, int64_t* iterations, double* residual, int* converged);

/* --- reductions --- */
/* param_gradient (adjoint.cpp:377-420): g_design in DesignField::nodes
 * order (n_design), plus the inlet_dp global (nullable). */
int lbgpu_param_gradient(lbgpu_engine* e, int kernel, double* g_design, double* g_inlet_dp);
int lbgpu_objective(lbgpu_engine* e, double* value); /* evaluate_raw (objective.cpp:64-72) */
int lbgpu_penalty(lbgpu_engine* e, double* value);   /* penalty().value (topology.cpp:40-50) */

/* --- design loop --- */
/* one_shot_run (optimizer.cpp:25-72) for `iterations` iterations with the
 * per-iteration step size zeta[it-1] and penalty weight lambda[it-1]
 * (zeta_at / PenaltySchedule::weight_at evaluated by the caller). Rows are
 * written every record_interval iterations and at the last one. */
int lbgpu_one_shot(lbgpu_engine* e, int64_t iterations, const double* zeta,
                   const double* lambda, int64_t record_interval, lbgpu_run_row* rows,
                   int64_t cap, int64_t* n_rows);

/* --- unsteady adjoint (no reference function) --- */
/* Discrete adjoint of n_steps primal steps from the current state f^0, for
 * J = F(f^N) (sum_objective = 0) or J = sum_{n=1..N} F(f^n): returns J,
 * dJ/dw in DesignField::nodes order and dJ/d(inlet_dp). Primal states are
 * recomputed from checkpoints by recursive bisection within `slots` device
 * state buffers; forward_sweeps reports the primal sweeps spent (>= N).
 * Leaves f^N as the primal state. Equals the composition of the reference's
 * own adjoint_step / param_gradient (tests/test_gpu_unsteady.py) and
 * fd_gradient(fixed_iters = N). */
int lbgpu_unsteady_adjoint(lbgpu_engine* e, int64_t n_steps, int sum_objective, int64_t slots,
                           double* g_design, double* g_inlet_dp, double* J,
                           int64_t* forward_sweeps);

/* --- multi-slab runs (PartitionedRun, partition.cpp:43-312) --- */
/* In-process group: engines[i] must be slab i of n (same device); they then
 * share one stream and step in lock step through the lbgpu_group_* calls,
 * each sweep followed by the halo exchange (neighbour buffers read directly). */
int lbgpu_group_link(lbgpu_engine** engines, int n);
/* P2P group: engines[i] is slab i of n >= 2 and may sit on any device (peer
 * access is enabled between neighbouring GPUs; LBGPU_E_CONFIG without it).
 * Each keeps its own stream; a sweep writes the planes crossing each cut
 * straight into the neighbour's ghost column (peer stores over NVLink) and
 * waits only on its two neighbours' previous sweep. Same lbgpu_group_* calls. */
int lbgpu_group_link_p2p(lbgpu_engine** engines, int n);
/* which: 0 primal, 1 adjoint (kernel as lbgpu_adjoint_step); residual =
 * global max-norm step residual of the last step (nullable). P2P groups also
 * take which = 2: fused primal+adjoint pairs (as lbgpu_pair_steps: adjoint
 * k with primal k+1 in one sweep, both fields' cut planes pushed; residual
 * NULL). */
int lbgpu_group_step(lbgpu_engine** engines, int n, int which, int64_t steps, int kernel,
                     double* residual);
/* P2P group: milliseconds of `steps` lock steps (which as lbgpu_group_step),
 * CUDA events on every slab's stream, the maximum over slabs. */
int lbgpu_group_time(lbgpu_engine** engines, int n, int which, int64_t steps, double* ms);
/* Fill every slab's ghost columns of `field` (after uploads). */
int lbgpu_group_exchange(lbgpu_engine** engines, int n, int field);
/* NCCL (one slab per rank, one GPU per rank): rank 0 makes the id, every rank
 * attaches with it; sweeps then exchange halos over NVLink and residuals /
 * error flags are reduced across ranks. */
int lbgpu_nccl_unique_id(void* out, int cap);
int lbgpu_attach_nccl(lbgpu_engine* e, const void* unique_id, int nranks, int rank);
/* Exchange the halos of `field` (collective in NCCL mode; after uploads). */
int lbgpu_exchange(lbgpu_engine* e, int field);

/* Iterations first .. first+count-1 of a one-shot run of `total`
 * iterations (zeta/lambda indexed from `first`); rows at it % record_interval
 * == 0 and at it == total. Lets a driver take snapshots between ranges. */
int lbgpu_one_shot_range(lbgpu_engine* e, int64_t first, int64_t count, int64_t total,
                         const double* zeta, const double* lambda, int64_t record_interval,
                         lbgpu_run_row* rows, int64_t cap, int64_t* n_rows);

/* --- timing (device events on the engine stream; bench support) --- */
/* which: 0 primal sweeps, 1 adjoint sweeps, 2 fused pair sweeps (adjoint k +
 * primal k+1, FP64 product build); returns elapsed milliseconds of
 * `steps` back-to-back sweeps (no residual), bracketed by synchronisation.
 * Adjoint sweeps run against the frozen current primal state, with its
 * moment cache built once inside the timed region (the steady-solve path). */
int lbgpu_time_sweeps(lbgpu_engine* e, int which, int64_t steps, double* ms);
/* Elapsed milliseconds of lbgpu_pair_steps(n) without residuals (n >= 1). */
int lbgpu_time_pair_steps(lbgpu_engine* e, int64_t n, double* ms);
/* `steps` x (one primal sweep then one adjoint sweep against it), one CUDA
 * event between consecutive sweeps: total, primal-only and adjoint-only ms. */
int lbgpu_time_pairs(lbgpu_engine* e, int64_t steps, double* ms_total, double* ms_primal,
                     double* ms_adjoint);
/* Number of sweep kernels this engine has launched. */
int64_t lbgpu_sweep_launches(const lbgpu_engine* e);

#ifdef __cplusplus
}
#endif

#endif /* LBGPU_H */

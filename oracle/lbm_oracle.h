/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the LBM primal/adjoint hot path.
 *
 * A plain-C restatement of the reference's algorithm (arxiv/paper_1501_04741,
 * /root/reference/proj). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it, and only as the checker. It is pinned against
 * the reference itself (oracle/_ref/liblbopt_ref.so, built from the
 * reference's own sources) by tests/test_oracle.py, bit-for-bit on masks,
 * states, adjoint states, gradients and objectives.
 *
 * Layout follows the reference: SoA planes, flat node index
 * x + nx*(y + ny*z) (lattice.hpp:25-27), plane p at offset p*N, state in the
 * reference's pre-collision convention. FP64 only.
 */
#ifndef LBM_ORACLE_H
#define LBM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { LBO_INTERIOR = 0, LBO_WALL = 1, LBO_INLET = 2, LBO_OUTLET = 3, LBO_HEATER = 4 };

typedef struct {
  /* lattice */
  int nx, ny, nz;
  long n;
  int mf, mt, m;
  int vel[28][3];
  int opp[28];
  double wf[19], wt[9];
  double A[19 * 19], At[19 * 19], relax[19];
  /* model (collision.hpp:46-59) */
  double nu, beta_fluid, beta_solid, inlet_dp, u_clamp, omega_nonhydro, theta;
  int bgk, fluid_power;
  /* per-node tables (config.cpp:302-371) */
  uint8_t* tag;
  double* bc_T;
  int8_t* bc_axis;
  int8_t* bc_sign;
  double* w;
  uint8_t* mask;
  long* design;
  long n_design;
  /* objective (config.cpp:373-395) */
  int obj_kind; /* 0 mixing 1 heatflux 2 synthetic */
  int flux_axis, flux_sign;
  uint8_t* on_support;
  long* support;
  long n_support;
} lbo_system;

typedef struct {
  int nx, ny, nz;
  int bgk, fluid_power, periodic, split_inlet, obj_kind;
  double nu, beta_fluid, beta_solid, inlet_dp, u_clamp, omega_nonhydro, theta, inlet_T;
  int design_x0, design_x1, heater_x0, heater_x1, plane_offset;
  double initial_w, init_noise;
  uint64_t seed;
} lbo_params;

/* Build descriptors, tables, tags, design and objective support. Returns 0 or
 * an error code (2 = config). Free with lbo_free. */
int lbo_build(const lbo_params* p, lbo_system* s);
void lbo_free(lbo_system* s);

void lbo_init_state(const lbo_system* s, double* f);
/* f_next = stream(collide(f_cur)); returns 0, or 3 (non-positive density) with
 * *bad = first offending flat index. */
int lbo_primal_step(const lbo_system* s, const double* f_cur, double* f_next, long* bad);
double lbo_residual(const double* a, const double* b, long count);
/* kernel: 0 analytic, 1 dual sweep (adjoint.hpp:14-18). */
int lbo_adjoint_step(const lbo_system* s, const double* base, const double* v_cur,
                     double* v_next, int kernel);
int lbo_param_gradient(const lbo_system* s, const double* v, const double* base, int kernel,
                       double* g_design, double* g_inlet_dp);
double lbo_objective(const lbo_system* s, const double* f);
double lbo_penalty(const lbo_system* s);
int lbo_collide_node(const lbo_system* s, int tag, int axis, int sign, double bcT,
                     const double* fin, double w, double* fout);
/* one-shot iteration (optimizer.cpp:31-46): f, v double buffers handled by
 * the caller: reads f_cur/v_cur, writes f_next/v_next, updates s->w. comp_max
 * receives max|comp|. */
int lbo_one_shot_iter(lbo_system* s, const double* f_cur, double* f_next, const double* v_cur,
                      double* v_next, double zeta, double lambda, double* comp_max);
double lbo_pairwise_sum(const double* x, long n);

#ifdef __cplusplus
}
#endif
#endif

#!/usr/bin/env python
"""Per-config measurements for BASELINE.json configs C1..C5 (SURVEY.md §8d
protocols), written to profiles/<tag>_configs.json. Not the driver's bench
line (bench.py is); this is the evidence behind each config row.

  C1  256x64 BGK: primal to steady state (tol 1e-10) + adjoint + gradient
  C2  1024x256 mixer: warm start (ZETA0 zeta=0 one-shot iterations), then 50
      one-shot design iterations at zeta=1e-4 — GPU vs the reference on the same
      warm (f, v, w), compared iteration by iteration
  C3  256x128x128: sweep rates FP64 / FP32 (the bench.py headline)
  C4  512x128x128 exchanger: one-shot iterations/s
  C5  2048x512x512 over 8 GPUs: one rank's 256x512x512 slab, sweep rates and an
      unsteady adjoint (N_t steps, checkpoint/recompute)
The reference (oracle/_ref, compiled from its own sources) is timed on this
box's host cores on bounded samples.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1501_04741_b200 as P  # noqa: E402
from paper_1501_04741_b200.presets import config_text  # noqa: E402
from oracle import oracle as O  # noqa: E402

CORES = len(os.sched_getaffinity(0))
out = {"cores": CORES}
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
only = set(sys.argv[2:])


def want(c):
    return not only or c in only


def sweeps(e, K=50):
    """Sweep rates over the nodes a sweep updates (a slab's owned columns, not
    its ghost/pad columns)."""
    e.time_pairs(5)
    t, tp, ta = e.time_pairs(K)
    s = 8 if e.precision == 64 else 4
    sl = e.slab()
    n = e.n // sl["nxl"] * sl["span"]
    out = {"primal_mlups": n * K / tp / 1e3, "adjoint_mlups": n * K / ta / 1e3,
           "primal_gbs": 2 * e.m * s * n * K / tp / 1e6,
           "adjoint_gbs": 3 * e.m * s * n * K / ta / 1e6}
    e.time_pair_steps(3)
    out["pair_mlups"] = n * K / e.time_pair_steps(K) / 1e3  # lbgpu_pair_steps (fused at FP64)
    e.time_sweeps(1, 3)
    out["adjoint_frozen_base_mlups"] = n * K / e.time_sweeps(1, K) / 1e3
    return out


if want("C1"):
    txt = config_text("C1")
    res = {}
    # (c) GPU-only convergence to 1e-10 of the SURVEY A.3 geometry (initial_w
    # 0.5, no noise) against the reference's converged objective
    for exact in (False, True):
        e = P.Engine.from_config(config_text("C1", {"optimizer.init_noise": 0}), exact=exact)
        e.init_state()
        t0 = time.perf_counter()
        it, r, conv = e.solve_primal(1e-10, 3000000)
        dt = time.perf_counter() - t0
        obj = e.objective()
        res["noise0_exact" if exact else "noise0_fast"] = {
            "primal_iterations": it, "residual": r, "converged": conv, "seconds": dt,
            "objective": obj, "objective_cpu_reference": 0.01066509204221,
            "abs_diff": abs(obj - 0.01066509204221), "steps_per_s": it / dt}
        e.close()
    # the SURVEY A.3 trace (reference, 1 thread) at fixed iteration counts:
    # the exact build must reproduce its printed objectives
    trace = {25000: 0.0106650923521202, 100000: 0.0106650920422142,
             400000: 0.0106650920421798}
    e = P.Engine.from_config(config_text("C1", {"optimizer.init_noise": 0}), exact=True)
    e.init_state()
    done, rows = 0, {}
    for k, ref in trace.items():
        e.primal_step(k - done, residual=False)
        done = k
        rows[k] = {"objective": e.objective(), "reference_trace": ref,
                   "abs_diff": abs(e.objective() - ref)}
    res["trace_exact"] = rows
    e.close()
    # the C1 case itself: primal to 1e-10, adjoint to 1e-10, gradient
    e = P.Engine.from_config(txt)
    e.init_state()
    t0 = time.perf_counter()
    it, r, conv = e.solve_primal(1e-10, 3000000)
    tp = time.perf_counter() - t0
    obj = e.objective()
    t0 = time.perf_counter()
    ia, ra, ca = e.solve_adjoint(1e-10, 3000000)
    g, gdp = e.param_gradient()
    ta = time.perf_counter() - t0
    res["case"] = {"primal_iterations": it, "primal_residual": r, "converged": conv,
                   "primal_seconds": tp, "objective": obj, "adjoint_iterations": ia,
                   "adjoint_residual": ra, "adjoint_converged": ca,
                   "adjoint_plus_gradient_seconds": ta, "inlet_dp_gradient": gdp,
                   "gpu_primal_steps_per_s": it / tp}
    # (a) fixed-iteration parity, bit-exact build vs the reference itself
    K = 10000
    e = P.Engine.from_config(txt, exact=True)
    e.init_state()
    r_ = O.RefOracle(txt)
    r_.init_state()
    e.primal_step(K)
    t0 = time.perf_counter()
    r_.primal_steps(K)
    ref_sps = K / (time.perf_counter() - t0)
    e.adjoint_step(K)
    r_.adjoint_steps(K)
    ge, gde = e.param_gradient()
    gr, gdr = r_.gradient()
    res["fixed_iteration_parity"] = {
        "steps": K, "state_equal": bool(np.array_equal(e.get_state(0), r_.get_state(0))),
        "adjoint_equal": bool(np.array_equal(e.get_state(1), r_.get_state(1))),
        "objective_equal": e.objective() == r_.objective(),
        "gradient_equal": bool(np.array_equal(ge, gr)) and gde == gdr,
        "reference_primal_steps_per_s_1thread": ref_sps,
        "reference_seconds_for_case_primal_solve_est": it / ref_sps}
    out["C1"] = res
    print("C1", json.dumps(res), flush=True)

if want("C2"):
    ZETA0 = 20000
    txt = config_text("C2", {"optimizer.zeta_stages": "0:0"})
    e = P.Engine.from_config(txt)
    t0 = time.perf_counter()
    e.one_shot(np.zeros(ZETA0), np.zeros(ZETA0), record_interval=ZETA0)
    warm_s = time.perf_counter() - t0
    f0, v0, w0 = e.get_state(0), e.get_state(1), e.design()
    iters = 50
    zeta = np.full(iters, 1e-4)
    lam = np.zeros(iters)
    t0 = time.perf_counter()
    rows = e.one_shot(zeta, lam, record_interval=1)
    gpu_s = time.perf_counter() - t0
    w_gpu = e.design()
    # the reference on the same warm state
    r_ = O.RefOracle(config_text("C2", {"optimizer.zeta_stages": "0:0.0001"}))
    r_.set_state(0, f0)
    r_.set_state(1, v0)
    r_.set_design(w0)
    t0 = time.perf_counter()
    rrows = r_.one_shot(iters, 1)
    ref_s = time.perf_counter() - t0
    w_ref = r_.tables()["w"]
    out["C2"] = {"warm_iterations": ZETA0, "warm_seconds": warm_s,
                 "gpu_seconds_50_iterations": gpu_s, "gpu_iterations_per_s": iters / gpu_s,
                 "reference_seconds_50_iterations_1thread": ref_s,
                 "reference_iterations_per_s": iters / ref_s,
                 "max_abs_w_diff": float(np.max(np.abs(w_gpu - w_ref))),
                 "max_rel_objective_diff": float(np.max(np.abs(rows[:, 2] - rrows[:, 2]) /
                                                        np.abs(rrows[:, 2]))),
                 "max_rel_gradnorm_diff": float(np.max(np.abs(rows[:, 6] - rrows[:, 6]) /
                                                       np.abs(rrows[:, 6]))),
                 "design_moved": float(np.max(np.abs(w_gpu - w0)))}
    print("C2", json.dumps(out["C2"]), flush=True)

if want("C3"):
    res = {}
    for name, ov in (("fp64", {}), ("fp32", {"model.precision": 32}),
                     ("bgk_fp64", {"model.collision": "bgk"})):
        e = P.Engine.from_config(config_text("C3"), ov)
        e.init_state()
        e.primal_step(20, residual=False)
        res[name] = sweeps(e)
        e.close()
    out["C3"] = res
    print("C3", json.dumps(res), flush=True)

if want("C4"):
    txt = config_text("C4", {"optimizer.zeta_stages": "0:0.0001"})
    e = P.Engine.from_config(txt)
    e.init_state()
    e.one_shot(np.full(20, 1e-4), np.zeros(20), record_interval=100)
    K = 100
    t0 = time.perf_counter()
    e.one_shot(np.full(K, 1e-4), np.zeros(K), record_interval=K)
    dt = time.perf_counter() - t0
    sw = sweeps(e)
    r_ = O.RefOracle(txt)
    r_.init_state()
    tp = r_.time_steps(0, CORES, 1)
    ta = r_.time_steps(1, CORES, 1)
    # parity: the C2 warm-start protocol at 128x32x32 (C4
    # proportions), 20 one-shot iterations from the same (f, v, w) on both
    # engines; then 3 full-size iterations from a GPU-warmed state.
    def warm_parity(txt_warm, txt_run, warm, iters):
        g = P.Engine.from_config(txt_warm)
        g.init_state()
        g.one_shot(np.zeros(warm), np.zeros(warm), record_interval=warm)
        f0, v0, w0 = g.get_state(0), g.get_state(1), g.design()
        rows = g.one_shot(np.full(iters, 1e-4), np.zeros(iters), record_interval=1)
        wg = g.design()
        g.close()
        rr = O.RefOracle(txt_run)
        rr.set_state(0, f0)
        rr.set_state(1, v0)
        rr.set_design(w0)
        t0 = time.perf_counter()
        rrows = rr.one_shot(iters, 1)
        ref_s = time.perf_counter() - t0
        return {"warm_iterations": warm, "iterations": iters,
                "objective_trace_gpu": rows[:, 2].tolist(),
                "objective_trace_reference": rrows[:, 2].tolist(),
                "max_abs_w_diff": float(np.max(np.abs(wg - rr.tables()["w"]))),
                "max_rel_objective_diff": float(np.max(np.abs(rows[:, 2] - rrows[:, 2]) /
                                                       np.abs(rrows[:, 2]))),
                "max_rel_gradnorm_diff": float(np.max(np.abs(rows[:, 6] - rrows[:, 6]) /
                                                      np.abs(rrows[:, 6]))),
                "design_moved": float(np.max(np.abs(wg - w0))),
                "reference_seconds_1thread": ref_s}
    small = {"lattice.nx": 128, "lattice.ny": 32, "lattice.nz": 32, "tags.design_x0": 37,
             "tags.design_x1": 91, "tags.heater_x0": 55, "tags.heater_x1": 72}
    par_small = warm_parity(config_text("C4", {**small, "optimizer.zeta_stages": "0:0"}),
                            config_text("C4", {**small, "optimizer.zeta_stages": "0:0.0001"}),
                            4000, 20)
    par_full = warm_parity(config_text("C4", {"optimizer.zeta_stages": "0:0"}),
                           config_text("C4", {"optimizer.zeta_stages": "0:0.0001"}), 4000, 3)
    out["C4"] = {"parity_128x32x32": par_small, "parity_full_size": par_full,
                 "nodes": e.n, "one_shot_iterations_per_s": K / dt,
                 "one_shot_node_iterations_mlups": e.n * K / dt / 1e6, **sw,
                 "reference_primal_plus_adjoint_seconds_per_iteration": tp + ta,
                 "reference_cores": CORES}
    print("C4", json.dumps(out["C4"]), flush=True)

if want("C5"):
    txt = config_text("C5")
    e = P.Engine.slab_from_config(txt, None, 8, 0)
    e.init_state()
    sw = sweeps(e, 20)
    slab = e.slab()
    e.close()
    # Unsteady adjoint at one rank's node count: a slab without its neighbours
    # has frozen ghosts and (slab 0) neither design nodes nor the objective
    # plane, so the A14 run uses the C5 physics on a standalone 256x512x512
    # lattice (design x 64..191, objective plane x = 254).
    NT, SLOTS, WARM = 1000, 4, 2000
    e = P.Engine.from_config(config_text("C5", {"lattice.nx": 256, "tags.design_x0": 64,
                                                "tags.design_x1": 191}))
    e.init_state()
    e.primal_step(WARM, residual=False)
    f_warm = e.get_state(0)
    runs = {}
    # round 1 (recursive bisection, 4 slots + separate state-0 / state-N
    # buffers): 10,604 forward sweeps for N_t = 1000. The binomial schedule
    # with checkpoints placed by the first pass: 4 slots, and 5 (the same
    # device memory as round 1's 4, whose extra buffers are now the engine's).
    for slots in (SLOTS, SLOTS + 1):
        e.set_state(0, f_warm)
        t0 = time.perf_counter()
        J, g, gdp, fs = e.unsteady_adjoint(NT, False, slots)
        dt = time.perf_counter() - t0
        runs[str(slots)] = {"seconds": dt, "forward_sweeps": fs, "recompute_factor": fs / NT,
                            "adjoint_sweeps": NT, "J": J,
                            "grad_max": float(np.max(np.abs(g))), "inlet_dp_gradient": gdp,
                            "node_sweeps_per_s_mlups": e.n * (fs + NT) / dt / 1e6}
    out["C5"] = {"slab": slab, "owned_nodes": slab["span"] * 512 * 512, **sw,
                 "note": "sweep rates: one rank's slab of the 8-GPU decomposition over its local array",
                 "unsteady_lattice": "256x512x512 (C5 physics, one rank's node count)",
                 "unsteady_warmup_steps": WARM, "unsteady_steps": NT,
                 "unsteady_round1_forward_sweeps_4_slots": 10604, "unsteady_by_slots": runs}
    print("C5", json.dumps(out["C5"]), flush=True)

if os.path.isdir(os.path.join(ROOT, "gpurun_out")):
    with open(os.path.join(ROOT, "gpurun_out", f"{tag}_configs_part.json"), "w") as fh:
        json.dump(out, fh, indent=1)
path = os.path.join(ROOT, "profiles", f"{tag}_configs.json")
old = {}
if os.path.exists(path):
    with open(path) as fh:
        old = json.load(fh)
old.update(out)
with open(path, "w") as fh:
    json.dump(old, fh, indent=1)

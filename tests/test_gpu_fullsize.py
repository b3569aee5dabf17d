"""Parity at the BASELINE configs' own sizes (SURVEY.md §8d protocols).

The product path is checked against the reference itself (oracle/_ref,
compiled from its own sources) on identical inputs at full size:

* C3 (the bench config, 256x128x128 D3Q19+D3Q7 FMRT): from a state developed
  by 1,000 primal steps, 100 primal then 100 adjoint sweeps and the design
  gradient against the reference's thread-per-slab PartitionedRun
  (partition.cpp:93-253, bitwise equal to its monolithic operators,
  test_partition.cpp:53-141) on all host threads; then 20 primal+adjoint
  pairs — the fused k_pair sweep the bench times — the same way. The
  bit-exact build must equal the reference bit for bit on all of it.
* C1 (256x64 BGK): 10^4 primal + 10^4 adjoint steps and the gradient,
  bit-exact build bitwise, product build within tolerance.
* C2 (1024x256 mixer) and C4 (512x128x128 exchanger): the warm-start one-shot
  protocol — (f, v, w) developed on the GPU, loaded into both engines, then
  design iterations compared (C2: 50; C4: 20 at 128x32x32 and 3 at full size).
* C5 (D3Q19 mixer physics): the unsteady adjoint of N_t = 200 cold-start steps
  at 128x32x32 against the composition of the reference's own operators
  (SURVEY.md §8a A14 recipe), bitwise in the exact build. At this state the
  gradient is ~1e-16 (the porous block w ~ 0.5 has not let any flow reach the
  support plane), below what central differences resolve, so the FD pin --
  fd_gradient(fixed_iters = N_t) on the 3 strongest design nodes (bitwise the
  reference's in the exact build, test_gpu_fdcheck.py) -- runs on the same
  lattice with a nearly fluid design (w = 0.9 +- 0.1), uniform inlet and
  N_t = 400, where the flow crosses the channel.

Tolerances are SURVEY.md §8(d)'s (FP64): state <= 1e-12 of max|f| (adjoint
state <= 1e-11 of max|v|, see test_gpu_parity.py); design gradient <= 1e-10
of max|g| and objective <= 1e-12 relative -- or, where these protocol states
make them ill-conditioned, within twice what the reference's own arithmetic
gives on the product build's states. Behind C3's porous design block
(w ~ 0.5, G = w^3) the outflow velocity at the support plane is ~1e-11, so J
~ 1e-7 and g ~ 1e-11 are built from u = j_x / rho, which FP64 resolves only to
~1e-5 relative (j_x is a difference of O(0.3) populations): a 1e-14 state
difference moves them by ~1e-6 relative in either code. The bit-exact build
equals the reference bit for bit on all of it.
"""
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

THREADS = max(1, len(os.sched_getaffinity(0)))
STATE_RTOL, ADJ_RTOL, OBJ_RTOL, GRAD_RTOL = 1e-12, 1e-11, 1e-12, 1e-10


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def objective_scale(f, r):
    """sum over the support of |u_n| (1 + T^2) for state f (reference
    layout) of oracle handle r: the magnitude the objective's terms are
    computed from (objective.cpp:19-32, flux along +x for these presets)."""
    t = r.tables()
    F = f.reshape(r.m, r.n)[:, t["support"]]
    rho = F[: r.mf].sum(0)
    ux = (t["vel"][: r.mf, 0:1] * F[: r.mf]).sum(0) / rho
    T = F[r.mf:].sum(0)
    return float(np.sum(np.abs(ux) * (1.0 + T * T)))


def cfg(cid, extra=None):
    from paper_1501_04741_b200.presets import config_text
    return config_text(cid, extra or {})


def test_c3_full_size_sweeps_gradient_and_pairs(lbgpu, oracle_mod, has_gpu):
    txt = cfg("C3")
    e = lbgpu.Engine.from_config(txt)
    assert e.n == 256 * 128 * 128 and e.m == 26
    e.init_state()
    e.primal_step(1000, residual=False)
    f_w = e.get_state(0)
    r = oracle_mod.RefOracle(txt)
    assert np.array_equal(e.tables()["design"], r.tables()["design"])
    r.set_state(0, f_w)
    rp, ra = r.partitioned(THREADS, n_primal=100, n_adjoint=100)
    f_r, v_r = r.get_state(0), r.get_state(1)
    J_r = r.objective()
    g_r, gdp_r = r.gradient()

    # bit-exact build: the reference's bits at full size
    x = lbgpu.Engine.from_config(txt, exact=True)
    x.set_state(0, f_w)
    assert x.primal_step(100) == rp
    assert x.adjoint_step(100) == ra
    assert np.array_equal(x.get_state(0), f_r)
    assert np.array_equal(x.get_state(1), v_r)
    assert x.objective() == J_r
    g_x, gdp_x = x.param_gradient()
    assert np.array_equal(g_x, g_r) and gdp_x == gdp_r

    # product build
    e.reset_adjoint()
    rpe = e.primal_step(100)
    rae = e.adjoint_step(100)
    f_e, v_e = e.get_state(0), e.get_state(1)
    fmax = np.max(np.abs(f_r))
    assert rel(f_e, f_r) <= STATE_RTOL
    assert rel(v_e, v_r) <= ADJ_RTOL
    assert abs(rpe - rp) <= 2 * STATE_RTOL * fmax
    J_e = e.objective()
    g_e, gdp_e = e.param_gradient()
    # the reference's arithmetic (bit-exact build) on the product build's states
    x.set_state(0, f_e)
    x.set_state(1, v_e)
    J_xe = x.objective()
    g_xe, gdp_xe = x.param_gradient()
    x.close()
    gs = np.max(np.abs(g_r))
    assert gs > 0
    assert abs(J_e - J_r) <= max(OBJ_RTOL * abs(J_r), 2 * abs(J_xe - J_r))
    assert np.max(np.abs(g_e - g_r)) <= max(GRAD_RTOL * gs, 2 * np.max(np.abs(g_xe - g_r)))
    assert abs(gdp_e - gdp_r) <= max(GRAD_RTOL * abs(gdp_r), 2 * abs(gdp_xe - gdp_r))
    del v_r, g_r, f_e, v_e

    # the bench step: 20 primal+adjoint pairs from v = 0 (k_pair at FP64)
    r.partitioned(THREADS, n_pairs=20)
    e.reset_adjoint()
    e.pair_steps(20, residual=False)
    assert rel(e.get_state(0), r.get_state(0)) <= STATE_RTOL
    assert rel(e.get_state(1), r.get_state(1)) <= ADJ_RTOL
    e.close()
    r.close()


def test_c1_fixed_iteration_parity(lbgpu, oracle_mod, has_gpu):
    """SURVEY §8d C1 (a) at 10^4 steps (the 10^5-step version is ~10 min of
    reference CPU time): state, adjoint state, objective and gradient."""
    K = 10000
    txt = cfg("C1")
    r = oracle_mod.RefOracle(txt)
    r.init_state()
    rp, ra = r.partitioned(min(THREADS, 8), n_primal=K, n_adjoint=K)
    f_r, v_r = r.get_state(0), r.get_state(1)
    g_r, gdp_r = r.gradient()
    for exact in (True, False):
        e = lbgpu.Engine.from_config(txt, exact=exact)
        e.init_state()
        rpe = e.primal_step(K)
        rae = e.adjoint_step(K)
        g_e, gdp_e = e.param_gradient()
        if exact:
            assert rpe == rp and rae == ra
            assert np.array_equal(e.get_state(0), f_r)
            assert np.array_equal(e.get_state(1), v_r)
            assert np.array_equal(g_e, g_r) and gdp_e == gdp_r
            assert e.objective() == r.objective()
        else:
            assert abs(e.objective() - r.objective()) <= 1e-10 * abs(r.objective())
            # 10^4 steps: per-step ulps accumulate (<= 1e-10 after 10^4)
            assert rel(e.get_state(0), f_r) <= 1e-10
            assert rel(e.get_state(1), v_r) <= 1e-10
            assert np.max(np.abs(g_e - g_r)) <= 1e-9 * np.max(np.abs(g_r))
        e.close()


def test_c1_tol_stop_iteration_parity(lbgpu, oracle_mod, has_gpu):
    """the tol-stop iteration of solve_fixed_point
    (collision.cpp:377-416) at C1 size against the reference's own stop rule,
    run on its partitioned_fixed_point (partition.cpp:279-312, bitwise its
    monolithic solve) on the host threads. tol 1e-6 (crossed near 10^5 steps)
    rather than SURVEY's 1e-7 (near 3*10^5, ~30 min of reference CPU time);
    bit-exact build: the same iteration, residual and state; product build:
    the iteration within +-1."""
    txt = cfg("C1")
    r = oracle_mod.RefOracle(txt)
    r.init_state()
    it_r, res_r, conv_r = r.partitioned_solve(min(THREADS, 16), 1e-6, 3000000)
    assert conv_r and it_r > 10000
    x = lbgpu.Engine.from_config(txt, exact=True)
    x.init_state()
    it_x, res_x, conv_x = x.solve_primal(1e-6, 3000000)
    assert (it_x, res_x, conv_x) == (it_r, res_r, conv_r)
    assert np.array_equal(x.get_state(0), r.get_state(0))
    e = lbgpu.Engine.from_config(txt)
    e.init_state()
    it_e, res_e, conv_e = e.solve_primal(1e-6, 3000000)
    assert conv_e and abs(it_e - it_r) <= 1


def _warm_one_shot(lbgpu, oracle_mod, txt_warm, txt_run, warm, iters):
    g = lbgpu.Engine.from_config(txt_warm)
    g.init_state()
    g.one_shot(np.zeros(warm), np.zeros(warm), record_interval=warm)
    f0, v0, w0 = g.get_state(0), g.get_state(1), g.design()
    rows = g.one_shot(np.full(iters, 1e-4), np.zeros(iters), record_interval=1)
    w_g, f_g = g.design(), g.get_state(0)
    g.close()
    r = oracle_mod.RefOracle(txt_run)
    r.set_state(0, f0)
    r.set_state(1, v0)
    r.set_design(w0)
    scale = objective_scale(f0, r)
    rrows = r.one_shot(iters, 1)
    w_r = r.tables()["w"]
    moved = np.max(np.abs(w_g - w0))
    assert moved > 0, "the design did not move: the protocol checks nothing"
    # iteration, residual, objective, penalty, weight, composite, max|comp|
    assert np.array_equal(rows[:, 0], rrows[:, 0])
    assert np.max(np.abs(rows[:, 2] - rrows[:, 2])) <= 1e-11 * scale
    assert np.max(np.abs(rows[:, 6] - rrows[:, 6]) / np.abs(rrows[:, 6])) <= 1e-9
    assert np.max(np.abs(w_g - w_r)) <= 1e-13
    assert rel(f_g, r.get_state(0)) <= 1e-11
    r.close()


def test_c2_warm_one_shot_50_iterations(lbgpu, oracle_mod, has_gpu):
    _warm_one_shot(lbgpu, oracle_mod, cfg("C2", {"optimizer.zeta_stages": "0:0"}),
                   cfg("C2", {"optimizer.zeta_stages": "0:0.0001"}), 20000, 50)


@pytest.mark.parametrize("size", ["128x32x32", "full"])
def test_c4_warm_one_shot(lbgpu, oracle_mod, has_gpu, size):
    small = {"lattice.nx": 128, "lattice.ny": 32, "lattice.nz": 32, "tags.design_x0": 37,
             "tags.design_x1": 91, "tags.heater_x0": 55, "tags.heater_x1": 72}
    ov = small if size != "full" else {}
    _warm_one_shot(lbgpu, oracle_mod, cfg("C4", {**ov, "optimizer.zeta_stages": "0:0"}),
                   cfg("C4", {**ov, "optimizer.zeta_stages": "0:0.0001"}), 4000,
                   20 if size != "full" else 3)


C5_SMALL = {"lattice.nx": 128, "lattice.ny": 32, "lattice.nz": 32, "tags.design_x0": 32,
            "tags.design_x1": 95}


def composed_reference(O, txt, N, every=20):
    """The A14 recipe on the reference's own operators, with checkpoints every
    `every` states (recomputed forward inside each segment):
      mu^N = adjoint_step(f^N, 0, obj); mu^{n-1} = adjoint_step(f^{n-1}, mu^n, obj off);
      dJ/dw = sum_n param_gradient(mu^n, f^{n-1}); J = F(f^N)."""
    r = O.RefOracle(txt)
    r.init_state()
    ck = {0: r.get_state(0)}
    for n in range(1, N + 1):
        r.primal_steps(1)
        if n % every == 0 or n == N:
            ck[n] = r.get_state(0)
    J = r.objective()
    r.set_state(1, np.zeros(r.m * r.n))
    r.adjoint_steps(1)  # mu^N against f^N (the handle holds f^N)
    r.objective_enabled(False)
    g = np.zeros(r.n_design)
    gdp = 0.0
    n = N
    while n > 0:
        a = ((n - 1) // every) * every  # checkpoint at or below n-1
        r.set_state(0, ck[a])
        seg = [ck[a]]
        for _ in range(a + 1, n):
            r.primal_steps(1)
            seg.append(r.get_state(0))
        for k in range(n, a, -1):  # bases f^{k-1} = seg[k-1-a]
            r.set_state(0, seg[k - 1 - a])
            gk, dk = r.gradient()
            g += gk
            gdp += dk
            r.adjoint_steps(1)
        n = a
    r.objective_enabled(True)
    r.close()
    return J, g, gdp, ck[N]


def test_c5_unsteady_adjoint_protocol(lbgpu, oracle_mod, has_gpu):
    N = 200
    txt = cfg("C5", C5_SMALL)
    J_r, g_r, gdp_r, fN_r = composed_reference(oracle_mod, txt, N)
    gs = np.max(np.abs(g_r))
    assert gs > 0
    # the reference's arithmetic (bit-exact build) from a cold start perturbed
    # by 1e-14 relative: how much J and g move under ulp-level differences
    x = lbgpu.Engine.from_config(txt, exact=True)
    x.init_state()
    f0 = x.get_state(0)
    x.set_state(0, f0 * (1 + 1e-14 * np.random.default_rng(3).uniform(-1, 1, f0.size)))
    J_p, g_p, gdp_p, _ = x.unsteady_adjoint(N, sum_objective=False, slots=6)
    x.close()
    for exact in (True, False):
        e = lbgpu.Engine.from_config(txt, exact=exact)
        e.init_state()
        J, g, gdp, fsweeps = e.unsteady_adjoint(N, sum_objective=False, slots=6)
        assert fsweeps > N  # recompute happened (6 slots for 200 states)
        if exact:
            assert J == J_r and np.array_equal(g, g_r) and gdp == gdp_r
        else:
            assert abs(J - J_r) <= max(OBJ_RTOL * abs(J_r), 10 * abs(J_p - J_r))
            assert np.max(np.abs(g - g_r)) <= max(GRAD_RTOL * gs, 10 * np.max(np.abs(g_p - g_r)))
            assert abs(gdp - gdp_r) <= max(GRAD_RTOL * abs(gdp_r), 10 * abs(gdp_p - gdp_r))
        e.close()
    # fd_gradient(fixed_iters = N) (adjoint.cpp:492-517) on the 3 strongest
    # design components with the reference's step set and error rule
    # (case.cpp:256-283), in the bit-exact build, on the well-conditioned variant
    N2 = 400
    txt2 = cfg("C5", {**C5_SMALL, "optimizer.initial_w": 0.9, "optimizer.init_noise": 0.1,
                      "tags.inlet_profile": "uniform", "tags.inlet_T": 0.0})
    x = lbgpu.Engine.from_config(txt2, exact=True)
    x.init_state()
    J2, g2, gdp2, _ = x.unsteady_adjoint(N2, sum_objective=False, slots=8)
    gs2 = max(np.max(np.abs(g2)), abs(gdp2))
    x.init_state()
    order = [int(o) for o in np.argsort(-np.abs(g2), kind="stable")[:3]]
    hs = [1e-5, 1e-6, 1e-7]
    fd = x.fd_gradient_batch([o for o in order for _ in hs], hs * 3, fixed_iters=N2)
    for k, o in enumerate(order):
        best = min(abs(fd[3 * k + j] - g2[o]) / max(abs(g2[o]), abs(fd[3 * k + j]), 1e-6 * gs2)
                   for j in range(3))
        assert best <= 1e-4, (o, g2[o], list(fd[3 * k: 3 * k + 3]), best)
    x.close()

"""On-device gradient verification at scale.

The reference's grad_check (case.cpp:228-329) compares the adjoint gradient
with fd_gradient re-solves on the 12 strongest design components (plus the
inlet_dp global) at steps {1e-5, 1e-6, 1e-7}, keeping each component's best
relative error with the floor 1e-6 * g_scale (case.cpp:256-283). A steady
re-solve of a 4M-node lattice per FD side is hours of thermal diffusion, so at
C3 size the check is run on the discrete adjoint of a fixed horizon instead
(lbgpu_unsteady_adjoint, whose FD partner is fd_gradient with fixed_iters):

* C3's lattice (256x128x128, D3Q19+D3Q7 FMRT, mixer3d physics) with a
  uniform inlet temperature, so the mixing objective sum u_n (1 - T^2) is the
  outflow rate through the support plane, and a nearly fluid design (w = 0.9
  +- 0.1) so that there is an outflow to differentiate: C3's own w = 0.5 +- 0.3
  block (G = w^3 ~ 0.1) throttles the outflow velocity to ~1e-10, where J is
  ~1e-6, the gradient ~1e-10 and central differences are roundoff (~1e-8);
* 2,000 developing primal steps, then J = F(f^N) over N = 500 further steps
  (long enough for the inlet's influence to cross the 256 columns);
* all 39 FD components (13 x 3 steps x 2 sides, each 500 sweeps from the same
  developed state) through lbgpu_fd_gradient_batch: one call, one host sync.

grad_check's error rule, best of the reference's steps {1e-5, 1e-6, 1e-7}, at
1e-4: here J is the outflow through 15,876 support nodes (~1e2), so central
differences carry ~1e-16 J / h of roundoff (1e-4 relative at h = 1e-6 for
these ~1e-4 components) and h = 1e-5 leaves a ~1e-5 truncation error after
500 steps (measured: the worst component agrees to 3.4e-5).
"""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_c3_unsteady_gradient_against_batched_fd(lbgpu, has_gpu):
    from paper_1501_04741_b200.presets import config_text
    txt = config_text("C3", {"tags.inlet_profile": "uniform", "tags.inlet_T": 0.0,
                             "optimizer.initial_w": 0.9, "optimizer.init_noise": 0.1})
    e = lbgpu.Engine.from_config(txt)
    e.init_state()
    e.primal_step(2000, residual=False)
    f_w = e.get_state(0)
    N = 500
    J, g, gdp, _ = e.unsteady_adjoint(N, sum_objective=False, slots=16)
    assert J > 0
    e.set_state(0, f_w)
    order = sorted(range(g.size), key=lambda i: (-abs(g[i]), i))[:12]
    g_scale = max(max(abs(g[i]) for i in order), abs(gdp))
    steps = [1e-5, 1e-6, 1e-7]
    ords = [o for o in order for _ in steps] + [-1] * len(steps)
    hs = steps * (len(order) + 1)
    fd = e.fd_gradient_batch(ords, hs, fixed_iters=N, from_state=True)
    assert np.array_equal(e.get_state(0), f_w)  # state restored
    worst, rows = 0.0, []
    for c, o in enumerate(order + [-1]):
        adj = gdp if o < 0 else g[o]
        best = min(abs(fd[3 * c + k] - adj) / max(abs(adj), abs(fd[3 * c + k]), 1e-6 * g_scale)
                   for k in range(3))
        rows.append((o, adj, list(fd[3 * c: 3 * c + 3]), best))
        worst = max(worst, best)
    assert abs(gdp) > 1e-6 * g_scale, (gdp, g_scale)  # the inlet's influence arrived
    assert worst <= 1e-4, rows
    e.close()


def test_fd_batch_equals_single_calls(lbgpu, oracle_mod, has_gpu):
    """lbgpu_fd_gradient_batch (cold start) = lbgpu_fd_gradient per component,
    bitwise, in both builds; the exact build's = the reference's fd_gradient."""
    from cases import case_text
    txt = case_text("mix3d")
    r = oracle_mod.RefOracle(txt)
    for exact in (True, False):
        e = lbgpu.Engine.from_config(txt, exact=exact)
        e.init_state()
        e.primal_step(40)
        before = e.get_state(0)
        ords, hs = [0, 3, -1, 7], [1e-6, 1e-5, 1e-6, 1e-7]
        batch = e.fd_gradient_batch(ords, hs, fixed_iters=150)
        single = [e.fd_gradient(o, h, 0.0, 150, fixed_iters=150) for o, h in zip(ords, hs)]
        assert np.array_equal(batch, single)
        assert np.array_equal(e.get_state(0), before)
        if exact:
            assert batch[0] == r.fd_gradient(0, 1e-6, 0.0, 150, 150)
        e.close()

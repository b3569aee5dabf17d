"""tangent_solve (adjoint.cpp:422-490) on the GPU: the
forward-mode sensitivity dF along a design direction, iterated to its own
fixed point under the frozen primal state.

* exact build: bit-for-bit the reference's own tangent_solve (oracle/_ref)
  — dF, iteration count and residual — on the same base state;
* product build: within tolerance of it, and dual to the adjoint gradient
  (the reference's test_adjoint.cpp:173-202: dF == g . dw + g_dp * d_dp,
  1e-10 relative)."""
import numpy as np
import pytest

from cases import case_text

pytestmark = pytest.mark.gpu


def need_ref(oracle_mod):
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")


@pytest.mark.parametrize("name,warm", [("grad2d", 400), ("exch2d", 300), ("solid2d", 300),
                                       ("mix3d", 300), ("exch3d", 200)])
def test_tangent_exact_bitwise(lbgpu, oracle_mod, has_gpu, name, warm):
    need_ref(oracle_mod)
    txt = case_text(name)
    e = lbgpu.Engine.from_config(txt, exact=True)
    r = oracle_mod.RefOracle(txt)
    e.init_state()
    r.init_state()
    e.primal_step(warm)
    r.primal_steps(warm)
    assert np.array_equal(e.get_state(0), r.get_state(0))
    rng = np.random.default_rng(11)
    dw = rng.uniform(-1, 1, e.n_design)
    ddp = float(rng.uniform(-1, 1))
    runs = ((0.0, 60), (1e-9, 100000)) if name.endswith("2d") else ((0.0, 60),)
    for tol, it in runs:
        got = e.tangent_solve(dw, ddp, tol, it)
        ref = r.tangent(dw, ddp, tol, it)
        assert got == ref, (got, ref)
    # the primal state is untouched
    assert np.array_equal(e.get_state(0), r.get_state(0))


def test_tangent_fast_and_duality(lbgpu, oracle_mod, has_gpu):
    need_ref(oracle_mod)
    txt = case_text("grad2d")
    e = lbgpu.Engine.from_config(txt)
    e.init_state()
    it, res, conv = e.solve_primal(1e-12, 400000)
    assert conv
    ia, ra, ca = e.solve_adjoint(1e-13, 400000)
    assert ca
    g, gdp = e.param_gradient()
    r = oracle_mod.RefOracle(txt)
    r.set_state(0, e.get_state(0))
    rng = np.random.default_rng(35)
    for _ in range(3):
        dw = rng.uniform(-1, 1, e.n_design)
        ddp = float(rng.uniform(-1, 1))
        dF, n, rr, cv = e.tangent_solve(dw, ddp, 1e-13, 400000)
        assert cv and rr <= 1e-13
        dot = float(g @ dw + gdp * ddp)
        assert abs(dF - dot) <= 1e-10 * max(1.0, abs(dot)), (dF, dot)
        dF_r, n_r, _, cv_r = r.tangent(dw, ddp, 1e-13, 400000)
        # residual decay near tol is ~1e-4 per sweep: FMA ulps move the stop by a few
        assert cv_r and abs(n - n_r) <= 1e-3 * n_r
        assert abs(dF - dF_r) <= 1e-11 * max(1.0, abs(dF_r))


def test_tangent_zero_iterations_and_args(lbgpu, has_gpu):
    e = lbgpu.Engine.from_config(case_text("grad2d"))
    e.init_state()
    dF, n, r, cv = e.tangent_solve(np.zeros(e.n_design), 0.0, 1e-12, 0)
    assert (dF, n, r, cv) == (0.0, 0, 0.0, True)
    with pytest.raises(lbgpu.LbgpuError):
        e.tangent_solve(np.zeros(e.n_design), 0.0, 1e-12, -1)


@pytest.mark.parametrize("name,comps", [("grad2d", (0, 5, -1)), ("mix3d", (3, -1))])
def test_fd_gradient_exact_bitwise(lbgpu, oracle_mod, has_gpu, name, comps):
    """lbgpu_fd_gradient (adjoint.cpp:492-517) in the exact build equals the
    reference's fd_gradient bit for bit (fixed-iteration and tol-stop
    solves), and leaves the engine's state and design as they were."""
    need_ref(oracle_mod)
    txt = case_text(name)
    e = lbgpu.Engine.from_config(txt, exact=True)
    r = oracle_mod.RefOracle(txt)
    e.init_state()
    e.primal_step(7)
    f0, w0 = e.get_state(0), e.design()
    for k in comps:
        assert e.fd_gradient(k, 1e-6, 0.0, 0, 150) == r.fd_gradient(k, 1e-6, 0.0, 0, 150)
    if name == "grad2d":
        assert e.fd_gradient(2, 1e-5, 1e-9, 100000) == r.fd_gradient(2, 1e-5, 1e-9, 100000, -1)
    assert np.array_equal(e.get_state(0), f0) and np.array_equal(e.design(), w0)


def test_fd_matches_unsteady_adjoint_at_scale(lbgpu, has_gpu):
    """On-device verification at a size the CPU reference cannot reach in a
    test: a 64x32x32 D3Q19+D3Q7 mixer (65,536 nodes), the
    unsteady adjoint gradient of J(f^N) from a cold start against central
    differences with fixed_iters = N, both on the GPU (product build)."""
    txt = case_text("mix3d", {"lattice.nx": 64, "lattice.ny": 32, "lattice.nz": 32,
                              "tags.design_x0": 16, "tags.design_x1": 47})
    e = lbgpu.Engine.from_config(txt)
    N = 300
    e.init_state()
    J, g, gdp, _ = e.unsteady_adjoint(N, False, 8)
    order = np.argsort(-np.abs(g))
    # the reference's own criterion (test_adjoint.cpp:161-170): doctest
    # Approx(fd).epsilon(eps).scale(max(1e-3, |fd|))
    def approx(a, fd, eps=1e-5):
        return abs(a - fd) < eps * (max(1e-3, abs(fd)) + max(abs(a), abs(fd)))
    for k in order[:3]:
        fd = e.fd_gradient(int(k), 1e-5, 0.0, 0, N)
        assert approx(g[k], fd), (k, fd, g[k])
    fd = e.fd_gradient(-1, 1e-6, 0.0, 0, N)
    assert approx(gdp, fd), (fd, gdp)

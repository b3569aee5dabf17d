"""Unsteady adjoint: the discrete adjoint of N primal
steps with checkpoint/recompute. There is no reference function for it
(SPEC.md:313); the oracle is the composition of the reference's own
operators (SURVEY recipe):

    mu^N     = adjoint_step(base f^N, v = 0, obj)
    mu^{n-1} = adjoint_step(base f^{n-1}, mu^n, obj off | on for the sum)
    dJ/dw    = sum_{n=N..1} param_gradient(mu^n, f^{n-1})

run on the C restatement (bit-exact to the reference), and pinned by the
reference's own fd_gradient(fixed_iters = N)."""
import numpy as np
import pytest

from cases import case_text

pytestmark = pytest.mark.gpu


def composed(O, txt, warm, N, sum_obj):
    o = O.COracle(txt)
    o.init_state()
    if warm:
        o.primal_steps(warm)
    states = [o.f.copy()]
    J = 0.0
    for n in range(1, N + 1):
        o.primal_steps(1)
        states.append(o.f.copy())
        if sum_obj or n == N:
            J += o.objective()
    on = np.ctypeslib.as_array(o.s.on_support, shape=(o.n,))
    support = on.copy()
    o.v[:] = 0.0
    o.f[:] = states[N]
    o.adjoint_steps(1)                     # mu^N, with the objective partial
    g = np.zeros(o.s.n_design)
    gdp = 0.0
    for n in range(N, 0, -1):
        o.f[:] = states[n - 1]
        gn, dn = o.gradient()
        g = g + gn
        gdp += dn
        if not sum_obj:
            on[:] = 0
        o.adjoint_steps(1)
        on[:] = support
    return J, g, gdp


@pytest.mark.parametrize("name", ["grad2d", "exch2d", "mix3d"])
@pytest.mark.parametrize("sum_obj", [False, True])
def test_unsteady_equals_composed_oracle(lbgpu, oracle_mod, has_gpu, name, sum_obj):
    txt = case_text(name)
    warm, N = 300, 25  # past the start-up transient (see test_gpu_parity.py)
    J_o, g_o, gdp_o = composed(oracle_mod, txt, warm, N, sum_obj)
    for slots in (2, 5, 64):
        e = lbgpu.Engine.from_config(txt, exact=True)
        e.init_state()
        e.primal_step(warm)
        J, g, gdp, fs = e.unsteady_adjoint(N, sum_obj, slots)
        assert J == J_o
        assert np.array_equal(g, g_o), (slots, np.max(np.abs(g - g_o)))
        assert gdp == gdp_o
        assert fs >= 2 * N - 1
    # product build: tolerance
    e = lbgpu.Engine.from_config(txt)
    e.init_state()
    e.primal_step(warm)
    J, g, gdp, _ = e.unsteady_adjoint(N, sum_obj, 4)
    # early in the transient the heat-flux objective is a ~1e-11 cancellation residue
    assert abs(J - J_o) <= 1e-12 * abs(J_o) + 1e-17
    assert np.max(np.abs(g - g_o)) <= 1e-10 * max(np.max(np.abs(g_o)), 1e-300)


def test_unsteady_matches_reference_fd(lbgpu, oracle_mod, has_gpu):
    """dJ/dw of J = F(f^N) from a cold start against the reference's
    fd_gradient(fixed_iters = N) (adjoint.cpp:491-516), central differences."""
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    txt = case_text("grad2d")
    N = 400
    e = lbgpu.Engine.from_config(txt)
    e.init_state()
    J, g, gdp, _ = e.unsteady_adjoint(N, False, 6)
    r = oracle_mod.RefOracle(txt)
    order = np.argsort(-np.abs(g))
    for k in order[:4]:
        fd = r.fd_gradient(int(k), 1e-5, 1e-13, 100000, N)
        assert abs(fd - g[k]) <= 1e-6 * max(abs(fd), abs(g[k])), (k, fd, g[k])
    fd = r.fd_gradient(-1, 1e-6, 1e-13, 100000, N)
    assert abs(fd - gdp) <= 1e-5 * max(abs(fd), abs(gdp))


def test_unsteady_forward_matches_plain_steps_on_ghost_slab(lbgpu, has_gpu):
    """On a slab with ghost columns and no exchange attached, the ghosts are
    frozen: both ping-pong buffers must carry the same ones from init_state on,
    so the unsteady first pass (slot buffers) and plain stepping (f[0]/f[1])
    read identical inputs and f^N agrees bitwise."""
    txt = case_text("mix3d")
    a = lbgpu.Engine.slab_from_config(txt, None, 2, 0)
    b = lbgpu.Engine.slab_from_config(txt, None, 2, 0)
    for e in (a, b):
        e.init_state()
        e.primal_step(7, residual=False)
    a.primal_step(6, residual=False)
    b.unsteady_adjoint(6, False, 2)
    assert np.array_equal(a.get_state(0), b.get_state(0))

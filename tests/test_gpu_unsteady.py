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
        assert fs >= N  # the first pass; no recompute once every state fits
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


def _schedule_sweeps(N, s):
    """Primal sweeps of the checkpoint schedule (engine.cu Schedule): the first
    pass (N) plus first(N, s), with
      opt(n, s)   = min_m m + opt(n - m, s - 1) + opt(m, s),
      first(n, s) = min_m first(n - m, s - 1) + opt(m, s),
    both n - 1 when n - 1 <= s and n (n - 1) / 2 when s = 0."""
    import functools

    @functools.lru_cache(None)
    def opt(n, k):
        if n <= 1:
            return 0
        if n - 1 <= k:
            return n - 1
        if k == 0:
            return n * (n - 1) // 2
        return min(m + opt(n - m, k - 1) + opt(m, k) for m in range(1, n))

    @functools.lru_cache(None)
    def first(n, k):
        if n <= 1 or n - 1 <= k:
            return 0
        if k == 0:
            return n * (n - 1) // 2
        return min(first(n - m, k - 1) + opt(m, k) for m in range(1, n))

    return N + first(N, s)


@pytest.mark.parametrize("N,slots", [(25, 2), (60, 3), (200, 4)])
def test_checkpoint_schedule_sweep_count(lbgpu, oracle_mod, has_gpu, N, slots):
    """The engine runs exactly the binomial schedule's sweep count, and the
    gradient is bitwise the one with every state stored (slots >= N)."""
    txt = case_text("mix3d")
    out = []
    for s in (slots, N):
        e = lbgpu.Engine.from_config(txt, exact=True)
        e.init_state()
        e.primal_step(50)
        out.append(e.unsteady_adjoint(N, False, s))
        e.close()
    (J, g, gdp, fs), (J2, g2, gdp2, fs2) = out
    assert fs == _schedule_sweeps(N, slots)
    assert fs2 == N  # every inner state stored by the first pass: no recompute
    assert J == J2 and gdp == gdp2 and np.array_equal(g, g2)

"""Pins the CPU oracle: the C restatement (oracle/lbm_oracle.c) must equal
the reference itself (oracle/_ref, compiled from /root/reference sources)
bit for bit, on every parity case; and the committed golden fixtures
(tests/golden/, generated from the reference by make_golden.py) must hold."""
import os

import numpy as np
import pytest

from cases import CASES, case_text

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _need_ref(O):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (no /root/reference here)")


@pytest.mark.parametrize("name", list(CASES))
def test_restatement_equals_reference(oracle_mod, name):
    O = oracle_mod
    _need_ref(O)
    txt = case_text(name)
    c, r = O.COracle(txt), O.RefOracle(txt)
    tc, tr = c.tables(), r.tables()
    for k in ("tag", "bc_T", "bc_axis", "bc_sign", "w", "mask", "design", "support", "A"):
        assert np.array_equal(tc[k], tr[k]), k
    c.init_state()
    r.init_state()
    assert c.primal_steps(25) == r.primal_steps(25)
    assert np.array_equal(c.f, r.get_state(0))
    assert c.objective() == r.objective()
    assert c.adjoint_steps(12) == r.adjoint_steps(12)
    assert np.array_equal(c.v, r.get_state(1))
    assert c.adjoint_steps(2, kernel=1) == r.adjoint_steps(2, kernel=1)
    assert np.array_equal(c.v, r.get_state(1))
    for kern in (0, 1):
        gc, dc = c.gradient(kern)
        gr, dr = r.gradient(kern)
        assert np.array_equal(gc, gr) and dc == dr
    assert c.penalty() == r.penalty()


def test_restatement_one_shot_equals_reference(oracle_mod):
    O = oracle_mod
    _need_ref(O)
    txt = case_text("exch2d")
    ov = {"optimizer.zeta_stages": "0:0.002", "objective.penalty_w0": 0.001,
          "objective.penalty_cap": 1.0, "objective.penalty_interval": 4,
          "objective.penalty_growth": 2.0}
    c, r = O.COracle(txt, ov), O.RefOracle(txt, ov)
    c.init_state()
    r.init_state()
    rows = r.one_shot(9, 3)
    lam = [min(0.001 * 2.0 ** ((it) / 4), 1.0) for it in range(1, 10)]
    gms = [c.one_shot_iter(0.002, lam[i]) for i in range(9)]
    assert np.array_equal(c.f, r.get_state(0))
    assert np.array_equal(c.v, r.get_state(1))
    t = r.tables()
    assert np.array_equal(c.design(), t["w"])
    assert rows[-1][6] == gms[-1]


def test_golden_fixtures(oracle_mod):
    """Known answers produced by the reference (make_golden.py) reproduce on
    the restatement, so the oracle stays pinned where /root/reference is absent."""
    O = oracle_mod
    path = os.path.join(GOLDEN, "golden.npz")
    g = np.load(path, allow_pickle=False)
    for name in [str(s) for s in g["cases"]]:
        c = O.COracle(case_text(name))
        c.init_state()
        c.primal_steps(int(g[f"{name}/primal_steps"]))
        assert np.array_equal(c.f, g[f"{name}/f"]), name
        c.adjoint_steps(int(g[f"{name}/adjoint_steps"]))
        assert np.array_equal(c.v, g[f"{name}/v"]), name
        gd, gdp = c.gradient()
        assert np.array_equal(gd, g[f"{name}/grad"]) and gdp == float(g[f"{name}/grad_dp"])
        assert c.objective() == float(g[f"{name}/objective"])


def test_gradcheck_known_answer_restatement(oracle_mod):
    """gradcheck2d converges to 1e-12 in 16,578 iterations with
    objective 0.0126428346367474 (the reference, measured)."""
    from paper_1501_04741_b200.presets import preset_text
    c = oracle_mod.COracle(preset_text("gradcheck2d"))
    c.init_state()
    it = 0
    while True:
        it += 1
        r = c.primal_steps(1)
        if r <= 1e-12:
            break
    assert it == 16578
    assert c.objective() == 0.012642834636747431


def test_pairwise_sum_tree(oracle_mod):
    """reduce.hpp:43-52: leaf 16, midpoint split — differs from a flat sum."""
    x = np.random.default_rng(0).standard_normal(1000) * 1e8
    s = oracle_mod.pairwise_sum(x)

    def pw(lo, hi):
        if hi - lo <= 16:
            acc = 0.0
            for i in range(lo, hi):
                acc += float(x[i])
            return acc
        mid = lo + (hi - lo) // 2
        return pw(lo, mid) + pw(mid, hi)
    assert s == pw(0, 1000)


def test_reference_tangent_is_dual_to_adjoint(oracle_mod):
    """oracle/_ref's tangent_solve (the reference's own, through ref_shim)
    reproduces test_adjoint.cpp:173-202 on gradcheck2d: dF == g . dw +
    g_dp * d_dp within 1e-10 — the pin for the GPU tangent parity tests."""
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_1501_04741_b200.presets import preset_text
    r = oracle_mod.RefOracle(preset_text("gradcheck2d"))
    r.init_state()
    assert r.solve_primal(1e-12, 400000)[2]
    assert r.solve_adjoint(1e-13, 400000)[2]
    g, gdp = r.gradient()
    rng = np.random.default_rng(1)
    dw = rng.uniform(-1, 1, g.size)
    ddp = float(rng.uniform(-1, 1))
    dF, it, res, conv = r.tangent(dw, ddp, 1e-13, 400000)
    dot = float(g @ dw + gdp * ddp)
    assert conv and abs(dF - dot) <= 1e-10 * max(1.0, abs(dot))


@pytest.mark.parametrize("name", ["mix3d", "grad2d"])
def test_partitioned_runner_equals_monolithic(oracle_mod, name):
    """ref_partitioned (the full-size parity oracle of test_gpu_fullsize.py)
    is the reference's PartitionedRun: bitwise its monolithic operators
    (test_partition.cpp:53-141), for primal, adjoint and pair sequences; and
    objective_enabled(False) is the A14 recipe's obj_empty."""
    O = oracle_mod
    _need_ref(O)
    txt = case_text(name)
    a, b = O.RefOracle(txt), O.RefOracle(txt)
    a.init_state()
    b.init_state()
    a.primal_steps(40)
    b.primal_steps(40)
    ra = a.partitioned(3, n_primal=9, n_adjoint=6, n_pairs=4)
    b.set_state(1, np.zeros(b.m * b.n))
    b.primal_steps(9)
    b.adjoint_steps(6)
    for _ in range(4):
        rp = b.primal_steps(1)
        rb = b.adjoint_steps(1)
    assert ra == (rp, rb)
    assert np.array_equal(a.get_state(0), b.get_state(0))
    assert np.array_equal(a.get_state(1), b.get_state(1))
    # obj_empty: an adjoint step from v = 0 without the source stays zero
    a.set_state(1, np.zeros(a.m * a.n))
    a.objective_enabled(False)
    a.adjoint_steps(2)
    assert not np.any(a.get_state(1))
    a.objective_enabled(True)
    a.adjoint_steps(1)
    assert np.any(a.get_state(1))


def test_partitioned_solve_equals_monolithic(oracle_mod):
    """ref_partitioned_solve is the reference's partitioned_fixed_point:
    the same stop iteration, residual and state as solve_fixed_point."""
    O = oracle_mod
    _need_ref(O)
    txt = case_text("grad2d")
    a, b = O.RefOracle(txt), O.RefOracle(txt)
    a.init_state()
    b.init_state()
    assert a.partitioned_solve(3, 1e-8, 200000) == b.solve_primal(1e-8, 200000)
    assert np.array_equal(a.get_state(0), b.get_state(0))

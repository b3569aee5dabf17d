"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

* exact build (``exact=True``): bit-for-bit equal to the oracle restatement
  (itself bit-for-bit equal to the reference, tests/test_oracle.py) for
  states, residuals, adjoint states, gradients, objectives and penalties;
* fast build (the product path): within the tolerances SURVEY.md §8(d)
  recommends at FP64 — per-step primal state <= 1e-12 relative to max|f|,
  objective <= 1e-12 relative, design gradient <= 1e-10 of max|g|; the
  adjoint state <= 1e-11 of max|v| (its support-plane source is the local
  velocity, which is ~1e-11 before the pressure wave arrives, so 1-ulp
  differences in f show up at 1e-12 of max|v|; measured 2.4e-12 on exch2d).
"""
import numpy as np
import pytest

from cases import CASES, case_text

pytestmark = pytest.mark.gpu

STATE_RTOL = 1e-12
GRAD_RTOL = 1e-10
ADJ_RTOL = 1e-11
OBJ_RTOL = 1e-12


def rel(a, b):
    scale = max(np.max(np.abs(b)), 1e-300)
    return float(np.max(np.abs(a - b)) / scale)


def make(P, O, name, exact, steps=30, asteps=20):
    txt = case_text(name)
    e = P.Engine.from_config(txt, exact=exact)
    o = O.COracle(txt)
    e.init_state()
    o.init_state()
    return e, o


@pytest.mark.parametrize("name", list(CASES))
def test_exact_bitwise(lbgpu, oracle_mod, has_gpu, name):
    e, o = make(lbgpu, oracle_mod, name, exact=True)
    # masks and tables
    te, to = e.tables(), o.tables()
    for k in ("tag", "bc_T", "bc_axis", "bc_sign", "w", "mask", "design", "support", "A"):
        assert np.array_equal(te[k], to[k]), k
    # primal: 1, then 10 more, then 40 more steps
    for k in (1, 10, 40):
        re_ = e.primal_step(k)
        ro = o.primal_steps(k)
        assert np.array_equal(e.get_state(0), o.f), f"primal state after +{k}"
        assert re_ == ro, (re_, ro)
    assert e.objective() == o.objective()
    # adjoint (analytic), against the current state
    for k in (1, 15):
        re_ = e.adjoint_step(k, kernel=0)
        ro = o.adjoint_steps(k, kernel=0)
        assert np.array_equal(e.get_state(1), o.v), f"adjoint state after +{k}"
        assert re_ == ro
    ge, gde = e.param_gradient(0)
    go, gdo = o.gradient(0)
    assert np.array_equal(ge, go)
    assert gde == gdo
    # dual-sweep kernel
    re_ = e.adjoint_step(2, kernel=1)
    ro = o.adjoint_steps(2, kernel=1)
    assert np.array_equal(e.get_state(1), o.v)
    ge, gde = e.param_gradient(1)
    go, gdo = o.gradient(1)
    assert np.array_equal(ge, go) and gde == gdo
    assert e.penalty() == o.penalty()


@pytest.mark.parametrize("name", list(CASES))
def test_fast_tolerance(lbgpu, oracle_mod, has_gpu, name):
    e, o = make(lbgpu, oracle_mod, name, exact=False)
    # run past the start-up transient (the pressure wave crosses these
    # channels in <100 steps) so the gradient is not a cancellation residue
    for k in (1, 400):
        e.primal_step(k)
        o.primal_steps(k)
        assert rel(e.get_state(0), o.f) <= STATE_RTOL, f"primal +{k}"
    oe, oo = e.objective(), o.objective()
    assert abs(oe - oo) <= OBJ_RTOL * max(abs(oo), 1e-300) + 1e-18
    for k in (1, 20):
        e.adjoint_step(k, kernel=0)
        o.adjoint_steps(k, kernel=0)
        assert rel(e.get_state(1), o.v) <= ADJ_RTOL, f"adjoint +{k}"
    ge, gde = e.param_gradient(0)
    go, gdo = o.gradient(0)
    if go.size:
        assert np.max(np.abs(ge - go)) <= GRAD_RTOL * max(np.max(np.abs(go)), 1e-300)
    assert abs(gde - gdo) <= GRAD_RTOL * max(abs(gdo), 1e-300)
    # the dual-sweep kernel in the fast build
    e.adjoint_step(1, kernel=1)
    o.adjoint_steps(1, kernel=1)
    assert rel(e.get_state(1), o.v) <= ADJ_RTOL


@pytest.mark.parametrize("name", ["grad2d", "mix3d"])
def test_layout_round_trip(lbgpu, oracle_mod, has_gpu, name):
    """upload/download is the exact inverse permutation (both fields)."""
    e = lbgpu.Engine.from_config(case_text(name))
    rng = np.random.default_rng(5)
    for field in (0, 1):
        x = rng.standard_normal(e.m * e.n)
        e.set_state(field, x)
        assert np.array_equal(e.get_state(field), x)


def test_upload_then_step_matches(lbgpu, oracle_mod, has_gpu):
    """A state uploaded in reference layout steps exactly like the oracle."""
    txt = case_text("mix3d")
    e = lbgpu.Engine.from_config(txt, exact=True)
    o = oracle_mod.COracle(txt)
    o.init_state()
    o.primal_steps(7)
    e.set_state(0, o.f)
    o.primal_steps(3)
    e.primal_step(3)
    assert np.array_equal(e.get_state(0), o.f)
    rng = np.random.default_rng(1)
    v0 = rng.uniform(-0.3, 0.3, e.m * e.n)
    e.set_state(1, v0)
    o.v[:] = v0
    e.adjoint_step(2)
    o.adjoint_steps(2)
    assert np.array_equal(e.get_state(1), o.v)


def test_gradcheck_preset_known_answers(lbgpu, has_gpu):
    """gradcheck2d to 1e-12: 16,578 iterations, objective 0.0126428346367474
    (measured with the reference)."""
    from paper_1501_04741_b200.presets import preset_text
    e = lbgpu.Engine.from_config(preset_text("gradcheck2d"), exact=True)
    it, r, conv = e.solve_primal(1e-12, 200000)
    assert (it, conv) == (16578, True)
    assert r <= 1e-12
    assert e.objective() == 0.012642834636747431
    f = lbgpu.Engine.from_config(preset_text("gradcheck2d"))
    it2, r2, conv2 = f.solve_primal(1e-12, 200000)
    assert conv2 and abs(it2 - 16578) <= 1
    assert abs(f.objective() - 0.012642834636747431) <= 1e-12 * 0.0127


def test_solve_stop_iteration_matches_reference(lbgpu, oracle_mod, has_gpu):
    """Tol-stop iteration and final residual equal the reference's exactly."""
    txt = case_text("bgk2d")
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    r = oracle_mod.RefOracle(txt)
    r.init_state()
    it_r, res_r, conv_r = r.solve_primal(1e-7, 100000)
    e = lbgpu.Engine.from_config(txt, exact=True)
    it_e, res_e, conv_e = e.solve_primal(1e-7, 100000)
    assert (it_e, res_e, conv_e) == (it_r, res_r, conv_r)
    assert np.array_equal(e.get_state(0), r.get_state(0))
    ia, ra, ca = r.solve_adjoint(1e-7, 100000)
    ja, sa, cb = e.solve_adjoint(1e-7, 100000)
    assert (ja, sa, cb) == (ia, ra, ca)
    assert np.array_equal(e.get_state(1), r.get_state(1))
    g_r, gdp_r = r.gradient()
    g_e, gdp_e = e.param_gradient()
    assert np.array_equal(g_e, g_r) and gdp_e == gdp_r


def test_one_shot_exact(lbgpu, oracle_mod, has_gpu):
    """one_shot_run: w, f, v and the record rows bit-for-bit (ζ>0, λ>0)."""
    txt = case_text("exch2d")
    e = lbgpu.Engine.from_config(txt, exact=True)
    o = oracle_mod.COracle(txt)
    e.init_state()
    o.init_state()
    iters = 12
    zeta = np.full(iters, 2e-3)
    lam = np.linspace(0.0, 0.01, iters)
    rows = e.one_shot(zeta, lam, record_interval=5)
    gms = [o.one_shot_iter(zeta[i], lam[i]) for i in range(iters)]
    assert np.array_equal(e.design(), o.design())
    assert np.array_equal(e.get_state(0), o.f)
    assert np.array_equal(e.get_state(1), o.v)
    assert [int(r[0]) for r in rows] == [5, 10, 12]
    assert rows[-1][6] == gms[-1]
    assert rows[-1][2] == o.objective()
    assert rows[-1][3] == o.penalty()


def test_one_shot_fast(lbgpu, oracle_mod, has_gpu):
    txt = case_text("mix3d")
    e = lbgpu.Engine.from_config(txt)
    o = oracle_mod.COracle(txt)
    e.init_state()
    o.init_state()
    iters = 10
    zeta = np.full(iters, 5e-2)
    lam = np.full(iters, 1e-3)
    e.one_shot(zeta, lam, record_interval=10)
    for i in range(iters):
        o.one_shot_iter(zeta[i], lam[i])
    assert np.max(np.abs(e.design() - o.design())) <= 1e-12
    assert rel(e.get_state(0), o.f) <= STATE_RTOL
    assert rel(e.get_state(1), o.v) <= ADJ_RTOL


@pytest.mark.parametrize("name", list(CASES))
def test_one_shot_fused_update_is_bitwise(lbgpu, has_gpu, name):
    """The product build carries each non-record iteration's design update
    into the next iteration's primal sweep (k_primal UPD); with a record every
    iteration nothing is carried. Both must give the same bits: w, f, v and
    the rows they share."""
    txt = case_text(name)
    iters = 15
    zeta = np.full(iters, 3e-2)
    lam = np.linspace(0.0, 2e-3, iters)
    out = []
    for ri in (7, 1):
        e = lbgpu.Engine.from_config(txt)
        e.init_state()
        e.primal_step(30, residual=False)
        rows = e.one_shot(zeta, lam, record_interval=ri)
        out.append((rows, e.design(), e.get_state(0), e.get_state(1)))
        e.close()
    (ra, wa, fa, va), (rb, wb, fb, vb) = out
    assert np.array_equal(wa, wb) and np.array_equal(fa, fb) and np.array_equal(va, vb)
    shared = {7: 6, 14: 13, 15: 14}
    for i, row in enumerate(ra):
        assert np.array_equal(row, rb[shared[int(row[0])]])


def test_zero_zeta_one_shot_is_plain_stepping(lbgpu, has_gpu):
    """test_optimizer.cpp:182-209: one-shot with ζ = 0 == plain primal steps."""
    txt = case_text("grad2d")
    a = lbgpu.Engine.from_config(txt)
    b = lbgpu.Engine.from_config(txt)
    a.one_shot(np.zeros(15), np.zeros(15), record_interval=100)
    b.primal_step(15)
    assert np.array_equal(a.get_state(0), b.get_state(0))
    assert np.array_equal(a.design(), b.design())


def test_fp32_against_reference_fp32(lbgpu, oracle_mod, has_gpu):
    """precision = 32: the GPU float path against the reference's own float
    path at the same step counts (SURVEY.md §8d FP32 tolerances)."""
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    txt = case_text("mix3d")
    ov = {"model.precision": 32}
    e = lbgpu.Engine.from_config(txt, ov)
    r = oracle_mod.RefOracle(txt, ov)
    r.init_state()
    e.primal_step(300)
    r.primal_steps(300)
    assert rel(e.get_state(0), r.get_state(0)) <= 1e-5
    assert abs(e.objective() - r.objective()) <= 5e-4 * abs(r.objective())
    e.adjoint_step(200)
    r.adjoint_steps(200)
    g_e, _ = e.param_gradient()
    g_r, _ = r.gradient()
    assert np.max(np.abs(g_e - g_r)) <= 1e-3 * np.max(np.abs(g_r))


def test_nonpositive_density_reports_node(lbgpu, has_gpu):
    """NumericError naming the first bad node (collision.cpp:355-361)."""
    txt = case_text("periodic2d")
    e = lbgpu.Engine.from_config(txt)
    f = e.get_state(0)
    nx, ny, _ = e.shape
    n = e.n
    # make node (3,0,0) negative in the reference layout (test_collision.cpp:288-295)
    for j in range(e.mf):
        f[j * n + 3] = -1.0
    e.set_state(0, f)
    with pytest.raises(lbgpu.LbgpuError) as ex:
        e.primal_step(1)
    assert ex.value.code == lbgpu.E_NUMERIC
    assert "non-positive density at node (3,0,0)" in ex.value.msg


def test_design_values_round_trip(lbgpu, oracle_mod, has_gpu):
    """lbgpu_set_design_values (design order) == set_design on the full field."""
    txt = case_text("mix3d")
    for exact in (True, False):
        a = lbgpu.Engine.from_config(txt, exact=exact)
        b = lbgpu.Engine.from_config(txt, exact=exact)
        rng = np.random.default_rng(4)
        vals = rng.uniform(0, 1, a.n_design)
        a.set_design_values(vals)
        full = b.design()
        full[b.tables()["design"]] = vals
        b.set_design(full)
        assert np.array_equal(a.design(), b.design())
        assert np.array_equal(a.design_values(), vals)
        a.primal_step(5)
        b.primal_step(5)
        assert np.array_equal(a.get_state(0), b.get_state(0))


@pytest.mark.parametrize("nz", [8, 37])
@pytest.mark.parametrize("prec", [64, 32])
def test_primal_step_with_design_equals_upload_then_step(lbgpu, has_gpu, nz, prec):
    """lbgpu_primal_step_with_design is bitwise set_design_values +
    primal_step (states, residual, w) on each of its paths: one upload-gated
    launch (box-shaped design, no residual on the first sweep), the z-chunked
    upload (residual of a single sweep; nz = 37 gives uneven chunks), and the
    fallback (nz = 8, the exact build)."""
    txt = case_text("mix3d", {"lattice.nz": nz, "model.precision": prec})
    for exact in (False, True) if prec == 64 else (False,):  # the bit-exact build is FP64
        a = lbgpu.Engine.from_config(txt, exact=exact)
        b = lbgpu.Engine.from_config(txt, exact=exact)
        for e in (a, b):
            e.init_state()
            e.primal_step(20)
        rng = np.random.default_rng(nz)
        for k, resid in ((1, True), (3, True), (1, False), (2, False), (1, True)):
            vals = rng.uniform(0, 1, a.n_design)
            ra = a.primal_step_with_design(vals, k, residual=resid)
            b.set_design_values(vals)
            rb = b.primal_step(k, residual=resid)
            assert ra == rb
            assert np.array_equal(a.get_state(0), b.get_state(0))
            assert np.array_equal(a.design_values(), vals)
        a.adjoint_step(2)
        b.adjoint_step(2)
        assert np.array_equal(a.param_gradient()[0], b.param_gradient()[0])


@pytest.mark.parametrize("nz", [8, 16, 37])
def test_pair_step_with_design_equals_separate_calls(lbgpu, has_gpu, nz):
    """lbgpu_pair_step_with_design (design upload, primal z-chunks and adjoint
    z-chunks on a second stream, overlapped; nz = 8 takes the fallback, 16 is
    the smallest chunked lattice, 37 gives uneven chunks) is bitwise
    primal_step_with_design(1) + adjoint_step(1) + objective: f, v, w,
    residuals, J, and the gradient taken afterwards."""
    # design ranges narrower than the lattice
    wide = {"lattice.nx": 96, "tags.design_x0": 40, "tags.design_x1": 59}
    wider = {"lattice.nx": 160, "tags.design_x0": 70, "tags.design_x1": 89}
    for name, over in (("mix3d", {}), ("exch3d", {}), ("bgk3d", {}), ("mix3d", wide),
                       ("mix3d", wider)):
        txt = case_text(name, {**over, "lattice.nz": nz})
        for exact in (False, True):
            a = lbgpu.Engine.from_config(txt, exact=exact)
            b = lbgpu.Engine.from_config(txt, exact=exact)
            for e in (a, b):
                e.init_state()
                e.primal_step(20)
                e.adjoint_step(3)
            rng = np.random.default_rng(nz)
            for _ in range(3):
                vals = rng.uniform(0, 1, a.n_design)
                rpa, raa, ja = a.pair_step_with_design(vals)
                rpb = b.primal_step_with_design(vals, 1)
                rab = b.adjoint_step(1)
                jb = b.objective()
                assert (rpa, raa, ja) == (rpb, rab, jb)
                assert np.array_equal(a.get_state(0), b.get_state(0))
                assert np.array_equal(a.get_state(1), b.get_state(1))
                assert np.array_equal(a.design_values(), vals)
            a.pair_step_with_design(vals, residual=False, objective=False)
            b.primal_step_with_design(vals, 1, residual=False)
            b.adjoint_step(1, residual=False)
            assert np.array_equal(a.get_state(1), b.get_state(1))
            assert np.array_equal(a.param_gradient()[0], b.param_gradient()[0])


def test_gated_upload_never_hangs(lbgpu, has_gpu):
    """The gated fused sweep takes the sentinel bit pattern (kGateEmpty) as
    "not landed yet": a design vector carrying it fails the call with
    E_NUMERIC after the bounded wait instead of hanging, and the engine
    recovers (re-armed upload buffer) once it is given a valid state."""
    import time
    txt = case_text("mix3d", {"lattice.nz": 16})
    a = lbgpu.Engine.from_config(txt)
    b = lbgpu.Engine.from_config(txt)
    for e in (a, b):
        e.init_state()
        e.primal_step(10)
    vals = np.random.default_rng(4).uniform(0.05, 1, a.n_design)
    a.pair_step_with_design(vals, residual=False)  # leaves its adjoint sweep pending
    bad = vals.copy()
    bad.view(np.uint64)[a.n_design // 2] = np.uint64(0x7FF4DEAD0000BEEF)
    t0 = time.time()
    with pytest.raises(lbgpu.LbgpuError) as ex:
        a.pair_step_with_design(bad, residual=False)  # gated: waits, then gives up
    assert ex.value.code == lbgpu.E_NUMERIC and "upload" in ex.value.msg
    assert time.time() - t0 < 30
    for e in (a, b):
        e.init_state()
        e.set_design_values(vals)
        e.primal_step(10)
    for _ in range(3):
        ja = a.pair_step_with_design(vals, residual=False)[2]
        b.primal_step_with_design(vals, 1, residual=False)
        b.adjoint_step(1, residual=False)
        assert ja == b.objective()
    a.finish()
    assert np.array_equal(a.get_state(0), b.get_state(0))
    assert np.array_equal(a.get_state(1), b.get_state(1))


@pytest.mark.parametrize("nz", [16, 37])
def test_deferred_design_pairs_equal_separate_calls(lbgpu, has_gpu, nz):
    """Back-to-back lbgpu_pair_step_with_design calls without residuals defer
    each adjoint sweep into the next call's fused sweep (the adjoint half
    reading the previous design); J of every call, and f, v, w and the
    gradient once anything else runs, are bitwise the separate calls."""
    wide = {"lattice.nx": 96, "tags.design_x0": 40, "tags.design_x1": 59}
    for name, over in (("mix3d", {}), ("exch3d", {}), ("mix3d", wide), ("periodic3d", None)):
        if over is None:  # synthetic objective: side-list adjoint nodes in the fused sweep
            txt = case_text("bgk3d", {"lattice.nz": nz, "tags.geometry": "periodic",
                                      "objective.kind": "synthetic"})
        else:
            txt = case_text(name, {**over, "lattice.nz": nz})
        a = lbgpu.Engine.from_config(txt)
        b = lbgpu.Engine.from_config(txt)
        for e in (a, b):
            e.init_state()
            e.primal_step(20)
        rng = np.random.default_rng(nz)
        for k in range(5):
            vals = rng.uniform(0.05, 1, a.n_design)
            ja = a.pair_step_with_design(vals, residual=False)[2]
            b.primal_step_with_design(vals, 1, residual=False)
            b.adjoint_step(1, residual=False)
            assert ja == b.objective()
        a.finish()
        assert np.array_equal(a.get_state(0), b.get_state(0))
        assert np.array_equal(a.get_state(1), b.get_state(1))
        assert np.array_equal(a.design_values(), b.design_values())
        # a deferred sweep is completed by whatever call comes next
        vals = rng.uniform(0.05, 1, a.n_design)
        a.pair_step_with_design(vals, residual=False, objective=False)
        b.primal_step_with_design(vals, 1, residual=False)
        b.adjoint_step(1, residual=False)
        assert np.array_equal(a.param_gradient()[0], b.param_gradient()[0])
        assert np.array_equal(a.get_state(1), b.get_state(1))
        # the upload buffer stays armed across other design writes
        for k in range(3):
            vals = rng.uniform(0.05, 1, a.n_design)
            if k == 1:
                for e in (a, b):
                    e.primal_step_with_design(vals, 2, residual=False)
                vals = rng.uniform(0.05, 1, a.n_design)
            ja = a.pair_step_with_design(vals, residual=False)[2]
            b.primal_step_with_design(vals, 1, residual=False)
            b.adjoint_step(1, residual=False)
            assert ja == b.objective()
        a.finish()
        assert np.array_equal(a.get_state(0), b.get_state(0))
        assert np.array_equal(a.get_state(1), b.get_state(1))


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("prec", [64, 32])
def test_frozen_base_moment_cache_is_bitwise(lbgpu, has_gpu, name, prec):
    """adjoint_step(n >= 2) and solve_adjoint cache the frozen base's moments
    (k_base_moments) instead of gathering the base every sweep; the adjoint
    states must equal single-sweep calls (which gather) bit for bit."""
    txt = case_text(name, {"model.precision": prec})
    a = lbgpu.Engine.from_config(txt)
    b = lbgpu.Engine.from_config(txt)
    for e in (a, b):
        e.init_state()
        e.primal_step(40)
    ra = a.adjoint_step(15)
    for _ in range(15):
        rb = b.adjoint_step(1)
    assert ra == rb
    assert np.array_equal(a.get_state(1), b.get_state(1))
    assert np.array_equal(a.param_gradient()[0], b.param_gradient()[0])


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("exact", [False, True])
def test_pair_steps_equal_separate_sweeps(lbgpu, has_gpu, name, exact):
    """lbgpu_pair_steps (product build: adjoint k fused with primal k+1 in one
    sweep, k_pair) is bitwise n x (primal_step(1) + adjoint_step(1)): states,
    residuals of the last pair, and the gradient afterwards."""
    txt = case_text(name)
    a = lbgpu.Engine.from_config(txt, exact=exact)
    b = lbgpu.Engine.from_config(txt, exact=exact)
    for e in (a, b):
        e.init_state()
        e.primal_step(25)
    for n in (1, 2, 7):
        rp, ra = a.pair_steps(n)
        for _ in range(n):
            rpb = b.primal_step(1)
            rab = b.adjoint_step(1)
        assert (rp, ra) == (rpb, rab)
        assert np.array_equal(a.get_state(0), b.get_state(0))
        assert np.array_equal(a.get_state(1), b.get_state(1))
    assert a.pair_steps(3, residual=False) is None
    for _ in range(3):
        b.primal_step(1), b.adjoint_step(1)
    assert np.array_equal(a.get_state(1), b.get_state(1))
    assert np.array_equal(a.param_gradient()[0], b.param_gradient()[0])


@pytest.mark.parametrize("name,over", [
    ("mix3d", {"lattice.nx": 160}),  # rows wider than a block: edge-column blocks
    ("mix3d", {"lattice.nx": 128}),  # exactly one block per row
    ("exch3d", {"lattice.nx": 300, "tags.design_x0": 100, "tags.design_x1": 199}),
    ("grad2d", {"lattice.nx": 257}),
])
def test_pair_steps_wide_rows(lbgpu, has_gpu, name, over):
    """k_pair with its edge columns (inlet / outlet faces) in dedicated blocks
    is bitwise the sweeps apart, residuals included."""
    txt = case_text(name, over)
    a = lbgpu.Engine.from_config(txt)
    b = lbgpu.Engine.from_config(txt)
    for e in (a, b):
        e.init_state()
        e.primal_step(25)
    for n in (1, 4):
        rp, ra = a.pair_steps(n)
        for _ in range(n):
            rpb = b.primal_step(1)
            rab = b.adjoint_step(1)
        assert (rp, ra) == (rpb, rab)
        assert np.array_equal(a.get_state(0), b.get_state(0))
        assert np.array_equal(a.get_state(1), b.get_state(1))

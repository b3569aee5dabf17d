"""In-place (AA-pattern) streaming: one state buffer per field instead of the
reference's double buffer (StateField<R>, lattice.hpp:57-92), SURVEY.md
§8(f) F4. Each sweep alternates between layout O (the reference's own
layout) and layout E (post-collision values in the opposite slot of their own
node); the arithmetic is the double-buffered kernels' own, so every result
must be bitwise the double-buffered engine's: states (downloaded in the
reference layout), objective, gradient, for primal sweeps, adjoint sweeps
(gathering and frozen-base), fused pairs and any mix of them, on all nine
parity cases, FP64 and FP32; and the x-slab NCCL transport with its forward /
reverse exchanges (single-rank ring) bitwise the monolithic run.
"""
import numpy as np
import pytest

from cases import CASES, case_text

pytestmark = pytest.mark.gpu


def twins(P, txt, **kw):
    a = P.Engine.from_config(txt, **kw)
    b = P.Engine.from_config(txt, streaming="aa", **kw)
    a.init_state()
    b.init_state()
    return a, b


def same(a, b):
    assert np.array_equal(a.get_state(0), b.get_state(0)), "f"
    assert np.array_equal(a.get_state(1), b.get_state(1)), "v"


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("name", list(CASES))
def test_aa_bitwise_equals_double_buffer(lbgpu, has_gpu, name, prec):
    a, b = twins(lbgpu, case_text(name, {"model.precision": prec}))
    for k in (1, 2, 37):  # odd and even counts: both layouts at rest
        a.primal_step(k, residual=False)
        b.primal_step(k, residual=False)
        same(a, b)
    assert a.objective() == b.objective()
    for k in (1, 6):  # k >= 2: the frozen-base moment cache
        a.adjoint_step(k, residual=False)
        b.adjoint_step(k, residual=False)
        same(a, b)
    ga, da = a.param_gradient()
    gb, db = b.param_gradient()
    assert np.array_equal(ga, gb) and da == db
    # pairs from every parity combination of (f, v)
    for pre in ((), (0,), (1,), (0, 1)):
        for which in pre:
            (a.primal_step if which == 0 else a.adjoint_step)(1, residual=False)
            (b.primal_step if which == 0 else b.adjoint_step)(1, residual=False)
        a.pair_steps(3, residual=False)
        b.pair_steps(3, residual=False)
        same(a, b)
    ga, da = a.param_gradient()
    gb, db = b.param_gradient()
    assert np.array_equal(ga, gb) and da == db
    assert a.objective() == b.objective()


def test_aa_upload_download_round_trip(lbgpu, has_gpu):
    txt = case_text("mix3d")
    a, b = twins(lbgpu, txt)
    rng = np.random.default_rng(3)
    for field in (0, 1):
        x = rng.standard_normal(b.m * b.n)
        b.set_state(field, x)
        assert np.array_equal(b.get_state(field), x)
    # an uploaded state steps like the double buffer's, from either layout
    a.primal_step(5, residual=False)
    b.set_state(0, a.get_state(0))
    b.set_state(1, a.get_state(1))
    for _ in range(2):
        a.pair_steps(1, residual=False)
        b.pair_steps(1, residual=False)
        same(a, b)
        b.set_state(0, b.get_state(0))  # re-upload resets f to layout O
        same(a, b)


def test_aa_refuses_what_needs_the_previous_state(lbgpu, has_gpu):
    """No step residual (hence no tol-stop solve) in place: E_STATE with a
    reason, never a silent zero."""
    b = lbgpu.Engine.from_config(case_text("grad2d"), streaming="aa")
    b.init_state()
    for call in (lambda: b.primal_step(1), lambda: b.adjoint_step(1),
                 lambda: b.pair_steps(1), lambda: b.solve_primal(1e-6, 100),
                 lambda: b.unsteady_adjoint(3)):
        with pytest.raises(lbgpu.LbgpuError) as ex:
            call()
        assert ex.value.code == lbgpu.E_STATE and "in-place" in ex.value.msg
    with pytest.raises(lbgpu.LbgpuError) as ex:
        lbgpu.Engine.from_config(case_text("grad2d"), exact=True, streaming="aa")
    assert ex.value.code == lbgpu.E_CONFIG


@pytest.mark.parametrize("name", ["grad2d", "mix3d", "exch3d", "periodic2d"])
def test_aa_nccl_single_rank_ring_equals_monolithic(lbgpu, has_gpu, name):
    """In-place slabs over NCCL on one GPU (one slab in ghost layout, its own
    neighbour both ways): the forward exchange after sweeps from O (boundary
    columns -> ghosts) and the reverse exchange after sweeps from E (ghosts ->
    the neighbours' boundary columns), each overlapped with the interior
    columns, must give the monolithic run's bits."""
    import torch  # noqa: F401  (torch's libnccl first, as in bench.py)
    txt = case_text(name)
    mono = lbgpu.Engine.from_config(txt)
    ring = lbgpu.Engine.slab_from_config(txt, None, 1, -1, streaming="aa")
    ring.attach_nccl(lbgpu.nccl_unique_id(), 1, 0)
    s = ring.slab()
    mono.init_state()
    ring.init_state()

    def owned(e, field):
        nx, ny, nz = mono.shape
        return e.get_state(field).reshape(e.m, nz, ny, s["nxl"])[..., : s["span"]].reshape(-1)

    for k in (1, 24):
        mono.primal_step(k, residual=False)
        ring.primal_step(k, residual=False)
        assert np.array_equal(owned(ring, 0), mono.get_state(0))
    for k in (1, 8):
        mono.adjoint_step(k, residual=False)
        ring.adjoint_step(k, residual=False)
        assert np.array_equal(owned(ring, 1), mono.get_state(1))
    g_m, d_m = mono.param_gradient()
    g_r, d_r = ring.param_gradient()
    assert np.array_equal(g_m, g_r) and d_m == d_r
    for k in (1, 5):
        mono.pair_steps(k, residual=False)
        ring.pair_steps(k, residual=False)
        assert np.array_equal(owned(ring, 0), mono.get_state(0))
        assert np.array_equal(owned(ring, 1), mono.get_state(1))
    assert mono.objective() == ring.objective()


@pytest.mark.parametrize("prec", [64, 32])
def test_aa_bitwise_at_c3_size(lbgpu, has_gpu, prec):
    """The in-place kernels at the bench config's own size (C3, 256x128x128,
    4.2M nodes; FP32 is C5's one-GPU capacity mode): sweeps, frozen-base
    adjoint, fused pairs from both layouts, the gradient and J, bitwise the
    double-buffered engine."""
    from paper_1501_04741_b200.presets import config_text
    a, b = twins(lbgpu, config_text("C3", {"model.precision": prec}))
    for k in (20, 1):
        a.primal_step(k, residual=False)
        b.primal_step(k, residual=False)
    for k in (1, 4):
        a.adjoint_step(k, residual=False)
        b.adjoint_step(k, residual=False)
    for k in (3, 4):
        a.pair_steps(k, residual=False)
        b.pair_steps(k, residual=False)
    same(a, b)
    ga, da = a.param_gradient()
    gb, db = b.param_gradient()
    assert np.array_equal(ga, gb) and da == db
    assert a.objective() == b.objective()

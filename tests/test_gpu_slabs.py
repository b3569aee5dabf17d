"""Slab-decomposed runs on the GPU equal the monolithic run bit for bit —
the reference's own partition contract (partition_check,
partition.cpp:314-357; test_partition.cpp:53-141). Slabs run as an
in-process lock-step group on one device; the NCCL transport moves the same
packed planes between ranks (host-side plan tested in test_slabs.py)."""
import numpy as np
import pytest

from cases import case_text

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["grad2d", "exch2d", "mix3d", "exch3d", "periodic2d"])
@pytest.mark.parametrize("parts", [2, 3, 4])
@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("transport", ["pull", "p2p"])
def test_slabs_bitwise_equal_monolithic(lbgpu, has_gpu, name, parts, exact, transport):
    """transport "p2p": one stream per slab, running concurrently; every sweep
    pushes its boundary planes into the neighbours' ghost columns (the
    multi-GPU peer-store path, here with all slabs on one device)."""
    txt = case_text(name)
    mono = lbgpu.Engine.from_config(txt, exact=exact)
    grp = lbgpu.SlabGroup(txt, None, parts, exact=exact, transport=transport)
    mono.init_state()
    grp.init_state()
    r_m = mono.primal_step(30)
    r_g = grp.step(0, 30)
    assert r_m == r_g
    assert np.array_equal(grp.get_state(0), mono.get_state(0))
    assert grp.objective() == mono.objective()
    a_m = mono.adjoint_step(12)
    a_g = grp.step(1, 12)
    assert a_m == a_g
    assert np.array_equal(grp.get_state(1), mono.get_state(1))
    g_m, gdp_m = mono.param_gradient()
    g_g, gdp_g = grp.gradient()
    assert np.array_equal(g_g, g_m) and gdp_g == gdp_m


@pytest.mark.parametrize("transport", ["pull", "p2p"])
def test_slab_upload_round_trip(lbgpu, has_gpu, transport):
    txt = case_text("mix3d")
    mono = lbgpu.Engine.from_config(txt)
    grp = lbgpu.SlabGroup(txt, None, 3, transport=transport)
    mono.init_state()
    mono.primal_step(9)
    f = mono.get_state(0)
    grp.set_state(0, f)
    assert np.array_equal(grp.get_state(0), f)
    mono.primal_step(4)
    grp.step(0, 4)
    assert np.array_equal(grp.get_state(0), mono.get_state(0))


@pytest.mark.parametrize("name", ["grad2d", "mix3d", "exch3d"])
def test_nccl_single_rank_ring_equals_monolithic(lbgpu, has_gpu, name):
    """The NCCL transport (pack -> ncclSend/ncclRecv -> unpack on a comm
    stream, boundary columns first, interior overlapped) exercised on one GPU:
    one slab in ghost layout whose left and right neighbour is itself. Must
    equal the monolithic periodic-wrap run bit for bit, for both sweeps and
    for the batched tol-stop solver with its cross-rank flag reductions."""
    import torch  # noqa: F401  (loads torch's libnccl first, as in bench.py)
    txt = case_text(name)
    mono = lbgpu.Engine.from_config(txt)
    ring = lbgpu.Engine.slab_from_config(txt, None, 1, -1)
    ring.attach_nccl(lbgpu.nccl_unique_id(), 1, 0)
    s = ring.slab()
    assert s["nxl"] > s["span"] == s["gnx"]
    mono.init_state()
    ring.init_state()

    def owned(e, field):
        nx, ny, nz = mono.shape
        return e.get_state(field).reshape(e.m, nz, ny, s["nxl"])[..., : s["span"]].reshape(-1)

    assert mono.primal_step(25) == ring.primal_step(25)
    assert np.array_equal(owned(ring, 0), mono.get_state(0))
    assert mono.adjoint_step(9) == ring.adjoint_step(9)
    assert np.array_equal(owned(ring, 1), mono.get_state(1))
    g_m, d_m = mono.param_gradient()
    g_r, d_r = ring.param_gradient()
    assert np.array_equal(g_m, g_r) and d_m == d_r
    assert mono.solve_primal(1e-6, 20000) == ring.solve_primal(1e-6, 20000)
    assert np.array_equal(owned(ring, 0), mono.get_state(0))
    # fused pairs: both fields' halos after every k_pair (boundary columns
    # first, interior overlapped with the two exchanges)
    assert mono.pair_steps(6) == ring.pair_steps(6)
    assert np.array_equal(owned(ring, 0), mono.get_state(0))
    assert np.array_equal(owned(ring, 1), mono.get_state(1))


def test_p2p_group_long_run_is_race_free(lbgpu, has_gpu):
    """Many lock-step sweeps of four concurrently running slabs (separate
    streams, cross-stream event waits only between neighbours) at a size where
    the slabs' kernels overlap in time: still bitwise the monolithic run."""
    txt = case_text("mix3d", {"lattice.nx": 64, "lattice.ny": 48, "lattice.nz": 40,
                              "tags.design_x0": 16, "tags.design_x1": 47})
    mono = lbgpu.Engine.from_config(txt)
    grp = lbgpu.SlabGroup(txt, None, 4, transport="p2p")
    mono.init_state()
    grp.init_state()
    assert mono.primal_step(300) == grp.step(0, 300)
    assert np.array_equal(grp.get_state(0), mono.get_state(0))
    assert mono.adjoint_step(150) == grp.step(1, 150)
    assert np.array_equal(grp.get_state(1), mono.get_state(1))


def test_p2p_link_rejects_a_non_group(lbgpu, has_gpu):
    txt = case_text("grad2d")
    e = lbgpu.Engine.from_config(txt)
    import ctypes as C
    arr = (C.c_void_p * 2)(e.h.value, e.h.value)
    assert lbgpu.load_library().lbgpu_group_link_p2p(arr, 2) == lbgpu.E_ARG


@pytest.mark.parametrize("name", ["mix3d", "exch3d", "grad2d", "periodic2d"])
def test_p2p_group_fused_pairs_equal_monolithic(lbgpu, has_gpu, name):
    """Fused pair sweeps in the P2P group (each slab's k_pair pushes both
    fields' cut planes into its neighbours' ghosts): bitwise the monolithic
    lbgpu_pair_steps; the group timer reports a positive device time."""
    txt = case_text(name)
    mono = lbgpu.Engine.from_config(txt)
    grp = lbgpu.SlabGroup(txt, None, 3, transport="p2p")
    mono.init_state()
    grp.init_state()
    mono.primal_step(12, residual=False)
    grp.step(0, 12, residual=False)
    for n in (1, 2, 6):
        mono.pair_steps(n, residual=False)
        grp.pair_steps(n)
        assert np.array_equal(grp.get_state(0), mono.get_state(0))
        assert np.array_equal(grp.get_state(1), mono.get_state(1))
    assert grp.time(2, 5) > 0


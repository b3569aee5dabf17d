"""x-slab decomposition (partition.cpp:9-188) — host logic.

* slab tables (local layout with ghost columns) equal the global tables
  cut per slab, bit for bit, including the mt19937_64 design noise;
* decompose matches the reference's sizes (test_partition.cpp:15-38);
* the halo plan — which planes cross, which ghost they land in, the
  transposed plan for the adjoint, the NCCL posting order — reproduces
  periodic pull streaming exactly, on world_size 2 and 3 with the gloo
  backend (CPU).
"""
import ctypes as C
import os

import numpy as np
import pytest

from cases import CASES, case_text

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def slab_tables(P, txt, count, sid):
    L = P.load_library()
    fn = L.lbgpu_case_slab_tables
    fn.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                   C.c_void_p] + [C.c_void_p] * 8
    sl = (C.c_int * 6)()
    dims = (C.c_int * 8)()
    cnt = (C.c_int64 * 4)()
    rc = fn(txt.encode(), b"", count, sid, sl, dims, cnt, *([None] * 8))
    assert rc == 0, L.lbgpu_last_create_error()
    n, nd, ns = cnt[0], cnt[1], cnt[2]
    t = {"tag": np.zeros(n, np.uint8), "bc_T": np.zeros(n), "bc_axis": np.zeros(n, np.int8),
         "bc_sign": np.zeros(n, np.int8), "w": np.zeros(n), "mask": np.zeros(n, np.uint8),
         "design": np.zeros(max(nd, 1), np.int64), "support": np.zeros(max(ns, 1), np.int64)}
    keys = ("tag", "bc_T", "bc_axis", "bc_sign", "w", "mask", "design", "support")
    assert fn(txt.encode(), b"", count, sid, sl, dims, cnt, *[t[k].ctypes.data for k in keys]) == 0
    t["design"], t["support"] = t["design"][:nd], t["support"][:ns]
    return dict(zip(("gnx", "x0", "span", "nxl", "count", "id"), list(sl))), t


def test_decompose_matches_reference(lbgpu):
    """decompose (partition.cpp:9-21): contiguous, sizes differ by <= 1, the
    first nx % n slabs get the extra column (test_partition.cpp:15-38)."""
    txt = "[lattice]\nnx = 37\nny = 8\n[tags]\ngeometry = periodic\n[objective]\nkind = synthetic\n"
    for parts in (1, 2, 3, 4, 5):
        covered = 0
        for i in range(parts):
            s, _ = slab_tables(lbgpu, txt, parts, i)
            assert s["x0"] == covered
            assert s["span"] == 37 // parts + (1 if i < 37 % parts else 0)
            if parts > 1:
                assert s["nxl"] % 16 == 0 and s["nxl"] >= s["span"] + 2
            else:
                assert s["nxl"] == 37  # one slab: the periodic lattice itself
            covered += s["span"]
        assert covered == 37


@pytest.mark.parametrize("name", ["grad2d", "exch2d", "mix3d", "exch3d", "periodic2d"])
@pytest.mark.parametrize("parts", [2, 3])
def test_slab_tables_equal_global(lbgpu, name, parts):
    from test_masks import engine_tables
    txt = case_text(name)
    g = engine_tables(lbgpu, txt)
    s0, _ = slab_tables(lbgpu, txt, parts, 0)
    nx = s0["gnx"]
    n = g["tag"].size
    ny_nz = n // nx
    design_all, support_all = [], []
    for i in range(parts):
        s, t = slab_tables(lbgpu, txt, parts, i)
        nxl, span, x0 = s["nxl"], s["span"], s["x0"]
        for k in ("tag", "bc_T", "bc_axis", "bc_sign", "w", "mask"):
            loc = t[k].reshape(ny_nz, nxl)
            glob = g[k].reshape(ny_nz, nx)
            if k in ("w", "mask"):  # design data is owned-only
                assert np.array_equal(loc[:, :span], glob[:, x0:x0 + span]), (k, i)
            else:
                assert np.array_equal(loc[:, :span], glob[:, x0:x0 + span]), (k, i)
                assert np.array_equal(loc[:, span], glob[:, (x0 + span) % nx]), (k, i)
                assert np.array_equal(loc[:, nxl - 1], glob[:, (x0 - 1) % nx]), (k, i)
        to_glob = lambda a: (a % nxl) + x0 + nx * (a // nxl)
        design_all.append(to_glob(t["design"]))
        support_all.append(to_glob(t["support"]))
    assert np.array_equal(np.sort(np.concatenate(design_all)), g["design"])
    assert np.array_equal(np.sort(np.concatenate(support_all)), g["support"])


# ---------------------------------------------------------------------------
# the halo plan over gloo

VEL2 = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (1, 1, 0), (-1, 1, 0),
        (1, -1, 0), (-1, -1, 0)] * 2
VEL3 = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1),
        (1, 1, 0), (-1, 1, 0), (1, -1, 0), (-1, -1, 0), (1, 0, 1), (-1, 0, 1), (1, 0, -1),
        (-1, 0, -1), (0, 1, 1), (0, -1, 1), (0, 1, -1), (0, -1, -1)] + \
       [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]


def pull(buf, vel, D):
    """Periodic pull streaming: out_p(x) = buf_p(x + D e_p) on (M, nz, ny, nx)."""
    out = np.empty_like(buf)
    for p, (ex, ey, ez) in enumerate(vel):
        out[p] = np.roll(buf[p], shift=(-D * ez, -D * ey, -D * ex), axis=(0, 1, 2))
    return out


def _worker(rank, world, port, D, dims, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, ny, nz = dims
    vel = VEL3 if nz > 1 else VEL2
    M = len(vel)
    rng = np.random.default_rng(11)
    glob = rng.standard_normal((M, nz, ny, nx))
    # this rank's slab in the engine's local layout
    base, rem = nx // world, nx % world
    x0 = rank * base + min(rank, rem)
    span = base + (1 if rank < rem else 0)
    nxl = (span + 2 + 15) // 16 * 16
    loc = np.zeros((M, nz, ny, nxl))
    loc[..., :span] = glob[..., x0:x0 + span]
    # halo plan (kernels.cuh k_halo_pack / k_halo_unpack)
    to_right = [p for p, e in enumerate(vel) if D * e[0] == -1]
    to_left = [p for p, e in enumerate(vel) if D * e[0] == +1]
    assert len(to_right) == 6 and len(to_left) == 6
    send_r = torch.from_numpy(np.ascontiguousarray(loc[to_right, :, :, span - 1]))
    send_l = torch.from_numpy(np.ascontiguousarray(loc[to_left, :, :, 0]))
    recv_l, recv_r = torch.empty_like(send_r), torch.empty_like(send_l)
    left, right = (rank - 1) % world, (rank + 1) % world
    # engine.cu exchange(): send right, recv left, send left, recv right
    reqs = [dist.isend(send_r, right), dist.irecv(recv_l, left),
            dist.isend(send_l, left), dist.irecv(recv_r, right)]
    for r in reqs:
        r.wait()
    loc[to_right, :, :, nxl - 1] = recv_l.numpy()
    loc[to_left, :, :, span] = recv_r.numpy()
    # the next sweep's pull over owned columns, with the kernels' local wrap
    got = pull(loc, vel, D)[..., :span]
    want = pull(glob, vel, D)[..., x0:x0 + span]
    q.put((rank, bool(np.array_equal(got, want))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("D", [-1, +1])
@pytest.mark.parametrize("dims", [(13, 6, 1), (11, 5, 4)])
def test_halo_plan_over_gloo(world, D, dims):
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, D, dims, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res

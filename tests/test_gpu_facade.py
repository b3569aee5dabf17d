"""lbopt.h on the B200 engine: the reference's own C API
(oracle/_ref/liblbopt_ref.so, capi.cpp) and ours (liblbgpu.so,
include/lbopt_gpu.h) driven through identical call sequences. With the
bit-exact build (LBOPT_GPU_EXACT=1) statuses, iteration counts and every
output file are byte-identical; the product build is checked within the
parity tolerances."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_1501_04741_b200.presets import preset_text

pytestmark = pytest.mark.gpu


def lib(path):
    L = C.CDLL(path)
    vp = C.c_void_p
    L.lbopt_open_text.argtypes = [C.c_char_p, C.POINTER(vp)]
    L.lbopt_close.argtypes = [vp]
    L.lbopt_last_open_error.restype = C.c_char_p
    L.lbopt_error_message.restype = C.c_char_p
    L.lbopt_error_message.argtypes = [vp]
    L.lbopt_set.argtypes = [vp, C.c_char_p, C.c_char_p]
    L.lbopt_save_config.argtypes = [vp, C.c_char_p]
    for f in ("lbopt_simulate", "lbopt_solve_adjoint", "lbopt_optimize"):
        getattr(L, f).argtypes = [vp]
    L.lbopt_grad_check.argtypes = [vp, C.POINTER(C.c_double)]
    L.lbopt_threshold_sweep.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.lbopt_partition_check.argtypes = [vp, C.c_long, C.POINTER(C.c_double)]
    L.lbopt_cost_ratio.argtypes = [vp, C.c_long, C.POINTER(C.c_double)]
    L.lbopt_generate_fins.argtypes = [vp, C.c_int, C.c_int]
    L.lbopt_load_state_csv.argtypes = [vp, C.c_char_p]
    L.lbopt_load_design_csv.argtypes = [vp, C.c_char_p]
    L.lbopt_write_fields.argtypes = [vp, C.c_char_p, C.c_char_p]
    L.lbopt_objective_value.argtypes = [vp, C.POINTER(C.c_double)]
    L.lbopt_iterations.argtypes = [vp, C.POINTER(C.c_long)]
    L.lbopt_converged.argtypes = [vp, C.POINTER(C.c_int)]
    L.lbopt_residual.argtypes = [vp, C.POINTER(C.c_double)]
    return L


class Case:
    def __init__(self, L, text, out_dir, sets=()):
        self.L = L
        self.h = C.c_void_p()
        rc = L.lbopt_open_text(text.encode(), C.byref(self.h))
        assert rc == 0, L.lbopt_last_open_error()
        self.set("output.dir", out_dir)
        for k, v in sets:
            self.set(k, v)

    def set(self, k, v):
        assert self.L.lbopt_set(self.h, k.encode(), str(v).encode()) == 0

    def call(self, name, *args):
        return getattr(self.L, name)(self.h, *args)

    def status(self):
        o, r = C.c_double(), C.c_double()
        it, cv = C.c_long(), C.c_int()
        self.L.lbopt_objective_value(self.h, C.byref(o))
        self.L.lbopt_residual(self.h, C.byref(r))
        self.L.lbopt_iterations(self.h, C.byref(it))
        self.L.lbopt_converged(self.h, C.byref(cv))
        return (o.value, r.value, it.value, cv.value)

    def msg(self):
        return self.L.lbopt_error_message(self.h).decode()

    def close(self):
        self.L.lbopt_close(self.h)


@pytest.fixture(scope="module")
def libs(oracle_mod):
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    import paper_1501_04741_b200 as P
    return lib(oracle_mod.REF_SO), lib(P.LIB_PATH)


@pytest.fixture()
def exact_env(monkeypatch):
    monkeypatch.setenv("LBOPT_GPU_EXACT", "1")


def same_files(d1, d2, names):
    for n in names:
        a = open(os.path.join(d1, n)).read()
        b = open(os.path.join(d2, n)).read()
        assert a == b, n


def test_simulate_adjoint_byte_identical(libs, tmp_path, exact_env, has_gpu):
    R, G = libs
    text = preset_text("gradcheck2d")
    sets = [("optimizer.record_interval", 500), ("output.write_vtk", "true")]
    r = Case(R, text, str(tmp_path / "ref"), sets)
    g = Case(G, text, str(tmp_path / "gpu"), sets)
    assert r.call("lbopt_simulate") == 0 and g.call("lbopt_simulate") == 0
    assert r.status() == g.status()
    assert g.status()[2] == 16578
    same_files(tmp_path / "ref", tmp_path / "gpu", ["fields.csv", "state.csv", "record.csv",
                                                      "fields.vtk"])
    assert r.call("lbopt_solve_adjoint") == 0 and g.call("lbopt_solve_adjoint") == 0
    assert r.status() == g.status()
    same_files(tmp_path / "ref", tmp_path / "gpu", ["gradient.csv", "adjoint_record.csv"])


def test_one_shot_and_mma_byte_identical(libs, tmp_path, exact_env, has_gpu):
    R, G = libs
    text = preset_text("mixer2d", {"lattice.nx": 40, "lattice.ny": 10, "tags.design_x0": 10,
                                   "tags.design_x1": 29, "optimizer.iterations": 30,
                                   "optimizer.zeta_stages": "0:0,5:0.01",
                                   "optimizer.record_interval": 4,
                                   "objective.penalty_w0": 0.001, "objective.penalty_cap": 0.1,
                                   "objective.penalty_interval": 10, "optimizer.primal_tol": 1e-7,
                                   "output.write_vtk": "false"})
    files = ["design.csv", "fields.csv", "state.csv", "convergence.csv", "optimize_record.csv",
             "design_000006.csv", "fields_000030.csv"]
    for method in ("oneshot", "mma"):
        sets = [("optimizer.method", method), ("optimizer.outer_iterations", 3),
                ("optimizer.primal_tol", 1e-6), ("optimizer.adjoint_tol", 1e-6)]
        r = Case(R, text, str(tmp_path / f"ref_{method}"), sets)
        g = Case(G, text, str(tmp_path / f"gpu_{method}"), sets)
        assert r.call("lbopt_optimize") == 0, r.msg()
        assert g.call("lbopt_optimize") == 0, g.msg()
        assert r.status() == g.status(), method
        names = files if method == "oneshot" else files[:5] + ["design_000003.csv"]
        same_files(tmp_path / f"ref_{method}", tmp_path / f"gpu_{method}", names)


def test_grad_check_threshold_partition(libs, tmp_path, exact_env, has_gpu):
    R, G = libs
    text = preset_text("gradcheck2d", {"optimizer.primal_tol": 1e-10,
                                       "optimizer.adjoint_tol": 1e-10,
                                       "optimizer.threshold_points": 4,
                                       "optimizer.workers": 2})
    r = Case(R, text, str(tmp_path / "ref"))
    g = Case(G, text, str(tmp_path / "gpu"))
    er, eg = C.c_double(), C.c_double()
    assert r.call("lbopt_grad_check", C.byref(er)) == 0
    assert g.call("lbopt_grad_check", C.byref(eg)) == 0
    assert er.value == eg.value and eg.value < 1e-5
    same_files(tmp_path / "ref", tmp_path / "gpu", ["gradcheck.csv"])
    be_r, bo_r, be_g, bo_g = C.c_double(), C.c_double(), C.c_double(), C.c_double()
    assert r.call("lbopt_threshold_sweep", C.byref(be_r), C.byref(bo_r)) == 0
    assert g.call("lbopt_threshold_sweep", C.byref(be_g), C.byref(bo_g)) == 0
    assert (be_r.value, bo_r.value) == (be_g.value, bo_g.value)
    same_files(tmp_path / "ref", tmp_path / "gpu", ["threshold.csv"])
    d = C.c_double(-1.0)
    assert g.call("lbopt_partition_check", 20, C.byref(d)) == 0 and d.value == 0.0
    ratio = C.c_double()
    assert g.call("lbopt_cost_ratio", 20, C.byref(ratio)) == 0 and ratio.value > 0


def test_state_and_design_io_and_errors(libs, tmp_path, exact_env, has_gpu):
    R, G = libs
    text = preset_text("gradcheck2d", {"optimizer.primal_tol": 1e-6})
    g = Case(G, text, str(tmp_path / "gpu"))
    r = Case(R, text, str(tmp_path / "ref"))
    # adjoint before any primal: StateError, same message
    assert g.call("lbopt_solve_adjoint") == 5 == r.call("lbopt_solve_adjoint")
    assert g.msg() == r.msg()
    # unknown key: immediate config error
    assert G.lbopt_set(g.h, b"model.bogus", b"1") == 2 == R.lbopt_set(r.h, b"model.bogus", b"1")
    assert g.msg() == r.msg()
    # simulate on one engine, hand its state.csv to the other through load_state_csv
    assert r.call("lbopt_simulate") == 0
    assert g.call("lbopt_load_state_csv", str(tmp_path / "ref" / "state.csv").encode()) == 0
    assert r.call("lbopt_solve_adjoint") == 0 and g.call("lbopt_solve_adjoint") == 0
    same_files(tmp_path / "ref", tmp_path / "gpu", ["gradient.csv"])
    # fins + design round trip
    assert r.call("lbopt_generate_fins", 2, 1) == 0 and g.call("lbopt_generate_fins", 2, 1) == 0
    assert r.call("lbopt_write_fields", str(tmp_path / "fr.csv").encode(), None) == 0
    assert g.call("lbopt_write_fields", str(tmp_path / "fg.csv").encode(), None) == 0
    assert open(tmp_path / "fr.csv").read() == open(tmp_path / "fg.csv").read()
    # save_config: canonical serialisation is identical
    r.set("output.dir", str(tmp_path / "same"))
    g.set("output.dir", str(tmp_path / "same"))
    R.lbopt_save_config(r.h, str(tmp_path / "r.cfg").encode())
    G.lbopt_save_config(g.h, str(tmp_path / "g.cfg").encode())
    assert open(tmp_path / "r.cfg").read() == open(tmp_path / "g.cfg").read()


def test_product_build_within_tolerance(libs, tmp_path, has_gpu, monkeypatch):
    monkeypatch.delenv("LBOPT_GPU_EXACT", raising=False)
    R, G = libs
    text = preset_text("gradcheck2d")
    r = Case(R, text, str(tmp_path / "ref"))
    g = Case(G, text, str(tmp_path / "gpu"))
    assert r.call("lbopt_simulate") == 0 and g.call("lbopt_simulate") == 0
    so, sg = r.status(), g.status()
    assert abs(so[2] - sg[2]) <= 1 and so[3] == sg[3] == 1
    assert abs(so[0] - sg[0]) <= 1e-12 * abs(so[0])
    assert r.call("lbopt_solve_adjoint") == 0 and g.call("lbopt_solve_adjoint") == 0
    gr = np.loadtxt(tmp_path / "ref" / "gradient.csv", delimiter=",", skiprows=1, usecols=3)
    gg = np.loadtxt(tmp_path / "gpu" / "gradient.csv", delimiter=",", skiprows=1, usecols=3)
    assert np.max(np.abs(gr - gg)) <= 1e-9 * np.max(np.abs(gr))

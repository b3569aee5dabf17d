"""TEST INFRASTRUCTURE ONLY — Python handles on the two CPU checkers.

* ``COracle``  — the plain-C restatement (oracle/lbm_oracle.c, built as
  oracle/liblbm_oracle.so).
* ``RefOracle`` — the reference itself, compiled from its own sources
  (oracle/Makefile -> oracle/_ref/liblbopt_ref.so) behind oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
``--impl reference``) may import this module, and only as the checker. The
product (paper_1501_04741_b200/) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "liblbopt_ref.so")
ORACLE_SO = os.path.join(HERE, "liblbm_oracle.so")
REF_SRC = "/root/reference/proj"


def build(ref: bool = True) -> None:
    """Build the C restatement, and the reference when its sources exist."""
    targets = ["oracle"]
    if ref and os.path.isdir(os.path.join(REF_SRC, "src")):
        targets.append("ref")
        if os.path.exists(os.path.join(os.path.dirname(HERE), "paper_1501_04741_b200", "liblbgpu.so")):
            targets.append("drop_in")  # the reference-side binding
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


# ---------------------------------------------------------------------------
# configuration (defaults and keys of CaseConfig, config.hpp:16-83)

DEFAULTS = {
    "lattice.nx": "0", "lattice.ny": "0", "lattice.nz": "1",
    "model.nu": "0.02", "model.beta_fluid": "0.003", "model.beta_solid": "0.003",
    "model.inlet_dp": "0", "model.u_clamp": "0.05", "model.collision": "fmrt",
    "model.precision": "64", "model.omega_nonhydro": "1", "model.switch_theta": "3",
    "model.switch_form": "solid_power",
    "tags.geometry": "channel", "tags.design_x0": "-1", "tags.design_x1": "-1",
    "tags.heater_x0": "-1", "tags.heater_x1": "-1", "tags.inlet_profile": "uniform",
    "tags.inlet_T": "0",
    "objective.kind": "mixing", "objective.plane_offset": "1",
    "optimizer.initial_w": "1", "optimizer.init_noise": "0", "optimizer.seed": "0",
}


def parse_cfg(text: str, overrides: dict | None = None) -> dict:
    out = dict(DEFAULTS)
    sec = ""
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if line.startswith("["):
            sec = line[1:-1].strip()
            continue
        k, v = line.split("=", 1)
        key = f"{sec}.{k.strip()}"
        if key == "output.dir":
            continue
        out[key] = v.strip()
    for k, v in (overrides or {}).items():
        out[k] = str(v)
    return out


def overrides_text(overrides: dict | None) -> bytes | None:
    if not overrides:
        return None
    return "\n".join(f"{k}={v}" for k, v in overrides.items()).encode()


# ---------------------------------------------------------------------------
# C restatement


class _Params(C.Structure):
    _fields_ = [
        ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
        ("bgk", C.c_int), ("fluid_power", C.c_int), ("periodic", C.c_int),
        ("split_inlet", C.c_int), ("obj_kind", C.c_int),
        ("nu", C.c_double), ("beta_fluid", C.c_double), ("beta_solid", C.c_double),
        ("inlet_dp", C.c_double), ("u_clamp", C.c_double), ("omega_nonhydro", C.c_double),
        ("theta", C.c_double), ("inlet_T", C.c_double),
        ("design_x0", C.c_int), ("design_x1", C.c_int), ("heater_x0", C.c_int),
        ("heater_x1", C.c_int), ("plane_offset", C.c_int),
        ("initial_w", C.c_double), ("init_noise", C.c_double), ("seed", C.c_uint64),
    ]


class _System(C.Structure):
    _fields_ = [
        ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("n", C.c_long),
        ("mf", C.c_int), ("mt", C.c_int), ("m", C.c_int),
        ("vel", (C.c_int * 3) * 28), ("opp", C.c_int * 28),
        ("wf", C.c_double * 19), ("wt", C.c_double * 9),
        ("A", C.c_double * 361), ("At", C.c_double * 361), ("relax", C.c_double * 19),
        ("nu", C.c_double), ("beta_fluid", C.c_double), ("beta_solid", C.c_double),
        ("inlet_dp", C.c_double), ("u_clamp", C.c_double), ("omega_nonhydro", C.c_double),
        ("theta", C.c_double), ("bgk", C.c_int), ("fluid_power", C.c_int),
        ("tag", C.POINTER(C.c_uint8)), ("bc_T", C.POINTER(C.c_double)),
        ("bc_axis", C.POINTER(C.c_int8)), ("bc_sign", C.POINTER(C.c_int8)),
        ("w", C.POINTER(C.c_double)), ("mask", C.POINTER(C.c_uint8)),
        ("design", C.POINTER(C.c_long)), ("n_design", C.c_long),
        ("obj_kind", C.c_int), ("flux_axis", C.c_int), ("flux_sign", C.c_int),
        ("on_support", C.POINTER(C.c_uint8)), ("support", C.POINTER(C.c_long)),
        ("n_support", C.c_long),
    ]


_DP = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_olib = None


def _load_oracle():
    global _olib
    if _olib is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        L = C.CDLL(ORACLE_SO)
        L.lbo_build.argtypes = [C.POINTER(_Params), C.POINTER(_System)]
        L.lbo_free.argtypes = [C.POINTER(_System)]
        L.lbo_init_state.argtypes = [C.POINTER(_System), _DP]
        L.lbo_primal_step.argtypes = [C.POINTER(_System), _DP, _DP, C.POINTER(C.c_long)]
        L.lbo_residual.argtypes = [_DP, _DP, C.c_long]
        L.lbo_residual.restype = C.c_double
        L.lbo_adjoint_step.argtypes = [C.POINTER(_System), _DP, _DP, _DP, C.c_int]
        L.lbo_param_gradient.argtypes = [C.POINTER(_System), _DP, _DP, C.c_int, _DP,
                                         C.POINTER(C.c_double)]
        L.lbo_objective.argtypes = [C.POINTER(_System), _DP]
        L.lbo_objective.restype = C.c_double
        L.lbo_penalty.argtypes = [C.POINTER(_System)]
        L.lbo_penalty.restype = C.c_double
        L.lbo_collide_node.argtypes = [C.POINTER(_System), C.c_int, C.c_int, C.c_int, C.c_double,
                                       _DP, C.c_double, _DP]
        L.lbo_one_shot_iter.argtypes = [C.POINTER(_System), _DP, _DP, _DP, _DP, C.c_double,
                                        C.c_double, C.POINTER(C.c_double)]
        L.lbo_pairwise_sum.argtypes = [_DP, C.c_long]
        L.lbo_pairwise_sum.restype = C.c_double
        _olib = L
    return _olib


class COracle:
    """The C restatement with its own state arrays (reference layout, FP64)."""

    def __init__(self, cfg_text: str, overrides: dict | None = None):
        self.L = _load_oracle()
        c = parse_cfg(cfg_text, overrides)
        p = _Params()
        p.nx, p.ny, p.nz = int(c["lattice.nx"]), int(c["lattice.ny"]), int(c["lattice.nz"])
        p.bgk = c["model.collision"] == "bgk"
        p.fluid_power = c["model.switch_form"] == "fluid_power"
        p.periodic = c["tags.geometry"] == "periodic"
        p.split_inlet = c["tags.inlet_profile"] == "split"
        p.obj_kind = {"mixing": 0, "heatflux": 1, "synthetic": 2}[c["objective.kind"]]
        for k in ("nu", "beta_fluid", "beta_solid", "inlet_dp", "u_clamp", "omega_nonhydro"):
            setattr(p, k, float(c["model." + k]))
        p.theta = float(c["model.switch_theta"])
        p.inlet_T = float(c["tags.inlet_T"])
        for k in ("design_x0", "design_x1", "heater_x0", "heater_x1"):
            setattr(p, k, int(c["tags." + k]))
        p.plane_offset = int(c["objective.plane_offset"])
        p.initial_w = float(c["optimizer.initial_w"])
        p.init_noise = float(c["optimizer.init_noise"])
        p.seed = int(c["optimizer.seed"])
        self.s = _System()
        rc = self.L.lbo_build(C.byref(p), C.byref(self.s))
        if rc:
            raise ValueError(f"oracle build failed ({rc})")
        s = self.s
        self.shape = (s.nx, s.ny, s.nz)
        self.n, self.m, self.mf, self.mt = s.n, s.m, s.mf, s.mt
        self.f = np.zeros(self.m * self.n)
        self.v = np.zeros(self.m * self.n)
        self.f2 = np.zeros_like(self.f)
        self.v2 = np.zeros_like(self.v)
        self.last_primal_residual = 0.0
        self.last_adjoint_residual = 0.0

    def __del__(self):
        try:
            self.L.lbo_free(C.byref(self.s))
        except Exception:
            pass

    # --- tables -----------------------------------------------------------
    def tables(self) -> dict:
        s, n = self.s, self.n
        arr = lambda p, k, dt: np.ctypeslib.as_array(p, shape=(k,)).astype(dt).copy()
        return {
            "tag": arr(s.tag, n, np.uint8), "bc_T": arr(s.bc_T, n, np.float64),
            "bc_axis": arr(s.bc_axis, n, np.int8), "bc_sign": arr(s.bc_sign, n, np.int8),
            "w": arr(s.w, n, np.float64), "mask": arr(s.mask, n, np.uint8),
            "design": arr(s.design, s.n_design, np.int64) if s.n_design else np.zeros(0, np.int64),
            "support": arr(s.support, s.n_support, np.int64),
            "A": np.array(s.A[: s.mf * s.mf]).reshape(s.mf, s.mf),
        }

    def set_design(self, w_full: np.ndarray) -> None:
        w = np.ctypeslib.as_array(self.s.w, shape=(self.n,))
        w[:] = w_full

    def design(self) -> np.ndarray:
        return np.ctypeslib.as_array(self.s.w, shape=(self.n,)).copy()

    # --- operators ----------------------------------------------------------
    def init_state(self) -> None:
        self.L.lbo_init_state(C.byref(self.s), self.f)
        self.v[:] = 0.0

    def primal_steps(self, k: int = 1) -> float:
        bad = C.c_long(-1)
        for _ in range(k):
            if self.L.lbo_primal_step(C.byref(self.s), self.f, self.f2, C.byref(bad)):
                raise FloatingPointError(f"non-positive density at flat index {bad.value}")
            self.f, self.f2 = self.f2, self.f
        self.last_primal_residual = self.L.lbo_residual(self.f, self.f2, self.f.size)
        return self.last_primal_residual

    def adjoint_steps(self, k: int = 1, kernel: int = 0) -> float:
        for _ in range(k):
            if self.L.lbo_adjoint_step(C.byref(self.s), self.f, self.v, self.v2, kernel):
                raise FloatingPointError("non-positive density")
            self.v, self.v2 = self.v2, self.v
        self.last_adjoint_residual = self.L.lbo_residual(self.v, self.v2, self.v.size)
        return self.last_adjoint_residual

    def gradient(self, kernel: int = 0):
        g = np.zeros(max(self.s.n_design, 1))
        gdp = C.c_double()
        if self.L.lbo_param_gradient(C.byref(self.s), self.v, self.f, kernel, g, C.byref(gdp)):
            raise FloatingPointError("non-positive density")
        return g[: self.s.n_design], gdp.value

    def objective(self) -> float:
        return self.L.lbo_objective(C.byref(self.s), self.f)

    def penalty(self) -> float:
        return self.L.lbo_penalty(C.byref(self.s))

    def collide_node(self, tag, axis, sign, bcT, fin, w):
        out = np.zeros(self.m)
        self.L.lbo_collide_node(C.byref(self.s), tag, axis, sign, bcT,
                                np.ascontiguousarray(fin, np.float64), w, out)
        return out

    def one_shot_iter(self, zeta: float, lam: float) -> float:
        gm = C.c_double()
        rc = self.L.lbo_one_shot_iter(C.byref(self.s), self.f, self.f2, self.v, self.v2,
                                      zeta, lam, C.byref(gm))
        if rc:
            raise FloatingPointError("non-positive density")
        self.f, self.f2 = self.f2, self.f
        self.v, self.v2 = self.v2, self.v
        return gm.value


def pairwise_sum(x: np.ndarray) -> float:
    L = _load_oracle()
    x = np.ascontiguousarray(x, np.float64)
    return L.lbo_pairwise_sum(x, x.size)


# ---------------------------------------------------------------------------
# the reference itself

_rlib = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _load_ref():
    global _rlib
    if _rlib is None:
        if not os.path.exists(REF_SO):
            build(ref=True)
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_open.restype = C.c_void_p
        L.ref_open.argtypes = [C.c_char_p, C.c_char_p]
        L.ref_close.argtypes = [C.c_void_p]
        vp = C.c_void_p
        L.ref_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_long)]
        L.ref_set_design.argtypes = [vp, _DP]
        L.ref_init_state.argtypes = [vp]
        L.ref_get_state.argtypes = [vp, C.c_int, _DP]
        L.ref_set_state.argtypes = [vp, C.c_int, _DP]
        L.ref_primal_steps.argtypes = [vp, C.c_long, C.POINTER(C.c_double)]
        L.ref_adjoint_steps.argtypes = [vp, C.c_long, C.c_int, C.POINTER(C.c_double)]
        L.ref_solve_primal.argtypes = [vp, C.c_double, C.c_long, C.c_long, C.POINTER(C.c_long),
                                       C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.ref_solve_adjoint.argtypes = [vp, C.c_double, C.c_long, C.c_long, C.c_int,
                                        C.POINTER(C.c_long), C.POINTER(C.c_double),
                                        C.POINTER(C.c_int)]
        L.ref_gradient.argtypes = [vp, C.c_int, _DP, C.POINTER(C.c_double)]
        L.ref_objective.argtypes = [vp, C.POINTER(C.c_double)]
        L.ref_penalty.argtypes = [vp, C.POINTER(C.c_double)]
        L.ref_one_shot.argtypes = [vp, C.c_long, C.c_long, _DP, C.c_long, C.POINTER(C.c_long)]
        L.ref_collide_node.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_double, _DP, C.c_double,
                                       _DP]
        L.ref_fd_gradient.argtypes = [vp, C.c_long, C.c_double, C.c_double, C.c_long, C.c_long,
                                      C.POINTER(C.c_double)]
        L.ref_partition_check.argtypes = [vp, C.c_int, C.c_long, C.POINTER(C.c_double),
                                          C.POINTER(C.c_double)]
        L.ref_time.argtypes = [vp, C.c_int, C.c_int, C.c_long, C.POINTER(C.c_double)]
        L.ref_partitioned.argtypes = [vp, C.c_int, C.c_long, C.c_long, C.c_long, _DP]
        L.ref_objective_enabled.argtypes = [vp, C.c_int]
        L.ref_partitioned_solve.argtypes = [vp, C.c_int, C.c_double, C.c_long, C.c_long,
                                            C.POINTER(C.c_long), C.POINTER(C.c_double),
                                            C.POINTER(C.c_int)]
        L.ref_tangent.argtypes = [vp, vp, C.c_double, C.c_double, C.c_long,
                                  C.POINTER(C.c_double), C.POINTER(C.c_long),
                                  C.POINTER(C.c_double), C.POINTER(C.c_int)]
        _rlib = L
    return _rlib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class RefOracle:
    """The reference's own operators (compiled from /root/reference sources)."""

    def __init__(self, cfg_text: str, overrides: dict | None = None):
        self.L = _load_ref()
        h = self.L.ref_open(cfg_text.encode(), overrides_text(overrides))
        if not h:
            raise RefError(2, self.L.ref_last_error().decode())
        self.h = C.c_void_p(h)
        dims = (C.c_int * 7)()
        cnt = (C.c_long * 3)()
        self._ok(self.L.ref_info(self.h, dims, cnt))
        self.shape = (dims[0], dims[1], dims[2])
        self.m, self.mf, self.mt, self.precision = dims[3], dims[4], dims[5], dims[6]
        self.n, self.n_design, self.n_support = cnt[0], cnt[1], cnt[2]

    def _ok(self, rc):
        if rc:
            raise RefError(rc, self.L.ref_last_error().decode())

    def close(self):
        if getattr(self, "h", None):
            self.L.ref_close(self.h)
            self.h = None

    __del__ = close

    def tables(self) -> dict:
        n, m, mf = self.n, self.m, self.mf
        t = {
            "tag": np.zeros(n, np.uint8), "bc_T": np.zeros(n), "bc_axis": np.zeros(n, np.int8),
            "bc_sign": np.zeros(n, np.int8), "w": np.zeros(n), "mask": np.zeros(n, np.uint8),
            "design": np.zeros(max(self.n_design, 1), np.int64),
            "support": np.zeros(max(self.n_support, 1), np.int64),
            "A": np.zeros((mf, mf)), "relax": np.zeros(mf),
            "vel": np.zeros((m, 3), np.int32), "opp": np.zeros(m, np.int32),
        }
        P = lambda a: a.ctypes.data_as(C.c_void_p)
        fn = self.L.ref_tables
        fn.argtypes = [C.c_void_p] + [C.c_void_p] * 12
        self._ok(fn(self.h, *[P(t[k]) for k in ("tag", "bc_T", "bc_axis", "bc_sign", "w", "mask",
                                                "design", "support", "A", "relax", "vel", "opp")]))
        t["design"] = t["design"][: self.n_design]
        t["support"] = t["support"][: self.n_support]
        return t

    def set_design(self, w_full):
        self._ok(self.L.ref_set_design(self.h, np.ascontiguousarray(w_full, np.float64)))

    def init_state(self):
        self._ok(self.L.ref_init_state(self.h))

    def get_state(self, field: int = 0) -> np.ndarray:
        out = np.zeros(self.m * self.n)
        self._ok(self.L.ref_get_state(self.h, field, out))
        return out

    def set_state(self, field: int, data: np.ndarray) -> None:
        self._ok(self.L.ref_set_state(self.h, field, np.ascontiguousarray(data, np.float64)))

    def primal_steps(self, k: int = 1) -> float:
        r = C.c_double()
        self._ok(self.L.ref_primal_steps(self.h, k, C.byref(r)))
        return r.value

    def adjoint_steps(self, k: int = 1, kernel: int = 0) -> float:
        r = C.c_double()
        self._ok(self.L.ref_adjoint_steps(self.h, k, kernel, C.byref(r)))
        return r.value

    def solve_primal(self, tol, max_iter=200000, fixed=-1):
        it, res, conv = C.c_long(), C.c_double(), C.c_int()
        self._ok(self.L.ref_solve_primal(self.h, tol, max_iter, fixed, C.byref(it), C.byref(res),
                                         C.byref(conv)))
        return it.value, res.value, bool(conv.value)

    def solve_adjoint(self, tol, max_iter=200000, fixed=-1, kernel=0):
        it, res, conv = C.c_long(), C.c_double(), C.c_int()
        self._ok(self.L.ref_solve_adjoint(self.h, tol, max_iter, fixed, kernel, C.byref(it),
                                          C.byref(res), C.byref(conv)))
        return it.value, res.value, bool(conv.value)

    def gradient(self, kernel: int = 0):
        g = np.zeros(max(self.n_design, 1))
        gdp = C.c_double()
        self._ok(self.L.ref_gradient(self.h, kernel, g, C.byref(gdp)))
        return g[: self.n_design], gdp.value

    def objective(self) -> float:
        v = C.c_double()
        self._ok(self.L.ref_objective(self.h, C.byref(v)))
        return v.value

    def penalty(self) -> float:
        v = C.c_double()
        self._ok(self.L.ref_penalty(self.h, C.byref(v)))
        return v.value

    def one_shot(self, iterations: int, record_interval: int):
        cap = iterations // record_interval + 2
        rows = np.zeros(7 * cap)
        nr = C.c_long()
        self._ok(self.L.ref_one_shot(self.h, iterations, record_interval, rows, cap, C.byref(nr)))
        return rows.reshape(cap, 7)[: nr.value]

    def collide_node(self, tag, axis, sign, bcT, fin, w):
        out = np.zeros(self.m)
        self._ok(self.L.ref_collide_node(self.h, tag, axis, sign, bcT,
                                         np.ascontiguousarray(fin, np.float64), w, out))
        return out

    def fd_gradient(self, ordinal, step, tol, max_iter, fixed):
        v = C.c_double()
        self._ok(self.L.ref_fd_gradient(self.h, ordinal, step, tol, max_iter, fixed, C.byref(v)))
        return v.value

    def tangent(self, dw, d_inlet_dp, tol, max_iter):
        """tangent_solve (adjoint.cpp:422-489) from the current primal state:
        (dF, iterations, residual, converged)."""
        dw = np.ascontiguousarray(dw, np.float64)
        dF, r = C.c_double(), C.c_double()
        it, cv = C.c_long(), C.c_int()
        self._ok(self.L.ref_tangent(self.h, dw.ctypes.data, d_inlet_dp, tol, max_iter,
                                    C.byref(dF), C.byref(it), C.byref(r), C.byref(cv)))
        return dF.value, it.value, r.value, bool(cv.value)

    def partition_check(self, parts, steps):
        a, b = C.c_double(), C.c_double()
        self._ok(self.L.ref_partition_check(self.h, parts, steps, C.byref(a), C.byref(b)))
        return a.value, b.value

    def partitioned(self, threads: int, n_primal: int = 0, n_adjoint: int = 0,
                    n_pairs: int = 0):
        """The reference's PartitionedRun on `threads` host threads from the
        handle's f with v = 0: n_primal primal steps, n_adjoint adjoint steps,
        n_pairs (primal, adjoint) pairs; f and v gathered back. Returns the
        last primal and adjoint residuals."""
        r = np.zeros(2)
        self._ok(self.L.ref_partitioned(self.h, threads, n_primal, n_adjoint, n_pairs, r))
        return float(r[0]), float(r[1])

    def partitioned_solve(self, threads: int, tol: float, max_iter: int = 200000,
                          fixed: int = -1):
        """partitioned_fixed_point on `threads` host threads from the handle's
        f: (iterations, residual, converged); f gathered back."""
        it, res, conv = C.c_long(), C.c_double(), C.c_int()
        self._ok(self.L.ref_partitioned_solve(self.h, threads, tol, max_iter, fixed, C.byref(it),
                                              C.byref(res), C.byref(conv)))
        return it.value, res.value, bool(conv.value)

    def objective_enabled(self, on: bool) -> None:
        """obj_empty of the A14 composition recipe: adjoint steps without
        the objective source while off."""
        self._ok(self.L.ref_objective_enabled(self.h, 1 if on else 0))

    def time_steps(self, which: int, threads: int, steps: int) -> float:
        s = C.c_double()
        self._ok(self.L.ref_time(self.h, which, threads, steps, C.byref(s)))
        return s.value


def preset(name: str) -> str:
    """INI text of a reference preset, from the product's preset registry
    (paper_1501_04741_b200/presets.py restates proj/presets/*.cfg)."""
    import sys
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_1501_04741_b200.presets import preset_text
    return preset_text(name)

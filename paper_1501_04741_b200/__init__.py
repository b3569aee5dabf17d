"""B200-native LBM primal / discrete-adjoint hot path (arxiv/paper_1501_04741).

Python host mirror of the reference's inner operator seam, over the C ABI in
include/lbgpu.h (liblbgpu.so, built in-tree by ``build.py``). Method names
follow the reference operators they replace:

=====================  ===========================================
``Engine`` method      reference operator (proj/...)
=====================  ===========================================
``init_state``         initialize_state (src/collision.cpp:296-306)
``primal_step``        primal_step + step_residual (:308-375)
``solve_primal``       solve_fixed_point (:377-416)
``adjoint_step``       adjoint_step (src/adjoint.cpp:206-254)
``solve_adjoint``      solve_adjoint (:256-297)
``param_gradient``     param_gradient (:377-420)
``objective``          evaluate_raw (src/objective.cpp:64-72)
``penalty``            penalty (src/topology.cpp:40-50)
``one_shot``           one_shot_run (src/optimizer.cpp:25-72)
=====================  ===========================================

Errors raise ``LbgpuError`` carrying the reference's status code
(lbopt.h:18-25). There is no CPU fallback: without liblbgpu.so or without a
GPU the constructor raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LBGPU_LIB") or os.path.join(HERE, "liblbgpu.so")

OK, E_ARG, E_CONFIG, E_NUMERIC, E_IO, E_STATE = range(6)


class LbgpuError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


class RunRow(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("iteration", "residual", "objective", "penalty",
                                          "penalty_weight", "composite", "grad_norm")]


class SystemDesc(C.Structure):
    _fields_ = [
        ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
        ("precision", C.c_int), ("exact", C.c_int), ("device", C.c_int),
        ("collision", C.c_int),
        ("nu", C.c_double), ("beta_fluid", C.c_double), ("beta_solid", C.c_double),
        ("inlet_dp", C.c_double), ("u_clamp", C.c_double), ("omega_nonhydro", C.c_double),
        ("switch_theta", C.c_double), ("switch_form", C.c_int),
        ("A", C.c_void_p), ("relax", C.c_void_p), ("vel", C.c_void_p), ("opp", C.c_void_p),
        ("tag", C.c_void_p), ("bc_T", C.c_void_p), ("bc_axis", C.c_void_p),
        ("bc_sign", C.c_void_p), ("w", C.c_void_p), ("design_mask", C.c_void_p),
        ("obj_kind", C.c_int), ("flux_axis", C.c_int), ("flux_sign", C.c_int),
        ("support", C.c_void_p), ("n_support", C.c_int64),
        ("slab_count", C.c_int), ("slab_id", C.c_int),
        ("streaming", C.c_int),
    ]


_lib = None


def build(verbose: bool = False) -> str:
    from . import builder as _b
    return _b.build(verbose=verbose)


def load_library() -> C.CDLL:
    """Load liblbgpu.so (fails loudly when it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LbgpuError(E_STATE, f"{LIB_PATH} is not built; run paper_1501_04741_b200/builder.py")
    L = C.CDLL(LIB_PATH)
    vp, i64, dp = C.c_void_p, C.c_int64, C.POINTER(C.c_double)
    L.lbgpu_version.restype = C.c_char_p
    L.lbgpu_last_create_error.restype = C.c_char_p
    L.lbgpu_error_message.restype = C.c_char_p
    L.lbgpu_error_message.argtypes = [vp]
    L.lbgpu_create.argtypes = [C.POINTER(SystemDesc), C.POINTER(vp)]
    L.lbgpu_create_from_config.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.POINTER(vp)]
    L.lbgpu_create_from_config_ex.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_int,
                                              C.c_int, C.c_int, C.POINTER(vp)]
    L.lbgpu_destroy.argtypes = [vp]
    L.lbgpu_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(i64)]
    L.lbgpu_get_tables.argtypes = [vp] + [vp] * 9
    L.lbgpu_counters.argtypes = [vp, C.POINTER(i64), C.POINTER(i64)]
    L.lbgpu_stream.argtypes = [vp]
    L.lbgpu_stream.restype = vp
    for name in ("lbgpu_init_state", "lbgpu_reset_adjoint"):
        getattr(L, name).argtypes = [vp]
    for name in ("lbgpu_upload_state", "lbgpu_download_state", "lbgpu_upload_state_device",
                 "lbgpu_download_state_device"):
        getattr(L, name).argtypes = [vp, C.c_int, vp]
    L.lbgpu_set_design.argtypes = [vp, vp]
    L.lbgpu_get_design.argtypes = [vp, vp]
    L.lbgpu_set_design_values.argtypes = [vp, vp]
    L.lbgpu_get_design_values.argtypes = [vp, vp]
    L.lbgpu_primal_step.argtypes = [vp, i64, dp]
    L.lbgpu_primal_step_with_design.argtypes = [vp, vp, i64, dp]
    L.lbgpu_pair_steps.argtypes = [vp, i64, dp, dp]
    L.lbgpu_pair_step_with_design.argtypes = [vp, vp, dp, dp, dp]
    L.lbgpu_finish.argtypes = [vp]
    L.lbgpu_time_pair_steps.argtypes = [vp, i64, dp]
    L.lbgpu_fd_gradient.argtypes = [vp, i64, C.c_double, C.c_double, i64, i64, dp]
    L.lbgpu_fd_gradient_batch.argtypes = [vp, i64, vp, vp, C.c_double, i64, i64, C.c_int, vp]
    L.lbgpu_tangent_solve.argtypes = [vp, vp, C.c_double, C.c_double, i64, dp, C.POINTER(i64), dp,
                                      C.POINTER(C.c_int)]
    L.lbgpu_adjoint_step.argtypes = [vp, i64, C.c_int, dp]
    L.lbgpu_solve_primal.argtypes = [vp, C.c_double, i64, i64, C.POINTER(i64), dp,
                                     C.POINTER(C.c_int)]
    L.lbgpu_solve_adjoint.argtypes = [vp, C.c_double, i64, i64, C.c_int, C.POINTER(i64), dp,
                                      C.POINTER(C.c_int)]
    L.lbgpu_param_gradient.argtypes = [vp, C.c_int, vp, dp]
    L.lbgpu_objective.argtypes = [vp, dp]
    L.lbgpu_penalty.argtypes = [vp, dp]
    L.lbgpu_one_shot.argtypes = [vp, i64, vp, vp, i64, vp, i64, C.POINTER(i64)]
    L.lbgpu_time_sweeps.argtypes = [vp, C.c_int, i64, dp]
    L.lbgpu_time_pairs.argtypes = [vp, i64, dp, dp, dp]
    L.lbgpu_slab_nxl.argtypes = [C.c_int]
    L.lbgpu_create_slab_from_config.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_int,
                                                C.c_int, C.POINTER(vp)]
    L.lbgpu_slab_info.argtypes = [vp, C.POINTER(C.c_int)]
    L.lbgpu_group_link.argtypes = [C.POINTER(vp), C.c_int]
    L.lbgpu_group_link_p2p.argtypes = [C.POINTER(vp), C.c_int]
    L.lbgpu_group_step.argtypes = [C.POINTER(vp), C.c_int, C.c_int, i64, C.c_int, dp]
    L.lbgpu_group_time.argtypes = [C.POINTER(vp), C.c_int, C.c_int, i64, dp]
    L.lbgpu_group_exchange.argtypes = [C.POINTER(vp), C.c_int, C.c_int]
    L.lbgpu_nccl_unique_id.argtypes = [vp, C.c_int]
    L.lbgpu_attach_nccl.argtypes = [vp, vp, C.c_int, C.c_int]
    L.lbgpu_exchange.argtypes = [vp, C.c_int]
    L.lbgpu_unsteady_adjoint.argtypes = [vp, i64, C.c_int, i64, vp, dp, dp, C.POINTER(i64)]
    L.lbgpu_sweep_launches.argtypes = [vp]
    L.lbgpu_sweep_launches.restype = i64
    _lib = L
    return L


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class Engine:
    """One lattice on one B200 (see include/lbgpu.h)."""

    def __init__(self, handle: int):
        self.L = load_library()
        self.h = C.c_void_p(handle)
        dims = (C.c_int * 8)()
        cnt = (C.c_int64 * 4)()
        self._ok(self.L.lbgpu_info(self.h, dims, cnt))
        self.shape = (dims[0], dims[1], dims[2])
        self.m, self.mf, self.mt, self.precision, self.exact = dims[3], dims[4], dims[5], dims[6], dims[7]
        self.n, self.n_design, self.n_support, self.n_inlets = cnt[0], cnt[1], cnt[2], cnt[3]
        self._wd_cache = (None, None)  # (design buffer, its address): pair_step_with_design

    # --- construction -------------------------------------------------------
    @classmethod
    def from_config(cls, cfg_text: str, overrides: dict | None = None, device: int = 0,
                    exact: bool = False, streaming: str = "double") -> "Engine":
        """CaseConfig text (+ dotted overrides) -> build_case -> engine.
        streaming: "double" (two state buffers per field, every operation) or
        "aa" (in place, one buffer per field: fixed-step sweeps, pairs,
        objective and gradient only)."""
        return cls._create(cfg_text, overrides, device, exact, 1, 0, streaming)

    @classmethod
    def _create(cls, cfg_text, overrides, device, exact, slab_count, slab_id, streaming):
        L = load_library()
        ov = "\n".join(f"{k}={v}" for k, v in (overrides or {}).items()).encode()
        if streaming not in ("double", "aa"):
            raise LbgpuError(E_ARG, f"streaming must be 'double' or 'aa', not {streaming!r}")
        h = C.c_void_p()
        rc = L.lbgpu_create_from_config_ex(cfg_text.encode(), ov, device, int(exact), slab_count,
                                           slab_id, int(streaming == "aa"), C.byref(h))
        if rc:
            raise LbgpuError(rc, L.lbgpu_last_create_error().decode())
        return cls(h.value)

    @classmethod
    def from_tables(cls, *, shape, tag, bc_T, bc_axis, bc_sign, w, mask, support,
                    nu=0.02, beta_fluid=0.003, beta_solid=0.003, inlet_dp=0.0, u_clamp=0.05,
                    omega_nonhydro=1.0, switch_theta=3.0, fluid_power=False, bgk=False,
                    obj_kind=0, precision=64, exact=False, device=0, A=None, vel=None,
                    opp=None, relax=None, flux_axis=0, flux_sign=1,
                    streaming: str = "double") -> "Engine":
        """Flattened System arrays (the drop-in seam fed by the reference's own
        System)."""
        L = load_library()
        keep = []

        def arr(a, dt):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a.ctypes.data

        d = SystemDesc()
        d.nx, d.ny, d.nz = shape
        d.precision, d.exact, d.device = precision, int(exact), device
        d.collision = int(bgk)
        d.nu, d.beta_fluid, d.beta_solid, d.inlet_dp = nu, beta_fluid, beta_solid, inlet_dp
        d.u_clamp, d.omega_nonhydro, d.switch_theta = u_clamp, omega_nonhydro, switch_theta
        d.switch_form = int(fluid_power)
        d.A = arr(A, np.float64)
        d.relax = arr(relax, np.float64)
        d.vel = arr(vel, np.int32)
        d.opp = arr(opp, np.int32)
        d.tag, d.bc_T = arr(tag, np.uint8), arr(bc_T, np.float64)
        d.bc_axis, d.bc_sign = arr(bc_axis, np.int8), arr(bc_sign, np.int8)
        d.w, d.design_mask = arr(w, np.float64), arr(mask, np.uint8)
        d.obj_kind, d.flux_axis, d.flux_sign = obj_kind, flux_axis, flux_sign
        d.streaming = int(streaming == "aa")
        d.support = arr(support, np.int64)
        d.n_support = len(support)
        h = C.c_void_p()
        rc = L.lbgpu_create(C.byref(d), C.byref(h))
        if rc:
            raise LbgpuError(rc, L.lbgpu_last_create_error().decode())
        return cls(h.value)

    @classmethod
    def slab_from_config(cls, cfg_text: str, overrides: dict | None, slab_count: int,
                         slab_id: int, device: int = 0, exact: bool = False,
                         streaming: str = "double") -> "Engine":
        """Slab `slab_id` of decompose(nx, slab_count) (partition.cpp:9-21);
        slab_id -1 with slab_count 1: the whole lattice in ghost layout."""
        return cls._create(cfg_text, overrides, device, exact, slab_count, slab_id, streaming)

    def slab(self) -> dict:
        v = (C.c_int * 6)()
        self._ok(self.L.lbgpu_slab_info(self.h, v))
        return dict(zip(("gnx", "x0", "span", "nxl", "count", "id"), list(v)))

    def attach_nccl(self, unique_id: bytes, nranks: int, rank: int) -> None:
        buf = C.create_string_buffer(unique_id, len(unique_id))
        self._ok(self.L.lbgpu_attach_nccl(self.h, buf, nranks, rank))

    def exchange(self, field: int) -> None:
        self._ok(self.L.lbgpu_exchange(self.h, field))

    def close(self) -> None:
        if getattr(self, "h", None):
            self.L.lbgpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ok(self, rc: int) -> None:
        if rc:
            raise LbgpuError(rc, self.L.lbgpu_error_message(self.h).decode())

    # --- tables / state -------------------------------------------------------
    def tables(self) -> dict:
        n = self.n
        t = {"tag": np.zeros(n, np.uint8), "bc_T": np.zeros(n), "bc_axis": np.zeros(n, np.int8),
             "bc_sign": np.zeros(n, np.int8), "w": np.zeros(n), "mask": np.zeros(n, np.uint8),
             "design": np.zeros(max(self.n_design, 1), np.int64),
             "support": np.zeros(max(self.n_support, 1), np.int64),
             "A": np.zeros((self.mf, self.mf))}
        self._ok(self.L.lbgpu_get_tables(self.h, *[_ptr(t[k]) for k in (
            "tag", "bc_T", "bc_axis", "bc_sign", "w", "mask", "design", "support", "A")]))
        t["design"] = t["design"][: self.n_design]
        t["support"] = t["support"][: self.n_support]
        return t

    def counters(self) -> tuple[int, int]:
        p, a = C.c_int64(), C.c_int64()
        self._ok(self.L.lbgpu_counters(self.h, C.byref(p), C.byref(a)))
        return p.value, a.value

    def stream(self) -> int:
        return self.L.lbgpu_stream(self.h)

    def init_state(self) -> None:
        self._ok(self.L.lbgpu_init_state(self.h))

    def reset_adjoint(self) -> None:
        self._ok(self.L.lbgpu_reset_adjoint(self.h))

    def get_state(self, field: int = 0) -> np.ndarray:
        out = np.empty(self.m * self.n)
        self._ok(self.L.lbgpu_download_state(self.h, field, _ptr(out)))
        return out

    def set_state(self, field: int, data: np.ndarray) -> None:
        data = np.ascontiguousarray(data, np.float64)
        assert data.size == self.m * self.n
        self._ok(self.L.lbgpu_upload_state(self.h, field, _ptr(data)))

    def set_design(self, w_full: np.ndarray) -> None:
        w_full = np.ascontiguousarray(w_full, np.float64)
        self._ok(self.L.lbgpu_set_design(self.h, _ptr(w_full)))

    def set_design_values(self, w_design: np.ndarray) -> None:
        """Design values in DesignField::nodes order (host buffer, may be pinned)."""
        w_design = np.ascontiguousarray(w_design, np.float64)
        assert w_design.size == self.n_design
        self._ok(self.L.lbgpu_set_design_values(self.h, _ptr(w_design)))

    def primal_step_with_design(self, w_design: np.ndarray, n: int = 1,
                                residual: bool = True) -> float | None:
        """New design values (DesignField::nodes order) then n primal steps,
        the upload pipelined under the first sweep (optimizer.cpp:200-202)."""
        w_design = np.ascontiguousarray(w_design, np.float64)
        assert w_design.size == self.n_design
        r = C.c_double()
        self._ok(self.L.lbgpu_primal_step_with_design(self.h, _ptr(w_design), n,
                                                      C.byref(r) if residual else None))
        return r.value if residual else None

    def pair_step_with_design(self, w_design: np.ndarray, residual: bool = True,
                              objective: bool = True):
        """New design values, one primal step, one adjoint step against the new
        state and J of that state (optimizer.cpp:33-34, :200-202), as one
        overlapped pipeline. Returns (primal_residual, adjoint_residual, J),
        None where not requested."""
        w_design = np.ascontiguousarray(w_design, np.float64)
        if self._wd_cache[0] is not w_design:  # one optimizer buffer, reused every call
            assert w_design.size == self.n_design
            self._wd_cache = (w_design, _ptr(w_design))
        rp, ra, j = C.c_double(), C.c_double(), C.c_double()
        self._ok(self.L.lbgpu_pair_step_with_design(
            self.h, self._wd_cache[1], C.byref(rp) if residual else None,
            C.byref(ra) if residual else None, C.byref(j) if objective else None))
        return (rp.value if residual else None, ra.value if residual else None,
                j.value if objective else None)

    def finish(self) -> None:
        """Complete any deferred sweep (pair_step_with_design) and synchronize."""
        self._ok(self.L.lbgpu_finish(self.h))

    def pair_steps(self, n: int = 1, residual: bool = True):
        """n primal+adjoint pairs (one-shot at zeta = 0 without the gradient);
        (primal, adjoint) residuals of the last pair, or None."""
        rp, ra = C.c_double(), C.c_double()
        if residual:
            self._ok(self.L.lbgpu_pair_steps(self.h, n, C.byref(rp), C.byref(ra)))
            return rp.value, ra.value
        self._ok(self.L.lbgpu_pair_steps(self.h, n, None, None))
        return None

    def time_pair_steps(self, n: int) -> float:
        """Milliseconds (CUDA events) of pair_steps(n) without residuals."""
        ms = C.c_double()
        self._ok(self.L.lbgpu_time_pair_steps(self.h, n, C.byref(ms)))
        return ms.value

    def fd_gradient(self, ordinal: int, h: float, tol: float, max_iter: int = 200000,
                    fixed_iters: int = -1) -> float:
        """fd_gradient (adjoint.cpp:492-517): ordinal in DesignField::nodes order,
        < 0 for inlet_dp."""
        out = C.c_double()
        self._ok(self.L.lbgpu_fd_gradient(self.h, ordinal, h, tol, max_iter, fixed_iters,
                                          C.byref(out)))
        return out.value

    def fd_gradient_batch(self, ordinals, steps, tol: float = 0.0, max_iter: int = 200000,
                          fixed_iters: int = -1, from_state: bool = False) -> np.ndarray:
        """fd_gradient for many (ordinal, step) components in one call (one
        host sync with fixed_iters >= 0); from_state: each side restarts from
        the current primal state instead of initialize_state."""
        o = np.ascontiguousarray(ordinals, np.int64)
        h = np.ascontiguousarray(steps, np.float64)
        assert o.size == h.size
        out = np.zeros(max(o.size, 1))
        self._ok(self.L.lbgpu_fd_gradient_batch(self.h, o.size, _ptr(o), _ptr(h), tol, max_iter,
                                                fixed_iters, int(from_state), _ptr(out)))
        return out[: o.size]

    def tangent_solve(self, dw: np.ndarray, d_inlet_dp: float, tol: float,
                      max_iter: int = 200000) -> tuple[float, int, float, bool]:
        """tangent_solve (adjoint.cpp:422-490) from the current primal state:
        (dF, iterations, residual, converged)."""
        dw = np.ascontiguousarray(dw, np.float64)
        assert dw.size == self.n_design
        dF, r = C.c_double(), C.c_double()
        it, cv = C.c_int64(), C.c_int()
        self._ok(self.L.lbgpu_tangent_solve(self.h, _ptr(dw), d_inlet_dp, tol, max_iter,
                                            C.byref(dF), C.byref(it), C.byref(r), C.byref(cv)))
        return dF.value, it.value, r.value, bool(cv.value)

    def design_values(self) -> np.ndarray:
        out = np.empty(max(self.n_design, 1))
        self._ok(self.L.lbgpu_get_design_values(self.h, _ptr(out)))
        return out[: self.n_design]

    def design(self) -> np.ndarray:
        out = np.empty(self.n)
        self._ok(self.L.lbgpu_get_design(self.h, _ptr(out)))
        return out

    # --- operators --------------------------------------------------------------
    def primal_step(self, n: int = 1, residual: bool = True) -> float | None:
        r = C.c_double()
        self._ok(self.L.lbgpu_primal_step(self.h, n, C.byref(r) if residual else None))
        return r.value if residual else None

    def adjoint_step(self, n: int = 1, kernel: int = 0, residual: bool = True) -> float | None:
        r = C.c_double()
        self._ok(self.L.lbgpu_adjoint_step(self.h, n, kernel, C.byref(r) if residual else None))
        return r.value if residual else None

    def solve_primal(self, tol: float, max_iter: int = 200000, fixed_iters: int = -1):
        it, r, cv = C.c_int64(), C.c_double(), C.c_int()
        self._ok(self.L.lbgpu_solve_primal(self.h, tol, max_iter, fixed_iters, C.byref(it),
                                           C.byref(r), C.byref(cv)))
        return it.value, r.value, bool(cv.value)

    def solve_adjoint(self, tol: float, max_iter: int = 200000, fixed_iters: int = -1,
                      kernel: int = 0):
        it, r, cv = C.c_int64(), C.c_double(), C.c_int()
        self._ok(self.L.lbgpu_solve_adjoint(self.h, tol, max_iter, fixed_iters, kernel,
                                            C.byref(it), C.byref(r), C.byref(cv)))
        return it.value, r.value, bool(cv.value)

    def param_gradient(self, kernel: int = 0):
        g = np.zeros(max(self.n_design, 1))
        gdp = C.c_double()
        self._ok(self.L.lbgpu_param_gradient(self.h, kernel, _ptr(g), C.byref(gdp)))
        return g[: self.n_design], gdp.value

    def objective(self) -> float:
        v = C.c_double()
        self._ok(self.L.lbgpu_objective(self.h, C.byref(v)))
        return v.value

    def penalty(self) -> float:
        v = C.c_double()
        self._ok(self.L.lbgpu_penalty(self.h, C.byref(v)))
        return v.value

    def one_shot(self, zeta, lam, record_interval: int = 100) -> np.ndarray:
        zeta = np.ascontiguousarray(zeta, np.float64)
        lam = np.ascontiguousarray(lam, np.float64)
        iters = zeta.size
        cap = iters // record_interval + 2
        rows = (RunRow * cap)()
        nr = C.c_int64()
        self._ok(self.L.lbgpu_one_shot(self.h, iters, _ptr(zeta), _ptr(lam), record_interval,
                                       C.addressof(rows), cap, C.byref(nr)))
        return np.array([[getattr(r, k) for k, _ in RunRow._fields_] for r in rows[: nr.value]])

    def unsteady_adjoint(self, n_steps: int, sum_objective: bool = False, slots: int = 8):
        """Discrete adjoint of n_steps primal steps from the current state
        (checkpoint + recompute). Returns (J, dJ/dw design order, dJ/d inlet_dp,
        primal sweeps spent)."""
        g = np.zeros(max(self.n_design, 1))
        gdp, J, fs = C.c_double(), C.c_double(), C.c_int64()
        self._ok(self.L.lbgpu_unsteady_adjoint(self.h, n_steps, int(sum_objective), slots, _ptr(g),
                                               C.byref(gdp), C.byref(J), C.byref(fs)))
        return J.value, g[: self.n_design], gdp.value, fs.value

    def time_sweeps(self, which: int, steps: int) -> float:
        """Milliseconds of `steps` back-to-back sweeps (CUDA events on the
        engine stream). which: 0 primal, 1 adjoint."""
        ms = C.c_double()
        self._ok(self.L.lbgpu_time_sweeps(self.h, which, steps, C.byref(ms)))
        return ms.value


    def time_pairs(self, steps: int) -> tuple[float, float, float]:
        """(total, primal, adjoint) milliseconds of `steps` primal+adjoint
        sweep pairs, CUDA events between sweeps on the engine stream."""
        t, p, a = C.c_double(), C.c_double(), C.c_double()
        self._ok(self.L.lbgpu_time_pairs(self.h, steps, C.byref(t), C.byref(p), C.byref(a)))
        return t.value, p.value, a.value

    def sweep_launches(self) -> int:
        return int(self.L.lbgpu_sweep_launches(self.h))


def nccl_unique_id() -> bytes:
    L = load_library()
    buf = C.create_string_buffer(256)
    rc = L.lbgpu_nccl_unique_id(buf, 256)
    if rc:
        raise LbgpuError(rc, "ncclGetUniqueId failed")
    return buf.raw[:128]


class SlabGroup:
    """In-process lock-step group of slab engines: the PartitionedRun of
    partition.cpp:43-312.

    transport "pull": one device, one shared stream, the halo exchange done by
    a kernel that reads the neighbour slabs' buffers after each sweep.
    transport "p2p": one stream per slab, slabs on `devices` (round robin;
    default all on `device`); each sweep stores its boundary planes straight
    into the neighbours' ghost columns (peer memory across GPUs) and waits only
    on its two neighbours' previous sweep."""

    def __init__(self, cfg_text: str, overrides: dict | None, n: int, device: int = 0,
                 exact: bool = False, transport: str = "pull", devices=None):
        devs = list(devices) if devices else [device]
        self.engines = [Engine.slab_from_config(cfg_text, overrides, n, i, devs[i % len(devs)],
                                                exact) for i in range(n)]
        self.L = load_library()
        self._arr = (C.c_void_p * n)(*[e.h.value for e in self.engines])
        if transport == "p2p" and n > 1:
            rc = self.L.lbgpu_group_link_p2p(self._arr, n)
        elif transport in ("pull", "p2p"):
            rc = self.L.lbgpu_group_link(self._arr, n)
        else:
            raise ValueError(f"unknown transport {transport!r}")
        if rc:
            raise LbgpuError(rc, self.L.lbgpu_error_message(self._arr[0]).decode()
                             or "lbgpu_group_link failed")
        self.n = n
        self.slabs = [e.slab() for e in self.engines]
        e0 = self.engines[0]
        self.m, self.mf = e0.m, e0.mf
        self.shape = (self.slabs[0]["gnx"], e0.shape[1], e0.shape[2])

    def _ok(self, rc):
        if rc:
            raise LbgpuError(rc, self.L.lbgpu_error_message(self._arr[0]).decode())

    def init_state(self):
        for e in self.engines:
            e.init_state()

    def step(self, which: int, steps: int = 1, kernel: int = 0, residual: bool = True):
        """which: 0 primal, 1 adjoint, 2 fused pair sweeps (P2P groups; no
        residual). Returns the global residual of the last step, or None."""
        r = C.c_double()
        self._ok(self.L.lbgpu_group_step(self._arr, self.n, which, steps, kernel,
                                         C.byref(r) if residual and which != 2 else None))
        return r.value if residual and which != 2 else None

    def pair_steps(self, n: int = 1) -> None:
        """lbgpu_pair_steps over the group: primal, n-1 fused pair sweeps, adjoint."""
        if n <= 0:
            return
        self.step(0, 1, residual=False)
        if n > 1:
            self.step(2, n - 1)
        self.step(1, 1, residual=False)

    def time(self, which: int, steps: int) -> float:
        """P2P group: milliseconds of `steps` lock steps (max over slabs)."""
        ms = C.c_double()
        self._ok(self.L.lbgpu_group_time(self._arr, self.n, which, steps, C.byref(ms)))
        return ms.value

    def exchange(self, field: int):
        self._ok(self.L.lbgpu_group_exchange(self._arr, self.n, field))

    def get_state(self, field: int) -> np.ndarray:
        nx, ny, nz = self.shape
        out = np.empty((self.m, nz, ny, nx))
        for e, s in zip(self.engines, self.slabs):
            loc = e.get_state(field).reshape(self.m, nz, ny, s["nxl"])
            out[..., s["x0"]: s["x0"] + s["span"]] = loc[..., : s["span"]]
        return out.reshape(-1)

    def set_state(self, field: int, data: np.ndarray):
        for e, s in zip(self.engines, self.slabs):
            e.set_state(field, slab_cut(data, self.m, self.shape, s))
        self.exchange(field)

    def gradient(self, kernel: int = 0):
        """Design gradient in global DesignField::nodes order + inlet_dp."""
        idx, vals, gdp = [], [], 0.0
        nx, ny, _ = self.shape
        for e, s in zip(self.engines, self.slabs):
            g, d = e.param_gradient(kernel)
            loc = e.tables()["design"]
            lx, rest = loc % s["nxl"], loc // s["nxl"]
            idx.append(lx + s["x0"] + nx * rest)
            vals.append(g)
            gdp += d
        idx = np.concatenate(idx)
        order = np.argsort(idx, kind="stable")
        return np.concatenate(vals)[order], gdp

    def objective(self) -> float:
        return sum(e.objective() for e in self.engines)


def slab_cut(data: np.ndarray, m: int, shape, s: dict) -> np.ndarray:
    """Local reference-layout array of slab s (owned columns + both ghosts)."""
    nx, ny, nz = shape
    g = np.asarray(data, np.float64).reshape(m, nz, ny, nx)
    loc = np.zeros((m, nz, ny, s["nxl"]))
    span, x0 = s["span"], s["x0"]
    loc[..., :span] = g[..., x0: x0 + span]
    loc[..., span] = g[..., (x0 + span) % nx]
    loc[..., s["nxl"] - 1] = g[..., (x0 - 1) % nx]
    return loc.reshape(-1)


def version() -> str:
    return load_library().lbgpu_version().decode()

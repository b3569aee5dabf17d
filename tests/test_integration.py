"""The drop-in boundary seen from the reference's side.

* CPU: the binding a maintainer adds to the reference (integration/gpu_engine.cpp,
  INTEGRATION.md §2) compiles against the reference's own headers
  (/root/reference/proj/include) and this repo's include/lbgpu.h, warnings as
  errors; skipped where the reference tree is absent.
* GPU: oracle/_ref/drop_in_check -- that binding linked with the reference's
  own objects -- builds a case with the reference's parse_text/build_case,
  solves it with the reference on the CPU and, through make_gpu_engine (the
  reference's System: tags, bc arrays, design, support, ModelTables::A and
  relax, vel/opp fed to lbgpu_create), on the GPU. In the bit-exact build the
  two agree bit for bit: states, residuals, objective, gradient, and one
  MMA-shaped outer iteration (design write-back, solve_fixed_point,
  solve_adjoint, param_gradient).
* GPU: the same through the Python mirror -- RefOracle.tables() fed to
  Engine.from_tables (lbgpu_create) -- against oracle/_ref.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from cases import case_text

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
DROP_IN = os.path.join(ROOT, "oracle", "_ref", "drop_in_check")


def test_binding_compiles_against_reference_headers(tmp_path):
    if not os.path.isdir(REF_INC):
        pytest.skip("no /root/reference here")
    for src in ("gpu_engine.cpp", "drop_in_check.cpp"):
        subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-c",
                        f"-I{REF_INC}", f"-I{ROOT}/include", f"-I{ROOT}/integration",
                        os.path.join(ROOT, "integration", src), "-o", str(tmp_path / (src + ".o"))],
                       check=True)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["grad2d", "mix3d", "exch3d", "bgk3d", "pois2d"])
def test_reference_system_through_the_binding(has_gpu, tmp_path, name):
    if not os.path.exists(DROP_IN):
        pytest.skip("oracle/_ref/drop_in_check not built (needs /root/reference at build time)")
    cfg = tmp_path / "case.cfg"
    cfg.write_text(case_text(name))
    for exact in (1, 0):
        out = subprocess.run([DROP_IN, str(cfg), str(exact), "120", "40"], check=True,
                             capture_output=True, text=True).stdout
        d = json.loads(out.strip().splitlines()[-1])
        assert d["primal_iters"][0] == d["primal_iters"][1] == 120
        if exact:
            assert d["f_maxdiff"] == 0 and d["v_maxdiff"] == 0, d
            assert d["primal_residual"][0] == d["primal_residual"][1]
            assert d["adjoint_residual"][0] == d["adjoint_residual"][1]
            assert d["J"][0] == d["J"][1] and d["gdp"][0] == d["gdp"][1]
            assert d["g_maxdiff"] == 0 and d["mma_g_maxdiff"] == 0, d
        else:
            assert d["f_maxdiff"] <= 1e-12 * d["f_max"]
            assert d["v_maxdiff"] <= 1e-11 * d["v_max"]
            assert d["g_maxdiff"] <= 1e-10 * d["g_max"]
            assert d["mma_g_maxdiff"] <= 1e-10 * d["mma_g_max"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["grad2d", "mix3d", "exch3d", "solid2d"])
def test_from_reference_tables_bitwise(lbgpu, oracle_mod, has_gpu, name):
    """lbgpu_create fed with the reference's own System arrays (A, relax,
    vel, opp included) through the Python mirror: bitwise the reference."""
    txt = case_text(name)
    r = oracle_mod.RefOracle(txt)
    t = r.tables()
    c = oracle_mod.parse_cfg(txt)
    e = lbgpu.Engine.from_tables(
        shape=r.shape, tag=t["tag"], bc_T=t["bc_T"], bc_axis=t["bc_axis"], bc_sign=t["bc_sign"],
        w=t["w"], mask=t["mask"], support=t["support"], nu=float(c["model.nu"]),
        beta_fluid=float(c["model.beta_fluid"]), beta_solid=float(c["model.beta_solid"]),
        inlet_dp=float(c["model.inlet_dp"]), u_clamp=float(c["model.u_clamp"]),
        omega_nonhydro=float(c["model.omega_nonhydro"]),
        switch_theta=float(c["model.switch_theta"]),
        fluid_power=c["model.switch_form"] == "fluid_power", bgk=c["model.collision"] == "bgk",
        obj_kind={"mixing": 0, "heatflux": 1, "synthetic": 2}[c["objective.kind"]],
        exact=True, A=t["A"], relax=t["relax"], vel=t["vel"], opp=t["opp"])
    r.init_state()
    e.init_state()
    assert e.primal_step(60) == r.primal_steps(60)
    assert np.array_equal(e.get_state(0), r.get_state(0))
    assert e.adjoint_step(25) == r.adjoint_steps(25)
    assert np.array_equal(e.get_state(1), r.get_state(1))
    ge, de = e.param_gradient()
    gr, dr = r.gradient()
    assert np.array_equal(ge, gr) and de == dr
    assert e.objective() == r.objective()

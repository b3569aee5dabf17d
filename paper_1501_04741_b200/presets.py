"""Reference presets (proj/presets/*.cfg) restated as dotted-key tables.

The reference ships six case files; they are the inputs every BASELINE config
starts from. They are kept here as data so the GPU boxes, which
have no /root/reference, see the same inputs; ``preset_text`` renders the INI
form the reference parser (config.cpp:129-154) and ours both accept.
"""
from __future__ import annotations

PRESETS: dict[str, dict[str, object]] = {
    # proj/presets/gradcheck2d.cfg: small channel for adjoint-vs-FD checks
    "gradcheck2d": {
        "lattice.nx": 12, "lattice.ny": 8,
        "model.nu": 0.02, "model.beta_fluid": 0.003, "model.beta_solid": 0.003,
        "model.inlet_dp": 0.002,
        "tags.design_x0": 3, "tags.design_x1": 8, "tags.inlet_profile": "split",
        "objective.kind": "mixing", "objective.plane_offset": 1,
        "optimizer.initial_w": 0.5, "optimizer.primal_tol": 1e-12,
        "optimizer.adjoint_tol": 1e-12,
        "output.dir": "out/gradcheck2d", "output.write_vtk": "false",
    },
    # proj/presets/mixer2d.cfg: desk-scale two-stream mixer
    "mixer2d": {
        "lattice.nx": 90, "lattice.ny": 10,
        "model.nu": 0.02, "model.inlet_dp": 0.016666, "model.beta_fluid": 0.003,
        "model.beta_solid": 0.003, "model.switch_form": "fluid_power",
        "tags.design_x0": 20, "tags.design_x1": 70, "tags.inlet_profile": "split",
        "objective.kind": "mixing", "objective.plane_offset": 1,
        "optimizer.method": "oneshot", "optimizer.iterations": 200000,
        "optimizer.zeta_stages": "0:0,15000:0.0001,90000:0.00003",
        "optimizer.initial_w": 1.0, "optimizer.primal_tol": 1e-9,
        "optimizer.adjoint_tol": 1e-9, "optimizer.record_interval": 1000,
        "output.dir": "out/mixer2d",
    },
    # proj/presets/mixer3d.cfg: full-scale 3D mixer
    "mixer3d": {
        "lattice.nx": 450, "lattice.ny": 50, "lattice.nz": 50,
        "model.nu": 0.02, "model.inlet_dp": 0.016666, "model.beta_fluid": 0.003,
        "model.beta_solid": 0.003, "model.switch_form": "fluid_power",
        "tags.design_x0": 61, "tags.design_x1": 390, "tags.inlet_profile": "split",
        "objective.kind": "mixing", "objective.plane_offset": 1,
        "optimizer.method": "oneshot", "optimizer.iterations": 1000000,
        "optimizer.zeta_stages": "0:0,20000:0.0001,120000:0.00003",
        "optimizer.initial_w": 1.0, "optimizer.primal_tol": 1e-9,
        "optimizer.adjoint_tol": 1e-9, "optimizer.record_interval": 5000,
        "output.dir": "out/mixer3d",
    },
    # proj/presets/exchanger2d.cfg: desk-scale heat exchanger
    "exchanger2d": {
        "lattice.nx": 70, "lattice.ny": 10,
        "model.nu": 0.01, "model.inlet_dp": 0.03, "model.beta_fluid": 0.003,
        "model.beta_solid": 1.0, "model.switch_form": "fluid_power",
        "tags.design_x0": 20, "tags.design_x1": 49, "tags.heater_x0": 30,
        "tags.heater_x1": 39, "tags.inlet_profile": "uniform", "tags.inlet_T": 0,
        "objective.kind": "heatflux", "objective.plane_offset": 1,
        "optimizer.method": "oneshot", "optimizer.iterations": 150000,
        "optimizer.zeta_stages": "0:0,10000:0.0001,60000:0.00003",
        "optimizer.initial_w": 1.0, "optimizer.primal_tol": 1e-9,
        "optimizer.adjoint_tol": 1e-9, "optimizer.record_interval": 1000,
        "output.dir": "out/exchanger2d",
    },
    # proj/presets/exchanger3d.cfg: full-scale 3D heat exchanger
    "exchanger3d": {
        "lattice.nx": 352, "lattice.ny": 50, "lattice.nz": 50,
        "model.nu": 0.01, "model.inlet_dp": 0.03, "model.beta_fluid": 0.003,
        "model.beta_solid": 1.0, "model.switch_form": "fluid_power",
        "tags.design_x0": 101, "tags.design_x1": 252, "tags.heater_x0": 151,
        "tags.heater_x1": 200, "tags.inlet_profile": "uniform", "tags.inlet_T": 0,
        "objective.kind": "heatflux", "objective.plane_offset": 1,
        "optimizer.method": "oneshot", "optimizer.iterations": 1000000,
        "optimizer.zeta_stages": "0:0,20000:0.0001,120000:0.00003",
        "optimizer.initial_w": 1.0, "optimizer.primal_tol": 1e-9,
        "optimizer.adjoint_tol": 1e-9, "optimizer.record_interval": 5000,
        "output.dir": "out/exchanger3d",
    },
    # proj/presets/poiseuille2d.cfg: plane Poiseuille benchmark (TRT magic omega)
    "poiseuille2d": {
        "lattice.nx": 201, "lattice.ny": 15,
        "model.nu": 0.02, "model.inlet_dp": 0.002,
        "model.omega_nonhydro": 0.27586206896551724,
        "tags.inlet_profile": "uniform", "tags.inlet_T": 0,
        "objective.kind": "mixing", "objective.plane_offset": 1,
        "optimizer.primal_tol": 1e-11,
        "output.dir": "out/poiseuille2d", "output.write_vtk": "false",
    },
}

# BASELINE.json configs C1..C5 as preset + overrides.
CONFIGS: dict[str, tuple[str, dict[str, object]]] = {
    "C1": ("gradcheck2d", {
        "lattice.nx": 256, "lattice.ny": 64, "model.collision": "bgk",
        "tags.design_x0": 85, "tags.design_x1": 170, "optimizer.initial_w": 0.5,
        "optimizer.init_noise": 0.3, "optimizer.seed": 7, "optimizer.primal_tol": 1e-10,
        "optimizer.adjoint_tol": 1e-10, "optimizer.max_inner": 3000000}),
    "C2": ("mixer2d", {
        "lattice.nx": 1024, "lattice.ny": 256, "tags.design_x0": 256,
        "tags.design_x1": 767, "optimizer.zeta_stages": "0:0.0001"}),
    "C3": ("mixer3d", {
        "lattice.nx": 256, "lattice.ny": 128, "lattice.nz": 128, "tags.design_x0": 64,
        "tags.design_x1": 191, "optimizer.initial_w": 0.5, "optimizer.init_noise": 0.3,
        "optimizer.seed": 7}),
    "C4": ("exchanger3d", {
        "lattice.nx": 512, "lattice.ny": 128, "lattice.nz": 128, "tags.design_x0": 147,
        "tags.design_x1": 366, "tags.heater_x0": 219, "tags.heater_x1": 291}),
    "C5": ("mixer3d", {
        "lattice.nx": 2048, "lattice.ny": 512, "lattice.nz": 512, "tags.design_x0": 512,
        "tags.design_x1": 1535, "optimizer.initial_w": 0.5, "optimizer.init_noise": 0.3,
        "optimizer.seed": 7}),
}


def _fmt(v: object) -> str:
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, float):
        return repr(v)
    return str(v)


def preset_text(name: str, overrides: dict[str, object] | None = None) -> str:
    """Render a preset (plus dotted-key overrides) as INI text."""
    table = dict(PRESETS[name])
    for k, v in (overrides or {}).items():
        table[k] = v
    sections: dict[str, list[str]] = {}
    for key, v in table.items():
        sec, k = key.split(".", 1)
        sections.setdefault(sec, []).append(f"{k} = {_fmt(v)}")
    out = []
    for sec, lines in sections.items():
        out.append(f"[{sec}]")
        out.extend(lines)
        out.append("")
    return "\n".join(out)


def config_text(cid: str, extra: dict[str, object] | None = None) -> str:
    """INI text for BASELINE config C1..C5 (optionally with more overrides)."""
    name, ov = CONFIGS[cid]
    ov = dict(ov)
    ov.update(extra or {})
    return preset_text(name, ov)

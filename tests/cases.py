"""Parity cases: reference presets + overrides at sizes the CPU oracle
finishes in seconds (configs C1-C5 are larger versions of the
same presets)."""
from paper_1501_04741_b200.presets import preset_text

CASES = {
    # gradcheck2d preset (proj/presets/gradcheck2d.cfg): FMRT, split inlet
    "grad2d": ("gradcheck2d", {}),
    # C1 in miniature: BGK with init noise
    "bgk2d": ("gradcheck2d", {"lattice.nx": 20, "lattice.ny": 10, "model.collision": "bgk",
                              "tags.design_x0": 6, "tags.design_x1": 13,
                              "optimizer.init_noise": 0.3, "optimizer.seed": 7}),
    # 2D exchanger with the heater plate and solid conduction (heatflux)
    "exch2d": ("exchanger2d", {"lattice.nx": 40, "tags.design_x0": 10, "tags.design_x1": 29,
                               "tags.heater_x0": 15, "tags.heater_x1": 24,
                               "optimizer.initial_w": 0.6, "optimizer.init_noise": 0.3,
                               "optimizer.seed": 11}),
    # Poiseuille preset: omega_nonhydro = 8/29 (all MRT rows relax)
    "pois2d": ("poiseuille2d", {"lattice.nx": 30, "lattice.ny": 9}),
    # solid_power switching, uniform inlet temperature
    "solid2d": ("gradcheck2d", {"lattice.nx": 16, "model.switch_form": "solid_power",
                                "tags.inlet_profile": "uniform", "tags.inlet_T": 0.25,
                                "optimizer.initial_w": 0.4, "optimizer.init_noise": 0.35,
                                "optimizer.seed": 3, "model.inlet_dp": 0.01}),
    # C3 in miniature: D3Q19+D3Q7 FMRT mixer
    "mix3d": ("mixer3d", {"lattice.nx": 20, "lattice.ny": 9, "lattice.nz": 8,
                          "tags.design_x0": 5, "tags.design_x1": 14, "optimizer.initial_w": 0.5,
                          "optimizer.init_noise": 0.3, "optimizer.seed": 7}),
    # C4 in miniature: 3D exchanger with a heater plate
    "exch3d": ("exchanger3d", {"lattice.nx": 24, "lattice.ny": 10, "lattice.nz": 12,
                               "tags.design_x0": 6, "tags.design_x1": 17, "tags.heater_x0": 9,
                               "tags.heater_x1": 14, "optimizer.initial_w": 0.7,
                               "optimizer.init_noise": 0.2, "optimizer.seed": 5}),
    # 3D BGK
    "bgk3d": ("mixer3d", {"lattice.nx": 16, "lattice.ny": 8, "lattice.nz": 9,
                          "model.collision": "bgk", "tags.design_x0": 4, "tags.design_x1": 11,
                          "optimizer.initial_w": 0.5, "optimizer.init_noise": 0.3,
                          "optimizer.seed": 2}),
    # all-interior periodic box with the synthetic objective (oracles.hpp:46-55)
    "periodic2d": ("gradcheck2d", {"lattice.nx": 10, "lattice.ny": 7, "tags.geometry": "periodic",
                                   "tags.design_x0": 1, "tags.design_x1": 8,
                                   "objective.kind": "synthetic", "model.beta_solid": 0.01,
                                   "optimizer.init_noise": 0.3, "optimizer.seed": 9}),
}


def case_text(name: str, extra: dict | None = None) -> str:
    preset, ov = CASES[name]
    return preset_text(preset, {**ov, **(extra or {})})

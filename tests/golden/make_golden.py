"""Generate tests/golden/golden.npz from the reference itself.

Runs the reference (oracle/_ref/liblbopt_ref.so, compiled from the sources
under /root/reference by oracle/Makefile) on small parity cases and records
states after fixed step counts, adjoint states, gradients and objectives.
Only this container has /root/reference; the fixture travels with the repo.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from cases import case_text  # noqa: E402
from oracle import oracle as O  # noqa: E402

SPEC = {"grad2d": (40, 20), "exch2d": (60, 30), "bgk3d": (30, 15)}


def main():
    O.build(ref=True)
    out = {"cases": np.array(list(SPEC))}
    for name, (ps, as_) in SPEC.items():
        r = O.RefOracle(case_text(name))
        r.init_state()
        r.primal_steps(ps)
        out[f"{name}/primal_steps"] = np.array(ps)
        out[f"{name}/f"] = r.get_state(0)
        out[f"{name}/objective"] = np.array(r.objective())
        r.adjoint_steps(as_)
        out[f"{name}/adjoint_steps"] = np.array(as_)
        out[f"{name}/v"] = r.get_state(1)
        g, gdp = r.gradient()
        out[f"{name}/grad"] = g
        out[f"{name}/grad_dp"] = np.array(gdp)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)


if __name__ == "__main__":
    main()

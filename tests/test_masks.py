"""Node masks and indexing bit-exact against the reference (SURVEY.md §8a
A1-A4): tags, bc arrays, design mask/nodes/initial w (mt19937_64 noise),
objective support and the relaxation matrix A — from our host builder
(lbgpu_case_tables, no GPU) vs the reference's build_case (oracle/_ref)."""
import ctypes as C

import numpy as np
import pytest

from cases import CASES, case_text
from paper_1501_04741_b200.presets import CONFIGS, config_text


def engine_tables(P, txt, ov=None):
    L = P.load_library()
    ovb = "\n".join(f"{k}={v}" for k, v in (ov or {}).items()).encode()
    dims = (C.c_int * 8)()
    cnt = (C.c_int64 * 4)()
    fn = L.lbgpu_case_tables
    fn.argtypes = [C.c_char_p, C.c_char_p, C.c_void_p, C.c_void_p] + [C.c_void_p] * 9
    rc = fn(txt.encode(), ovb, dims, cnt, *([None] * 9))
    assert rc == 0, L.lbgpu_last_create_error()
    n, nd, ns = cnt[0], cnt[1], cnt[2]
    mf = dims[4]
    t = {"tag": np.zeros(n, np.uint8), "bc_T": np.zeros(n), "bc_axis": np.zeros(n, np.int8),
         "bc_sign": np.zeros(n, np.int8), "w": np.zeros(n), "mask": np.zeros(n, np.uint8),
         "design": np.zeros(max(nd, 1), np.int64), "support": np.zeros(max(ns, 1), np.int64),
         "A": np.zeros((mf, mf))}
    keys = ("tag", "bc_T", "bc_axis", "bc_sign", "w", "mask", "design", "support", "A")
    rc = fn(txt.encode(), ovb, dims, cnt, *[t[k].ctypes.data for k in keys])
    assert rc == 0
    t["design"] = t["design"][:nd]
    t["support"] = t["support"][:ns]
    return t


@pytest.mark.parametrize("name", list(CASES))
def test_case_masks_bit_exact(lbgpu, oracle_mod, name):
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    txt = case_text(name)
    te = engine_tables(lbgpu, txt)
    tr = oracle_mod.RefOracle(txt).tables()
    for k in te:
        assert np.array_equal(te[k], tr[k]), k


@pytest.mark.parametrize("cid", ["C1", "C2", "C3", "C4"])
def test_baseline_config_masks_bit_exact(lbgpu, oracle_mod, cid):
    """Full-size BASELINE configs C1-C4 (C5's 537M nodes is checked by
    construction on its C3-shaped slabs in the multi-slab tests)."""
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    txt = config_text(cid)
    te = engine_tables(lbgpu, txt)
    tr = oracle_mod.RefOracle(txt).tables()
    for k in te:
        assert np.array_equal(te[k], tr[k]), (cid, k)


def test_mask_counts_match_survey(lbgpu):
    """C1 has 5,332 design nodes, C2 130,048, C3 2,032,128."""
    assert len(engine_tables(lbgpu, config_text("C1"))["design"]) == 5332
    assert len(engine_tables(lbgpu, config_text("C2"))["design"]) == 130048
    assert len(engine_tables(lbgpu, config_text("C3"))["design"]) == 2032128

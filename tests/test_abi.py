"""The drop-in boundary: liblbgpu.so loads and exports every symbol
include/lbgpu.h declares; host-only entry points work without a GPU."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols(header="lbgpu.h", prefix="lbgpu_"):
    text = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"\b(" + prefix + r"[a-z_0-9]+)\s*\(", text)))


def test_exports_every_declared_symbol(lbgpu):
    L = lbgpu.load_library()
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_exports_the_reference_case_api(lbgpu):
    """include/lbopt_gpu.h: every function of the reference's lbopt.h
    (lbopt.h:26-61) is exported by liblbgpu.so."""
    L = lbgpu.load_library()
    syms = declared_symbols("lbopt_gpu.h", "lbopt_")
    assert len(syms) == 27
    assert not [s for s in syms if not hasattr(L, s)]
    import ctypes as C
    L.lbopt_version.restype = C.c_char_p
    assert L.lbopt_version() == b"0.1.0"


def test_version(lbgpu):
    assert lbgpu.version().startswith("0.1.0")


def test_bad_config_is_config_error(lbgpu):
    import ctypes as C
    L = lbgpu.load_library()
    dims = (C.c_int * 8)()
    cnt = (C.c_int64 * 4)()
    fn = L.lbgpu_case_tables
    fn.argtypes = [C.c_char_p, C.c_char_p, C.c_void_p, C.c_void_p] + [C.c_void_p] * 9
    rc = fn(b"[lattice]\nnx = 5\nny = 5\n[model]\nbogus = 1\n", None, dims, cnt, *([None] * 9))
    assert rc == lbgpu.E_CONFIG
    assert b"unknown key 'bogus' in section [model]" in L.lbgpu_last_create_error()
    rc = fn(b"[lattice]\nnx = 2\nny = 5\n", None, dims, cnt, *([None] * 9))
    assert rc == lbgpu.E_CONFIG
    assert L.lbgpu_last_create_error() == b"channel geometry needs nx >= 3 and ny >= 3"


def test_null_handle_is_arg_error(lbgpu):
    L = lbgpu.load_library()
    import ctypes as C
    assert L.lbgpu_init_state(None) == lbgpu.E_ARG
    assert L.lbgpu_error_message(None) == b"null handle"
    r = C.c_double()
    assert L.lbgpu_primal_step(None, 1, C.byref(r)) == lbgpu.E_ARG


def test_headers_compile_as_c_and_link(lbgpu, tmp_path):
    """include/lbgpu.h and include/lbopt_gpu.h are plain C: a C99 consumer
    compiles with -Wall -Werror, links against liblbgpu.so and runs its
    host-only calls."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if not gcc:
        pytest.skip("no gcc")
    lib = os.path.dirname(lbgpu.LIB_PATH)
    exe = str(tmp_path / "consumer")
    subprocess.run([gcc, "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "consumer.c"), "-o", exe, "-L", lib,
                    "-llbgpu", "-Wl,-rpath," + lib], check=True)
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, (out.returncode, out.stderr)
    assert out.stdout.startswith("ok 0.1.0")

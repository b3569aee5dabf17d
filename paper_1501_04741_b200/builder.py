"""Build liblbgpu.so (the sm_100a CUDA engine) in-tree.

nvcc -gencode arch=compute_100a,code=sm_100a, one object per translation
unit compiled in parallel; the k_exact_* units with -fmad=false (bit-exact
reference-order build). Incremental: a unit is recompiled when it or any
header in csrc/ is newer than its object.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.environ.get("LBGPU_BUILD_DIR") or os.path.join(HERE, "_build")
LIB = os.environ.get("LBGPU_LIB") or os.path.join(HERE, "liblbgpu.so")
NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
EXTRA = os.environ.get("LBGPU_NVCC_EXTRA", "").split()
COMMON = [*EXTRA, "-std=c++20", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
          "--expt-relaxed-constexpr", "-diag-suppress", "20058",
          f"-I{os.path.join(os.path.dirname(HERE), 'include')}"]
# 20058: "#pragma unroll must precede a loop" — LBGPU_FOR bodies contain
# compile-time-unrolled lambdas; the pragmas there are harmless


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers_mtime() -> float:
    hs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    hs += glob.glob(os.path.join(os.path.dirname(HERE), "include", "*.h"))
    return max((os.path.getmtime(h) for h in hs), default=0.0)


def _compile(src: str, hdr_mtime: float, verbose: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime):
        return obj
    if src.endswith(".cpp"):  # host-only C++ (no device code): the host compiler
        cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else os.environ.get("CXX", "g++")
        cmd = [cxx, "-std=c++20", "-O2", "-fPIC",
               f"-I{os.path.join(os.path.dirname(HERE), 'include')}", "-c", src, "-o", obj]
    else:
        cmd = [NVCC, *ARCH, *COMMON]
        if os.path.basename(src).startswith("k_exact_"):
            cmd.append("-fmad=false")
        cmd += ["-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return obj


def build(verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hm = _headers_mtime()
    srcs = _sources()
    with ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, hm, verbose), srcs))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        subprocess.run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-ldl"], check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))

"""Build libspmv_b200.so in-tree (nvcc for sm_100a + g++), no torch involved.

    python -m paper_1203_2739_b200.build [--force] [--verbose]

The CUDA runtime is linked statically (the library is built with nvcc 12.9;
torch in the same process carries its own 12.8 runtime), NCCL is the venv's
libnccl.so.2 that torch itself loads (one NCCL per process), found by rpath.
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libspmv_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir() -> str:
    for base in [sysconfig.get_paths()["purelib"], sysconfig.get_paths()["platlib"]]:
        d = os.path.join(base, "nvidia", "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("venv NCCL (nvidia/nccl) not found")


SOURCES = {
    "kernels.cu": "cu",
    "rowtile.cu": "cu",
    "split.cu": "cu",
    "panel.cu": "cu",
    "order.cu": "cu",
    "xstaged.cu": "cu",
    "plan_panel.cpp": "cpp",
    "host.cpp": "cpp",
    "exchange.cpp": "cpp",
    "test_hooks.cpp": "cpp",
}
HEADERS = ["internal.h", "plan_panel.h", "handle.h", "exchange.h", os.path.join("..", "..", "include", "spmv.h"),
           os.path.join("..", "..", "include", "spmv_test.h")]
# measurement microkernels: a separate library (include/spmv_diag.h), not the SpMxV path
DIAG_DIR = os.path.join(HERE, "diag")
DIAG_SOURCES = ["diag.cu", "diag2.cu", "api.cu"]
DIAG_LIB = os.path.join(HERE, "libspmv_diag.so")


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    nccl = _nccl_dir()
    inc = ["-I" + CSRC, "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(nccl, "include"),
           "-I" + os.path.join(CUDA, "include")]
    hdrs = [os.path.join(CSRC, h) for h in HEADERS]
    # build-time experiments only (e.g. "-DSPMV_PN_PEND=64"); the library reads no environment at run time
    defs = os.environ.get("SPMV_BUILD_DEFS", "").split()
    objs = []
    for src, kind in SOURCES.items():
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if not force and not _newer(o, [s, __file__] + hdrs):
            continue
        if kind == "cu":
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                   "--expt-relaxed-constexpr", "-Xptxas", "-v", "-c", s, "-o", o, *inc, *defs]
        else:
            cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-fopenmp", "-Wall", "-Wno-unused-function",
                   "-c", s, "-o", o, *inc, *defs]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stdout.write(r.stdout)
            sys.stdout.write(r.stderr)
        if r.returncode:
            raise RuntimeError(f"compile failed: {src}")
    if force or _newer(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        nccl_lib = os.path.join(nccl, "lib")
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
               "-Xcompiler", "-fopenmp", "-lgomp",
               "-L" + nccl_lib, "-Xlinker", "-l:libnccl.so.2",
               "-Xlinker", "-rpath," + nccl_lib]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.stdout.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
        os.replace(tmp, LIB)
    build_diag(force, verbose)
    return LIB


def build_diag(force: bool = False, verbose: bool = False) -> str:
    """libspmv_diag.so: the measurement microkernels bench.py uses for its live peaks."""
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    hdrs = [os.path.join(DIAG_DIR, "diag.h"), os.path.join(ROOT, "include", "spmv_diag.h")]
    for src in DIAG_SOURCES:
        s = os.path.join(DIAG_DIR, src)
        o = os.path.join(BUILD, "diag_" + src + ".o")
        objs.append(o)
        if not force and not _newer(o, [s, __file__] + hdrs):
            continue
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-c", s, "-o", o,
               "-I" + DIAG_DIR, "-I" + os.path.join(ROOT, "include")]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stdout.write(r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"compile failed: diag/{src}")
    if force or _newer(DIAG_LIB, objs):
        tmp = DIAG_LIB + f".tmp{os.getpid()}"
        r = subprocess.run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs], capture_output=True, text=True)
        if r.returncode:
            sys.stdout.write(r.stdout + r.stderr)
            raise RuntimeError("link failed: libspmv_diag.so")
        os.replace(tmp, DIAG_LIB)
    return DIAG_LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv or "-v" in sys.argv)
    print(LIB)

"""Measurement microkernels (``libspmv_diag.so``, ``include/spmv_diag.h``).

Not part of the SpMxV path: bench.py uses them to measure, live in the same
run, the bounds the SpMxV kernels are judged against (the L2 -> SM stream and
random x gathers).  Vectors are CUDA tensors; stream None = torch's current.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspmv_diag.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1203_2739_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        L.spmv_diag_read.argtypes = [vp, i64, i32, vp, vp]
        L.spmv_diag_gather.argtypes = [vp, i64, i64, vp, vp]
        L.spmv_diag_gather_mode.argtypes = [vp, i64, i64, i32, i32, vp, vp]
        L.spmv_diag_micro.argtypes = [i32, i32, vp, i64, i64, vp, vp]
        for f in (L.spmv_diag_read, L.spmv_diag_gather, L.spmv_diag_gather_mode, L.spmv_diag_micro):
            f.restype = i32
        _lib = L
    return _lib


EXPORTED = ["spmv_diag_read", "spmv_diag_gather", "spmv_diag_gather_mode", "spmv_diag_micro"]


def _s(stream):
    import torch
    return (torch.cuda.current_stream() if stream is None else stream).cuda_stream


def _ok(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed (status {rc})")


def read(buf, nbytes: int, out, blocks_per_sm: int = 4, stream=None):
    _ok(lib().spmv_diag_read(buf.data_ptr(), nbytes, blocks_per_sm, out.data_ptr(), _s(stream)), "spmv_diag_read")


def gather_mode(x, count: int, mode: int, out, blocks_per_sm: int = 8, stream=None):
    _ok(lib().spmv_diag_gather_mode(x.data_ptr(), x.numel(), count, mode, blocks_per_sm, out.data_ptr(), _s(stream)),
        "spmv_diag_gather_mode")


def micro(kind: int, param: int, buf, nbytes: int, count: int, out, stream=None):
    _ok(lib().spmv_diag_micro(kind, param, 0 if buf is None else buf.data_ptr(), nbytes, count, out.data_ptr(),
                              _s(stream)), "spmv_diag_micro")

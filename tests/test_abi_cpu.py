"""C-ABI checks that need no GPU (-m "not gpu"): the library loads, exports
every symbol include/spmv.h declares, and rejects bad input on the host-side
validation path (which runs before any CUDA call)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1203_2739_b200 as sp
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_1203_2739_b200 import build
    build.build()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "spmv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spmv_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    names = declared_functions()
    assert {"spmv_create", "spmv_apply", "spmv_split_apply", "spmv_destroy"} <= set(names)
    L = ctypes.CDLL(sp.LIB_PATH)
    for n in names:
        assert hasattr(L, n), n
    assert set(names) <= set(sp.EXPORTED)


def test_status_strings_and_version():
    assert sp.spmv_status_string(0) == "ok"
    assert sp.spmv_status_string(2) == "data error"
    assert sp.spmv_version() >= 100


def test_destroy_null_ok():
    assert sp.lib().spmv_destroy(None) == 0


def _create_status(m, n, rp, col, val, **kw):
    try:
        sp.spmv_create(m, n, rp, col, val, **kw)
    except sp.SpmvError as e:
        return e.status
    return 0


@pytest.mark.parametrize("case,expect", [
    ("dup", sp.SPMV_ERR_DATA),
    ("col_range", sp.SPMV_ERR_DATA),
    ("rowptr", sp.SPMV_ERR_DATA),
    ("rowperm", sp.SPMV_ERR_DATA),
    ("colperm", sp.SPMV_ERR_DATA),
    ("envelope", sp.SPMV_ERR_DATA),
    ("part", sp.SPMV_ERR_DATA),
    ("blocks_cover", sp.SPMV_ERR_DATA),
    ("dist_db", sp.SPMV_ERR_UNSUPPORTED),
])
def test_create_rejects(case, expect):
    rp = np.array([0, 2, 3, 5])
    col = np.array([0, 2, 1, 0, 2], np.int32)
    val = np.arange(1.0, 6.0)
    kw = {}
    if case == "dup":
        col = np.array([0, 0, 1, 0, 2], np.int32)
    elif case == "col_range":
        col = np.array([0, 3, 1, 0, 2], np.int32)
    elif case == "rowptr":
        rp = np.array([0, 3, 2, 5])
    elif case == "rowperm":
        kw["row_perm"] = [0, 0, 1]
    elif case == "colperm":
        kw["col_perm"] = [0, 1, 3]
    elif case == "envelope":
        # SB with K=2: rows {0},{1,2}; C_1={0}, C_2={1}, C_B={2}; row 0 touches col 1 -> outside
        col = np.array([1, 2, 1, 0, 2], np.int32)
        kw["blocks"] = dict(kind=1, K=2, row_block_ptr=[0, 1, 3, 3], col_block_ptr=[0, 1, 2, 3])
    elif case == "part":
        kw["parts"] = [0, 1, 2, 0, 1]
        kw["n_parts"] = 2
    elif case == "blocks_cover":
        kw["blocks"] = dict(kind=1, K=1, row_block_ptr=[0, 2, 2], col_block_ptr=[0, 2, 3])
    elif case == "dist_db":
        kw["blocks"] = dict(kind=2, K=1, row_block_ptr=[0, 2, 3], col_block_ptr=[0, 2, 3])
        kw["dist"] = dict(rank=0, world=2, device=0, nccl_unique_id=bytes(128))
    assert _create_status(3, 3, rp, col, val, **kw) == expect


def test_shard_plan_partitions():
    p = synth.make("c5s", scramble=0)
    L = sp.lib()

    class Shard(ctypes.Structure):
        _fields_ = [(k, ctypes.c_int64) for k in (
            "block_begin", "block_end", "row_begin", "row_end", "x_interior_begin", "x_interior_len",
            "x_border_begin", "x_border_len", "x_local_len", "border_begin", "border_total")]

    b = p.blocks
    rbp = np.ascontiguousarray(b["row_block_ptr"], np.int64)
    cbp = np.ascontiguousarray(b["col_block_ptr"], np.int64)
    blk = sp._Blocks(1, b["K"], rbp.ctypes.data, cbp.ctypes.data, None)
    for world in (1, 2, 4, 8):
        rows, cols = [], []
        for r in range(world):
            s = Shard()
            assert L.spmv_shard_plan(ctypes.byref(blk), ctypes.c_int64(p.m), ctypes.c_int64(p.n), r, world,
                                     ctypes.byref(s)) == 0
            rows.append((s.row_begin, s.row_end))
            if world > 1:
                cols += list(range(s.x_interior_begin, s.x_interior_begin + s.x_interior_len))
                cols += list(range(s.x_border_begin, s.x_border_begin + s.x_border_len))
                assert s.x_local_len == s.x_interior_len + s.x_border_len
                # owner-aligned layout (A17): owned columns == owned rows in count
                assert s.x_local_len == s.row_end - s.row_begin
            else:
                cols = list(range(p.n))
        assert rows[0][0] == 0 and rows[-1][1] == p.m
        assert all(rows[i][1] == rows[i + 1][0] for i in range(world - 1))
        assert sorted(cols) == list(range(p.n))

"""C-ABI checks that need no GPU (-m "not gpu"): the libraries load, export
every symbol include/*.h declares (spmv.h and spmv_test.h: libspmv_b200.so;
spmv_diag.h: libspmv_diag.so), and reject bad input on the host-side
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


def declared_functions(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spmv_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    names = declared_functions("spmv.h")
    assert {"spmv_create", "spmv_apply", "spmv_split_apply", "spmv_destroy"} <= set(names)
    L = ctypes.CDLL(sp.LIB_PATH)
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(sp.EXPORTED)
    test_names = declared_functions("spmv_test.h")
    assert test_names and not set(test_names) & set(names), "test hooks live in spmv_test.h only"
    for n in test_names:
        assert hasattr(L, n), n
    assert set(test_names) == set(sp.EXPORTED_TEST)


def test_diag_library_separate():
    from paper_1203_2739_b200 import diag
    names = declared_functions("spmv_diag.h")
    D = ctypes.CDLL(diag.LIB_PATH)
    L = ctypes.CDLL(sp.LIB_PATH)
    for n in names:
        assert hasattr(D, n), n
        assert not hasattr(L, n), f"{n} must not be in the SpMxV library"
    assert set(names) == set(diag.EXPORTED)


def test_no_environment_switches():
    """The library reads no environment variables: behaviour is set through
    spmv_options_t only (env vars changed create semantics)."""
    csrc = os.path.join(ROOT, "paper_1203_2739_b200", "csrc")
    for f in os.listdir(csrc):
        txt = open(os.path.join(csrc, f)).read()
        assert "getenv" not in txt, f
    assert "environ" not in open(os.path.join(ROOT, "paper_1203_2739_b200", "__init__.py")).read()


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
    ("dist_none", sp.SPMV_ERR_UNSUPPORTED),
    ("options", sp.SPMV_ERR_USAGE),
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
    elif case == "dist_db":     # fewer blocks than ranks
        kw["blocks"] = dict(kind=2, K=1, row_block_ptr=[0, 2, 3], col_block_ptr=[0, 2, 3])
        kw["dist"] = dict(rank=0, world=2, device=0, nccl_unique_id=bytes(128))
    elif case == "dist_none":   # world > 1 needs a block descriptor
        kw["dist"] = dict(rank=0, world=2, device=0, nccl_unique_id=bytes(128))
    elif case == "options":
        kw["options"] = dict(panel_rows=-5)
    assert _create_status(3, 3, rp, col, val, **kw) == expect


def test_shard_plan_partitions():
    p = synth.make("c5s", scramble=0)
    for world in (1, 2, 4, 8):
        rows, cols = [], []
        for r in range(world):
            s = sp.spmv_shard_plan(p.blocks, p.m, p.n, r, world)
            rows.append((s["row_begin"], s["row_end"]))
            if world > 1:
                cols += list(range(s["x_interior_begin"], s["x_interior_begin"] + s["x_interior_len"]))
                cols += list(range(s["x_border_begin"], s["x_border_begin"] + s["x_border_len"]))
                assert s["x_local_len"] == s["x_interior_len"] + s["x_border_len"]
                # owner-aligned layout (A17): owned columns == owned rows in count
                assert s["x_local_len"] == s["row_end"] - s["row_begin"] == s["y_local_len"]
            else:
                cols = list(range(p.n))
        assert rows[0][0] == 0 and rows[-1][1] == p.m
        assert all(rows[i][1] == rows[i + 1][0] for i in range(world - 1))
        assert sorted(cols) == list(range(p.n))


def test_shard_plan_db_rows():
    """DB across GPUs (f1): rank g owns its blocks' rows and a slice of the row
    border R_B; together the ranks own every row exactly once."""
    p = synth.make("c3s")
    K = p.blocks["K"]
    for world in (2, 4):
        owned = []
        for r in range(world):
            s = sp.spmv_shard_plan(p.blocks, p.m, p.n, r, world)
            owned += list(range(s["row_begin"], s["row_end"]))
            owned += list(range(s["y_border_begin"], s["y_border_begin"] + s["y_border_len"]))
            assert s["y_local_len"] == s["row_end"] - s["row_begin"] + s["y_border_len"]
            assert s["y_border_begin"] >= p.blocks["row_block_ptr"][K]
        assert sorted(owned) == list(range(p.m))

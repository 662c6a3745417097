"""GPU parity of the SB default kernel -- column-sorted panels (panel.cu),
y in shared memory, epoch barriers -- against the CPU oracle (oracle/), forced
onto small panels through spmv_options_t: odd block widths, blocks without a
border, empty and dense rows, bit-exact integer data, determinism, the fused
multiple-SpMxV on panels and the row-major fallback."""
import os

import numpy as np
import pytest

import oracle
import paper_1203_2739_b200 as sp
import paper_1203_2739_b200.testing as T
import synth
from gpu_util import assert_parity, create, gpu_apply, oracle_permuted
from gpu_util import panel
from test_plan_cpu import _c5_like, _random_sb

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    sp.lib()


def _run(m, n, rp, col, val, blocks, x, flags=0, rows=700):
    h = sp.spmv_create(m, n, rp, col, val, blocks=blocks, options=panel(rows))
    assert sp.spmv_get_info(h)["kernel"] == 7
    return h, gpu_apply(h, x, m, flags=flags)


@pytest.mark.parametrize("seed", [0, 1])
@pytest.mark.parametrize("variant", ["int", "real"])
def test_random_sb_odd_blocks(seed, variant):
    m, n, rp, col, val, blocks = _random_sb(seed, 4, [37, 600, 1201, 90], [1, 2047, 2049, 5001], 333, 0.01, 0.01)
    rng = np.random.default_rng(seed + 10)
    if variant == "int":
        val = rng.integers(-4, 5, len(val)).astype(np.float64)
        x = rng.integers(-4, 5, n).astype(np.float64)
    else:
        x = rng.uniform(-1, 1, n)
    yref, S = oracle.spmv(rp, col, val, x)
    _, y = _run(m, n, rp, col, val, blocks, x)
    assert_parity(y, yref, S, exact=(variant == "int"), what=f"random_sb/{seed}/{variant}")


def test_no_border_dense_rows():
    m, n, rp, col, val, blocks = _random_sb(5, 3, [40, 1, 300], [3000, 17, 4100], 0, 0.3, 0.0)
    x = np.random.default_rng(3).uniform(-1, 1, n)
    yref, S = oracle.spmv(rp, col, val, x)
    _, y = _run(m, n, rp, col, val, blocks, x)
    assert_parity(y, yref, S, what="no_border")


@pytest.mark.parametrize("name", ["c5s", "c2s"])
@pytest.mark.parametrize("variant", ["int", "dyadic", "real"])
def test_presets(name, variant):
    p = synth.make(name, variant=variant)
    x = p.x()
    xh, yh_ref, S = oracle_permuted(p, x)
    h = create(p, options=panel(700))
    assert sp.spmv_get_info(h)["kernel"] == 7
    yh = gpu_apply(h, xh, p.m)
    assert_parity(yh, yh_ref, S, exact=(variant != "real"), what=f"panel/{name}/{variant}")


@pytest.mark.parametrize("variant", ["int", "real"])
def test_c5_like_default_geometry(variant):
    """The SB default (panel kernel) on a C5-shaped block pair, at the panel size
    the default plan picks for full C5 (16,384 rows; this small matrix would
    otherwise get 1,024-row panels)."""
    p = _c5_like(seed=3)
    if variant == "int":
        rng = np.random.default_rng(1)
        p.val[:] = rng.integers(-4, 5, p.nnz)
    x = synth.vector(p.n, 3, 0, variant)
    yref, S = oracle.spmv(p.row_ptr, p.col, p.val, x, nthreads=oracle.max_threads())
    h = create(p, options=dict(panel_rows=16384))
    info = sp.spmv_get_info(h)
    assert info["kernel"] == 7 and info["pad_slots"] < 0.05 * 32 * info["groups"]
    y = gpu_apply(h, x, p.m)
    assert_parity(y, yref, S, exact=(variant == "int"), what=f"c5_like/{variant}")


@pytest.mark.parametrize("name", ["c5s", "c4s"])
def test_deterministic(name):
    p = synth.make(name)
    h = create(p, options=panel(2000))
    x = torch.from_numpy(oracle.permute_x(p.col_perm, p.x()) if p.col_perm is not None else p.x()).cuda()
    y = torch.empty(p.m, dtype=torch.float64, device="cuda")
    sp.spmv_apply(h, x, y)
    y1 = y.clone()
    for _ in range(3):
        sp.spmv_apply(h, x, y)
    torch.cuda.synchronize()
    assert torch.equal(y, y1), "run-to-run deterministic"


@pytest.mark.parametrize("variant", ["int", "real"])
def test_split_on_panels(variant):
    """Fused multiple-SpMxV on the panel kernel: each (row, part) segment is its
    own virtual row, folded per row.  Forced onto small panels."""
    p = synth.make("c3s", variant=variant)
    x = p.x()
    h = create(p, options=panel(900))
    assert sp.spmv_get_info(h)["split_kernel"] == 7
    y = gpu_apply(h, x, p.m, split=True)
    yref = oracle.split(p.row_ptr, p.col, p.val, p.parts, p.n_parts, x)
    S = oracle.spmv(p.row_ptr, p.col, p.val, x)[1]
    assert_parity(y, yref, S, exact=(variant == "int"), what=f"split-on-panels/{variant}")
    # literal sequence and single SpMxV on the same handle agree with the oracle too
    yl = gpu_apply(h, x, p.m, flags=sp.SPMV_SPLIT_LITERAL, split=True)
    assert_parity(yl, yref, S, exact=(variant == "int"), what="literal")


def test_split_on_panels_random_parts():
    p = synth.make("c4s", variant="int")      # rows up to 3,000 nonzeros: long segments split further
    rng = np.random.default_rng(7)
    parts = rng.integers(0, 5, p.nnz).astype(np.int32)
    x = p.x()
    h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, parts=parts, n_parts=5, options=panel(3000))
    y = gpu_apply(h, x, p.m, split=True)
    yref = oracle.split(p.row_ptr, p.col, p.val, parts, 5, x)
    assert_parity(y, yref, None, exact=True, what="split-on-panels/random parts")


def test_split_rowmajor_kernel():
    """The row-major segment kernel (used when the panel plan is rejected)."""
    p = synth.make("c3s", variant="int")
    x = p.x()
    h = create(p, options=dict(split_kernel="rows"))
    assert sp.spmv_get_info(h)["split_kernel"] == 3
    y = gpu_apply(h, x, p.m, split=True)
    yref = oracle.split(p.row_ptr, p.col, p.val, p.parts, p.n_parts, x)
    assert_parity(y, yref, None, exact=True, what="split row-major")




# ---------------------------------------- debug checks (sanitizer stand-in)
@pytest.mark.parametrize("name,opts,split", [
    ("c5s", dict(kernel="panel", panel_rows=2000), False),
    ("c4s", dict(kernel="panel", panel_rows=2000), False),
    ("c1", dict(kernel="panel", panel_rows=700), False),
    ("c3s", dict(split_kernel="panel", panel_rows=900), True),
    ("_c5like_dbg", dict(kernel="panel", panel_rows=16384), False)])
def test_debug_checks_clean(name, opts, split):
    """compute-sanitizer is closed on this GPU pool, so the panel kernel has a
    checked variant (spmv_options_t.debug_checks): every y slot and x column
    bounds-checked, every y update stamping its slot with the epoch.  On the
    planner's output it must count no violation -- the shared-memory y
    updates of an epoch never race (distinct rows) -- and still match the
    oracle."""
    if name == "_c5like_dbg":
        synth.PRESETS[name] = lambda **kw: synth._sb(2, 40_000, 39_200, 800, 12, 20, 0, 3, **kw)
    p = synth.make(name)
    h = create(p, options=dict(opts, debug_checks=1))
    x = p.x()
    if split:
        y = gpu_apply(h, x, p.m, split=True)
        assert_parity(y, oracle.split(p.row_ptr, p.col, p.val, p.parts, p.n_parts, x),
                      oracle.spmv(p.row_ptr, p.col, p.val, x)[1], what=name)
    else:
        xh, yh, S = oracle_permuted(p, x)
        assert_parity(gpu_apply(h, xh, p.m), yh, S, what=name)
    assert sp.spmv_get_info(h)["debug_violations"] == [0, 0, 0]
    sp.spmv_destroy(h)


@pytest.mark.parametrize("kind,slot", [(1, 2), (2, 0), (3, 1)])
def test_debug_checks_have_teeth(kind, slot):
    """A corrupted plan is caught: a row updated twice in one epoch (a
    shared-memory race), a y slot out of bounds, an x column out of bounds."""
    p = synth.make("c5s", scramble=0)
    h = create(p, options=dict(kernel="panel", panel_rows=2000, debug_checks=1))
    T.corrupt_panel(h, kind)
    gpu_apply(h, oracle_permuted(p, p.x())[0], p.m)
    v = sp.spmv_get_info(h)["debug_violations"]
    assert v[slot] > 0, v
    sp.spmv_destroy(h)


def test_csr_released_on_panel_handles():
    """A panel handle frees its device CSR copy after planning (the kernel
    reads only its group stream; C5: 13.7 GB per GPU); the debug copy is then
    refused, unless created with retain_csr, and the SpMxV is unaffected."""
    p = synth.make("c5s", scramble=0)
    x = p.x()
    xh, yh, S = oracle_permuted(p, x)
    h = create(p, options=panel(2000))
    free0 = torch.cuda.mem_get_info()[0]
    with pytest.raises(sp.SpmvError) as e:
        T.debug_copy_csr(h)
    assert e.value.status == sp.SPMV_ERR_UNSUPPORTED
    assert_parity(gpu_apply(h, xh, p.m), yh, S, what="released CSR")
    h2 = create(p, options=dict(panel(2000), retain_csr=1))
    rp, col, val = T.debug_copy_csr(h2)
    assert len(col) == p.nnz
    assert np.array_equal(gpu_apply(h2, xh, p.m), gpu_apply(h, xh, p.m))
    sp.spmv_destroy(h)
    sp.spmv_destroy(h2)
    assert free0 > 0


@pytest.mark.parametrize("variant", ["int", "real"])
@pytest.mark.parametrize("checks", [0, 1])
def test_far_stream_heavy_runs(variant, checks):
    """Rows whose nonzeros all sit in one 40-column window: most of them are
    still deferred when a small panel's sweep ends and run through the far
    phase (one lane per y slot, register sums, barrier-free); parity with the
    oracle (bit for bit on integer data), and the checked kernel variant sees
    no out-of-bounds slot or column."""
    rng = np.random.default_rng(7)
    m = n = 3000
    rows, cols = [], []
    for r in range(m):
        c0 = (r * 7) % (n - 40)
        cs = np.sort(rng.choice(40, size=30, replace=False)) + c0
        rows += [r] * len(cs)
        cols += cs.tolist()
    rp = np.zeros(m + 1, np.int64)
    np.add.at(rp, np.asarray(rows) + 1, 1)
    rp = np.cumsum(rp)
    col = np.asarray(cols, np.int32)
    if variant == "int":
        val = rng.integers(-4, 5, len(col)).astype(np.float64)
        x = rng.integers(-4, 5, n).astype(np.float64)
    else:
        val = rng.uniform(-1, 1, len(col))
        x = rng.uniform(-1, 1, n)
    st = T.pn_plan_check(m, n, rp, col, val, None, 1024)
    assert st["far"] > len(col) // 20, st
    yref, S = oracle.spmv(rp, col, val, x)
    h = sp.spmv_create(m, n, rp, col, val, options=dict(kernel="panel", panel_rows=1024, debug_checks=checks))
    assert sp.spmv_get_info(h)["kernel"] == 7
    y = gpu_apply(h, x, m)
    assert_parity(y, yref, S, exact=(variant == "int"), what=f"far_runs/{variant}")
    if checks:
        assert sp.spmv_get_info(h)["debug_violations"] == [0, 0, 0]

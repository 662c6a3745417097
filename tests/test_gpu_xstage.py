"""GPU parity of the SB panel kernels against the CPU oracle (oracle/):
  panel  (panel.cu, kernel 7, the SB default): column-sorted panels, y in
         shared memory, epoch barriers;
  xstage (xstage.cu, kernel 6): x chunks streamed through shared memory.
Odd block widths and chunk-straddling blocks, blocks without a border, empty
and dense rows, bit-exact integer data, alignment errors, determinism."""
import os

import numpy as np
import pytest

import oracle
import paper_1203_2739_b200 as sp
import synth
from gpu_util import assert_parity, create, gpu_apply, oracle_permuted
from test_xs_plan_cpu import _c5_like, _random_sb

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

KERNEL_ID = {"xstage": 6, "panel": 7}


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    sp.lib()


@pytest.fixture(params=["panel", "xstage"])
def kernel(request, monkeypatch):
    monkeypatch.setenv("SPMV_KERNEL", request.param)
    monkeypatch.setenv("SPMV_PN_ROWS", "700")
    return request.param


def _run(kernel, m, n, rp, col, val, blocks, x, flags=0):
    h = sp.spmv_create(m, n, rp, col, val, blocks=blocks)
    assert sp.spmv_get_info(h)["kernel"] == KERNEL_ID[kernel]
    return h, gpu_apply(h, x, m, flags=flags)


@pytest.mark.parametrize("seed", [0, 1])
@pytest.mark.parametrize("variant", ["int", "real"])
def test_random_sb_odd_blocks(kernel, seed, variant):
    m, n, rp, col, val, blocks = _random_sb(seed, 4, [37, 600, 1201, 90], [1, 2047, 2049, 5001], 333, 0.01, 0.01)
    rng = np.random.default_rng(seed + 10)
    if variant == "int":
        val = rng.integers(-4, 5, len(val)).astype(np.float64)
        x = rng.integers(-4, 5, n).astype(np.float64)
    else:
        x = rng.uniform(-1, 1, n)
    yref, S = oracle.spmv(rp, col, val, x)
    _, y = _run(kernel, m, n, rp, col, val, blocks, x)
    assert_parity(y, yref, S, exact=(variant == "int"), what=f"{kernel}/random_sb/{seed}/{variant}")


def test_no_border_dense_rows(kernel):
    m, n, rp, col, val, blocks = _random_sb(5, 3, [40, 1, 300], [3000, 17, 4100], 0, 0.3, 0.0)
    x = np.random.default_rng(3).uniform(-1, 1, n)
    yref, S = oracle.spmv(rp, col, val, x)
    _, y = _run(kernel, m, n, rp, col, val, blocks, x)
    assert_parity(y, yref, S, what=f"{kernel}/no_border")


@pytest.mark.parametrize("name", ["c5s", "c2s"])
@pytest.mark.parametrize("variant", ["int", "dyadic", "real"])
def test_presets(kernel, name, variant):
    p = synth.make(name, variant=variant)
    x = p.x()
    xh, yh_ref, S = oracle_permuted(p, x)
    h = create(p)
    assert sp.spmv_get_info(h)["kernel"] == KERNEL_ID[kernel]
    yh = gpu_apply(h, xh, p.m)
    assert_parity(yh, yh_ref, S, exact=(variant != "real"), what=f"{kernel}/{name}/{variant}")


@pytest.mark.parametrize("variant", ["int", "real"])
def test_c5_like_default_geometry(monkeypatch, variant):
    """The SB default (panel kernel) on a C5-shaped block pair, at the panel size
    the default plan picks for full C5 (16,384 rows; this small matrix would
    otherwise get 1,024-row panels)."""
    monkeypatch.delenv("SPMV_KERNEL", raising=False)
    monkeypatch.setenv("SPMV_PN_ROWS", "16384")
    p = _c5_like(seed=3)
    if variant == "int":
        rng = np.random.default_rng(1)
        p.val[:] = rng.integers(-4, 5, p.nnz)
    x = synth.vector(p.n, 3, 0, variant)
    yref, S = oracle.spmv(p.row_ptr, p.col, p.val, x, nthreads=oracle.max_threads())
    h = create(p)
    info = sp.spmv_get_info(h)
    assert info["kernel"] == 7 and info["xs_pad_slots"] < 0.05 * 32 * info["xs_groups"]
    y = gpu_apply(h, x, p.m)
    assert_parity(y, yref, S, exact=(variant == "int"), what=f"c5_like/{variant}")


def test_misaligned_x_and_deterministic(kernel):
    p = synth.make("c5s")
    h = create(p)
    x = torch.from_numpy(oracle.permute_x(p.col_perm, p.x())).cuda()
    y = torch.empty(p.m, dtype=torch.float64, device="cuda")
    if kernel == "xstage":
        buf = torch.zeros(p.n + 1, dtype=torch.float64, device="cuda")
        buf[1:].copy_(x)
        with pytest.raises(sp.SpmvError):
            sp.spmv_apply(h, buf[1:], y)           # 8-byte aligned only: the bulk copy needs 16
    sp.spmv_apply(h, x, y)
    y1 = y.clone()
    for _ in range(3):
        sp.spmv_apply(h, x, y)
    torch.cuda.synchronize()
    assert torch.equal(y, y1), "run-to-run deterministic"


@pytest.mark.parametrize("variant", ["int", "real"])
def test_split_on_panels(monkeypatch, variant):
    """Fused multiple-SpMxV on the panel kernel: each (row, part) segment is its
    own virtual row, folded per row.  Forced onto small panels."""
    monkeypatch.setenv("SPMV_KERNEL", "panel")
    monkeypatch.setenv("SPMV_PN_ROWS", "900")
    p = synth.make("c3s", variant=variant)
    x = p.x()
    h = create(p)
    assert sp.spmv_get_info(h)["split_kernel"] == 7
    y = gpu_apply(h, x, p.m, split=True)
    yref = oracle.split(p.row_ptr, p.col, p.val, p.parts, p.n_parts, x)
    S = oracle.spmv(p.row_ptr, p.col, p.val, x)[1]
    assert_parity(y, yref, S, exact=(variant == "int"), what=f"split-on-panels/{variant}")
    # literal sequence and single SpMxV on the same handle agree with the oracle too
    yl = gpu_apply(h, x, p.m, flags=sp.SPMV_SPLIT_LITERAL, split=True)
    assert_parity(yl, yref, S, exact=(variant == "int"), what="literal")


def test_split_on_panels_random_parts(monkeypatch):
    monkeypatch.setenv("SPMV_KERNEL", "panel")
    monkeypatch.setenv("SPMV_PN_ROWS", "3000")
    p = synth.make("c4s", variant="int")      # rows up to 3,000 nonzeros: long segments split further
    rng = np.random.default_rng(7)
    parts = rng.integers(0, 5, p.nnz).astype(np.int32)
    x = p.x()
    h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, parts=parts, n_parts=5)
    y = gpu_apply(h, x, p.m, split=True)
    yref = oracle.split(p.row_ptr, p.col, p.val, parts, 5, x)
    assert_parity(y, yref, None, exact=True, what="split-on-panels/random parts")


def test_split_rowmajor_kernel(monkeypatch):
    """The row-major segment kernel (used when the panel plan is rejected)."""
    monkeypatch.setenv("SPMV_SPLIT_ROWTILE", "1")
    p = synth.make("c3s", variant="int")
    x = p.x()
    h = create(p)
    assert sp.spmv_get_info(h)["split_kernel"] == 3
    y = gpu_apply(h, x, p.m, split=True)
    yref = oracle.split(p.row_ptr, p.col, p.val, p.parts, p.n_parts, x)
    assert_parity(y, yref, None, exact=True, what="split row-major")


@pytest.mark.parametrize("name", ["c5s", "c2s"])
def test_panel_x_split_path(monkeypatch, name):
    """The kernel's two-buffer x path (world > 1: interior | gathered border)
    on one GPU: SPMV_PN_XS_TEST splits the same x into x_lo = x and
    x_hi = x + C_B start.  Same values through other pointers: y must equal
    the one-buffer path bit for bit (and the oracle)."""
    monkeypatch.setenv("SPMV_KERNEL", "panel")
    monkeypatch.setenv("SPMV_PN_ROWS", "2000")
    p = synth.make(name, variant="real")
    x = p.x()
    xh, yh_ref, S = oracle_permuted(p, x)
    h1 = create(p)
    y1 = gpu_apply(h1, xh, p.m)
    monkeypatch.setenv("SPMV_PN_XS_TEST", "1")
    h2 = create(p)
    assert sp.spmv_get_info(h2)["kernel"] == 7
    y2 = gpu_apply(h2, xh, p.m)
    assert np.array_equal(y1.view(np.int64), y2.view(np.int64))
    assert_parity(y2, yh_ref, S, what=f"x-split path/{name}")


@pytest.mark.parametrize("name", ["c5s", "c4s"])
def test_persistent_panels(monkeypatch, name):
    """SPMV_PN_PERSIST: one CTA per SM walks the panels (measurement switch);
    same plan, same per-row order, so y equals the one-CTA-per-panel launch
    bit for bit."""
    monkeypatch.setenv("SPMV_KERNEL", "panel")
    monkeypatch.setenv("SPMV_PN_ROWS", "700")
    p = synth.make(name, variant="real")
    x = p.x()
    xh, yh_ref, S = oracle_permuted(p, x)
    y1 = gpu_apply(create(p), xh, p.m)
    monkeypatch.setenv("SPMV_PN_PERSIST", "1")
    y2 = gpu_apply(create(p), xh, p.m)
    assert np.array_equal(y1.view(np.int64), y2.view(np.int64))
    assert_parity(y2, yh_ref, S, what=f"persistent/{name}")

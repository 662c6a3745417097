"""The x-staged SB kernel (xstaged.cu, -m gpu): each CTA stages its SB
block's x(C_k) and x(C_B) in shared memory once and gathers from there --
the paper's cache-fit rule (Theorem 1) with one SM's shared
memory as the cache.  Checked against the oracle: integer data bit for bit,
real data within the north_star tolerance; C2 and the scaled configs, odd/uneven blocks, rows longer than a
tile, empty rows, ORIGINAL index space and the power-iteration glue.  (Not
the default kernel: slower than the row tiles on C2.)"""
import numpy as np
import pytest

import oracle
import paper_1203_2739_b200 as sp
import synth
from gpu_util import assert_parity, create, gpu_apply, oracle_permuted
from test_gpu_parity import _teacher_forced
from test_plan_cpu import _random_sb

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

XS = dict(kernel="xstaged")


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    sp.lib()


@pytest.mark.parametrize("name", ["c2s", "c5s", "c2"])
@pytest.mark.parametrize("variant", ["int", "real"])
def test_presets(name, variant):
    p = synth.make(name, variant=variant)
    x = p.x()
    xh, yh, S = oracle_permuted(p, x)
    h = create(p, options=XS)
    assert sp.spmv_get_info(h)["kernel"] == 8
    assert_parity(gpu_apply(h, xh, p.m), yh, S, exact=(variant == "int"), what=f"{name}/{variant}")
    y = gpu_apply(h, x, p.m, flags=sp.SPMV_VEC_ORIGINAL)
    assert_parity(y, oracle.spmv(p.row_ptr, p.col, p.val, x)[0], oracle.spmv(p.row_ptr, p.col, p.val, x)[1],
                  exact=(variant == "int"), what="original space")
    sp.spmv_destroy(h)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_odd_blocks_long_and_empty_rows(seed):
    """Uneven blocks starting at odd columns, a dense row longer than a tile
    (the CTA-per-row path), empty rows, a border-free block."""
    m, n, rp, col, val, blocks = _random_sb(seed, 5, [37, 600, 1201, 90, 3000], [1, 2047, 2049, 5001, 700],
                                            333, 0.01, 0.01)
    # one row of block 3 dense over its interior + border (> 2048 nonzeros)
    r = int(blocks["row_block_ptr"][3]) + 5
    cb = blocks["col_block_ptr"]
    dense = np.concatenate([np.arange(cb[3], cb[4]), np.arange(cb[5], n)]).astype(np.int32)
    rows = [col[rp[i]:rp[i + 1]] for i in range(m)]
    vals = [val[rp[i]:rp[i + 1]] for i in range(m)]
    rows[r] = dense
    vals[r] = np.random.default_rng(seed).integers(-3, 4, len(dense)).astype(np.float64)
    for i in range(0, m, 7):         # empty rows
        if i != r:
            rows[i] = rows[i][:0]
            vals[i] = vals[i][:0]
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum([len(c) for c in rows])
    col = np.concatenate(rows).astype(np.int32)
    val = np.round(np.concatenate(vals) * 4)   # integers: exact sums
    x = np.random.default_rng(seed + 9).integers(-4, 5, n).astype(np.float64)
    h = sp.spmv_create(m, n, rp, col, val, blocks=blocks, options=XS)
    assert sp.spmv_get_info(h)["kernel"] == 8
    y_ref = oracle.spmv(rp, col, val, x)[0]
    assert_parity(gpu_apply(h, x, m), y_ref, None, exact=True, what=f"seed {seed}")
    sp.spmv_destroy(h)


def test_power_iteration():
    """Teacher-forced power steps on the x-staged kernel: the fused max-abs
    of its epilogue exact, x_{t+1} bit for bit."""
    _teacher_forced(synth.make("c5s"), XS, 4, expect_kernel=8)


def test_too_big_is_unsupported():
    """C5-shaped blocks (x(C_k) of 39,200 + 800 entries) do not fit: forcing
    the kernel is UNSUPPORTED, the default takes another kernel."""
    synth.PRESETS["_xs_big"] = lambda **kw: synth._sb(2, 40_000, 39_200, 800, 12, 20, 0, 3, **kw)
    p = synth.make("_xs_big")
    with pytest.raises(sp.SpmvError) as e:
        create(p, options=XS)
    assert e.value.status == sp.SPMV_ERR_UNSUPPORTED
    h = create(p)
    assert sp.spmv_get_info(h)["kernel"] in (0, 7)
    sp.spmv_destroy(h)

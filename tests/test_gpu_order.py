"""f4 on the GPU (-m gpu): spmv_order_sbfs -- the sBFS ordering of P:L134 and
the SB extraction of reading R5 -- bit for bit against oracle.sbfs (the serial
queue BFS), on the worked example, the configs' scrambled inputs and shapes
with empty rows, untouched columns and several components; and the produced
order driven end to end through spmv_create / spmv_apply."""
import json
import os

import numpy as np
import pytest

import oracle
import paper_1203_2739_b200 as sp
import synth
from gpu_util import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    sp.lib()


KEYS = ("row_perm", "col_perm", "row_block_ptr", "col_block_ptr")


def both(m, n, rp, col, K):
    g = sp.spmv_order_sbfs(m, n, rp, col, K)
    o = oracle.sbfs(m, n, rp, col, K)
    for k in KEYS:
        assert np.array_equal(g[k], o[k]), f"{k} differs (m={m} n={n} K={K})"
    assert g["border_cols"] == n - o["col_block_ptr"][K]
    return g


def test_worked_example(golden_dir):
    gd = json.load(open(os.path.join(golden_dir, "sbfs_6x6.json")))
    g = both(gd["m"], gd["n"], np.array(gd["row_ptr"]), np.array(gd["col"]), gd["K"])
    for k in KEYS:
        assert g[k].tolist() == gd[k]


@pytest.mark.parametrize("name,K", [("c1", 4), ("c2s", 4), ("c5s", 8), ("c4s", 16), ("c3s", 3), ("c2s", 1)])
def test_presets(name, K):
    p = synth.make(name)          # the ORIGINAL (scrambled where the preset hides a permutation) CSR
    both(p.m, p.n, p.row_ptr, p.col, K)


def test_irregular_shapes():
    """Empty rows (roots of their own), untouched columns (numbered last),
    several components, a dense row, rectangular both ways."""
    rng = np.random.default_rng(7)
    for m, n, K in [(3000, 1000, 5), (800, 4000, 3), (1, 1, 1), (5, 0, 2), (0, 4, 2)]:
        rows = []
        for i in range(m):
            r = rng.random()
            k = 0 if r < 0.2 else (min(n, 900) if r > 0.999 else int(rng.integers(1, 4)))
            k = min(k, n)
            # three column bands -> several components
            band = (i % 3) * (n // 3)
            hi = max(1, n // 3) if n >= 3 else n
            c = (band + rng.choice(hi, size=min(k, hi), replace=False)) % max(n, 1) if k else np.zeros(0, int)
            rows.append(np.unique(c).astype(np.int32))
        rp = np.zeros(m + 1, np.int64)
        rp[1:] = np.cumsum([len(r) for r in rows]) if m else []
        col = np.concatenate(rows).astype(np.int32) if m else np.zeros(0, np.int32)
        both(m, n, rp, col, K)


def test_full_size_c2():
    p = synth.make("c2")
    g = both(p.m, p.n, p.row_ptr, p.col, 16)
    assert g["components"] >= 1 and g["levels"] > 0


def test_order_drives_spmv():
    """The produced (row_perm, col_perm, SB blocks) is accepted by spmv_create
    (envelope check of Eq.(1)) and the product matches the oracle, in both
    index spaces."""
    p = synth.make("c2s", scramble=1)
    g = sp.spmv_order_sbfs(p.m, p.n, p.row_ptr, p.col, 4)
    h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=g["row_perm"], col_perm=g["col_perm"],
                       blocks=g["blocks"])
    x = p.x()
    y_ref, S = oracle.spmv(p.row_ptr, p.col, p.val, x)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty(p.m, dtype=torch.float64, device="cuda")
    sp.spmv_apply(h, xd, yd, sp.SPMV_VEC_ORIGINAL)
    torch.cuda.synchronize()
    assert_parity(yd.cpu().numpy(), y_ref, S, what="sBFS-ordered SpMxV")
    sp.spmv_destroy(h)


def test_bad_input():
    rp = np.array([0, 2, 3], np.int64)
    with pytest.raises(sp.SpmvError) as e:
        sp.spmv_order_sbfs(2, 3, rp, np.array([0, 5, 1], np.int32), 2)
    assert e.value.status == sp.SPMV_ERR_DATA
    with pytest.raises(sp.SpmvError) as e:
        sp.spmv_order_sbfs(2, 3, rp, np.array([0, 1, 1], np.int32), 0)
    assert e.value.status == sp.SPMV_ERR_USAGE

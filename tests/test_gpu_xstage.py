"""GPU parity of the x-staged SB kernel (xstage.cu, the default for SB
handles): odd block widths and chunk-straddling blocks, blocks without a
border, empty rows, dense rows, bit-exact integer data, alignment errors,
and run-to-run determinism.  Oracle: the CPU reference (oracle/)."""
import numpy as np
import pytest

import oracle
import paper_1203_2739_b200 as sp
import synth
from gpu_util import assert_parity, create, gpu_apply, oracle_permuted
from test_xs_plan_cpu import _random_sb

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    sp.lib()


def _run(m, n, rp, col, val, blocks, x, flags=0):
    h = sp.spmv_create(m, n, rp, col, val, blocks=blocks)
    info = sp.spmv_get_info(h)
    assert info["kernel"] == 6, "SB handles use the x-staged kernel"
    y = gpu_apply(h, x, m, flags=flags)
    return h, y


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


def test_no_border_dense_and_empty_rows():
    m, n, rp, col, val, blocks = _random_sb(5, 3, [40, 1, 300], [3000, 17, 4100], 0, 0.3, 0.0)
    # make some rows empty
    x = np.random.default_rng(3).uniform(-1, 1, n)
    yref, S = oracle.spmv(rp, col, val, x)
    _, y = _run(m, n, rp, col, val, blocks, x)
    assert_parity(y, yref, S, what="no_border")


@pytest.mark.parametrize("name", ["c5s", "c2s"])
@pytest.mark.parametrize("variant", ["int", "dyadic"])
def test_presets_bit_exact(name, variant):
    p = synth.make(name, variant=variant)
    x = p.x()
    xh, yh_ref, _ = oracle_permuted(p, x)
    h = create(p)
    assert sp.spmv_get_info(h)["kernel"] == 6
    yh = gpu_apply(h, xh, p.m)
    assert_parity(yh, yh_ref, None, exact=True, what=f"{name}/{variant}")


def test_misaligned_x_rejected_and_deterministic():
    p = synth.make("c5s")
    h = create(p)
    x = torch.from_numpy(oracle.permute_x(p.col_perm, p.x())).cuda()
    buf = torch.zeros(p.n + 1, dtype=torch.float64, device="cuda")
    buf[1:].copy_(x)
    y = torch.empty(p.m, dtype=torch.float64, device="cuda")
    with pytest.raises(sp.SpmvError):
        sp.spmv_apply(h, buf[1:], y)           # 8-byte aligned only
    sp.spmv_apply(h, x, y)
    y1 = y.clone()
    for _ in range(3):
        sp.spmv_apply(h, x, y)
    torch.cuda.synchronize()
    assert torch.equal(y, y1), "x-staged kernel must be run-to-run deterministic"

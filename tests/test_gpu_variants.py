"""GPU parity of the single-SpMxV kernels selectable with SPMV_KERNEL against
the CPU oracle: the panel kernel forced onto small matrices (panel.cu; c4s
has rows of up to 3,000 nonzeros -> virtual rows and warp folds), the
row-tile family (rowtile.cu: quad and lane-consecutive streaming,
128/256/512-thread CTAs), rowseg, pipe and the first tile kernel.  Integer data: bit-exact; real data:
the north_star tolerance."""
import pytest

import paper_1203_2739_b200 as sp
import synth
from gpu_util import assert_parity, create, gpu_apply, oracle_permuted

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

VARIANTS = {"rowtile": 0, "pipe": 1, "tile": 2, "rowtile512": 3, "rowseg": 4, "rowtile128": 5, "rowlin": 8,
            "panel": 7}


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    sp.lib()


@pytest.mark.parametrize("kernel", sorted(VARIANTS))
@pytest.mark.parametrize("name,variant", [("c4s", "int"), ("c5s", "int"), ("c4s", "real"), ("c1", "dyadic")])
def test_variant_parity(monkeypatch, kernel, name, variant):
    monkeypatch.setenv("SPMV_KERNEL", kernel)
    monkeypatch.setenv("SPMV_PN_ROWS", "2000")   # panel: several panels, c4s's long rows become virtual rows
    p = synth.make(name, variant=variant)
    x = p.x()
    xh, yh_ref, S = oracle_permuted(p, x)
    h = create(p, with_parts=False)
    assert sp.spmv_get_info(h)["kernel"] == VARIANTS[kernel]
    yh = gpu_apply(h, xh, p.m)
    assert_parity(yh, yh_ref, S, exact=(variant != "real"), what=f"{kernel}/{name}/{variant}")

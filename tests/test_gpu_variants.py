"""GPU parity of the two single-SpMxV kernels, each forced through
spmv_options_t, against the CPU oracle: the column-sorted panel kernel
(panel.cu; c4s has rows of up to 3,000 nonzeros -> virtual rows and warp
folds) and the row-tile kernel (rowtile.cu).  Integer / dyadic data:
bit-exact; real data: the north_star tolerance."""
import pytest

import paper_1203_2739_b200 as sp
import synth
from gpu_util import assert_parity, create, gpu_apply, oracle_permuted

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

VARIANTS = {"rowtile": (dict(kernel="rowtile"), 0), "panel": (dict(kernel="panel", panel_rows=2000), 7)}


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    sp.lib()


@pytest.mark.parametrize("kernel", sorted(VARIANTS))
@pytest.mark.parametrize("name,variant", [("c4s", "int"), ("c5s", "int"), ("c4s", "real"), ("c1", "dyadic"),
                                          ("c2s", "real"), ("c3s", "int")])
def test_variant_parity(kernel, name, variant):
    opts, kid = VARIANTS[kernel]
    p = synth.make(name, variant=variant)
    x = p.x()
    xh, yh_ref, S = oracle_permuted(p, x)
    h = create(p, with_parts=False, options=opts)
    assert sp.spmv_get_info(h)["kernel"] == kid
    yh = gpu_apply(h, xh, p.m)
    assert_parity(yh, yh_ref, S, exact=(variant != "real"), what=f"{kernel}/{name}/{variant}")

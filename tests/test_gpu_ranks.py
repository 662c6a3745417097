"""The multi-GPU SB path on one GPU (-m gpu): every rank of world 2 / 4 is
created as a real shard -- its rows, local CSR, x layout [interior | C_B],
panel plan from the global per-block counts, the kernel's two-buffer x path
-- without a communicator (SPMV_TEST_RANKS_NO_NCCL; spmv_test_set_border
supplies the x(C_B) the NCCL all-gather would deliver).  Each rank's y must
equal its rows of the single-GPU y bit for bit (y does not
depend on the GPU count) and match the oracle.  Only the collective itself
is not exercised here (one GPU per call)."""
import numpy as np
import pytest

import paper_1203_2739_b200 as sp
import synth
from gpu_util import assert_parity, create, gpu_apply, oracle_permuted

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name,kernel", [("c5s", "panel"), ("c5s", "default"), ("c2s", "default")])
def test_ranks_match_single_gpu(monkeypatch, name, kernel, world):
    if kernel == "panel":
        monkeypatch.setenv("SPMV_KERNEL", "panel")
    p = synth.make(name)
    x = p.x()
    xh, yh_ref, S = oracle_permuted(p, x)
    h1 = create(p)
    y1 = gpu_apply(h1, xh, p.m)
    k1 = sp.spmv_get_info(h1)["kernel"]
    monkeypatch.setenv("SPMV_TEST_RANKS_NO_NCCL", "1")
    K = p.blocks["K"]
    cb0 = int(p.blocks["col_block_ptr"][K])
    rows = 0
    for r in range(world):
        h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm,
                           blocks=p.blocks, dist=dict(rank=r, world=world, device=0, nccl_unique_id=None))
        info = sp.spmv_get_info(h)
        assert info["world"] == world and info["kernel"] == k1
        a, L = info["x_interior_begin"], info["x_interior_len"]
        b, Lb = info["x_border_begin"], info["x_border_len"]
        xl = np.concatenate([xh[a:a + L], xh[b:b + Lb]])
        sp.spmv_test_set_border(h, torch.from_numpy(np.ascontiguousarray(xh[cb0:cb0 + info["border_total"]])).cuda())
        yl = gpu_apply(h, xl, info["m_local"])
        r0, ml = info["row_begin"], info["m_local"]
        assert np.array_equal(yl.view(np.int64), y1[r0:r0 + ml].view(np.int64)), f"rank {r} of {world}"
        assert_parity(yl, yh_ref[r0:r0 + ml], S[r0:r0 + ml], what=f"{name} rank {r}/{world}")
        rows += ml
        sp.spmv_destroy(h)
    assert rows == p.m

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


@pytest.mark.parametrize("world", [2, 4])
def test_ranks_power_step(monkeypatch, world):
    """a9 at world > 1 on emulated ranks: each rank's fused local max (the
    max all-reduce done on the host here) and its owner-local x-update
    x^_{t+1}[c] = y^_t[r(c)] / m reproduce the single-GPU step bit for bit
    on the rank's x layout [interior | owned border slice], two steps."""
    p = synth.make("c5s")
    x = p.x()
    xh, _, _ = oracle_permuted(p, x)
    h1 = create(p)
    dev = "cuda"
    monkeypatch.setenv("SPMV_TEST_RANKS_NO_NCCL", "1")
    K = p.blocks["K"]
    cb0 = int(p.blocks["col_block_ptr"][K])
    hs = [sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm,
                         blocks=p.blocks, dist=dict(rank=r, world=world, device=0, nccl_unique_id=None))
          for r in range(world)]
    infos = [sp.spmv_get_info(h) for h in hs]
    xg = torch.from_numpy(xh).to(dev)
    xl = [torch.from_numpy(np.concatenate([xh[i["x_interior_begin"]:i["x_interior_begin"] + i["x_interior_len"]],
                                           xh[i["x_border_begin"]:i["x_border_begin"] + i["x_border_len"]]])).to(dev)
          for i in infos]
    for t in range(2):
        # single GPU step
        y1 = torch.empty(p.m, dtype=torch.float64, device=dev)
        m1 = torch.empty(1, dtype=torch.float64, device=dev)
        sp.spmv_apply(h1, xg, y1, sp.SPMV_FUSE_MAXABS)
        sp.spmv_maxabs(h1, m1)
        xg_next = torch.empty_like(xg)
        sp.spmv_normalize(h1, y1, m1, xg_next)
        # ranks: SpMxV with the fused local max, host all-reduce(MAX), x-update
        border = xg[cb0:cb0 + infos[0]["border_total"]].contiguous()
        ys, ms = [], []
        for h, i, xr in zip(hs, infos, xl):
            sp.spmv_test_set_border(h, border)
            yr = torch.empty(i["m_local"], dtype=torch.float64, device=dev)
            mr = torch.empty(1, dtype=torch.float64, device=dev)
            sp.spmv_apply(h, xr, yr, sp.SPMV_FUSE_MAXABS)
            sp.spmv_maxabs(h, mr)   # no communicator: this rank's max
            ys.append(yr)
            ms.append(mr)
        mg = torch.max(torch.cat(ms)).reshape(1)
        assert mg.item() == m1.item(), f"step {t}: max over ranks"
        for h, i, yr, r in zip(hs, infos, ys, range(world)):
            r0 = i["row_begin"]
            assert torch.equal(yr, y1[r0:r0 + i["m_local"]]), f"step {t} rank {r}: y"
            xn = torch.empty_like(xl[r])
            sp.spmv_normalize(h, yr, mg, xn)
            a, L = i["x_interior_begin"], i["x_interior_len"]
            b, Lb = i["x_border_begin"], i["x_border_len"]
            ref = torch.cat([xg_next[a:a + L], xg_next[b:b + Lb]])
            assert torch.equal(xn.view(torch.int64), ref.view(torch.int64)), f"step {t} rank {r}: x-update"
            xl[r] = xn
        torch.cuda.synchronize()
        xg = xg_next

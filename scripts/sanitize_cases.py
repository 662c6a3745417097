"""Small cases through every kernel of the apply path, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run): the panel kernel forced
on c5s (SB border groups), c4s (virtual rows, warp folds) and C1; the row-tile
kernel with 16- and 32-bit column ids; the fused split on panels, the
row-major split and the literal K-pass split on c3s; ORIGINAL-mode gathers;
the power-iteration glue; the sBFS ordering (f4).  Each result is checked
against the oracle, so a run that completes also shows parity."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import oracle
import paper_1203_2739_b200 as sp
import synth
from gpu_util import assert_parity, create, gpu_apply, oracle_permuted

small = "--small" in sys.argv
done = []
for name, opts in [("c5s", dict(kernel="panel", panel_rows=2000)), ("c4s", dict(kernel="panel", panel_rows=2000)),
                   ("c1", dict(kernel="panel", panel_rows=700)), ("c1", dict(kernel="rowtile")),
                   ("c2s", dict(kernel="rowtile", index16=1)), ("c2s", dict(kernel="rowtile"))]:
    if small and name == "c4s":
        continue
    p = synth.make(name)
    x = p.x()
    xh, yh, S = oracle_permuted(p, x)
    h = create(p, options=opts)
    xd = torch.from_numpy(xh).cuda()
    yd = torch.empty(p.m, dtype=torch.float64, device="cuda")
    sp.spmv_apply(h, xd, yd, sp.SPMV_FUSE_MAXABS)
    if p.m == p.n and sp.spmv_get_info(h)["has_owner_map"]:
        md = torch.empty(1, dtype=torch.float64, device="cuda")
        sp.spmv_maxabs(h, md)
        xn = torch.empty_like(xd)
        sp.spmv_normalize(h, yd, md, xn)
    torch.cuda.synchronize()
    assert_parity(yd.cpu().numpy(), yh, S, what=f"{name} {opts}")
    if p.row_perm is not None:
        yo = gpu_apply(h, x, p.m, flags=sp.SPMV_VEC_ORIGINAL)
        assert_parity(yo, oracle.spmv(p.row_ptr, p.col, p.val, x)[0], oracle.spmv(p.row_ptr, p.col, p.val, x)[1])
    sp.spmv_destroy(h)
    done.append(f"{name}:{opts}")
q = synth.make("c3s")
xq = q.x()
yq_ref = oracle.split(q.row_ptr, q.col, q.val, q.parts, q.n_parts, xq)
Sq = oracle.spmv(q.row_ptr, q.col, q.val, xq)[1]
for opts, flags in [(dict(split_kernel="panel", panel_rows=900), 0), (dict(split_kernel="rows"), 0),
                    (None, sp.SPMV_SPLIT_LITERAL)]:
    h = create(q, options=opts)
    y = gpu_apply(h, xq, q.m, split=True, flags=flags)
    assert_parity(y, yq_ref, Sq, what=f"split {opts} {flags}")
    sp.spmv_destroy(h)
    done.append(f"c3s split:{opts}:{flags}")
r = synth.make("c2s")
g = sp.spmv_order_sbfs(r.m, r.n, r.row_ptr, r.col, 4)
o = oracle.sbfs(r.m, r.n, r.row_ptr, r.col, 4)
assert np.array_equal(g["row_perm"], o["row_perm"]) and np.array_equal(g["col_perm"], o["col_perm"])
done.append("sbfs c2s")
print("sanitize cases ok:", "; ".join(done))

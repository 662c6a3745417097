"""Panel vs row-tile on C5 geometry (K blocks) with x made L2-resident right
before each timed apply (x.sum() touches all of x): do x misses explain the
panel kernel's gap?"""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_2739_b200 as sp, synth
K = int(os.environ.get("K", "4"))
synth.PRESETS["c5q"] = lambda **kw: synth._sb(K, 1_000_000, 980_000, 20_000, 12, 20, 0, 3, **kw)
p = synth.make("c5q")
out = {}
for kern in os.environ.get("KERNELS", "panel,rowtile").split(","):
    os.environ["SPMV_KERNEL"] = kern
    h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm, blocks=p.blocks)
    info = sp.spmv_get_info(h)
    x = torch.rand(info["n"], dtype=torch.float64, device="cuda")
    y = torch.empty(info["m"], dtype=torch.float64, device="cuda")
    for warm in (False, True):
        ts = []
        for it in range(13):
            if warm:
                s = x.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); sp.spmv_apply(h, x, y); b.record(); torch.cuda.synchronize()
            if it >= 3:
                ts.append(a.elapsed_time(b))
        ts.sort()
        out[f"{kern}_{'xwarm' if warm else 'plain'}_ms"] = ts[len(ts) // 2]
    sp.spmv_destroy(h)
print(json.dumps(out))

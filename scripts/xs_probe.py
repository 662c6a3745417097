"""x-staged kernel probe on a C5-geometry matrix with fewer blocks (K blocks of
1M rows, 980K interior + 20K border columns each): times xstage vs rowtile."""
import json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_2739_b200 as sp, synth
from roofline import timeit
K = int(os.environ.get("K", "4"))
synth.PRESETS["c5q"] = lambda **kw: synth._sb(K, 1_000_000, 980_000, 20_000, 12, 20, 0, 3, **kw)
p = synth.make("c5q")
out = {"nnz": p.nnz}
x = None
for kern in (os.environ.get("KERNELS", "xstage,rowtile").split(",")):
    os.environ["SPMV_KERNEL"] = kern
    t0 = time.time()
    h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm, blocks=p.blocks)
    info = sp.spmv_get_info(h)
    out[f"{kern}_create_s"] = time.time() - t0
    out[f"{kern}_info"] = {k: info[k] for k in ("kernel", "xs_panels", "xs_groups", "xs_pad_slots", "bytes_alg", "bytes_stream")}
    if x is None:
        x = torch.rand(info["n"], dtype=torch.float64, device="cuda")
        y = torch.empty(info["m"], dtype=torch.float64, device="cuda")
    ms = timeit(lambda: sp.spmv_apply(h, x, y), reps=10)
    out[f"{kern}_ms"] = ms
    out[f"{kern}_GBs_alg"] = info["bytes_alg"] / ms / 1e6
    if os.environ.get("PROFILE_ONE"):
        torch.cuda.synchronize()
        sp.spmv_apply(h, x, y)
        torch.cuda.synchronize()
    sp.spmv_destroy(h)
print(json.dumps(out, indent=1))

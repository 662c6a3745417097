"""C5 gather diagnosis: stream+gather variants over the real C5 CSR."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_2739_b200 as sp, synth
from roofline import timeit
w = sys.argv[1] if len(sys.argv) > 1 else "c5"
p = synth.make(w)
h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm, blocks=p.blocks)
nnz = p.nnz
del p
info = sp.spmv_get_info(h)
x = torch.rand(info["n"], dtype=torch.float64, device="cuda")
y = torch.empty(info["m"], dtype=torch.float64, device="cuda")
sink = torch.zeros(1, dtype=torch.float64, device="cuda")
out = {}
for mode in range(4):
    ms = timeit(lambda: sp.spmv_diag_csr(h, x, mode, sink), reps=5)
    out[f"mode{mode}_ms"] = ms
    out[f"mode{mode}_Gnnz_s"] = nnz / ms / 1e6
out["spmv_ms"] = timeit(lambda: sp.spmv_apply(h, x, y), reps=5)
if os.environ.get("AB"):
    q = synth.make(w)
    for k in ("rowtile512", "rowtile128"):
        os.environ["SPMV_KERNEL"] = k
        h2 = sp.spmv_create(q.m, q.n, q.row_ptr, q.col, q.val, row_perm=q.row_perm, col_perm=q.col_perm, blocks=q.blocks)
        out[f"spmv_{k}_ms"] = timeit(lambda: sp.spmv_apply(h2, x, y), reps=5)
        sp.spmv_destroy(h2)
    del os.environ["SPMV_KERNEL"]
print(json.dumps(out, indent=1))
if os.environ.get("PROFILE_ONE"):
    torch.cuda.synchronize()
    for mode in (1, 3):
        sp.spmv_diag_csr(h, x, mode, sink)
    sp.spmv_apply(h, x, y)
    torch.cuda.synchronize()

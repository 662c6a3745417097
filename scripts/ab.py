"""A/B of SPMV_KERNEL variants on one workload: python ab.py c4 rowtile,rowlin"""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_2739_b200 as sp, synth
from roofline import timeit
w, kernels = sys.argv[1], sys.argv[2].split(",")
p = synth.make(w)
out = {"workload": w, "nnz": p.nnz}
for k in kernels:
    os.environ["SPMV_KERNEL"] = k
    h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm, blocks=p.blocks)
    info = sp.spmv_get_info(h)
    x = torch.rand(info["n"], dtype=torch.float64, device="cuda")
    y = torch.empty(info["m"], dtype=torch.float64, device="cuda")
    ms = timeit(lambda: sp.spmv_apply(h, x, y), reps=20)
    out[k] = {"ms": ms, "GBs": info["bytes_alg"] / ms / 1e6, "kernel": info["kernel"]}
    sp.spmv_destroy(h)
print(json.dumps(out))

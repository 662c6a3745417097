"""C3: fused multiple-SpMxV vs single-SpMxV vs the literal K-pass sequence on the
same matrix (the GPU analog of the paper's mHP_RCN vs sHP_eRCN comparison)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_2739_b200 as sp, synth
from timing import timeit
p = synth.make("c3")
h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, blocks=p.blocks, parts=p.parts, n_parts=p.n_parts)
info = sp.spmv_get_info(h)
x = torch.rand(info["n"], dtype=torch.float64, device="cuda")
y = torch.empty(info["m"], dtype=torch.float64, device="cuda")
flush = torch.empty(512 << 17, dtype=torch.float64, device="cuda")
out = {"nnz": p.nnz, "bytes_alg": info["bytes_alg"], "bytes_alg_split": info["bytes_alg_split"]}
for name, fn in [("single", lambda: sp.spmv_apply(h, x, y)),
                 ("split_fused", lambda: sp.spmv_split_apply(h, x, y)),
                 ("split_literal", lambda: sp.spmv_split_apply(h, x, y, sp.SPMV_SPLIT_LITERAL))]:
    out[name + "_warm_ms"] = timeit(fn, reps=20)
    def cold():
        flush.fill_(1.0)
        fn()
    t_all = timeit(cold, reps=10)
    t_flush = timeit(lambda: flush.fill_(1.0), reps=10)
    out[name + "_cold_ms"] = t_all - t_flush
print(json.dumps(out, indent=1))

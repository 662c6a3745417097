"""Interleaved timing of kernel choices on one workload (spmv_options_t.kernel),
L2 flushed before each call (cold) and back to back (warm).
    python scripts/ab_kernels.py c2 rowtile xstaged panel"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1203_2739_b200 as sp
import synth

name, kernels = sys.argv[1], sys.argv[2:]
p = synth.make(name)
hs = {}
for k in kernels:
    try:
        hs[k] = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm,
                               blocks=p.blocks, options=dict(kernel=k))
    except sp.SpmvError as e:
        print(k, "unsupported:", e)
x = torch.rand(p.n, dtype=torch.float64, device="cuda")
y = torch.empty(p.m, dtype=torch.float64, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
res = {k: {"cold": [], "warm": []} for k in hs}
for rnd in range(5):
    for k, h in hs.items():
        for mode in ("cold", "warm"):
            evs = []
            for _ in range(10):
                if mode == "cold":
                    flush.fill_(1.0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                sp.spmv_apply(h, x, y)
                b.record()
                evs.append((a, b))
            torch.cuda.synchronize()
            res[k][mode] += [a.elapsed_time(b) for a, b in evs]
for k in hs:
    i = sp.spmv_get_info(hs[k])
    print(f"{name} {k:8s} kernel {i['kernel']}: cold {statistics.median(res[k]['cold']) * 1e3:.1f} us, "
          f"warm {statistics.median(res[k]['warm']) * 1e3:.1f} us")

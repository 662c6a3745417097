"""Gather-flavour microbenchmark (see diag.cu modes): which path serves random
8-byte x gathers fastest on B200."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_2739_b200 as sp
from roofline import timeit

out = {}
sink = torch.zeros(1, dtype=torch.float64, device="cuda")
names = ["ldg_nc", "ld_ca", "ld_cg", "nc_noalloc", "pairs16B", "v2_16B", "8lanes_line", "bulk16B", "smem96KB"]
for mb in (8, 32):
    x = torch.rand(mb * (1 << 20) // 8, dtype=torch.float64, device="cuda")
    for mode, name in enumerate(names):
        for bps in (4, 8):
            cnt = 1 << 29
            try:
                ms = timeit(lambda: sp.spmv_diag_gather_mode(x, cnt, mode, sink, bps), reps=5, warm=2)
                out[f"{mb}MB_{name}_bps{bps}_Gps"] = round(cnt / ms / 1e6, 1)
            except Exception as e:
                out[f"{mb}MB_{name}_bps{bps}_Gps"] = str(e)[:80]
print(json.dumps(out, indent=1))

"""Interleaved timing of spmv_options_t variants on one workload:
    python scripts/ab_opts.py c4 '{"panel_rows": 8192}' '{}' ...
Each variant's SpMxV is timed 20 times back to back per round, 3 rounds."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1203_2739_b200 as sp
import synth

name, variants = sys.argv[1], [json.loads(a) for a in sys.argv[2:]]
p = synth.make(name)
hs = []
for v in variants:
    h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm,
                       blocks=p.blocks, options=v or None)
    hs.append(h)
x = torch.rand(p.n, dtype=torch.float64, device="cuda")
y = torch.empty(p.m, dtype=torch.float64, device="cuda")
res = [[] for _ in hs]
for rnd in range(3):
    for k, h in enumerate(hs):
        for _ in range(3):
            sp.spmv_apply(h, x, y)
        evs = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            sp.spmv_apply(h, x, y)
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        res[k] += [a.elapsed_time(b) for a, b in evs]
for v, h, r in zip(variants, hs, res):
    i = sp.spmv_get_info(h)
    print(f"{name} {json.dumps(v):32s} kernel {i['kernel']} panels {i['panels']:5d}: {statistics.median(r):.4f} ms")

"""Sustained (power-capped) interleaved timing of spmv_options_t variants:
    python scripts/ab_opts_sustained.py c5 '{}' '{"panel_rows": 20480}' ...
Each variant runs 150 SpMxVs back to back per round (the first 50 untimed, so
the power cap has set the clock), 3 interleaved rounds; prints the median
SpMxV time and the SM clock sampled at the end of each timed block."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1203_2739_b200 as sp
import synth


def sm_clock():
    try:
        o = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-i", "0"],
                           capture_output=True, text=True, timeout=10).stdout.strip()
        return o
    except Exception:
        return "?"


name, variants = sys.argv[1], [json.loads(a) for a in sys.argv[2:]]
p = synth.make(name)
hs = [sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm,
                     blocks=p.blocks, options=v or None) for v in variants]
x = torch.rand(p.n, dtype=torch.float64, device="cuda")
y = torch.empty(p.m, dtype=torch.float64, device="cuda")
res = [[] for _ in hs]
clk = [[] for _ in hs]
for rnd in range(3):
    for k, h in enumerate(hs):
        for _ in range(50):
            sp.spmv_apply(h, x, y)
        evs = []
        for _ in range(100):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            sp.spmv_apply(h, x, y)
            b.record()
            evs.append((a, b))
        clk[k].append(sm_clock())
        torch.cuda.synchronize()
        res[k].append(statistics.median(a.elapsed_time(b) for a, b in evs))
for v, h, r, c in zip(variants, hs, res, clk):
    i = sp.spmv_get_info(h)
    print(f"{name} {json.dumps(v):28s} panels {i['panels']:5d}: rounds {[round(t, 4) for t in r]} ms, clocks/power {c}", flush=True)

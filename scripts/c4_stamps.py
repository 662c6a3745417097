"""Per-CTA timeline of the panel kernel (spmv_test_panel_stamps) on one workload:
phase split (prologue / epochs / epilogue), per-panel durations vs groups, wave
structure and the tail.    python scripts/c4_stamps.py c4 [options-json]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1203_2739_b200 as sp
import synth
from paper_1203_2739_b200 import testing as T

name = sys.argv[1]
opts = json.loads(sys.argv[2]) if len(sys.argv) > 2 else None
p = synth.make(name)
h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm, blocks=p.blocks,
                   options=opts)
x = torch.rand(p.n, dtype=torch.float64, device="cuda")
y = torch.empty(p.m, dtype=torch.float64, device="cuda")
for _ in range(5):
    sp.spmv_apply(h, x, y)
T.panel_stamps_arm(h)
for _ in range(3):
    sp.spmv_apply(h, x, y)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
sp.spmv_apply(h, x, y)
b.record()
torch.cuda.synchronize()
S = T.panel_stamps_read(h).astype(np.int64)
ms = a.elapsed_time(b)
sm, g0, g1, c0, c1, c2, c3, ce = S[:, 0], S[:, 1], S[:, 2], S[:, 3], S[:, 4], S[:, 5], S[:, 6], S[:, 7]
t0 = g0.min()
dur = (g1 - g0) / 1e3
pro, loop, epi = (c1 - c0), (c2 - c1), (c3 - c2)
tot = c3 - c0
print(f"{name} {opts}: event {ms * 1e3:.1f} us, panels {len(S)}, span {(g1.max() - t0) / 1e3:.1f} us")
print(f"  CTA us: mean {dur.mean():.1f} min {dur.min():.1f} max {dur.max():.1f}")
print(f"  far phase (+ first slot loads) share {(c2 - ce).sum() / tot.sum():.3f}")
print(f"  phase share of CTA clocks: prologue {pro.sum() / tot.sum():.3f} epochs {loop.sum() / tot.sum():.3f} "
      f"epilogue {epi.sum() / tot.sum():.3f}; mean clocks pro {pro.mean():.0f} loop {loop.mean():.0f} epi {epi.mean():.0f}")
# per SM: busy time vs span
busy = np.zeros(sm.max() + 1)
last = np.zeros(sm.max() + 1)
first = np.full(sm.max() + 1, np.inf)
for i in range(len(S)):
    busy[sm[i]] += (g1[i] - g0[i]) / 1e3
    last[sm[i]] = max(last[sm[i]], (g1[i] - t0) / 1e3)
    first[sm[i]] = min(first[sm[i]], (g0[i] - t0) / 1e3)
used = busy > 0
print(f"  SMs used {used.sum()}, busy us mean {busy[used].mean():.1f} min {busy[used].min():.1f} max {busy[used].max():.1f}; "
      f"last end min {last[used].min():.1f} max {last[used].max():.1f}; first start max {first[used].max():.1f}")
# start-time histogram (waves)
st = (g0 - t0) / 1e3
print("  CTA starts (us) quantiles:", np.round(np.quantile(st, [0, .1, .25, .33, .5, .66, .75, .9, 1]), 1).tolist())
print("  CTA durations (us) quantiles:", np.round(np.quantile(dur, [0, .1, .25, .5, .75, .9, 1]), 1).tolist())
info = sp.spmv_get_info(h)
print(f"  groups {info['groups']}, deferred {info['deferred']}, pad {info['pad_slots']}")

"""Cost split of C4's SpMxV: the full matrix against its band part (|c - r| <= 2000,
70 % of the nonzeros) and its far part (uniform columns, 30 %), each on the panel
and the row-tile kernel, interleaved, back to back (inputs > L2).
    python scripts/c4_parts.py [c4]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1203_2739_b200 as sp
import synth

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
p = synth.make(name)
rp = np.asarray(p.row_ptr, dtype=np.int64)
col = np.asarray(p.col, dtype=np.int32)
val = np.asarray(p.val, dtype=np.float64)
rows = np.repeat(np.arange(p.m, dtype=np.int64), np.diff(rp))
band = np.abs(col.astype(np.int64) - rows) <= 2000
print(f"{name}: nnz {len(col)}, band {band.mean():.3f}")


def sub(mask):
    cnt = np.bincount(rows[mask], minlength=p.m)
    r2 = np.zeros(p.m + 1, dtype=np.int64)
    np.cumsum(cnt, out=r2[1:])
    return r2, col[mask], val[mask]


mats = {"full": (rp, col, val), "band": sub(band), "far": sub(~band)}
hs = {}
for mn, (r, c, v) in mats.items():
    for k in ("panel", "rowtile"):
        hs[(mn, k)] = sp.spmv_create(p.m, p.n, r, c, v, options=dict(kernel=k))
x = torch.rand(p.n, dtype=torch.float64, device="cuda")
y = torch.empty(p.m, dtype=torch.float64, device="cuda")
res = {k: [] for k in hs}
for rnd in range(7):
    for k, h in hs.items():
        evs = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            sp.spmv_apply(h, x, y)
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        res[k] += [a.elapsed_time(b) for a, b in evs]
for k, h in hs.items():
    i = sp.spmv_get_info(h)
    print(f"{k[0]:5s} {k[1]:8s} kernel {i['kernel']}: {statistics.median(res[k]) * 1e3:.1f} us "
          f"(nnz {mats[k[0]][1].size}, groups {i.get('groups')}, deferred {i.get('deferred')}, panels {i.get('panels')})")

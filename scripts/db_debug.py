"""Debug of the DB split across loopback ranks: which rows go wrong."""
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import oracle
import paper_1203_2739_b200 as sp
import paper_1203_2739_b200.testing as T
import synth
from test_gpu_ranks import apply_ranks, make_ranks, x_local, y_rows

name, world = sys.argv[1], int(sys.argv[2])
prow = int(sys.argv[3]) if len(sys.argv) > 3 else 0
if name == "_c3w8":
    synth.PRESETS["_c3w8"] = lambda **kw: synth._db(8, 3000, 1000, 10, 16, 0, 4, 10, 20, **kw)
p = synth.make(name, variant="int")
x = p.x()
y_ref = oracle.split(p.row_ptr, p.col, p.val, p.parts, p.n_parts, x)
rbp = p.blocks["row_block_ptr"]
cbp = p.blocks["col_block_ptr"]
K = p.blocks["K"]
xz = x.copy()
xz[cbp[K]:] = 0.0
y_nob = oracle.split(p.row_ptr, p.col, p.val, p.parts, p.n_parts, xz)
hs, infos = make_ranks(p, world, options=dict(panel_rows=prow) if prow else None)
for r, i in enumerate(infos):
    print("rank", r, {k: i[k] for k in ("row_begin", "m_local", "y_local_len", "y_border_begin", "y_border_len",
                                      "x_interior_begin", "x_interior_len", "x_border_begin", "x_border_len",
                                      "panels", "kernel", "split_kernel")})
import time
for rep in range(4):
    t0 = time.time()
    try:
        ys = apply_ranks(hs, infos, [x_local(x, i) for i in infos], split=True)
    except Exception as e:
        print("rep", rep, "raised", str(e)[:120], "timeouts", [sp.spmv_get_info(h)["exchange_timeouts"] for h in hs])
        break
    print(f"rep {rep} took {time.time() - t0:.2f} s, timeouts", [sp.spmv_get_info(h)["exchange_timeouts"] for h in hs])
    y = np.full(p.m, np.nan)
    for i, yd in zip(infos, ys):
        y[y_rows(i)] = yd.cpu().numpy()
    bad = np.flatnonzero(y != y_ref)
    border = bad >= rbp[K]
    nob = (y[bad] == y_nob[bad])
    print(f"rep {rep}: bad {bad.size} (border rows {border.sum()}, block rows {(~border).sum()}); "
          f"equal to 'border x = 0' result: {nob.sum()}; first {bad[:8]}")
    for r, i in enumerate(infos):
        rr = y_rows(i)
        print(f"   rank {r}: bad {np.isin(bad, rr).sum()} of {len(rr)}")
print("timeouts", [sp.spmv_get_info(h)["exchange_timeouts"] for h in hs])

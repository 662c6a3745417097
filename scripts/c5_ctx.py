"""C5 SpMxV time in context: standalone vs inside the power-iteration step
(after max-abs + x-update) vs after a 512 MB memset (dirty L2)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_2739_b200 as sp, synth
w = sys.argv[1] if len(sys.argv) > 1 else "c5"
p = synth.make(w)
h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm, blocks=p.blocks)
info = sp.spmv_get_info(h)
dev = torch.device("cuda")
x = [torch.rand(info["n"], dtype=torch.float64, device=dev) for _ in range(2)]
y = torch.empty(info["m"], dtype=torch.float64, device=dev)
md = torch.zeros(1, dtype=torch.float64, device=dev)
junk = torch.empty(64 << 20, dtype=torch.float64, device=dev)
out = {"workload": w}

def run(label, pre, fuse, reps=20):
    ts = []
    for i in range(reps + 3):
        pre(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sp.spmv_apply(h, x[i % 2], y, sp.SPMV_FUSE_MAXABS if fuse else 0)
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    out[label] = {"median": float(np.median(ts)), "mean": float(np.mean(ts)), "min": float(np.min(ts))}

def glue(i):
    sp.spmv_maxabs(h, md)
    sp.spmv_normalize(h, y, md, x[(i + 1) % 2])
    md.zero_()

run("standalone", lambda i: None, False)
run("standalone_maxabs", lambda i: None, True)
run("after_memset_512MB", lambda i: junk.fill_(1.0), False)
run("power_step", glue, True)
run("standalone_again", lambda i: None, False)
print(json.dumps(out))

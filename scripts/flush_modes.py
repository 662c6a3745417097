"""Cold-L2 protocol check on the small configs: SpMxV time after a 512 MB
write flush (L2 left full of dirty lines, written back during the SpMxV)
vs after write + read of another 512 MB buffer (L2 left clean)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_2739_b200 as sp, synth
out = {}
fb = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
rb = torch.ones(64 << 20, dtype=torch.float64, device="cuda")
sink = torch.zeros(1, dtype=torch.float64, device="cuda")
for w in sys.argv[1:] or ["c2", "c3"]:
    p = synth.make(w)
    kw = dict(row_perm=p.row_perm, col_perm=p.col_perm, blocks=p.blocks)
    if p.n_parts:
        kw.update(parts=p.parts, n_parts=p.n_parts)
    h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, **kw)
    info = sp.spmv_get_info(h)
    x = torch.rand(info["n"], dtype=torch.float64, device="cuda")
    y = torch.empty(info["m"], dtype=torch.float64, device="cuda")
    f = (lambda: sp.spmv_split_apply(h, x, y)) if p.n_parts else (lambda: sp.spmv_apply(h, x, y))
    r = {}
    for mode in ("write", "write+read", "none"):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        for a, b in evs:
            if mode != "none":
                fb.fill_(1.0)
            if mode == "write+read":
                torch.sum(rb, dim=0, keepdim=True, out=sink)
            a.record(); f(); b.record()
        torch.cuda.synchronize()
        r[mode] = float(np.median([a.elapsed_time(b) for a, b in evs]))
    out[w] = r
    sp.spmv_destroy(h)
print(json.dumps(out))

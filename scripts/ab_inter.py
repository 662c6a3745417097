"""Interleaved A/B of create-time variants on one workload, robust to the
power-cap clock drift: all handles are built first, then timed in rounds
(10 back-to-back applies each, variants alternating).
  python ab_inter.py c5 "SPMV_PN_ROWS=16384" "SPMV_PN_ROWS=20480,SPMV_PN_GATHER_NA=1"
A spec's LIB=path runs that variant on another build of the library (loaded
side by side, RTLD_LOCAL; the binding's library handle is swapped per call).
"""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_2739_b200 as sp, synth
w, specs = sys.argv[1], sys.argv[2:]
rounds = int(os.environ.get("ROUNDS", "6"))
p = synth.make(w)
hs, libs = [], []
default_lib = sp.lib()
for s in specs:
    env = dict(kv.split("=", 1) for kv in s.split(",") if kv)
    lp = env.pop("LIB", None)
    if lp:
        sp._lib, sp.LIB_PATH = None, lp
        libs.append(sp.lib())
    else:
        libs.append(default_lib)
    sp._lib = libs[-1]
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm, blocks=p.blocks)
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    hs.append(h)
sp._lib = libs[0]
info = sp.spmv_get_info(hs[0])
x = torch.rand(info["n"], dtype=torch.float64, device="cuda")
y = torch.empty(info["m"], dtype=torch.float64, device="cuda")
for h, L in zip(hs, libs):
    sp._lib = L
    for _ in range(2):
        sp.spmv_apply(h, x, y)
torch.cuda.synchronize()
res = {s: [] for s in specs}
for r in range(rounds):
    order = list(range(len(specs))) if r % 2 == 0 else list(reversed(range(len(specs))))
    for i in order:
        sp._lib = libs[i]
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        for a, b in evs:
            a.record(); sp.spmv_apply(hs[i], x, y); b.record()
        torch.cuda.synchronize()
        res[specs[i]].append(float(np.median([a.elapsed_time(b) for a, b in evs])))
out = {"workload": w, "rounds": rounds}
for s in specs:
    out[s or "default"] = {"median_ms": float(np.median(res[s])), "per_round": [round(v, 4) for v in res[s]]}
print(json.dumps(out))

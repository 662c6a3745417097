"""C5 SpMxV time drift over a sustained run: blocks of 20 back-to-back
standalone SpMxVs, with NVML clocks / temperature / power per block."""
import json, os, sys, time
import numpy as np
import torch
import pynvml
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_2739_b200 as sp, synth
w = sys.argv[1] if len(sys.argv) > 1 else "c5"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 8
pynvml.nvmlInit()
nh = pynvml.nvmlDeviceGetHandleByIndex(0)
p = synth.make(w)
h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm, blocks=p.blocks)
info = sp.spmv_get_info(h)
x = torch.rand(info["n"], dtype=torch.float64, device="cuda")
y = torch.empty(info["m"], dtype=torch.float64, device="cuda")
rows = []
for blk in range(nb):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for a, b in evs:
        a.record(); sp.spmv_apply(h, x, y); b.record()
    time.sleep(0.03)
    s = dict(sm=pynvml.nvmlDeviceGetClockInfo(nh, pynvml.NVML_CLOCK_SM), mem=pynvml.nvmlDeviceGetClockInfo(nh, pynvml.NVML_CLOCK_MEM),
             temp=pynvml.nvmlDeviceGetTemperature(nh, pynvml.NVML_TEMPERATURE_GPU), power=pynvml.nvmlDeviceGetPowerUsage(nh) / 1000,
             reasons=pynvml.nvmlDeviceGetCurrentClocksEventReasons(nh))
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) for a, b in evs]
    s.update(block=blk, median_ms=float(np.median(t)), min_ms=float(np.min(t)), max_ms=float(np.max(t)))
    rows.append(s)
    print(json.dumps(s), flush=True)

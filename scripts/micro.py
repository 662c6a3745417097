"""Design microbenchmarks (diag2.cu): L2->SM bandwidth (LDG, bulk copy,
cluster multicast), shared-memory y += v*x update rate, line-shared gathers."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_2739_b200 as sp
from paper_1203_2739_b200 import diag
from timing import timeit

out = {}
sink = torch.zeros(1, dtype=torch.float64, device="cuda")
for mb in (16, 64):
    buf = torch.rand(mb * (1 << 20) // 8, dtype=torch.float64, device="cuda")
    cnt = 16 << 30
    ms = timeit(lambda: diag.micro(1, 0, buf, buf.numel() * 8, cnt, sink), reps=5, warm=2)
    out[f"l2read_ldg_{mb}MB_GBs"] = round(cnt / ms / 1e6, 1)
    for cl in (1, 2, 4, 8):
        try:
            ms = timeit(lambda: diag.micro(2, cl, buf, buf.numel() * 8, cnt, sink), reps=5, warm=2)
            out[f"tma_{mb}MB_cl{cl}_delivered_GBs"] = round(cnt / ms / 1e6, 1)
        except Exception as e:
            out[f"tma_{mb}MB_cl{cl}_delivered_GBs"] = str(e)[:100]
for mode in (0, 1):
    cnt = 1 << 32
    ms = timeit(lambda: diag.micro(3, mode, None, 0, cnt, sink), reps=5, warm=2)
    out[f"smem_rmw_mode{mode}_Gupd_s"] = round(cnt / ms / 1e6, 1)
x = torch.rand((32 << 20) // 8, dtype=torch.float64, device="cuda")
for g in (1, 2, 4, 8, 16, 32):
    cnt = 1 << 30
    ms = timeit(lambda: diag.micro(4, g, x, x.numel() * 8, cnt, sink), reps=5, warm=2)
    out[f"gather_{g}lanes_per_line_Gps"] = round(cnt / ms / 1e6, 1)
print(json.dumps(out, indent=1))

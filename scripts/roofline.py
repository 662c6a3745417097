"""Roofline microbenchmarks on the B200: HBM read peak,
random x-gather rate from L2, and the speed of light of the SpMxV memory
pattern (stream col/val, +gather x) over the real C4/C5 matrices, next to the
SpMxV kernel itself.  Prints one JSON object; CUDA-event timing, warm-up
first, median of repeats."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1203_2739_b200 as sp  # noqa: E402
import synth  # noqa: E402


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    workloads = sys.argv[1:] or ["c5", "c4"]
    out = {}
    dev = torch.device("cuda")
    sink = torch.zeros(1, dtype=torch.float64, device=dev)
    nbytes = 8 << 30
    buf = torch.empty(nbytes // 8, dtype=torch.float64, device=dev).fill_(1.0)
    for bps in (2, 4, 8):
        ms = timeit(lambda: sp.spmv_diag_read(buf, nbytes, sink, bps))
        out[f"read_gbs_bps{bps}"] = nbytes / ms / 1e6
    copy_dst = torch.empty_like(buf)
    ms = timeit(lambda: copy_dst.copy_(buf))
    out["torch_copy_gbs"] = 2 * nbytes / ms / 1e6
    del copy_dst
    for mb in (1, 8, 32, 128, 1024):
        x = torch.rand(mb * (1 << 20) // 8, dtype=torch.float64, device=dev)
        cnt = 1 << 30
        ms = timeit(lambda: sp.spmv_diag_gather(x, cnt, sink), reps=5)
        out[f"gather_{mb}MB_Gps"] = cnt / ms / 1e6
        out[f"gather_{mb}MB_sector_GBs"] = cnt * 32 / ms / 1e6
    del buf
    torch.cuda.empty_cache()
    for w in workloads:
        t0 = time.time()
        p = synth.make(w)
        h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm,
                           blocks=p.blocks, parts=p.parts, n_parts=p.n_parts)
        info = sp.spmv_get_info(h)
        nnz = p.nnz
        x = torch.rand(info["n"], dtype=torch.float64, device=dev)
        y = torch.empty(info["m"], dtype=torch.float64, device=dev)
        r = {"nnz": nnz, "bytes_alg": info["bytes_alg"], "setup_s": time.time() - t0}
        ms0 = timeit(lambda: sp.spmv_diag_csr(h, x, 0, sink))
        ms1 = timeit(lambda: sp.spmv_diag_csr(h, x, 1, sink))
        ms2 = timeit(lambda: sp.spmv_apply(h, x, y))
        if os.environ.get("ROOFLINE_AB"):
            os.environ["SPMV_KERNEL"] = "tile"
            h2 = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm,
                                blocks=p.blocks, parts=p.parts, n_parts=p.n_parts)
            del os.environ["SPMV_KERNEL"]
            r["spmv_tile_kernel_ms"] = timeit(lambda: sp.spmv_apply(h2, x, y))
            sp.spmv_destroy(h2)
        r["stream_only_ms"] = ms0
        r["stream_only_gbs"] = 12 * nnz / ms0 / 1e6
        r["stream_gather_ms"] = ms1
        r["stream_gather_alg_gbs"] = info["bytes_alg"] / ms1 / 1e6
        r["spmv_ms"] = ms2
        r["spmv_alg_gbs"] = info["bytes_alg"] / ms2 / 1e6
        out[w] = r
        del p
        sp.spmv_destroy(h)
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark of the SpMxV hot path (arXiv 1203.2739) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5|c4|c3|c2|c1]
                    [--impl ours|reference] [--quick]

One JSON line on rank 0.  A "step" is one pass of the whole hot path over the
workload:
  c5/c4 (power iterations, BJ configs 5/4): y^ = A^ x^ with the fused max-abs
        (+ NCCL border-x allgather when N > 1), max all-reduce, x-update;
  c3    (multiple-SpMxV, BJ config 3): y = sum_k A^k x, fused split pass;
  c2/c1: one SpMxV with L2 flushed before each call (their matrices fit L2).
`value` = 2 nnz / step time (GFLOP/s, whole job); `roofline` is the SpMxV
kernel's algorithmic bytes / its average CUDA-event duration against the
measured HBM copy peak; `cpu_baseline` times the CPU oracle (test
infrastructure) on a bounded sample; `e2e` repeats the step through the C ABI
with the input x copied from pinned host memory and y read back every step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMxV GFLOP/s and achieved HBM GB/s (fraction of ~8 TB/s) at 1/2/4/8 B200"
WORKLOAD_DESC = {
    "c1": "tiny irregular 2,000^2, U{4..16} nnz/row, identity perms (BJ configs[0])",
    "c2": "SB 200,000^2, 16 blocks x 12,500 rows, 5% border, hidden perm (BJ configs[1])",
    "c3": "DB 500,000^2, K=8 nonzero-disjoint 2D-block split, fused multiple-SpMxV (BJ configs[2])",
    "c4": "power-law 4,000,000^2, Zipf-Mandelbrot rows, 70% +-2,000 band, 100 power iterations (BJ configs[3])",
    "c5": "SB 64,000,000^2, 64 blocks x 1M rows, 2% border, hidden perm, power iterations (BJ configs[4])",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------------------
# clocks during the timed region (pynvml sampling thread)
# --------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int, period_s: float = 0.02):
        self.idx, self.period = device_index, period_s
        self.samples, self.reasons = [], set()
        self.mem, self.temp, self.power = [], [], []
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:   # pragma: no cover
            log("clock sampler unavailable:", e)
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.mem.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_MEM))
                self.temp.append(self.nv.nvmlDeviceGetTemperature(self.h, self.nv.NVML_TEMPERATURE_GPU))
                self.power.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        out = {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
               "reasons": sorted(self.reasons), "samples": len(self.samples)}
        if self.mem:
            out["mem_mhz"] = statistics.median(self.mem)
        if self.temp:
            out["gpu_temp_c_max"] = max(self.temp)
        if self.power:
            out["power_w_max"] = max(self.power)
        return out


# --------------------------------------------------------------------------
# workload
# --------------------------------------------------------------------------
def make_problem(name: str, rank: int, world: int):
    """Generate the synthetic problem; for world > 1 rank 0 generates it once
    and shares it through a memory-mapped cache (/dev/shm, else /tmp, whichever
    has room: C5 is 14 GB); if neither has room, or writing fails, every rank
    generates it (the generator is counter-based, so all ranks get the same
    matrix)."""
    import synth
    if world == 1:
        return synth.make(name)
    import pickle
    import shutil
    import torch.distributed as dist
    keys = ("row_ptr", "col", "val", "row_perm", "col_perm", "parts", "owner")
    port = os.environ.get("MASTER_PORT", "0")
    p, cache = None, None
    if rank == 0:
        p = synth.make(name)
        need = sum(getattr(p, k).nbytes for k in keys if getattr(p, k) is not None) * 1.05 + (64 << 20)
        for root in ("/dev/shm", "/tmp"):
            try:
                if shutil.disk_usage(root).free < need:
                    continue
                c = os.path.join(root, f"spmv_bench_{name}_{port}")
                os.makedirs(c, exist_ok=True)
                for k in keys:
                    a = getattr(p, k)
                    if a is not None:
                        np.save(os.path.join(c, k + ".npy"), a)
                with open(os.path.join(c, "meta.pkl"), "wb") as f:
                    pickle.dump({"p": {k: v for k, v in p.__dict__.items() if not isinstance(v, np.ndarray)}}, f)
                cache = c
                break
            except OSError as e:
                log(f"problem cache in {root} failed ({e}); trying the next")
                shutil.rmtree(os.path.join(root, f"spmv_bench_{name}_{port}"), ignore_errors=True)
    obj = [cache]
    dist.broadcast_object_list(obj, src=0)
    cache = obj[0]
    if rank != 0:
        if cache is None:
            p = synth.make(name)
        else:
            with open(os.path.join(cache, "meta.pkl"), "rb") as f:
                d = pickle.load(f)["p"]
            for k in keys:
                fn = os.path.join(cache, k + ".npy")
                d[k] = np.load(fn, mmap_mode="r") if os.path.exists(fn) else None
            p = synth.Problem(**d)
    dist.barrier()   # every rank has mapped the files (pages stay mapped after the unlink)
    if rank == 0 and cache is not None:
        shutil.rmtree(cache, ignore_errors=True)
    return p


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


def load_traffic(workload: str):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


# --------------------------------------------------------------------------
# CPU baseline: the oracle on a bounded sample (test infrastructure)
# --------------------------------------------------------------------------
_XCACHE = {}


def oracle_sample(p, target_s: float, nthreads: int, start_row: int = 0, max_rows=None):
    import oracle
    if id(p) not in _XCACHE:
        _XCACHE[id(p)] = p.x()
    x = _XCACHE[id(p)]
    rows = min(p.m, 1 << 16) if max_rows is None else max_rows
    while True:
        r0 = start_row % p.m
        r1 = min(p.m, r0 + rows)
        a, b = int(p.row_ptr[r0]), int(p.row_ptr[r1])
        rp = np.asarray(p.row_ptr[r0:r1 + 1]) - a
        col, val = np.asarray(p.col[a:b]), np.asarray(p.val[a:b])
        t0 = time.perf_counter()
        oracle.spmv(rp, col, val, x, nthreads=nthreads)
        dt = time.perf_counter() - t0
        if dt >= target_s or r1 - r0 >= p.m or max_rows is not None:
            return {"rows": r1 - r0, "nnz": b - a, "seconds": dt, "gflops": 2.0 * (b - a) / dt / 1e9,
                    "row_range": [r0, r1]}
        rows = int(min(p.m, max(rows * 2, rows * target_s / max(dt, 1e-3) * 1.1)))


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_one_core(p, target_s: float):
    """The oracle on ONE pinned host core (sched_setaffinity): the paper's
    single-threaded setting (OSKI on one core)."""
    old = os.sched_getaffinity(0)
    core = min(old)
    try:
        os.sched_setaffinity(0, {core})
        return oracle_sample(p, target_s, 1), core
    finally:
        os.sched_setaffinity(0, old)


def cpu_leg(args, p, split, x_gpu, y_gpu, m_gpu=None, xn_gpu=None):
    """The only place the timed arm touches oracle/: the CPU baseline (all
    cores and one pinned core) and the teacher-forced parity check of the last
    timed step (y_t on sampled rows, m_t and x_{t+1} on every entry)."""
    import oracle
    cpu = parity = None
    if not args.no_cpu_baseline:
        nthreads = len(os.sched_getaffinity(0)) or os.cpu_count() or 1
        r = oracle_sample(p, args.cpu_seconds, nthreads)
        r1, core = oracle_one_core(p, max(2.0, args.cpu_seconds / 2))
        cpu = {"value": r["gflops"], "unit": "GFLOP/s", "cores": nthreads, "kind": "oracle",
               "cpu_model": cpu_model(), "nproc": os.cpu_count(),
               "sample": f"{r['rows']} consecutive original-order rows ({r['nnz']} nnz) of {args.workload}, "
                         f"oracle.spmv (serial per-row fp64, rows over {nthreads} threads), {r['seconds']:.1f} s",
               "one_core": {"value": r1["gflops"], "unit": "GFLOP/s", "cores": 1, "pinned_core": core,
                            "sample": f"{r1['rows']} rows ({r1['nnz']} nnz), 1 thread pinned with "
                                      f"sched_setaffinity, {r1['seconds']:.1f} s (the paper's single-core "
                                      "setting, P:L142)"}}
    if not args.no_parity and x_gpu is not None:
        rng = np.random.default_rng(1234)
        nsamp = min(p.m, args.parity_rows)
        prow = np.sort(rng.choice(p.m, nsamp, replace=False))          # permuted rows checked
        x_orig = x_gpu[p.col_perm] if p.col_perm is not None else x_gpu  # x[j] = x^[col_perm[j]]
        if p.row_perm is not None:
            inv = np.empty_like(p.row_perm)
            inv[p.row_perm] = np.arange(p.m, dtype=p.row_perm.dtype)
            orow = inv[prow]
        else:
            orow = prow
        yref, S = oracle.spmv_rows(orow, p.row_ptr, p.col, p.val, x_orig)
        if split:
            yref = oracle.split(p.row_ptr, p.col, p.val, p.parts, p.n_parts, x_orig)[orow]
        nbad, worst, _ = oracle.check(y_gpu[prow], yref, S)
        parity = {"rows_checked": int(nsamp), "failures": int(nbad), "max_err_over_S": worst,
                  "tol": 1e-12, "teacher_forced": True, "step": "last timed step"}
        if m_gpu is not None and xn_gpu is not None:
            # a9: m_t = max |y_t| exactly (over all rows), x_{t+1} = y_t / m_t bitwise (every entry)
            y_orig = oracle.unpermute_y(p.row_perm, y_gpu) if p.row_perm is not None else y_gpu
            m_ref = oracle.maxabs(y_orig)
            xn_orig = xn_gpu[p.col_perm] if p.col_perm is not None else xn_gpu
            xn_ref = oracle.scale(y_orig, m_gpu)
            parity["maxabs_exact"] = bool(m_gpu == m_ref)
            parity["x_next_bitwise"] = bool(np.array_equal(xn_orig.view(np.int64), xn_ref.view(np.int64)))
            parity["x_next_entries"] = int(len(xn_ref))
            if not (parity["maxabs_exact"] and parity["x_next_bitwise"]):
                parity["failures"] += 1
    return cpu, parity


# --------------------------------------------------------------------------
# reference arm: the oracle as it stands, on the host cores
# --------------------------------------------------------------------------
def run_reference(args, rank, world):
    if rank != 0:
        return 0
    p = make_problem(args.workload, 0, 1)
    nthreads = len(os.sched_getaffinity(0)) or os.cpu_count() or 1
    import oracle
    # calibrate a per-step sample of ~1 s (bounded), then time W + K steps
    cal = oracle_sample(p, 1.0, nthreads)
    rows = cal["rows"]
    for w in range(args.warmup):
        oracle_sample(p, 0, nthreads, start_row=w * rows, max_rows=rows)
    tot_nnz, tot_s = 0, 0.0
    for k in range(args.steps):
        r = oracle_sample(p, 0, nthreads, start_row=(args.warmup + k) * rows, max_rows=rows)
        tot_nnz += r["nnz"]
        tot_s += r["seconds"]
    gf = 2.0 * tot_nnz / tot_s / 1e9
    sample = f"{args.steps} steps x {rows} consecutive original-order rows of {args.workload} (oracle.spmv, {nthreads} threads)"
    line = {"impl": "reference", "metric": METRIC, "value": gf, "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_s / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": args.workload, "desc": WORKLOAD_DESC[args.workload]},
            "cpu_baseline": {"value": gf, "unit": "GFLOP/s", "cores": nthreads, "kind": "oracle",
                             "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": gf, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    del oracle
    return 0


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import torch
    import paper_1203_2739_b200 as sp
    from paper_1203_2739_b200 import diag

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
    t0 = time.time()
    p = make_problem(args.workload, rank, world)
    t_gen = time.time() - t0
    uid = None
    if world > 1:
        obj = [sp.spmv_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    t0 = time.time()
    split = p.parts is not None
    h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm,
                       blocks=p.blocks, parts=p.parts, n_parts=p.n_parts,
                       dist=None if world == 1 else dict(rank=rank, world=world, device=local_rank,
                                                         nccl_unique_id=uid))
    t_create = time.time() - t0
    info = sp.spmv_get_info(h)
    log(f"[rank {rank}] gen {t_gen:.1f}s create {t_create:.1f}s nnz {p.nnz} local {info['nnz_local']} "
        f"tiles {info['n_tiles']} long {info['n_long_rows']}")

    # x^ (permuted, this rank's layout)
    x = p.x()
    xhat = np.empty_like(x)                 # input preparation: x^[col_perm[j]] = x[j]
    if p.col_perm is not None:
        xhat[p.col_perm] = x
    else:
        xhat[:] = x
    if world > 1:
        a, L = info["x_interior_begin"], info["x_interior_len"]
        b, Lb = info["x_border_begin"], info["x_border_len"]
        xloc = np.concatenate([xhat[a:a + L], xhat[b:b + Lb]])
    else:
        xloc = xhat
    xd = torch.from_numpy(np.ascontiguousarray(xloc)).to(dev)
    x_in = xd.clone()
    yd = torch.empty(info["m_local"], dtype=torch.float64, device=dev)
    md = torch.zeros(1, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    power = args.workload in ("c4", "c5") and info["has_owner_map"]
    l2_flush = args.workload in ("c1", "c2", "c3")
    flush_buf = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device=dev) if l2_flush else None
    xbuf = [xd, torch.empty_like(xd)]
    launches_per_step = 0

    def apply(xcur):
        if split:
            sp.spmv_split_apply(h, xcur, yd, sp.SPMV_FUSE_MAXABS if power else 0, stream=stream)
        else:
            sp.spmv_apply(h, xcur, yd, sp.SPMV_FUSE_MAXABS if power else 0, stream=stream)

    def glue(xcur, xnext):
        sp.spmv_maxabs(h, md, stream=stream)
        sp.spmv_normalize(h, yd, md, xnext, stream=stream)

    # our kernels per step: the SpMxV kernel (panel or row-tile), max-abs finish
    # and x-update for the power iterations
    launches_per_step = 1 + (2 if power else 0)
    cur = 0
    for _ in range(args.warmup):
        if l2_flush:
            flush_buf.fill_(1.0)
        apply(xbuf[cur])
        if power:
            glue(xbuf[cur], xbuf[1 - cur])
            cur = 1 - cur
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()

    K = args.steps
    ev_a = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev_b = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    st_all = torch.cuda.Event(enable_timing=True)
    en_all = torch.cuda.Event(enable_timing=True)
    x_last = None
    with ClockSampler(local_rank) as clk:
        st_all.record(stream)
        for k in range(K):
            if l2_flush:
                flush_buf.fill_(1.0)
            ev_a[k].record(stream)
            apply(xbuf[cur])
            ev_b[k].record(stream)
            if power:
                if k == K - 1:
                    x_last = xbuf[cur]
                glue(xbuf[cur], xbuf[1 - cur])
                cur = 1 - cur
        en_all.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    spmv_ms = [a.elapsed_time(b) for a, b in zip(ev_a, ev_b)]
    total_ms = st_all.elapsed_time(en_all)
    if l2_flush:   # the flush is not part of the path: step time = SpMxV time
        total_ms = sum(spmv_ms)
    avg_spmv_ms = sum(spmv_ms) / K
    if dist:
        t = torch.tensor([total_ms, avg_spmv_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, avg_spmv_max = t.tolist()
    else:
        avg_spmv_max = avg_spmv_ms
    ms_per_step = total_ms / K
    gflops = 2.0 * p.nnz / (ms_per_step * 1e-3) / 1e9

    # device copies of the last step's x_t, y_t, m_t and x_{t+1} for the CPU
    # leg's parity check (teacher-forced: the oracle recomputes from x_t)
    if not power:
        x_last = xbuf[cur]
    y_gpu = yd.cpu().numpy() if world == 1 else None
    x_gpu = x_last.cpu().numpy() if world == 1 else None
    m_gpu = float(md.item()) if (power and world == 1) else None
    xn_gpu = xbuf[cur].cpu().numpy() if (power and world == 1) else None

    # ---------------- e2e through the C ABI with host buffers
    # Every step copies its input x from pinned host memory and reads its
    # result y (and the max) back.  The steps are pipelined over three
    # streams: step i+1's host->device copy and step i-1's device->host copy
    # run while step i computes (PCIe is full duplex); buffers are double-
    # buffered and ordered with events.
    e2e = None
    if not args.no_e2e:
        hx = torch.from_numpy(np.ascontiguousarray(xloc)).pin_memory()
        hy = [torch.empty(info["m_local"], dtype=torch.float64).pin_memory() for _ in range(2)]
        hm = [torch.empty(1, dtype=torch.float64).pin_memory() for _ in range(2)]
        xin = [torch.empty_like(xd) for _ in range(2)]
        yb = [torch.empty(info["m_local"], dtype=torch.float64, device=dev) for _ in range(2)]
        mb = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(2)]
        xn = torch.empty_like(xd)
        s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_c = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        for e in ev_c + ev_out:
            e.record(stream)
        flags = sp.SPMV_FUSE_MAXABS if power else 0

        def e2e_step(i):
            j = i % 2
            s_in.wait_event(ev_c[j])                 # xin[j] last read by step i-2
            with torch.cuda.stream(s_in):
                xin[j].copy_(hx, non_blocking=True)
            ev_in[j].record(s_in)
            stream.wait_event(ev_in[j])
            stream.wait_event(ev_out[j])             # yb[j] last read by step i-2's copy-out
            if split:
                sp.spmv_split_apply(h, xin[j], yb[j], flags, stream=stream)
            else:
                sp.spmv_apply(h, xin[j], yb[j], flags, stream=stream)
            if power:
                sp.spmv_maxabs(h, mb[j], stream=stream)
                sp.spmv_normalize(h, yb[j], mb[j], xn, stream=stream)
            ev_c[j].record(stream)
            s_out.wait_event(ev_c[j])
            with torch.cuda.stream(s_out):
                hy[j].copy_(yb[j], non_blocking=True)
                if power:
                    hm[j].copy_(mb[j], non_blocking=True)
            ev_out[j].record(s_out)

        Ke = max(3, min(K, args.e2e_steps))
        for i in range(2):
            e2e_step(i)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(Ke):
            e2e_step(i)
        for j in range(2):
            stream.wait_event(ev_out[j])
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / Ke
        if dist:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = t.item()
        # the e2e step's own bound: the same H2D and D2H copies, concurrent on
        # their two streams, with no compute (the host link, full duplex)
        l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        l0.record(stream)
        s_in.wait_stream(stream)
        s_out.wait_stream(stream)
        for i in range(Ke):
            with torch.cuda.stream(s_in):
                xin[i % 2].copy_(hx, non_blocking=True)
            with torch.cuda.stream(s_out):
                hy[i % 2].copy_(yb[i % 2], non_blocking=True)
        stream.wait_stream(s_in)
        stream.wait_stream(s_out)
        l1.record(stream)
        torch.cuda.synchronize()
        lms = l0.elapsed_time(l1) / Ke
        e2e = {"value": 2.0 * p.nnz / (ems * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": ems,
               "h2d_bytes_per_step": int(hx.numel() * 8),
               "d2h_bytes_per_step": int(hy[0].numel() * 8 + (8 if power else 0)),
               "steps": Ke, "pipelined": "3 streams: H2D(i+1) and D2H(i-1) overlap compute(i), double-buffered",
               "link_bound_ms_per_step": lms, "frac_of_link_bound": lms / ems,
               "link_note": "the same H2D + D2H copies concurrently, no compute, measured in this run"}
        del xin, yb, hy

    # ---------------- second roofline: the LSU x-gather rate, measured live
    gather = None
    if not args.no_gather_peak and info["kernel"] == 7 and not split and info["gather_sectors"] > 0:
        # the panel kernel's second roofline: bytes crossing L2 -> SM per launch
        # (its group stream + the distinct 32-byte x sectors its gathers request,
        # counted at plan time) against an L2-resident LDG stream measured live
        gb = torch.rand((16 << 20) // 8, dtype=torch.float64, device=dev)    # 16 MB, L2-resident
        sink = torch.zeros(1, dtype=torch.float64, device=dev)
        cnt = 8 << 30
        for _ in range(2):
            diag.micro(1, 0, gb, gb.numel() * 8, cnt, sink, stream=stream)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(3):
            diag.micro(1, 0, gb, gb.numel() * 8, cnt, sink, stream=stream)
        g1.record(stream)
        torch.cuda.synchronize()
        fpeak = 3 * cnt / (g0.elapsed_time(g1) * 1e-3) / 1e9
        fbytes = info["bytes_stream"] + 32 * info["gather_sectors"]
        fach = fbytes / (avg_spmv_ms * 1e-3) / 1e9
        gather = {"bound": "l2_to_sm", "achieved": fach, "peak": fpeak, "unit": "GB/s", "frac": fach / fpeak,
                  "bytes_per_launch": fbytes,
                  "note": "group stream + distinct 32-byte x sectors of the gathers (plan-time count) per launch / "
                          "SpMxV time; peak = 128-bit LDG stream over a 16 MB L2-resident buffer, measured in this "
                          "run (libspmv_diag.so spmv_diag_micro kind 1)"}
        del gb
    if not args.no_gather_peak and info["kernel"] != 7:   # the panel kernel does not gather once per nonzero
        gx = torch.rand(4 << 20, dtype=torch.float64, device=dev)      # 32 MB, L2-resident
        sink = torch.zeros(1, dtype=torch.float64, device=dev)
        cnt = 1 << 29
        for _ in range(2):
            diag.gather_mode(gx, cnt, 0, sink, stream=stream)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(3):
            diag.gather_mode(gx, cnt, 0, sink, stream=stream)
        g1.record(stream)
        torch.cuda.synchronize()
        gpeak = 3 * cnt / (g0.elapsed_time(g1) * 1e-3) / 1e9
        nnz_loc = info["nnz_local"]
        gach = nnz_loc / (avg_spmv_ms * 1e-3) / 1e9
        gather = {"bound": "lsu_gather", "achieved": gach, "peak": gpeak, "unit": "Ggathers/s", "frac": gach / gpeak,
                  "note": "one x gather per nonzero; peak = random 8-byte __ldg gathers from a 32 MB L2-resident "
                          "vector, measured in this run (spmv_diag_gather_mode)"}
        del gx

    # ---------------- roofline of the SpMxV kernel
    peaks, peak_src = load_peaks()
    bytes_alg = info["bytes_alg_split"] if split else info["bytes_alg"]
    if dist:
        t = torch.tensor([bytes_alg], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        bytes_tot = t.item()
    else:
        bytes_tot = bytes_alg
    achieved = bytes_alg / (avg_spmv_ms * 1e-3) / 1e9       # this rank's kernel
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    tr = load_traffic(args.workload)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": tr.get("dram_bytes_per_launch") if tr else None,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src}, copy read+write)",
                "bytes_alg_per_launch": bytes_alg, "kernel_ms": avg_spmv_ms,
                "frac_of_8TBs": achieved / 8000.0}

    # ---------------- CPU leg (rank 0, N = 1 only): oracle baseline + sampled parity
    cpu, parity = None, None
    if rank == 0 and world == 1:
        cpu, parity = cpu_leg(args, p, split, x_gpu, y_gpu, m_gpu, xn_gpu)

    # ---------------- warm-L2 time (C1-C3 are otherwise timed with L2 flushed)
    extra = {}
    if l2_flush:
        wm = []
        for _ in range(3):
            apply(xbuf[cur])
        # queued back to back (one sync at the end), as in the timed loop: a
        # per-call sync would put the host's launch latency inside the events
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        for a_, b_ in evs:
            a_.record(stream)
            apply(xbuf[cur])
            b_.record(stream)
        torch.cuda.synchronize()
        wm = [a_.elapsed_time(b_) for a_, b_ in evs]
        extra["warm_l2_spmv_ms"] = statistics.median(wm)

    # ---------------- reordering effect (the paper's Table 2 analog)
    if world == 1 and not args.no_reorder_ref and p.row_perm is not None and not split:
        # the same matrix in its ORIGINAL (scrambled) order, no permutation, no
        # blocks: what the SpMxV costs without the SB reordering;
        # same L2 protocol as the main timing
        sp.spmv_destroy(h)
        h = None
        torch.cuda.empty_cache()
        xs_ = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
        ys_ = torch.empty(p.m, dtype=torch.float64, device=dev)

        def time_scrambled(kernel):
            # "rowtile" keeps the input CSR order (the paper's unordered
            # baseline); "auto" lets the default planner run, whose panels sort
            # each row panel's nonzeros by column by themselves
            hs = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, options=dict(kernel=kernel))
            kern = sp.spmv_get_info(hs)["kernel"]
            for _ in range(3):
                sp.spmv_apply(hs, xs_, ys_, stream=stream)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
            for a_, b_ in evs:   # queued back to back, one sync (no host launch latency inside the events)
                if l2_flush:
                    flush_buf.fill_(1.0)
                a_.record(stream)
                sp.spmv_apply(hs, xs_, ys_, stream=stream)
                b_.record(stream)
            torch.cuda.synchronize()
            tms = [a_.elapsed_time(b_) for a_, b_ in evs]
            sp.spmv_destroy(hs)
            return statistics.median(tms), KERNEL_NAMES.get(kern, str(kern))

        sms, skern = time_scrambled("rowtile")
        pms, pkern = time_scrambled("auto")
        extra["reordering"] = {"scrambled_spmv_ms": sms, "reordered_spmv_ms": avg_spmv_ms,
                               "speedup": sms / avg_spmv_ms,
                               "scrambled_kernel": skern + " on the input (scrambled) CSR order, no blocks",
                               "scrambled_default_ms": pms,
                               "scrambled_default_kernel": pkern + " on the scrambled matrix, no blocks "
                                                           "(the panel's own column sort recovers part of the locality)",
                               "note": "same matrix and x: input order vs SB-reordered (Table 2 analog, P:L51-55)"}
        if not args.no_sbfs:
            # f4: the order produced on the GPU instead of received -- the sBFS
            # analog + SB extraction with the planted form's K --
            # and its Table 3 analog: the ordering (+ ingest)
            # time in SpMxVs of the unordered matrix, and the SpMxVs it
            # takes to amortize against the unordered SpMxV
            K = int(p.blocks["K"])
            torch.cuda.synchronize()
            t0 = time.time()
            g = sp.spmv_order_sbfs(p.m, p.n, p.row_ptr, p.col, K)
            t_order = time.time() - t0
            t0 = time.time()
            hb = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=g["row_perm"], col_perm=g["col_perm"],
                                blocks=g["blocks"])
            t_create = time.time() - t0
            xb_ = torch.empty(p.n, dtype=torch.float64, device=dev)
            xb_[torch.from_numpy(g["col_perm"].astype(np.int64)).to(dev)] = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
            ys_ = torch.empty(p.m, dtype=torch.float64, device=dev)
            for _ in range(3):
                sp.spmv_apply(hb, xb_, ys_, stream=stream)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
            for a_, b_ in evs:
                if l2_flush:
                    flush_buf.fill_(1.0)
                a_.record(stream)
                sp.spmv_apply(hb, xb_, ys_, stream=stream)
                b_.record(stream)
            torch.cuda.synchronize()
            bms = statistics.median([a_.elapsed_time(b_) for a_, b_ in evs])
            bkern = KERNEL_NAMES.get(sp.spmv_get_info(hb)["kernel"], "?")
            sp.spmv_destroy(hb)
            gain = sms - bms
            extra["reordering"]["sbfs"] = {
                "K": K, "border_cols": int(g["border_cols"]), "planted_border_cols": int(p.n - p.blocks["col_block_ptr"][K]),
                "bfs_levels": int(g["levels"]), "components": int(g["components"]),
                "order_device_ms": g["bfs_ms"] + g["extract_ms"], "order_wall_s": t_order, "create_s": t_create,
                "spmv_ms": bms, "kernel": bkern, "speedup_vs_scrambled": sms / bms,
                "overhead_spmvs": (t_order * 1e3) / sms, "overhead_with_create_spmvs": ((t_order + t_create) * 1e3) / sms,
                "amortization_spmvs": ((t_order * 1e3) / gain) if gain > 0 else None,
                "amortization_with_create_spmvs": (((t_order + t_create) * 1e3) / gain) if gain > 0 else None,
                "note": "spmv_order_sbfs on the scrambled input (GPU BFS on the bipartite graph + SB extraction), "
                        "then spmv_create with that order; overhead in unordered SpMxVs and amortization = "
                        "ordering time / (unordered - sBFS-ordered SpMxV time), Table 3's definition"}
            del xb_
        del xs_, ys_

    # ---------------- the smem-staging effect: the x-staged
    # kernel (each CTA stages its SB block's x(C_k) + x(C_B) in shared
    # memory) against the default, same protocol; only where it fits
    xs_fits = False
    if world == 1 and p.blocks is not None and int(p.blocks.get("kind", 0)) == 1 and not split:
        cb_ = np.asarray(p.blocks["col_block_ptr"])
        K_ = int(p.blocks["K"])
        xs_fits = int(np.max(np.diff(cb_[:K_ + 1]))) + int(cb_[K_ + 1] - cb_[K_]) <= 227 * 1024 // 8
    if xs_fits:
        try:
            hx = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm,
                                blocks=p.blocks, options=dict(kernel="xstaged"))
        except sp.SpmvError:
            hx = None
        if hx is not None:
            xq_ = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
            yq_ = torch.empty(p.m, dtype=torch.float64, device=dev)
            for _ in range(3):
                sp.spmv_apply(hx, xq_, yq_, sp.SPMV_VEC_ORIGINAL, stream=stream)
            xh_ = torch.empty_like(xq_)
            xh_[torch.from_numpy(np.asarray(p.col_perm).astype(np.int64)).to(dev)] = xq_
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
            for a_, b_ in evs:
                if l2_flush:
                    flush_buf.fill_(1.0)
                a_.record(stream)
                sp.spmv_apply(hx, xh_, yq_, stream=stream)
                b_.record(stream)
            torch.cuda.synchronize()
            xms = statistics.median([a_.elapsed_time(b_) for a_, b_ in evs])
            extra["xstaged"] = {"spmv_ms": xms, "default_spmv_ms": avg_spmv_ms, "speedup_vs_default": avg_spmv_ms / xms,
                                "note": "x-staged kernel (block x in shared memory, 16-bit block-local ids) vs the "
                                        "default kernel, same L2 protocol"}
            sp.spmv_destroy(hx)
            del xq_, yq_, xh_

    # ---------------- cuSPARSE comparator (informational): the
    # vendor CSR SpMV (torch.mv on a CSR tensor -> cusparseSpMV, fp64, int32
    # indices) on the same reordered matrix, same L2 protocol; not the product
    # path and not a baseline arm
    if world == 1 and not args.no_cusparse:
        try:
            if h is not None:
                sp.spmv_destroy(h)
                h = None
            torch.cuda.empty_cache()
            import synth
            q = synth.make(args.workload, scramble=0) if p.row_perm is not None else p
            idt = np.int32 if q.nnz < 2**31 else np.int64
            crow = torch.from_numpy(np.asarray(q.row_ptr).astype(idt)).to(dev)
            colq = torch.from_numpy(np.asarray(q.col).astype(idt)).to(dev)
            valq = torch.from_numpy(np.asarray(q.val)).to(dev)
            Acs = torch.sparse_csr_tensor(crow, colq, valq, size=(q.m, q.n))
            xq = torch.rand(q.n, dtype=torch.float64, device=dev)
            with torch.cuda.stream(stream):
                for _ in range(3):
                    yq = torch.mv(Acs, xq)
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
                for a_, b_ in evs:   # queued back to back, as for our kernel
                    if l2_flush:
                        flush_buf.fill_(1.0)
                    a_.record(stream)
                    yq = torch.mv(Acs, xq)
                    b_.record(stream)
                torch.cuda.synchronize()
                tcs = [a_.elapsed_time(b_) for a_, b_ in evs]
            cms = statistics.median(tcs)
            extra["cusparse"] = {"spmv_ms": cms, "ours_spmv_ms": avg_spmv_ms, "speedup_ours": cms / avg_spmv_ms,
                                 "gflops": 2.0 * q.nnz / (cms * 1e-3) / 1e9,
                                 "what": "torch.mv(CSR fp64, int32 indices) -> cusparseSpMV on the reordered matrix"}
            del Acs, crow, colq, valq, xq, yq, q
            torch.cuda.empty_cache()
        except Exception as e:   # informational only
            extra["cusparse"] = {"error": f"{type(e).__name__}: {str(e)[:200]}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": gflops, "unit": "GFLOP/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "desc": WORKLOAD_DESC[args.workload],
                       "m": p.m, "n": p.n, "nnz": p.nnz,
                       "step": ("SpMxV+maxabs+x-update (power iteration)" if power else
                                "fused multiple-SpMxV" if split else "SpMxV"),
                       "l2": ("flushed (512 MB write) before every SpMxV; step time = SpMxV time" if l2_flush
                              else f"inputs larger than L2 ({bytes_tot / 1e9:.1f} GB vs 126 MB)"),
                       "parallelism": f"sb-rowblock{world}" if world > 1 else "1gpu",
                       "kernel": (SPLIT_KERNEL_NAMES.get(info["split_kernel"], str(info["split_kernel"]))
                                  if split else KERNEL_NAMES.get(info["kernel"], str(info["kernel"])))},
            "hbm_gbs": bytes_tot / (avg_spmv_max * 1e-3) / 1e9,
            "spmv_ms": avg_spmv_max,
            "roofline": roofline,
            "roofline_gather": gather,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * K,
            "clocks": clk.summary(),
            "parity": parity,
            "setup_s": {"generate": t_gen, "create": t_create,
                        "create_phases": dict(zip(("validate_descriptor_shard", "permute", "tiles_csr_upload",
                                                   "split_layouts", "panel_plans_upload", "maps_buffers"),
                                                  [round(v, 3) for v in info["create_s"]]))},
            **extra,
        }
        print(json.dumps(line), flush=True)
    if h is not None:
        sp.spmv_destroy(h)
    return 0


KERNEL_NAMES = {7: "panel (column-sorted, y in shared memory)", 0: "row-tile"}
SPLIT_KERNEL_NAMES = {7: "fused multiple-SpMxV on panels (a y slot per (row, part) segment)",
                      3: "fused multiple-SpMxV (row-major part segments)",
                      1: "fused multiple-SpMxV (part-major tiles)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOAD_DESC))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gather-peak", action="store_true")
    ap.add_argument("--no-reorder-ref", action="store_true", help="skip the scrambled-order reference timing")
    ap.add_argument("--no-cusparse", action="store_true", help="skip the cuSPARSE comparator timing")
    ap.add_argument("--no-sbfs", action="store_true", help="skip the GPU sBFS ordering (f4) timing")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--parity-rows", type=int, default=200000)
    ap.add_argument("--e2e-steps", type=int, default=10)
    args = ap.parse_args()
    if args.steps is None:
        args.steps = {"c5": 50, "c4": 100, "c3": 100, "c2": 100, "c1": 100}[args.workload]
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        log(f"note: WORLD_SIZE={world} but --gpus {args.gpus}; using WORLD_SIZE")
        args.gpus = world
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.impl == "reference":
            rc = run_reference(args, rank, world)
        else:
            rc = run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())

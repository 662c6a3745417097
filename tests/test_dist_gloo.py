"""Multi-rank SB sharding on CPU (-m "not gpu"): world_size 2 and 4 with the
gloo backend.  Each rank takes its shard from the library's host-side shard
planner (spmv_shard_plan, the routine spmv_create uses), holds only its owned
x entries, exchanges the border x slices with an all-gather (the NCCL
allgather of the GPU path: the row slices R_k share only the coupling
columns), computes its rows, and must match the single-process oracle
bit-for-bit (every row is summed in the same order on its owner).  The
power-iteration glue (max all-reduce + owner-local x-update, reading A17) is
checked the same way."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_1203_2739_b200 as sp
import synth


class _S:
    def __init__(self, d):
        self.__dict__.update(d)


def shard_plan(p, rank, world):
    return _S(sp.spmv_shard_plan(p.blocks, p.m, p.n, rank, world))


def _worker(rank, world, port, name, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = synth.make(name, variant="real")
        s = shard_plan(p, rank, world)
        # permuted CSR (test infrastructure: the oracle's permuter) and x^
        rp, col, val, _ = oracle.permute(p.m, p.n, p.row_ptr, p.col, p.val, p.row_perm, p.col_perm)
        x = p.x()
        xh = oracle.permute_x(p.col_perm, x)
        # the rank owns only these x entries
        x_int = xh[s.x_interior_begin:s.x_interior_begin + s.x_interior_len].copy()
        x_own_b = xh[s.x_border_begin:s.x_border_begin + s.x_border_len].copy()
        # border exchange: all-gather of the owned slices (equal sizes here)
        parts = [torch.empty(s.x_border_len, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(x_own_b))
        x_border = torch.cat(parts).numpy()
        assert len(x_border) == s.border_total
        # local rows with columns in the local layout [interior | C_B]
        r0, r1 = s.row_begin, s.row_end
        a, b = rp[r0], rp[r1]
        lrp = rp[r0:r1 + 1] - a
        lcol = col[a:b].astype(np.int64)
        inside = lcol < s.border_begin
        assert np.all(lcol[inside] >= s.x_interior_begin)
        assert np.all(lcol[inside] < s.x_interior_begin + s.x_interior_len)   # Eq.(1) envelope
        lcol = np.where(inside, lcol - s.x_interior_begin, s.x_interior_len + (lcol - s.border_begin))
        xloc = np.concatenate([x_int, x_border])
        y_loc, _ = oracle.spmv(lrp, lcol.astype(np.int32), val[a:b], xloc)
        y_ref, _ = oracle.spmv(rp, col, val, xh)
        ok_spmv = bool(np.array_equal(y_loc, y_ref[r0:r1]))
        # power-iteration glue: global max, owner-local update x^[c] = y^[r(c)]/m
        mloc = torch.tensor([oracle.maxabs(y_loc)], dtype=torch.float64)
        dist.all_reduce(mloc, op=dist.ReduceOp.MAX)
        mt = mloc.item()
        owned = np.concatenate([np.arange(s.x_interior_begin, s.x_interior_begin + s.x_interior_len),
                                np.arange(s.x_border_begin, s.x_border_begin + s.x_border_len)])
        own_rows = p.owner[owned]
        ok_owner = bool(np.all((own_rows >= r0) & (own_rows < r1)))
        x_next_loc = y_loc[own_rows - r0] / mt
        x_next_ref = oracle.permute_x(p.col_perm, oracle.scale(oracle.unpermute_y(p.row_perm, y_ref),
                                                               oracle.maxabs(y_ref)))
        ok_update = bool(np.array_equal(x_next_loc, x_next_ref[owned]))
        result_q.put((rank, ok_spmv, ok_owner, ok_update, int(r1 - r0)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
def test_sb_sharding_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, "c5s", q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort()
    assert all(r[1] for r in res), res
    assert all(r[2] for r in res), res
    assert all(r[3] for r in res), res
    assert sum(r[4] for r in res) == synth.make("c5s").m


def _bench_problem_worker(rank, world, port, shm_limit, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import shutil
    import bench
    if shm_limit:   # pretend neither cache root has room: every rank generates
        real = shutil.disk_usage
        shutil.disk_usage = lambda path: real(path)._replace(free=0)
    p = bench.make_problem("c5s", rank, world)
    q = synth.make("c5s")
    same = all(np.array_equal(np.asarray(getattr(p, k)), getattr(q, k))
               for k in ("row_ptr", "col", "val", "row_perm", "col_perm"))
    dist.barrier()
    dist.destroy_process_group()
    result_q.put((rank, same))


@pytest.mark.parametrize("shm_limit", [False, True])
def test_bench_problem_sharing_gloo(shm_limit):
    """bench.py's multi-rank problem setup: rank 0 generates and shares the
    matrix through a memory-mapped cache, or (no room) every rank generates
    it; either way each rank sees the generator's matrix bit for bit."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_problem_worker, args=(r, 2, port, shm_limit, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert all(r[1] for r in res), res

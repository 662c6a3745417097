"""The multi-GPU path on one GPU (-m gpu): the loopback fake of SURVEY §4.

Every rank of world G is built as a real shard (spmv_test_create_rank: its
rows, local CSR, x / y layouts, panel plan) and the G ranks are linked into a
loopback group (spmv_test_loopback_link): each rank's apply then runs the
P2P exchange protocol of the multi-GPU path -- copy-engine pushes of its
border-x slice (and, DB, its border-row temporaries) into the other ranks'
buffers on its comm stream, stream-memory-operation flags, the kernel's
device-side wait before its first border epoch, the double-buffered parity
-- with the peers' buffers on the same GPU.  Each rank runs on its own
stream, as each would on its own GPU.

  * SB (Eq.(1)): every rank's y equals its rows of the single-GPU y
    bit for bit (the plan does not depend on the GPU count) and matches the
    oracle; the power-iteration glue reproduces the single-GPU steps bit for
    bit over several applies (both buffer parities).
  * DB split across GPUs (f1): y = sum_k A^k x with part k on
    block k's rank and the border rows' temporaries folded in part order on
    their owner -- integer data bit-exact against the oracle's literal split,
    real data within the north_star tolerance.
  * a4: the kernel's interior epochs run while a peer's border slice is still
    in flight (event timing with a late peer).
Only NCCL and CUDA IPC themselves are not exercised (one GPU per call)."""
import time

import numpy as np
import pytest

import oracle
import paper_1203_2739_b200 as sp
import paper_1203_2739_b200.testing as T
import synth
from gpu_util import assert_parity, create, oracle_permuted

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    sp.lib()


def make_ranks(p, world, parts=True, options=None):
    hs = [T.test_create_rank(p.m, p.n, p.row_ptr, p.col, p.val, r, world, row_perm=p.row_perm,
                             col_perm=p.col_perm, blocks=p.blocks, parts=p.parts if parts else None,
                             n_parts=p.n_parts if parts else 0, options=options) for r in range(world)]
    T.loopback_link(hs)
    return hs, [sp.spmv_get_info(h) for h in hs]


def x_local(xh, info):
    a, L = info["x_interior_begin"], info["x_interior_len"]
    b, Lb = info["x_border_begin"], info["x_border_len"]
    return np.concatenate([xh[a:a + L], xh[b:b + Lb]])


def y_rows(info):
    """Global permuted rows of the rank's y_local: its block rows, then (DB) its border-row slice."""
    r0, nb = info["row_begin"], info["y_local_len"] - info["y_border_len"]
    return np.concatenate([np.arange(r0, r0 + nb), np.arange(info["y_border_begin"],
                                                             info["y_border_begin"] + info["y_border_len"])])


def apply_ranks(hs, infos, xls, split=False, flags=0):
    """One apply per rank, each on its own stream (as on its own GPU).  All
    inputs and outputs are allocated and ready before the first apply, so
    nothing on the host waits between the ranks' applies (a rank's apply
    completes only once its peers have pushed their slices)."""
    streams = [T.rank_stream(h) for h in hs]   # each rank's own hardware queue (spmv_test_rank_stream)
    xds = [xl if torch.is_tensor(xl) else torch.from_numpy(np.ascontiguousarray(xl)).cuda() for xl in xls]
    ys = [torch.full((i["y_local_len"],), float("nan"), dtype=torch.float64, device="cuda") for i in infos]
    torch.cuda.synchronize()
    for h, xd, yd, s in zip(hs, xds, ys, streams):
        (sp.spmv_split_apply if split else sp.spmv_apply)(h, xd, yd, flags, stream=s)
    torch.cuda.synchronize()
    return ys


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name", ["c5s", "c2s"])
def test_sb_ranks_match_single_gpu(name, world):
    p = synth.make(name)
    x = p.x()
    xh, yh_ref, S = oracle_permuted(p, x)
    h1 = create(p, options=dict(kernel="panel"))
    yd1 = torch.empty(p.m, dtype=torch.float64, device="cuda")
    sp.spmv_apply(h1, torch.from_numpy(xh).cuda(), yd1)
    y1 = yd1.cpu().numpy()
    hs, infos = make_ranks(p, world)
    assert all(i["exchange"] == 3 and i["kernel"] == 7 for i in infos)
    for rep in range(3):   # both parities of the double-buffered exchange
        ys = apply_ranks(hs, infos, [x_local(xh, i) for i in infos])
        rows = 0
        for r, (i, yd) in enumerate(zip(infos, ys)):
            rr = y_rows(i)
            yl = yd.cpu().numpy()
            assert np.array_equal(yl.view(np.int64), y1[rr].view(np.int64)), f"rep {rep} rank {r} of {world}"
            assert_parity(yl, yh_ref[rr], S[rr], what=f"{name} rank {r}/{world}")
            rows += len(rr)
        assert rows == p.m
    assert all(sp.spmv_get_info(h)["exchange_timeouts"] == 0 for h in hs)


@pytest.mark.parametrize("world", [2, 4])
def test_sb_ranks_power_steps(world):
    """a9 at world > 1: each rank's fused local max (folded across ranks on the
    host: the test ranks have no communicator), its owner-local x-update
    x^_{t+1}[c] = y^_t[r(c)] / m on the rank's [interior | owned border]
    layout, and the exchange of the new border slices reproduce the
    single-GPU power steps bit for bit."""
    p = synth.make("c5s")
    xh, _, _ = oracle_permuted(p, p.x())
    h1 = create(p, options=dict(kernel="panel"))
    hs, infos = make_ranks(p, world)
    xg = torch.from_numpy(xh).cuda()
    xl = [torch.from_numpy(x_local(xh, i)).cuda() for i in infos]
    for t in range(4):
        y1 = torch.empty(p.m, dtype=torch.float64, device="cuda")
        m1 = torch.empty(1, dtype=torch.float64, device="cuda")
        sp.spmv_apply(h1, xg, y1, sp.SPMV_FUSE_MAXABS)
        sp.spmv_maxabs(h1, m1)
        xg_next = torch.empty_like(xg)
        sp.spmv_normalize(h1, y1, m1, xg_next)
        ys = apply_ranks(hs, infos, xl, flags=sp.SPMV_FUSE_MAXABS)
        ms = []
        for h in hs:
            mr = torch.empty(1, dtype=torch.float64, device="cuda")
            sp.spmv_maxabs(h, mr)
            ms.append(mr)
        mg = torch.max(torch.cat(ms)).reshape(1)
        assert mg.item() == m1.item(), f"step {t}: max over ranks"
        for r, (h, i, yr) in enumerate(zip(hs, infos, ys)):
            assert torch.equal(yr.view(torch.int64), y1[torch.from_numpy(y_rows(i)).cuda()].view(torch.int64))
            xn = torch.empty_like(xl[r])
            sp.spmv_normalize(h, yr, mg, xn)
            ref = torch.from_numpy(x_local(xg_next.cpu().numpy(), i)).cuda()
            assert torch.equal(xn.view(torch.int64), ref.view(torch.int64)), f"step {t} rank {r}: x-update"
            xl[r] = xn
        torch.cuda.synchronize()
        xg = xg_next


# C3's DB structure with K = 8 blocks, small enough that all eight ranks'
# kernels are co-resident on the one GPU of the loopback fake: a rank's CTAs
# spin (bounded) until every peer's slice lands, and on one GPU a peer whose
# kernel cannot get an SM never pushes (full C3 at world 8 has 632 CTAs of
# 1 per SM; on a real run each rank has a GPU of its own).
synth.PRESETS["_c3w8"] = lambda **kw: synth._db(8, 3000, 1000, 10, 16, 0, 4, 10, 20, **kw)


@pytest.mark.parametrize("name,world", [("c3s", 2), ("c3s", 4), ("_c3w8", 8)])
@pytest.mark.parametrize("variant", ["int", "real"])
def test_db_split_across_ranks(name, world, variant):
    """f1: the multiple-SpMxV across GPUs on C3's DB structure (K parts, A13's
    2D block assignment): part k on block k's rank, border-row temporaries
    folded in part order by the row's owner."""
    p = synth.make(name, variant=variant)
    x = p.x()
    y_ref = oracle.split(p.row_ptr, p.col, p.val, p.parts, p.n_parts, x)
    S = oracle.spmv(p.row_ptr, p.col, p.val, x)[1]
    hs, infos = make_ranks(p, world)
    assert all(i["exchange"] == 3 and i["split_kernel"] == 7 for i in infos)
    for rep in range(3):
        ys = apply_ranks(hs, infos, [x_local(x, i) for i in infos], split=True)
        y = np.full(p.m, np.nan)
        for i, yd in zip(infos, ys):
            y[y_rows(i)] = yd.cpu().numpy()
        assert_parity(y, y_ref, S, exact=(variant == "int"), what=f"DB split world {world} rep {rep}")
    # apply on the same handles: the same sum (single SpMxV semantics)
    ys = apply_ranks(hs, infos, [x_local(x, i) for i in infos])
    y = np.full(p.m, np.nan)
    for i, yd in zip(infos, ys):
        y[y_rows(i)] = yd.cpu().numpy()
    assert_parity(y, y_ref, S, exact=(variant == "int"), what="DB apply")
    assert all(sp.spmv_get_info(h)["exchange_timeouts"] == 0 for h in hs)


@pytest.mark.parametrize("world", [2, 4])
def test_db_without_split_across_ranks(world):
    """DB across GPUs without a user split: the library derives the 2D block
    assignment (reading A13) itself; y = A x."""
    p = synth.make("c3s", variant="int")
    x = p.x()
    y_ref, _ = oracle.spmv(p.row_ptr, p.col, p.val, x)
    hs, infos = make_ranks(p, world, parts=False)
    ys = apply_ranks(hs, infos, [x_local(x, i) for i in infos])
    y = np.full(p.m, np.nan)
    for i, yd in zip(infos, ys):
        y[y_rows(i)] = yd.cpu().numpy()
    assert np.array_equal(y, y_ref)


def test_db_power_steps_across_ranks():
    """The power-iteration glue on DB ranks: y_local = [block rows | owned
    border-row slice], x_local = [interior | owned border-column slice] (owner
    aligned for C3), x-update bit for bit against the oracle's."""
    p = synth.make("c3s")
    world = 4
    hs, infos = make_ranks(p, world)
    assert all(i["has_owner_map"] == 1 for i in infos)
    x = p.x()
    xl = [torch.from_numpy(x_local(x, i)).cuda() for i in infos]
    for t in range(3):
        ys = apply_ranks(hs, infos, xl, split=True, flags=sp.SPMV_FUSE_MAXABS)
        xg = np.full(p.n, np.nan)
        for i, xr in zip(infos, xl):
            a, L, b, Lb = i["x_interior_begin"], i["x_interior_len"], i["x_border_begin"], i["x_border_len"]
            v = xr.cpu().numpy()
            xg[a:a + L], xg[b:b + Lb] = v[:L], v[L:]
        y = np.full(p.m, np.nan)
        for i, yd in zip(infos, ys):
            y[y_rows(i)] = yd.cpu().numpy()
        y_ref = oracle.split(p.row_ptr, p.col, p.val, p.parts, p.n_parts, xg)
        S = oracle.spmv(p.row_ptr, p.col, p.val, xg)[1]
        assert_parity(y, y_ref, S, what=f"step {t}")
        ms = []
        for h in hs:
            mr = torch.empty(1, dtype=torch.float64, device="cuda")
            sp.spmv_maxabs(h, mr)
            ms.append(mr)
        mg = torch.max(torch.cat(ms)).reshape(1)
        assert mg.item() == oracle.maxabs(y)
        xref = oracle.scale(y, mg.item())
        for r, (h, i, yr) in enumerate(zip(hs, infos, ys)):
            xn = torch.empty_like(xl[r])
            sp.spmv_normalize(h, yr, mg, xn)
            assert np.array_equal(xn.cpu().numpy(), x_local(xref, i)), f"step {t} rank {r}"
            xl[r] = xn


def test_unlinked_rank_refuses():
    p = synth.make("c5s")
    h = T.test_create_rank(p.m, p.n, p.row_ptr, p.col, p.val, 0, 2, row_perm=p.row_perm, col_perm=p.col_perm,
                           blocks=p.blocks)
    i = sp.spmv_get_info(h)
    x = torch.zeros(i["x_local_len"], dtype=torch.float64, device="cuda")
    y = torch.zeros(i["y_local_len"], dtype=torch.float64, device="cuda")
    with pytest.raises(sp.SpmvError) as e:
        sp.spmv_apply(h, x, y)
    assert e.value.status == sp.SPMV_ERR_USAGE


def test_exchange_overlaps_interior():
    """a4: rank 0's kernel starts at once and runs its interior epochs while
    rank 1's border slice is still to come (rank 1 applies 20 ms late, as a
    slow peer would); once the slice lands, only the border epochs remain.
    Measured with CUDA events: the time rank 0 still needs after rank 1 starts
    pushing is well below rank 0's whole kernel time with every slice ready."""
    # large enough that rank 0's kernel (~0.2 ms) dwarfs the push latency
    synth.PRESETS["_overlap"] = lambda **kw: synth._sb(2, 1_200_000, 1_188_000, 12_000, 12, 20, 0, 3, **kw)
    p = synth.make("_overlap", scramble=0)
    hs, infos = make_ranks(p, 2)
    x = p.x()
    xl = [torch.from_numpy(x_local(x, i)).cuda() for i in infos]
    ys = [torch.empty(i["y_local_len"], dtype=torch.float64, device="cuda") for i in infos]
    s0, s1 = T.rank_stream(hs[0]), T.rank_stream(hs[1])
    ev = lambda: torch.cuda.Event(enable_timing=True)   # noqa: E731

    def both(delay_s):
        a0, b0, e1 = ev(), ev(), ev()
        a0.record(s0)
        sp.spmv_apply(hs[0], xl[0], ys[0], stream=s0)
        b0.record(s0)
        if delay_s:
            time.sleep(delay_s)
        e1.record(s1)
        sp.spmv_apply(hs[1], xl[1], ys[1], stream=s1)
        torch.cuda.synchronize()
        return a0, b0, e1

    for _ in range(3):
        both(0)
    full = []
    for _ in range(5):   # rank 0's kernel with rank 1 right behind (slices land early)
        a0, b0, _ = both(0)
        full.append(a0.elapsed_time(b0))
    t_full = float(np.median(full))
    tails, leads = [], []
    for _ in range(5):
        a0, b0, e1 = both(0.02)
        leads.append(a0.elapsed_time(e1))     # rank 0 was running for this long before rank 1 pushed
        tails.append(e1.elapsed_time(b0))     # what rank 0 still did after rank 1's push began
    t_tail = float(np.median(tails))
    assert min(leads) > 10.0, "rank 1 applied late"
    print(f"overlap: rank 0 kernel {t_full:.3f} ms with slices ready; {t_tail:.3f} ms left after the late "
          f"peer's push began (interior share done early: {1 - t_tail / t_full:.2f})")
    assert t_tail < 0.7 * t_full, (t_tail, t_full)
    assert all(sp.spmv_get_info(h)["exchange_timeouts"] == 0 for h in hs)


def test_peer_gone_is_sticky():
    """A rank whose peer never applies: its kernel's device-side wait for the
    border slice gives up after a bound (no hang), counts the timeout, and
    the handle's next apply fails with SPMV_ERR_INTERNAL instead of
    returning results computed from a stale border."""
    p = synth.make("c5s", scramble=0)
    hs, infos = make_ranks(p, 2)
    x0 = torch.from_numpy(x_local(p.x(), infos[0])).cuda()
    y0 = torch.empty(infos[0]["y_local_len"], dtype=torch.float64, device="cuda")
    s0 = T.rank_stream(hs[0])
    t0 = time.time()
    sp.spmv_apply(hs[0], x0, y0, stream=s0)     # rank 1 never pushes its slice
    torch.cuda.synchronize()
    assert time.time() - t0 < 120
    assert sp.spmv_get_info(hs[0])["exchange_timeouts"] > 0
    with pytest.raises(sp.SpmvError) as e:
        sp.spmv_apply(hs[0], x0, y0, stream=s0)
    assert e.value.status == sp.SPMV_ERR_INTERNAL

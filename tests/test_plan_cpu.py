"""Host-only checks of the column-sorted panel planner (plan_panel.cpp): the
packed groups decode back to the permuted CSR bit for bit, with the format's
invariants (distinct rows per epoch, groups on one side of the border split,
border groups last, every panel within 227 KB of shared memory), and the SB
plan does not depend on the GPU count.  The kernel itself is checked on the
GPU (tests/test_gpu_*.py)."""
import numpy as np
import pytest

import paper_1203_2739_b200 as sp
import paper_1203_2739_b200.testing as T
import synth


def _random_sb(seed, K, rows, cols, border, dens_int, dens_b):
    """SB form with uneven, odd-sized blocks (chunk starts at odd columns)."""
    rng = np.random.default_rng(seed)
    rb = np.concatenate([[0], np.cumsum(rows)])
    cb = np.concatenate([[0], np.cumsum(cols)])
    m, nint = int(rb[-1]), int(cb[-1])
    n = nint + border
    rp = [0]
    col, val = [], []
    for k in range(K):
        for r in range(rb[k], rb[k + 1]):
            ci = np.flatnonzero(rng.random(cols[k]) < dens_int) + cb[k]
            cbo = np.flatnonzero(rng.random(border) < dens_b) + nint if border else np.array([], dtype=np.int64)
            c = np.concatenate([ci, cbo]).astype(np.int32)
            col.append(c)
            val.append(rng.standard_normal(len(c)))
            rp.append(rp[-1] + len(c))
    blocks = {"kind": 1, "K": K, "row_block_ptr": np.array(list(rb) + [m], dtype=np.int64),
              "col_block_ptr": np.array(list(cb) + [n], dtype=np.int64)}
    return m, n, np.array(rp, dtype=np.int64), np.concatenate(col), np.concatenate(val), blocks


# ---------------------------------------------------------------- panel planner
def _c5_like(K=2, rows=60_000, cols=58_800, border=1_200, seed=0):
    synth.PRESETS["_c5like"] = lambda **kw: synth._sb(K, rows, cols, border // K, 12, 20, 0, 3, **kw)
    return synth.make("_c5like", scramble=0, seed=seed)


@pytest.mark.parametrize("target", [30_000, 7_000])
def test_panel_plan_round_trip_c5_like(target):
    p = _c5_like()
    st = T.pn_plan_check(p.m, p.n, p.row_ptr, p.col, p.val, p.blocks, target)
    assert st["entries"] == p.nnz
    assert st["epochs"] * 64 == st["groups"]
    # big panels: little padding, few deferred nonzeros (the kernel's premise)
    if target == 30_000:
        assert st["pads"] < 0.05 * 32 * st["groups"]
        assert st["deferred"] < 0.1 * p.nnz


@pytest.mark.parametrize("name,target", [("c5s", 2000), ("c2s", 300), ("c4s", 5000)])
def test_panel_plan_round_trip_small(name, target):
    # small panels pad heavily (the library then keeps the row-tile kernel),
    # but the round trip must still be exact; c4s has rows of up to 3,000 nonzeros
    p = synth.make(name) if name == "c4s" else synth.make(name, scramble=0)
    st = T.pn_plan_check(p.m, p.n, p.row_ptr, p.col, p.val, p.blocks if name != "c4s" else None, target)
    assert st["entries"] == p.nnz


def test_panel_plan_random_sb_odd_blocks():
    m, n, rp, col, val, blocks = _random_sb(7, 4, [37, 600, 1201, 90], [1, 2047, 2049, 5001], 333, 0.01, 0.01)
    st = T.pn_plan_check(m, n, rp, col, val, blocks, 400)
    assert st["entries"] == len(col)


@pytest.mark.parametrize("world,rank", [(2, 0), (2, 1), (4, 3)])
def test_panel_plan_rank_local_layout(world, rank):
    """A rank's shard at world > 1: rows of its SB blocks, columns in the local
    layout [interior columns | full C_B] (host.cpp), border columns read from
    the exchange buffer -- so no group may mix the two sides (x_split = C_B's
    local start).  Built from the scrambled C5 stand-in through the shard plan."""
    p = synth.make("c5s")
    sh = sp.spmv_shard_plan(p.blocks, p.m, p.n, rank, world)
    rp_g, col_g, val_g = synth_permuted(p)
    r0, r1 = sh["row_begin"], sh["row_end"]
    q0, nint, b0 = sh["x_interior_begin"], sh["x_interior_len"], sh["border_begin"]
    a, b = int(rp_g[r0]), int(rp_g[r1])
    rp = rp_g[r0:r1 + 1] - a
    c = col_g[a:b].astype(np.int64)
    loc = np.where(c >= b0, nint + (c - b0), c - q0).astype(np.int32)
    assert loc.min() >= 0 and loc.max() < nint + sh["border_total"]
    k0, k1 = sh["block_begin"], sh["block_end"]
    rbp, cbp = p.blocks["row_block_ptr"], p.blocks["col_block_ptr"]
    K = k1 - k0
    blocks = {"kind": 1, "K": K,
              "row_block_ptr": np.array([rbp[k] - r0 for k in range(k0, k1 + 1)] + [r1 - r0], dtype=np.int64),
              "col_block_ptr": np.array([cbp[k] - q0 for k in range(k0, k1 + 1)] + [nint + sh["border_total"]],
                                        dtype=np.int64)}
    st = T.pn_plan_check(r1 - r0, nint + sh["border_total"], rp, loc, val_g[a:b], blocks, 1500)
    assert st["entries"] == b - a


def synth_permuted(p):
    import oracle
    rp, col, val, _ = oracle.permute(p.m, p.n, p.row_ptr, p.col, p.val, p.row_perm, p.col_perm)
    return rp, col, val


@pytest.mark.parametrize("name", ["c5s", "c2s"])
def test_panel_plan_independent_of_gpu_count(name):
    """every rank plans its SB blocks' panels from the global
    per-block slot counts, in its own x layout, so each block's panels and
    every row's summation order (hash of each group's rows, virtual rows,
    global columns and values in issue order) are the same at world 1, 2, 4
    -- y is then bit-identical across GPU counts."""
    p = synth.make(name, scramble=0)
    K = p.blocks["K"]
    ref = T.pn_shard_hash(p.m, p.n, p.row_ptr, p.col, p.val, p.blocks, 1)[0]
    assert np.all(ref != 0)
    for world in (2, 4):
        h = T.pn_shard_hash(p.m, p.n, p.row_ptr, p.col, p.val, p.blocks, world)
        owned = (h != 0).sum(axis=0)
        assert np.all(owned == 1), f"each block on exactly one rank (world {world})"
        assert np.array_equal(h.sum(axis=0), ref), f"world {world} plans differ from world 1"
    # the hash has teeth: another whole-wave count cuts other panels
    other = T.pn_shard_hash(p.m, p.n, p.row_ptr, p.col, p.val, p.blocks, 1, sms=1)[0]
    assert not np.array_equal(other, ref)


def test_panel_smem_cap_split_rows():
    """rows of 33-64 nonzeros become two virtual rows, and a
    split row also costs 2 B per slot and 12 B per row of fold lists, so a
    panel of ~16 K slots can exceed 227 KB; the planner must cut panels by
    shared-memory bytes, whatever the slot target."""
    rng = np.random.default_rng(11)
    m = n = 40_000
    L = 40
    col = np.concatenate([np.sort(rng.choice(n, L, replace=False)) for _ in range(m)]).astype(np.int32)
    rp = np.arange(0, (m + 1) * L, L, dtype=np.int64)
    val = rng.uniform(-1, 1, m * L)
    st = T.pn_plan_check(m, n, rp, col, val, None, 16384)
    assert st["entries"] == m * L
    assert st["smem_max"] <= 227 * 1024


def test_border_groups_last():
    """Columns of C_B (Eq.(1)) come after every interior column in each panel,
    so the border groups form the panel's last epochs (the world > 1 exchange
    overlaps the interior epochs); the check itself runs in pn_plan_check."""
    p = _c5_like()
    st = T.pn_plan_check(p.m, p.n, p.row_ptr, p.col, p.val, p.blocks, 7_000)
    assert st["panels_with_border"] == st["panels"]


@pytest.mark.parametrize("name", ["c4s", "c3s"])
def test_far_stream_takes_the_drain(name):
    """Nonzeros still deferred when a panel's sweep ends go to the far stream
    (panel.cu's barrier-free phase) instead of near-empty epochs: no drain
    padding, and the round trip (runs owned by one lane each, flagged at their
    last entry, every nonzero once) holds."""
    p = synth.make(name)
    blocks = p.blocks if name != "c4s" else None
    st = T.pn_plan_check(p.m, p.n, p.row_ptr, p.col, p.val, blocks, 5000)
    assert st["far"] > 0, st
    assert st["pads_drain"] == 0 and st["epochs_drain"] == 0, st
    assert st["entries"] == p.nnz


def test_far_stream_heavy_column_runs():
    """A panel whose rows all repeat one dense column window (every row's
    nonzeros within 40 columns): deferrals pile up, the far stream carries
    long runs, and the plan still round-trips bit for bit."""
    rng = np.random.default_rng(5)
    m = n = 3000
    rows, cols = [], []
    for r in range(m):
        c0 = (r * 7) % (n - 40)
        cs = np.sort(rng.choice(40, size=30, replace=False)) + c0
        rows += [r] * len(cs)
        cols += cs.tolist()
    rp = np.zeros(m + 1, np.int64)
    np.add.at(rp, np.asarray(rows) + 1, 1)
    rp = np.cumsum(rp)
    col = np.asarray(cols, np.int32)
    val = rng.uniform(-1, 1, len(col))
    st = T.pn_plan_check(m, n, rp, col, val, None, 1024)
    assert st["entries"] == len(col) and st["pads_drain"] == 0, st


def test_bank_colouring_lowers_predicted_y_wavefronts():
    """The y-slot colouring (plan_panel.cpp colour_slots, directed bank swaps):
    on C5-like panels (12-20 nonzeros per row, columns random inside the
    block) the predicted wavefronts of a warp-wide 64-bit y access must fall
    well below the slot = row layout's (4.84 -> 3.75 at the
    production panel size); both are at least 2 (two half-warps)."""
    p = _c5_like()
    st = T.pn_plan_check(p.m, p.n, p.row_ptr, p.col, p.val, p.blocks, 16384)
    nat, colr = st["y_wavefronts_natural"], st["y_wavefronts_coloured"]
    assert 2.0 <= colr < nat
    assert colr <= nat - 0.8, (nat, colr)
    assert colr <= 3.9, colr

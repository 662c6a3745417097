"""Pins of oracle.sbfs (the sBFS ordering of P:L134 and the
SB extraction of reading R5) against things other than itself: the hand-
derived worked example, scipy's breadth-first order on the bipartite graph,
closed forms (tridiagonal -> identity, block-diagonal components), and the
SB envelope of Eq.(1) checked directly on the permuted matrix."""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sps
from scipy.sparse.csgraph import breadth_first_order

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))


def _rand_csr(m, n, per_row, seed, shuffle=True):
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(m):
        k = int(rng.integers(0, per_row + 1))
        c = rng.choice(n, size=min(k, n), replace=False).astype(np.int32)
        if not shuffle:
            c.sort()
        rows.append(c)
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    col = np.concatenate(rows) if rows else np.zeros(0, np.int32)
    return rp, col.astype(np.int32)


def _scipy_bfs(m, n, rp, col):
    """BFS numbers from scipy on B = [[0, A], [A^T, 0]] (sorted indices, so a
    vertex's neighbours are visited in ascending number), restarted from the
    lowest unvisited row while any row is unvisited; untouched columns last."""
    A = sps.csr_matrix((np.ones(len(col)), col, rp), shape=(m, n))
    A.sum_duplicates()
    B = sps.bmat([[None, A], [A.T, None]], format="csr")
    B.sort_indices()
    bfs_row = -np.ones(m, np.int64)
    bfs_col = -np.ones(n, np.int64)
    nr = nc = 0
    while (bfs_row < 0).any():
        root = int(np.flatnonzero(bfs_row < 0)[0])
        order = breadth_first_order(B, root, directed=False, return_predecessors=False)
        for v in order:
            if v < m:
                assert bfs_row[v] < 0
                bfs_row[v] = nr
                nr += 1
            else:
                assert bfs_col[v - m] < 0
                bfs_col[v - m] = nc
                nc += 1
    for j in range(n):
        if bfs_col[j] < 0:
            bfs_col[j] = nc
            nc += 1
    return bfs_row, bfs_col


def _check_sb(m, n, rp, col, K, o):
    """Eq.(1): every entry of row block k lies in C_k or C_B; the extraction
    rule of reading R5 (nonzero-prefix blocks, minimal border) holds."""
    rperm, cperm = o["row_perm"], o["col_perm"]
    assert np.array_equal(np.sort(rperm), np.arange(m)) and np.array_equal(np.sort(cperm), np.arange(n))
    rbp, cbp = o["row_block_ptr"], o["col_block_ptr"]
    assert rbp[0] == 0 and rbp[K] == m and rbp[K + 1] == m and np.all(np.diff(rbp) >= 0)
    assert cbp[0] == 0 and cbp[K + 1] == n and np.all(np.diff(cbp) >= 0)
    blk_of_new_row = np.searchsorted(rbp[1:K + 1], np.arange(m), side="right")
    blocks_of_col = [set() for _ in range(n)]
    lens = np.diff(rp)
    nnz = int(rp[-1])
    # nonzero-prefix block rule, computed independently from the new row order
    new_len = np.empty(m, np.int64)
    new_len[rperm] = lens
    P = np.concatenate([[0], np.cumsum(new_len)[:-1]])
    want = np.minimum(K - 1, (K * P) // max(nnz, 1)) if nnz else np.minimum(K - 1, (K * np.arange(m)) // max(m, 1))
    assert np.array_equal(blk_of_new_row, want)
    for i in range(m):
        b = blk_of_new_row[rperm[i]]
        for j in col[rp[i]:rp[i + 1]]:
            blocks_of_col[j].add(int(b))
            q = cperm[j]
            assert (cbp[b] <= q < cbp[b + 1]) or q >= cbp[K], "entry outside the SB envelope"
    for j in range(n):
        q = cperm[j]
        if q >= cbp[K]:
            assert len(blocks_of_col[j]) != 1, "a border column touched by one block only"
        else:
            k = int(np.searchsorted(cbp[1:K + 1], q, side="right"))
            assert blocks_of_col[j] == {k}


def test_worked_example(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "sbfs_6x6.json")))
    o = oracle.sbfs(g["m"], g["n"], np.array(g["row_ptr"]), np.array(g["col"]), g["K"])
    for k in ("bfs_row", "bfs_col", "row_perm", "col_perm", "row_block_ptr", "col_block_ptr"):
        assert o[k].tolist() == g[k], k


@pytest.mark.parametrize("m,n,per_row,seed", [(300, 250, 6, 0), (200, 400, 3, 1), (500, 500, 2, 2),
                                              (50, 60, 1, 3)])
def test_bfs_matches_scipy(m, n, per_row, seed):
    rp, col = _rand_csr(m, n, per_row, seed)
    o = oracle.sbfs(m, n, rp, col, 4)
    br, bc = _scipy_bfs(m, n, rp, col)
    assert np.array_equal(o["bfs_row"], br)
    assert np.array_equal(o["bfs_col"], bc)


@pytest.mark.parametrize("K", [1, 2, 3, 7])
@pytest.mark.parametrize("seed", [0, 1])
def test_sb_envelope(K, seed):
    m, n = 400, 350
    rp, col = _rand_csr(m, n, 5, seed)
    o = oracle.sbfs(m, n, rp, col, K)
    _check_sb(m, n, rp, col, K, o)


def test_tridiagonal_is_identity():
    m = 50
    rows = [[j for j in (i - 1, i, i + 1) if 0 <= j < m] for i in range(m)]
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    col = np.array([j for r in rows for j in r], np.int32)
    o = oracle.sbfs(m, m, rp, col, 1)
    assert np.array_equal(o["bfs_row"], np.arange(m)) and np.array_equal(o["bfs_col"], np.arange(m))
    assert o["col_block_ptr"].tolist() == [0, m, m]          # K = 1: no border


def test_components_and_empty():
    """Two disconnected diagonal blocks given interleaved (rows 0,2,4 x cols
    0,2 and rows 1,3 x cols 1,3), an empty row, an untouched column: the
    BFS restarts from the lowest unvisited row, the empty row is its own
    component, the untouched column comes last; with K = 2 the blocks are
    recovered with an empty border (plus the untouched column)."""
    A = np.zeros((6, 5))
    for i in (0, 2, 4):
        for j in (0, 2):
            A[i, j] = 1
    for i in (1, 3):
        for j in (1, 3):
            A[i, j] = 1
    S = sps.csr_matrix(A)
    rp, col = S.indptr.astype(np.int64), S.indices.astype(np.int32)
    o = oracle.sbfs(6, 5, rp, col, 2)
    assert o["bfs_row"].tolist() == [0, 3, 1, 4, 2, 5]
    assert o["bfs_col"].tolist() == [0, 2, 1, 3, 4]
    _check_sb(6, 5, rp, col, 2, o)
    # block 0 = rows {0,2,4} (6 of 10 nonzeros), block 1 = rows {1,3} + the empty row 5
    assert o["row_block_ptr"].tolist() == [0, 3, 6, 6]
    assert o["col_block_ptr"].tolist() == [0, 2, 4, 5]


def test_unsorted_rows_same_as_sorted():
    m, n = 200, 180
    rp, col = _rand_csr(m, n, 6, 5, shuffle=True)
    cs = col.copy()
    for i in range(m):
        cs[rp[i]:rp[i + 1]].sort()
    a, b = oracle.sbfs(m, n, rp, col, 3), oracle.sbfs(m, n, rp, cs, 3)
    for k in a:
        assert np.array_equal(a[k], b[k])

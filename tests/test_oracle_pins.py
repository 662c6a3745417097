"""Pins for the CPU oracle (-m "not gpu").

Each test ties an oracle routine to something other than itself: hand
arithmetic (golden), brute-force dense matvec, closed forms, exact integer /
dyadic arithmetic, an independent library (scipy.sparse), or the generator's
own construction (closed loop).  A dropped term, wrong sign/index or
transposed operand in oracle.c fails at least one of them.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth


# ---------------------------------------------------------------- helpers ---
def dense_of(m, n, row_ptr, col, val):
    A = np.zeros((m, n))
    for i in range(m):
        for t in range(row_ptr[i], row_ptr[i + 1]):
            A[i, col[t]] = val[t]
    return A


def dense_matvec_serial(A, x):
    """Brute force: y_i = sum_j a_ij x_j in ascending j, one rounding per op,
    skipping structural zeros (CSR order for sorted rows)."""
    m, n = A.shape
    y = np.zeros(m)
    for i in range(m):
        s = 0.0
        for j in range(n):
            if A[i, j] != 0.0:
                s = s + float(A[i, j]) * float(x[j])
        y[i] = s
    return y


def perm_matrix(p):
    """(P)_{new,old} = 1 for an old->new array p."""
    P = np.zeros((len(p), len(p)))
    P[np.asarray(p), np.arange(len(p))] = 1.0
    return P


# ------------------------------------------------------ golden worked ex. ---
@pytest.fixture(scope="module")
def W(golden_dir):
    with open(os.path.join(golden_dir, "worked_example_6x6.json")) as f:
        return json.load(f)


def test_worked_example_permute(W):
    rp, c, v, _ = oracle.permute(6, 6, W["orig_row_ptr"], W["orig_col"], np.array(W["orig_val"], float),
                                 W["row_perm"], W["col_perm"])
    assert rp.tolist() == W["perm_row_ptr"]
    assert c.tolist() == W["perm_col"]
    assert v.tolist() == W["perm_val"]
    assert oracle.permute_x(W["col_perm"], np.array(W["x"], float)).tolist() == W["xhat"]


def test_worked_example_spmv(W):
    yh, S = oracle.spmv(W["perm_row_ptr"], W["perm_col"], np.array(W["perm_val"], float),
                        np.array(W["xhat"], float))
    assert yh.tolist() == W["yhat"]
    y, _ = oracle.spmv(W["orig_row_ptr"], W["orig_col"], np.array(W["orig_val"], float),
                       np.array(W["x"], float))
    assert y.tolist() == W["y"]
    assert oracle.unpermute_y(W["row_perm"], yh).tolist() == W["y"]
    assert S.tolist() == W["yhat"]          # all products positive here


def test_worked_example_split(W):
    rp, c, v = W["orig_row_ptr"], W["orig_col"], np.array(W["orig_val"], float)
    parts = np.array(W["part_of_nnz"], np.int32)
    x = np.array(W["x"], float)
    y = oracle.split(rp, c, v, parts, 2, x)
    assert y.tolist() == W["y"]
    # single parts via a K=2 split where the other part is masked to part ids only
    y0 = oracle.split(rp, c, v * (parts == 0), parts, 2, x)
    y1 = oracle.split(rp, c, v * (parts == 1), parts, 2, x)
    assert y0.tolist() == W["y_part0"]
    assert y1.tolist() == W["y_part1"]
    lr, lc = oracle.split_lambda(6, 6, rp, c, parts, 2)
    assert (lr, lc) == (W["sum_lambda_r_split"], W["sum_lambda_c_split"])
    assert lr + lc == W["corollary4_bound"]


def test_worked_example_sb_lambda(W):
    rb = np.repeat(np.arange(2, dtype=np.int32), 3)
    s, lam = oracle.sb_lambda(6, 6, W["perm_row_ptr"], W["perm_col"], rb)
    assert s == W["sum_lambda_c_SB"]
    assert lam.tolist() == [1, 1, 1, 1, 2, 2]


# --------------------------------------------------------- hand examples ---
def test_spec_hand_examples():
    # [[1,2],[0,3]] . [1,1] = [3,3]
    y, _ = oracle.spmv([0, 2, 3], [0, 1, 1], np.array([1.0, 2.0, 3.0]), np.array([1.0, 1.0]))
    assert y.tolist() == [3.0, 3.0]
    # single nonzero 2 at (3,7), x[7] = 4 -> y[3] = 8, all else 0
    rp = [0, 0, 0, 0, 1, 1]
    x = np.zeros(8); x[7] = 4.0
    y, S = oracle.spmv(rp, [7], np.array([2.0]), x)
    assert y.tolist() == [0, 0, 0, 8, 0]
    assert S.tolist() == [0, 0, 0, 8, 0]
    # 2x2 antidiagonal with a row swap -> diagonal
    rp2, c2, v2, _ = oracle.permute(2, 2, [0, 1, 2], [1, 0], np.array([5.0, 7.0]), [1, 0], None)
    assert rp2.tolist() == [0, 1, 2] and c2.tolist() == [0, 1] and v2.tolist() == [7.0, 5.0]


def test_closed_forms():
    rng = np.random.default_rng(3)
    n = 50
    x = rng.uniform(-1, 1, n)
    # identity -> y = x bitwise
    y, _ = oracle.spmv(np.arange(n + 1), np.arange(n), np.ones(n), x)
    assert np.array_equal(y, x)
    # diagonal -> y_i = d_i x_i bitwise
    d = rng.uniform(-1, 1, n)
    y, _ = oracle.spmv(np.arange(n + 1), np.arange(n), d, x)
    assert np.array_equal(y, d * x)
    # permutation matrix -> gather
    p = rng.permutation(n)
    y, _ = oracle.spmv(np.arange(n + 1), p, np.ones(n), x)
    assert np.array_equal(y, x[p])
    # rank-1 u v^T with dyadic entries: exact closed form y = u (v . x)
    u = np.round(rng.uniform(-1, 1, 20) * 64) / 64
    v = np.round(rng.uniform(-1, 1, 30) * 64) / 64
    xs = np.round(rng.uniform(-1, 1, 30) * 64) / 64
    rp = np.arange(21) * 30
    col = np.tile(np.arange(30), 20)
    val = np.outer(u, v).ravel()
    y, _ = oracle.spmv(rp, col, val, xs)
    assert np.array_equal(y, u * float(np.dot(v, xs)))


# --------------------------------------------------------- brute force ---
@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("variant", ["real", "int"])
def test_brute_force_dense(seed, variant):
    rng = np.random.default_rng(seed)
    m, n = int(rng.integers(1, 64)), int(rng.integers(1, 64))
    rp, col, val = synth.random_csr(m, n, 0.2, variant=variant, rng=rng, empty_rows=0.1)
    x = rng.uniform(-1, 1, n) if variant == "real" else rng.integers(-4, 5, n).astype(float)
    y, S = oracle.spmv(rp, col, val, x)
    A = dense_of(m, n, rp, col, val)
    assert np.array_equal(y, dense_matvec_serial(A, x))          # same order -> bitwise
    assert np.array_equal(S, dense_matvec_serial(np.abs(A), np.abs(x)))


def test_permute_vs_dense_permutation_matrices():
    """A^ = P_r A P_c^T with (P)_{new,old} = 1 (reading A1)."""
    rng = np.random.default_rng(7)
    for m, n in [(6, 6), (17, 23), (40, 31)]:
        rp, col, val = synth.random_csr(m, n, 0.3, rng=rng)
        pr, pc = rng.permutation(m).astype(np.int32), rng.permutation(n).astype(np.int32)
        o = oracle.permute(m, n, rp, col, val, pr, pc)
        A = dense_of(m, n, rp, col, val)
        Ah = perm_matrix(pr) @ A @ perm_matrix(pc).T
        assert np.array_equal(dense_of(m, n, o[0], o[1], o[2]), Ah)
        # rows sorted by new column
        for i in range(m):
            assert np.all(np.diff(o[1][o[0][i]:o[0][i + 1]]) > 0)
        # permutation invariance y^ = P_r (A x) with x^ = P_c x; integer data -> exact
        x = rng.integers(-4, 5, n).astype(float)
        vi = np.round(val * 8)
        yh, _ = oracle.spmv(o[0], o[1], np.round(o[2] * 8), oracle.permute_x(pc, x))
        y, _ = oracle.spmv(rp, col, vi, x)
        assert np.array_equal(oracle.unpermute_y(pr, yh), y)


def test_scipy_independent_library():
    import scipy.sparse as sp
    for name in ["c1", "c2s", "c4s"]:
        p = synth.make(name)
        x = p.x()
        y, S = oracle.spmv(p.row_ptr, p.col, p.val, x)
        A = sp.csr_matrix((p.val, p.col, p.row_ptr), shape=(p.m, p.n))
        bad, worst, _ = oracle.check(A @ x, y, S)
        assert bad == 0, (name, worst)


# ------------------------------------------------- generator closed loop ---
@pytest.mark.parametrize("name", ["c2s", "c5s"])
def test_closed_loop_unscramble(name):
    """The generator builds the SB CSR, then hides it under a permutation;
    the oracle's permuter must reproduce the pre-scramble form bit-exactly."""
    hidden = synth.make(name, scramble=1)
    plain = synth.make(name, scramble=0)
    o = oracle.permute(hidden.m, hidden.n, hidden.row_ptr, hidden.col, hidden.val,
                       hidden.row_perm, hidden.col_perm)
    assert np.array_equal(o[0], plain.row_ptr)
    assert np.array_equal(o[1], plain.col)
    assert np.array_equal(o[2].view(np.int64), plain.val.view(np.int64))
    # SB envelope (Eq.(1)): every nonzero of block k lies in C_k or C_B
    rbp, cbp = plain.blocks["row_block_ptr"], plain.blocks["col_block_ptr"]
    K = plain.blocks["K"]
    rows_blk = np.repeat(np.arange(K), np.diff(rbp[:K + 1]))
    cblk = np.searchsorted(cbp, plain.col, side="right") - 1
    rblk = np.repeat(rows_blk, np.diff(plain.row_ptr))
    assert np.all((cblk == rblk) | (cblk == K))


def test_owner_map_update_is_local():
    """Reading A17/A18: x^_{t+1}[c] = y^_t[r(c)]/m equals the original-space
    update x_{t+1}[j] = y_t[j]/m, bitwise, and r(c) lies in c's owner block."""
    p = synth.make("c5s", scramble=1)
    x = p.x()
    y, _ = oracle.spmv(p.row_ptr, p.col, p.val, x)
    mt = oracle.maxabs(y)
    xn = oracle.scale(y, mt)
    o = oracle.permute(p.m, p.n, p.row_ptr, p.col, p.val, p.row_perm, p.col_perm)
    yh, _ = oracle.spmv(o[0], o[1], o[2], oracle.permute_x(p.col_perm, x))
    assert np.array_equal(oracle.unpermute_y(p.row_perm, yh), y) or oracle.check(
        oracle.unpermute_y(p.row_perm, yh), y, oracle.spmv(p.row_ptr, p.col, p.val, x)[1])[0] == 0
    xh_next = yh[p.owner] / oracle.maxabs(yh)
    assert np.array_equal(oracle.permute_x(p.col_perm, oracle.scale(oracle.unpermute_y(p.row_perm, yh),
                                                                    oracle.maxabs(yh))), xh_next)
    Rb = p.params["Rb"]; Ci = p.params["Ci"]; Bs = p.params["Bs"]; K = p.params["K"]
    c = np.arange(p.n)
    blk_c = np.where(c < K * Ci, c // Ci, (c - K * Ci) // Bs)
    assert np.array_equal(p.owner // Rb, blk_c)
    assert np.array_equal(np.sort(p.owner), np.arange(p.m))
    del xn


# ----------------------------------------------------------------- split ---
@pytest.mark.parametrize("variant", ["int", "dyadic", "real"])
def test_split_equals_single(variant):
    """Sum_k A^k x = A x: bitwise on integer/dyadic data."""
    p = synth.make("c3s", variant=variant)
    x = p.x()
    ys = oracle.split(p.row_ptr, p.col, p.val, p.parts, p.n_parts, x)
    y, S = oracle.spmv(p.row_ptr, p.col, p.val, x)
    if variant == "real":
        assert oracle.check(ys, y, S)[0] == 0
    else:
        assert np.array_equal(ys, y)


def test_split_k1_and_columns():
    rng = np.random.default_rng(11)
    rp, col, val = synth.random_csr(60, 60, 0.1, rng=rng)
    x = rng.uniform(-1, 1, 60)
    y, S = oracle.spmv(rp, col, val, x)
    assert np.array_equal(oracle.split(rp, col, val, np.zeros(len(col), np.int32), 1, x), y)
    # 2x2 dense split by columns is exact
    ys = oracle.split([0, 2, 4], [0, 1, 0, 1], np.array([1.0, 2.0, 3.0, 4.0]),
                      np.array([0, 1, 0, 1], np.int32), 2, np.array([0.5, 0.25]))
    assert ys.tolist() == [1.0, 2.5]
    # random 4-way split within tolerance, and literal per-part check
    parts = rng.integers(0, 4, len(col)).astype(np.int32)
    ys = oracle.split(rp, col, val, parts, 4, x)
    assert oracle.check(ys, y, S)[0] == 0
    yk = sum(dense_of(60, 60, rp, col, val * (parts == k)) @ x for k in range(4))
    assert oracle.check(ys, yk, S)[0] == 0
    with pytest.raises(ValueError):
        oracle.split(rp, col, val, parts + 4, 4, x)


def test_split_lambda_bruteforce():
    p = synth.make("c3s")
    lr, lc = oracle.split_lambda(p.m, p.n, p.row_ptr, p.col, p.parts, p.n_parts)
    rows = np.repeat(np.arange(p.m), np.diff(p.row_ptr))
    assert lr == len(set(zip(rows.tolist(), p.parts.tolist())))
    assert lc == len(set(zip(p.col.tolist(), p.parts.tolist())))


# -------------------------------------------------- validation / compare ---
def test_validation():
    assert oracle.validate_csr(2, 3, [0, 1, 2], [0, 2]) == 0
    assert oracle.validate_csr(2, 3, [0, 2, 1], [0, 2]) == 1
    assert oracle.validate_csr(2, 3, [1, 1, 2], [0, 2]) == 1
    assert oracle.validate_csr(2, 3, [0, 1, 2], [0, 3]) == 2
    assert oracle.validate_csr(2, 3, [0, 1, 2], [0, -1]) == 2
    assert oracle.validate_csr(1, 3, [0, 2], [1, 1]) == 3
    assert oracle.validate_csr(2, 3, [0, 1, 2], [1, 1]) == 0      # same column, different rows
    assert oracle.validate_perm([2, 0, 1]) == 0
    assert oracle.validate_perm([2, 0, 2]) == 1
    assert oracle.validate_perm([3, 0, 1]) == 1


def test_comparator():
    S = np.array([1.0, 0.0, 2.0, 1.0])
    yref = np.array([1.0, 0.0, 5.0, 1.0])
    ok = np.array([1.0 + 2.0**-41, -0.0, 5.0 - 2.0**-41, 1.0])   # well inside 1e-12*S
    assert oracle.check(ok, yref, S)[0] == 0
    # an exact tie |d| == tol*S passes, one ulp beyond fails
    assert oracle.check(np.array([1.25]), np.array([1.0]), np.array([1.0]), tol=0.25)[0] == 0
    assert oracle.check(np.array([np.nextafter(1.25, 2)]), np.array([1.0]), np.array([1.0]), tol=0.25)[0] == 1
    assert oracle.check(np.array([1.0 + 3e-12, 0.0, 5.0, 1.0]), yref, S)[:3:2] == (1, 0)
    assert oracle.check(np.array([1.0, 1e-300, 5.0, 1.0]), yref, S)[0] == 1     # S = 0 needs +-0
    assert oracle.check(np.array([1.0, 0.0, 5.0, np.nan]), yref, S)[2] == 3
    assert oracle.check(np.array([1.0, 0.0, np.inf, 1.0]), yref, S)[0] == 1


# ------------------------------------------------------- power iteration ---
def test_power_iteration_closed_forms():
    # diag(d): x_t -> e_argmax|d| (up to sign), m_t -> max|d|
    d = np.array([0.5, -2.0, 1.0, 0.25])
    x = np.ones(4)
    for _ in range(60):
        y, _ = oracle.spmv(np.arange(5), np.arange(4), d, x)
        mt = oracle.maxabs(y)
        x = oracle.scale(y, mt)
    assert mt == 2.0 and np.allclose(np.abs(x), [0, 1, 0, 0], atol=1e-15)
    # cyclic permutation: x_{t+1} = shift(x_t)/||x_t||_inf
    x0 = np.array([0.5, -1.0, 0.25, 0.75, -0.5])
    col = np.array([1, 2, 3, 4, 0], np.int32)
    y, _ = oracle.spmv(np.arange(6), col, np.ones(5), x0)
    assert oracle.maxabs(y) == np.max(np.abs(x0))
    assert np.array_equal(oracle.scale(y, oracle.maxabs(y)), x0[col] / 1.0)
    assert np.array_equal(oracle.scale(np.array([3.0, -6.0]), 6.0), np.array([0.5, -1.0]))


def test_generator_thread_independence(tmp_path):
    import subprocess, sys
    code = ("import synth,hashlib;p=synth.make('c4s');"
            "print(hashlib.sha1(p.row_ptr.tobytes()+p.col.tobytes()+p.val.tobytes()).hexdigest())")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for nt in ("1", "4"):
        env = dict(os.environ, OMP_NUM_THREADS=nt, PYTHONPATH=root)
        outs.append(subprocess.check_output([sys.executable, "-c", code], env=env, cwd=root).strip())
    assert outs[0] == outs[1]


# ------------------------------------------------------ sampled-row oracle ---
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_spmv_rows_pinned_to_brute_force(seed):
    """oracle_spmv_rows (the bench's full-size sampled parity, VERDICT r1:
    unpinned) against the brute-force dense matvec, bitwise, on row subsets
    with empty rows, repeated and unsorted row ids; S against |a_ij x_j|
    summed by brute force."""
    rng = np.random.default_rng(seed)
    m, n = 40, 33
    lens = rng.integers(0, 9, m)
    lens[[3, 17, 29]] = 0                                   # empty rows
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    col = np.concatenate([np.sort(rng.choice(n, L, replace=False)) for L in lens]).astype(np.int32)
    val = rng.uniform(-1, 1, int(rp[-1]))
    x = rng.uniform(-1, 1, n)
    A = dense_of(m, n, rp, col, val)
    y_bf = dense_matvec_serial(A, x)
    S_bf = dense_matvec_serial(np.abs(A), np.abs(x))
    rows = np.concatenate([rng.permutation(m)[:25], [3, 3, 17, 0, m - 1]]).astype(np.int64)
    y, S = oracle.spmv_rows(rows, rp, col, val, x)
    assert np.array_equal(y.view(np.int64), y_bf[rows].view(np.int64))
    assert np.array_equal(S, S_bf[rows])
    assert np.all(y[np.isin(rows, [3, 17, 29])] == 0.0)
    y0, S0 = oracle.spmv_rows(np.zeros(0, np.int64), rp, col, val, x)
    assert y0.size == 0 and S0.size == 0

"""GPU parity (-m gpu): the CUDA path through the C ABI against the CPU oracle,
element by element on the same seeded inputs (north_star tolerance
|y - y_ref| <= 1e-12 * sum_j |a_ij x_j|; integer/dyadic variants and all
index work bit-exact)."""
import dataclasses

import numpy as np
import pytest

import oracle
import paper_1203_2739_b200 as sp
import paper_1203_2739_b200.testing as T
import synth
from gpu_util import assert_parity, create, gpu_apply, oracle_permuted, panel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    sp.lib()   # raises if the library is missing: no fallback


# ------------------------------------------------------------ ingest (a1)
@pytest.mark.parametrize("name", ["c1", "c2s", "c5s", "c3s"])
def test_ingest_bit_exact(name):
    p = synth.make(name)
    h = create(p, options=dict(retain_csr=1))
    rp, col, val = T.debug_copy_csr(h)
    o = oracle.permute(p.m, p.n, p.row_ptr, p.col, p.val, p.row_perm, p.col_perm)
    assert np.array_equal(rp, o[0])
    assert np.array_equal(col, o[1])
    assert np.array_equal(val.view(np.int64), o[2].view(np.int64))


# -------------------------------------------------------- single SpMxV (a5-a7)
@pytest.mark.parametrize("variant", ["real", "int", "dyadic"])
@pytest.mark.parametrize("name", ["c1", "c2s", "c5s", "c4s", "c3s"])
def test_spmv_parity(name, variant):
    p = synth.make(name, variant=variant)
    x = p.x()
    xh, yh_ref, S = oracle_permuted(p, x)
    h = create(p)
    yh = gpu_apply(h, xh, p.m)
    assert_parity(yh, yh_ref, S, exact=(variant != "real"), what=f"{name}/{variant}")


@pytest.mark.parametrize("name", ["c2s", "c5s"])
def test_original_index_space(name):
    p = synth.make(name)
    x = p.x()
    y_ref, S = oracle.spmv(p.row_ptr, p.col, p.val, x)
    h = create(p)
    y = gpu_apply(h, x, p.m, flags=sp.SPMV_VEC_ORIGINAL)
    assert_parity(y, y_ref, S, what=name)
    pi = synth.make(name, variant="int")
    xi = pi.x()
    yi = gpu_apply(create(pi), xi, pi.m, flags=sp.SPMV_VEC_ORIGINAL)
    assert_parity(yi, oracle.spmv(pi.row_ptr, pi.col, pi.val, xi)[0], None, exact=True)


def _edge_matrix(lengths, n, seed=0, variant="int"):
    rng = np.random.default_rng(seed)
    rp = np.zeros(len(lengths) + 1, np.int64)
    rp[1:] = np.cumsum(lengths)
    col = np.concatenate([np.sort(rng.choice(n, L, replace=False)) for L in lengths] or [np.zeros(0)]).astype(np.int32)
    nnz = int(rp[-1])
    if variant == "int":
        val = (rng.integers(1, 5, nnz) * rng.choice([-1, 1], nnz)).astype(np.float64)
        x = rng.integers(-4, 5, n).astype(np.float64)
    else:
        val = rng.uniform(-1, 1, nnz)
        x = rng.uniform(-1, 1, n)
    return rp, col, val, x


@pytest.mark.parametrize("case", ["tile_edges", "long_rows", "empty_rows", "rect_wide", "rect_tall",
                                  "single", "all_empty", "ragged_mix"])
@pytest.mark.parametrize("variant", ["int", "real"])
@pytest.mark.parametrize("kernel", ["default", "panel", "rowtile32"])
def test_edge_shapes(case, variant, kernel):
    """Row lengths at every tile/class boundary +-1, rows longer than a tile,
    empty rows, m != n (Table 1's rectangular group), odd row
    starts (exercise the 128-bit quad peeling).  kernel=panel forces the
    column-sorted panel kernel on small panels (virtual rows of very long
    rows, the warp fold of rows with > 32 of them, empty panels' rows).
    The default here is the row-tile kernel with f3's 16-bit tile-local ids
    (every case fits them; a tile's boundary quads hold a neighbour's ids);
    rowtile32 forces 32-bit ids."""
    opts = panel(700) if kernel == "panel" else dict(kernel="rowtile", index16=1) if kernel == "rowtile32" else None
    TN = 2048   # kTileNnz
    rng = np.random.default_rng(5)
    if case == "tile_edges":
        lengths, n = [1, 3, TN - 1, TN, TN + 1, 2, 5, TN - 3, 7, 4 * TN + 1, 1, 0, 33, 31, 32], 20000
    elif case == "long_rows":
        lengths, n = [10000, 1, 6000, 2 * TN, 3], 12000
    elif case == "empty_rows":
        lengths, n = list(rng.choice([0, 0, 0, 1, 2, 17], 3000)), 500
    elif case == "rect_wide":
        lengths, n = list(rng.integers(0, 40, 700)), 50000
    elif case == "rect_tall":
        lengths, n = list(rng.integers(0, 9, 9000)), 64
    elif case == "single":
        lengths, n = [1], 1
    elif case == "all_empty":
        lengths, n = [0] * 1000, 77
    else:
        lengths, n = list(rng.integers(0, 600, 400)) + [TN + 5] + list(rng.integers(0, 3, 2000)), 4000
    rp, col, val, x = _edge_matrix(lengths, n, variant=variant)
    m = len(lengths)
    y_ref, S = oracle.spmv(rp, col, val, x)
    h = sp.spmv_create(m, n, rp, col, val, options=opts)
    if kernel == "panel" and case not in ("all_empty",):
        assert sp.spmv_get_info(h)["kernel"] == 7
    y = gpu_apply(h, x, m)
    assert_parity(y, y_ref, S, exact=(variant == "int"), what=case)


def test_random_perms_unsorted_rows():
    """Random (non-owner-aligned) perms; input rows given unsorted (A3)."""
    rng = np.random.default_rng(9)
    p = synth.make("c4s")
    m, n = p.m, p.n
    rp, col, val = p.row_ptr.copy(), p.col.copy(), p.val.copy()
    for i in range(0, m, 7):   # shuffle some rows' entry order
        a, b = rp[i], rp[i + 1]
        o = rng.permutation(b - a)
        col[a:b], val[a:b] = col[a:b][o], val[a:b][o]
    pr, pc = rng.permutation(m).astype(np.int32), rng.permutation(n).astype(np.int32)
    x = p.x()
    y_ref, S = oracle.spmv(rp, col, val, x)
    h = sp.spmv_create(m, n, rp, col, val, row_perm=pr, col_perm=pc)
    yh = gpu_apply(h, oracle.permute_x(pc, x), m)
    assert_parity(oracle.unpermute_y(pr, yh), y_ref, S)
    y = gpu_apply(h, x, m, flags=sp.SPMV_VEC_ORIGINAL)
    assert_parity(y, y_ref, S)


# ----------------------------------------------------------- split (a8)
@pytest.mark.parametrize("variant", ["real", "int"])
def test_split_parity(variant):
    p = synth.make("c3s", variant=variant)
    x = p.x()
    ys_ref = oracle.split(p.row_ptr, p.col, p.val, p.parts, p.n_parts, x)
    y_ref, S = oracle.spmv(p.row_ptr, p.col, p.val, x)
    h = create(p)
    ys = gpu_apply(h, x, p.m, split=True)           # identity perms: permuted == original space
    yl = gpu_apply(h, x, p.m, split=True, flags=sp.SPMV_SPLIT_LITERAL)
    yp = gpu_apply(h, x, p.m)
    exact = variant == "int"
    assert_parity(ys, ys_ref, S, exact=exact, what="fused split vs oracle split")
    assert_parity(yl, ys_ref, S, exact=exact, what="literal split vs oracle split")
    assert_parity(ys, y_ref, S, exact=exact, what="sum_k A^k x = A x")
    assert_parity(yp, y_ref, S, exact=exact, what="apply on a split handle")


def test_split_k1_and_random_parts():
    p = synth.make("c4s", variant="int")
    x = p.x()
    y_ref, _ = oracle.spmv(p.row_ptr, p.col, p.val, x)
    h1 = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, parts=np.zeros(p.nnz, np.int32), n_parts=1)
    assert np.array_equal(gpu_apply(h1, x, p.m, split=True), y_ref)
    rng = np.random.default_rng(1)
    parts = rng.integers(0, 5, p.nnz).astype(np.int32)
    h5 = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, parts=parts, n_parts=5)
    assert np.array_equal(gpu_apply(h5, x, p.m, split=True), oracle.split(p.row_ptr, p.col, p.val, parts, 5, x))
    assert np.array_equal(gpu_apply(h5, x, p.m, split=True, flags=sp.SPMV_SPLIT_LITERAL), y_ref)


def test_split_on_panels_edges():
    """Fused split on forced small panels: K = 1, parts that never occur, rows
    whose nonzeros all sit in one part, empty rows, long segments."""
    lengths = [0, 1, 40, 3000, 0, 7, 33, 2] * 150
    rp, col, val, x = _edge_matrix(lengths, 5000, seed=3)
    m, nnz = len(lengths), int(rp[-1])
    y_ref, _ = oracle.spmv(rp, col, val, x)
    rng = np.random.default_rng(4)
    cases = {
        "k1": (np.zeros(nnz, np.int32), 1),
        "sparse_ids": (rng.choice([0, 3, 6], nnz).astype(np.int32), 7),
        "row_parts": (np.repeat(np.arange(m) % 4, np.diff(rp)).astype(np.int32), 4),
        "random": (rng.integers(0, 9, nnz).astype(np.int32), 9),
    }
    for what, (parts, K) in cases.items():
        h = sp.spmv_create(m, 5000, rp, col, val, parts=parts, n_parts=K, options=panel(700))
        assert sp.spmv_get_info(h)["split_kernel"] == 7, what
        ys = gpu_apply(h, x, m, split=True)
        assert np.array_equal(ys, oracle.split(rp, col, val, parts, K, x)), what
        assert np.array_equal(ys, y_ref), what
        sp.spmv_destroy(h)


def test_split_with_permutation():
    p = synth.make("c2s", variant="int")
    rng = np.random.default_rng(2)
    parts = rng.integers(0, 3, p.nnz).astype(np.int32)
    x = p.x()
    ys_ref = oracle.split(p.row_ptr, p.col, p.val, parts, 3, x)
    h = sp.spmv_create(p.m, p.n, p.row_ptr, p.col, p.val, row_perm=p.row_perm, col_perm=p.col_perm,
                       blocks=p.blocks, parts=parts, n_parts=3)
    assert np.array_equal(gpu_apply(h, x, p.m, split=True, flags=sp.SPMV_VEC_ORIGINAL), ys_ref)


# ------------------------------------------------ power iteration glue (a9)
def _c5_like(seed=3):
    """Two C5-shaped SB blocks (identity perms) at the production panel size."""
    synth.PRESETS["_c5like_pi"] = lambda **kw: synth._sb(2, 40_000, 39_200, 800, 12, 20, 0, 3, **kw)
    return synth.make("_c5like_pi", scramble=0, seed=seed)


def _teacher_forced(p, opts, steps, split=False, expect_kernel=None, expect_runs=None):
    """Teacher-forced power iteration: at every step the
    oracle recomputes A x_t (or the split sum) from the GPU's own x_t and
    checks y_t within the north_star tolerance; m_t must equal the oracle's
    max |y_t| of the GPU's y_t exactly, and x_{t+1} must equal y_t / m_t bit
    for bit (IEEE division)."""
    h = create(p, options=opts)
    info = sp.spmv_get_info(h)
    assert info["has_owner_map"] == 1
    if expect_kernel is not None:
        assert (info["split_kernel"] if split else info["kernel"]) == expect_kernel
    if expect_runs is not None:
        assert info["owner_runs"] == expect_runs
    x = p.x()
    xh = torch.from_numpy(oracle.permute_x(p.col_perm, x) if p.col_perm is not None else x.copy()).cuda()
    yh = torch.empty(p.m, dtype=torch.float64, device="cuda")
    md = torch.empty(1, dtype=torch.float64, device="cuda")
    nth = oracle.max_threads()
    for t in range(steps):
        (sp.spmv_split_apply if split else sp.spmv_apply)(h, xh, yh, sp.SPMV_FUSE_MAXABS)
        sp.spmv_maxabs(h, md)
        xn = torch.empty_like(xh)
        sp.spmv_normalize(h, yh, md, xn)
        torch.cuda.synchronize()
        xg = xh.cpu().numpy()
        x_orig = xg[p.col_perm] if p.col_perm is not None else xg      # x[j] = x^[col_perm[j]]
        y_ref, S = oracle.spmv(p.row_ptr, p.col, p.val, x_orig, nthreads=nth)
        if split:
            y_ref = oracle.split(p.row_ptr, p.col, p.val, p.parts, p.n_parts, x_orig)
        yg = yh.cpu().numpy()
        y_gpu = oracle.unpermute_y(p.row_perm, yg) if p.row_perm is not None else yg
        assert_parity(y_gpu, y_ref, S, what=f"step {t}")
        m_gpu = float(md.item())
        assert m_gpu == oracle.maxabs(y_gpu), f"step {t}: max |y| folded on the GPU"
        xn_ref = oracle.scale(y_gpu, m_gpu)                             # x_{t+1}[j] = y_t[j] / m_t
        xnh = xn.cpu().numpy()
        xn_orig = xnh[p.col_perm] if p.col_perm is not None else xnh
        assert np.array_equal(xn_orig.view(np.int64), xn_ref.view(np.int64)), f"step {t}: x-update"
        xh = xn
    sp.spmv_destroy(h)


def test_power_iteration_teacher_forced():
    """c5s on its default kernel (the row-tile fallback at this size)."""
    _teacher_forced(synth.make("c5s"), None, 6)


def test_power_iteration_panel_c5_geometry():
    """The production kernel of C5 -- column-sorted panels at the full-C5 panel
    size (16,384 slots), SB border groups -- with the max |y| fold of its
    epilogue (untested on the default kernel)."""
    _teacher_forced(_c5_like(), panel(16384), 4, expect_kernel=7)


def test_power_iteration_panel_c4_virtual_rows():
    """C4's power-law rows on forced panels: rows above 32 nonzeros are split
    into virtual rows, folded by one thread (<= 32 of them) or a warp (more);
    both epilogue folds feed the max."""
    p = synth.make("c4s")
    assert int(np.diff(p.row_ptr).max()) > 32 * 32   # some rows get > 32 virtual rows (warp fold)
    _teacher_forced(p, panel(2000), 4, expect_kernel=7)


def test_power_iteration_owner_map_forms():
    """The x-update's two owner-map forms (a9): A17's owner-aligned SB layout
    held as runs (c5s: one run per block's interior columns and one per owned
    border slice; c4s: identity, one run), and a per-column array when the
    runs are short (independent random row and column permutations)."""
    p = synth.make("c5s")
    K = p.blocks["K"]
    _teacher_forced(p, None, 3, expect_runs=2 * K)
    q = synth.make("c4s")
    _teacher_forced(q, None, 2, expect_runs=1)
    rng = np.random.default_rng(11)
    q = dataclasses.replace(q, row_perm=rng.permutation(q.m).astype(np.int32),
                            col_perm=rng.permutation(q.n).astype(np.int32))
    _teacher_forced(q, None, 3, expect_runs=0)


def test_power_iteration_split_fused_maxabs():
    """The fused multiple-SpMxV on panels with SPMV_FUSE_MAXABS: the (row,
    part) fold of the epilogue feeds the max; teacher-forced against the
    oracle's literal split sequence."""
    _teacher_forced(synth.make("c3s"), panel(900), 3, split=True, expect_kernel=7)


# ------------------------------------------------------------ API behaviour
def test_errors_on_device():
    p = synth.make("c2s")
    h = create(p)
    x = torch.zeros(p.n, dtype=torch.float64, device="cuda")
    y = torch.zeros(p.m, dtype=torch.float64, device="cuda")
    with pytest.raises(sp.SpmvError) as e:
        sp.spmv_apply(h, x[:-1], y)
    assert e.value.status == sp.SPMV_ERR_DATA
    with pytest.raises(sp.SpmvError) as e:
        sp.spmv_apply(h, x, x)
    assert e.value.status in (sp.SPMV_ERR_USAGE, sp.SPMV_ERR_DATA)
    with pytest.raises(sp.SpmvError) as e:
        sp.spmv_split_apply(h, x, y)
    assert e.value.status == sp.SPMV_ERR_UNSUPPORTED
    with pytest.raises(sp.SpmvError) as e:
        sp.spmv_apply(h, x, y, flags=64)
    assert e.value.status == sp.SPMV_ERR_USAGE
    sp.spmv_destroy(h)
    with pytest.raises(sp.SpmvError):
        sp.spmv_apply(h, x, y)


def test_deterministic_and_graph_capturable():
    p = synth.make("c4s")
    h = create(p)
    xh = torch.from_numpy(p.x()).cuda()
    y1 = torch.empty(p.m, dtype=torch.float64, device="cuda")
    y2 = torch.empty_like(y1)
    sp.spmv_apply(h, xh, y1)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        sp.spmv_apply(h, xh, y2, stream=s)    # warm-up on the capture stream
        torch.cuda.synchronize()
        y2.zero_()
        with torch.cuda.graph(g, stream=s):
            sp.spmv_apply(h, xh, y2, stream=s)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y1.view(torch.int64), y2.view(torch.int64))


# ------------------------------------------------- full-size configs
@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_full_size_parity(name):
    """BASELINE configs C2-C4 at full size, every entry."""
    p = synth.make(name)
    x = p.x()
    xh, yh_ref, S = oracle_permuted(p, x)
    h = create(p)
    assert_parity(gpu_apply(h, xh, p.m), yh_ref, S, what=name)
    if p.parts is not None:
        ys_ref = oracle.split(p.row_ptr, p.col, p.val, p.parts, p.n_parts, x)
        assert_parity(gpu_apply(h, xh, p.m, split=True), ys_ref, S, what=name + " split")


def test_full_size_power_c4():
    """BASELINE config C4 at full size (4 M rows, 48 M nonzeros) on its default
    kernel: three teacher-forced power steps, every entry, m_t exact and
    x_{t+1} bitwise."""
    _teacher_forced(synth.make("c4"), None, 3, expect_kernel=7)


def test_full_size_power_c5():
    """BASELINE config C5 at full size (64 M rows, 1.12e9 nonzeros, hidden
    permutation) on its default kernel (panels, plan of the bench): two
    teacher-forced power steps checked on all 64 M rows (the bench
    samples 200,000 rows), m_t exact and x_{t+1} bitwise."""
    _teacher_forced(synth.make("c5"), None, 2, expect_kernel=7)


# ----------------------------------------------- f3: 16-bit column ids
@pytest.mark.parametrize("name", ["c1", "c2s", "c5s", "c4s", "c2"])
def test_index16_bitwise(name):
    """f3 (ICSR-style index compression): the row-tile kernel with
    16-bit tile-local column ids (two windows per tile: C_k and C_B for an SB
    block tile) gives the same y bit for bit as with 32-bit ids (integer
    decoding, same summation order), and matches the oracle."""
    p = synth.make(name)
    x = p.x()
    xh, yh_ref, S = oracle_permuted(p, x)
    ys = {}
    for mode in (0, 1):
        h = create(p, options=dict(kernel="rowtile", index16=mode))
        info = sp.spmv_get_info(h)
        ys[mode] = (gpu_apply(h, xh, p.m), info["index_bytes"])
        sp.spmv_destroy(h)
    assert ys[1][1] == 4
    if name != "c4s":   # c4s: a long row's columns span > 65,536 ids -> stays 32-bit
        assert ys[0][1] == 2, "16-bit ids expected"
    assert np.array_equal(ys[0][0].view(np.int64), ys[1][0].view(np.int64))
    assert_parity(ys[0][0], yh_ref, S, what=f"{name} 16-bit ids")

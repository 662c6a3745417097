"""GPU parity (-m gpu): the CUDA path through the C ABI against the CPU oracle,
element by element on the same seeded inputs (north_star tolerance
|y - y_ref| <= 1e-12 * sum_j |a_ij x_j|; integer/dyadic variants and all
index work bit-exact)."""
import numpy as np
import pytest

import oracle
import paper_1203_2739_b200 as sp
import synth
from gpu_util import assert_parity, create, gpu_apply, oracle_permuted

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
    h = create(p)
    rp, col, val = sp.spmv_debug_copy_csr(h)
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
@pytest.mark.parametrize("kernel", ["default", "panel"])
def test_edge_shapes(monkeypatch, case, variant, kernel):
    """Row lengths at every tile/class boundary +-1, rows longer than a tile,
    empty rows, m != n (Table 1's rectangular group), odd row
    starts (exercise the 128-bit quad peeling).  kernel=panel forces the
    column-sorted panel kernel on small panels (virtual rows of very long
    rows, the warp fold of rows with > 32 of them, empty panels' rows)."""
    if kernel == "panel":
        monkeypatch.setenv("SPMV_KERNEL", "panel")
        monkeypatch.setenv("SPMV_PN_ROWS", "700")
    T = 2048   # kTileNnz
    rng = np.random.default_rng(5)
    if case == "tile_edges":
        lengths, n = [1, 3, T - 1, T, T + 1, 2, 5, T - 3, 7, 4 * T + 1, 1, 0, 33, 31, 32], 20000
    elif case == "long_rows":
        lengths, n = [10000, 1, 6000, 2 * T, 3], 12000
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
        lengths, n = list(rng.integers(0, 600, 400)) + [T + 5] + list(rng.integers(0, 3, 2000)), 4000
    rp, col, val, x = _edge_matrix(lengths, n, variant=variant)
    m = len(lengths)
    y_ref, S = oracle.spmv(rp, col, val, x)
    h = sp.spmv_create(m, n, rp, col, val)
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


def test_split_on_panels_edges(monkeypatch):
    """Fused split on forced small panels: K = 1, parts that never occur, rows
    whose nonzeros all sit in one part, empty rows, long segments."""
    monkeypatch.setenv("SPMV_KERNEL", "panel")
    monkeypatch.setenv("SPMV_PN_ROWS", "700")
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
        h = sp.spmv_create(m, 5000, rp, col, val, parts=parts, n_parts=K)
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
def test_power_iteration_teacher_forced():
    p = synth.make("c5s")
    h = create(p)
    info = sp.spmv_get_info(h)
    assert info["has_owner_map"] == 1
    x = p.x()
    xh = torch.from_numpy(oracle.permute_x(p.col_perm, x)).cuda()
    yh = torch.empty(p.m, dtype=torch.float64, device="cuda")
    md = torch.empty(1, dtype=torch.float64, device="cuda")
    for t in range(6):
        sp.spmv_apply(h, xh, yh, sp.SPMV_FUSE_MAXABS)
        sp.spmv_maxabs(h, md)
        xn = torch.empty_like(xh)
        sp.spmv_normalize(h, yh, md, xn)
        torch.cuda.synchronize()
        # teacher forcing: the oracle recomputes A x_t from the GPU's own x_t
        xg = xh.cpu().numpy()
        x_orig = np.empty_like(xg)
        x_orig[:] = xg[p.col_perm]            # x[j] = x^[col_perm[j]]
        y_ref, S = oracle.spmv(p.row_ptr, p.col, p.val, x_orig)
        y_gpu = oracle.unpermute_y(p.row_perm, yh.cpu().numpy())
        assert_parity(y_gpu, y_ref, S, what=f"step {t}")
        m_gpu = float(md.item())
        assert m_gpu == oracle.maxabs(y_gpu)                     # exact max
        xn_ref = oracle.scale(y_gpu, m_gpu)                      # x_{t+1}[j] = y_t[j] / m_t
        assert np.array_equal(xn.cpu().numpy()[p.col_perm], xn_ref)
        xh = xn


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

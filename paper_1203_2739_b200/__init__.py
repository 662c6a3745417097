"""B200-native SpMxV on SB/DB-reordered matrices (arXiv 1203.2739 hot path).

Thin ctypes binding over the C ABI in ``include/spmv.h`` (libspmv_b200.so,
built by ``python -m paper_1203_2739_b200.build``).  Argument marshalling
only: every step of the path -- ingest, planning, the SpMxV and split
kernels, the NCCL border exchange, the power-iteration glue -- runs in the
library.  There is no CPU or PyTorch fallback: if the library is missing,
importing the binding's entry points raises.

Names follow the ABI: ``spmv_create`` (-> ``spmv_create_ex``), ``spmv_apply``,
``spmv_split_apply``, ``spmv_destroy`` plus the helpers ``spmv_get_info``,
``spmv_maxabs``, ``spmv_normalize``, ``spmv_shard_plan``,
``spmv_nccl_unique_id``, and ``spmv_order_sbfs`` (f4: the sBFS ordering + SB
extraction that produces the permutations and blocks).  The test hooks of ``include/spmv_test.h`` are in
``paper_1203_2739_b200.testing``; the measurement microkernels
(``include/spmv_diag.h``, a separate library) in ``paper_1203_2739_b200.diag``.
Vectors are CUDA float64 torch tensors (or raw device addresses); the stream
argument is a ``torch.cuda.Stream``, a raw ``cudaStream_t`` int, or None for
torch's current stream.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspmv_b200.so")

SPMV_OK, SPMV_ERR_USAGE, SPMV_ERR_DATA, SPMV_ERR_INTERNAL, SPMV_ERR_UNSUPPORTED = range(5)
SPMV_SB, SPMV_DB = 1, 2
SPMV_VEC_PERMUTED = 0
SPMV_VEC_ORIGINAL = 1
SPMV_FUSE_MAXABS = 2
SPMV_SPLIT_LITERAL = 4

EXPORTED = ["spmv_create", "spmv_create_ex", "spmv_apply", "spmv_split_apply", "spmv_destroy", "spmv_get_info",
            "spmv_maxabs", "spmv_normalize", "spmv_nccl_unique_id", "spmv_status_string", "spmv_last_error",
            "spmv_version", "spmv_shard_plan", "spmv_order_sbfs"]
# include/spmv_test.h (test and debug hooks, same library)
EXPORTED_TEST = ["spmv_debug_copy_csr", "spmv_pn_plan_check", "spmv_pn_shard_hash", "spmv_test_create_rank",
                 "spmv_test_loopback_link", "spmv_test_rank_stream", "spmv_test_corrupt_panel", "spmv_test_panel_stamps"]

KERNELS = {"auto": 0, "panel": 1, "rowtile": 2, "xstaged": 3}
SPLIT_KERNELS = {"auto": 0, "panel": 1, "rows": 2}
EXCHANGES = {"auto": 0, "nccl": 1, "p2p": 2}


class SpmvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{msg} (status {status})")
        self.status = status


class _Blocks(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("K", ctypes.c_int32),
                ("row_block_ptr", ctypes.c_void_p), ("col_block_ptr", ctypes.c_void_p),
                ("border_owner_ptr", ctypes.c_void_p), ("row_border_owner_ptr", ctypes.c_void_p)]


class _Options(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_int32), ("kernel", ctypes.c_int32), ("panel_rows", ctypes.c_int32),
                ("split_kernel", ctypes.c_int32), ("exchange", ctypes.c_int32), ("index16", ctypes.c_int32),
                ("debug_checks", ctypes.c_int32), ("retain_csr", ctypes.c_int32), ("reserved", ctypes.c_int32 * 8)]


class _Dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("device", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("nccl_unique_id", ctypes.c_void_p)]


class spmv_info_t(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in (
        "m", "n", "nnz", "m_local", "nnz_local", "row_begin", "x_local_len", "x_interior_begin",
        "x_interior_len", "x_border_begin", "x_border_len", "border_total", "n_tiles", "n_long_rows",
        "bytes_alg", "bytes_alg_split", "split_segments", "panels", "groups", "pad_slots",
        "bytes_stream")] + [
        (k, ctypes.c_int32) for k in ("n_parts", "rank", "world", "kind", "has_owner_map", "kernel",
                                      "split_kernel", "exchange")] + [
        (k, ctypes.c_int64) for k in ("gather_sectors", "y_local_len", "y_border_begin", "y_border_len",
                                      "deferred", "y_wavefronts_x1000", "exchange_timeouts", "index_bytes")] + [
        ("debug_violations", ctypes.c_int64 * 3), ("create_s", ctypes.c_double * 6), ("far_nonzeros", ctypes.c_int64),
        ("owner_runs", ctypes.c_int64)]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["debug_violations"] = list(self.debug_violations)
        d["create_s"] = list(self.create_s)
        return d


class spmv_order_info_t(ctypes.Structure):
    _fields_ = [("bfs_ms", ctypes.c_double), ("extract_ms", ctypes.c_double), ("levels", ctypes.c_int64),
                ("components", ctypes.c_int64), ("border_cols", ctypes.c_int64)]


_lib = None


def lib():
    """Load libspmv_b200.so; raises if it is missing (no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1203_2739_b200.build` "
                              "(the SpMxV path has no CPU or PyTorch fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
        L.spmv_create.argtypes = [i64, i64, i64, vp, vp, vp, vp, vp, vp, i32, vp, vp, ctypes.POINTER(vp)]
        L.spmv_create_ex.argtypes = [i64, i64, i64, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, ctypes.POINTER(vp)]
        L.spmv_apply.argtypes = [vp, vp, i64, vp, i64, u32, vp]
        L.spmv_split_apply.argtypes = [vp, vp, i64, vp, i64, u32, vp]
        L.spmv_destroy.argtypes = [vp]
        L.spmv_get_info.argtypes = [vp, ctypes.POINTER(spmv_info_t)]
        L.spmv_maxabs.argtypes = [vp, vp, vp]
        L.spmv_normalize.argtypes = [vp, vp, vp, vp, vp]
        L.spmv_nccl_unique_id.argtypes = [vp, ctypes.c_size_t]
        L.spmv_shard_plan.argtypes = [vp, i64, i64, i32, i32, vp]
        L.spmv_status_string.argtypes = [i32]
        L.spmv_status_string.restype = ctypes.c_char_p
        L.spmv_last_error.argtypes = []
        L.spmv_last_error.restype = ctypes.c_char_p
        L.spmv_version.restype = i32
        L.spmv_order_sbfs.argtypes = [i64, i64, i64, vp, vp, i32, vp, vp, vp, vp, ctypes.POINTER(spmv_order_info_t)]
        L.spmv_debug_copy_csr.argtypes = [vp, vp, vp, vp]
        L.spmv_pn_plan_check.argtypes = [i64, i64, vp, vp, vp, vp, i64, vp]
        L.spmv_pn_shard_hash.argtypes = [i64, i64, vp, vp, vp, vp, i32, i32, vp]
        L.spmv_test_create_rank.argtypes = [i64, i64, i64, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, ctypes.POINTER(vp)]
        L.spmv_test_loopback_link.argtypes = [vp, i32]
        L.spmv_test_rank_stream.argtypes = [vp, vp]
        L.spmv_test_corrupt_panel.argtypes = [vp, i32]
        L.spmv_test_panel_stamps.argtypes = [vp, i32, vp, i64]
        for name in EXPORTED_TEST:
            getattr(L, name).restype = i32
        for name in EXPORTED:
            if name not in ("spmv_status_string", "spmv_last_error", "spmv_version"):
                getattr(L, name).restype = i32
        _lib = L
    return _lib


def _check(status: int, what: str):
    if status != SPMV_OK:
        msg = lib().spmv_last_error().decode(errors="replace")
        raise SpmvError(status, f"{what}: {msg}")


def _np(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


def _addr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _dev(t) -> int:
    """Device address of a torch tensor (float64, contiguous) or a raw int."""
    if t is None:
        return 0
    if isinstance(t, int):
        return t
    import torch
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise SpmvError(SPMV_ERR_USAGE, "vectors must be contiguous float64 CUDA tensors")
    return t.data_ptr()


def _len(t, n):
    if n is not None:
        return n
    return 0 if t is None or isinstance(t, int) else t.numel()


def _stream(s) -> int:
    if s is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(s, int):
        return s
    return s.cuda_stream


class Handle:
    """Owns an spmv_handle_t; destroyed by spmv_destroy (or on GC)."""

    def __init__(self, ptr: int):
        self.ptr = ptr

    def __del__(self):
        try:
            if self.ptr:
                lib().spmv_destroy(ctypes.c_void_p(self.ptr))
                self.ptr = 0
        except Exception:
            pass

    @property
    def info(self) -> dict:
        return spmv_get_info(self)


def _h(h) -> ctypes.c_void_p:
    p = h.ptr if isinstance(h, Handle) else h
    if not p:
        raise SpmvError(SPMV_ERR_USAGE, "handle already destroyed")
    return ctypes.c_void_p(p)


def _blocks_struct(blocks, keep):
    if blocks is None:
        return None
    rbp = _np(blocks["row_block_ptr"], np.int64)
    cbp = _np(blocks["col_block_ptr"], np.int64)
    bop = _np(blocks.get("border_owner_ptr"), np.int64)
    rop = _np(blocks.get("row_border_owner_ptr"), np.int64)
    b = _Blocks(int(blocks["kind"]), int(blocks["K"]), rbp.ctypes.data, cbp.ctypes.data,
                None if bop is None else bop.ctypes.data, None if rop is None else rop.ctypes.data)
    keep += [rbp, cbp, bop, rop, b]
    return ctypes.byref(b)


def _options_struct(options, keep):
    if not options:
        return None
    o = _Options()
    o.struct_size = ctypes.sizeof(_Options)
    o.kernel = KERNELS[options.get("kernel", "auto")]
    o.panel_rows = int(options.get("panel_rows", 0))
    o.split_kernel = SPLIT_KERNELS[options.get("split_kernel", "auto")]
    o.exchange = EXCHANGES[options.get("exchange", "auto")]
    o.index16 = int(options.get("index16", 0))
    o.debug_checks = int(options.get("debug_checks", 0))
    o.retain_csr = int(options.get("retain_csr", 0))
    unknown = set(options) - {"kernel", "panel_rows", "split_kernel", "exchange", "index16", "debug_checks",
                              "retain_csr"}
    if unknown:
        raise ValueError(f"unknown spmv options: {sorted(unknown)}")
    keep.append(o)
    return ctypes.byref(o)


def _create_args(m, n, row_ptr, col_idx, val, row_perm, col_perm, blocks, parts, n_parts, dist, options, keep):
    rp = _np(row_ptr, np.int64)
    ci = _np(col_idx, np.int32)
    va = _np(val, np.float64)
    pr = _np(row_perm, np.int32)
    pc = _np(col_perm, np.int32)
    pa = _np(parts, np.int32)
    keep += [rp, ci, va, pr, pc, pa]
    nnz = int(rp[-1]) if rp is not None and len(rp) else 0
    bptr = _blocks_struct(blocks, keep)
    dptr = None
    if dist is not None:
        uid_ptr = None
        if dist.get("nccl_unique_id") is not None:
            uid = ctypes.create_string_buffer(bytes(dist["nccl_unique_id"]), 128)
            keep.append(uid)
            uid_ptr = ctypes.cast(uid, ctypes.c_void_p).value
        d = _Dist(int(dist["rank"]), int(dist["world"]), int(dist.get("device", 0)), 0, uid_ptr)
        keep.append(d)
        dptr = ctypes.byref(d)
    return (m, n, nnz, _addr(rp), _addr(ci), _addr(va), _addr(pr), _addr(pc), bptr,
            int(n_parts if pa is not None else 0), _addr(pa), dptr, _options_struct(options, keep))


def spmv_create(m: int, n: int, row_ptr, col_idx, val, row_perm=None, col_perm=None, blocks=None,
                parts=None, n_parts: int = 0, dist=None, options=None) -> Handle:
    """Ingest an ORIGINAL-space CSR plus old->new permutations.

    blocks: dict(kind=1|2, K=.., row_block_ptr=[K+2], col_block_ptr=[K+2],
    border_owner_ptr=[K+1] or None, row_border_owner_ptr=[K+1] or None) in
    PERMUTED space.  parts: int32 part id per nonzero in input order (split Pi,
    P:L107).  dist: dict(rank, world, device, nccl_unique_id=bytes(128)) for
    one-process-per-GPU runs.  options: dict(kernel="auto"|"panel"|"rowtile",
    panel_rows=int, split_kernel="auto"|"panel"|"rows", exchange="auto"|"nccl"|"p2p")
    (spmv_options_t)."""
    keep = []
    args = _create_args(m, n, row_ptr, col_idx, val, row_perm, col_perm, blocks, parts, n_parts, dist, options, keep)
    out = ctypes.c_void_p(0)
    _check(lib().spmv_create_ex(*args, ctypes.byref(out)), "spmv_create")
    return Handle(out.value)


class _Shard(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in (
        "block_begin", "block_end", "row_begin", "row_end", "x_interior_begin", "x_interior_len",
        "x_border_begin", "x_border_len", "x_local_len", "border_begin", "border_total",
        "y_border_begin", "y_border_len", "y_local_len")]


def spmv_shard_plan(blocks, m: int, n: int, rank: int, world: int) -> dict:
    """Host-side SB shard plan of rank `rank` of `world` (see spmv.h)."""
    keep = []
    b = _blocks_struct(blocks, keep)
    out = _Shard()
    _check(lib().spmv_shard_plan(b, m, n, rank, world, ctypes.byref(out)), "spmv_shard_plan")
    return {k: int(getattr(out, k)) for k, _ in _Shard._fields_}


def spmv_apply(h, x, y, flags: int = 0, stream=None, x_len: int | None = None, y_len: int | None = None):
    """y^ <- A^ x^; asynchronous on `stream`."""
    _check(lib().spmv_apply(_h(h), ctypes.c_void_p(_dev(x)), _len(x, x_len), ctypes.c_void_p(_dev(y)),
                            _len(y, y_len), flags, ctypes.c_void_p(_stream(stream))), "spmv_apply")


def spmv_split_apply(h, x, y, flags: int = 0, stream=None, x_len: int | None = None, y_len: int | None = None):
    """y = 0; y <- y + A^k x, k = 1..K; fused unless SPMV_SPLIT_LITERAL."""
    _check(lib().spmv_split_apply(_h(h), ctypes.c_void_p(_dev(x)), _len(x, x_len), ctypes.c_void_p(_dev(y)),
                                  _len(y, y_len), flags, ctypes.c_void_p(_stream(stream))), "spmv_split_apply")


def spmv_destroy(h):
    if isinstance(h, Handle):
        if h.ptr:
            _check(lib().spmv_destroy(ctypes.c_void_p(h.ptr)), "spmv_destroy")
            h.ptr = 0
    else:
        _check(lib().spmv_destroy(ctypes.c_void_p(h)), "spmv_destroy")


def spmv_get_info(h) -> dict:
    info = spmv_info_t()
    _check(lib().spmv_get_info(_h(h), ctypes.byref(info)), "spmv_get_info")
    return info.as_dict()


def spmv_maxabs(h, m_dev, stream=None):
    """*m_dev = max_i |y_i| of the last SPMV_FUSE_MAXABS apply (all ranks)."""
    _check(lib().spmv_maxabs(_h(h), ctypes.c_void_p(_dev(m_dev)), ctypes.c_void_p(_stream(stream))), "spmv_maxabs")


def spmv_normalize(h, y, m_dev, x_next, stream=None):
    """x^_{t+1}[c] = y^_t[r(c)] / *m_dev (power-iteration glue)."""
    _check(lib().spmv_normalize(_h(h), ctypes.c_void_p(_dev(y)), ctypes.c_void_p(_dev(m_dev)),
                                ctypes.c_void_p(_dev(x_next)), ctypes.c_void_p(_stream(stream))),
           "spmv_normalize")


def spmv_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().spmv_nccl_unique_id(buf, 128), "spmv_nccl_unique_id")
    return buf.raw


def spmv_status_string(s: int) -> str:
    return lib().spmv_status_string(s).decode()


def spmv_version() -> int:
    return int(lib().spmv_version())


def spmv_order_sbfs(m: int, n: int, row_ptr, col, K: int) -> dict:
    """sBFS ordering + SB extraction on the current CUDA device (f4).
    Host CSR in, host permutations (old -> new) and an SB block descriptor out
    (``blocks`` is ready for ``spmv_create``), plus the device timings."""
    rp = _np(row_ptr, np.int64)
    ci = _np(col, np.int32)
    rperm = np.empty(m, np.int32)
    cperm = np.empty(n, np.int32)
    rbp = np.empty(K + 2, np.int64)
    cbp = np.empty(K + 2, np.int64)
    info = spmv_order_info_t()
    _check(lib().spmv_order_sbfs(m, n, int(rp[-1]), _addr(rp), _addr(ci), K, _addr(rperm), _addr(cperm),
                                 _addr(rbp), _addr(cbp), ctypes.byref(info)), "spmv_order_sbfs")
    return {"row_perm": rperm, "col_perm": cperm, "row_block_ptr": rbp, "col_block_ptr": cbp,
            "blocks": {"kind": SPMV_SB, "K": K, "row_block_ptr": rbp, "col_block_ptr": cbp},
            "bfs_ms": info.bfs_ms, "extract_ms": info.extract_ms, "levels": info.levels,
            "components": info.components, "border_cols": info.border_cols}

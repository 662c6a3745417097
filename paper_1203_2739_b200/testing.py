"""Test and debug hooks of libspmv_b200.so (``include/spmv_test.h``).

Argument marshalling only, like the main binding.  The parity tests use these
to read the device CSR back, to round-trip the panel planner on the host, and
to run the multi-GPU path on one GPU (the loopback fake of SURVEY.md §4:
``test_create_rank`` + ``loopback_link``).  Nothing here changes what a handle
made by ``spmv_create`` computes.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import Handle, _addr, _blocks_struct, _check, _create_args, _h, _np, lib, spmv_get_info


def debug_copy_csr(h):
    """The device copy of the permuted local CSR, back on the host (global column ids)."""
    info = spmv_get_info(h)
    rp = np.empty(info["m_local"] + 1, np.int64)
    col = np.empty(info["nnz_local"], np.int32)
    val = np.empty(info["nnz_local"], np.float64)
    _check(lib().spmv_debug_copy_csr(_h(h), _addr(rp), _addr(col), _addr(val)), "spmv_debug_copy_csr")
    return rp, col, val


def pn_plan_check(m: int, n: int, row_ptr, col, val, blocks, rows_target: int) -> dict:
    """Host-only round trip of the column-sorted panel planner; raises on mismatch."""
    rp = _np(row_ptr, np.int64)
    ci = _np(col, np.int32)
    va = _np(val, np.float64)
    keep = []
    bptr = _blocks_struct(blocks, keep)
    stats = np.zeros(15, dtype=np.int64)
    _check(lib().spmv_pn_plan_check(m, n, _addr(rp), _addr(ci), _addr(va), bptr, rows_target, stats.ctypes.data),
           "spmv_pn_plan_check")
    d = dict(zip(("panels", "groups", "pads", "deferred", "epochs", "entries"), (int(v) for v in stats[:6])))
    d["y_wavefronts_natural"] = stats[6] / 1000.0
    d["y_wavefronts_coloured"] = stats[7] / 1000.0
    d["smem_max"] = int(stats[8])
    d["panels_with_border"] = int(stats[9])
    d["gather_sectors"] = int(stats[10])
    d["pads_drain"] = int(stats[11])
    d["epochs_drain"] = int(stats[12])
    d["far"] = int(stats[13])
    d["far_steps"] = int(stats[14])
    return d


def pn_shard_hash(m: int, n: int, row_ptr, col, val, blocks, world: int, sms: int = 148) -> np.ndarray:
    """Host-only: per-rank, per-block hashes of the SB panel plan's summation order; int64 [world, K]."""
    rp = _np(row_ptr, np.int64)
    ci = _np(col, np.int32)
    va = _np(val, np.float64)
    keep = []
    bptr = _blocks_struct(blocks, keep)
    out = np.zeros((world, int(blocks["K"])), dtype=np.int64)
    _check(lib().spmv_pn_shard_hash(m, n, _addr(rp), _addr(ci), _addr(va), bptr, world, sms, out.ctypes.data),
           "spmv_pn_shard_hash")
    return out


def test_create_rank(m: int, n: int, row_ptr, col_idx, val, rank: int, world: int, row_perm=None, col_perm=None,
                     blocks=None, parts=None, n_parts: int = 0, device: int = 0, options=None) -> Handle:
    """Rank `rank` of `world` on the current GPU without a communicator (loopback fake)."""
    keep = []
    args = _create_args(m, n, row_ptr, col_idx, val, row_perm, col_perm, blocks, parts, n_parts,
                        dict(rank=rank, world=world, device=device), options, keep)
    out = ctypes.c_void_p(0)
    _check(lib().spmv_test_create_rank(*args, ctypes.byref(out)), "spmv_test_create_rank")
    return Handle(out.value)


def loopback_link(handles) -> None:
    """Link test ranks 0..G-1 (in order) into one loopback group (P2P protocol on one GPU)."""
    arr = (ctypes.c_void_p * len(handles))(*[_h(h).value for h in handles])
    _check(lib().spmv_test_loopback_link(arr, len(handles)), "spmv_test_loopback_link")


def rank_stream(h):
    """The apply stream of a linked loopback test rank, as a torch.cuda.ExternalStream."""
    import torch
    out = ctypes.c_void_p(0)
    _check(lib().spmv_test_rank_stream(_h(h), ctypes.byref(out)), "spmv_test_rank_stream")
    return torch.cuda.ExternalStream(out.value)


def corrupt_panel(h, kind: int) -> None:
    """Corrupt a panel handle's plan on the device (tests of debug_checks)."""
    _check(lib().spmv_test_corrupt_panel(_h(h), kind), "spmv_test_corrupt_panel")


def panel_stamps_arm(h) -> None:
    """Record the per-CTA timeline of the handle's next panel-kernel launches."""
    _check(lib().spmv_test_panel_stamps(_h(h), 1, None, 0), "spmv_test_panel_stamps")


def panel_stamps_read(h) -> np.ndarray:
    """[panels, 8] uint64: SM id, globaltimer start/end (ns), clock64 at start, after the
    prologue, after the far phase, at the end, after the epochs -- of the last launch; disarms."""
    n = spmv_get_info(h)["panels"]
    out = np.zeros((n, 8), np.uint64)
    _check(lib().spmv_test_panel_stamps(_h(h), 0, _addr(out), out.size), "spmv_test_panel_stamps")
    return out

"""Seeded synthetic inputs for the SpMxV hot path (BASELINE.json configs C1-C5).

This package is the only code shared between the oracle side (``oracle/``,
``tests/``) and the product side (``bench.py`` driving
``paper_1203_2739_b200``).  It builds inputs only -- original-space CSR,
old->new permutations, the SB/DB block descriptor, split part ids, dense
vectors -- and holds none of the method's arithmetic.  The recipes (sizes,
distributions, readings A13-A18 of SURVEY.md §8(c)) are restated in DESIGN.md
"Input recipe".

The heavy lifting is ``gen.c`` (plain C + OpenMP, counter-based RNG, so the
output does not depend on the thread count); it is compiled on first use.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_SO = os.path.join(_HERE, "libsynth.so")

UNIFORM, SB, DB, POWERLAW = 1, 2, 3, 4
VARIANTS = {"real": 0, "int": 1, "dyadic": 2}


class _Params(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("variant", ctypes.c_int32),
        ("scramble", ctypes.c_int32), ("pad0", ctypes.c_int32),
        ("m", ctypes.c_int64), ("n", ctypes.c_int64), ("seed", ctypes.c_uint64),
        ("lo", ctypes.c_int64), ("hi", ctypes.c_int64),
        ("K", ctypes.c_int64), ("Rb", ctypes.c_int64), ("Ci", ctypes.c_int64), ("Bs", ctypes.c_int64),
        ("int_lo", ctypes.c_int64), ("int_hi", ctypes.c_int64),
        ("bord_lo", ctypes.c_int64), ("bord_hi", ctypes.c_int64),
        ("RB", ctypes.c_int64), ("CB", ctypes.c_int64),
        ("brow_lo", ctypes.c_int64), ("brow_hi", ctypes.c_int64),
        ("q", ctypes.c_double), ("Lmax", ctypes.c_int64), ("band", ctypes.c_int64),
        ("band_frac", ctypes.c_double),
    ]


def build(force: bool = False) -> str:
    """Compile gen.c into libsynth.so (gcc, OpenMP)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P = ctypes.POINTER
        lib.synth_check.argtypes = [P(_Params)]
        lib.synth_structure.argtypes = [P(_Params), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.synth_fill.argtypes = [P(_Params), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.synth_vector.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int32,
                                     ctypes.c_void_p]
        lib.synth_vector.restype = None
        lib.synth_sb_owner.argtypes = [P(_Params), ctypes.c_void_p]
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


@dataclass
class Problem:
    """One synthetic SpMxV instance.  Everything is host numpy, ORIGINAL space
    except ``blocks`` (PERMUTED space, the reordered form the library computes
    in)."""
    name: str
    m: int
    n: int
    row_ptr: np.ndarray          # int64 [m+1]
    col: np.ndarray              # int32 [nnz]
    val: np.ndarray              # float64 [nnz]
    row_perm: np.ndarray | None  # int32 [m] old->new, None = identity
    col_perm: np.ndarray | None  # int32 [n] old->new, None = identity
    blocks: dict | None          # {"kind": 1|2, "K", "row_block_ptr", "col_block_ptr"}
    parts: np.ndarray | None     # int32 [nnz] split part id, canonical (input CSR) order
    n_parts: int
    owner: np.ndarray | None     # int32 [n] r(c): permuted col -> permuted row (A17), SB only
    variant: str
    seed: int
    params: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def x(self, stream: int = 0) -> np.ndarray:
        """Dense x in ORIGINAL space, U(-1,1) (or the variant's exact set)."""
        return vector(self.n, self.seed, stream, self.variant)


def vector(n: int, seed: int = 0, stream: int = 0, variant: str = "real") -> np.ndarray:
    lib = _load()
    out = np.empty(n, dtype=np.float64)
    lib.synth_vector(n, seed, stream, VARIANTS[variant], _ptr(out))
    return out


# ---------------------------------------------------------------------------
# Config presets (BASELINE.json configs[0..4]; readings in SURVEY.md §8(c))
# ---------------------------------------------------------------------------
def _c1(**kw):
    return dict(kind=UNIFORM, m=2000, n=2000, lo=4, hi=16) | kw


def _sb(K, Rb, Ci, Bs, int_lo, int_hi, bord_lo, bord_hi, scramble=1, **kw):
    return dict(kind=SB, m=K * Rb, n=K * Ci + K * Bs, K=K, Rb=Rb, Ci=Ci, Bs=Bs,
                int_lo=int_lo, int_hi=int_hi, bord_lo=bord_lo, bord_hi=bord_hi, scramble=scramble) | kw


def _db(K, Rb, RB, int_lo, int_hi, bord_lo, bord_hi, brow_lo, brow_hi, **kw):
    return dict(kind=DB, m=K * Rb + RB, n=K * Rb + RB, K=K, Rb=Rb, Ci=Rb, RB=RB, CB=RB,
                int_lo=int_lo, int_hi=int_hi, bord_lo=bord_lo, bord_hi=bord_hi,
                brow_lo=brow_lo, brow_hi=brow_hi, scramble=0) | kw


def _pl(n, q=0.9043, Lmax=10000, band=2000, band_frac=0.7, **kw):
    return dict(kind=POWERLAW, m=n, n=n, q=q, Lmax=Lmax, band=band, band_frac=band_frac, scramble=0) | kw


PRESETS = {
    # C1: tiny irregular, 2,000^2, U{4..16}, identity perms, seed 0
    "c1": lambda **kw: _c1(**kw),
    # C2: SB 200,000^2, 16 blocks x 12,500 rows, 5% border (10,000 cols = 625/block)
    "c2": lambda **kw: _sb(16, 12500, 11875, 625, 15, 25, 0, 4, **kw),
    # C3: DB 500,000^2, 8 blocks x 59,375 + 25,000 border rows/cols, K=8 split (A13)
    "c3": lambda **kw: _db(8, 59375, 25000, 10, 16, 0, 4, 10, 20, **kw),
    # C4: power-law 4,000,000^2 (A14/A15)
    "c4": lambda **kw: _pl(4_000_000, **kw),
    # C5: SB 64,000,000^2, 64 blocks x 1M rows, 2% border (1.28M cols = 20,000/block)
    "c5": lambda **kw: _sb(64, 1_000_000, 980_000, 20_000, 12, 20, 0, 3, **kw),
    # scaled-down stand-ins with the same structure (tests; oracle finishes in seconds)
    "c2s": lambda **kw: _sb(4, 1250, 1190, 60, 15, 25, 0, 4, **kw),
    "c3s": lambda **kw: _db(4, 2400, 400, 10, 16, 0, 4, 10, 20, **kw),
    "c4s": lambda **kw: _pl(60_000, Lmax=3000, band=2000, **kw),
    "c5s": lambda **kw: _sb(8, 5000, 4900, 100, 12, 20, 0, 3, **kw),
}


def params(name: str, **kw) -> dict:
    return PRESETS[name](**kw)


def make(name: str, variant: str = "real", seed: int = 0, **kw) -> Problem:
    """Generate preset ``name`` (c1..c5, or a scaled c2s..c5s) with overrides."""
    p = params(name, **kw)
    P = _Params()
    for k, v in p.items():
        setattr(P, k, v)
    P.variant = VARIANTS[variant]
    P.seed = seed
    lib = _load()
    rc = lib.synth_check(ctypes.byref(P))
    if rc:
        raise ValueError(f"synth: bad parameters for {name}: {rc}")
    m, n = int(P.m), int(P.n)
    row_perm = np.empty(m, dtype=np.int32)
    col_perm = np.empty(n, dtype=np.int32)
    row_len = np.empty(m, dtype=np.int64)
    assert lib.synth_structure(ctypes.byref(P), _ptr(row_perm), _ptr(col_perm), _ptr(row_len)) == 0
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(row_len, out=row_ptr[1:])
    del row_len
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float64)
    parts = np.empty(nnz, dtype=np.int32) if p["kind"] == DB else None
    col_inv = None
    if p.get("scramble"):
        col_inv = np.empty(n, dtype=np.int32)
        col_inv[col_perm] = np.arange(n, dtype=np.int32)
    assert lib.synth_fill(ctypes.byref(P), _ptr(row_perm), _ptr(col_inv), _ptr(row_ptr),
                          _ptr(col), _ptr(val), _ptr(parts)) == 0
    del col_inv
    blocks = None
    owner = None
    if p["kind"] == SB:
        K = p["K"]
        rbp = np.array([k * p["Rb"] for k in range(K + 1)] + [K * p["Rb"]], dtype=np.int64)
        cbp = np.array([k * p["Ci"] for k in range(K + 1)] + [n], dtype=np.int64)
        blocks = {"kind": 1, "K": K, "row_block_ptr": rbp, "col_block_ptr": cbp}
        if p["Rb"] == p["Ci"] + p["Bs"]:
            owner = np.empty(n, dtype=np.int32)
            assert lib.synth_sb_owner(ctypes.byref(P), _ptr(owner)) == 0
    elif p["kind"] == DB:
        K = p["K"]
        rbp = np.array([k * p["Rb"] for k in range(K + 1)] + [m], dtype=np.int64)
        cbp = np.array([k * p["Ci"] for k in range(K + 1)] + [n], dtype=np.int64)
        blocks = {"kind": 2, "K": K, "row_block_ptr": rbp, "col_block_ptr": cbp}
    scr = bool(p.get("scramble"))
    return Problem(name=name, m=m, n=n, row_ptr=row_ptr, col=col, val=val,
                   row_perm=row_perm if scr else None, col_perm=col_perm if scr else None,
                   blocks=blocks, parts=parts, n_parts=(p["K"] if p["kind"] == DB else 0),
                   owner=owner, variant=variant, seed=seed, params=p)


def random_csr(m: int, n: int, density: float, seed: int = 0, variant: str = "real",
               empty_rows: float = 0.0, rng=None):
    """Small random CSR (numpy; tests only): each row picks distinct sorted
    columns.  Returns (row_ptr int64, col int32, val float64)."""
    g = rng if rng is not None else np.random.default_rng(seed)
    rows = []
    for i in range(m):
        if empty_rows and g.random() < empty_rows:
            rows.append(np.zeros(0, dtype=np.int64))
            continue
        k = g.binomial(n, density) if n else 0
        rows.append(np.sort(g.choice(n, size=k, replace=False)) if k else np.zeros(0, dtype=np.int64))
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    row_ptr[1:] = np.cumsum([len(r) for r in rows])
    col = np.concatenate(rows).astype(np.int32) if rows else np.zeros(0, np.int32)
    nnz = len(col)
    if variant == "int":
        v = g.integers(1, 5, size=nnz) * g.choice([-1, 1], size=nnz)
        val = v.astype(np.float64)
    elif variant == "dyadic":
        val = np.round(g.uniform(-1, 1, size=nnz) * 1024) / 1024
    else:
        val = g.uniform(-1, 1, size=nnz)
    return row_ptr, col, val

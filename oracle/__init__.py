"""TEST INFRASTRUCTURE -- the CPU oracle for the convex-hull pre-filter.

Plain sequential fp64 implementation of Algorithm 1 of Carrasco et al.,
arXiv 2303.10581: eight extremes, octagon
(P:124), octagon test, stable compaction and an
exact monotone-chain hull.  The arithmetic lives in
``ch_oracle.c`` (compiled with ``-ffp-contract=off``); this module only
marshals numpy arrays.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with ``paper_2303_10581_b200`` and never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ch_oracle.c")
_LIB = os.path.join(_HERE, "libchoracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]

OK, EMPTY, NONFINITE = 0, 2, 3
SLOTS = ("R", "TR", "T", "TL", "L", "BL", "B", "BR")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Octagon(ctypes.Structure):
    _fields_ = [
        ("nv", ctypes.c_int32),
        ("degenerate", ctypes.c_int32),
        ("vidx", ctypes.c_int64 * 8),
        ("vx", ctypes.c_double * 8),
        ("vy", ctypes.c_double * 8),
        ("ex", ctypes.c_double * 8),
        ("ey", ctypes.c_double * 8),
        ("thr", ctypes.c_double * 8),
        ("xmin", ctypes.c_double),
        ("xmax", ctypes.c_double),
        ("ymin", ctypes.c_double),
        ("ymax", ctypes.c_double),
    ]


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        lib.oracle_admit.argtypes = [P, I64]
        lib.oracle_admit.restype = ctypes.c_int
        lib.oracle_extremes8.argtypes = [P, I64, P]
        lib.oracle_extremes8.restype = None
        lib.oracle_octagon_build.argtypes = [P, P, ctypes.c_int, ctypes.POINTER(_Octagon)]
        lib.oracle_octagon_build.restype = None
        lib.oracle_flags.argtypes = [P, I64, ctypes.POINTER(_Octagon), P]
        lib.oracle_flags.restype = None
        lib.oracle_compact.argtypes = [P, I64, I64, P]
        lib.oracle_compact.restype = I64
        lib.oracle_filter_compact.argtypes = [P, I64, ctypes.c_int, P, ctypes.POINTER(_Octagon), P, P]
        lib.oracle_filter_compact.restype = ctypes.c_int
        lib.oracle_filter_compact_exact.argtypes = [P, I64, P, P, P]
        lib.oracle_filter_compact_exact.restype = ctypes.c_int
        lib.oracle_orient_sign.argtypes = [ctypes.c_double] * 6
        lib.oracle_orient_sign.restype = ctypes.c_int
        lib.oracle_hull.argtypes = [P, P, I64, P]
        lib.oracle_hull.restype = I64
        _lib = lib
    return _lib


def _xy(xy) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(xy, dtype=np.float64).reshape(-1, 2))
    return a


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def admit(xy) -> int:
    a = _xy(xy)
    return _load().oracle_admit(_p(a), a.shape[0])


def extremes8(xy) -> np.ndarray:
    """Indices [R, TR, T, TL, L, BL, B, BR] (lowest index on ties)."""
    a = _xy(xy)
    if a.shape[0] < 1:
        raise ValueError("EmptySet")
    out = np.zeros(8, dtype=np.int64)
    _load().oracle_extremes8(_p(a), a.shape[0], _p(out))
    return out


def octagon(xy, idx8=None, certified: bool = True) -> dict:
    a = _xy(xy)
    if idx8 is None:
        idx8 = extremes8(a)
    idx8 = np.ascontiguousarray(idx8, dtype=np.int64)
    o = _Octagon()
    _load().oracle_octagon_build(_p(a), _p(idx8), int(certified), ctypes.byref(o))
    nv = o.nv
    return {
        "nv": nv,
        "degenerate": bool(o.degenerate),
        "vidx": np.array(o.vidx[:nv], dtype=np.int64),
        "vx": np.array(o.vx[:nv]),
        "vy": np.array(o.vy[:nv]),
        "ex": np.array(o.ex[:nv]),
        "ey": np.array(o.ey[:nv]),
        "thr": np.array(o.thr[:nv]),
        "bbox": (o.xmin, o.xmax, o.ymin, o.ymax),
        "_c": o,
    }


def flags(xy, certified: bool = True, oct_=None) -> np.ndarray:
    """uint8 keep flags: 1 = hull candidate."""
    a = _xy(xy)
    if oct_ is None:
        oct_ = octagon(a, certified=certified)
    out = np.zeros(a.shape[0], dtype=np.uint8)
    _load().oracle_flags(_p(a), a.shape[0], ctypes.byref(oct_["_c"]), _p(out))
    return out


def compact(keep, index_base: int = 0) -> np.ndarray:
    k = np.ascontiguousarray(keep, dtype=np.uint8)
    out = np.zeros(k.shape[0], dtype=np.int64)
    c = _load().oracle_compact(_p(k), k.shape[0], index_base, _p(out))
    return out[:c].copy()


def filter_compact(xy, certified: bool = True):
    """Algorithm 1 lines 1-3.  Returns (survivor indices, idx8, octagon dict)."""
    a = _xy(xy)
    n = a.shape[0]
    surv = np.zeros(max(n, 1), dtype=np.int64)
    idx8 = np.zeros(8, dtype=np.int64)
    cnt = np.zeros(1, dtype=np.int64)
    o = _Octagon()
    st = _load().oracle_filter_compact(_p(a), n, int(certified), _p(idx8), ctypes.byref(o), _p(surv), _p(cnt))
    if st == EMPTY:
        raise ValueError("EmptySet")
    if st == NONFINITE:
        raise ValueError("NonFinite")
    return surv[: cnt[0]].copy(), idx8


def filter_compact_exact(xy):
    """f3: survivors of the exact strict predicate (discard iff the exact
    orientation is > 0 on every octagon edge).  Returns (survivors, idx8)."""
    a = _xy(xy)
    n = a.shape[0]
    surv = np.zeros(max(n, 1), dtype=np.int64)
    idx8 = np.zeros(8, dtype=np.int64)
    cnt = np.zeros(1, dtype=np.int64)
    st = _load().oracle_filter_compact_exact(_p(a), n, _p(idx8), _p(surv), _p(cnt))
    if st == EMPTY:
        raise ValueError("EmptySet")
    if st == NONFINITE:
        raise ValueError("NonFinite")
    return surv[: cnt[0]].copy(), idx8


def orient_sign(a, b, c) -> int:
    return _load().oracle_orient_sign(float(a[0]), float(a[1]), float(b[0]), float(b[1]), float(c[0]), float(c[1]))


def hull(xy, idx=None) -> np.ndarray:
    """Strict CCW hull (input indices) of the points xy[idx], from the lexicographic minimum."""
    a = _xy(xy)
    if idx is None:
        idx = np.arange(a.shape[0], dtype=np.int64)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.zeros(idx.shape[0] + 1, dtype=np.int64)
    h = _load().oracle_hull(_p(a), _p(idx), idx.shape[0], _p(out))
    return out[:h].copy()


def hull_end_to_end(xy, certified: bool = True):
    """Algorithm 1: filter, compact, hull of the candidates."""
    surv, idx8 = filter_compact(xy, certified)
    return hull(xy, surv), surv, idx8

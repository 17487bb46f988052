"""ctypes loader for libchfilter.so (the C ABI of include/chfilter.h).

There is no fallback: if the shared library is missing and cannot be built,
or a call fails, this raises.  The filter never runs on the CPU.
"""
from __future__ import annotations

import ctypes
import os

from . import build as _build

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
DBL = ctypes.c_double
SZ = ctypes.c_size_t

CH_OK, CH_ERR_INVALID_ARG, CH_ERR_EMPTY, CH_ERR_NONFINITE = 0, 1, 2, 3
CH_ERR_MISALIGNED, CH_ERR_WORKSPACE, CH_ERR_CUDA, CH_ERR_PEER, CH_ERR_NCCL = 4, 5, 6, 7, 8
ABI_VERSION = 3
CH_NCCL_ID_BYTES = 128
CH_MAX_PEERS = 16
CH_CERTIFIED, CH_PLAIN, CH_EXACT = 0, 1, 2
CH_HULL_HOST = 4


class Extremes(ctypes.Structure):
    _fields_ = [("idx", I64 * 8), ("x", DBL * 8), ("y", DBL * 8)]


class Octagon(ctypes.Structure):
    _fields_ = [
        ("nv", I32), ("degenerate", I32), ("vidx", I64 * 8),
        ("vx", DBL * 8), ("vy", DBL * 8), ("ex", DBL * 8), ("ey", DBL * 8), ("thr", DBL * 8),
        ("bbox", DBL * 4), ("box", DBL * 4), ("has_box", I32), ("plain", I32),
        ("guess_edge", I32 * 8), ("cx", DBL), ("cy", DBL),
        ("f32_a", ctypes.c_float * 8), ("f32_b", ctypes.c_float * 8), ("f32_c", ctypes.c_float * 8),
        ("f32_dk", ctypes.c_float * 8), ("f32_delta", ctypes.c_float), ("has_f32", I32), ("exact", I32),
    ]


class Result(ctypes.Structure):
    _fields_ = [("count", I64), ("nonfinite", I32), ("degenerate", I32)]


class Stats(ctypes.Structure):
    _fields_ = [("n", I64), ("n_survivors", I64), ("n_hull", I64),
                ("ms_filter", DBL), ("ms_gather", DBL), ("ms_hull", DBL),
                ("ms_pass1", DBL), ("ms_pass2", DBL), ("ms_exchange", DBL)]


# name -> (restype, argtypes); every symbol declared in include/chfilter.h
SIGNATURES = {
    "ch_abi_version": (ctypes.c_int, []),
    "ch_status_str": (ctypes.c_char_p, [ctypes.c_int]),
    "ch_last_error": (ctypes.c_char_p, []),
    "ch_occupancy": (ctypes.c_int, [ctypes.c_int]),
    "ch_workspace_bytes": (SZ, [I64]),
    "ch_workspace_init": (ctypes.c_int, [P, SZ, P]),
    "ch_extremes8": (ctypes.c_int, [P, I64, I64, ctypes.c_int, P, ctypes.POINTER(Extremes),
                                    ctypes.POINTER(Octagon), P, SZ, P]),
    "ch_extremes8_f32": (ctypes.c_int, [P, I64, I64, ctypes.c_int, P, ctypes.POINTER(Extremes),
                                        ctypes.POINTER(Octagon), P, SZ, P]),
    "ch_combine8": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, P, SZ, P]),
    "ch_octagon_build": (ctypes.c_int, [ctypes.POINTER(Extremes), ctypes.c_int, ctypes.POINTER(Octagon)]),
    "ch_octagon_filter": (ctypes.c_int, [P, I64, ctypes.POINTER(Octagon), P, P, SZ, P]),
    "ch_filter_compact": (ctypes.c_int, [P, I64, I64, ctypes.POINTER(Octagon), P, P, P, SZ, P]),
    "ch_filter_compact_f32": (ctypes.c_int, [P, I64, I64, ctypes.POINTER(Octagon), P, P, P, SZ, P]),
    "ch_filter_f32": (ctypes.c_int, [P, I64, ctypes.c_int, P, ctypes.POINTER(I64), P, SZ, P]),
    "ch_read_result": (ctypes.c_int, [P, ctypes.POINTER(Result), P]),
    "ch_read_octagon": (ctypes.c_int, [P, ctypes.POINTER(Extremes), ctypes.POINTER(Octagon), P]),
    "ch_filter": (ctypes.c_int, [P, I64, ctypes.c_int, P, ctypes.POINTER(I64), P, SZ, P]),
    "ch_filter_async": (ctypes.c_int, [P, I64, ctypes.c_int, P, P, P, SZ, P]),
    "ch_filter_async_f32": (ctypes.c_int, [P, I64, ctypes.c_int, P, P, P, SZ, P]),
    "ch_filter_graph_create": (ctypes.c_int, [P, I64, ctypes.c_int, P, P, P, SZ, ctypes.POINTER(P)]),
    "ch_filter_graph_create_f32": (ctypes.c_int, [P, I64, ctypes.c_int, P, P, P, SZ, ctypes.POINTER(P)]),
    "ch_graph_launch": (ctypes.c_int, [P, P]),
    "ch_peer_handle_bytes": (SZ, []),
    "ch_peer_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.POINTER(P), P]),
    "ch_peer_open": (ctypes.c_int, [P, P]),
    "ch_peer_destroy": (ctypes.c_int, [P]),
    "ch_filter_step_peer": (ctypes.c_int, [P, P, I64, I64, ctypes.c_int, P, P, SZ, P]),
    "ch_filter_step_peer_f32": (ctypes.c_int, [P, P, I64, I64, ctypes.c_int, P, P, SZ, P]),
    "ch_peer_counts": (ctypes.c_int, [P, P, ctypes.POINTER(I64), ctypes.POINTER(I64), P]),
    "ch_exclusive_offset": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(I64), ctypes.POINTER(I64)]),
    "ch_comm_unique_id": (ctypes.c_int, [P]),
    "ch_comm_nccl_version": (ctypes.c_int, []),
    "ch_comm_init": (ctypes.c_int, [ctypes.POINTER(P), P, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "ch_comm_destroy": (ctypes.c_int, [P]),
    "ch_filter_compact_dist": (ctypes.c_int, [P, P, I64, I64, ctypes.c_int, P, ctypes.POINTER(I64),
                                              ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(Extremes),
                                              P, SZ, P]),
    "ch_filter_compact_dist_f32": (ctypes.c_int, [P, P, I64, I64, ctypes.c_int, P, ctypes.POINTER(I64),
                                                  ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(Extremes),
                                                  P, SZ, P]),
    "ch_comm_result": (ctypes.c_int, [P, P, ctypes.POINTER(I64), ctypes.POINTER(I64), P]),
    "ch_comm_step_times": (ctypes.c_int, [P, ctypes.POINTER(DBL), ctypes.POINTER(DBL), ctypes.POINTER(DBL)]),
    "ch_gather_survivors": (ctypes.c_int, [P, P, P, ctypes.c_int, ctypes.c_int, P, P, P, SZ, P]),
    "ch_hull_end_to_end_dist": (ctypes.c_int, [P, P, I64, I64, ctypes.c_int, P, ctypes.c_int, P,
                                               ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(Stats),
                                               P, SZ, P]),
    "ch_hull_gpu_pts_async": (ctypes.c_int, [P, P, I64, P, P, P, SZ, P]),
    "ch_graph_destroy": (ctypes.c_int, [P]),
    "ch_filter_host": (ctypes.c_int, [P, I64, ctypes.c_int, P, P, P, ctypes.POINTER(I64), P, SZ, P]),
    "ch_gather_points": (ctypes.c_int, [P, I64, P, I64, P, P]),
    "ch_hull_points": (ctypes.c_int, [P, P, I64, P, ctypes.POINTER(I64)]),
    "ch_hull_gpu_temp_bytes": (SZ, [I64]),
    "ch_hull_gpu": (ctypes.c_int, [P, I64, P, I64, P, ctypes.POINTER(I64), P, SZ, P]),
    "ch_hull_gpu_async": (ctypes.c_int, [P, I64, P, I64, P, P, P, SZ, P]),
    "ch_hull_workspace_bytes": (SZ, [I64]),
    "ch_hull_end_to_end": (ctypes.c_int, [P, I64, ctypes.c_int, P, ctypes.POINTER(I64), P,
                                          ctypes.POINTER(I64), ctypes.POINTER(Stats), P, SZ, P]),
}

_lib = None


class CHError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: status {status} ({detail})")
        self.status = status


def lib_path() -> str:
    return _build.LIB


def load():
    """Load (building in-tree first if stale and nvcc exists) the library."""
    global _lib
    if _lib is not None:
        return _lib
    path = _build.LIB
    try:
        path = _build.build()
    except Exception:
        if not os.path.exists(path):
            raise
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    lib.ch_orient_sign.restype = ctypes.c_int
    lib.ch_orient_sign.argtypes = [DBL] * 6
    if lib.ch_abi_version() != ABI_VERSION:
        raise RuntimeError("libchfilter ABI mismatch")
    _lib = lib
    return lib


def check(status: int, where: str):
    if status != CH_OK:
        lib = load()
        detail = (lib.ch_last_error() or b"").decode()
        raise CHError(status, where, f"{lib.ch_status_str(status).decode()}: {detail}")

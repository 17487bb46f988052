"""paper_2303_10581_b200 -- B200-native GPU octagon pre-filter for the 2D convex
hull (Carrasco et al., arXiv 2303.10581), exposed through a thin binding of
the C ABI in include/chfilter.h.

Every step of the filter runs in the CUDA kernels of libchfilter.so; this
module only marshals torch tensors (device memory, streams) into the C calls.
There is no CPU fallback: without a CUDA device or the library, calls raise.

Typical use::

    import torch, paper_2303_10581_b200 as chf
    xy = torch.randn(10**8, 2, dtype=torch.float64, device="cuda")
    ws = chf.Workspace(xy.shape[0])
    surv = chf.filter(xy, ws)                    # int64 survivor indices (Algorithm 1 l.1-3)
    hull, surv, stats = chf.hull_end_to_end(xy, ws)   # + the exact hull (l.4)
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import CHError, Extremes, Octagon, Result, Stats  # noqa: F401

SLOTS = ("R", "TR", "T", "TL", "L", "BL", "B", "BR")


def _stream(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor | None) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _points(xy: torch.Tensor) -> torch.Tensor:
    if not isinstance(xy, torch.Tensor) or xy.dtype not in (torch.float64, torch.float32):
        raise TypeError("points must be a float64 (or float32) torch tensor of shape [n, 2]")
    if xy.dim() != 2 or xy.shape[1] != 2 or not xy.is_contiguous():
        raise ValueError("points must be a contiguous [n, 2] tensor (AoS x, y)")
    if not xy.is_cuda:
        raise ValueError("points must be on a CUDA device (no CPU path)")
    return xy


def _points64(xy: torch.Tensor, what: str) -> torch.Tensor:
    """float64 points only: the hull and gather entry points read const double*."""
    xy = _points(xy)
    if xy.dtype != torch.float64:
        raise TypeError(f"{what} takes float64 points (got {xy.dtype}); widen float32 storage with .double()")
    return xy


def _ids(idx: torch.Tensor, xy: torch.Tensor, what: str) -> torch.Tensor:
    if not isinstance(idx, torch.Tensor) or idx.dtype != torch.int64 or idx.dim() != 1 or not idx.is_contiguous():
        raise TypeError(f"{what}: indices must be a contiguous 1-D int64 tensor")
    if idx.device != xy.device:
        raise ValueError(f"{what}: indices must be on the points' device")
    return idx


def _plain(plain: bool) -> int:
    """Predicate flags: True / "plain" -> CH_PLAIN, "exact" -> CH_EXACT,
    False / "certified" -> CH_CERTIFIED (DESIGN R4, f3)."""
    if plain == "exact":
        return _lib.CH_EXACT
    if plain is True or plain == "plain":
        return _lib.CH_PLAIN
    return _lib.CH_CERTIFIED


def _fn(lib, name: str, xy: torch.Tensor):
    """The float64 entry point, or its _f32 twin for float32 storage."""
    return getattr(lib, name + "_f32") if xy.dtype == torch.float32 else getattr(lib, name)


class Workspace:
    """Caller-owned scratch of ch_workspace_bytes(n) bytes, zero-filled once.
    hull=True sizes it for ch_hull_end_to_end's device hull too
    (ch_hull_workspace_bytes), so that call allocates nothing."""

    def __init__(self, n: int, device=None, stream=None, hull: bool = False):
        lib = _lib.load()
        self.capacity = int(n)
        self.hull = bool(hull)
        self.nbytes = int(lib.ch_hull_workspace_bytes(self.capacity) if hull else lib.ch_workspace_bytes(self.capacity))
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.buf = torch.zeros(self.nbytes, dtype=torch.uint8, device=dev)

    def ensure(self, n: int) -> "Workspace":
        if n > self.capacity:
            raise ValueError(f"workspace sized for {self.capacity} points, got {n}")
        return self

    @property
    def ptr(self):
        return ctypes.c_void_p(self.buf.data_ptr())


def _ws(ws: Workspace | None, n: int, device) -> Workspace:
    return ws.ensure(n) if ws is not None else Workspace(max(n, 1), device=device)


def extremes8(xy: torch.Tensor, ws: Workspace | None = None, index_base: int = 0, plain: bool = False,
              ext_out: torch.Tensor | None = None, stream=None):
    """Algorithm 1 line 1: the eight extremes and the octagon.
    Returns (Extremes, Octagon) host structs (synchronizes)."""
    lib = _lib.load()
    xy = _points(xy)
    n = xy.shape[0]
    ws = _ws(ws, n, xy.device)
    e, o = Extremes(), Octagon()
    _lib.check(_fn(lib, "ch_extremes8", xy)(_ptr(xy), n, index_base, _plain(plain), _ptr(ext_out), ctypes.byref(e),
                                ctypes.byref(o), ws.ptr, ws.nbytes, _stream(stream)), "ch_extremes8")
    return e, o


def extremes8_async(xy: torch.Tensor, ws: Workspace, index_base: int = 0, plain: bool = False,
                    ext_out: torch.Tensor | None = None, stream=None):
    """Enqueue K1 only (no synchronization)."""
    lib = _lib.load()
    xy = _points(xy)
    _lib.check(_fn(lib, "ch_extremes8", xy)(_ptr(xy), xy.shape[0], index_base, _plain(plain), _ptr(ext_out), None, None,
                                ws.ptr, ws.nbytes, _stream(stream)), "ch_extremes8")


def combine8(ext_all: torch.Tensor, world: int, ws: Workspace, plain: bool = False, stream=None):
    """Multi-GPU exchange step: combine `world` device ch_extremes records."""
    lib = _lib.load()
    _lib.check(lib.ch_combine8(_ptr(ext_all), world, _plain(plain), ws.ptr, ws.nbytes, _stream(stream)),
               "ch_combine8")


def octagon_build(ext: Extremes, plain: bool = False) -> Octagon:
    lib = _lib.load()
    o = Octagon()
    _lib.check(lib.ch_octagon_build(ctypes.byref(ext), _plain(plain), ctypes.byref(o)), "ch_octagon_build")
    return o


def octagon_filter(xy: torch.Tensor, ws: Workspace | None = None, oct_: Octagon | None = None,
                   out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Algorithm 1 line 2: the n-bit candidate vector as int32
    words (bit i%32 of word i//32).  Uses the workspace octagon unless oct_."""
    lib = _lib.load()
    xy = _points(xy)
    if xy.dtype != torch.float64:
        raise TypeError("octagon_filter takes float64 points")
    n = xy.shape[0]
    ws = _ws(ws, 0, xy.device)
    words = (n + 31) // 32
    if out is None:
        out = torch.empty(words, dtype=torch.int32, device=xy.device)
    _lib.check(lib.ch_octagon_filter(_ptr(xy), n, ctypes.byref(oct_) if oct_ is not None else None, _ptr(out),
                                     ws.ptr, ws.nbytes, _stream(stream)), "ch_octagon_filter")
    return out


def filter_compact(xy: torch.Tensor, ws: Workspace, index_base: int = 0, oct_: Octagon | None = None,
                   out: torch.Tensor | None = None, count: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Algorithm 1 lines 2-3 fused: enqueue K2 (async).  Survivors go to `out`
    (int64, capacity n); the count to `count` (device int64[1]) if given."""
    lib = _lib.load()
    xy = _points(xy)
    n = xy.shape[0]
    if out is None:
        out = torch.empty(max(n, 1), dtype=torch.int64, device=xy.device)
    _lib.check(_fn(lib, "ch_filter_compact", xy)(_ptr(xy), n, index_base, ctypes.byref(oct_) if oct_ is not None else None,
                                     _ptr(out), _ptr(count), ws.ptr, ws.nbytes, _stream(stream)),
               "ch_filter_compact")
    return out


def read_result(ws: Workspace, stream=None) -> Result:
    lib = _lib.load()
    r = Result()
    _lib.check(lib.ch_read_result(ws.ptr, ctypes.byref(r), _stream(stream)), "ch_read_result")
    return r


def read_octagon(ws: Workspace, stream=None):
    """(Extremes, Octagon) the last step on `ws` built on the device."""
    lib = _lib.load()
    e, o = Extremes(), Octagon()
    _lib.check(lib.ch_read_octagon(ws.ptr, ctypes.byref(e), ctypes.byref(o), _stream(stream)), "ch_read_octagon")
    return e, o


def filter(xy: torch.Tensor, ws: Workspace | None = None, plain: bool = False, out: torch.Tensor | None = None,
           stream=None) -> torch.Tensor:
    """One filter step (K1 + K2 + count readback): the survivor indices, in
    increasing order, as a view of `out`."""
    lib = _lib.load()
    xy = _points(xy)
    n = xy.shape[0]
    ws = _ws(ws, n, xy.device)
    if out is None:
        out = torch.empty(max(n, 1), dtype=torch.int64, device=xy.device)
    cnt = ctypes.c_int64(0)
    _lib.check(_fn(lib, "ch_filter", xy)(_ptr(xy), n, _plain(plain), _ptr(out), ctypes.byref(cnt), ws.ptr, ws.nbytes,
                             _stream(stream)), "ch_filter")
    return out[: cnt.value]


def filter_async(xy: torch.Tensor, ws: Workspace, out: torch.Tensor, count: torch.Tensor | None = None,
                 plain: bool = False, stream=None):
    """One filter step without synchronizing (K5 for n <= 2048, K6 for n <= 32768, else K1 + K2);
    the count goes to `count` (device int64[1]) and the workspace result."""
    lib = _lib.load()
    xy = _points(xy)
    _lib.check(_fn(lib, "ch_filter_async", xy)(_ptr(xy), xy.shape[0], _plain(plain), _ptr(out), _ptr(count),
                                                ws.ptr, ws.nbytes, _stream(stream)), "ch_filter_async")


class FilterGraph:
    """The filter_async step captured once as a CUDA graph (ch_filter_graph_create)
    and replayed by launch(): one host call per step.  The tensors are baked
    into the graph, so they are kept referenced here and must not move."""

    def __init__(self, xy: torch.Tensor, ws: Workspace, out: torch.Tensor, count: torch.Tensor | None = None,
                 plain: bool = False):
        lib = _lib.load()
        self._xy = _points(xy)
        self._keep = (ws, out, count)
        h = ctypes.c_void_p()
        _lib.check(_fn(lib, "ch_filter_graph_create", self._xy)(
            _ptr(self._xy), self._xy.shape[0], _plain(plain), _ptr(out), _ptr(count), ws.ptr, ws.nbytes,
            ctypes.byref(h)), "ch_filter_graph_create")
        self._h = h

    def launch(self, stream=None):
        _lib.check(_lib.load().ch_graph_launch(self._h, _stream(stream)), "ch_graph_launch")

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().ch_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def filter_host(h_xy: torch.Tensor, ws: Workspace, d_staging: torch.Tensor, d_out: torch.Tensor,
                h_out: torch.Tensor, plain: bool = False, stream=None) -> int:
    """End-to-end step from host memory (H2D copy, filter, D2H survivors)."""
    lib = _lib.load()
    if h_xy.is_cuda or h_xy.dtype != torch.float64 or not h_xy.is_contiguous():
        raise ValueError("h_xy must be a contiguous float64 host tensor")
    n = h_xy.shape[0]
    cnt = ctypes.c_int64(0)
    _lib.check(lib.ch_filter_host(_ptr(h_xy), n, _plain(plain), _ptr(d_staging), _ptr(d_out), _ptr(h_out),
                                  ctypes.byref(cnt), ws.ptr, ws.nbytes, _stream(stream)), "ch_filter_host")
    return cnt.value


def gather_points(xy: torch.Tensor, idx: torch.Tensor, index_base: int = 0, stream=None) -> torch.Tensor:
    """The coordinates of points idx - index_base of xy (device, [m, 2] float64)."""
    lib = _lib.load()
    xy = _points64(xy, "gather_points")
    idx = _ids(idx, xy, "gather_points")
    m = idx.shape[0]
    out = torch.empty(m, 2, dtype=torch.float64, device=xy.device)
    _lib.check(lib.ch_gather_points(_ptr(xy), index_base, _ptr(idx), m, _ptr(out), _stream(stream)),
               "ch_gather_points")
    return out


def hull_points(pts: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """Exact strict CCW hull (host, Algorithm 1 line 4) of pts[j] with ids[j]."""
    lib = _lib.load()
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    out = np.zeros(max(len(ids), 1), dtype=np.int64)
    h = ctypes.c_int64(0)
    _lib.check(lib.ch_hull_points(pts.ctypes.data_as(ctypes.c_void_p), ids.ctypes.data_as(ctypes.c_void_p),
                                  len(ids), out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(h)), "ch_hull_points")
    return out[: h.value].copy()


def hull_gpu(xy: torch.Tensor, surv: torch.Tensor, stream=None) -> np.ndarray:
    """f1: exact strict hull of the survivors `surv` (int64 device indices
    into xy) computed on the device; returns the hull ids (host)."""
    lib = _lib.load()
    xy = _points64(xy, "hull_gpu")
    surv = _ids(surv, xy, "hull_gpu")
    m = int(surv.shape[0])
    tb = int(lib.ch_hull_gpu_temp_bytes(m))
    tmp = torch.empty(max(tb, 1), dtype=torch.uint8, device=xy.device)
    # the ids land in pinned host memory (torch's caching host allocator):
    # a pageable buffer would make the copy, not the hull, the cost
    out = torch.empty(max(m, 1), dtype=torch.int64, pin_memory=True)
    h = ctypes.c_int64(0)
    _lib.check(lib.ch_hull_gpu(_ptr(xy), xy.shape[0], _ptr(surv), m, ctypes.c_void_p(out.data_ptr()),
                               ctypes.byref(h), _ptr(tmp), tb, _stream(stream)), "ch_hull_gpu")
    return out[: h.value].numpy()


def hull_gpu_async(xy: torch.Tensor, surv: torch.Tensor, tmp: torch.Tensor | None = None, stream=None):
    """f1 without host round trip: (hull ids, count) as device int64 tensors
    (the ids valid up to the count).  `tmp`: uint8 device scratch of
    ch_hull_gpu_temp_bytes(len(surv)) bytes (allocated if None)."""
    lib = _lib.load()
    xy = _points64(xy, "hull_gpu_async")
    surv = _ids(surv, xy, "hull_gpu_async")
    m = int(surv.shape[0])
    tb = int(lib.ch_hull_gpu_temp_bytes(m))
    if tmp is None or tmp.numel() < tb:
        tmp = torch.empty(max(tb, 1), dtype=torch.uint8, device=xy.device)
    ids = torch.empty(max(m, 1), dtype=torch.int64, device=xy.device)
    cnt = torch.empty(1, dtype=torch.int64, device=xy.device)
    _lib.check(lib.ch_hull_gpu_async(_ptr(xy), xy.shape[0], _ptr(surv), m, _ptr(ids), _ptr(cnt), _ptr(tmp), tb,
                                     _stream(stream)), "ch_hull_gpu_async")
    return ids, cnt


def hull_end_to_end(xy: torch.Tensor, ws: Workspace | None = None, plain: bool = False,
                    out: torch.Tensor | None = None, stream=None, host_hull: bool = False):
    """Algorithm 1: filter on the GPU, then the exact hull of the
    survivors on the device (default, f1) or on the host (host_hull=True).
    Returns (hull ids np.ndarray, survivors tensor, Stats).  A workspace made
    with Workspace(n, hull=True) also holds the device hull's scratch."""
    lib = _lib.load()
    xy = _points(xy)
    if xy.dtype != torch.float64:
        raise TypeError("hull_end_to_end takes float64 points")
    n = xy.shape[0]
    ws = ws.ensure(n) if ws is not None else Workspace(max(n, 1), device=xy.device, hull=not host_hull)
    if out is None:
        out = torch.empty(max(n, 1), dtype=torch.int64, device=xy.device)
    # pinned (page-locked, cached by torch) so the hull ids come back at full PCIe speed
    hull_t = torch.empty(max(n, 1), dtype=torch.int64, pin_memory=True)
    hull = hull_t.numpy()
    ns, nh, st = ctypes.c_int64(0), ctypes.c_int64(0), Stats()
    flags = _plain(plain) | (_lib.CH_HULL_HOST if host_hull else 0)
    _lib.check(lib.ch_hull_end_to_end(_ptr(xy), n, flags, _ptr(out), ctypes.byref(ns),
                                      hull.ctypes.data_as(ctypes.c_void_p), ctypes.byref(nh), ctypes.byref(st),
                                      ws.ptr, ws.nbytes, _stream(stream)), "ch_hull_end_to_end")
    return hull[: nh.value], out[: ns.value], st  # a view of the pinned buffer (no 0.8 GB copy)


def orient_sign(a, b, c) -> int:
    """The hull's exact orientation predicate (test hook)."""
    return _lib.load().ch_orient_sign(float(a[0]), float(a[1]), float(b[0]), float(b[1]), float(c[0]), float(c[1]))


def extremes_tuple(e: Extremes):
    return (np.array(e.idx[:], dtype=np.int64), np.array(e.x[:]), np.array(e.y[:]))


def octagon_dict(o: Octagon) -> dict:
    nv = o.nv
    return {"nv": nv, "degenerate": bool(o.degenerate), "vidx": np.array(o.vidx[:nv], dtype=np.int64),
            "vx": np.array(o.vx[:nv]), "vy": np.array(o.vy[:nv]), "ex": np.array(o.ex[:nv]),
            "ey": np.array(o.ey[:nv]), "thr": np.array(o.thr[:nv]), "bbox": tuple(o.bbox),
            "box": tuple(o.box), "has_box": bool(o.has_box)}

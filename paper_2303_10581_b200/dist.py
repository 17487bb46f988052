"""Multi-GPU filter: one process per GPU, points sharded by contiguous index
ranges (DESIGN R14), and the two real exchange steps of the path
(north_star):

  a4  all-gather of each rank's eight extremes (one 192-byte ch_extremes
      record per rank), then K3 (combine8 + octagon) repeated identically on
      every rank -> the global octagon, bit-identical to the 1-GPU result;
  a7  all-gather of the per-rank survivor counts and their exclusive scan ->
      each rank's offset in the one logical, globally ordered survivor array.

The survivors stay distributed (rank r owns [off_r, off_r + cnt_r)); the
physical gather to a root belongs to the separately timed hull stage
(`NcclComm.gather`, `NcclComm.hull_end_to_end`).

Three transports for the exchanges (DistFilter(exchange=...)), all driving
the same kernels through the C ABI:
  "nccl"   a library-owned NCCL communicator (ch_comm_*): the step is ONE C
           call (ch_filter_compact_dist: K1, ncclAllGather, K3, K2,
           ncclAllGather, scan); torch.distributed only broadcasts the
           128-byte ncclUniqueId once;
  "peer"   fused into the kernels over cudaIpc-mapped peer memory
           (ch_filter_step_peer): K1's last CTA stores its record into every
           peer's buffer, K3 acquires them, K2's last CTA stores its count --
           no collective launches at all;
  "torch"  torch.distributed all-gathers (NCCL or gloo) around ch_extremes8 /
           ch_combine8 / ch_filter_compact; the offsets from
           ch_exclusive_offset.  Works with gloo, so several ranks can share
           one GPU in tests (NCCL refuses two ranks on one device).

This module only marshals arguments; every step of the path, including the
scan, runs in the library.  The collective helpers also work on CPU tensors
with gloo, which is how the host logic is tested without GPUs
(tests/test_dist_gloo.py).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import Workspace, _fn, _lib, _plain, _points, _ptr, _stream, combine8, extremes8_async, filter_compact
from ._lib import CHError

EXT_WORDS = 24  # ch_extremes = int64 idx[8] + double x[8] + double y[8]
EXCHANGES = ("nccl", "peer", "torch")


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Rank r owns global points [floor(r n / W), floor((r + 1) n / W))."""
    return (rank * n) // world, ((rank + 1) * n) // world


def pack_extremes(idx, x, y) -> torch.Tensor:
    """A ch_extremes record as 24 int64 words (x, y as their bit patterns).
    idx = -1 marks an empty shard (ignored by the combine)."""
    w = np.empty(EXT_WORDS, dtype=np.int64)
    w[0:8] = np.asarray(idx, dtype=np.int64)
    w[8:16] = np.asarray(x, dtype=np.float64).view(np.int64)
    w[16:24] = np.asarray(y, dtype=np.float64).view(np.int64)
    return torch.from_numpy(w)


def unpack_extremes(words) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    w = np.asarray(words.cpu() if isinstance(words, torch.Tensor) else words, dtype=np.int64).reshape(-1, EXT_WORDS)
    return w[:, 0:8].copy(), w[:, 8:16].view(np.float64).copy(), w[:, 16:24].view(np.float64).copy()


def empty_record(device) -> torch.Tensor:
    t = pack_extremes([-1] * 8, [0.0] * 8, [0.0] * 8)
    return t.to(device)


def _all_gather_flat(out: torch.Tensor, inp: torch.Tensor, group=None) -> torch.Tensor:
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp, group=group)   # one NCCL all-gather, in place
    else:  # gloo (CPU tests, and single-GPU multi-rank tests: staged through host memory)
        hin = inp.cpu()
        parts = list(torch.empty(out.numel(), dtype=out.dtype).chunk(dist.get_world_size(group)))
        dist.all_gather(parts, hin, group=group)
        out.copy_(torch.cat(parts))
    return out


def exchange_extremes(ext_local: torch.Tensor, group=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """a4 over torch.distributed: all-gather one record per rank ->
    [world * 24] int64 (rank order)."""
    world = dist.get_world_size(group)
    if out is None:
        out = torch.empty(world * EXT_WORDS, dtype=torch.int64, device=ext_local.device)
    return _all_gather_flat(out, ext_local, group)


def exclusive_offsets(count: torch.Tensor, group=None, out: torch.Tensor | None = None):
    """a7 over torch.distributed: all-gather of the int64 counts (device);
    `offsets_from_counts` turns them into (offset, total)."""
    world = dist.get_world_size(group)
    if out is None:
        out = torch.empty(world, dtype=torch.int64, device=count.device)
    return _all_gather_flat(out, count.reshape(1), group)


def offsets_from_counts(counts, rank: int) -> tuple[int, int]:
    """(exclusive offset of `rank`, total) -- ch_exclusive_offset (the scan
    runs in the library)."""
    c = np.ascontiguousarray([int(v) for v in (counts.tolist() if isinstance(counts, torch.Tensor) else counts)],
                             dtype=np.int64)
    off, tot = ctypes.c_int64(0), ctypes.c_int64(0)
    _lib.check(_lib.load().ch_exclusive_offset(c.ctypes.data_as(ctypes.c_void_p), len(c), rank, ctypes.byref(off),
                                               ctypes.byref(tot)), "ch_exclusive_offset")
    return off.value, tot.value


def agree_status(status: int, group=None) -> int:
    """The worst (largest) ch_status over the ranks, known to every rank, so
    that a non-finite coordinate or a late peer seen by one rank makes every
    rank raise instead of some ranks returning a result built from it."""
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([int(status)], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(t.item())


def broadcast_bytes(payload: bytes | None, nbytes: int, src: int = 0, group=None) -> bytes:
    """Broadcast `nbytes` bytes from rank `src` over the process group (the
    ncclUniqueId hand-off; a CUDA tensor for the NCCL backend)."""
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    if dist.get_rank(group) == src:
        assert payload is not None and len(payload) == nbytes
        t.copy_(torch.tensor(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(t, src=dist.get_global_rank(group, src) if group is not None else src, group=group)
    return bytes(t.cpu().numpy())


class NcclComm:
    """The library-owned NCCL communicator of one rank (ch_comm_*).  Rank 0
    creates the ncclUniqueId; torch.distributed broadcasts it (with a status
    byte, so a failure on rank 0 fails every rank); every rank then calls the
    collective ch_comm_init.  Without an initialized process group it is a
    world-size-1 communicator (tests on one GPU)."""

    def __init__(self, group=None, device=None):
        lib = _lib.load()
        self._h = None
        grouped = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if grouped else 0
        self.world = dist.get_world_size(group) if grouped else 1
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        nb = _lib.CH_NCCL_ID_BYTES
        uid = (ctypes.c_uint8 * nb)()
        ok = 1
        if self.rank == 0:
            ok = int(lib.ch_comm_unique_id(uid) == _lib.CH_OK)
        payload = bytes([ok]) + bytes(uid)
        if grouped and self.world > 1:
            payload = broadcast_bytes(payload if self.rank == 0 else None, nb + 1, 0, group)
        if not payload[0]:
            detail = (lib.ch_last_error() or b"").decode() if self.rank == 0 else "on rank 0"
            raise CHError(_lib.CH_ERR_NCCL, "ch_comm_unique_id", detail)
        uid = (ctypes.c_uint8 * nb).from_buffer_copy(payload[1:])
        h = ctypes.c_void_p()
        _lib.check(lib.ch_comm_init(ctypes.byref(h), uid, self.rank, self.world, dev.index or 0), "ch_comm_init")
        self._h = h

    @property
    def handle(self):
        return self._h

    def step(self, xy, n_local: int, n_global: int, ws: Workspace, out: torch.Tensor, plain=False, sync=False,
             stream=None):
        """One sharded step (ch_filter_compact_dist).  sync=False: enqueue only
        (result() later); sync=True: returns (count, offset, total)."""
        lib = _lib.load()
        c, o, t = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
        refs = (ctypes.byref(c), ctypes.byref(o), ctypes.byref(t)) if sync else (None, None, None)
        fn = lib.ch_filter_compact_dist_f32 if xy.dtype == torch.float32 else lib.ch_filter_compact_dist
        _lib.check(fn(self._h, _ptr(xy), n_local, n_global, _plain(plain), _ptr(out), *refs, None, ws.ptr,
                      ws.nbytes, _stream(stream)), "ch_filter_compact_dist")
        return (c.value, o.value, t.value) if sync else None

    def result(self, stream=None) -> tuple[list[int], int, int]:
        """(every rank's count, this rank's offset, total) of the last step;
        raises on every rank if any shard was non-finite."""
        counts = (ctypes.c_int64 * self.world)()
        o, t = ctypes.c_int64(0), ctypes.c_int64(0)
        _lib.check(_lib.load().ch_comm_result(self._h, counts, ctypes.byref(o), ctypes.byref(t), _stream(stream)),
                   "ch_comm_result")
        return list(counts), o.value, t.value

    def step_times(self) -> tuple[float, float, float]:
        """(pass 1, exchanges, pass 2) device milliseconds of the last step."""
        a, b, c = ctypes.c_double(0), ctypes.c_double(0), ctypes.c_double(0)
        _lib.check(_lib.load().ch_comm_step_times(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)),
                   "ch_comm_step_times")
        return a.value, b.value, c.value

    def gather(self, xy, local: torch.Tensor, root: int = 0, with_points: bool = True, stream=None):
        """The last step's survivors (ids, and coordinates) gathered to `root`
        in global order (ch_gather_survivors).  Returns (ids, pts) on the
        root, (None, None) elsewhere."""
        lib = _lib.load()
        counts, _, total = self.result(stream)
        dev = local.device
        is_root = self.rank == root
        ids = torch.empty(max(total, 1), dtype=torch.int64, device=dev) if is_root else None
        pts = torch.empty(max(total, 1), 2, dtype=torch.float64, device=dev) if is_root and with_points else None
        mine = counts[self.rank]
        tmp = (torch.empty(max(mine, 1), 2, dtype=torch.float64, device=dev)
               if with_points and not is_root else None)
        _lib.check(lib.ch_gather_survivors(self._h, _ptr(xy), _ptr(local), root, int(with_points), _ptr(ids),
                                           _ptr(pts), _ptr(tmp), 0 if tmp is None else tmp.numel() * 8,
                                           _stream(stream)), "ch_gather_survivors")
        if not is_root:
            return None, None
        return ids[:total], (pts[:total] if pts is not None else None)

    def hull_end_to_end(self, xy, n_local: int, n_global: int, ws: Workspace, out: torch.Tensor, root: int = 0,
                        plain=False, stream=None):
        """Algorithm 1 on W GPUs (ch_hull_end_to_end_dist): the step, the
        gather to `root` and the device hull there.  Returns (hull ids
        np.ndarray -- empty off the root, total survivors, Stats)."""
        lib = _lib.load()
        cap = max(n_global, 1) if self.rank == root else 1
        hull = np.zeros(cap, dtype=np.int64)
        nh, ns, st = ctypes.c_int64(0), ctypes.c_int64(0), _lib.Stats()
        _lib.check(lib.ch_hull_end_to_end_dist(self._h, _ptr(xy), n_local, n_global, _plain(plain), _ptr(out), root,
                                               hull.ctypes.data_as(ctypes.c_void_p), ctypes.byref(nh),
                                               ctypes.byref(ns), ctypes.byref(st), ws.ptr, ws.nbytes,
                                               _stream(stream)), "ch_hull_end_to_end_dist")
        return hull[: nh.value].copy(), ns.value, st

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().ch_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PeerExchange:
    """The fused-exchange endpoint of one rank (ch_peer_*): its exchange
    buffer's IPC handle is all-gathered once over the process group (the only
    use of torch.distributed on this path) and the peers' buffers mapped."""

    def __init__(self, group=None):
        lib = _lib.load()
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._h = None
        if self.world > _lib.CH_MAX_PEERS:
            raise ValueError(f"peer exchange supports at most {_lib.CH_MAX_PEERS} ranks")
        hb = int(lib.ch_peer_handle_bytes())
        mine = (ctypes.c_uint8 * hb)()
        h = ctypes.c_void_p()
        ok = lib.ch_peer_create(self.rank, self.world, ctypes.byref(h), mine) == _lib.CH_OK
        if ok:
            self._h = h
        # every rank takes part in both gathers, so a failure anywhere is
        # seen everywhere and all ranks fall back together
        allh = self._gather(bytes([int(ok)]) + bytes(mine), group)
        if not all(allh[r * (hb + 1)] for r in range(self.world)):
            self.close()
            raise RuntimeError("peer exchange unavailable on some rank (ch_peer_create)")
        handles = b"".join(allh[r * (hb + 1) + 1:(r + 1) * (hb + 1)] for r in range(self.world))
        buf = (ctypes.c_uint8 * len(handles)).from_buffer_copy(handles)
        st = lib.ch_peer_open(self._h, buf)
        oks = self._gather(bytes([int(st == _lib.CH_OK)]), group)
        if not all(oks):
            detail = (lib.ch_last_error() or b"").decode() if st != _lib.CH_OK else "on another rank"
            self.close()
            raise RuntimeError(f"peer exchange unavailable (ch_peer_open: {detail})")

    @staticmethod
    def _gather(payload: bytes, group) -> bytes:
        t = torch.tensor(bytearray(payload), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        out = torch.empty(dist.get_world_size(group) * len(payload), dtype=torch.uint8, device=t.device)
        _all_gather_flat(out, t, group)
        return bytes(out.cpu().numpy())

    @property
    def handle(self):
        return self._h

    def step(self, xy, n_local: int, index_base: int, ws: Workspace, out: torch.Tensor, plain=False, stream=None):
        lib = _lib.load()
        _lib.check(_fn(lib, "ch_filter_step_peer", xy)(self._h, _ptr(xy), n_local, index_base, _plain(plain),
                                                       _ptr(out), ws.ptr, ws.nbytes, _stream(stream)),
                   "ch_filter_step_peer")

    def counts_status(self, stream=None) -> tuple[int, list[int], int, int]:
        """(ch_status, every rank's count, this rank's offset, total) without
        raising (the caller agrees on the status first)."""
        c = (ctypes.c_int64 * self.world)()
        o, t = ctypes.c_int64(0), ctypes.c_int64(0)
        st = _lib.load().ch_peer_counts(self._h, c, ctypes.byref(o), ctypes.byref(t), _stream(stream))
        return st, list(c), o.value, t.value

    def counts(self, stream=None) -> list[int]:
        st, c, _, _ = self.counts_status(stream)
        _lib.check(st, "ch_peer_counts")
        return c

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().ch_peer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DistFilter:
    """Per-rank state for the sharded filter step (all device buffers are
    allocated once; `step` only enqueues work)."""

    def __init__(self, n_global: int, xy_local: torch.Tensor, group=None, plain: bool = False,
                 exchange: str = "nccl"):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.n_global = int(n_global)
        self.lo, self.hi = shard_range(self.n_global, self.world, self.rank)
        self.n_local = self.hi - self.lo
        if xy_local.shape[0] != self.n_local:
            raise ValueError("local shard size does not match shard_range")
        self.xy = _points(xy_local) if self.n_local > 0 else xy_local
        dev = xy_local.device
        self.plain = plain
        self.ws = Workspace(max(self.n_local, 1), device=dev)
        self.out = torch.empty(max(self.n_local, 1), dtype=torch.int64, device=dev)
        if exchange not in EXCHANGES:
            raise ValueError(f"exchange must be one of {EXCHANGES}")
        self.exchange = exchange
        self.peer = PeerExchange(group) if exchange == "peer" else None
        self.comm = NcclComm(group, device=dev) if exchange == "nccl" else None
        if exchange == "torch":
            self.ext_local = empty_record(dev)
            self.ext_all = torch.empty(self.world * EXT_WORDS, dtype=torch.int64, device=dev)
            self.count = torch.zeros(1, dtype=torch.int64, device=dev)
            self.counts = torch.empty(self.world, dtype=torch.int64, device=dev)

    def step(self, xy_local: torch.Tensor | None = None):
        """One step, enqueued (no host synchronization)."""
        xy = self.xy if xy_local is None else xy_local
        if self.comm is not None:   # one C call: K1, NCCL all-gather, K3, K2, NCCL all-gather, scan
            self.comm.step(xy, self.n_local, self.n_global, self.ws, self.out, plain=self.plain)
            return
        if self.peer is not None:   # the exchanges fused into K1 / K3 / K2
            self.peer.step(xy, self.n_local, self.lo, self.ws, self.out, plain=self.plain)
            return
        if self.n_local > 0:
            extremes8_async(xy, self.ws, index_base=self.lo, plain=self.plain, ext_out=self.ext_local)
        exchange_extremes(self.ext_local, self.group, out=self.ext_all)
        combine8(self.ext_all, self.world, self.ws, plain=self.plain)
        if self.n_local > 0:
            filter_compact(xy, self.ws, index_base=self.lo, out=self.out, count=self.count)
        exclusive_offsets(self.count, self.group, out=self.counts)

    def _check_all_ranks(self, st_local: int):
        """This rank's workspace status (non-finite input, late peer) combined
        with every other rank's: all ranks raise, or none does."""
        lib = _lib.load()
        res = _lib.Result()
        st = lib.ch_read_result(self.ws.ptr, ctypes.byref(res), _stream(None))
        if st_local != _lib.CH_OK:
            st = st_local
        worst = agree_status(st, self.group)
        if worst != _lib.CH_OK:
            detail = (lib.ch_last_error() or b"").decode() if st != _lib.CH_OK else "reported by another rank"
            raise CHError(worst, "DistFilter.step", f"{lib.ch_status_str(worst).decode()}: {detail}")

    def result(self):
        """(local survivor indices (device view), offset, total) -- synchronizes.
        Raises CHError on every rank if any rank saw a non-finite coordinate
        or a peer exchange timeout."""
        if self.comm is not None:   # every rank sees every rank's flags (library)
            counts, off, total = self.comm.result()
            return self.out[: counts[self.rank]], off, total
        if self.peer is not None:
            st, c, off, total = self.peer.counts_status()
            self._check_all_ranks(st)
            return self.out[: c[self.rank]], off, total
        self._check_all_ranks(_lib.CH_OK)
        off, total = offsets_from_counts(self.counts, self.rank)
        cnt = int(self.counts[self.rank].item())
        return self.out[:cnt], off, total

    def close(self):
        for x in (self.peer, self.comm):
            if x is not None:
                x.close()

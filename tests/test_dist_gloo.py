"""Multi-process (world_size 2, gloo, CPU) tests of the sharded path's host
logic: contiguous shards, the extremes exchange (a4), the count exchange and
exclusive scan (a7).  The per-shard compute is played by the oracle here (no
GPU); the GPU kernels of the same decomposition are covered by
tests/test_gpu_parity.py::test_index_base_and_sharded_combine_world_independence."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2303_10581_b200 import dist as chdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _combine_oracle(recs_idx, recs_x, recs_y):
    """Global extremes from per-rank candidates: the oracle's own argmax over
    the candidate points ordered by global index (lowest index wins ties)."""
    cand = {}
    for r in range(recs_idx.shape[0]):
        for k in range(8):
            i = int(recs_idx[r, k])
            if i >= 0:
                cand[i] = (recs_x[r, k], recs_y[r, k])
    gids = sorted(cand)
    pts = np.array([cand[g] for g in gids], dtype=np.float64)
    loc = oracle.extremes8(pts)
    return np.array([gids[i] for i in loc], dtype=np.int64)


def _worker(rank, world, port, n, dist_name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = synth.points(dist_name, n, seed=3).numpy()
        lo, hi = chdist.shard_range(n, world, rank)
        shard = synth.points(dist_name, n, seed=3, lo=lo, hi=hi).numpy()
        assert np.array_equal(shard, full[lo:hi])          # generator is world-size independent
        # a4: local extremes (global indices) -> exchange -> combine
        if hi > lo:
            li = oracle.extremes8(shard)
            rec = chdist.pack_extremes(li + lo, shard[li, 0], shard[li, 1])
        else:
            rec = chdist.empty_record("cpu")
        allrec = chdist.exchange_extremes(rec)
        ri, rx, ry = chdist.unpack_extremes(allrec)
        assert ri.shape == (world, 8)
        gidx = _combine_oracle(ri, rx, ry)
        assert np.array_equal(gidx, oracle.extremes8(full))
        # a7: survivors of the shard under the global octagon, counts exchanged
        o = oracle.octagon(full, gidx)
        keep = oracle.flags(shard, oct_=o) if hi > lo else np.zeros(0, np.uint8)
        surv = oracle.compact(keep, index_base=lo)
        counts = chdist.exclusive_offsets(torch.tensor([len(surv)], dtype=torch.int64))
        off, total = chdist.offsets_from_counts(counts, rank)
        want, _ = oracle.filter_compact(full)
        assert total == len(want)
        assert np.array_equal(want[off: off + len(surv)], surv)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dist_name,n", [("normal", 20_011), ("displaced", 9_999), ("circle", 3), ("normal", 1)])
def test_gloo_world2_exchange_matches_single(dist_name, n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, dist_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}:\n{msg}"


def test_shard_range_partition():
    for n in (0, 1, 7, 10 ** 9 + 3):
        for W in (1, 2, 3, 4, 8):
            rs = [chdist.shard_range(n, W, r) for r in range(W)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            for (a, b), (c, d) in zip(rs, rs[1:]):
                assert b == c
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def test_pack_unpack_roundtrip():
    idx = np.arange(8, dtype=np.int64) * 1000 + 5
    x = np.array([0.5, -0.0, 1e-300, -3.25, 7.0, 1.0 / 3, 2.0 ** 60, -1e10])
    y = x[::-1].copy()
    t = chdist.pack_extremes(idx, x, y)
    assert t.dtype == torch.int64 and t.numel() == 24
    i2, x2, y2 = chdist.unpack_extremes(t)
    assert np.array_equal(i2[0], idx)
    assert np.array_equal(x2[0].view(np.int64), x.view(np.int64))
    assert np.array_equal(y2[0].view(np.int64), y.view(np.int64))


def _peer_fallback_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        try:
            chdist.PeerExchange()
            q.put((rank, "created"))
        except RuntimeError as e:
            q.put((rank, "unavailable: " + str(e)))
        dist.barrier()   # no rank is left hanging in a collective
        q.put((rank, "done"))
    finally:
        dist.destroy_process_group()


def test_peer_exchange_failure_is_collective():
    """Without a GPU ch_peer_create fails; every rank must see the failure
    (and fall back together) rather than some ranks waiting in the handle
    all-gather -- the consistency logic of PeerExchange, on CPU."""
    if torch.cuda.is_available():
        pytest.skip("needs a machine without a GPU")
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_peer_fallback_worker, args=(r, world, port, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    msgs = [q.get(timeout=120) for _ in range(2 * world)]
    for p_ in procs:
        p_.join(timeout=60)
    status = [m[1] for m in msgs if m[1] != "done"]
    assert len(status) == world and all(m.startswith("unavailable") for m in status), status
    assert sum(m[1] == "done" for m in msgs) == world


def _comm_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # the ncclUniqueId hand-off: rank 0's bytes reach every rank
        payload = bytes(range(129)) if rank == 0 else None
        got = chdist.broadcast_bytes(payload, 129, 0)
        assert got == bytes(range(129)), got[:8]
        # a status seen on one rank is raised on every rank
        worst = chdist.agree_status(3 if rank == world - 1 else 0)
        assert worst == 3
        # a7's scan runs in the library (ch_exclusive_offset)
        counts = [5, 0, 7, 11][:world]
        assert chdist.offsets_from_counts(counts, rank) == (sum(counts[:rank]), sum(counts))
        # without a GPU ch_comm_init fails on every rank, none hangs
        try:
            chdist.NcclComm(device="cuda:0")
            q.put((rank, "created"))
        except Exception as e:
            q.put((rank, "failed: " + type(e).__name__))
        dist.barrier()
        q.put((rank, "done"))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_nccl_comm_host_logic_world(world):
    """The host side of the library-owned NCCL communicator over gloo on CPU:
    unique-id broadcast, status agreement, the scan, and a collective failure
    of ch_comm_init when there is no GPU."""
    if torch.cuda.is_available():
        pytest.skip("needs a machine without a GPU")
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_comm_worker, args=(r, world, port, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    msgs = [q.get(timeout=120) for _ in range(2 * world)]
    for p_ in procs:
        p_.join(timeout=60)
    status = [m[1] for m in msgs if m[1] != "done"]
    assert len(status) == world and all(m.startswith("failed") for m in status), status


def test_exclusive_offset_abi():
    import ctypes
    from paper_2303_10581_b200 import _lib
    lib = _lib.load()
    c = np.array([3, 0, 9, 2], dtype=np.int64)
    o, t = ctypes.c_int64(0), ctypes.c_int64(0)
    for r in range(4):
        assert lib.ch_exclusive_offset(c.ctypes.data_as(ctypes.c_void_p), 4, r, ctypes.byref(o), ctypes.byref(t)) == 0
        assert (o.value, t.value) == (int(c[:r].sum()), 14)
    assert lib.ch_exclusive_offset(c.ctypes.data_as(ctypes.c_void_p), 4, 4, None, None) == 1
    bad = np.array([1, -1], dtype=np.int64)
    assert lib.ch_exclusive_offset(bad.ctypes.data_as(ctypes.c_void_p), 2, 0, None, None) == 1

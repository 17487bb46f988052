"""Multi-GPU paths through the C ABI against the oracle:

* the library-owned NCCL communicator (ch_comm_*, ch_filter_compact_dist,
  ch_gather_survivors, ch_hull_end_to_end_dist) at world size 1 on one GPU;
* one process per GPU over NCCL -- exchange "nccl" (library comm), "peer"
  (cudaIpc over NVLink) and "torch" (torch.distributed NCCL all-gathers) --
  at W = 2 and W = every GPU of the box, skipped on a 1-GPU box.

Every rank's survivors, offsets and totals, the extremes, and the hull
gathered to the root must equal the oracle on the full array."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import paper_2303_10581_b200 as chf
import synth
from paper_2303_10581_b200 import dist as chdist

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ------------------------------------------------------------ world size 1 --
@pytest.mark.parametrize("dist_name,storage", [("displaced", "f64"), ("normal", "f64"), ("circle", "f32")])
def test_nccl_comm_world1_step_gather_hull(dist_name, storage):
    """ch_comm at W = 1 (NCCL collectives on one rank): the step equals the
    oracle; the gather to the root returns the survivors and their
    coordinates; the distributed end-to-end hull equals the oracle hull."""
    assert chf._lib.load().ch_comm_nccl_version() > 0
    n = 1_000_003
    xy = synth.points(dist_name, n, seed=6, device=DEV)
    if storage == "f32":
        xy = xy.float()
    xn = xy.double().cpu().numpy()
    want, idx8 = oracle.filter_compact(xn)
    comm = chdist.NcclComm()
    ws = chf.Workspace(n)
    out = torch.empty(n, dtype=torch.int64, device=DEV)
    for k in range(3):                      # sync and async steps, repeated
        if k == 1:
            comm.step(xy, n, n, ws, out)
            counts, off, total = comm.result()
            cnt = counts[0]
        else:
            cnt, off, total = comm.step(xy, n, n, ws, out, sync=True)
        assert (off, total, cnt) == (0, len(want), len(want))
        assert np.array_equal(out[:cnt].cpu().numpy(), want)
    e, o = chf.read_octagon(ws)
    assert np.array_equal(np.array(e.idx[:]), idx8)
    p1, ex, p2 = comm.step_times()
    assert p1 > 0 and ex > 0 and p2 > 0
    if storage == "f64":
        ids, pts = comm.gather(xy, out[:cnt])
        assert np.array_equal(ids.cpu().numpy(), want)
        assert np.array_equal(pts.cpu().numpy(), xn[want])
        hull, total, st = comm.hull_end_to_end(xy, n, n, ws, out)
        assert total == len(want)
        assert np.array_equal(hull, oracle.hull(xn, want))
        assert st.n_hull == len(hull) and st.ms_pass1 > 0 and st.ms_pass2 > 0
    comm.close()


def test_nccl_comm_world1_nonfinite_and_arguments():
    comm = chdist.NcclComm()
    n = 100_000
    xy = synth.points("normal", n, seed=1, device=DEV)
    xy[777, 1] = float("nan")
    ws = chf.Workspace(n)
    out = torch.empty(n, dtype=torch.int64, device=DEV)
    with pytest.raises(chf.CHError) as ei:
        comm.step(xy, n, n, ws, out, sync=True)
    assert ei.value.status == 3
    with pytest.raises(chf.CHError) as ei:
        comm.step(xy, n - 1, n, ws, out, sync=True)      # not the R14 shard size
    assert ei.value.status == 1
    comm.close()


def test_hull_gpu_pts_matches_hull_gpu():
    """ch_hull_gpu_pts_async (the root's hull of gathered coordinates) equals
    ch_hull_gpu on the same survivors, for sets with duplicates and ties."""
    import ctypes
    lib = chf._lib.load()
    rng = np.random.default_rng(3)
    grid = rng.integers(-40, 41, size=(200_000, 2)).astype(np.float64)
    for xy_np in (grid, synth.points("circle", 300_000, seed=2).numpy()):
        xy = torch.tensor(xy_np, device=DEV)
        surv = chf.filter(xy)
        m = int(surv.shape[0])
        pts = chf.gather_points(xy, surv)
        tb = int(lib.ch_hull_gpu_temp_bytes(m))
        tmp = torch.empty(tb, dtype=torch.uint8, device=DEV)
        hull = torch.empty(m + 1, dtype=torch.int64, device=DEV)
        nh = torch.zeros(1, dtype=torch.int64, device=DEV)
        assert lib.ch_hull_gpu_pts_async(chf._ptr(pts), chf._ptr(surv), m, chf._ptr(hull), chf._ptr(nh),
                                         chf._ptr(tmp), tb, chf._stream(None)) == 0
        got = hull[: int(nh.item())].cpu().numpy()
        assert np.array_equal(got, chf.hull_gpu(xy, surv))
        assert np.array_equal(got, oracle.hull(xy_np, surv.cpu().numpy()))


# --------------------------------------------------- one process per GPU --
def _rank_worker(rank, world, port, n, dist_name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["CH_PEER_TIMEOUT_MS"] = "20000"
    import torch.distributed as tdist
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    tdist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        lo, hi = chdist.shard_range(n, world, rank)
        xy = synth.points(dist_name, n, seed=8, device=dev, lo=lo, hi=hi)
        res = {}
        for exchange in chdist.EXCHANGES:
            df = chdist.DistFilter(n, xy, exchange=exchange)
            steps = []
            for _ in range(3):
                df.out.fill_(-1)
                df.step()
                loc, off, total = df.result()
                steps.append((off, total, loc.cpu().numpy()))
            res[exchange] = steps
            tdist.barrier()
            df.close()
        comm = chdist.NcclComm(device=dev)
        ws = chf.Workspace(max(hi - lo, 1), device=dev)
        out = torch.empty(max(hi - lo, 1), dtype=torch.int64, device=dev)
        hull, total, st = comm.hull_end_to_end(xy, hi - lo, n, ws, out, root=0)
        comm.close()
        q.put((rank, res, hull, total))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world", sorted({2, min(8, max(2, torch.cuda.device_count() if torch.cuda.is_available()
                                                               else 2))}))
@pytest.mark.parametrize("dist_name,n", [("displaced", 2_000_003), ("normal", 5_000_011)])
def test_one_process_per_gpu_all_exchanges(world, dist_name, n):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (this box has {torch.cuda.device_count()})")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_worker, args=(r, world, port, n, dist_name, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda r: r[0])
    for p_ in procs:
        p_.join(timeout=120)
    for r in res:
        assert len(r) == 4, r[1]
    full = synth.points(dist_name, n, seed=8, device=DEV).cpu().numpy()
    want, _ = oracle.filter_compact(full)
    for exchange in chdist.EXCHANGES:
        for k in range(3):
            parts = [r[1][exchange][k] for r in res]
            assert np.array_equal(np.concatenate([p[2] for p in parts]), want), (exchange, k)
            sizes = [len(p[2]) for p in parts]
            assert [p[0] for p in parts] == [sum(sizes[:i]) for i in range(world)], exchange
            assert all(p[1] == len(want) for p in parts), exchange
    assert np.array_equal(res[0][2], oracle.hull(full, want))
    assert all(len(r[2]) == 0 for r in res[1:]) and all(r[3] == len(want) for r in res)

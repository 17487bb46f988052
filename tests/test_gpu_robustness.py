"""GPU tests of the library's guards (VERDICT r1 "weak" 7-8):
workspace octagons reused on other points, caller-supplied octagons whose
shortcuts are wrong, the look-back epoch wrap, a late peer record, and the
float64-only hull / gather entry points.  Every result is compared with the
oracle (or with the definition the oracle implements) element by element."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import paper_2303_10581_b200 as chf
import synth
from exact import load_golden

pytestmark = pytest.mark.gpu
DEV = "cuda"

# WsHeader layout (csrc/chfilter.cu): k1_ticket, k2_claim, k2_exit, epoch, ...
EPOCH_OFF = 12
STATUS_OFF = 4096 + 2048 * 144     # WS_HEADER + K1_MAX_CTAS * sizeof(Partial)


def _want_flags(xy_np, build_np, certified=True):
    """Survivors of xy under the octagon the oracle builds from build_np."""
    wo = oracle.octagon(build_np, certified=certified)
    return np.flatnonzero(oracle.flags(xy_np, oct_=wo))


def test_workspace_octagon_reused_on_other_points():
    """ch_filter_compact(h_oct = NULL) on points the workspace octagon was NOT
    built from: the result is the definition (D_k > T_k with that octagon),
    so K2 must not use the fp32 certificates, whose bound assumes every
    point inside the octagon's bbox (data tag)."""
    rng = np.random.default_rng(5)
    a = synth.points("normal", 300_000, seed=1, device=DEV)
    an = a.cpu().numpy()
    wo = oracle.octagon(an)
    # B: half inside A's octagon region, points far outside A's bbox at large
    # scales (fp32 overflow range), and points within ulps of A's edges
    inner = (an[:100_000] - 0.5) * 0.3 + 0.5
    far = rng.normal(size=(50_000, 2)) * np.array([1e30, 1e36])
    from exact import near_edge_points
    V = list(zip(wo["vx"], wo["vy"]))
    edge = near_edge_points(rng, V, 50_000, ulps=3)
    b = np.concatenate([inner, far, edge, an[100_000:150_000] * 3.0])
    bd = torch.tensor(b, device=DEV)
    ws = chf.Workspace(max(len(b), a.shape[0]))
    for storage in ("f64", "f32"):
        aa = a if storage == "f64" else a.float()
        bb = bd if storage == "f64" else bd.float()
        bref = b if storage == "f64" else bb.double().cpu().numpy()
        aref = an if storage == "f64" else aa.double().cpu().numpy()
        chf.extremes8(aa, ws)
        cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
        out = chf.filter_compact(bb, ws, count=cnt)
        got = out[: int(cnt.item())].cpu().numpy()
        assert np.array_equal(got, _want_flags(bref, aref)), storage
        # and the same workspace octagon on its own points still matches
        out = chf.filter_compact(aa, ws, count=cnt)
        got = out[: int(cnt.item())].cpu().numpy()
        assert np.array_equal(got, _want_flags(aref, aref)), storage


def test_caller_octagon_with_invalid_box_is_not_trusted():
    """A caller octagon whose accept box does not lie inside the octagon:
    the box is dropped (sanitize_octagon), so the survivors are still the
    definition's.  Trusting it would discard every point in [-10, 10]^2."""
    xy = synth.points("displaced", 200_003, seed=3, device=DEV)
    xn = xy.cpu().numpy()
    e, o = chf.extremes8(xy)
    o.box[0], o.box[1], o.box[2], o.box[3] = -10.0, 10.0, -10.0, 10.0
    o.has_box = 1
    for k in range(8):
        o.guess_edge[k] = 77          # out of range: sanitized to 0
    want = _want_flags(xn, xn)
    ws = chf.Workspace(xy.shape[0])
    got = chf.filter_compact(xy, ws, oct_=o)
    cnt = chf.read_result(ws).count
    assert np.array_equal(got[:cnt].cpu().numpy(), want)
    bits = chf.octagon_filter(xy, ws, oct_=o).cpu().numpy().view(np.uint32)
    keep = np.unpackbits(bits.view(np.uint8), bitorder="little")[: len(xn)]
    assert np.array_equal(np.flatnonzero(keep), want)
    # a valid box is kept and gives the same survivors
    e2, o2 = chf.extremes8(xy)
    assert o2.has_box
    got = chf.filter_compact(xy, ws, oct_=o2)
    assert np.array_equal(got[: chf.read_result(ws).count].cpu().numpy(), want)


def test_epoch_wrap_clears_lookback_status_words():
    """The look-back status words carry a 22-bit launch epoch.  When it wraps
    the last CTA clears every status word of the workspace, so a word written
    2^22 launches earlier cannot pass for a current one.
    Simulated: a large step at epoch 5, a launch that wraps, epoch 5 again on
    different data -- stale words would carry epoch 5 and flag P."""
    n = 3_000_000
    a = synth.points("displaced", n, seed=11, device=DEV)
    b = synth.points("circle", n, seed=12, device=DEV)
    small = synth.points("normal", 100_000, seed=13, device=DEV)
    ws = chf.Workspace(n)
    ep = ws.buf[EPOCH_OFF:EPOCH_OFF + 4].view(torch.int32)
    ep.fill_(5)
    sa = chf.filter(a, ws).cpu().numpy()
    assert int(ep.item()) == 6
    st = ws.buf[STATUS_OFF:].view(torch.int64)
    assert int((st != 0).sum().item()) > 0
    ep.fill_((1 << 22) - 1)
    chf.filter(small, ws)
    torch.cuda.synchronize()
    assert int(ep.item()) == 0
    assert int((st != 0).sum().item()) == 0          # every status word cleared
    ep.fill_(5)
    sb = chf.filter(b, ws).cpu().numpy()
    want_b, _ = oracle.filter_compact(b.cpu().numpy())
    assert np.array_equal(sb, want_b)
    want_a, _ = oracle.filter_compact(a.cpu().numpy())
    assert np.array_equal(sa, want_a)


def test_hull_and_gather_take_float64_only():
    """the hull and gather entry points read const double*."""
    xy = synth.points("normal", 10_000, seed=2, device=DEV)
    surv = chf.filter(xy)
    for fn in (chf.hull_gpu, chf.hull_gpu_async, chf.gather_points):
        with pytest.raises(TypeError):
            fn(xy.float(), surv)
        with pytest.raises(TypeError):
            fn(xy, surv.int())
    assert len(chf.hull_gpu(xy, surv)) > 2


def test_device_hull_golden_scaled_tiny():
    """The device hull's exact orientation at magnitudes where every product
    of coordinate differences underflows (scale invariance of the golden
    hulls)."""
    for s in (2.0 ** -470, 2.0 ** -540, 2.0 ** -700):
        for ex in load_golden():
            d = torch.tensor(np.array(ex["points"]) * s, device=DEV)
            sv = torch.tensor(ex["survivors"], dtype=torch.int64, device=DEV)
            assert list(chf.hull_gpu(d, sv)) == ex["hull"], (ex["name"], s)


def _late_peer_worker(rank, world, port, n, q):
    import os
    import time
    import torch.distributed as tdist
    from paper_2303_10581_b200 import dist as chdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["CH_PEER_TIMEOUT_MS"] = "300"
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = chdist.shard_range(n, world, rank)
        xy = synth.points("displaced", n, seed=4, device="cuda", lo=lo, hi=hi)
        df = chdist.DistFilter(n, xy, exchange="peer")
        tdist.barrier()
        if rank == 1:
            time.sleep(2.0)           # rank 0's K3 gives up on this record
        df.step()
        torch.cuda.synchronize()
        tdist.barrier()
        err = None
        try:
            df.result()
        except chf.CHError as e:
            err = e.status
        df.step()                     # the next step is healthy again
        loc, off, total = df.result()
        tdist.barrier()
        df.peer.close()
        q.put((rank, err, off, total, loc.cpu().numpy()))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        tdist.destroy_process_group()


def test_late_peer_record_fails_its_step_only():
    """a record that misses K3's wait is combined as an empty shard
    (never the zero-filled slot), the step raises CH_ERR_PEER on every rank,
    and the flag is reset by the next step, which matches the oracle."""
    import socket
    import torch.multiprocessing as mp
    n, world = 500_003, 2
    s0 = socket.socket(); s0.bind(("127.0.0.1", 0)); port = s0.getsockname()[1]; s0.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_late_peer_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p_ in procs:
        p_.join(timeout=60)
    for r in res:
        assert len(r) == 5, r[1]
    assert [r[1] for r in res] == [7, 7]          # CH_ERR_PEER on both ranks
    full = synth.points("displaced", n, seed=4, device="cuda")
    want, _ = oracle.filter_compact(full.cpu().numpy())
    assert np.array_equal(np.concatenate([r[4] for r in res]), want)
    assert all(r[3] == len(want) for r in res)

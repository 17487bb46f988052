#!/usr/bin/env python
"""Benchmark of the B200 octagon pre-filter (arXiv 2303.10581 hot path).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)

A step is one pass of the whole hot path over the
resident synthetic input: K1 (extremes + octagon) then K2 (octagon test +
stable compaction), plus at N > 1 the extremes all-gather + K3 combine and
the count all-gather.  Default workload: 10^9 normal points (the north_star
target, BASELINE.json configs[4] at one GPU), float64.  Prints ONE JSON line
on rank 0.  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gpts/s filtered and % of HBM peak at 1/2/4/8 B200; survivor ratio per distribution"
L2_BYTES = 126 * 1024 * 1024   # B200 L2
UNIT = "Gpts/s"

NVML_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
                0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference", "cub", "thrust-scan", "thrust-copy"], default="ours",
                    help="ours | reference (the CPU oracle arm) | cub (the paper's Variant #4 rebuilt "
                         "with CUB on this GPU, SURVEY f4: an in-box prior-art bar, not a driver arm)")
    ap.add_argument("--dist", choices=["normal", "circle", "displaced"], default="normal")
    ap.add_argument("--points", "--n", dest="n", type=float, default=1e9,
                    help="points (total for strong scaling, per GPU for weak)")
    ap.add_argument("--p", type=float, default=0.1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong")
    ap.add_argument("--predicate", choices=["certified", "plain", "exact"], default="certified",
                    help="certified (default, DESIGN R4) | plain (T_k = 0) | exact (f3)")
    ap.add_argument("--plain", action="store_true", help="alias of --predicate plain")
    ap.add_argument("--storage", choices=["f64", "f32"], default="f64",
                    help="point storage precision (f32: the paper's, widened exactly to f64)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--timed-events", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--exchange", choices=["auto", "peer", "nccl", "torch"], default="auto",
                    help="N > 1: extremes / count exchange fused into the kernels over peer memory (peer), the "
                         "library-owned NCCL communicator (nccl: one C call per step), or torch.distributed "
                         "all-gathers (torch); auto = peer if it initializes AND its first step agrees with nccl, "
                         "else nccl")
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",  # noqa: E501
                    help="replay the step as a CUDA graph (ch_graph_launch); auto: 1 GPU and n <= 2^20")
    ap.add_argument("--hull-reps", type=int, default=3,
                    help="a8: time the hull of the step's survivors this many times after the filter's timed "
                         "region (0: off; 1 GPU, float64 storage)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="target CPU work for the oracle baseline")
    return ap.parse_args()


def env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_name(a) -> str:
    n = int(a.n)
    e = int(round(math.log10(n))) if n > 0 and 10 ** round(math.log10(n)) == n else None
    size = f"1e{e}" if e is not None else str(n)
    d = a.dist if a.dist != "displaced" else f"displaced_p{a.p:g}"
    return f"{d}_{size}_fp{'32' if getattr(a, 'storage', 'f64') == 'f32' else '64'}"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.ok = False
        self.samples, self.reasons = [], 0
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        names = [v for k, v in NVML_REASONS.items() if self.reasons & k]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": int(self.max_mhz),
                "reasons": names, "samples": len(self.samples)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy kernel)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def ncu_traffic(kernel: str, workload: str):
    """dram bytes per launch from the committed ncu capture, if it matches."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d[workload][kernel]
        return float(e["dram_read_bytes"]) + float(e["dram_write_bytes"])
    except Exception:
        return None


def cpu_model() -> str | None:
    """The host CPU model (lscpu "Model name", else /proc/cpuinfo)."""
    try:
        import subprocess
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.strip().startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def oracle_rate(xy_host: np.ndarray, seconds: float):
    """Time the CPU oracle (single thread) on a bounded prefix of the input."""
    import oracle
    oracle.build()
    n = xy_host.shape[0]
    m0 = min(n, 1 << 20)
    t0 = time.perf_counter()
    oracle.filter_compact(xy_host[:m0])
    dt0 = time.perf_counter() - t0
    m = int(min(n, max(m0, m0 * seconds / max(dt0, 1e-9))))
    t0 = time.perf_counter()
    surv, _ = oracle.filter_compact(xy_host[:m])
    dt = time.perf_counter() - t0
    return m, dt, len(surv)


# --------------------------------------------------------------------------- #
def run_reference(a):
    """The reference arm: the CPU oracle, as it stands, on the host cores."""
    rank, world, local = env()
    if rank != 0:
        return 0
    import oracle
    import synth
    oracle.build()
    n = int(a.n)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    # a bounded prefix of the same workload (same generator, same device)
    m0 = min(n, 1 << 20)
    probe = synth.points(a.dist, n, seed=a.seed, p=a.p, device=dev, lo=0, hi=m0).cpu().numpy()
    t0 = time.perf_counter()
    ofc = (lambda v: oracle.filter_compact_exact(v)) if a.predicate == "exact" else \
        (lambda v: oracle.filter_compact(v, certified=a.predicate != "plain"))
    ofc(probe)
    dt0 = time.perf_counter() - t0
    per_step_s = 120.0 / max(a.steps + a.warmup, 1)
    m = int(min(n, max(m0, m0 * min(per_step_s, 2.0) / max(dt0, 1e-9))))
    xy = synth.points(a.dist, n, seed=a.seed, p=a.p, device=dev, lo=0, hi=m).cpu().numpy()
    if a.storage == "f32":
        xy = xy.astype(np.float32).astype(np.float64)   # the widened f32 workload
    for _ in range(a.warmup):
        ofc(xy)
    times = []
    s = 0
    for _ in range(a.steps):
        t0 = time.perf_counter()
        surv, _ = ofc(xy)
        times.append(time.perf_counter() - t0)
        s = len(surv)
    ms = 1e3 * float(np.mean(times))
    val = m / (ms / 1e3) / 1e9
    sample = f"first {m} of {n} points of {workload_name(a)} (same generator), per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": a.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(a), "n": n, "dist": a.dist, "seed": a.seed,
                   "sample_points": m, "survivors_in_sample": s},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model(), "nproc": os.cpu_count()},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- #
def run_ours(a):
    import torch.distributed as dist
    import paper_2303_10581_b200 as chf
    from paper_2303_10581_b200 import dist as chdist
    import synth

    rank, world, local = env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU path)")
    # the sharded path: N > 1, or an explicit --exchange (also at N = 1, to
    # run the distributed step's code on one GPU)
    multi = world > 1 or a.exchange != "auto"
    # stdout carries exactly one JSON line: NCCL's own messages (e.g. its
    # version banner when the environment sets NCCL_DEBUG=VERSION) go to stderr
    if "CH_KEEP_NCCL_DEBUG" not in os.environ:
        os.environ["NCCL_DEBUG"] = "WARN"
        os.environ["NCCL_DEBUG_FILE"] = "/dev/stderr"
    # CH_BENCH_SHARE_GPU=1: every rank on cuda:0 with gloo collectives -- only
    # to exercise the N > 1 code path on a 1-GPU box; never a measurement.
    share = os.environ.get("CH_BENCH_SHARE_GPU") == "1"
    gpu = 0 if share else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if multi:
        if world == 1:   # a one-rank group without torchrun
            import socket
            s0 = socket.socket()
            s0.bind(("127.0.0.1", 0))
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(s0.getsockname()[1]))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
            s0.close()
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def reduce_host(v, op):
        """All-reduce a python scalar over ranks (device tensor for NCCL)."""
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64 if isinstance(v, float) else torch.int64,
                         device="cpu" if share else dev)
        dist.all_reduce(t, op=op)
        return t.item()
    n_arg = int(a.n)
    n_total = n_arg if a.scaling == "strong" else n_arg * world
    lo, hi = chdist.shard_range(n_total, world, rank)
    n_local = hi - lo
    xy = synth.points(a.dist, n_total, seed=a.seed, p=a.p, device=dev, lo=lo, hi=hi)
    if a.storage == "f32":
        xy = xy.float()
    torch.cuda.synchronize()
    bpp = 8.0 if a.storage == "f32" else 16.0   # bytes per point per pass
    stream = torch.cuda.current_stream()

    small = not multi and n_local <= 4096   # latency-bound C1: the single-kernel step (K5)
    peer, exchange = False, None
    # launch-bound sizes: the whole step replayed as one CUDA graph
    graphed = not multi and (a.graph == "on" or (a.graph == "auto" and n_local <= (1 << 20)))
    if not multi:
        ws = chf.Workspace(n_local, device=dev)
        out = torch.empty(max(n_local, 1), dtype=torch.int64, device=dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        launches_per_step = 1 if small else 2
        graph = chf.FilterGraph(xy, ws, out, cnt, plain=a.plain) if graphed else None

        def k1():
            if graphed:
                graph.launch()
            elif small:
                chf.filter_async(xy, ws, out, cnt, plain=a.plain)
            else:
                chf.extremes8_async(xy, ws, plain=a.plain)

        def exch():
            pass

        def k2():
            if not small and not graphed:
                chf.filter_compact(xy, ws, out=out, count=cnt)

        def exch2():
            pass

        def one_call():
            """The product's one-call step (ch_filter_async: K1 then K2 with
            programmatic dependent launch; K5/K6 for small n; or the graph)."""
            if graphed:
                graph.launch()
            else:
                chf.filter_async(xy, ws, out, cnt, plain=a.plain)
    else:
        exchange = a.exchange if a.exchange != "auto" else "nccl"
        if share and exchange == "nccl":
            exchange = "torch"   # NCCL refuses two ranks on one device: gloo all-gathers instead
        df = chdist.DistFilter(n_total, xy, plain=a.plain, exchange=exchange)
        if a.exchange == "auto" and not share:
            # the peer transport (no collective launches) if it initializes on
            # every rank AND its first step gives the same placement as NCCL's
            df.step()
            ref = df.result()
            ok = 1
            try:
                os.environ.setdefault("CH_PEER_TIMEOUT_MS", "10000")
                dp = chdist.DistFilter(n_total, xy, plain=a.plain, exchange="peer")
                dp.step()
                got = dp.result()
                ok = int(got[1:] == ref[1:] and torch.equal(got[0], ref[0]))
            except Exception as e:
                print(f"[bench] rank {rank}: peer exchange unavailable ({e})", file=sys.stderr)
                dp, ok = None, 0
            if int(reduce_host(int(ok), dist.ReduceOp.MIN)) == 1:
                df.close()
                df, exchange = dp, "peer"
            elif dp is not None:
                dp.close()
        ws = df.ws
        peer = exchange == "peer"
        # our kernels per step: K1, K3, K2 (+ the status pack and scan kernels of the NCCL step)
        launches_per_step = 5 if exchange == "nccl" else 3

        def k1():
            if exchange != "torch":
                df.step()   # one C call: the whole step (see DistFilter)
                return
            chf.extremes8_async(xy, df.ws, index_base=df.lo, plain=a.plain, ext_out=df.ext_local)

        def exch():
            if exchange == "torch":
                chdist.exchange_extremes(df.ext_local, out=df.ext_all)
                chf.combine8(df.ext_all, world, df.ws, plain=a.plain)

        def k2():
            if exchange == "torch":
                chf.filter_compact(xy, df.ws, index_base=df.lo, out=df.out, count=df.count)

        def exch2():
            if exchange == "torch":
                chdist.exclusive_offsets(df.count, out=df.counts)

        def one_call():
            k1(); exch(); k2(); exch2()

    def step():
        one_call()

    for _ in range(max(a.warmup, 0)):
        step()
    torch.cuda.synchronize()
    res = chf.read_result(ws)   # raises on non-finite input

    K = a.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if not (bpp * n_local < 2 * L2_BYTES) and not graphed:
        # the per-kernel split (for the roofline) from a pass with events
        # between the kernels, before the timed region; `value` comes from
        # the timed region, which has no events between the kernels (K2's
        # programmatic launch overlaps K1's tail only when they are adjacent)
        for k in range(K):
            ev[k][0].record(stream)
            k1()
            ev[k][1].record(stream)
            exch()
            ev[k][2].record(stream)
            k2()
            ev[k][3].record(stream)
            exch2()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    # inputs smaller than 2x the 126 MB L2: flush L2 before every timed step
    # (a 512 MB memset, outside the step's own events) and time steps alone
    flush = bpp * n_local < 2 * L2_BYTES
    fbuf = torch.empty(4 * L2_BYTES, dtype=torch.uint8, device=dev) if flush else None
    step_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)] if flush else None
    with ClockSampler(local) as clk:
        t_start.record(stream)
        if flush:
            for k in range(K):
                fbuf.zero_()
                step_ev[k][0].record(stream)
                if graphed:
                    k1()
                else:
                    ev[k][0].record(stream)
                    k1()
                    ev[k][1].record(stream)
                    exch()
                    ev[k][2].record(stream)
                    k2()
                    ev[k][3].record(stream)
                    exch2()
                step_ev[k][1].record(stream)
        elif a.timed_events:   # developer A/B: events between the kernels in the timed region
            for k in range(K):
                ev[k][0].record(stream)
                k1()
                ev[k][1].record(stream)
                exch()
                ev[k][2].record(stream)
                k2()
                ev[k][3].record(stream)
                exch2()
        else:   # the one-call step, no events between the kernels (see the split pass above)
            for k in range(K):
                one_call()
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = t_start.elapsed_time(t_end)
    if flush:   # the steps' own time: L2 flushes excluded
        total_ms = float(np.sum([e[0].elapsed_time(e[1]) for e in step_ev]))
    if graphed:
        k1_ms, k2_ms, ex_ms = total_ms / K, 0.0, 0.0
    else:
        k1_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
        k2_ms = float(np.mean([e[2].elapsed_time(e[3]) for e in ev]))
        ex_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
    if multi and exchange == "nccl":
        # the library's own events around the phases of the last timed step
        k1_ms, ex_ms, k2_ms = df.comm.step_times()
    res = chf.read_result(ws)
    s_local = int(res.count)
    if world > 1:
        total_ms = float(reduce_host(float(total_ms), dist.ReduceOp.MAX))
        s_total = int(reduce_host(int(s_local), dist.ReduceOp.SUM))
    else:
        s_total = s_local
    ms_step = total_ms / K
    value = n_total / (ms_step / 1e3) / 1e9

    # ---- roofline of the dominant kernel (algorithmic bytes) ----
    peak, peak_src = measured_peaks()
    k1_bytes = bpp * n_local
    k2_bytes = bpp * n_local + 8.0 * s_local
    if graphed:
        dom = ("graph(k5_small_filter)" if small else "graph(k6_cluster_filter)" if n_local <= 32768
               else "graph(k1_extremes8+k2_filter_compact)")
        dom_bytes, dom_ms = k1_bytes + k2_bytes, k1_ms
    elif peer:   # one call enqueues K1, K3 and K2: the whole step is timed
        dom, dom_bytes, dom_ms = "step(k1_extremes8+k3_combine8_peer+k2_filter_compact)", k1_bytes + k2_bytes, k1_ms
    elif small:
        dom, dom_bytes, dom_ms = "k5_small_filter", k1_bytes + k2_bytes, k1_ms
    elif k2_ms >= k1_ms:
        dom, dom_bytes, dom_ms = "k2_filter_compact", k2_bytes, k2_ms
    else:
        dom, dom_bytes, dom_ms = "k1_extremes8", k1_bytes, k1_ms
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    step_bytes = k1_bytes + k2_bytes
    traffic = ncu_traffic(dom, workload_name(a))
    roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
            "traffic_source": ("dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed "
                               "ncu --set full capture of this kernel and workload (profiles/ncu_traffic.json), "
                               "not measured in this run") if traffic is not None else None,
            "kernel_ms_source": ("a pass of the same K steps with CUDA events between the kernels (separate "
                                 "calls, no programmatic launch), run just before the timed region; value and "
                                 "ms_per_step time the one-call step") if not (graphed or peer or small) else
                                "the timed region (one launch or one graph per step)",
            "k1_ms": k1_ms, "k2_ms": k2_ms, "k1_gbs": k1_bytes / (k1_ms / 1e3) / 1e9 if not (graphed or peer) else None,
            "k2_gbs": k2_bytes / (k2_ms / 1e3) / 1e9 if k2_ms > 0 else None,
            "step_gbs_per_gpu": step_bytes / (ms_step / 1e3) / 1e9,
            "step_frac": step_bytes / (ms_step / 1e3) / 1e9 / peak,
            "step_frac_theoretical_8184": step_bytes / (ms_step / 1e3) / 1e9 / 8184.0}

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not a.no_e2e and a.e2e_steps > 0 and a.storage == "f64":
        h_xy = torch.empty(n_local, 2, dtype=torch.float64, pin_memory=True)
        h_xy.copy_(xy)
        h_out = torch.empty(max(n_local, 1), dtype=torch.int64)
        d_stage = torch.empty_like(xy)
        e_s = torch.cuda.Event(enable_timing=True)
        e_e = torch.cuda.Event(enable_timing=True)
        # one untimed warm-up
        if not multi:
            d2h = 0
            chf.filter_host(h_xy, ws, d_stage, out, h_out, plain=a.plain)
            torch.cuda.synchronize()
            e_s.record(stream)
            for _ in range(a.e2e_steps):
                c = chf.filter_host(h_xy, ws, d_stage, out, h_out, plain=a.plain)
                d2h = 8 * c + 8
            e_e.record(stream)
            torch.cuda.synchronize()
            e2e_ms = e_s.elapsed_time(e_e) / a.e2e_steps
        else:
            df2 = chdist.DistFilter(n_total, d_stage, plain=a.plain, exchange=exchange)
            d2h = 0

            def e2e_step():
                d_stage.copy_(h_xy, non_blocking=True)
                df2.step(d_stage)
                loc, off, tot = df2.result()
                h_out[: loc.shape[0]].copy_(loc)
                return 8 * loc.shape[0] + 8 * world

            e2e_step()
            torch.cuda.synchronize()
            dist.barrier()
            e_s.record(stream)
            for _ in range(a.e2e_steps):
                d2h = e2e_step()
            e_e.record(stream)
            torch.cuda.synchronize()
            e2e_ms = float(reduce_host(float(e_s.elapsed_time(e_e) / a.e2e_steps), dist.ReduceOp.MAX))
        e2e = {"value": n_total / (e2e_ms / 1e3) / 1e9, "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": 16 * n_local, "d2h_bytes_per_step": int(d2h),
               "api": "ch_filter_host (C ABI, pinned host input)" if not multi else "DistFilter + host copies"}
        del h_xy, h_out, d_stage

    # ---- a8: the hull of the survivors, timed separately (north_star), after
    # the filter's timed region; CUDA events around each call ----
    hull = None
    if not multi and a.hull_reps > 0 and a.storage == "f64":
        lib = chf._lib.load()
        tb = int(lib.ch_hull_gpu_temp_bytes(max(s_local, 1)))
        if 2 * tb + 16 * s_local < 0.9 * torch.cuda.mem_get_info()[0]:   # ch_hull_gpu allocates its own
            surv = out[:s_local].clone()
            tmp = torch.empty(max(tb, 1), dtype=torch.uint8, device=dev)
            h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t_sync, t_async, nh = [], [], 0
            for r in range(a.hull_reps + 1):            # the first call is an untimed warm-up
                torch.cuda.synchronize()
                h0.record(stream)
                ids = chf.hull_gpu(xy, surv)            # ch_hull_gpu: synchronizes, ids to host
                h1.record(stream)
                torch.cuda.synchronize()
                if r:
                    t_sync.append(h0.elapsed_time(h1))
                h0.record(stream)
                hd, hc = chf.hull_gpu_async(xy, surv, tmp)
                h1.record(stream)
                torch.cuda.synchronize()
                if r:
                    t_async.append(h0.elapsed_time(h1))
                nh = len(ids)
                assert int(hc.item()) == nh
            hull = {"ms": float(np.median(t_sync)), "ms_on_device": float(np.median(t_async)), "n_hull": nh,
                    "survivors": s_local, "reps": a.hull_reps,
                    "api": "ms: ch_hull_gpu (second filtering round, radix sort by x, exact monotone chains; "
                           "hull ids copied to the host); ms_on_device: ch_hull_gpu_async (ids stay on the "
                           "device, no second round); median over reps, CUDA events; not part of value"}
            del tmp, surv, hd, hc

    # ---- CPU oracle baseline (rank 0, N = 1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        m_cap = n_local
        host = xy[:m_cap].double().cpu().numpy()
        m, dt, s = oracle_rate(host, a.cpu_seconds)
        cpu = {"value": m / dt / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
               "cpu_model": cpu_model(), "nproc": os.cpu_count(),
               "sample": f"first {m} points of the same {workload_name(a)} input (oracle: extremes + octagon + "
                         f"filter + compaction, single thread, {dt:.2f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": a.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": a.scaling if world > 1 else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(a), "n": n_total, "n_per_gpu": n_local, "dist": a.dist,
                       "seed": a.seed, "p": a.p if a.dist == "displaced" else None,
                       "predicate": a.predicate, "storage": a.storage,
                       "parallelism": f"dp{world}",
                       "l2": (f"L2 flushed before every step (512 MB memset outside the step events); "
                              f"inputs {bpp * n_local / 1e6:.3g} MB" if flush
                              else f"inputs larger than L2 ({int(bpp)} B/pt)"),
                       "cuda_graph": bool(graphed),
                       "exchange": exchange if multi else None},
            "survivors": s_total, "survivor_ratio": s_total / n_total,
            "hbm_frac": roof["step_frac"],
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "hull": hull,
            "gpu_launches": launches_per_step * K, "clocks": clk.summary(),
            "exchange_ms": ex_ms if multi else 0.0,
            "transport": ({"exchange": exchange, "ranks": world,
                           "collectives": {"nccl": "library-owned ncclComm (ch_comm_*): ncclAllGather x2 per step",
                                           "peer": "none (cudaIpc peer stores fused into K1/K2, acquired by K3)",
                                           "torch": "torch.distributed all_gather_into_tensor x2 per step"}[exchange],
                           "nccl_version": chf._lib.load().ch_comm_nccl_version(),
                           "backend": "gloo (shared GPU, functional check only)" if share else "nccl"}
                          if multi else None),
            "ctas_per_sm": {"k1": chf._lib.load().ch_occupancy(0),
                            "k2": chf._lib.load().ch_occupancy(2 if a.storage == "f32" else 1)},
        }
        print(json.dumps(line), flush=True)
    if multi:
        dist.destroy_process_group()
    return 0


def run_cub(a):
    """the paper's library variants on the same GPU, same
    input: #4 CUB (8 ArgMin/ArgMax reductions, a flag kernel,
    DeviceSelect::Flagged), #2 Thrust scan + scatter, #3 Thrust copy_if."""
    import ctypes
    import paper_2303_10581_b200 as chf
    import synth
    sys.path.insert(0, os.path.join(ROOT, "baselines"))
    import build as bbuild  # baselines/build.py
    lib = ctypes.CDLL(bbuild.build())
    P, SZ, I64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int64
    for f in ("chb_cub_temp_bytes", "chb_thrust_temp_bytes"):
        getattr(lib, f).restype = SZ
        getattr(lib, f).argtypes = [I64]
    lib.chb_cub_filter.restype = ctypes.c_int
    lib.chb_cub_filter.argtypes = [P, I64, P, ctypes.POINTER(I64), P, SZ, P]
    lib.chb_thrust_filter.restype = ctypes.c_int
    lib.chb_thrust_filter.argtypes = [ctypes.c_int, P, I64, P, ctypes.POINTER(I64), P, SZ, P]
    dev = torch.device("cuda", 0)
    n = int(a.n)
    xy = synth.points(a.dist, n, seed=a.seed, p=a.p, device=dev)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    variant = {"cub": 4, "thrust-scan": 2, "thrust-copy": 3}[a.impl]
    tb = int(lib.chb_cub_temp_bytes(n) if variant == 4 else lib.chb_thrust_temp_bytes(n))
    tmp = torch.empty(tb, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    cnt = ctypes.c_int64(0)

    def step():
        args = (P(xy.data_ptr()), n, P(out.data_ptr()), ctypes.byref(cnt), P(tmp.data_ptr()), tb,
                P(stream.cuda_stream))
        rc = lib.chb_cub_filter(*args) if variant == 4 else lib.chb_thrust_filter(variant, *args)
        assert rc == 0, rc

    for _ in range(a.warmup):
        step()
    mine = chf.filter(xy)                       # same survivors as the product path
    assert cnt.value == mine.shape[0] and torch.equal(out[: cnt.value], mine)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    desc = {4: "paper Variant #4 cub-flagged (P:237-242), rebuilt with CUB",
            2: "paper Variant #2 thrust-scan (P:219-222): min/max_element, transform, exclusive_scan, scatter",
            3: "paper Variant #3 thrust-copy (P:224-225): min/max_element, copy_if"}[variant]
    print(json.dumps({"impl": a.impl, "metric": METRIC, "value": n / (ms / 1e3) / 1e9, "unit": UNIT, "n_gpus": 1,
                      "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
                      "dtype": "f64", "data": "synthetic",
                      "config": {"workload": workload_name(a), "n": n, "survivors": int(cnt.value),
                                 "variant": desc}}),
          flush=True)
    return 0


def main():
    a = parse()
    if a.plain:
        a.predicate = "plain"
    # the binding's predicate argument: False (certified), True (plain), "exact"
    a.plain = {"certified": False, "plain": True, "exact": "exact"}[a.predicate]
    if a.impl == "reference":
        return run_reference(a)
    if a.impl in ("cub", "thrust-scan", "thrust-copy"):
        return run_cub(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())

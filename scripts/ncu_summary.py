#!/usr/bin/env python
"""Summarise an ncu report (raw page) into the numbers we track.

    python scripts/ncu_summary.py gpurun_out/prof_x.ncu-rep [--json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "lts__t_bytes.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        res.append((d, u))
    return res


def summarise(d, u):
    s = {"kernel": d.get("Kernel Name", "")[:90]}
    for k in KEYS:
        if k in d:
            s[k] = f"{d[k]} {u.get(k, '')}".strip()
    stalls = []
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    s["top_stalls_per_issue"] = [f"{n}={v:.2f}" for v, n in stalls[:6]]
    return s


def main():
    path = sys.argv[1]
    for d, u in load(path):
        s = summarise(d, u)
        if "--json" in sys.argv:
            print(json.dumps(s))
        else:
            for k, v in s.items():
                print(f"{k:60s} {v}")
            print()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Top stalled SASS instructions of an ncu report (needs -lineinfo builds).
    python scripts/ncu_hot.py report.ncu-rep [N]"""
import csv, io, subprocess, sys
path = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; data = rows[2:]; ix = {k: i for i, k in enumerate(h)}
S = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[ix[S]] or 0) for r in data)
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
order = sorted(range(len(data)), key=lambda i: -float(data[i][ix[S]] or 0))[:N]
for i in order:
    r = data[i]
    s = float(r[ix[S]] or 0)
    rs = sorted(((float(r[ix[k]] or 0), k[6:]) for k in reasons), reverse=True)[:3]
    prev = " | ".join(x[1].strip()[:28] for x in data[max(0, i - 2):i])
    print(f"{r[0][-5:]} {100*s/tot:5.1f}%  {r[1].strip()[:58]:58s} {[f'{n}:{int(v)}' for v, n in rs]}  prev: {prev}")

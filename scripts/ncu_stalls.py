#!/usr/bin/env python
"""Warp-stall samples per CUDA source line, with the top reasons:
python scripts/ncu_stalls.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
path, hdr, res = "", None, []
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0] not in ("", "Line No"):
        d = dict(zip(hdr, r))
        try:
            samp = float(d["Warp Stall Sampling (All Samples)"])
        except ValueError:
            continue
        reasons = sorted(((float(d[k]), k[6:]) for k in hdr if k.startswith("stall_") and "Not Issued" not in k
                          and d[k] not in ("", "-")), reverse=True)[:3]
        res.append((samp, path, r[0], r[1].strip()[:80], reasons))
tot = sum(x[0] for x in res) or 1
res.sort(key=lambda x: -x[0])
agg = {}
for s, *_, rs in res:
    pass
print(f"total samples {tot:.0f}")
for s, f, l, src, rs in res[:top]:
    print(f"{100 * s / tot:5.1f}%  {f}:{l:5s} {src:80s} " + " ".join(f"{n}={100 * v / tot:.1f}" for v, n in rs if v))

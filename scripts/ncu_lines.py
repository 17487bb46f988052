#!/usr/bin/env python
"""Instructions executed per CUDA source line (needs -lineinfo and
--import-source): python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
path, res = "", []
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif len(r) > 8 and r[0] not in ("", "Line No"):
        try:
            res.append((float(r[7]), path, r[0], r[1].strip()[:100], r[4]))
        except ValueError:
            pass
tot = sum(x[0] for x in res) or 1
res.sort(reverse=True)
print(f"total warp-instructions {tot:.4g}")
for v, f, l, s, st in res[:top]:
    print(f"{100 * v / tot:5.1f}%  stall={st:>6s}  {f}:{l}  {s}")

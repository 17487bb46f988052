#!/usr/bin/env python
"""Instruction-execution histogram of an ncu report by SASS opcode, and the
hottest address ranges.  python scripts/ncu_inst.py report.ncu-rep"""
import collections, csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; data = rows[2:]; ix = {k: i for i, k in enumerate(h)}
E = "Instructions Executed"
tot = sum(float(r[ix[E]] or 0) for r in data)
ops = collections.Counter()
for r in data:
    op = r[1].strip().split()
    if not op: continue
    o = op[0] if not op[0].startswith("@") else op[1]
    ops[o.split(".")[0]] += float(r[ix[E]] or 0)
print(f"total warp-instructions {tot:.4g}")
for o, c in ops.most_common(25):
    print(f"  {o:12s} {c:12.4g}  {100*c/tot:5.1f}%")
# contiguous hot regions (64-instruction windows)
win = 48
best = []
for i in range(0, len(data), win // 2):
    s = sum(float(r[ix[E]] or 0) for r in data[i:i + win])
    best.append((s, i))
best.sort(reverse=True)
print("hot windows (start addr, % of instructions):")
for s, i in best[:8]:
    print(f"  {data[i][0][-5:]}..{data[min(i+win, len(data)-1)][0][-5:]}  {100*s/tot:5.1f}%   first: {data[i][1].strip()[:50]}")

#!/usr/bin/env python
"""Executed warp-instructions by SASS opcode (SASS view: each instruction
counted once), as thread-instructions per point (x 32 / NPOINTS).
python scripts/ncu_opmix.py report.ncu-rep NPOINTS [top]"""
import collections, csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
npts = float(sys.argv[2]); top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; ix = {k: i for i, k in enumerate(hdr)}
agg = collections.Counter()
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    n = float(r[ix["Instructions Executed"]] or 0)
    s = r[ix["Source"]].split()
    if not s:
        continue
    op = (s[1] if s[0].startswith("@") else s[0]).split(".")[0]
    agg[op] += n
tot = sum(agg.values())
print(f"total {tot * 32 / npts:.1f} thread-instr/pt ({tot:.4g} warp-instr)")
for k, v in agg.most_common(top):
    print(f"  {k:10s} {v * 32 / npts:6.2f}")

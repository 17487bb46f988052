#!/usr/bin/env python
"""Per-source-line warp instructions and stall samples of ONE kernel in an ncu
report: python scripts/ncu_kernel_lines.py report.ncu-rep <kernel-regex> [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      "regex:" + kern, "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
ii, isamp = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
inst, st, src, cur = collections.Counter(), collections.Counter(), {}, None
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    if r[0]:
        cur = r[0]
        src[cur] = r[1]
        continue  # the CUDA line's own row repeats its SASS rows' sum
    try:
        inst[cur] += float(r[ii] or 0)
        st[cur] += float(r[isamp] or 0)
    except ValueError:
        pass
ti, ts = sum(inst.values()), sum(st.values())
print(f"warp instructions {ti:.4g}")
for l, v in inst.most_common(top):
    print(f"{100 * v / ti:5.1f}% inst {100 * st[l] / ts:5.1f}% stall  L{l}: {src[l].strip()[:90]}")

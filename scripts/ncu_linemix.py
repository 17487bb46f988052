#!/usr/bin/env python
"""Per CUDA source line: executed thread-instructions per point and the SASS
opcode mix.  python scripts/ncu_linemix.py report.ncu-rep NPOINTS [top]"""
import collections, csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
npts = float(sys.argv[2]); top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
hdr, cur, path = None, None, ""
lines = collections.OrderedDict()
seen = set()  # an inlined SASS instruction is listed under several source lines: count it once
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0]:
        cur = (path, r[0], r[1].strip()[:70]); lines.setdefault(cur, collections.Counter())
    elif cur and r[2].startswith("0x"):
        if r[2] in seen:
            continue
        seen.add(r[2])
        try: n = float(r[hdr.index("Thread Instructions Executed")])
        except ValueError: continue
        s = r[3].split()
        op = s[1] if s and s[0].startswith("@") else (s[0] if s else "?")
        lines[cur][op.split(".")[0]] += n
tot = sum(sum(c.values()) for c in lines.values())
print(f"total {tot / npts:.1f} thread-instr/pt")
for (f, l, src), c in sorted(lines.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
    s = sum(c.values())
    mix = " ".join(f"{k}:{v / npts:.2f}" for k, v in c.most_common(6))
    print(f"{s / npts:6.2f}  {f}:{l:5s} {src:70s} | {mix}")

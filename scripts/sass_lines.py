#!/usr/bin/env python
"""Static SASS size per source line (innermost, from nvdisasm -gi) of one
kernel: python scripts/sass_lines.py lib.so kernel_substring [top]"""
import collections, glob, os, re, subprocess, sys, tempfile
lib, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
for cub in glob.glob(os.path.join(d, "*.cubin")):
    txt = subprocess.run(["nvdisasm", "-gi", cub], capture_output=True, text=True).stdout
    for sec in re.split(r"\n(?=\.text\.)", txt):
        name = sec.split(":", 1)[0]
        if not name.startswith(".text.") or pat not in name:
            continue
        cnt, cur, fresh = collections.Counter(), None, True
        for l in sec.split("\n"):
            m = re.search(r'//## File "([^"]+)", line (\d+)', l)
            if m:
                if fresh:  # the first marker of a block is the innermost
                    cur = (os.path.basename(m.group(1)), int(m.group(2)))
                fresh = False
            elif re.search(r"/\*[0-9a-f]{4,}\*/", l):
                cnt[cur] += 1
                fresh = True
        tot = sum(cnt.values())
        print(f"{name[6:90]}  {tot} instructions")
        for k, v in cnt.most_common(top):
            print(f"  {v:6d} {100 * v / tot:5.1f}%  {k[0]}:{k[1]}" if k else f"  {v:6d}  ?")

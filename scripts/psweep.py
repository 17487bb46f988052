#!/usr/bin/env python
"""survivor ratio vs the displacement parameter p (the
paper's Table 1) on the GPU path, with the oracle re-counting
the 1e7 column.  Table 1 is context only (DESIGN R11: the reading
rho ~ U[r(1-p), r(1+p)] does not reproduce its p >= 0.08 rows).

    python scripts/psweep.py [--sizes 1e7 1e9] [--out profiles/r01_psweep.txt]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2303_10581_b200 as chf  # noqa: E402
import synth  # noqa: E402

PAPER = {  # Table 1: discarded % at n = 1e7 and 1e9
    0.00: (0.01, 0.01), 0.02: (13.08, 13.04), 0.04: (28.58, 28.69),
    0.06: (48.48, 48.51), 0.08: (81.88, 81.71), 0.10: (97.16, 97.17),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", nargs="+", type=float, default=[1e7, 1e9])
    ap.add_argument("--ps", nargs="+", type=float, default=[0.0, 0.02, 0.04, 0.06, 0.08, 0.10, 0.25, 1.0])
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_psweep.txt"))
    a = ap.parse_args()
    rows = []
    for p in a.ps:
        row = {"p": p}
        for nf in a.sizes:
            n = int(nf)
            xy = synth.points("displaced", n, seed=0, p=p, device="cuda")
            ws = chf.Workspace(n)
            s = int(chf.filter(xy, ws).shape[0])
            row[f"discarded_pct_{n:.0e}"] = 100.0 * (1 - s / n)
            if n <= 10 ** 7:
                want, _ = oracle.filter_compact(xy.cpu().numpy())
                row[f"oracle_agrees_{n:.0e}"] = bool(len(want) == s)
            del xy, ws
            torch.cuda.empty_cache()
        if round(p, 2) in PAPER:
            row["paper_discarded_pct_1e7"], row["paper_discarded_pct_1e9"] = PAPER[round(p, 2)]
        rows.append(row)
        print(json.dumps(row), flush=True)
    lines = ["# survivor sweep, displaced circumference r = 0.25, seed 0 (DESIGN R11); GPU path, oracle-checked at 1e7",
             "# paper = Table 1 of arXiv 2303.10581 (A100, FP32, its own generator): context only, parity unpinned",
             f"{'p':>5s} " + " ".join(f"{'ours %.0e' % s:>12s}" for s in a.sizes) + f" {'paper 1e7':>10s} {'paper 1e9':>10s}  oracle"]
    for r in rows:
        ours = " ".join(f"{r[f'discarded_pct_{int(s):.0e}']:12.4f}" for s in a.sizes)
        p7 = r.get("paper_discarded_pct_1e7", float("nan"))
        p9 = r.get("paper_discarded_pct_1e9", float("nan"))
        ok = all(v for k, v in r.items() if k.startswith("oracle_agrees"))
        lines.append(f"{r['p']:5.2f} {ours} {p7:10.2f} {p9:10.2f}  {'agree' if ok else 'DISAGREE'}")
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()

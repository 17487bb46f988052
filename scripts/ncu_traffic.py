#!/usr/bin/env python
"""Per-kernel launch list summary (ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv) -> profiles/ncu_traffic.json
entry for one workload.  python scripts/ncu_traffic.py launches.csv WORKLOAD"""
import collections, csv, json, os, re, sys

path, workload = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
hdr = rows[0]; ix = {k: i for i, k in enumerate(hdr)}
per = collections.defaultdict(lambda: collections.defaultdict(float))
ids = collections.defaultdict(set)
for r in rows[1:]:
    name = re.search(r"(k\d_\w+|k_gather)", r[ix["Kernel Name"]]).group(1)
    m = r[ix["Metric Name"]]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    if m == "gpu__time_duration.sum":
        v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
    elif unit in ("Kbyte", "Mbyte", "Gbyte"):
        v *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    per[name][m] += v
    ids[name].add(r[ix["ID"]])
tot = sum(d["gpu__time_duration.sum"] for d in per.values())
out = {}
for k, d in per.items():
    n = len(ids[k])
    out[k] = {"dram_read_bytes": d["dram__bytes_read.sum"] / n, "dram_write_bytes": d["dram__bytes_write.sum"] / n,
              "duration_ns": d["gpu__time_duration.sum"] / n, "launches": n,
              "share_of_step": d["gpu__time_duration.sum"] / tot}
pf = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
j = json.load(open(pf)) if os.path.exists(pf) else {}
j[workload] = out
j["_source"] = ("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
                "(cold-cache, serialised launches); per-launch averages")
json.dump(j, open(pf, "w"), indent=1)
print(json.dumps(out, indent=1))

#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics ... --csv) and an ncu --set full
report into a small JSON committed under profiles/.

    python tools/ncu_summary.py TAG [--alg-json bench.json]
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")


def launches(tag: str) -> list:
    path = os.path.join(OUT, f"launches_{tag}.csv")
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = {h: i for i, h in enumerate(rows[start])}
    agg = OrderedDict()
    for r in rows[start + 1:]:
        key = (int(r[hdr["ID"]]), r[hdr["Kernel Name"]])
        agg.setdefault(key, {})[r[hdr["Metric Name"]]] = float(r[hdr["Metric Value"]].replace(",", ""))
    out = []
    for (i, k), m in agg.items():
        out.append({"id": i, "kernel": k.split("(")[0].replace("void ", "").replace("<unnamed>::", ""),
                    "ms": m.get("gpu__time_duration.sum", 0) / 1e6,
                    "dram_read_GB": m.get("dram__bytes_read.sum", 0) / 1e9,
                    "dram_write_GB": m.get("dram__bytes_write.sum", 0) / 1e9})
    return out


def details(tag: str) -> list:
    path = os.path.join(OUT, f"prof_{tag}.ncu-rep")
    if not os.path.exists(path):
        return []
    txt = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    want = {"Duration", "DRAM Throughput", "Memory Throughput", "Achieved Occupancy",
            "Registers Per Thread", "Theoretical Occupancy", "Grid Size", "L2 Hit Rate",
            "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler"}
    per = OrderedDict()
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in want:
            k = per.setdefault(d["ID"], {"kernel": d["Kernel Name"].split("(")[0]})
            k[f"{d['Metric Name']} [{d.get('Metric Unit', '')}]"] = d["Metric Value"]
    return list(per.values())


def main():
    tag = sys.argv[1]
    ls = launches(tag) if os.path.exists(os.path.join(OUT, f"launches_{tag}.csv")) else []
    tot = sum(x["ms"] for x in ls)
    by = OrderedDict()
    for x in ls:
        b = by.setdefault(x["kernel"], {"launches": 0, "ms": 0.0, "dram_GB": 0.0})
        b["launches"] += 1
        b["ms"] += x["ms"]
        b["dram_GB"] += x["dram_read_GB"] + x["dram_write_GB"]
    for b in by.values():
        b["share"] = b["ms"] / tot if tot else 0
        b["dram_TBps"] = b["dram_GB"] / b["ms"] if b["ms"] else 0
    res = {"tag": tag, "note": "ncu launch list (cold-cache, serialised; compare shares) of "
           "bench.py --layers 2 --steps 2 --warmup 3 (cfg2 geometry), and --set full of the "
           "timed-step launches", "by_kernel": by, "launches_tail": ls[-12:],
           "full_set": details(tag)}
    path = os.path.join(ROOT, "profiles", f"ncu_{tag}.json")
    with open(path, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(by, indent=1))
    print("wrote", path)


if __name__ == "__main__":
    main()

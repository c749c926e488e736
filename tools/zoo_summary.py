#!/usr/bin/env python
"""Summarise a kernel-zoo run (tools/gpu_kernel_zoo.sh with NCU=1) into one
JSON + one markdown table under profiles/: per shipped kernel, the
CUDA-event rate of its stage (plain run), the ncu launch list (device time
and DRAM bytes summed over every launch of that kernel) and the --set full
capture (DRAM throughput %, registers, occupancy, issue slots, L2 hit rate,
top warp stall reasons).

    python tools/zoo_summary.py TAG      # reads gpurun_out/zoo_*_TAG*
"""

from __future__ import annotations

import csv
import glob
import json
import os
import re
import sys
from collections import OrderedDict, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
SHIPPED = re.compile(r"(reshard_fused_\w+|convert_gather_\w+|load_scatter_\w+|runtile_scan_kernel|"
                     r"gen_state_kernel|adam_step_kernel|compare_kernel)\(")
DETAIL = {"Duration": "duration_us", "DRAM Throughput": "dram_pct", "Memory Throughput": "mem",
          "Registers Per Thread": "regs", "Achieved Occupancy": "achieved_occupancy_pct",
          "Theoretical Occupancy": "theoretical_occupancy_pct", "Issue Slots Busy": "issue_slots_pct",
          "L2 Hit Rate": "l2_hit_pct", "Static Shared Memory Per Block": "smem_kb",
          "Grid Size": "grid"}


def _csv_rows(path):
    rows = list(csv.reader(open(path, errors="replace")))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    return rows[start], rows[start + 1:]


def short(name: str) -> str | None:
    m = SHIPPED.search(name)
    return m.group(1) if m else None


def launch_list(path):
    hdr, rows = _csv_rows(path)
    h = {k: i for i, k in enumerate(hdr)}
    per = OrderedDict()
    for r in rows:
        per.setdefault((r[h["ID"]], r[h["Kernel Name"]]), {})[r[h["Metric Name"]]] = float(
            r[h["Metric Value"]].replace(",", ""))
    agg = defaultdict(lambda: {"launches": 0, "ms": 0.0, "dram_GB": 0.0})
    for (_, k), m in per.items():
        s = short(k)
        if not s:
            continue
        a = agg[s]
        a["launches"] += 1
        a["ms"] += m.get("gpu__time_duration.sum", 0) / 1e6
        a["dram_GB"] += (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e9
    for a in agg.values():
        a["dram_TBps"] = a["dram_GB"] / a["ms"] if a["ms"] else 0.0
    return dict(agg)


def full_capture(details_path, raw_path):
    hdr, rows = _csv_rows(details_path)
    h = {k: i for i, k in enumerate(hdr)}
    launches = OrderedDict()
    for r in rows:
        s = short(r[h["Kernel Name"]])
        if not s:
            continue
        d = launches.setdefault(r[h["ID"]], {"kernel": s})
        key = DETAIL.get(r[h["Metric Name"]])
        if key and key not in d:
            v = r[h["Metric Value"]].replace(",", "")
            try:
                d[key] = float(v)
            except ValueError:
                d[key] = v
            if key == "mem":
                d[key] = f'{v} {r[h["Metric Unit"]]}'
    stalls = {}
    if os.path.exists(raw_path):
        rows = list(csv.reader(open(raw_path, errors="replace")))
        hdr = rows[0]
        idx = [(i, c.replace("smsp__pcsamp_warps_issue_stalled_", "")) for i, c in enumerate(hdr)
               if c.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in c]
        kcol = hdr.index("Kernel Name") if "Kernel Name" in hdr else None
        for r in rows[2:]:
            if kcol is None or not short(r[kcol]):
                continue
            tot = defaultdict(float)
            for i, n in idx:
                try:
                    tot[n] += float(r[i].replace(",", ""))
                except ValueError:
                    pass
            s = sum(tot.values()) or 1.0
            stalls[r[0]] = {n: round(v / s, 3) for n, v in
                            sorted(tot.items(), key=lambda x: -x[1])[:4]}
    for i, d in launches.items():
        d["top_stalls"] = stalls.get(i, {})
    return list(launches.values())


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02b"
    cases = OrderedDict()
    for p in sorted(glob.glob(os.path.join(OUT, f"zoo_*_{tag}.json"))):
        c = os.path.basename(p)[4:-len(f"_{tag}.json")]
        d = json.loads(open(p).read().strip().splitlines()[-1])
        row = {"case": c, "src": d["src"], "tgt": d["tgt"], "dtype": d["dtype"], "fused": d["fused"],
               "parity": d["parity"], "peak_GBps": d["peak_GBps"], "kernels": d["kernels"],
               "stages": {k: {"GBps": round(v["GBps"], 1), "frac": round(v["frac"], 4),
                              "bytes": v["bytes"]} for k, v in d["stages"].items()}}
        ll = os.path.join(OUT, f"zoo_{c}_{tag}.csv")
        if os.path.exists(ll):
            row["ncu_launch_list"] = launch_list(ll)
        det = os.path.join(OUT, f"zoo_{c}_{tag}_details.csv")
        if os.path.exists(det):
            row["ncu_full"] = full_capture(det, os.path.join(OUT, f"zoo_{c}_{tag}_raw.csv"))
        cases[c] = row
    json.dump(cases, open(os.path.join(ROOT, "profiles", f"ncu_zoo_{tag}.json"), "w"), indent=1)
    lines = [f"# Kernel zoo {tag}: one workload per shipped kernel (7B geometry, 2 layers)", "",
             "CUDA-event rate = algorithmic bytes of the stage / event time, vs MEASURED_PEAKS "
             "hbm_gbs. ncu launch list = DRAM bytes / device time over every launch of the kernel "
             "in a 2-step run (cold, serialised). ncu full = the first captured launch.", "",
             "| kernel | case | layout | stage GB/s (frac) | ncu list DRAM TB/s | ncu DRAM % | regs | "
             "occ. ach/theo % | issue % | top stalls |", "|---|---|---|---|---|---|---|---|---|---|"]
    for c, r in cases.items():
        for k in r["kernels"]:
            st = ("fused" if k.startswith("reshard") else "convert" if k.startswith("convert")
                  else "load")
            s = r["stages"].get(st, {})
            ll = r.get("ncu_launch_list", {}).get(k, {})
            fc = next((x for x in r.get("ncu_full", []) if x["kernel"] == k), {})
            stl = ", ".join(f"{n} {v:.2f}" for n, v in list(fc.get("top_stalls", {}).items())[:3])
            lines.append(
                f"| `{k}` | {c} | {r['src']} → {r['tgt']} {r['dtype']} | {s.get('GBps', 0):.0f} "
                f"({s.get('frac', 0):.3f}) | {ll.get('dram_TBps', 0):.2f} ({ll.get('launches', 0)} "
                f"launches) | {fc.get('dram_pct', '')} | {fc.get('regs', '')} | "
                f"{fc.get('achieved_occupancy_pct', '')}/{fc.get('theoretical_occupancy_pct', '')} | "
                f"{fc.get('issue_slots_pct', '')} | {stl} |")
    open(os.path.join(ROOT, "profiles", f"ncu_zoo_{tag}.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()

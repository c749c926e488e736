#!/usr/bin/env python
"""The reference's OWN benchmark harness (ucp.bench.bench: partition, then
timed convert + load of the same checkpoint over a workers sweep, warm
cache) run twice on the same box: on the unmodified reference, and with this
repo's B200 engine hot-swapped into it (paper_2406_18820_b200.hotswap).
Prints one JSON line per model with both arms' wall times.

    python tools/ref_harness_bench.py [--models DenseGPT:12:768 GQA:8:1024]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", nargs="+", default=["DenseGPT:12:768", "GQA:8:1024"])
    ap.add_argument("--workers", nargs="+", type=int, default=[4, os.cpu_count() or 4])
    args = ap.parse_args()
    import ucp
    from ucp.bench import bench

    from paper_2406_18820_b200 import hotswap

    for mdesc in args.models:
        fam, layers, hidden = mdesc.split(":")
        scale = {"n_layers": int(layers), "hidden": int(hidden)}
        res = {}
        for arm in ("reference", "b200"):
            undo = hotswap.install(ucp) if arm == "b200" else None
            try:
                rep = bench(fam, args.workers, [1], scale=scale)
            finally:
                if undo:
                    undo()
            res[arm] = [{"n_workers": r.n_workers, "convert_ms": r.wall_ms_convert,
                         "load_ms": r.wall_ms_load} for r in rep.rows]
            numel = rep.rows[0].params_numel
        best = {a: min(r["convert_ms"] + r["load_ms"] for r in rows) for a, rows in res.items()}
        print(json.dumps({"model": mdesc, "params_numel": numel, "state_GB": 12 * numel / 1e9,
                          "harness": "ucp.bench.bench (reference), warm cache, DP2/PP2 Z1 -> same",
                          "arms": res, "best_convert_plus_load_ms": best,
                          "speedup": best["reference"] / best["b200"]}), flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""File pipeline throughput of the drop-in convert()/load() on tmpfs
(SURVEY §8f row 1). Prints one JSON line.

    python tools/file_bench.py [--config cfg1] [--root /dev/shm/ucpbench] [--workers 16]

The source tree is written by the product's GPU partition() (outside the
timed region). convert() reads every rank file, reshards on the GPU and
writes the atomic tree; load() reads the atomic tree and materialises every
target shard in host memory. GB/s = S / t with S = 12 B x numel.
"""

from __future__ import annotations

import argparse
import json
import os
import shutil
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--root", default="/dev/shm/ucpbench")
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"],
                    help="reference: the unmodified reference's convert()/load() from "
                         "baseline/_ref on the same source tree (same box, same tmpfs)")
    args = ap.parse_args()
    import torch

    import paper_2406_18820_b200 as U
    from paper_2406_18820_b200 import api as A

    traces = {}

    spec, src, tgt, desc = U.bench_config(args.config, args.layers)
    S = 12 * spec.total_numel
    shutil.rmtree(args.root, ignore_errors=True)
    os.makedirs(args.root)
    src_dir = os.path.join(args.root, "src")
    t = time.perf_counter()
    U.partition(U.init_state(spec, 7), src, src_dir)
    t_part = time.perf_counter() - t
    if args.impl == "reference":
        run_reference(args, src_dir, tgt, S, desc, t_part)
        return
    conv, load, load_dev = [], [], []
    for r in range(args.reps + 1):
        out = os.path.join(args.root, f"atomic{r}")
        torch.cuda.synchronize()
        t = time.perf_counter()
        U.convert(src_dir, out, n_workers=args.workers)
        conv.append(time.perf_counter() - t)
        traces["convert"] = dict(A.PIPE_TRACE)
        t = time.perf_counter()
        world = U.load(out, tgt)
        load.append(time.perf_counter() - t)
        traces["load"] = dict(A.PIPE_TRACE)
        del world
        t = time.perf_counter()
        world = U.load(out, tgt, keep_on_device=True)
        torch.cuda.synchronize()
        load_dev.append(time.perf_counter() - t)
        traces["load_keep_on_device"] = dict(A.PIPE_TRACE)
        del world
        shutil.rmtree(out)
    res = {True: [], False: [], "dev": []}
    for r in range(args.reps + 1):
        for fused in (True, False, "dev"):
            scratch = os.path.join(args.root, f"scratch{r}{fused}")
            t = time.perf_counter()
            world = U.resume(src_dir, tgt, scratch, n_workers=args.workers, fused=bool(fused),
                             keep_on_device=fused == "dev")
            torch.cuda.synchronize()
            res[fused].append(time.perf_counter() - t)
            if fused is True:
                traces["resume_fused"] = dict(A.PIPE_TRACE)
            del world
            shutil.rmtree(scratch)
    c, lo = min(conv[1:]), min(load[1:])
    rf, ru = min(res[True][1:]), min(res[False][1:])
    print(json.dumps({
        "workload": desc, "config": args.config, "state_bytes": S, "root": args.root,
        "workers": args.workers, "partition_s": t_part,
        "convert_s": c, "convert_GBps": S / c / 1e9, "load_s": lo, "load_GBps": S / lo / 1e9,
        "convert_plus_load_GBps": S / (c + lo) / 1e9, "reps": args.reps,
        "resume_fused_s": rf, "resume_fused_GBps": S / rf / 1e9,
        "resume_two_pass_s": ru, "resume_two_pass_GBps": S / ru / 1e9,
        "resume_fused_keep_on_device_GBps": S / min(res["dev"][1:]) / 1e9,
        "load_keep_on_device_s": min(load_dev[1:]),
        "load_keep_on_device_GBps": S / min(load_dev[1:]) / 1e9,
        "all_convert_s": conv, "all_load_s": load, "io_chunk": A.IO_CHUNK,
        "pipeline_wait_s_last_rep": traces}))
    shutil.rmtree(args.root, ignore_errors=True)


def run_reference(args, src_dir, tgt, S, desc, t_part):
    """The reference's own file pipeline (ucp/convert.py:422, ucp/load.py:131)
    with n_workers = the host's cores, on the tree our partition() wrote
    (byte-identical to the reference's own, tests/golden src digests)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    sys.path.insert(0, ref)
    import ucp

    assert os.path.dirname(os.path.dirname(ucp.__file__)) == ref, ucp.__file__
    import paper_2406_18820_b200 as U

    rtgt = ucp.parse_config_string(U.format_config_string(tgt))
    conv, load = [], []
    for r in range(args.reps):
        out = os.path.join(args.root, f"ref_atomic{r}")
        t = time.perf_counter()
        ucp.convert(src_dir, out, n_workers=args.workers)
        conv.append(time.perf_counter() - t)
        t = time.perf_counter()
        world = ucp.load(out, rtgt)
        load.append(time.perf_counter() - t)
        del world
        shutil.rmtree(out)
    c, lo = min(conv), min(load)
    print(json.dumps({
        "impl": "reference", "workload": desc, "config": args.config, "state_bytes": S,
        "root": args.root, "workers": args.workers, "partition_s": t_part,
        "convert_s": c, "convert_GBps": S / c / 1e9, "load_s": lo, "load_GBps": S / lo / 1e9,
        "convert_plus_load_GBps": S / (c + lo) / 1e9, "reps": args.reps,
        "all_convert_s": conv, "all_load_s": load}))
    shutil.rmtree(args.root, ignore_errors=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Host-streamed reshard whose working set exceeds HBM (north_star item 4;
VERDICT r01 item 6): every source fragment of a BASELINE config sits in one
pinned host arena, is streamed H2D window by window through the plan's
multi-buffered device slots (cudaMemcpyAsync on a copy stream), resharded by
the fused kernel on a compute stream, and every target fragment stays in HBM
(a resume straight onto the GPU, ``ReshardPlan.run_pinned(dev_tgt=...)``).
For cfg2 that is 161.7 GB of sources in host memory plus 107.8 GB of targets
in HBM: 269.5 GB of working set on a 183 GB GPU, which no device-resident
plan can hold.

    python tools/host_stream.py [--config cfg2] [--window-gb 0.4] [--reps 3]

Guards the host: the pinned arena must fit MemAvailable minus --margin-gb,
else the model is truncated to the layers that fit (reported). Parity: every
window's targets in HBM are converted back and compared with the generator
state bit for bit (the full-size identity of ReshardPlan.verify).
Prints one JSON line (and writes --out)."""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2406_18820_b200 as U  # noqa: E402
from paper_2406_18820_b200.engine import compare, pinned_host  # noqa: E402
from paper_2406_18820_b200.reshard import ReshardPlan, layout_windows, make_windows  # noqa: E402

GB = 1e9


def mem_available() -> int:
    """MemAvailable, capped by the cgroup's headroom (memory.max - memory.current)
    when the process runs under a memory limit."""
    avail = 0
    with open("/proc/meminfo") as f:
        for line in f:
            if line.startswith("MemAvailable:"):
                avail = int(line.split()[1]) * 1024
    try:
        lim = open("/sys/fs/cgroup/memory.max").read().strip()
        cur = int(open("/sys/fs/cgroup/memory.current").read().strip())
        if lim != "max":
            avail = min(avail, int(lim) - cur)
    except (OSError, ValueError):
        pass
    return avail


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--window-gb", type=float, default=0.4)
    ap.add_argument("--slots", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--margin-gb", type=float, default=24.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    spec, src, tgt, desc = U.bench_config(a.config, a.layers)
    avail = mem_available()
    layers = a.layers or spec.n_layers
    while True:  # host layout only (no device work) until the arena fits
        spec, src, tgt, desc = U.bench_config(a.config, layers)
        wins = make_windows(list(spec.params), int(a.window_gb * GB))
        src_total, _ = layout_windows(spec, src, tgt, wins, U.DType.F32)
        if src_total + a.margin_gb * GB <= avail or layers <= 1:
            break
        layers -= 1
    plan = ReshardPlan(spec, src, tgt, fused=True, window_bytes=int(a.window_gb * GB))
    dev = plan.device
    free, total = torch.cuda.mem_get_info(dev)
    t0 = time.perf_counter()
    host_src = pinned_host(plan.src_total)
    t_pin = time.perf_counter() - t0
    # fill the host arena: each window synthesised on the GPU (the product's
    # generator + partition kernels, golden-pinned), copied to its slot
    t0 = time.perf_counter()
    win = plan.buf("src_win", plan.max_src)
    atom = plan.buf("atom", plan.max_atom)
    for W in plan.windows:
        plan.gen_atomic(W, atom, 7)
        W.synth.launch(False, atom.data_ptr(), win.data_ptr(), plan.status)
        host_src[W.src_base:W.src_base + W.src_bytes].copy_(win[:W.src_bytes])
    torch.cuda.synchronize(dev)
    t_fill = time.perf_counter() - t0
    plan._bufs.pop("src_win", None)
    dev_tgt = torch.empty(max(plan.tgt_total, 256), dtype=torch.uint8, device=dev)
    plan.host_slots = a.slots
    streams = plan.host_streams()
    stream = torch.cuda.current_stream(dev)
    plan.status.reset()
    plan.run_pinned(host_src, None, streams, dev_tgt=dev_tgt)  # warm-up, synced + checked
    ms = []
    for _ in range(a.reps):
        word = torch.empty(2, dtype=torch.int64, pin_memory=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for s_ in streams:
            s_.wait_stream(stream)
        plan.run_pinned(host_src, None, streams, status_out=word, sync=False, dev_tgt=dev_tgt)
        for s_ in streams:
            stream.wait_stream(s_)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if not plan.status_ok(word):
            plan._check_windows(host_src)
        ms.append(e0.elapsed_time(e1))
    # parity: targets in HBM -> convert back under the target layout == X
    back = plan.buf("atom_back", plan.max_atom)
    ref = plan.buf("atom_ref", plan.max_atom)
    mism = torch.zeros(1, dtype=torch.int64, device=dev)
    ok = True
    for W in plan.windows:
        plan.gen_atomic(W, ref, 7)
        plan._reverse(W).launch(True, dev_tgt.data_ptr() + W.tgt_base, back.data_ptr(), plan.status)
        compare(back.data_ptr(), ref.data_ptr(), W.atom_bytes, mism)
        torch.cuda.synchronize(dev)
        ok &= int(mism.item()) == -1
    link = bench.pcie_peaks(dev, stream)
    t = min(ms) / 1e3
    res = {"config": a.config, "workload": desc, "layers": layers, "state_bytes": plan.state_bytes,
           "host_src_bytes": plan.src_total, "hbm_tgt_bytes": plan.tgt_total,
           "working_set_bytes": plan.src_total + plan.tgt_total, "hbm_total_bytes": total,
           "exceeds_hbm": plan.src_total + plan.tgt_total > total,
           "windows": len(plan.windows), "slots": a.slots, "ms": ms,
           "state_GBps": plan.state_bytes / t / GB, "h2d_GBps": plan.src_total / t / GB,
           "link": link, "h2d_frac_of_peak": (plan.src_total / t / GB / link["h2d_GBps"]
                                              if link else None),
           "pin_s": t_pin, "fill_s": t_fill, "mem_available_bytes": avail,
           "target_parity": ok,
           "what": "all sources in one pinned host arena, streamed H2D per window through "
                   f"{a.slots} device slots on a copy stream, fused reshard on a compute "
                   "stream, every target fragment kept in HBM (run_pinned(dev_tgt=...)); "
                   "CUDA events around the whole call, best of reps"}
    line = json.dumps(res)
    print(line, flush=True)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()

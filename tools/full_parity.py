#!/usr/bin/env python
"""Full-scale independent parity of the GPU reshard against the reference
itself, every (param, kind) of a BASELINE config ("use all
layers for cfg2/cfg3").

    python tools/full_parity.py --config cfg2 [--threads 16] [--window-gb 2.5]

Window by window (one LLaMA layer, the embedding, ...):
  GPU   synthesise the window's state with the product's generator, partition
        it under the source layout, run the default fused reshard (atomic
        tensors + every target fragment of every target rank), copy sources,
        atomic and targets to the host;
  CPU   on the host cores, with the UNMODIFIED reference from baseline/_ref:
        ucp.convert.union over the GPU's source fragments == the GPU atomic,
        ucp.parallel.extract_fragment of that union == every GPU target
        fragment, byte for byte (pads included), and ucp.tensor.hash_unit
        over every element == the union (so the generator is checked too;
        v = |.|). Vocab-padded units (cfg3's embedding / output layer; the
        reference has no vocab padding) use the oracle restatement.
Prints one JSON line (and writes it to --out): units / fragments / bytes
compared, mismatches (must be 0), timings.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2406_18820_b200 as U  # noqa: E402
from oracle import ucp_oracle as O  # noqa: E402
from paper_2406_18820_b200.layout import vocab_padded_rows  # noqa: E402
from paper_2406_18820_b200.reshard import ReshardPlan  # noqa: E402

GEN_CHUNK = 1 << 24  # elements per hash_unit call (bounded temporaries per thread)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--window-gb", type=float, default=2.5)
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--no-gen-check", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("--windows", default=None,
                    help="A:B -- only windows A..B-1 (a long config split over calls); the "
                         "JSON then counts those windows' units only")
    a = ap.parse_args()
    ucp = bench.reference_ucp()
    if ucp is None:
        raise SystemExit("baseline/_ref (the unmodified reference) is not installed")
    from ucp import tensor as ref_tensor

    spec, src, tgt, desc = U.bench_config(a.config, a.layers)
    wdt = U.DType.F32 if a.dtype == "f32" else U.DType.BF16
    plan = ReshardPlan(spec, src, tgt, dtype=wdt, fused=True,
                       window_bytes=int(a.window_gb * 1e9))
    dev = plan.device
    arena = plan.buf("src_win", plan.max_src)
    atom = plan.buf("atom", plan.max_atom)
    tgtb = plan.buf("tgt0", plan.max_tgt)
    plain = lambda c: dataclasses.replace(c, vocab_multiple=1)
    pool = ThreadPoolExecutor(a.threads)
    res = {"config": a.config, "workload": desc, "src": U.format_config_string(src),
           "tgt": U.format_config_string(tgt), "target_weight_dtype": a.dtype,
           "threads": a.threads, "windows": len(plan.windows), "units": 0, "units_reference": 0,
           "units_port": 0, "fragments": 0, "bytes_compared": 0, "atomic_mismatch": [],
           "target_mismatch": [], "generator_mismatch": [], "state_bytes": plan.state_bytes}
    t_gpu = t_cpu = 0.0
    t0 = time.perf_counter()
    w_lo, w_hi = 0, len(plan.windows)
    if a.windows:
        lo_s, hi_s = a.windows.split(":")
        w_lo, w_hi = int(lo_s or 0), int(hi_s or len(plan.windows))
    res["window_range"] = [w_lo, w_hi]
    for wi, W in enumerate(plan.windows):
        if not w_lo <= wi < w_hi:
            continue
        tg = time.perf_counter()
        plan.status.reset()
        plan.gen_atomic(W, atom, 7)
        W.synth.launch(False, atom.data_ptr(), arena.data_ptr(), plan.status)
        W.fused.launch(arena.data_ptr(), atom.data_ptr(), tgtb.data_ptr(), plan.status)
        W.conv.launch(True, arena.data_ptr(), atom.data_ptr(), plan.status)
        W.load.launch(False, atom.data_ptr(), tgtb.data_ptr(), plan.status)
        torch.cuda.synchronize(dev)
        if plan.status.read()[0] != (1 << 64) - 1:
            raise SystemExit(f"window {wi}: the GPU reported a replica / pad failure")
        hs = arena[:W.src_bytes].cpu().numpy()
        ha = atom[:W.atom_bytes].cpu().numpy()
        ht = tgtb[:W.tgt_bytes].cpu().numpy()
        t_gpu += time.perf_counter() - tg
        tc = time.perf_counter()
        frags = {}
        for g, i, m, off, n in W.src_frags:
            frags.setdefault((m.param, m.kind), []).append(
                (m, hs[off:off + 4 * n].view("<f4").reshape(m.shape)))
        vocab = {k for k in frags if vocab_padded_rows(spec.param(k[0]), tgt) is not None
                 or vocab_padded_rows(spec.param(k[0]), src) is not None}
        arms = []
        if len(vocab) < len(frags):
            arms.append(bench.CpuArm(spec, plain(src), plain(tgt),
                                     {k: v for k, v in frags.items() if k not in vocab}))
        if vocab:
            arms.append(bench.CpuArm(spec, src, tgt, {k: v for k, v in frags.items() if k in vocab},
                                     prefer_reference=False))
        tgt_at = {(g, m.param, m.kind): (off, n, dt, m) for g, i, m, off, n, dt in W.tgt_frags}

        def check(arm, key):
            p = arm.spec.param(key[0])
            full = np.ascontiguousarray(arm.union(p, arm.src, arm.frags[key]), dtype=np.float32)
            out = {"key": key, "bad_atom": False, "bad_gen": False, "bad_tgt": [], "n": 0, "b": 0}
            ao = W.atom[key]
            got_a = ha[ao:ao + full.nbytes]
            out["bad_atom"] = not np.array_equal(full.reshape(-1).view(np.uint8), got_a)
            out["b"] += full.nbytes
            if not a.no_gen_check:
                base = ref_tensor.stream_base(7, spec.tied_leader(key[0]), key[1])
                flat = full.reshape(-1).view(np.uint32)
                for s0 in range(0, full.size, GEN_CHUNK):
                    want = ref_tensor.hash_unit(base, s0, min(GEN_CHUNK, full.size - s0))
                    if key[1] == "v":
                        want = np.abs(want)
                    if not np.array_equal(want.view(np.uint32), flat[s0:s0 + want.size]):
                        out["bad_gen"] = True
                        break
            for g, meta in arm.by_unit.get(key, ()):
                ref = np.ascontiguousarray(arm.extract(p, arm.tgt, meta, full))
                off, n, dt, m = tgt_at[(g, key[0], key[1])]
                if dt is not U.DType.F32:  # the load-side weight cast (ucp/load.py:204-205)
                    if arm.kind == "reference":
                        ref = ref_tensor.cast(ref_tensor.Tensor(ref_tensor.DType.F32, ref.shape, ref),
                                              ref_tensor.DType.BF16).data
                    else:
                        ref = O.cast_weight(ref, "BF16")
                rb = np.ascontiguousarray(ref).reshape(-1).view(np.uint8)
                gb = ht[off:off + dt.itemsize * n]
                if rb.size != gb.size or not np.array_equal(rb, gb):
                    out["bad_tgt"].append(g)
                out["n"] += 1
                out["b"] += rb.size
            return out

        jobs = [(arm, key) for arm in arms for key in arm.frags]
        for r in pool.map(lambda j: check(*j), jobs):
            res["units"] += 1
            res["fragments"] += r["n"]
            res["bytes_compared"] += r["b"]
            if r["bad_atom"]:
                res["atomic_mismatch"].append(list(r["key"]))
            if r["bad_gen"]:
                res["generator_mismatch"].append(list(r["key"]))
            if r["bad_tgt"]:
                res["target_mismatch"].append([*r["key"], r["bad_tgt"]])
        for arm in arms:
            res["units_reference" if arm.kind == "reference" else "units_port"] += len(arm.frags)
        t_cpu += time.perf_counter() - tc
        print(f"window {wi + 1}/{len(plan.windows)}: units {res['units']} fragments "
              f"{res['fragments']} mismatches {len(res['atomic_mismatch'])}/"
              f"{len(res['target_mismatch'])}/{len(res['generator_mismatch'])}",
              file=sys.stderr, flush=True)
    res.update({"gpu_s": t_gpu, "cpu_s": t_cpu, "wall_s": time.perf_counter() - t0,
                "expected_units": sum(3 * len(W.params) for W in plan.windows[w_lo:w_hi]),
                "expected_fragments": sum(len(W.tgt_frags) for W in plan.windows[w_lo:w_hi]),
                "identical": not (res["atomic_mismatch"] or res["target_mismatch"]
                                  or res["generator_mismatch"]),
                "what": "GPU fused reshard vs the unmodified reference (ucp.convert.union + "
                        "ucp.parallel.extract_fragment from baseline/_ref) on the GPU's own "
                        "source fragments, every unit of every layer; generator vs "
                        "ucp.tensor.hash_unit over every element; vocab-padded units vs the "
                        "oracle restatement"})
    line = json.dumps(res)
    print(line, flush=True)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""One workload per shipped kernel family, for per-kernel evidence:
CUDA-event rates (run plain) and ncu launch lists / --set full captures
(run under ncu by tools/gpu_kernel_zoo.sh).

    python tools/kernel_zoo.py --case fused_staged [--steps 10]

Every case is a ReshardPlan over a LLaMA-2-7B-geometry slice (2 layers,
cfg2 layouts unless the case changes them) or, for the general ops, a
synthetic model with one large averaged (ASYNC_PARTIAL) vector. It prints
one JSON line: per stage (fused / convert / load launches of a step) the
algorithmic bytes, mean ms per step from CUDA events, GB/s and the fraction
of MEASURED_PEAKS.json hbm_gbs, plus which kernels the stage launches.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2406_18820_b200 as U  # noqa: E402
from paper_2406_18820_b200.plan import NCLASS  # noqa: E402
from paper_2406_18820_b200.reshard import ReshardPlan  # noqa: E402
from paper_2406_18820_b200.spec import DType, ModelSpec, ParamKind, ParamSpec  # noqa: E402

GB = 1e9
CFG = lambda dp=1, tp=1, zero="z1": U.ParallelConfig(dp=dp, tp=tp, zero_stage=U.ZeroStage(zero))

# case -> (spec builder, src, tgt, fused, dtype, kernels it exists for)
CASES = {
    "fused_f32": ("llama", CFG(4, 2), CFG(2, 4), True, DType.F32, ["reshard_fused_f32"]),
    "fused_bf16": ("llama", CFG(4, 2), CFG(2, 4), True, DType.BF16, ["reshard_fused_bf16"]),
    "fused_f16": ("llama", CFG(4, 2), CFG(2, 4), True, DType.F16, ["reshard_fused_f16"]),
    "fused_staged": ("llama", CFG(3, 2), CFG(2, 4), True, DType.F32, ["reshard_fused_realign"]),
    "fused_staged5": ("llama", CFG(5, 2), CFG(2, 4), True, DType.F32, ["reshard_fused_realign"]),
    "unfused_f32": ("llama", CFG(4, 2), CFG(2, 4), False, DType.F32,
                    ["convert_gather_f32", "load_scatter_f32"]),
    "unfused_bf16": ("llama", CFG(4, 2), CFG(2, 4), False, DType.BF16, ["load_scatter_bf16"]),
    "unfused_f16": ("llama", CFG(4, 2), CFG(2, 4), False, DType.F16, ["load_scatter_f16"]),
    "unfused_staged": ("llama", CFG(3, 2), CFG(2, 4), False, DType.F32,
                       ["convert_gather_realign"]),
    "unfused_staged_load": ("llama", CFG(4, 2), CFG(3, 2), False, DType.F32,
                            ["load_scatter_realign"]),
    "fused_staged_bf16": ("llama", CFG(3, 2), CFG(2, 4), True, DType.BF16,
                          ["reshard_fused_realign"]),
    # f64 MEAN over tp=4 groups + ZeRO pad checks (convert); partial NOISE
    # + ZeRO re-pad (load): the GENERAL class of the move kernels
    "general_ops": ("partial", CFG(2, 4), CFG(3, 2), False, DType.F32,
                    ["convert_gather_ops", "load_scatter_ops"]),
    # the same ops with every source and destination on one 16-B phase
    # (n = 2^26, dp 2 -> 2): the vector branch of the OPS kernels alone
    "ops_vec": ("partial_even", CFG(2, 4), CFG(2, 2), False, DType.F32,
                ["convert_gather_ops", "load_scatter_ops"]),
}


def partial_spec(n: int = (1 << 26) + 1) -> ModelSpec:
    return ModelSpec("zoo-partial", 1, (), (ParamSpec("big.alibi", (n,), 0,
                                                      ParamKind.ASYNC_PARTIAL),))


def peak() -> float:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", required=True, choices=sorted(CASES))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--layers", type=int, default=2)
    a = ap.parse_args()
    kind, src, tgt, fused, dtype, kernels = CASES[a.case]
    spec = (U.llama_spec("7b", a.layers) if kind == "llama"
            else partial_spec(1 << 26) if kind == "partial_even" else partial_spec())
    plan = ReshardPlan(spec, src, tgt, dtype=dtype, fused=fused)
    plan.synthesize(7)
    par = plan.verify(7)
    plan.status.reset()
    for _ in range(a.warmup):
        plan.step_device()
    torch.cuda.synchronize()
    plan.check()
    evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in plan.windows]
           for _ in range(a.steps)]
    for k in range(a.steps):
        plan.step_device(None, evs[k])
    torch.cuda.synchronize()
    plan.check()
    ms = lambda i, j: sum(e[i].elapsed_time(e[j]) for st in evs for e in st) / a.steps
    pk = peak()
    stages = {
        "fused": (sum(plan.fused_bytes.values()), ms(0, 1), [W.fused for W in plan.windows]),
        "convert": (plan.bytes["R_c"] + plan.bytes["W_c"], ms(1, 2), [W.conv for W in plan.windows]),
        "load": (plan.bytes["R_l"] + plan.bytes["W_l"], ms(2, 3), [W.load for W in plan.windows]),
    }
    out = {"case": a.case, "kernels": kernels, "src": U.format_config_string(src),
           "tgt": U.format_config_string(tgt), "dtype": dtype.name, "fused": fused,
           "state_bytes": plan.state_bytes, "parity": par, "peak_GBps": pk, "stages": {}}
    for name, (nb, t, progs) in stages.items():
        if not nb:
            continue
        tiles = [int(sum(p.class_info[c] for p in progs)) for c in range(NCLASS)]
        out["stages"][name] = {"bytes": int(nb), "ms": t, "GBps": nb / (t / 1e3) / GB,
                               "frac": nb / (t / 1e3) / GB / pk, "tiles_per_class": tiles}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

"""One dp=3 window through the fused path, for ncu of reshard_fused_scalar."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2406_18820_b200 as U  # noqa: E402
from paper_2406_18820_b200.reshard import ReshardPlan  # noqa: E402

spec = U.llama_spec("7b", 2)
src = U.ParallelConfig(dp=3, tp=2, zero_stage=U.ZeroStage.Z1)
tgt = U.ParallelConfig(dp=2, tp=4, zero_stage=U.ZeroStage.Z1)
plan = ReshardPlan(spec, src, tgt, fused=True)
plan.synthesize(7)
for _ in range(3):
    plan.step_device()
torch.cuda.synchronize()
plan.check()
print("ok")

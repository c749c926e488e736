"""How fast is a layout whose ZeRO partitions do not share the atomic's
16-B phase (dp = 3: partition starts at k * ceil(n / 3) elements)? Times
ReshardPlan.step_device for a 7B-geometry slice under several source dp."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2406_18820_b200 as U  # noqa: E402
from paper_2406_18820_b200.reshard import ReshardPlan  # noqa: E402
from paper_2406_18820_b200.plan import CLASS_GENERAL  # noqa: E402

spec = U.llama_spec("7b", 4)
tgt = U.ParallelConfig(dp=2, tp=4, zero_stage=U.ZeroStage.Z1)
peak = 6536.4
fused = "unfused" not in sys.argv[1:]
for dp in (2, 3, 4, 5):
    src = U.ParallelConfig(dp=dp, tp=2, zero_stage=U.ZeroStage.Z1)
    plan = ReshardPlan(spec, src, tgt, fused=fused)
    plan.synthesize(7)
    res = plan.verify(7)
    gen = sum(int(W.conv.class_info[CLASS_GENERAL]) + int(W.load.class_info[CLASS_GENERAL])
              for W in plan.windows)
    plan.status.reset()
    for _ in range(3):
        plan.step_device()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        plan.step_device()
    b.record()
    torch.cuda.synchronize()
    plan.check()
    ms = a.elapsed_time(b) / 10
    hbm = plan.hbm_bytes
    print(f"src dp={dp}: {plan.state_bytes / ms / 1e6:.0f} GB/s of state, {hbm / ms / 1e6 / peak:.3f} of peak, "
          f"fused units {plan.n_fused_units}/{plan.n_units}, general tiles {gen}, parity {res}", flush=True)
    plan.free()
    del plan
    torch.cuda.empty_cache()

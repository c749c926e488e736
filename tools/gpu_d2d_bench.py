"""Device-to-device reshard() throughput: source fragments as separate CUDA
tensors (synthesised by the GPU generator + the load kernels), targets
allocated by reshard(); cfg2 geometry with N layers."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2406_18820_b200 as U  # noqa: E402
from paper_2406_18820_b200.reshard import ReshardPlan  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
spec, src, tgt, _ = U.bench_config("cfg2", layers)
plan = ReshardPlan(spec, src, tgt, fused=True)
arena = plan.synthesize(7)
torch.cuda.synchronize()
shards = {g: [None] * len(U.enumerate_rank_records(spec, src, g)) for g in range(src.world_size)}
for W in plan.windows:
    for g, i, m, off, n in W.src_frags:
        shards[g][i] = arena[W.src_base + off:W.src_base + off + 4 * n].view(torch.float32).clone()
plan.free()
del arena, plan
torch.cuda.empty_cache()
S = 12 * spec.total_numel
out = U.reshard(spec, src, tgt, shards)  # warm-up (compile + allocate)
del out
torch.cuda.synchronize()
import time  # noqa: E402

ts = []
for _ in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = U.reshard(spec, src, tgt, shards)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t)
    del out
print(f"device-to-device reshard(), cfg2 geometry {layers} layers, {S / 1e9:.2f} GB state: "
      f"best {min(ts) * 1e3:.1f} ms wall incl. plan compile + output allocation = "
      f"{S / min(ts) / 1e9:.0f} GB/s of state")

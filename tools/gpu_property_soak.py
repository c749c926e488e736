"""Soak the GPU property test: many more random (model, src, tgt, dtype)
draws through ReshardPlan (fused and unfused), the device-to-device
reshard() and the oracle. Usage: python tools/gpu_property_soak.py N"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402
import torch  # noqa: E402
from hypothesis import HealthCheck, given, settings  # noqa: E402

import paper_2406_18820_b200 as U  # noqa: E402
from oracle import ucp_oracle as O  # noqa: E402
from paper_2406_18820_b200.reshard import ReshardPlan  # noqa: E402
from paper_2406_18820_b200.spec import DType  # noqa: E402
from test_property_configs import cell  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
count = [0]


@settings(max_examples=N, deadline=None, suppress_health_check=list(HealthCheck), derandomize=False)
@given(cell())
def soak(c):
    spec, src, tgt, dt = c
    state = O.init_state(spec, 5)
    shards = O.partition_mem(spec, state, src)
    host = {g: [a for _, a in v] for g, v in shards.items()}
    want = O.world_digest(O.load_mem(spec, state, tgt, dt))
    recs = {g: U.enumerate_rank_records(spec, tgt, g) for g in range(tgt.world_size)}
    for fused in (False, True):
        plan = ReshardPlan(spec, src, tgt, dtype=DType[dt], fused=fused, window_bytes=1 << 15,
                           tile_bytes=1 << 13)
        out = plan.run_host(host)
        got = {g: list(zip(recs[g], out.get(g, []))) for g in range(tgt.world_size)}
        assert O.world_digest(got) == want, (fused, U.format_config_string(src),
                                             U.format_config_string(tgt), dt)
    dev = {g: [torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).cuda() for a in v]
           for g, v in host.items()}
    out = U.reshard(spec, src, tgt, dev, dtype=DType[dt])

    def bits(t):
        if t.dtype == torch.bfloat16:
            return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
        return t.cpu().numpy()

    got = {g: list(zip(recs[g], [bits(t) for t in out.get(g, [])])) for g in range(tgt.world_size)}
    assert O.world_digest(got) == want, ("d2d", U.format_config_string(src),
                                         U.format_config_string(tgt), dt)
    count[0] += 1


soak()
print(f"soak ok: {count[0]} random cells x (unfused, fused, device-to-device)")

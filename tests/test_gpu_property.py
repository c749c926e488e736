"""Random (model, source layout, target layout) triples through the real
kernels (fused and unfused ReshardPlan) vs the oracle."""

import pytest
from hypothesis import HealthCheck, given, settings

import paper_2406_18820_b200 as U
from oracle import ucp_oracle as O
from paper_2406_18820_b200.reshard import ReshardPlan
from paper_2406_18820_b200.spec import DType

from test_property_configs import cell

pytestmark = pytest.mark.gpu


@settings(max_examples=20, deadline=None, suppress_health_check=list(HealthCheck))
@given(cell())
def test_random_reshard_gpu(c):
    spec, src, tgt, dt = c
    state = O.init_state(spec, 5)
    shards = O.partition_mem(spec, state, src)
    host = {g: [a for _, a in v] for g, v in shards.items()}
    want = O.world_digest(O.load_mem(spec, state, tgt, dt))
    for fused in (False, True):
        plan = ReshardPlan(spec, src, tgt, dtype=DType[dt], fused=fused, window_bytes=1 << 15,
                           tile_bytes=1 << 13)
        out = plan.run_host(host)
        recs = {g: U.enumerate_rank_records(spec, tgt, g) for g in range(tgt.world_size)}
        got = {g: list(zip(recs[g], out.get(g, []))) for g in range(tgt.world_size)}
        assert O.world_digest(got) == want, (fused, U.format_config_string(src),
                                             U.format_config_string(tgt))

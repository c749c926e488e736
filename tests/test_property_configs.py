"""Property tests over random (model, source layout, target layout) triples,
in the spirit of the reference's hypothesis suites: the descriptor compiler
(unfused and fused) executed by the interpreter must reproduce the oracle for
every draw, including dp that does not divide the fragments (ZeRO pads,
misaligned pieces), interleaved PP, tp up to 8, ZeRO-3 and sp folding."""

import numpy as np
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import paper_2406_18820_b200 as U
from oracle import ucp_oracle as O
from paper_2406_18820_b200.spec import DType, ParallelConfig, PPSchedule, ZeroStage

from test_plan_interp import _arena_extract, _arena_union, _fused_world


@st.composite
def model(draw):
    fam = draw(st.sampled_from(["DenseGPT", "MoE", "GQA"]))
    hidden = draw(st.sampled_from([16, 32, 48, 64]))
    scale = {"n_layers": draw(st.integers(0, 4)), "hidden": hidden}
    if fam == "MoE":
        scale["n_experts"] = draw(st.integers(1, 3))
    if fam == "GQA":
        q = draw(st.sampled_from([h for h in (1, 2, 4, 8, 16) if hidden % h == 0]))
        scale.update(q_heads=q, kv_heads=draw(st.sampled_from([k for k in (1, 2, 4) if q % k == 0])))
    return U.make_model(fam, scale)


@st.composite
def config(draw, spec):
    for _ in range(50):
        zero = draw(st.sampled_from(["z0", "z1", "z3"]))
        dp = draw(st.integers(1, 4))
        tp = 1 if zero == "z3" else draw(st.sampled_from([1, 2, 4, 8]))
        pp = 1 if zero == "z3" else draw(st.integers(1, 3))
        v = draw(st.sampled_from([0, 2])) if pp > 1 else 0
        sp = draw(st.sampled_from([s for s in (1, 2) if dp % s == 0]))
        cfg = ParallelConfig(dp=dp, tp=tp, pp=pp, sp=sp, zero_stage=ZeroStage(zero),
                             pp_schedule=PPSchedule("interleaved", v) if v else PPSchedule())
        try:
            U.validate_model_config(spec, cfg)
            return cfg
        except U.UcpError:
            continue
    return ParallelConfig()


@st.composite
def cell(draw):
    spec = draw(model())
    return spec, draw(config(spec)), draw(config(spec)), draw(st.sampled_from(["F32", "BF16"]))


@settings(max_examples=25, deadline=None, suppress_health_check=list(HealthCheck))
@given(cell())
def test_random_reshard_matches_oracle(c):
    spec, src, tgt, dt = c
    state = O.init_state(spec, 3)
    shards = O.partition_mem(spec, state, src)
    got, fails, _ = _arena_union(spec, src, shards, tile_bytes=2048)
    assert fails == []
    for p in spec.params:
        for k in ("weight", "m", "v"):
            assert np.array_equal(got[(p.name, k)].view(np.uint32),
                                  state[p.name][k].view(np.uint32)), (p.name, k)
    want = O.world_digest(O.load_mem(spec, state, tgt, dt))
    world, _ = _arena_extract(spec, tgt, state, DType[dt], tile_bytes=2048)
    fixed = {g: [(m, a.reshape(U.plan.fragment_shape(spec.param(m.param), tgt, m))) for m, a in v]
             for g, v in world.items()}
    assert O.world_digest(fixed) == want
    fworld, fatom, _, _ = _fused_world(spec, src, tgt, shards, DType[dt], tile_bytes=2048)
    assert O.world_digest(fworld) == want

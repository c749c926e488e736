"""Vocab padding (extension, SURVEY G3 / BASELINE cfg3): embedding and
output-layer rows padded to ceil(V / (m * tp)) * m * tp in the sharded
layout, stripped by convert, zero re-padded by load. The reference has no
vocab padding, so parity is against the oracle's restatement plus the
size-independent round-trip identity."""

import numpy as np
import pytest

import paper_2406_18820_b200 as U
from oracle import ucp_oracle as O
from paper_2406_18820_b200.layout import all_rank_records, vocab_padded_rows
from paper_2406_18820_b200.spec import DType, ParallelConfig, ZeroStage

from test_plan_interp import _arena_extract, _arena_union, _fused_world

SPEC = U.make_model("GQA", {"n_layers": 2, "hidden": 64, "q_heads": 8, "kv_heads": 2})
SRC = ParallelConfig(dp=2, tp=2, zero_stage=ZeroStage.Z1, vocab_multiple=100)  # 512 -> 600
TGT = ParallelConfig(dp=3, tp=4, zero_stage=ZeroStage.Z1, vocab_multiple=36)   # 512 -> 576


def test_padded_rows_and_records():
    emb = SPEC.param("embed.tokens")
    assert vocab_padded_rows(emb, SRC) == 600 and vocab_padded_rows(emb, TGT) == 576
    assert vocab_padded_rows(SPEC.param("layers.0.attn_qkv"), SRC) is None
    assert U.llama_spec("13b").param("embed.tokens").shape[0] == 32000
    l13 = U.llama_spec("13b")
    assert vocab_padded_rows(l13.param("head.out"), ParallelConfig(tp=4, vocab_multiple=128)) == 32256
    assert vocab_padded_rows(l13.param("head.out"), ParallelConfig(tp=2, vocab_multiple=128)) == 32000
    for cfg in (SRC, TGT):
        recs = all_rank_records(SPEC, cfg)
        for g in range(cfg.world_size):
            ours = [O.record_tuple(m) for m in recs[g]]
            want = [O.record_tuple(r) for r in O.rank_records(SPEC, cfg, g)]
            assert ours == want
    d = U.spec.config_to_dict(TGT)
    assert d["vocab_multiple"] == 36 and U.spec.config_from_dict(d) == TGT
    assert "vocab_multiple" not in U.spec.config_to_dict(ParallelConfig())


def test_oracle_round_trip_strips_and_repads():
    state = O.init_state(SPEC, 7)
    shards = O.partition_mem(SPEC, state, SRC)
    atomic = O.convert_mem(SPEC, SRC, shards)
    for p in SPEC.params:
        for k in ("weight", "m", "v"):
            assert np.array_equal(atomic[p.name][k], state[p.name][k])
    world = O.load_mem(SPEC, atomic, TGT)
    # the last tp rank's embedding fragment ends in 576 - 512 = 64 zero rows
    last = TGT.rank_of(0, 3, 0)
    emb = next(a for r, a in world[last] if r["param"] == "embed.tokens" and r["kind"] == "weight")
    assert emb.shape == (144, 64) and not emb[80:].any() and emb[:80].any()


def test_interpreter_union_and_extract_match_oracle():
    state = O.init_state(SPEC, 7)
    shards = O.partition_mem(SPEC, state, SRC)
    got, fails, _ = _arena_union(SPEC, SRC, shards)
    assert fails == []
    for p in SPEC.params:
        for k in ("weight", "m", "v"):
            assert np.array_equal(got[(p.name, k)], state[p.name][k]), (p.name, k)
    for dt in (DType.F32, DType.BF16):
        world, _ = _arena_extract(SPEC, TGT, state, dt)
        want = O.load_mem(SPEC, state, TGT, dt.name)
        fixed = {g: [(m, a.reshape(U.plan.fragment_shape(SPEC.param(m.param), TGT, m)))
                     for m, a in items] for g, items in world.items()}
        assert O.world_digest(fixed) == O.world_digest(want)


def test_fused_matches_oracle():
    state = O.init_state(SPEC, 7)
    shards = O.partition_mem(SPEC, state, SRC)
    world, atomics, fused, _ = _fused_world(SPEC, SRC, TGT, shards, DType.BF16)
    assert O.world_digest(world) == O.world_digest(O.load_mem(SPEC, state, TGT, "BF16"))
    for (name, k), a in atomics.items():
        assert np.array_equal(a, state[name][k].reshape(-1))

"""Pin the CPU oracle to the reference's own outputs (tests/golden/*).

The golden files were produced by tests/golden/make_golden.py importing the
reference package; these tests prove the oracle restates it exactly, so the
oracle can stand in for the reference on the GPU box (where /root/reference
does not exist).
"""

import os

import numpy as np
import pytest

from helpers import PIPE_SPECS, cell_cfgs, cell_spec
from oracle import ucp_oracle as O
from paper_2406_18820_b200 import parse_config_string

FAST_CELLS = ("pad", "gqa", "moe")


def test_generator_bits(golden):
    for g in golden["generator"]:
        assert O.stream_base(g["seed"], g["name"], g["tag"]) == g["base"]
        got = O.hash_window(g["base"], g["start"], len(g["bits"])).view(np.uint32)
        assert [int(x) for x in got] == g["bits"], (g["name"], g["tag"])


def test_reference_frozen_table():
    # the reference test's FROZEN patterns (pkg/tests/test_tensor.py:36-53)
    frozen = {(7, "layers.0.attn_qkv", "weight"): [0x3F00DBD6, 0xBBD3F800, 0xBF7E6E4A,
                                                   0x3F317AC0, 0x3F72B0EC, 0x3E6F6380],
              (7, "layers.0.attn_qkv", "m"): [0xBF519234, 0xBE3EA338],
              (0, "embed.tokens", "weight"): [0xBF253D8E, 0xBEB5FBD8, 0x3EEA2528],
              (123456789, "pos.alibi", "v"): [0xBD2E4AC0]}
    for (seed, name, tag), want in frozen.items():
        got = O.gen_values(seed, name, tag, (len(want),)).view(np.uint32)
        assert [int(x) for x in got] == want
    assert int(O.gen_values(123456789, "pos.alibi", "v", (8,)).view(np.uint32)[7]) == 0x3BDC5600


def test_bf16_table(golden_arrays):
    x = golden_arrays["cast_in"].view(np.float32)
    assert np.array_equal(O.bf16_bits(x), golden_arrays["cast_bf16"])


def test_f16_table(golden_arrays):
    x = golden_arrays["cast_in"].view(np.float32)
    assert np.array_equal(O.f16_bits(x), golden_arrays["cast_f16"])


@pytest.mark.parametrize("tp", [2, 3, 4, 5, 8])
def test_partial_noise_table(golden_arrays, tp):
    x = golden_arrays["noise_in"].view(np.float32)
    for t in range(tp):
        got = O.partial_noise(x, t, tp).view(np.uint32)
        assert np.array_equal(got, golden_arrays[f"noise_tp{tp}_r{t}"]), (tp, t)


def test_partial_noise_mean_recovers_input(golden_arrays):
    # the property the reference relies on (ucp/parallel.py:340-349)
    x = golden_arrays["noise_in"].view(np.float32)
    x = x[np.isfinite(x)]
    for tp in (2, 3, 4, 8):
        acc = O.partial_noise(x, 0, tp).astype(np.float64)
        for t in range(1, tp):
            acc = acc + O.partial_noise(x, t, tp).astype(np.float64)
        back = (acc / float(tp)).astype(np.float32)
        assert np.array_equal(back.view(np.uint32), x.view(np.uint32)), tp


def test_record_digests(golden):
    import hashlib
    import json

    from helpers import SCALES
    from paper_2406_18820_b200.zoo import make_model

    for key, want in golden["records"].items():
        fam, cstr = key.split("|")
        spec = make_model(fam, SCALES[fam])
        cfg = parse_config_string(cstr)
        if "error" in want:
            with pytest.raises(O.OracleError) as ei:
                for g in range(cfg.world_size):
                    O.rank_records(spec, cfg, g)
                for p in spec.params:
                    O.tp_split_mode(p, cfg.tp)
            assert ei.value.name == want["error"]
            continue
        allr = []
        for g in range(cfg.world_size):
            allr.append([[r["param"], r["kind"], r["pattern"], list(r["placement"]),
                          list(r["shape"]),
                          None if r["segments"] is None else [list(s) for s in r["segments"]],
                          None if r["flat_range"] is None else list(r["flat_range"]),
                          r["pad_elems"]] for r in O.rank_records(spec, cfg, g)])
        assert hashlib.sha256(json.dumps(allr).encode()).hexdigest() == want["sha256"], key


def test_flat_split_known_answers():
    assert O.flat_split(1024, 3) == (1026, 2, [(0, 342), (342, 684), (684, 1026)])
    assert O.flat_split(1024, 2) == (1024, 0, [(0, 512), (512, 1024)])
    assert O.flat_split(7, 4) == (8, 1, [(0, 2), (2, 4), (4, 6), (6, 8)])


def _cells(golden, names=None):
    for row in golden["pipelines"]:
        if names is None or row["name"] in names:
            yield row


@pytest.mark.parametrize("name", list(FAST_CELLS) + ["DenseGPT.%d" % i for i in range(6)]
                         + ["MoE.%d" % i for i in range(6)] + ["GQA.%d" % i for i in range(6)])
def test_pipeline_digests(golden, tmp_path, name):
    row = next(_cells(golden, {name}))
    spec = cell_spec(golden, row)
    src_cfg, tgt_cfg = cell_cfgs(row)
    state = O.init_state(spec, 7)
    shards = O.partition_mem(spec, state, src_cfg)
    src = str(tmp_path / "src")
    O.write_tree(spec, src_cfg, shards, src)
    assert O.dir_digest(src) == row["src_digest"]
    atomic = O.convert_mem(spec, src_cfg, shards)
    adir = str(tmp_path / "atomic")
    O.write_atomic(spec, atomic, adir, fingerprint=O.config_fingerprint(src))
    assert O.dir_digest(adir) == row["atomic_digest"]
    for dt in ("F32", "BF16", "F16"):
        with np.errstate(all="ignore"):
            world = O.load_mem(spec, atomic, tgt_cfg, dt)
        assert O.world_digest(world) == row[f"world_{dt}"], dt


def test_golden_vec16_bytes():
    path = os.path.join(os.path.dirname(__file__), "golden", "golden_vec16.ucpt")
    want = open(path, "rb").read()
    assert O.ucpt_bytes(O.gen_values(7, "pos.alibi", "weight", (16,))) == want
    assert np.array_equal(O.ucpt_parse(want), O.gen_values(7, "pos.alibi", "weight", (16,)))


def test_union_unit_cases():
    # the reference's hand cases (pkg/tests/test_convert.py:61-205)
    from paper_2406_18820_b200 import ParallelConfig, ParamKind, ParamSpec, ZeroStage

    def rec(p, pattern, placement, shape, flat_range=None, pad=0, segments=None):
        return {"param": p.name, "kind": "weight", "pattern": pattern, "placement": placement,
                "shape": shape, "flat_range": flat_range, "pad_elems": pad, "segments": segments}

    p = ParamSpec("pos", (1,), 0, ParamKind.ASYNC_PARTIAL)
    cfg = ParallelConfig(tp=2)
    out = O.union(p, cfg, [(rec(p, "partial", (0, 0, 0), (1,)), np.float32([2.0])),
                           (rec(p, "partial", (0, 1, 0), (1,)), np.float32([4.0]))])
    assert out.tolist() == [3.0]
    p = ParamSpec("ln", (3,), 0, ParamKind.LAYERNORM_WEIGHT)
    cfg = ParallelConfig(dp=2, zero_stage=ZeroStage.Z3)
    out = O.union(p, cfg, [(rec(p, "shard_v", (0, 0, 1), (2,), (2, 4), 1), np.float32([3, 0])),
                           (rec(p, "shard_v", (0, 0, 0), (2,), (0, 2)), np.float32([1, 2]))])
    assert out.tolist() == [1.0, 2.0, 3.0]
    with pytest.raises(O.OracleError) as ei:
        O.union(p, cfg, [(rec(p, "shard_v", (0, 0, 1), (2,), (2, 4), 1), np.float32([3, -0.0])),
                         (rec(p, "shard_v", (0, 0, 0), (2,), (0, 2)), np.float32([1, 2]))])
    assert ei.value.name == "PaddingError"


def _grid_cells(golden):
    from helpers import SCALES
    from paper_2406_18820_b200.zoo import make_model

    specs = {f: make_model(f, sc) for f, sc in SCALES.items()}
    for row in golden["grid"]:
        yield row, specs[row["model"]], parse_config_string(row["src"]), parse_config_string(row["tgt"])


@pytest.mark.parametrize("chunk", range(6))
def test_reference_verify_grid(golden, tmp_path, chunk):
    # the reference's own acceptance grid (ucp/verify.py:301-357): 117 identity
    # cells + 21 cross-config cells, seed 11
    cells = list(_grid_cells(golden))
    assert len(cells) == 138
    for k, (row, spec, a, b) in enumerate(cells):
        if k % 6 != chunk:
            continue
        state = O.init_state(spec, 11)
        shards = O.partition_mem(spec, state, a)
        src = str(tmp_path / f"s{k}")
        O.write_tree(spec, a, shards, src)
        assert O.dir_digest(src) == row["src_digest"], (row["model"], row["src"])
        atomic = O.convert_mem(spec, a, shards)
        for p in spec.params:
            for kind in ("weight", "m", "v"):
                assert np.array_equal(atomic[p.name][kind], state[p.name][kind])
        for dt in ("F32", "BF16"):
            assert O.world_digest(O.load_mem(spec, atomic, b, dt)) == row[f"world_{dt}"]


def test_trainer_matches_reference(golden):
    from helpers import SCALES
    from paper_2406_18820_b200.zoo import make_model

    for row in golden["trained"]:
        spec = make_model(row["model"], SCALES[row["model"]])
        kw = row.get("cfg", {})
        kw = {"lr": kw.get("lr", 1e-3), "b1": kw.get("beta1", 0.9), "grad_seed": kw.get("grad_seed", 2024)}
        st = O.train_mem(spec, O.init_state(spec, 7), 0, row["steps"], **kw)
        assert O.state_digest(spec, st, row["steps"]) == row["digest"], row

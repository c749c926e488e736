"""Host logic of the product (no GPU): layout rules, spec/config codecs, the
UCPT container and manifests, pinned against the reference's golden data."""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2406_18820_b200 as U
from helpers import SCALES
from paper_2406_18820_b200 import codec
from paper_2406_18820_b200.layout import all_rank_records
from paper_2406_18820_b200.spec import DType, ParallelConfig, ZeroStage, spec_to_dict

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_make_model_matches_reference(golden):
    for key, d in golden["models"].items():
        if key in SCALES:
            spec = U.make_model(key, SCALES[key])
        elif key == "dense_l0_h16":
            spec = U.make_model("DenseGPT", {"n_layers": 0, "hidden": 16})
        elif key == "dense_l0_h1024":
            spec = U.make_model("DenseGPT", {"n_layers": 0, "hidden": 1024})
        else:
            from helpers import PIPE_SPECS
            fam, sc = PIPE_SPECS[key]
            spec = U.make_model(fam, sc)
        assert spec_to_dict(spec) == d, key
        assert U.spec_from_dict(d) == spec


def test_records_match_reference(golden):
    for key, want in golden["records"].items():
        fam, cstr = key.split("|")
        spec = U.make_model(fam, SCALES[fam])
        cfg = U.parse_config_string(cstr)
        if "error" in want:
            with pytest.raises(U.UcpError) as ei:
                U.validate_model_config(spec, cfg)
            assert type(ei.value).__name__ == want["error"]
            continue
        recs = all_rank_records(spec, cfg)
        allr = [[[r.param, r.kind, r.pattern, list(r.placement), list(r.shape),
                  None if r.segments is None else [list(s) for s in r.segments],
                  None if r.flat_range is None else list(r.flat_range), r.pad_elems]
                 for r in recs[g]] for g in range(cfg.world_size)]
        assert hashlib.sha256(json.dumps(allr).encode()).hexdigest() == want["sha256"], key
        assert sum(len(r) for r in recs) == want["n"]


def test_layout_known_answers():
    assert U.zero_flatten_meta(1024, 3) == (1026, 2, [(0, 342), (342, 684), (684, 1026)])
    seq = U.PPSchedule()
    assert U.pp_layer_map(10, 4, seq) == [[0, 1, 2], [3, 4, 5], [6, 7], [8, 9]]
    assert U.pp_layer_map(8, 2, U.PPSchedule("interleaved", 2)) == [[0, 1, 4, 5], [2, 3, 6, 7]]
    assert U.pp_layer_map(0, 1, seq) == [[0]]
    with pytest.raises(U.IncompatibleConfigError):
        U.pp_layer_map(6, 4, U.PPSchedule("interleaved", 2))
    cfg = ParallelConfig(dp=2, tp=2, pp=2)
    for g in range(8):
        assert cfg.rank_of(*cfg.coords_of(g)) == g


def test_config_strings():
    for s in ("2,1,4,1,z1,seq", "4,2,1,2,z1,seq", "1,1,4,1,z0,int2", "8,1,1,1,z3,seq",
              "4,2,1,2,z2,seq"):
        assert U.format_config_string(U.parse_config_string(s)) == s
    for bad in ("1,1,1,1,z1", "a,1,1,1,z1,seq", "1,1,1,1,z9,seq", "1,1,1,1,z1,foo",
                "1,2,1,1,z3,seq", "3,1,1,2,z1,seq"):
        with pytest.raises(U.IncompatibleConfigError):
            U.parse_config_string(bad)
    assert U.parse_config_string("4,2,1,2,z2,seq").zero_stage is ZeroStage.Z2


def test_z2_alias_lays_out_like_z1():
    spec = U.make_model("GQA", SCALES["GQA"])
    z1 = ParallelConfig(dp=4, tp=2, sp=2, zero_stage=ZeroStage.Z1)
    z2 = ParallelConfig(dp=4, tp=2, sp=2, zero_stage=ZeroStage.Z2)
    assert all_rank_records(spec, z1) == all_rank_records(spec, z2)


def test_llama_totals():
    # equal to the published LLaMA-2 parameter counts
    assert U.llama_spec("7b").total_numel == 6_738_415_616
    assert U.llama_spec("13b").total_numel == 13_015_864_320
    assert U.llama_spec("70b").total_numel == 68_976_648_192
    for name in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        spec, src, tgt, _ = U.bench_config(name)
        U.validate_model_config(spec, src)
        U.validate_model_config(spec, tgt)


def test_ucpt_round_trip(tmp_path):
    rng = np.random.default_rng(1)
    for i in range(300):
        dt = (DType.F32, DType.F16, DType.BF16)[i % 3]
        view = np.uint32 if dt is DType.F32 else np.uint16
        shape = tuple(int(x) for x in rng.integers(1, 7, size=rng.integers(0, 4)))
        bits = rng.integers(0, np.iinfo(view).max, size=shape, dtype=view)
        t = U.Tensor(dt, shape, bits.view(dt.storage).reshape(shape))
        path = str(tmp_path / "rt.ucpt")
        codec.write_tensor(path, t)
        back = codec.read_tensor(path)
        assert back.dtype is dt and back.shape == shape
        assert np.array_equal(back.data.view(view), bits)


def test_golden_vec16_and_shards(golden, tmp_path):
    from oracle import ucp_oracle as O

    t = U.make_tensor(DType.F32, O.gen_values(7, "pos.alibi", "weight", (16,)))
    path = str(tmp_path / "v.ucpt")
    codec.write_tensor(path, t)
    assert open(path, "rb").read() == open(os.path.join(GOLD, "golden_vec16.ucpt"), "rb").read()
    spec = U.make_model("DenseGPT", {"n_layers": 0, "hidden": 16})
    cfg = ParallelConfig()
    mpath = str(tmp_path / "shards.json")
    codec.write_json(mpath, codec.manifest_dict(cfg, 0, U.enumerate_rank_records(spec, cfg, 0)))
    assert hashlib.sha256(open(mpath, "rb").read()).hexdigest() == golden["golden_shards_sha256"]


@pytest.mark.parametrize("blob,err", [
    (b"UCP", U.CorruptHeaderError),
    (b"XXXX\x01\x00\x00\x01" + (4).to_bytes(8, "little") + b"\0" * 16, U.CorruptHeaderError),
    (b"UCPT\x02\x00\x00\x01" + (4).to_bytes(8, "little") + b"\0" * 16, U.CorruptHeaderError),
    (b"UCPT\x01\x00\x09\x01" + (4).to_bytes(8, "little") + b"\0" * 16, U.CorruptHeaderError),
    (b"UCPT\x01\x00\x00\x02" + (4).to_bytes(8, "little"), U.CorruptHeaderError),
    (b"UCPT\x01\x00\x00\x01" + (4).to_bytes(8, "little") + b"\0" * 15, U.TruncatedPayloadError),
    (b"UCPT\x01\x00\x00\x01" + (4).to_bytes(8, "little") + b"\0" * 17, U.TensorFileError),
    (b"UCPT\x01\x00\x00\x01" + (1 << 41).to_bytes(8, "little"), U.CorruptHeaderError),
])
def test_ucpt_errors(tmp_path, blob, err):
    path = str(tmp_path / "bad.ucpt")
    open(path, "wb").write(blob)
    with pytest.raises(err):
        codec.read_tensor(path)
    with pytest.raises(U.TensorIOError):
        codec.read_tensor(str(tmp_path / "missing.ucpt"))


def test_error_tree():
    assert issubclass(U.CorruptHeaderError, U.TensorFileError)
    assert issubclass(U.TensorIOError, U.TensorFileError)
    for cls in (U.ShapeError, U.ManifestError, U.PaddingError, U.ReplicateMismatchError,
                U.MissingFragmentError, U.OverlappingRangeError, U.CheckpointLayoutError,
                U.IncompatibleConfigError, U.PatternCoverageError, U.UnsupportedCastError):
        assert issubclass(cls, U.UcpError)


def test_public_names_are_the_api_functions():
    """Submodule imports must not shadow the drop-in functions of the same
    name (e.g. the `reshard` module vs the `reshard()` entry point)."""
    import inspect

    for name in ("convert", "load", "resume", "union", "extract_fragment", "reshard", "partition",
                 "init_state", "ucp_info", "cast", "load_atomic", "consolidate_world"):
        assert inspect.isfunction(getattr(U, name)), name
    assert inspect.isclass(U.ReshardPlan)


def test_d2d_template_rebind():
    """reshard_device's template patch: virtual source / target addresses
    map to the caller's real ones with offsets kept; real scratch addresses
    and zeros are untouched."""
    import sys

    import numpy as np

    R = sys.modules["paper_2406_18820_b200.reshard"]
    S, T = R._SRC_V, R._TGT_V
    starts = np.array([S, S + 256, S + 1024, T, T + 512], dtype=np.uint64)
    real = np.array([0x7000_0000, 0x7100_0100, 0x7200_0000, 0x7300_0000, 0x7400_0000],
                    dtype=np.uint64)
    v = np.array([S, S + 4, S + 256 + 12, S + 1024 + 1000, T + 8, T + 512 + 4, 0, 0x7f00_0000],
                 dtype=np.uint64)
    got = R._rebind(v, starts, real)
    want = [0x7000_0000, 0x7000_0004, 0x7100_010C, 0x7200_03E8, 0x7300_0008, 0x7400_0004, 0,
            0x7f00_0000]
    assert [int(x) for x in got] == want
    assert [int(x) for x in v][:1] == [S]  # input untouched

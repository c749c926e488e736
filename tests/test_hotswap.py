"""Host-side checks of the hot-swap shim (no GPU): every binding site is
patched and restored, results are rebuilt as the reference's own classes
around the same buffers, and errors map to the reference's classes. The
GPU suite (test_gpu_hotswap.py) runs the reference's verify grids on it."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = [os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"]
REF = next((c for c in CANDIDATES if os.path.isfile(os.path.join(c, "ucp", "__init__.py"))), None)
if REF is None:
    pytest.skip("reference package not present", allow_module_level=True)
sys.dont_write_bytecode = True
if REF not in sys.path:
    sys.path.insert(0, REF)
ucp = pytest.importorskip("ucp")

import paper_2406_18820_b200 as U  # noqa: E402
from paper_2406_18820_b200 import api, hotswap  # noqa: E402
from paper_2406_18820_b200.spec import DType, RecordMeta, Tensor  # noqa: E402


def test_install_patches_every_site_and_restores():
    before = {(sub, n): getattr(ucp if not sub else sys.modules[f"ucp.{sub}"], n)
              for sub, names in hotswap.SITES for n in names
              if hasattr(ucp if not sub else sys.modules.get(f"ucp.{sub}", object()), n)}
    assert len(before) >= 15
    undo = hotswap.install(ucp)
    try:
        for (sub, n), orig in before.items():
            mod = ucp if not sub else sys.modules[f"ucp.{sub}"]
            assert getattr(mod, n) is not orig, (sub, n)
            assert getattr(mod, n).__wrapped__.__module__.startswith("paper_2406_18820_b200")
        # the expected-value and input-generation paths stay the reference's
        assert ucp.parallel.extract_fragment.__module__ == "ucp.parallel"
        assert ucp.consolidate_world.__module__ == "ucp.oracle"
        assert ucp.conversions_invoked() == U.conversions_invoked()
    finally:
        undo()
    for (sub, n), orig in before.items():
        assert getattr(ucp if not sub else sys.modules[f"ucp.{sub}"], n) is orig


def test_world_is_rebuilt_as_reference_objects_without_copies():
    spec = U.make_model("DenseGPT", {"n_layers": 1, "hidden": 16})
    rspec = ucp.make_model("DenseGPT", {"n_layers": 1, "hidden": 16})
    tgt = ucp.ParallelConfig(dp=2)
    recs = ucp.enumerate_rank_records(rspec, tgt, 0)
    shards = {0: []}
    for m in recs:
        ours = RecordMeta(m.param, m.kind, m.pattern, m.placement, m.shape, m.segments,
                          m.flat_range, m.pad_elems)
        dt = DType.BF16 if m.kind == "weight" else DType.F32
        data = np.zeros(m.shape, dtype=dt.storage)
        shards[0].append(api.WorldShard(ours, Tensor(dt, tuple(m.shape), data)))
    stats = api.LoadStats(files_read=3, bytes_read=99, per_rank={0: {"files_read": 3}})
    world = api.LoadedWorld(U.ParallelConfig(dp=2), spec, 5, {"k": 1}, shards, stats)
    got = hotswap._Adapter(ucp).world_out(world, tgt)
    assert type(got) is ucp.LoadedWorld and got.cfg is tgt and got.step == 5
    assert type(got.spec) is ucp.ModelSpec and got.spec == rspec
    assert [s.meta for s in got.shards[0]] == recs
    for a, b in zip(got.shards[0], shards[0]):
        assert type(a) is ucp.WorldShard and type(a.tensor) is ucp.Tensor
        assert a.tensor.dtype is (ucp.DType.BF16 if a.meta.kind == "weight" else ucp.DType.F32)
        assert a.tensor.data is b.tensor.data  # same buffer
    assert type(got.stats) is ucp.LoadStats
    assert got.stats.to_dict() == stats.to_dict()


@pytest.mark.parametrize("name", ["ReplicateMismatchError", "PaddingError", "MissingFragmentError",
                                  "OverlappingRangeError", "ShapeError", "CheckpointLayoutError",
                                  "CorruptHeaderError", "IncompatibleConfigError"])
def test_errors_map_to_reference_classes(name):
    fns = hotswap.adapters(ucp)

    def boom(*a, **k):
        raise getattr(U, name)("x.weight: boom")

    wrapped = hotswap._guard(hotswap._Adapter(ucp), boom)
    with pytest.raises(getattr(ucp, name)) as ei:
        wrapped()
    assert type(ei.value) is getattr(ucp, name) and "x.weight: boom" in str(ei.value)
    assert isinstance(ei.value.__cause__, U.UcpError)
    assert set(fns) >= {"convert", "load", "resume", "union", "extract_fragment", "ucp_info"}


def test_reference_dtype_maps_by_name():
    for d in ucp.DType:
        assert hotswap._Adapter.dtype_in(d) is DType[d.name]


def test_config_identity_holds_across_packages():
    """resume() takes the lazy path iff the layouts match (ucp/load.py:250),
    also when tgt is the reference's ParallelConfig."""
    from paper_2406_18820_b200.layout import same_config

    for s in ("2,2,2,1,z1,seq", "4,1,1,2,z3,seq", "2,1,4,1,z0,int2"):
        r, o = ucp.parse_config_string(s), U.parse_config_string(s)
        assert r != o and same_config(r, o) and same_config(o, r)
    assert not same_config(ucp.parse_config_string("2,2,2,1,z1,seq"),
                           U.parse_config_string("2,2,2,1,z0,seq"))
    assert not same_config(U.ParallelConfig(dp=2), U.ParallelConfig(dp=2, vocab_multiple=128))

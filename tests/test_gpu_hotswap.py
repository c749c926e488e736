"""The reference package running unmodified on top of the B200 path.

``hotswap.install`` patches every binding site of an imported reference
``ucp``; the reference's own verification runner
(``ucp.verify.verify_roundtrip``, ucp/verify.py:154-231) then drives our
convert/load/resume over its stock grids and checks every cell with the
reference oracle (``consolidate_world``) and trainer. The original reference
functions, kept by the test, give the expected trees, worlds and LoadStats.

The reference is taken from ``baseline/_ref`` (the offline pip install of
/root/reference, git-ignored but shipped to the GPU box) or from
/root/reference itself; the module is skipped when neither exists.
"""

import os
import shutil
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = [os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"]
REF = next((c for c in CANDIDATES if os.path.isfile(os.path.join(c, "ucp", "__init__.py"))), None)
if REF is None:
    pytest.skip("reference package not present", allow_module_level=True)

pytestmark = pytest.mark.gpu

sys.dont_write_bytecode = True
if REF not in sys.path:
    sys.path.insert(0, REF)
ucp = pytest.importorskip("ucp")

import paper_2406_18820_b200 as U  # noqa: E402
from paper_2406_18820_b200 import hotswap  # noqa: E402

from oracle.ucp_oracle import dir_digest  # noqa: E402

ORIG = {n: getattr(sys.modules["ucp.convert"], n) for n in ("convert", "union")}
ORIG.update({n: getattr(sys.modules["ucp.load"], n) for n in ("load", "resume")})


@pytest.fixture
def swapped():
    undo = hotswap.install(ucp)
    try:
        yield
    finally:
        undo()


def _bits(world):
    return {g: [(s.meta, s.tensor.dtype.name, s.tensor.shape,
                 np.ascontiguousarray(s.tensor.data).tobytes()) for s in v]
            for g, v in world.shards.items()}


def test_install_patches_every_site_and_restores():
    undo = hotswap.install(ucp)
    try:
        assert ucp.convert is not ORIG["convert"]
        assert sys.modules["ucp.load"].resume is not ORIG["resume"]
        assert ucp.verify.convert.__wrapped__.__module__ == "paper_2406_18820_b200.hotswap"
        assert ucp.parallel.extract_fragment.__module__ == "ucp.parallel"  # left alone
    finally:
        undo()
    assert ucp.convert is ORIG["convert"] and sys.modules["ucp.load"].load is ORIG["load"]


@pytest.mark.parametrize("jobs", [1, 4])
def test_reference_verify_grids_pass_on_b200(swapped, jobs):
    """The reference's stock verification (identity round trips over its
    config grid + cross-config resume with continued training), run by the
    reference's own runner with our functions bound in; jobs=4 runs cells
    in threads, exercising our per-thread staging."""
    c0, r0 = U.conversions_invoked(), sys.modules["ucp.convert"].INVOCATIONS
    grids = ucp.default_grids(quick=(jobs > 1))
    report = ucp.merge_reports([ucp.verify_roundtrip(g, jobs=jobs) for g in grids])
    bad = [(r.cell.label(), r.detail) for r in report.results if not r.ok]
    assert not bad, bad[:5]
    n = len(report.results)
    n_resume = sum(1 for r in report.results if r.cell.resume_steps)
    assert n >= (138 if jobs == 1 else 10)
    # every conversion ran through this package, none through the reference
    assert U.conversions_invoked() - c0 == n + n_resume
    assert sys.modules["ucp.convert"].INVOCATIONS == r0


@pytest.mark.parametrize("fam,scale,src,tgt", [
    ("GQA", {"n_layers": 4, "hidden": 64, "q_heads": 8, "kv_heads": 2}, "2,2,2,1,z1,seq", "2,4,1,1,z1,seq"),
    ("MoE", {"n_layers": 4, "hidden": 64, "n_experts": 4}, "3,1,1,1,z3,seq", "2,2,2,1,z1,seq"),
    ("DenseGPT", {"n_layers": 2, "hidden": 32}, "3,1,1,1,z3,seq", "3,2,1,1,z1,seq"),
])
def test_swapped_equals_reference_functions(tmp_path, fam, scale, src, tgt):
    """Trees, worlds (f32/bf16/f16, bypass on/off), resume and LoadStats from
    the swapped functions equal the unswapped reference's, compared as
    reference objects (RecordMeta dataclass equality, DType identity)."""
    spec = ucp.make_model(fam, scale)
    s, t = ucp.parse_config_string(src), ucp.parse_config_string(tgt)
    ucp.partition(ucp.train_steps(ucp.init_state(spec, 7), ucp.TrainerConfig(), 0, 2), s,
                  str(tmp_path / "src"))
    cases = [(dt, bypass) for dt in (ucp.DType.F32, ucp.DType.BF16, ucp.DType.F16)
             for bypass in (True, False)]

    def run(tag):
        out = {"atomic": ucp.convert(str(tmp_path / "src"), str(tmp_path / tag))}
        for dt, bypass in cases:
            out[dt, bypass] = ucp.load(str(tmp_path / tag), t, dt, bypass)
        out["resume"] = ucp.resume(str(tmp_path / "src"), t, str(tmp_path / f"scr_{tag}"))
        out["lazy"] = ucp.resume(str(tmp_path / "src"), s, str(tmp_path / f"lazy_{tag}"))
        return out

    want = run("ref")
    undo = hotswap.install(ucp)
    try:
        got = run("ours")
    finally:
        undo()
    assert dir_digest(str(tmp_path / "ours")) == dir_digest(str(tmp_path / "ref"))
    assert dir_digest(str(tmp_path / "scr_ours" / "atomic")) == dir_digest(str(tmp_path / "scr_ref" / "atomic"))
    assert type(got["atomic"]) is type(want["atomic"])
    assert got["atomic"].spec == want["atomic"].spec and got["atomic"].step == want["atomic"].step
    assert got["atomic"].source_fingerprint == want["atomic"].source_fingerprint
    for key in cases + ["resume", "lazy"]:
        g, w = got[key], want[key]
        assert type(g) is type(w) and g.cfg == w.cfg and g.step == w.step and g.spec == w.spec
        assert g.stats.to_dict() == w.stats.to_dict(), key
        assert _bits(g) == _bits(w), key
    for dt, bypass in cases:
        for g, v in got[dt, bypass].shards.items():
            assert [sh.meta for sh in v] == ucp.enumerate_rank_records(spec, t, g)
            assert all(sh.tensor.dtype is dt for sh in v if sh.meta.kind == "weight")
    f32 = got[ucp.DType.F32, True]
    assert ucp.states_equal(ucp.consolidate_world(f32), ucp.consolidate_oracle(str(tmp_path / "src")))


def test_swapped_errors_are_reference_classes(tmp_path, swapped):
    """A corrupted replica raises the reference's ReplicateMismatchError and
    leaves the atomic tree torn (ucp/convert.py:503-504)."""
    spec = ucp.make_model("DenseGPT", {"n_layers": 2, "hidden": 32})
    cfg = ucp.parse_config_string("2,2,1,1,z0,seq")
    src = str(tmp_path / "src")
    ucp.partition(ucp.init_state(spec, 7), cfg, src)
    victim = os.path.join(src, "rank_1", "layers.0.ln_w.weight.ucpt")  # dp1 of tp0
    with open(victim, "r+b") as f:
        f.seek(-4, 2)
        f.write(np.float32(123.0).tobytes())
    with pytest.raises(ucp.ReplicateMismatchError):
        ucp.convert(src, str(tmp_path / "out"))
    assert not os.path.exists(tmp_path / "out" / "ucp_meta.json")
    for fn in (ucp.load, ORIG["load"]):
        with pytest.raises(ucp.UcpError) as ei:
            fn(str(tmp_path / "nothing"), ucp.ParallelConfig(dp=2))
        assert type(ei.value) is ucp.CheckpointLayoutError
    shutil.rmtree(tmp_path / "out", ignore_errors=True)


def test_swapped_union_matches_reference_union(swapped):
    """ucp.union on the reference's FragmentMsgs (its own test fixtures'
    shape: pkg/tests/test_convert.py:61-205) against the original."""
    spec = ucp.make_model("GQA", {"n_layers": 2, "hidden": 64, "q_heads": 8, "kv_heads": 2})
    cfg = ucp.ParallelConfig(dp=2, tp=2, pp=1, zero_stage=ucp.ZeroStage.Z1)
    state = ucp.init_state(spec, 7)
    FragmentMsg = sys.modules["ucp.convert"].FragmentMsg
    for p in spec.params:
        for kind in ("weight", "m", "v"):
            msgs = []
            for g in range(cfg.world_size):
                for m in ucp.enumerate_rank_records(spec, cfg, g):
                    if m.param == p.name and m.kind == kind:
                        full = getattr(state.params[p.name], kind).data
                        msgs.append(FragmentMsg(m, ucp.parallel.extract_fragment(p, cfg, m, full)))
            got, want = ucp.union(p, cfg, msgs), ORIG["union"](p, cfg, msgs)
            assert got.dtype == want.dtype and got.shape == want.shape
            assert got.tobytes() == want.tobytes(), (p.name, kind)

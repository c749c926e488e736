"""Duck-typing of the reference's own objects (ParamSpec / ParallelConfig /
RecordMeta from /root/reference) through the descriptor compiler, as the
hot-swap shim in INTEGRATION.md relies on. Runs only where the reference is
importable (baseline/_ref or /root/reference); skipped elsewhere."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = [os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"]
REF = next((c for c in CANDIDATES if os.path.isfile(os.path.join(c, "ucp", "__init__.py"))), None)
if REF is None:
    pytest.skip("reference package not present", allow_module_level=True)
if REF not in sys.path:
    sys.path.insert(0, REF)
sys.dont_write_bytecode = True
ucp = pytest.importorskip("ucp")

from descr_interp import execute  # noqa: E402
from paper_2406_18820_b200.engine import align_up  # noqa: E402
from paper_2406_18820_b200.plan import RunTable, compile_extract, compile_union  # noqa: E402
from paper_2406_18820_b200.spec import DType  # noqa: E402


@pytest.mark.parametrize("fam,scale", [("GQA", {"n_layers": 4, "hidden": 64, "q_heads": 8, "kv_heads": 2}),
                                       ("MoE", {"n_layers": 4, "hidden": 64, "n_experts": 4})])
def test_reference_types_drive_the_compiler(fam, scale):
    spec = ucp.make_model(fam, scale)
    src = ucp.ParallelConfig(dp=2, tp=2, pp=2, zero_stage=ucp.ZeroStage.Z1)
    tgt = ucp.ParallelConfig(dp=3, tp=2, zero_stage=ucp.ZeroStage.Z1)
    state = ucp.init_state(spec, 7)
    # union over the reference's own records and fragments
    frags, blobs, at = {}, [], 0
    for g in range(src.world_size):
        for m in ucp.enumerate_rank_records(spec, src, g):
            p = spec.param(m.param)
            a = ucp.parallel.extract_fragment(p, src, m, getattr(state.params[m.param], m.kind).data)
            frags.setdefault((m.param, m.kind), []).append((m, at, a.size))
            blobs.append((at, np.ascontiguousarray(a, dtype=np.float32)))
            at += align_up(a.nbytes)
    buf = np.zeros(at, dtype=np.uint8)
    for o, a in blobs:
        buf[o:o + a.nbytes] = a.view(np.uint8).reshape(-1)
    tab, outs, dat = RunTable(), [], 0
    for p in spec.params:
        for k in ("weight", "m", "v"):
            compile_union(tab, p, src, frags[(p.name, k)], dat, True)
            outs.append((p, k, dat))
            dat += align_up(4 * p.numel)
    runs, aux, tiles = tab.finish(8192)
    dst = np.zeros(dat, dtype=np.uint8)
    assert execute(runs, aux, tiles, buf, dst) == []
    for p, k, o in outs:
        got = dst[o:o + 4 * p.numel].view(np.float32).reshape(p.shape)
        assert np.array_equal(got, getattr(state.params[p.name], k).data), (p.name, k)
    # extract for the reference's target records, bf16 weights
    p = spec.param("layers.1.attn_qkv")
    full = state.params[p.name].weight.data
    src_buf = np.ascontiguousarray(full, dtype=np.float32).view(np.uint8).reshape(-1).copy()
    for g in range(tgt.world_size):
        m = next(r for r in ucp.enumerate_rank_records(spec, tgt, g)
                 if r.param == p.name and r.kind == "weight")
        want = ucp.cast(ucp.make_tensor(ucp.DType.F32, ucp.parallel.extract_fragment(p, tgt, m, full)),
                        ucp.DType.BF16).data
        t = RunTable()
        compile_extract(t, p, tgt, [(m, 0)], 0, DType.BF16)
        r, a, ti = t.finish(4096)
        out = np.zeros(want.nbytes, dtype=np.uint8)
        assert execute(r, a, ti, src_buf, out) == []
        assert np.array_equal(out.view(np.uint16).reshape(want.shape), want)

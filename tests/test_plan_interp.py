"""Descriptor compiler + tiler == oracle, executed by the numpy interpreter.

CPU-only proof that the run tables the GPU executes encode the reference's
union / extract_fragment / cast semantics for every golden cell, with tiny
tiles so column-split, row-block, head/tail and misaligned paths all occur.
"""

import numpy as np
import pytest

import paper_2406_18820_b200 as U
from descr_interp import execute
from helpers import cell_cfgs, cell_spec
from oracle import ucp_oracle as O
from paper_2406_18820_b200.engine import align_up
from paper_2406_18820_b200.layout import all_rank_records
from paper_2406_18820_b200.plan import (
    RunTable,
    compile_extract,
    compile_union,
    fragment_elems,
    expand_tiles,
    make_tiles,
    split_rows,
)
from paper_2406_18820_b200.spec import STATE_KINDS, DType, ParallelConfig, ParamKind, ParamSpec, RecordMeta, ZeroStage

CELLS = ["pad", "gqa", "moe"] + [f"{f}.{i}" for f in ("DenseGPT", "MoE", "GQA") for i in range(6)]


def _arena_union(spec, cfg, shards, strict=True, tile_bytes=4096):
    """Product union of every (param, kind) through the interpreter."""
    recs = all_rank_records(spec, cfg)
    frags, blobs, at = {}, [], 0
    for g in range(cfg.world_size):
        assert len(recs[g]) == len(shards[g])
        for meta, (orec, arr) in zip(recs[g], shards[g]):
            assert O.record_tuple(meta) == O.record_tuple(orec)
            frags.setdefault((meta.param, meta.kind), []).append((meta, at, arr.size))
            blobs.append((at, arr))
            at += align_up(arr.nbytes)
    src = np.zeros(max(at, 16), dtype=np.uint8)
    for o, a in blobs:
        src[o:o + a.nbytes] = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
    tab, outs, dat = RunTable(), [], 0
    for p in spec.params:
        for k in STATE_KINDS:
            compile_union(tab, p, cfg, frags[(p.name, k)], dat, strict)
            outs.append((p, k, dat))
            dat += align_up(4 * p.numel)
    runs, aux, tiles = tab.finish(tile_bytes)
    dst = np.full(max(dat, 16), 0xAB, dtype=np.uint8)
    fails = execute(runs, aux, tiles, src, dst)
    return {(p.name, k): dst[o:o + 4 * p.numel].view(np.float32).reshape(p.shape)
            for p, k, o in outs}, fails, tab


def _arena_extract(spec, cfg, atomic, dtype, tile_bytes=4096):
    src_blobs, at, soff = [], 0, {}
    for p in spec.params:
        for k in STATE_KINDS:
            soff[(p.name, k)] = at
            src_blobs.append((at, atomic[p.name][k]))
            at += align_up(4 * p.numel)
    src = np.zeros(max(at, 16), dtype=np.uint8)
    for o, a in src_blobs:
        src[o:o + a.nbytes] = a.view(np.uint8).reshape(-1)
    recs = all_rank_records(spec, cfg)
    by_unit, outs, tat = {}, [], 0
    for g in range(cfg.world_size):
        for m in recs[g]:
            p = spec.param(m.param)
            odt = dtype if m.kind == "weight" else DType.F32
            n = fragment_elems(p, cfg, m)
            by_unit.setdefault((m.param, m.kind), []).append((m, tat))
            outs.append((g, m, tat, n, odt))
            tat += align_up(n * odt.itemsize)
    tab = RunTable()
    for p in spec.params:
        for k in STATE_KINDS:
            odt = dtype if k == "weight" else DType.F32
            compile_extract(tab, p, cfg, by_unit.get((p.name, k), []), soff[(p.name, k)], odt)
    runs, aux, tiles = tab.finish(tile_bytes)
    dst = np.full(max(tat, 16), 0xCD, dtype=np.uint8)
    assert execute(runs, aux, tiles, src, dst) == []
    world = {}
    for g, m, o, n, odt in outs:
        world.setdefault(g, []).append((m, dst[o:o + n * odt.itemsize].view(odt.storage).copy()))
    return world, tab


@pytest.mark.parametrize("name", CELLS)
def test_union_matches_oracle(golden, name):
    row = next(r for r in golden["pipelines"] if r["name"] == name)
    spec = cell_spec(golden, row)
    src_cfg, _ = cell_cfgs(row)
    shards = O.partition_mem(spec, O.init_state(spec, 7), src_cfg)
    want = O.convert_mem(spec, src_cfg, shards)
    got, fails, _ = _arena_union(spec, src_cfg, shards)
    assert fails == []
    for p in spec.params:
        for k in STATE_KINDS:
            assert np.array_equal(got[(p.name, k)].view(np.uint32),
                                  want[p.name][k].view(np.uint32)), (p.name, k)


@pytest.mark.parametrize("name", CELLS)
@pytest.mark.parametrize("dtype", ["F32", "BF16", "F16"])
def test_extract_matches_golden_world(golden, name, dtype):
    row = next(r for r in golden["pipelines"] if r["name"] == name)
    spec = cell_spec(golden, row)
    _, tgt_cfg = cell_cfgs(row)
    atomic = O.init_state(spec, 7)
    world, _ = _arena_extract(spec, tgt_cfg, atomic, DType[dtype])
    # rebuild the digest in canonical order with shapes from the records
    fixed = {}
    for g, items in world.items():
        fixed[g] = []
        for m, a in items:
            p = spec.param(m.param)
            shape = U.plan.fragment_shape(p, tgt_cfg, m)
            fixed[g].append((m, a.reshape(shape)))
    assert O.world_digest(fixed) == row[f"world_{dtype}"]


def test_union_reports_bad_replica_and_pad():
    spec = U.make_model("DenseGPT", {"n_layers": 2, "hidden": 32})
    cfg = ParallelConfig(dp=3, tp=1, zero_stage=ZeroStage.Z1)
    shards = O.partition_mem(spec, O.init_state(spec, 7), cfg)
    # corrupt a weight replica on dp 2 and a pad element on the last dp rank
    for i, (r, a) in enumerate(shards[2]):
        if r["param"] == "layers.1.ln_w" and r["kind"] == "weight":
            a = a.copy()
            a[3] = np.float32(9.0)
            shards[2][i] = (r, a)
    _, fails, tab = _arena_union(spec, cfg, shards)
    assert fails and tab.units[int(tab.finish()[0][fails[0][0]]["tag"])].param == "layers.1.ln_w"


def _meta(p, kind="weight", pattern="replicate", placement=(0, 0, 0), shape=None,
          segments=None, flat_range=None, pad_elems=0):
    return RecordMeta(p.name, kind, pattern, placement, shape if shape is not None else p.shape,
                      segments, flat_range, pad_elems)


@pytest.mark.parametrize("case,err", [
    ("empty", U.MissingFragmentError),
    ("missing_tp", U.MissingFragmentError),
    ("overlap", U.OverlappingRangeError),
    ("gap", U.MissingFragmentError),
    ("dup_dp", U.OverlappingRangeError),
    ("mixed_flat", U.ManifestError),
    ("mixed_kind", U.ManifestError),
    ("tags", U.ManifestError),
    ("stages", U.ManifestError),
    ("pad_nonfinal", U.PaddingError),
    ("pad_arith", U.PaddingError),
    ("nc_segs", U.ManifestError),
    ("missing_dp", U.MissingFragmentError),
])
def test_union_metadata_errors(case, err):
    # mirrors pkg/tests/test_convert.py:143-205 plus the remaining branches of
    # ucp/convert.py:137-193, :232-262
    ln4 = ParamSpec("ln", (4,), 0, ParamKind.LAYERNORM_WEIGHT)
    ln6 = ParamSpec("ln", (6,), 0, ParamKind.LAYERNORM_WEIGHT)
    w = ParamSpec("w", (4, 2), 0, ParamKind.MATMUL2D, 0)
    z3 = lambda dp: ParallelConfig(dp=dp, zero_stage=ZeroStage.Z3)
    qkv = ParamSpec("qkv", (6, 2), 0, ParamKind.FUSED_QKV, 0, ((0, 4), (4, 2)))
    cases = {
        "empty": (w, ParallelConfig(), []),
        "missing_tp": (w, ParallelConfig(tp=2), [(_meta(w, pattern="shard_v", shape=(2, 2)), 0, 4)]),
        "overlap": (ln4, z3(2), [(_meta(ln4, pattern="shard_v", shape=(2,), flat_range=(0, 2)), 0, 2),
                                 (_meta(ln4, pattern="shard_v", placement=(0, 0, 1), shape=(2,),
                                        flat_range=(1, 3)), 256, 2)]),
        "gap": (ln6, z3(3), [(_meta(ln6, pattern="shard_v", shape=(2,), flat_range=(0, 2)), 0, 2),
                             (_meta(ln6, pattern="shard_v", placement=(0, 0, 2), shape=(2,),
                                    flat_range=(4, 6)), 256, 2),
                             (_meta(ln6, pattern="shard_v", placement=(0, 0, 1), shape=(2,),
                                    flat_range=(4, 6)), 512, 2)]),
        "dup_dp": (ln4, ParallelConfig(dp=2), [(_meta(ln4), 0, 4), (_meta(ln4), 256, 4),
                                               (_meta(ln4, placement=(0, 0, 1)), 512, 4)]),
        "mixed_flat": (ln4, z3(2), [(_meta(ln4, pattern="shard_v", shape=(2,), flat_range=(0, 2)), 0, 2),
                                    (_meta(ln4, pattern="shard_v", placement=(0, 0, 1)), 256, 4)]),
        "mixed_kind": (ln4, ParallelConfig(), [(_meta(ln4), 0, 4), (_meta(ln4, kind="m"), 256, 4)]),
        "tags": (ln4, ParallelConfig(dp=2), [(_meta(ln4), 0, 4),
                                             (_meta(ln4, pattern="unique", placement=(0, 0, 1)), 256, 4)]),
        "stages": (ln4, ParallelConfig(dp=2), [(_meta(ln4), 0, 4), (_meta(ln4, placement=(1, 0, 1)), 256, 4)]),
        "pad_nonfinal": (ln6, z3(2), [(_meta(ln6, pattern="shard_v", shape=(3,), flat_range=(0, 3),
                                             pad_elems=1), 0, 3),
                                      (_meta(ln6, pattern="shard_v", placement=(0, 0, 1), shape=(3,),
                                             flat_range=(3, 6)), 256, 3)]),
        "pad_arith": (ln4, z3(2), [(_meta(ln4, pattern="shard_v", shape=(2,), flat_range=(0, 2)), 0, 2),
                                   (_meta(ln4, pattern="shard_v", placement=(0, 0, 1), shape=(2,),
                                          flat_range=(2, 4), pad_elems=1), 256, 2)]),
        "nc_segs": (qkv, ParallelConfig(tp=2), [
            (_meta(qkv, pattern="shard_nc", placement=(0, t, 0), shape=(3, 2), segments=((0, 6),)),
             256 * t, 6) for t in range(2)]),
        "missing_dp": (ln4, ParallelConfig(dp=2), [(_meta(ln4), 0, 4)]),
    }
    p, cfg, frags = cases[case]
    with pytest.raises(err):
        compile_union(RunTable(), p, cfg, frags, 0, True)


def test_split_rows_covers_interval():
    corr = (10, 1000, 64, 7, 5)  # frag [10, 45) -> 7 rows of 5 at pitch 64
    for a in range(10, 45):
        for b in range(a + 1, 46):
            pieces = split_rows(corr, a, b)
            covered = []
            for fs, xs, xp, rows, cols in pieces:
                for i in range(rows):
                    for j in range(cols):
                        f = fs + i * cols + j
                        r, c = divmod(f - 10, 5)
                        assert xs + i * xp + j == 1000 + r * 64 + c
                        covered.append(f)
            assert covered == list(range(a, min(b, 45)))


def test_tiles_cover_every_element_once():
    from paper_2406_18820_b200.plan import RUN_ROWSPLIT

    tab = RunTable()
    tab.unit("x", "weight")
    tab.add(srcs=[0], dsts=[0], src_pitch=3000, dst_pitch=3000, rows=5, cols=3000, tag=0)
    tab.add(srcs=[4], dsts=[8], src_pitch=7, dst_pitch=9, rows=1000, cols=7, tag=0)
    tab.add(srcs=[12], dsts=[12, 4096], src_pitch=10 ** 6, dst_pitch=10 ** 6, rows=1,
            cols=10 ** 6, tag=0)
    base, _, _ = tab.finish()
    for tb in (2048, 1 << 15, 1 << 17, 1 << 24):
        runs = base.copy()
        tiles = make_tiles(runs, tb)
        for i, r in enumerate(runs):
            cover = np.zeros((int(r["rows"]), int(r["cols"])), dtype=np.int32)
            for t in tiles[tiles["run"] == i]:
                if r["flags"] & RUN_ROWSPLIT:
                    cover[t["row0"], t["col0"]:t["col0"] + t["count"]] += 1
                else:
                    assert t["col0"] == 0
                    cover[t["row0"]:t["row0"] + t["count"], :] += 1
            assert (cover == 1).all(), (tb, i)


def test_finish_classed_partitions_tiles():
    from paper_2406_18820_b200.plan import CLASS_GENERAL, CLASS_OPS, NCLASS, run_classes

    spec = U.make_model("DenseGPT", {"n_layers": 2, "hidden": 32})
    cfg = ParallelConfig(dp=3, tp=2, zero_stage=ZeroStage.Z1)
    atomic = O.init_state(spec, 7)
    _, tab = _arena_extract(spec, cfg, atomic, DType.BF16)
    runs, aux, rt, info, order = tab.finish_classed(4096)
    assert sorted(order) == list(range(len(runs)))
    assert len(info) == 2 * NCLASS
    assert info[:NCLASS].sum() == rt["ntiles"].sum() and info[NCLASS:].sum() == len(runs)
    cls = run_classes(runs)
    assert (np.diff(cls) >= 0).all()  # runs sorted by kernel class
    assert info[CLASS_GENERAL] > 0  # misaligned dp=3 pieces
    assert info[CLASS_OPS] > 0  # partial noise + ZeRO re-pads
    # the interpreter over the classed table reproduces the table-order result
    assert len(expand_tiles(runs, rt)) == info[:NCLASS].sum()


def _find_run(first, lo, hi, b):
    """Python mirror of find_run() in csrc/ucp_b200.cu (32-ary warp search)."""
    while hi - lo > 1:
        step = (hi - lo + 31) // 32
        le = [lo + i * step < hi and first[lo + i * step] <= b for i in range(32)]
        assert le == sorted(le, reverse=True)  # the ballot is a prefix of the lanes
        last = max(i for i in range(32) if le[i])
        lo += last * step
        hi = min(hi, lo + step)
    return lo


@pytest.mark.parametrize("tb", [512, 4096, 1 << 17])
def test_device_tile_derivation_matches_expansion(tb):
    """Per class, CTA b finds its run by the warp search over the
    class-relative `first` (what ucp_runtile_scan writes) and derives the
    same rectangle expand_tiles lists -- including zero-tile runs."""
    from paper_2406_18820_b200.plan import NCLASS, RUN_ROWSPLIT, classed, run_classes

    spec = U.make_model("GQA", {"n_layers": 2, "hidden": 64, "q_heads": 8, "kv_heads": 2})
    cfg = ParallelConfig(dp=3, tp=2, zero_stage=ZeroStage.Z1)
    _, tab = _arena_extract(spec, cfg, O.init_state(spec, 7), DType.BF16)
    runs0, aux = tab._runs_aux()
    empty = runs0[:1].copy()
    empty["rows"] = 0  # a zero-tile run in the middle of a class
    runs0 = np.concatenate([runs0[:3], empty, runs0[3:]])
    runs, aux, rt, info, _ = classed(runs0, aux, run_classes(runs0), tb)
    want = expand_tiles(runs, rt)
    got, r0 = [], 0
    for c in range(NCLASS):
        nr, nt = int(info[NCLASS + c]), int(info[c])
        first = rt["first"][r0:r0 + nr].astype(np.int64)
        assert nr == 0 or first[0] == 0
        for b in range(nt):
            run = r0 + _find_run(list(first), 0, nr, b)
            k = b - int(rt["first"][run])
            per, tpr, r = int(rt["per"][run]), int(rt["tpr"][run]), runs[run]
            assert 0 <= k < int(rt["ntiles"][run])
            if r["flags"] & RUN_ROWSPLIT:
                row0 = k // tpr
                col0 = (k - row0 * tpr) * per
                cnt = min(per, int(r["cols"]) - col0)
            else:
                row0, col0 = k * per, 0
                cnt = min(per, int(r["rows"]) - row0)
            got.append((run, row0, col0, cnt))
        r0 += nr
    assert got == [tuple(int(x) for x in t) for t in want]


def _fused_world(spec, src_cfg, tgt_cfg, shards, dtype, tile_bytes=4096, materialize=True,
                 fails=None):
    """Fused tables of every unit through the interpreter. ``fails``: a
    list collecting (table, run, elem) failures instead of asserting none."""
    from descr_interp import execute_fused
    from paper_2406_18820_b200.plan import XRunTable, compile_fused

    srecs, trecs = all_rank_records(spec, src_cfg), all_rank_records(spec, tgt_cfg)
    frags, blobs, at = {}, [], 0
    for g in range(src_cfg.world_size):
        for meta, (_, arr) in zip(srecs[g], shards[g]):
            frags.setdefault((meta.param, meta.kind), []).append((meta, at, arr.size))
            blobs.append((at, arr))
            at += align_up(arr.nbytes)
    src = np.zeros(max(at, 16), dtype=np.uint8)
    for o, a in blobs:
        src[o:o + a.nbytes] = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
    by_unit, outs, tat = {}, [], 0
    for g in range(tgt_cfg.world_size):
        for m in trecs[g]:
            p = spec.param(m.param)
            odt = dtype if m.kind == "weight" else DType.F32
            n = fragment_elems(p, tgt_cfg, m)
            by_unit.setdefault((m.param, m.kind), []).append((m, tat))
            outs.append((g, m, tat, n, odt))
            tat += align_up(n * odt.itemsize)
    fx, rc, rl = XRunTable(), RunTable(), RunTable()
    aoff, aat, fused = {}, 0, 0
    for p in spec.params:
        for k in STATE_KINDS:
            aoff[(p.name, k)] = aat
            odt = dtype if k == "weight" else DType.F32
            fused += compile_fused(fx, rc, rl, p, src_cfg, frags[(p.name, k)], aat, tgt_cfg,
                                   by_unit.get((p.name, k), []), odt, True, materialize)
            aat += align_up(4 * p.numel)
    atom = np.zeros(max(aat, 16), dtype=np.uint8)
    dst = np.full(max(tat, 16), 0xCD, dtype=np.uint8)
    xr, xa, xrt, _, _ = fx.finish_classed(tile_bytes)
    got = [("fused",) + f for f in execute_fused(xr, xa, expand_tiles(xr, xrt), src, atom, dst)]
    r1, a1, t1 = rc.finish(tile_bytes)
    got += [("conv",) + f for f in execute(r1, a1, t1, src, atom)]
    r2, a2, t2 = rl.finish(tile_bytes)
    got += [("load",) + f for f in execute(r2, a2, t2, atom, dst)]
    if fails is None:
        assert got == []
    else:
        fails.extend(got)
    world = {}
    for g, m, o, n, odt in outs:
        shape = U.plan.fragment_shape(spec.param(m.param), tgt_cfg, m)
        world.setdefault(g, []).append((m, dst[o:o + n * odt.itemsize].view(odt.storage).reshape(shape)))
    atomics = {k: atom[o:o + 4 * spec.param(k[0]).numel].view(np.float32) for k, o in aoff.items()}
    return world, atomics, fused, fx


@pytest.mark.parametrize("name", CELLS)
@pytest.mark.parametrize("dtype", ["F32", "BF16"])
def test_fused_matches_golden(golden, name, dtype):
    row = next(r for r in golden["pipelines"] if r["name"] == name)
    spec = cell_spec(golden, row)
    src_cfg, tgt_cfg = cell_cfgs(row)
    state = O.init_state(spec, 7)
    shards = O.partition_mem(spec, state, src_cfg)
    world, atomics, fused, _ = _fused_world(spec, src_cfg, tgt_cfg, shards, DType[dtype])
    assert O.world_digest(world) == row[f"world_{dtype}"]
    for (pname, k), a in atomics.items():
        assert np.array_equal(a.view(np.uint32), state[pname][k].reshape(-1).view(np.uint32))
    assert fused > 0


def test_fused_covers_llama_units():
    # every LLaMA unit fuses (no Partial params, all pieces 16-B phase aligned)
    spec = U.llama_spec("7b", n_layers=1)
    _, src, tgt, _ = U.bench_config("cfg2", n_layers=1)
    from paper_2406_18820_b200.plan import XRunTable, compile_fused

    srecs, trecs = all_rank_records(spec, src), all_rank_records(spec, tgt)
    n_f = 0
    for p in spec.params:
        for k in STATE_KINDS:
            frags = [(m, 1 << 40, fragment_elems(p, src, m)) for g in range(src.world_size)
                     for m in srecs[g] if (m.param, m.kind) == (p.name, k)]
            tg = [(m, 1 << 41) for g in range(tgt.world_size) for m in trecs[g]
                  if (m.param, m.kind) == (p.name, k)]
            n_f += compile_fused(XRunTable(), RunTable(), RunTable(), p, src, frags, 0, tgt, tg)
    assert n_f == 3 * len(spec.params)


def test_shard_hy_grid_union():
    # _union_hy (ucp/convert.py:196-218): blocks placed at (0, row, col)
    p = ParamSpec("g", (8, 6), 0, ParamKind.MATMUL2D, 0)
    full = np.arange(48, dtype=np.float32).reshape(8, 6)
    blocks = O.hy_blocks(full, 2, 3)
    src = np.zeros(48 * 4 + 256 * 6, dtype=np.uint8)
    frags = []
    for i, ((r, c), blk) in enumerate(blocks[::-1]):
        o = 256 * i
        src[o:o + blk.nbytes] = blk.view(np.uint8).reshape(-1)
        frags.append((RecordMeta(p.name, "weight", "shard_hy", (0, r, c), blk.shape), o, blk.size))
    tab = RunTable()
    compile_union(tab, p, ParallelConfig(), frags, 0, True)
    runs, aux, tiles = tab.finish(64)
    dst = np.zeros(48 * 4, dtype=np.uint8)
    assert execute(runs, aux, tiles, src, dst) == []
    assert np.array_equal(dst.view(np.float32).reshape(8, 6), full)
    assert np.array_equal(O.union(p, ParallelConfig(), [(f[0], blk) for f, (_, blk) in
                                                        zip(frags, blocks[::-1])]), full)
    with pytest.raises(U.OverlappingRangeError):
        compile_union(RunTable(), p, ParallelConfig(), frags + frags[:1], 0, True)
    with pytest.raises(U.MissingFragmentError):
        compile_union(RunTable(), p, ParallelConfig(), frags[1:], 0, True)


def test_fused_remainder_keeps_unit_provenance():
    # units that cannot fuse (Partial mean/noise) are re-homed into the
    # unfused tables; their runs must keep pointing at the right (param, kind)
    from paper_2406_18820_b200.plan import XRunTable, compile_fused

    spec = U.make_model("DenseGPT", {"n_layers": 2, "hidden": 32})
    src_cfg, tgt_cfg = ParallelConfig(dp=3, tp=2, zero_stage=ZeroStage.Z1), ParallelConfig(tp=4)
    srecs, trecs = all_rank_records(spec, src_cfg), all_rank_records(spec, tgt_cfg)
    fx, rc, rl = XRunTable(), RunTable(), RunTable()
    aoff, at = {}, 0
    for p in spec.params:
        for k in STATE_KINDS:
            aoff[(p.name, k)] = (at, at + 4 * p.numel)
            frags = [(m, 1 << 40, fragment_elems(p, src_cfg, m)) for g in range(src_cfg.world_size)
                     for m in srecs[g] if (m.param, m.kind) == (p.name, k)]
            tg = [(m, 1 << 41) for g in range(tgt_cfg.world_size) for m in trecs[g]
                  if (m.param, m.kind) == (p.name, k)]
            compile_fused(fx, rc, rl, p, src_cfg, frags, at, tgt_cfg, tg)
            at += align_up(4 * p.numel)
    assert len(rc) and len(rl)
    for table, field in ((rc, 1), (rl, 0)):
        for row in table._rows:
            if row[10] in (3, 4):  # ZERO / CHECKZERO do not touch the atomic
                continue
            unit = table.units[row[14]]
            lo, hi = aoff[(unit.param, unit.kind)]
            assert lo <= row[field] < hi, (unit.param, unit.kind)


def _ln_spec():
    return U.make_model("DenseGPT", {"n_layers": 1, "hidden": 32})


@pytest.mark.parametrize("bad_dp", [None, 3, 70, 79])
def test_fused_checks_every_replica_beyond_64(bad_dp):
    # dp = 80 Z0: every weight has 80 replicas, more than one run holds
    # (MAX_SRC); the verify-only continuation runs must still run when the
    # unit fuses, so a flipped late replica is reported like the reference
    # does (ucp/convert.py:163-172)
    spec = _ln_spec()
    src_cfg = ParallelConfig(dp=80, zero_stage=ZeroStage.Z0)
    tgt_cfg = ParallelConfig(dp=2, zero_stage=ZeroStage.Z1)
    state = O.init_state(spec, 7)
    shards = O.partition_mem(spec, state, src_cfg)
    target = "layers.0.ln_w"
    if bad_dp is not None:
        recs = all_rank_records(spec, src_cfg)
        g = next(g for g in range(src_cfg.world_size) if recs[g][0].placement[2] == bad_dp)
        i = next(i for i, m in enumerate(recs[g]) if (m.param, m.kind) == (target, "weight"))
        m, a = shards[g][i]
        a = a.copy()
        a.reshape(-1).view(np.uint32)[5] ^= 1
        shards[g][i] = (m, a)
    fails = []
    world, _, fused, _ = _fused_world(spec, src_cfg, tgt_cfg, shards, DType.F32, fails=fails)
    assert fused > 0
    if bad_dp is None:
        assert fails == []
        want = O.load_mem(spec, O.convert_mem(spec, src_cfg, shards), tgt_cfg, "F32")
        assert O.world_digest(world) == O.world_digest(want)
    else:
        assert fails, "a corrupted replica beyond the first run went unchecked"
        assert all(f[2] == 5 for f in fails)


@pytest.mark.parametrize("bad", [False, True])
def test_partial_mean_with_more_replicas_than_one_run(bad):
    # tp = 8, dp = 40 Z0: 320 sources for the averaged pos.alibi vector, more
    # than one averaged run can carry; the dp replicas are verified by
    # verify-only runs and the f64 mean reads one replica per tp rank
    spec = _ln_spec()
    src_cfg = ParallelConfig(dp=40, tp=8, zero_stage=ZeroStage.Z0)
    state = O.init_state(spec, 7)
    shards = O.partition_mem(spec, state, src_cfg)
    alibi = next(p for p in spec.params if p.kind == ParamKind.ASYNC_PARTIAL)
    if bad:
        recs = all_rank_records(spec, src_cfg)
        g = next(g for g in range(src_cfg.world_size) if recs[g][0].placement[1:] == (3, 33))
        i = next(i for i, m in enumerate(recs[g]) if (m.param, m.kind) == (alibi.name, "v"))
        m, a = shards[g][i]
        a = a.copy()
        a.reshape(-1).view(np.uint32)[2] ^= 1
        shards[g][i] = (m, a)
        with pytest.raises(O.OracleError, match="ReplicateMismatchError"):
            O.convert_mem(spec, src_cfg, shards)
    got, fails, _ = _arena_union(spec, src_cfg, shards)
    if bad:
        assert fails and all(e == 2 for _, e in fails)
        return
    assert fails == []
    want = O.convert_mem(spec, src_cfg, shards)
    for p in spec.params:
        for k in STATE_KINDS:
            assert np.array_equal(got[(p.name, k)].view(np.uint32),
                                  want[p.name][k].view(np.uint32)), (p.name, k)


def test_status_word_starts_ok():
    # a fresh status word decodes as "no failure" (first = ~0, n_bad = 0)
    import torch

    from paper_2406_18820_b200.engine import Status

    assert Status(torch.device("cpu")).read() == ((1 << 64) - 1, 0)

"""Descriptor compiler: (param, kind) units -> 2-D strided run tables + tiles.

This is the host half of the hot path. It turns the reference's union /
extract_fragment semantics into the device descriptor table that
``libucp_b200.so`` executes (include/ucp_b200.h):

* ``compile_union``   mirrors union() + _collapse_dp() + strip_pad()
                      (ucp/convert.py:115-308): all metadata validation
                      happens here, raising the reference's error classes in
                      the reference's order; data-dependent checks (replica
                      equality, zero pads) become COPY-with-replicas and
                      CHECKZERO runs whose failures come back via ucp_status.
* ``compile_extract`` mirrors extract_fragment() + partial_noise() + cast
                      (ucp/parallel.py:340-411, ucp/tensor.py:208-223); target
                      records with identical bytes (dp replicas, tp replicas
                      of replicated params) share one read and fan out.
* ``compile_grid``    mirrors _union_hy() (ucp/convert.py:196-218).

A TP fragment is addressed in its own row-major flat space. The TP pattern is
a list of *correspondences* (frag flat interval <-> 2-D region of the atomic
tensor, see ``tp_correspondences``); ZeRO flat pieces and replicas are
*source maps* over the same flat space. Runs are emitted per sub-interval
between all source-map boundaries, each split into head / body / tail rows.
"""

from __future__ import annotations

from collections import defaultdict
from dataclasses import dataclass, field

import numpy as np

from ._errors import (
    ManifestError,
    MissingFragmentError,
    OverlappingRangeError,
    PaddingError,
    PatternCoverageError,
    ShapeError,
)
from .layout import (
    PARTIAL,
    REPLICATE,
    SHARD_H,
    SHARD_HY,
    SHARD_NC,
    SHARD_V,
    frag_shape,
    mode_of,
    vocab_padded_rows,
)
from .spec import DType, ParallelConfig, ParamSpec, RecordMeta

# --------------------------------------------------------------------------- ABI

OP_COPY, OP_MEAN, OP_NOISE, OP_ZERO, OP_CHECKZERO = 0, 1, 2, 3, 4
RUN_VEC, RUN_ROWSPLIT = 1, 2
CLASS_VEC_F32, CLASS_VEC_BF16, CLASS_VEC_F16, CLASS_GENERAL, CLASS_OPS = 0, 1, 2, 3, 4
NCLASS = 5
SEG = 512            # elements per warp segment (kSeg in the kernel)
MAX_AUX = 256        # kMaxAux in the kernel
MAX_SRC = 64         # sources per run before verify-only continuation runs
MAX_DST = 64         # destinations per run before a second fan-out run

RUN_DTYPE = np.dtype({
    "names": ["src", "dst", "src_pitch", "dst_pitch", "rows", "cols", "aux", "n_src", "n_dst",
              "groups", "op", "dtype", "tp_rank", "tp", "tag", "flags"],
    "formats": ["<u8", "<u8", "<u4", "<u4", "<u4", "<u4", "<u4", "<u2", "<u2",
                "<u2", "u1", "u1", "<u2", "<u2", "<u4", "<u4"],
    "offsets": [0, 8, 16, 20, 24, 28, 32, 36, 38, 40, 42, 43, 44, 46, 48, 52],
    "itemsize": 64,
})
TILE_DTYPE = np.dtype([("run", "<u4"), ("row0", "<u4"), ("col0", "<u4"), ("count", "<u4")])
# ucp_runtile (include/ucp_b200.h): per-run tiling; `first` is filled on the
# device by ucp_runtile_scan (host copies keep it for the interpreter)
RUNTILE_DTYPE = np.dtype([("first", "<u4"), ("per", "<u4"), ("tpr", "<u4"), ("ntiles", "<u4")])
XRUN_DTYPE = np.dtype({
    "names": ["src", "atom", "dst", "src_pitch", "atom_pitch", "dst_pitch", "rows", "cols", "aux",
              "n_src", "n_dst", "dtype", "tag", "flags"],
    "formats": ["<u8", "<u8", "<u8", "<u4", "<u4", "<u4", "<u4", "<u4", "<u4", "<u2", "<u2", "u1",
                "<u4", "<u4"],
    "offsets": [0, 8, 16, 24, 28, 32, 36, 40, 44, 48, 50, 52, 56, 60],
    "itemsize": 64,
})
NO_ATOM = (1 << 64) - 1

_ESZ = {DType.F32: 4, DType.F16: 2, DType.BF16: 2}


def _numel(shape) -> int:
    n = 1
    for d in shape:
        n *= int(d)
    return n


# --------------------------------------------------------------------------- tables


@dataclass
class Unit:
    """Provenance of a (param, kind) unit, for error messages."""

    param: str
    kind: str
    labels: dict = field(default_factory=dict)  # run index -> list of source labels


class RunTable:
    """Accumulates runs + aux offsets for one kernel launch."""

    def __init__(self):
        self._rows: list = []
        self._aux: list = []
        self.units: list = []
        self.src_bytes = 0   # algorithmic bytes read
        self.dst_bytes = 0   # algorithmic bytes written

    def unit(self, param: str, kind: str) -> int:
        self.units.append(Unit(param, kind))
        return len(self.units) - 1

    def add(self, *, srcs, dsts, src_pitch, dst_pitch, rows, cols, op=OP_COPY, groups=1,
            dtype=DType.F32, tp_rank=0, tp=1, tag=0, labels=None) -> None:
        """srcs/dsts: byte offsets (group-major for sources)."""
        if rows == 0 or cols == 0:
            return
        if rows * cols >= 1 << 32:
            # keep rows*cols < 2^32 (element index inside a run is u32)
            per = max(1, ((1 << 31) // cols))
            for r0 in range(0, rows, per):
                n = min(per, rows - r0)
                self.add(srcs=[s + 4 * r0 * src_pitch for s in srcs],
                         dsts=[d + _ESZ[dtype] * r0 * dst_pitch for d in dsts],
                         src_pitch=src_pitch, dst_pitch=dst_pitch, rows=n, cols=cols, op=op,
                         groups=groups, dtype=dtype, tp_rank=tp_rank, tp=tp, tag=tag,
                         labels=labels)
            return
        if len(dsts) > MAX_DST:
            for i in range(0, len(dsts), MAX_DST):
                self.add(srcs=srcs if i == 0 else srcs[:1], dsts=dsts[i:i + MAX_DST],
                         src_pitch=src_pitch, dst_pitch=dst_pitch, rows=rows, cols=cols, op=op,
                         groups=groups, dtype=dtype, tp_rank=tp_rank, tp=tp, tag=tag,
                         labels=labels if i == 0 else None)
            return
        if len(srcs) > MAX_SRC and op == OP_COPY:
            # verify-only continuation runs compare extra replicas with replica 0
            head, rest = srcs[:MAX_SRC], srcs[MAX_SRC:]
            self.add(srcs=head, dsts=dsts, src_pitch=src_pitch, dst_pitch=dst_pitch, rows=rows,
                     cols=cols, op=op, dtype=dtype, tag=tag,
                     labels=None if labels is None else labels[:MAX_SRC])
            for i in range(0, len(rest), MAX_SRC - 1):
                chunk = rest[i:i + MAX_SRC - 1]
                self.add(srcs=[srcs[0]] + chunk, dsts=[], src_pitch=src_pitch,
                         dst_pitch=dst_pitch, rows=rows, cols=cols, op=op, tag=tag,
                         labels=None if labels is None else
                         [labels[0]] + labels[MAX_SRC + i:MAX_SRC + i + len(chunk)])
            return
        if len(srcs) + len(dsts) - 2 > MAX_AUX:
            raise ShapeError("too many sources for one averaged run")
        esz = _ESZ[dtype]
        ph = set()
        for s in srcs:
            ph.add((s // 4) % 4 if s % 4 == 0 else -1)
        for d in dsts:
            ph.add((d // esz) % 4 if d % esz == 0 else -1)
        vec = len(ph) == 1 and -1 not in ph and (
            rows == 1 or (src_pitch % 4 == 0 and dst_pitch % 4 == 0) or
            (not srcs and dst_pitch % 4 == 0) or (not dsts and src_pitch % 4 == 0))
        aux_at = len(self._aux)
        self._aux.extend(srcs[1:])
        self._aux.extend(dsts[1:])
        if labels is not None:
            self.units[tag].labels[len(self._rows)] = labels
        self._rows.append((srcs[0] if srcs else 0, dsts[0] if dsts else 0, src_pitch, dst_pitch,
                           rows, cols, aux_at, len(srcs), len(dsts), groups, op, dtype.value,
                           tp_rank, tp, tag, RUN_VEC if vec else 0))
        n = rows * cols
        self.src_bytes += 4 * n * len(srcs)
        self.dst_bytes += esz * n * len(dsts)

    def __len__(self):
        return len(self._rows)

    def finish(self, tile_bytes: int = 1 << 17) -> tuple:
        """(runs, aux, tiles) in table order, tiles expanded on the host
        (tests and the interpreter; the kernels derive them per CTA)."""
        runs, aux = self._runs_aux()
        return runs, aux, expand_tiles(runs, make_runtiles(runs, tile_bytes))

    def _runs_aux(self) -> tuple:
        runs = np.zeros(len(self._rows), dtype=RUN_DTYPE)
        if self._rows:
            cols = list(zip(*self._rows))
            for name, vals in zip(RUN_DTYPE.names, cols):
                runs[name] = vals
        aux = np.asarray(self._aux if self._aux else [0], dtype=np.uint64)
        return runs, aux

    def finish_classed(self, tile_bytes: int = 1 << 17):
        """(runs sorted by kernel class, aux, their ucp_runtile array,
        class_info = tiles per class then runs per class, sorted -> table
        index). Run order within a class is table order."""
        runs, aux = self._runs_aux()
        return classed(runs, aux, run_classes(runs), tile_bytes)


def run_classes(runs: np.ndarray) -> np.ndarray:
    """Kernel class of each run (UCP_CLASS_* in include/ucp_b200.h): the
    vector kernels take COPY runs with a shared 16-B phase, the GENERAL
    (realigning) kernels the other COPY runs, the OPS kernels MEAN / NOISE /
    ZERO / CHECKZERO."""
    copy = (runs["op"] == OP_COPY) & (runs["n_src"] >= 1)
    vec = ((runs["flags"] & RUN_VEC) != 0) & copy
    by_dt = np.select([runs["dtype"] == DType.F32.value, runs["dtype"] == DType.BF16.value],
                      [CLASS_VEC_F32, CLASS_VEC_BF16], CLASS_VEC_F16)
    return np.select([vec, copy], [by_dt, CLASS_GENERAL], CLASS_OPS).astype(np.int64)


def make_runtiles(runs: np.ndarray, tile_bytes: int, extra_bpe=None) -> np.ndarray:
    """Per-run tiling (ucp_runtile), one CTA per tile; a tile never
    straddles runs. Tile size is normalised by bytes moved per element so
    tiles cost about the same. Runs wider than a tile are cut into column
    tiles of single rows (UCP_RUN_ROWSPLIT, set here); the others into
    blocks of whole rows. ``first`` is the exclusive prefix of ``ntiles`` in
    array order (the device recomputes it per class, ucp_runtile_scan)."""
    rt = np.zeros(len(runs), dtype=RUNTILE_DTYPE)
    if len(runs) == 0:
        return rt
    esz = np.where(runs["dtype"] == 0, 4, 2).astype(np.int64)
    bpe = 4 * runs["n_src"].astype(np.int64) + esz * runs["n_dst"].astype(np.int64)
    if extra_bpe is not None:
        bpe = bpe + extra_bpe
    bpe = np.maximum(bpe, 4)
    telems = np.maximum(SEG, (tile_bytes // bpe) // SEG * SEG)
    rows = runs["rows"].astype(np.int64)
    cols = runs["cols"].astype(np.int64)
    split = cols > telems
    runs["flags"] = np.where(split, runs["flags"] | RUN_ROWSPLIT, runs["flags"] & ~np.uint32(RUN_ROWSPLIT))
    tpr = np.where(split, -(-cols // telems), 0)
    rpt = np.maximum(1, telems // np.maximum(cols, 1))
    rt["per"] = np.where(split, telems, rpt)
    rt["tpr"] = tpr
    ntiles = np.where(split, rows * tpr, -(-rows // rpt))
    if ntiles.sum() >= 1 << 31:
        raise ValueError("too many tiles for one launch; use smaller windows")
    rt["ntiles"] = ntiles
    rt["first"] = np.cumsum(ntiles) - ntiles
    return rt


def make_tiles(runs: np.ndarray, tile_bytes: int, extra_bpe=None) -> np.ndarray:
    """Expanded tile list of runs in table order (host-side view)."""
    return expand_tiles(runs, make_runtiles(runs, tile_bytes, extra_bpe))


def expand_tiles(runs: np.ndarray, rt: np.ndarray) -> np.ndarray:
    """Every tile of a classed table as the kernels derive it per CTA
    (ucp_tile: run, row0, col0, count), in launch order. Host mirror of
    tile_begin() in csrc/ucp_b200.cu, for the interpreter and the tests."""
    n = rt["ntiles"].astype(np.int64)
    run = np.repeat(np.arange(len(runs), dtype=np.int64), n)
    k = np.arange(int(n.sum()), dtype=np.int64) - np.repeat(np.cumsum(n) - n, n)
    per = rt["per"].astype(np.int64)[run]
    tpr = rt["tpr"].astype(np.int64)[run]
    split = (runs["flags"][run] & RUN_ROWSPLIT) != 0
    t = np.zeros(len(run), dtype=TILE_DTYPE)
    t["run"] = run
    row0 = np.where(split, k // np.maximum(tpr, 1), k * per)
    col0 = np.where(split, (k - row0 * np.maximum(tpr, 1)) * per, 0)
    t["row0"] = row0
    t["col0"] = col0
    t["count"] = np.where(split, np.minimum(per, runs["cols"][run].astype(np.int64) - col0),
                          np.minimum(per, runs["rows"][run].astype(np.int64) - row0))
    return t


def classed(runs: np.ndarray, aux: np.ndarray, cls: np.ndarray, tile_bytes: int,
            extra_bpe=None) -> tuple:
    """Stable-sort runs by kernel class and tile them: (runs, aux, rt,
    class_info[2 * NCLASS] = tiles per class, then runs per class, order)
    with order[i] = table index of sorted run i (run labels are keyed by
    table index)."""
    order = np.argsort(cls, kind="stable")
    runs = runs[order]
    cls = cls[order]
    extra = None if extra_bpe is None else np.asarray(extra_bpe)[order]
    rt = make_runtiles(runs, tile_bytes, extra)
    info = np.zeros(2 * NCLASS, dtype=np.int64)
    nt = rt["ntiles"].astype(np.int64)
    for c in range(NCLASS):
        sel = cls == c
        info[c] = int(nt[sel].sum())
        info[NCLASS + c] = int(sel.sum())
    # per-class exclusive prefix, as ucp_runtile_scan computes it on the device
    start = 0
    for c in range(NCLASS):
        n = int(info[NCLASS + c])
        seg = nt[start:start + n]
        rt["first"][start:start + n] = np.cumsum(seg) - seg
        start += n
    return runs, aux, rt, info, order


# --------------------------------------------------------------------------- geometry


def tp_correspondences(p: ParamSpec, mode: str, tp: int, t: int, vrows=None) -> list:
    """[(f0, x_off, x_pitch, rows, cols)]: TP fragment t's flat elements
    f0 + i*cols + j  <->  atomic element x_off + i*x_pitch + j.
    The inverse of extract_fragment's slicing (ucp/parallel.py:383-399).
    ``vrows``: padded vocab rows (extension); fragment rows beyond the real
    vocabulary have no atomic counterpart (stripped / zero-filled)."""
    shape = tuple(p.shape)
    n = _numel(shape)
    if n == 0:
        return []
    if vrows is not None:
        w = _numel(shape[1:])
        r = vrows // tp
        real = max(0, min(r, shape[0] - t * r))
        return [(0, t * r * w, real * w, 1, real * w)] if real else []
    if mode in ("full", REPLICATE, PARTIAL):
        return [(0, 0, n, 1, n)]
    if mode == SHARD_V:
        fn = n // tp
        return [(0, t * fn, fn, 1, fn)]
    if mode == SHARD_H:
        inner = _numel(shape[2:])
        c = shape[1] // tp * inner
        return [(0, t * c, shape[1] * inner, shape[0], c)]
    if mode == SHARD_NC:
        w = _numel(shape[1:])
        out, cum = [], 0
        for start, length in p.nc_segments:
            k = length // tp
            out.append((cum * w, (start + t * k) * w, k * w, 1, k * w))
            cum += k
        return out
    raise PatternCoverageError(f"mode {mode} not extractable")


def split_rows(corr, a: int, b: int) -> list:
    """Pieces (frag_start, x_start, x_pitch, rows, cols) of frag interval
    [a, b) under one correspondence: head partial row, full rows, tail."""
    f0, x0, xp, R, C = corr
    a, b = max(a, f0), min(b, f0 + R * C)
    if a >= b:
        return []
    out = []
    i, j = divmod(a - f0, C)
    if j:
        n = min(C - j, b - a)
        out.append((a, x0 + i * xp + j, xp, 1, n))
        a += n
        i += 1
        if a >= b:
            return out
    full = (b - a) // C
    if full:
        out.append((a, x0 + i * xp, xp, full, C))
        a += full * C
        i += full
    if a < b:
        out.append((a, x0 + i * xp, xp, 1, b - a))
    return out


class SourceMap:
    """Where a TP fragment's flat elements [0, n) live: sorted segments
    (lo, hi, byte_offset_of_lo)."""

    __slots__ = ("segs", "label")

    def __init__(self, segs, label):
        self.segs = segs
        self.label = label

    def offset(self, pos: int) -> int:
        for lo, hi, off in self.segs:
            if lo <= pos < hi:
                return off + 4 * (pos - lo)
        raise ShapeError(f"flat position {pos} not covered")

    def bounds(self):
        for lo, hi, _ in self.segs:
            yield lo
            yield hi


def _cuts(maps, lo: int, hi: int) -> list:
    pts = {lo, hi}
    for m in maps:
        for x in m.bounds():
            if lo < x < hi:
                pts.add(x)
    return sorted(pts)


# --------------------------------------------------------------------------- union


def _where(p, frags) -> str:
    return f"{p.name}.{frags[0][0].kind if frags else '?'}"


def _collapse(p, cfg, t, items, mode, strict, where):
    """_collapse_dp validation (ucp/convert.py:137-193). items: [(meta, off,
    n)]. Returns (replica source maps, pad check segments)."""
    ctx = f"{where} tp_rank {t}"
    flat = items[0][0].flat_range is not None
    for m, _, _ in items:
        if (m.flat_range is not None) != flat:
            raise ManifestError(f"{ctx}: mixed flat and non-flat fragments")
    seen = defaultdict(list)
    for it in items:
        seen[it[0].placement[2]].append(it)
    missing = [d for d in range(cfg.dp) if d not in seen]
    if missing:
        raise MissingFragmentError(f"{ctx}: no fragment from dp ranks {missing}")
    if not flat:
        dups = [d for d, grp in seen.items() if len(grp) > 1]
        if dups:
            raise OverlappingRangeError(f"{ctx}: duplicate fragments from dp ranks {dups}")
        fshape = _mode_shape(p, mode, cfg)
        fn = _numel(fshape)
        maps = []
        for d in range(cfg.dp if strict else 1):
            m, off, n = seen[d][0]
            if n != fn:
                raise ShapeError(f"{ctx}: fragment of {n} elements, expected {fshape}")
            maps.append(SourceMap([(0, fn, off)], (t, d)))
        return maps, []
    ranged = sorted(items, key=lambda it: tuple(it[0].flat_range))
    pos = 0
    segs = []
    for i, (m, off, n) in enumerate(ranged):
        lo, hi = m.flat_range
        if lo < pos:
            raise OverlappingRangeError(f"{ctx}: flat range [{lo},{hi}) overlaps previous end {pos}")
        if lo > pos:
            raise MissingFragmentError(f"{ctx}: flat gap [{pos},{lo})")
        if hi - lo != n:
            raise ManifestError(f"{ctx}: payload size != flat range extent")
        pos = hi
        if i != len(ranged) - 1 and m.pad_elems:
            raise PaddingError(f"{ctx}: pad recorded on a non-final flat shard")
        segs.append((lo, hi, off))
    pad = ranged[-1][0].pad_elems
    fn = _numel(frag_shape(p, mode, cfg))
    if pad < 0 or fn + pad != pos:
        raise PaddingError(
            f"pad arithmetic mismatch: {pos} elements != {fn} + pad {pad}")
    smap = SourceMap(segs, (t, None))
    pad_runs = []
    if pad:
        for lo, hi, off in segs:
            a, b = max(lo, fn), min(hi, pos)
            if a < b:
                pad_runs.append((off + 4 * (a - lo), b - a))
    return [smap], pad_runs


def _mode_shape(p, mode, cfg):
    if mode in ("full", REPLICATE, PARTIAL, SHARD_V, SHARD_H, SHARD_NC):
        return frag_shape(p, mode, cfg)
    raise ManifestError(f"{p.name}: unknown pattern tag {mode!r}")


def _emit_group(tab, p, groups, corrs, fn, dst_off, op, tag, G):
    """Runs writing atomic regions from `groups` (list over G of replica
    source maps) through `corrs`. dst_off None: verify-only runs (replica
    checks with no destination)."""
    maps = [m for grp in groups for m in grp]
    labels = [m.label for m in maps]
    cuts = _cuts(maps, 0, fn)
    for a, b in zip(cuts[:-1], cuts[1:]):
        for corr in corrs:
            for fs, xs, xp, rows, cols in split_rows(corr, a, b):
                tab.add(srcs=[m.offset(fs) for m in maps],
                        dsts=[] if dst_off is None else [dst_off + 4 * xs],
                        src_pitch=corr[4], dst_pitch=xp, rows=rows, cols=cols, op=op,
                        groups=G, tag=tag, labels=labels)


def compile_union(tab: RunTable, p: ParamSpec, cfg: ParallelConfig, frags: list,
                  dst_off: int, strict: bool = True) -> int:
    """Runs that consolidate one (param, kind) into the atomic tensor at byte
    offset dst_off. frags: [(RecordMeta, src_byte_off, n_elems)]."""
    if not frags:
        raise MissingFragmentError(f"{p.name}: no fragments at all")
    where = _where(p, frags)
    kinds = {m.kind for m, _, _ in frags}
    names = {m.param for m, _, _ in frags}
    tags = {m.pattern for m, _, _ in frags}
    if len(kinds) != 1 or names != {p.name}:
        raise ManifestError(f"{where}: mixed params/kinds in one union call")
    if len(tags) != 1:
        raise ManifestError(f"{where}: inconsistent pattern tags {sorted(tags)}")
    tag_name = frags[0][0].pattern
    tag = tab.unit(p.name, frags[0][0].kind)
    if tag_name == SHARD_HY:
        return compile_grid(tab, p, frags, dst_off, tag, where)
    stages = {m.placement[0] for m, _, _ in frags}
    if len(stages) != 1:
        raise ManifestError(f"{where}: fragments from multiple pp stages {sorted(stages)}")
    mode = "full" if cfg.tp == 1 else tag_name
    by_tp = defaultdict(list)
    for it in frags:
        by_tp[it[0].placement[1]].append(it)
    expect = {0} if mode == "full" else set(range(cfg.tp))
    if set(by_tp) != expect:
        raise MissingFragmentError(f"{where}: tp ranks {sorted(by_tp)} != expected {sorted(expect)}")
    per_tp = {}
    pads = []
    for t, items in by_tp.items():
        per_tp[t], pr = _collapse(p, cfg, t, items, mode, strict, where)
        pads += pr
    if mode not in ("full", REPLICATE, PARTIAL, SHARD_V, SHARD_H, SHARD_NC):
        raise ManifestError(f"{where}: unknown pattern tag {tag_name!r}")
    if mode == SHARD_NC:
        segs = frags[0][0].segments
        if segs is None or tuple(map(tuple, segs)) != tuple(map(tuple, p.nc_segments or ())):
            raise ManifestError(f"{where}: nc segments disagree with the model spec")
    fshape = frag_shape(p, mode, cfg)
    vrows = vocab_padded_rows(p, cfg)
    if vrows is None:
        _check_assembled(p, mode, fshape, cfg.tp, where)
    fn = _numel(fshape)

    for off, n in pads:
        tab.add(srcs=[off], dsts=[], src_pitch=n, dst_pitch=n, rows=1, cols=n,
                op=OP_CHECKZERO, tag=tag, labels=[("pad",)])
    if mode == "full":
        _emit_group(tab, p, [per_tp[0]], tp_correspondences(p, "full", 1, 0, vrows), fn,
                    dst_off, OP_COPY, tag, 1)
    elif mode == REPLICATE:
        grp = [m for t in range(cfg.tp) for m in per_tp[t]] if strict else per_tp[0][:1]
        _emit_group(tab, p, [grp], tp_correspondences(p, mode, cfg.tp, 0), fn, dst_off,
                    OP_COPY, tag, 1)
    elif mode == PARTIAL:
        groups = [per_tp[t] for t in range(cfg.tp)]
        corrs = tp_correspondences(p, mode, cfg.tp, 0)
        if sum(len(g) for g in groups) - 1 > MAX_AUX:
            # too many sources for one averaged run (tp x dp replicas): each
            # tp rank's dp replicas are checked by verify-only COPY runs
            # (split further by RunTable.add), then the MEAN reads one
            # replica per tp rank -- the same bytes, in _collapse_dp order
            for grp in groups:
                if len(grp) > 1:
                    _emit_group(tab, p, [grp], corrs, fn, None, OP_COPY, tag, 1)
            groups = [grp[:1] for grp in groups]
        _emit_group(tab, p, groups, corrs, fn, dst_off, OP_MEAN, tag, cfg.tp)
    else:
        for t in range(cfg.tp):
            _emit_group(tab, p, [per_tp[t]], tp_correspondences(p, mode, cfg.tp, t, vrows), fn,
                        dst_off, OP_COPY, tag, 1)
    return tag


def _check_assembled(p, mode, fshape, tp, where):
    s = tuple(p.shape)
    if mode in ("full", REPLICATE, PARTIAL):
        got = fshape
    elif mode == SHARD_V:
        got = (fshape[0] * tp,) + fshape[1:]
    elif mode == SHARD_H:
        got = (fshape[0], fshape[1] * tp) + fshape[2:] if len(fshape) > 1 else fshape
    else:
        got = s if sum(n for _, n in p.nc_segments) == s[0] and all(
            n % tp == 0 for _, n in p.nc_segments) else (-1,)
    if tuple(got) != s:
        raise ShapeError(f"{where}: assembled {tuple(got)} != spec {s}")


def compile_grid(tab, p, frags, dst_off, tag, where) -> int:
    """Shard-Hy block grid, placement (0, row, col) (ucp/convert.py:196-218)."""
    grid = {}
    for m, off, n in frags:
        key = (m.placement[1], m.placement[2])
        if key in grid:
            raise OverlappingRangeError(f"{where}: duplicate block {key}")
        grid[key] = (m, off, n)
    R = 1 + max(k[0] for k in grid)
    C = 1 + max(k[1] for k in grid)
    missing = [(r, c) for r in range(R) for c in range(C) if (r, c) not in grid]
    if missing:
        raise MissingFragmentError(f"{where}: missing blocks {missing[:4]}")
    if len(p.shape) != 2:
        raise ShapeError(f"{where}: shard_hy needs a 2-D param")
    rows = [tuple(grid[(r, 0)][0].shape)[0] for r in range(R)]
    cols = [tuple(grid[(0, c)][0].shape)[1] for c in range(C)]
    for (r, c), (m, _, n) in grid.items():
        if tuple(m.shape) != (rows[r], cols[c]) or n != rows[r] * cols[c]:
            raise ShapeError(f"{where}: block {(r, c)} shape {m.shape}")
    if (sum(rows), sum(cols)) != tuple(p.shape):
        raise ShapeError(f"{where}: assembled {(sum(rows), sum(cols))} != {p.shape}")
    W = p.shape[1]
    r0 = 0
    for r in range(R):
        c0 = 0
        for c in range(C):
            m, off, n = grid[(r, c)]
            tab.add(srcs=[off], dsts=[dst_off + 4 * (r0 * W + c0)], src_pitch=cols[c],
                    dst_pitch=W, rows=rows[r], cols=cols[c], tag=tag, labels=[(r, c)])
            c0 += cols[c]
        r0 += rows[r]
    return tag


# --------------------------------------------------------------------------- extract


def noise_is_identity(t: int, tp: int) -> bool:
    return tp == 1 or (tp % 2 == 1 and t == tp - 1)


def compile_extract(tab: RunTable, p: ParamSpec, cfg: ParallelConfig, targets: list,
                    src_off: int, dtype: DType = DType.F32) -> int:
    """Runs slicing one atomic tensor (f32 at byte offset src_off) into every
    target record in `targets` = [(RecordMeta, dst_byte_off)], writing
    `dtype` (the weight cast; moments pass DType.F32)."""
    if not targets:
        return -1
    tag = tab.unit(p.name, targets[0][0].kind)
    mode = mode_of(p, cfg)
    fshape = frag_shape(p, mode, cfg)
    vrows = vocab_padded_rows(p, cfg)
    fn = _numel(fshape)
    esz = _ESZ[dtype]
    groups = defaultdict(list)
    for meta, off in targets:
        t = meta.placement[1]
        if mode in (SHARD_V, SHARD_H, SHARD_NC):
            key_t = t
        elif mode == PARTIAL and not noise_is_identity(t, cfg.tp):
            key_t = t
        else:
            key_t = -1
        fr = None if meta.flat_range is None else tuple(meta.flat_range)
        groups[(key_t, fr)].append(off)
    padded = -(-fn // cfg.dp) * cfg.dp if fn else 0
    for (key_t, fr), dsts in groups.items():
        t = max(key_t, 0)
        corrs = tp_correspondences(p, mode if mode != PARTIAL else "full", cfg.tp, t, vrows)
        op = OP_NOISE if mode == PARTIAL and key_t >= 0 else OP_COPY
        if fr is None:
            lo, hi = 0, fn
        else:
            lo, hi = min(fr[0], padded), min(max(fr[1], fr[0]), padded)
        covered = []
        for corr in corrs:
            for fs, xs, xp, rows, cols in split_rows(corr, lo, min(hi, fn)):
                tab.add(srcs=[src_off + 4 * xs], dsts=[d + esz * (fs - lo) for d in dsts],
                        src_pitch=xp, dst_pitch=corr[4], rows=rows, cols=cols, op=op,
                        dtype=dtype, tp_rank=t, tp=cfg.tp, tag=tag)
                covered.append((fs, fs + rows * cols))
        # zero-fill whatever no correspondence covers: the ZeRO pad tail and
        # (extension) padded vocabulary rows
        at = lo
        for a, b in sorted(covered) + [(hi, hi)]:
            if a > at:
                tab.add(srcs=[], dsts=[d + esz * (at - lo) for d in dsts], src_pitch=a - at,
                        dst_pitch=a - at, rows=1, cols=a - at, op=OP_ZERO, dtype=dtype, tag=tag)
            at = max(at, b)
    return tag


def fragment_elems(p: ParamSpec, cfg: ParallelConfig, meta: RecordMeta) -> int:
    """Element count of the fragment extract_fragment returns for meta."""
    fshape = frag_shape(p, mode_of(p, cfg), cfg)
    if meta.flat_range is None:
        return _numel(fshape)
    fn = _numel(fshape)
    padded = -(-fn // cfg.dp) * cfg.dp if fn else 0
    lo, hi = meta.flat_range
    lo, hi = min(lo, padded), min(max(hi, lo), padded)
    return max(hi - lo, 0)


def fragment_shape(p: ParamSpec, cfg: ParallelConfig, meta: RecordMeta) -> tuple:
    if meta.flat_range is None:
        return tuple(frag_shape(p, mode_of(p, cfg), cfg))
    return (fragment_elems(p, cfg, meta),)


# --------------------------------------------------------------------------- fused


class XRunTable:
    """Fused convert+load runs (ucp_xrun) for one ucp_reshard_fused launch."""

    def __init__(self):
        self._rows: list = []
        self._aux: list = []
        self.units: list = []
        self.src_bytes = 0
        self.atom_bytes = 0
        self.dst_bytes = 0

    def unit(self, param: str, kind: str) -> int:
        self.units.append(Unit(param, kind))
        return len(self.units) - 1

    def add(self, *, srcs, atom, dsts, src_pitch, atom_pitch, dst_pitch, rows, cols, dtype, tag,
            labels=None, vec: bool = True) -> None:
        """vec: every source, the atomic and every destination share one
        16-B phase (the vector kernels); otherwise the cell runs on the
        scalar fused path (coalesced 4-B accesses, reshard_fused_mixed)."""
        if rows == 0 or cols == 0:
            return
        if labels is not None:
            self.units[tag].labels[len(self._rows)] = labels
        aux_at = len(self._aux)
        self._aux.extend(srcs[1:])
        self._aux.extend(dsts[1:])
        self._rows.append((srcs[0], atom, dsts[0] if dsts else 0, src_pitch, atom_pitch, dst_pitch,
                           rows, cols, aux_at, len(srcs), len(dsts), dtype.value, tag,
                           RUN_VEC if vec else 0))
        n = rows * cols
        self.src_bytes += 4 * n * len(srcs)
        self.atom_bytes += 0 if atom == NO_ATOM else 4 * n
        self.dst_bytes += _ESZ[dtype] * n * len(dsts)

    def __len__(self):
        return len(self._rows)

    def finish_classed(self, tile_bytes: int = 1 << 17):
        runs = np.zeros(len(self._rows), dtype=XRUN_DTYPE)
        if self._rows:
            for name, vals in zip(XRUN_DTYPE.names, zip(*self._rows)):
                runs[name] = vals
        aux = np.asarray(self._aux if self._aux else [0], dtype=np.uint64)
        extra = np.where(runs["atom"] == np.uint64(NO_ATOM), 0, 4).astype(np.int64)
        cls = np.select([runs["dtype"] == DType.F32.value, runs["dtype"] == DType.BF16.value],
                        [CLASS_VEC_F32, CLASS_VEC_BF16], CLASS_VEC_F16).astype(np.int64)
        # phase-mismatched cells: the scalar fused path (reshard_fused_scalar)
        cls = np.where((runs["flags"] & RUN_VEC) != 0, cls, CLASS_GENERAL).astype(np.int64)
        return classed(runs, aux, cls, tile_bytes, extra)


def _rects(x0, xp, rows, cols, exts, ep, esz, R, W):
    """Pieces of one run's atomic-side region as rectangles of the [R, W] grid:
    (r0, c0, rows, cols, ext offsets at (r0, c0), ext pitch)."""
    if rows == 1:
        out = []
        for fs, xs, _, r, c in split_rows((0, 0, W, R, W), x0, x0 + cols):
            sh = esz * (fs - x0)
            out.append((xs // W, xs % W, r, c, [e + sh for e in exts], W if r > 1 else c))
        return out
    if xp != W:
        return None
    return [(x0 // W, x0 % W, rows, cols, list(exts), ep)]


def compile_fused(fx: XRunTable, rest_conv: RunTable, rest_load: RunTable, p: ParamSpec,
                  src: ParallelConfig, frags: list, atom_off: int, tgt: ParallelConfig,
                  targets: list, dtype: DType = DType.F32, strict: bool = True,
                  materialize: bool = True) -> bool:
    """Fused convert+load of one (param, kind): every atomic element is
    gathered (with replica checks), written to the atomic tensor at atom_off
    (unless materialize=False) and scattered to its target fragments in the
    same pass. Validation and error behaviour are compile_union's and
    compile_extract's (they run first). Units that cannot fuse (Partial
    mean/noise, phase-mismatched pieces, very wide fan-in/out) are emitted
    unfused into rest_conv / rest_load instead. Returns True when fused."""
    conv, load = RunTable(), RunTable()
    compile_union(conv, p, src, frags, atom_off, strict)
    compile_extract(load, p, tgt, targets, atom_off, dtype)
    n = _numel(p.shape)
    W = _numel(p.shape[1:]) if len(p.shape) > 1 else max(n, 1)
    R = n // W if W else 0
    esz = _ESZ[dtype]
    crects, lrects, extra_conv, extra_load = [], [], [], []
    ok = n > 0
    for i, r in enumerate(conv._rows):
        (s0, d0, sp, dp, rows, cols, aux, ns, nd, groups, op, dt, tpr, tp, tag, flags) = r
        if op == OP_CHECKZERO or (op == OP_COPY and nd == 0):
            # pad checks and the verify-only continuation runs of units with
            # more than MAX_SRC replicas (RunTable.add) have no atomic
            # destination: they run unfused, reading only their sources
            extra_conv.append(i)
            continue
        if op != OP_COPY or ns > MAX_SRC:
            ok = False
            break
        srcs = [s0] + conv._aux[aux:aux + ns - 1]
        got = _rects((d0 - atom_off) // 4, dp, rows, cols, srcs, sp, 4, R, W)
        if got is None:
            ok = False
            break
        crects += [(g, i) for g in got]
    if ok:
        for i, r in enumerate(load._rows):
            (s0, d0, sp, dp, rows, cols, aux, ns, nd, groups, op, dt, tpr, tp, tag, flags) = r
            if op == OP_ZERO:
                extra_load.append(i)
                continue
            if op != OP_COPY or nd > MAX_DST:
                ok = False
                break
            dsts = [d0] + load._aux[aux + ns - 1:aux + ns - 1 + nd - 1]
            got = _rects((s0 - atom_off) // 4, sp, rows, cols, dsts, dp, esz, R, W)
            if got is None:
                ok = False
                break
            lrects += [(g, i) for g in got]
    cells = []
    if ok:
        for (a, ai) in crects:
            ar0, ac0, ar, ac, aext, aep = a
            for (b, bi) in lrects:
                br0, bc0, br, bc, bext, bep = b
                r0, r1 = max(ar0, br0), min(ar0 + ar, br0 + br)
                c0, c1 = max(ac0, bc0), min(ac0 + ac, bc0 + bc)
                if r0 >= r1 or c0 >= c1:
                    continue
                srcs = [e + 4 * ((r0 - ar0) * aep + (c0 - ac0)) for e in aext]
                dsts = [e + esz * ((r0 - br0) * bep + (c0 - bc0)) for e in bext]
                atom = atom_off + 4 * (r0 * W + c0)
                ph = {(x // 4) % 4 for x in srcs} | {(atom // 4) % 4} | {(x // esz) % 4 for x in dsts}
                pit = r1 - r0 == 1 or (aep % 4 == 0 and bep % 4 == 0 and W % 4 == 0)
                if any(x % 4 for x in srcs) or any(x % esz for x in dsts):
                    ok = False
                    break
                # cells whose pieces do not share one 16-B phase (e.g. ZeRO
                # partitions of dp = 3) take the scalar fused path
                cells.append((srcs, atom, dsts, aep, bep, r1 - r0, c1 - c0, ai,
                              len(ph) == 1 and pit))
            if not ok:
                break
        if ok and sum(c[5] * c[6] for c in cells) != n:
            ok = False
    if not ok:
        _absorb(rest_conv, conv)
        _absorb(rest_load, load)
        return False
    cmap, lmap = {}, {}
    tag = fx.unit(p.name, frags[0][0].kind)
    for srcs, atom, dsts, sp, dp, rows, cols, ci, vec in cells:
        fx.add(srcs=srcs, atom=atom if materialize else NO_ATOM, dsts=dsts, src_pitch=sp,
               atom_pitch=W, dst_pitch=dp, rows=rows, cols=cols, dtype=dtype, tag=tag,
               labels=conv.units[0].labels.get(ci) if conv.units else None, vec=vec)
    for i in extra_conv:
        _absorb_row(rest_conv, conv, i, cmap)
    for i in extra_load:
        _absorb_row(rest_load, load, i, lmap)
    return True


def _absorb_row(dst: RunTable, src: RunTable, i: int, tags: dict) -> None:
    """Copy run i of src into dst; ``tags`` maps src unit ids to dst unit
    ids for this (src, dst) pair."""
    (s0, d0, sp, dp, rows, cols, aux, ns, nd, groups, op, dt, tpr, tp, tag, flags) = src._rows[i]
    unit = src.units[tag]
    new_tag = tags.get(tag)
    if new_tag is None:
        new_tag = tags[tag] = dst.unit(unit.param, unit.kind)
    nsx = max(ns - 1, 0)
    srcs = ([s0] + src._aux[aux:aux + nsx]) if ns else []
    dsts = ([d0] + src._aux[aux + nsx:aux + nsx + nd - 1]) if nd else []
    dst.add(srcs=srcs, dsts=dsts, src_pitch=sp, dst_pitch=dp, rows=rows, cols=cols, op=op,
            groups=groups, dtype=DType(dt), tp_rank=tpr, tp=tp, tag=new_tag,
            labels=unit.labels.get(i))


def _absorb(dst: RunTable, src: RunTable) -> None:
    tags: dict = {}
    for i in range(len(src._rows)):
        _absorb_row(dst, src, i, tags)

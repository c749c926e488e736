"""Layout rules: which elements of which parameter live on which rank.

Host-side integer logic that feeds the descriptor compiler (plan.py). It
restates the reference's layout arithmetic (ucp/parallel.py:88-332):

* rank numbering g = (pp*tp + tp_rank)*dp + dp_rank       (:69-75)
* compatibility rules                                      (:77-104)
* pp stage -> layers, sequential / interleaved(v)          (:112-141)
* TP pattern per param kind                                (:177-226)
* ZeRO flat split, pad on the last dp rank                 (:156-164, :229-235)
* manifest pattern tags                                    (:251-259)
* per-rank records in canonical order                      (:288-332)

Records are memoised per (spec, cfg): the reshard planner asks for them once
per plan, and ``ucp_info``/``load`` reuse them.
"""

from __future__ import annotations

from functools import lru_cache

from ._errors import IncompatibleConfigError, PatternCoverageError
from .spec import STATE_KINDS, ModelSpec, ParallelConfig, ParamKind, ParamSpec, RecordMeta, ZeroStage

UNIQUE, REPLICATE, PARTIAL = "unique", "replicate", "partial"
SHARD_V, SHARD_H, SHARD_HY, SHARD_NC = "shard_v", "shard_h", "shard_hy", "shard_nc"
PATTERNS = (UNIQUE, REPLICATE, PARTIAL, SHARD_V, SHARD_H, SHARD_HY, SHARD_NC)

_REPLICATED = {ParamKind.LAYERNORM_WEIGHT, ParamKind.LAYERNORM_BIAS}
_FUSED = {ParamKind.FUSED_QKV, ParamKind.FUSED_EXPERT}
_VOCAB = {ParamKind.EMBEDDING, ParamKind.TIED_EMBEDDING}


def kind_of(p) -> ParamKind:
    """The param's kind as this package's enum (duck-types the reference's
    ParamSpec objects, whose enum class differs but whose values match)."""
    k = p.kind
    return k if isinstance(k, ParamKind) else ParamKind(getattr(k, "value", k))


def zero_of(cfg) -> ZeroStage:
    z = cfg.zero_stage
    return z if isinstance(z, ZeroStage) else ZeroStage(getattr(z, "value", z))


def config_key(cfg) -> tuple:
    """Field-wise identity of a ParallelConfig that also holds across the
    reference's class (its dataclass ``==`` compares class first)."""
    s = cfg.pp_schedule
    return (cfg.dp, cfg.tp, cfg.pp, cfg.sp, zero_of(cfg), s.kind, s.v,
            getattr(cfg, "vocab_multiple", 1))


def same_config(a, b) -> bool:
    """``a == b`` as ucp/load.py:250 means it, for either package's configs."""
    return config_key(a) == config_key(b)


def validate_model_config(spec: ModelSpec, cfg: ParallelConfig) -> None:
    cfg.validate()
    if cfg.pp > max(spec.n_layers, 1):
        raise IncompatibleConfigError(
            f"pp={cfg.pp} exceeds layer depth {max(spec.n_layers, 1)} of {spec.name}")
    if cfg.pp_schedule.kind == "interleaved":
        chunks = cfg.pp * cfg.pp_schedule.v
        if spec.n_layers % chunks:
            raise IncompatibleConfigError(
                f"interleaved(v={cfg.pp_schedule.v}) needs n_layers divisible by pp*v = "
                f"{chunks}, got {spec.n_layers}")
    for p in spec.params:
        mode_of(p, cfg)


def vocab_padded_rows(p: ParamSpec, cfg: ParallelConfig):
    """Padded row count of an embedding / output layer under Megatron-style
    vocab padding (extension): ceil(V / (m * tp)) * m * tp, or
    None when cfg.vocab_multiple == 1 or the param is not vocab-sized."""
    m = getattr(cfg, "vocab_multiple", 1)
    if m <= 1 or kind_of(p) not in _VOCAB or not p.shape:
        return None
    unit = m * cfg.tp
    return -(-p.shape[0] // unit) * unit


def mode_of(p: ParamSpec, cfg: ParallelConfig) -> str:
    """tp_mode with the vocab-padding extension: a padded vocab param is
    Shard-V over its padded rows (always divisible)."""
    if vocab_padded_rows(p, cfg) is not None:
        return "full" if cfg.tp == 1 else SHARD_V
    return tp_mode(p, cfg.tp)


def frag_shape(p: ParamSpec, mode: str, cfg: ParallelConfig) -> tuple:
    """tp_fragment_shape with the vocab-padding extension."""
    rows = vocab_padded_rows(p, cfg)
    if rows is not None:
        return (rows // cfg.tp,) + tuple(p.shape[1:])
    return tp_fragment_shape(p, mode, cfg.tp)


def pp_layer_map(n_layers: int, pp: int, schedule) -> list:
    depth = max(n_layers, 1)
    if not 1 <= pp <= depth:
        raise IncompatibleConfigError(f"pp={pp} invalid for {n_layers} layers")
    if schedule.kind == "sequential":
        if n_layers == 0:
            return [[0]] + [[] for _ in range(pp - 1)]
        q, r = divmod(depth, pp)
        bounds = [0]
        for s in range(pp):
            bounds.append(bounds[-1] + q + (1 if s < r else 0))
        return [list(range(bounds[s], bounds[s + 1])) for s in range(pp)]
    chunks = pp * schedule.v
    if n_layers % chunks:
        raise IncompatibleConfigError(
            f"interleaved needs n_layers % (pp*v) == 0, got {n_layers} % {chunks}")
    size = n_layers // chunks
    stages = [[] for _ in range(pp)]
    for j in range(chunks):
        stages[j % pp] += list(range(j * size, (j + 1) * size))
    return stages


def stage_of_layer(n_layers: int, pp: int, schedule, layer: int) -> int:
    for s, layers in enumerate(pp_layer_map(n_layers, pp, schedule)):
        if layer in layers:
            return s
    raise IncompatibleConfigError(f"layer {layer} outside [0, {max(n_layers, 1)})")


def zero_flatten_meta(numel: int, dp: int) -> tuple:
    if dp < 1:
        raise IncompatibleConfigError("dp must be >= 1")
    per = -(-numel // dp)
    return per * dp, per * dp - numel, [(r * per, (r + 1) * per) for r in range(dp)]


def _divisible(p: ParamSpec, axis: int, tp: int) -> None:
    if len(p.shape) <= axis:
        raise PatternCoverageError(f"{p.name}: shape {p.shape} lacks axis {axis}")
    if p.shape[axis] % tp:
        raise PatternCoverageError(
            f"{p.name}: axis {axis} extent {p.shape[axis]} not divisible by tp={tp}")


def tp_mode(p: ParamSpec, tp: int) -> str:
    if tp == 1:
        return "full"
    k = kind_of(p)
    if k in _REPLICATED:
        return REPLICATE
    if k is ParamKind.ASYNC_PARTIAL:
        return PARTIAL
    if k in _VOCAB:
        _divisible(p, 0, tp)
        return SHARD_V
    if k is ParamKind.MATMUL2D:
        if p.tp_axis_hint not in (0, 1):
            raise PatternCoverageError(
                f"{p.name}: matmul2d without a tp axis hint cannot shard under tp={tp}")
        _divisible(p, p.tp_axis_hint, tp)
        return SHARD_V if p.tp_axis_hint == 0 else SHARD_H
    if k in _FUSED:
        if not p.nc_segments:
            raise PatternCoverageError(f"{p.name}: fused param lacks nc_segments")
        at = 0
        for s, (start, length) in enumerate(p.nc_segments):
            if start != at or length <= 0:
                raise PatternCoverageError(f"{p.name}: nc_segments must tile axis 0 contiguously")
            if length % tp:
                raise PatternCoverageError(
                    f"{p.name}: segment {s} of length {length} not divisible by tp={tp}")
            at += length
        if at != p.shape[0]:
            raise PatternCoverageError(f"{p.name}: nc_segments do not cover axis 0")
        return SHARD_NC
    raise PatternCoverageError(f"{p.name}: no rule for kind {k.value} under tp={tp}")


def zero_flattens(kind: str, zero: ZeroStage) -> bool:
    zero = ZeroStage(getattr(zero, "value", zero))
    if zero is ZeroStage.Z0:
        return False
    if zero in (ZeroStage.Z1, ZeroStage.Z2):
        return kind in ("m", "v")
    return True


def tp_fragment_shape(p: ParamSpec, mode: str, tp: int) -> tuple:
    s = tuple(p.shape)
    if mode in ("full", REPLICATE, PARTIAL):
        return s
    if mode == SHARD_V:
        return (s[0] // tp,) + s[1:]
    if mode == SHARD_H:
        return (s[0], s[1] // tp) + s[2:]
    if mode == SHARD_NC:
        return (sum(n // tp for _, n in p.nc_segments),) + s[1:]
    raise PatternCoverageError(f"no fragment shape for mode {mode}")


def pattern_tag(mode: str, flat: bool, dp: int) -> str:
    if mode != "full":
        return mode
    if flat:
        return SHARD_V
    return REPLICATE if dp > 1 else UNIQUE


def _numel(shape) -> int:
    n = 1
    for d in shape:
        n *= int(d)
    return n


@lru_cache(maxsize=64)
def _all_records(spec: ModelSpec, cfg: ParallelConfig) -> tuple:
    stages = pp_layer_map(spec.n_layers, cfg.pp, cfg.pp_schedule)
    last = max(spec.n_layers - 1, 0)
    modes = [mode_of(p, cfg) for p in spec.params]
    out = []
    for g in range(cfg.world_size):
        pp_r, tp_r, dp_r = cfg.coords_of(g)
        mine = set(stages[pp_r])
        recs = []
        for p, mode in zip(spec.params, modes):
            if min(p.layer_index, last) not in mine:
                continue
            fshape = frag_shape(p, mode, cfg)
            fnumel = _numel(fshape)
            segs = p.nc_segments if mode == SHARD_NC else None
            for kind in STATE_KINDS:
                if zero_flattens(kind, zero_of(cfg)):
                    _, pad, ranges = zero_flatten_meta(fnumel, cfg.dp)
                    lo, hi = ranges[dp_r]
                    recs.append(RecordMeta(p.name, kind, pattern_tag(mode, True, cfg.dp),
                                           (pp_r, tp_r, dp_r), (hi - lo,), segs, (lo, hi),
                                           pad if dp_r == cfg.dp - 1 else 0))
                else:
                    recs.append(RecordMeta(p.name, kind, pattern_tag(mode, False, cfg.dp),
                                           (pp_r, tp_r, dp_r), fshape, segs))
        out.append(tuple(recs))
    return tuple(out)


def enumerate_rank_records(spec: ModelSpec, cfg: ParallelConfig, g: int) -> list:
    return list(_all_records(spec, cfg)[g])


def all_rank_records(spec: ModelSpec, cfg: ParallelConfig) -> tuple:
    """Records of every rank (tuple indexed by g); memoised."""
    return _all_records(spec, cfg)


def layer_of(spec: ModelSpec, p: ParamSpec) -> int:
    return min(p.layer_index, max(spec.n_layers, 1) - 1)

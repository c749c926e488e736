"""Value types of the drop-in surface: tensors, model specs, parallel configs.

These mirror the reference's public types so callers only swap the import:

* ``DType`` / ``Tensor`` / ``make_tensor``        -- ucp/tensor.py:43-110
* ``ParamKind`` / ``ParamSpec`` / ``ModelSpec``   -- ucp/models.py:32-83
* ``ZeroStage`` / ``PPSchedule`` / ``ParallelConfig`` -- ucp/parallel.py:36-85
* ``RecordMeta``                                   -- ucp/parallel.py:269-285
* model.json / config.json / config-string codecs  -- ucp/models.py:374-421,
  ucp/parallel.py:441-503

Extension: ``ZeroStage.Z2`` ("z2") is accepted and lays out
exactly like Z1 (the reference omits ZeRO-2 because its checkpoint content
equals Z1).
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from enum import Enum
from functools import cached_property

import numpy as np

from ._errors import IncompatibleConfigError, ModelConfigError, ShapeError

# ---------------------------------------------------------------------------
# tensors
# ---------------------------------------------------------------------------


class DType(Enum):
    """Storage dtypes; values are the UCPT header codes."""

    F32 = 0
    F16 = 1
    BF16 = 2

    @property
    def itemsize(self) -> int:
        return 4 if self is DType.F32 else 2

    @property
    def storage(self) -> np.dtype:
        return _STORAGE[self]


_STORAGE = {DType.F32: np.dtype("<f4"), DType.F16: np.dtype("<f2"), DType.BF16: np.dtype("<u2")}


@dataclass(frozen=True)
class Tensor:
    """Read-only dense tensor; bf16 payloads are raw uint16 bit patterns."""

    dtype: DType
    shape: tuple
    data: np.ndarray

    def __post_init__(self):
        if tuple(self.data.shape) != tuple(self.shape):
            raise ShapeError(f"data shape {self.data.shape} != {self.shape}")
        if self.data.dtype != self.dtype.storage:
            raise ShapeError(f"storage dtype {self.data.dtype} does not match {self.dtype}")

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape, dtype=np.int64)) if self.shape else 1

    @property
    def nbytes(self) -> int:
        return self.numel * self.dtype.itemsize

    def tobytes(self) -> bytes:
        return np.ascontiguousarray(self.data).tobytes()

    def bits_equal(self, other: "Tensor") -> bool:
        return (self.dtype is other.dtype and tuple(self.shape) == tuple(other.shape)
                and self.tobytes() == other.tobytes())


def make_tensor(dtype: DType, array) -> Tensor:
    arr = np.asarray(array, dtype=dtype.storage)
    if not arr.flags["C_CONTIGUOUS"]:
        arr = np.ascontiguousarray(arr)
    return Tensor(dtype, tuple(arr.shape), arr)


# ---------------------------------------------------------------------------
# model description
# ---------------------------------------------------------------------------


class ParamKind(Enum):
    MATMUL2D = "matmul2d"
    FUSED_QKV = "fused_qkv"
    FUSED_EXPERT = "fused_expert"
    LAYERNORM_WEIGHT = "layernorm_weight"
    LAYERNORM_BIAS = "layernorm_bias"
    EMBEDDING = "embedding"
    TIED_EMBEDDING = "tied_embedding"
    ASYNC_PARTIAL = "async_partial"


@dataclass(frozen=True)
class ParamSpec:
    name: str
    shape: tuple
    layer_index: int
    kind: ParamKind
    tp_axis_hint: int | None = None
    nc_segments: tuple | None = None

    @property
    def numel(self) -> int:
        n = 1
        for d in self.shape:
            n *= int(d)
        return n


@dataclass(frozen=True)
class ModelSpec:
    name: str
    n_layers: int
    tied_pairs: tuple
    params: tuple

    @cached_property
    def _by_name(self) -> dict:
        return {p.name: p for p in self.params}

    def param(self, name: str) -> ParamSpec:
        try:
            return self._by_name[name]
        except KeyError:
            raise ModelConfigError(f"unknown param {name!r}") from None

    def tied_leader(self, name: str) -> str:
        for leader, follower in self.tied_pairs:
            if follower == name:
                return leader
        return name

    @property
    def total_numel(self) -> int:
        return sum(p.numel for p in self.params)


STATE_KINDS = ("weight", "m", "v")
FORMAT_VERSION = 1

# ---------------------------------------------------------------------------
# parallel configs
# ---------------------------------------------------------------------------


class ZeroStage(Enum):
    Z0 = "z0"
    Z1 = "z1"
    Z2 = "z2"  # extension: same checkpoint layout as Z1
    Z3 = "z3"


@dataclass(frozen=True)
class PPSchedule:
    kind: str = "sequential"
    v: int = 1

    def __post_init__(self):
        if self.kind == "sequential":
            if self.v != 1:
                raise IncompatibleConfigError("sequential schedule has no interleave")
        elif self.kind == "interleaved":
            if self.v < 2:
                raise IncompatibleConfigError("interleaved schedule needs v >= 2")
        else:
            raise IncompatibleConfigError(f"unknown pp schedule {self.kind!r}")


@dataclass(frozen=True)
class ParallelConfig:
    dp: int = 1
    tp: int = 1
    pp: int = 1
    sp: int = 1
    zero_stage: ZeroStage = ZeroStage.Z0
    pp_schedule: PPSchedule = field(default_factory=PPSchedule)
    # extension: Megatron-style vocab padding of embedding /
    # output-layer rows to a multiple of vocab_multiple * tp; 1 = none (the
    # reference has no vocab padding)
    vocab_multiple: int = 1

    @property
    def world_size(self) -> int:
        return self.dp * self.tp * self.pp

    def rank_of(self, pp_rank: int, tp_rank: int, dp_rank: int) -> int:
        # pp outermost, dp innermost (ucp/parallel.py:9-11)
        return (pp_rank * self.tp + tp_rank) * self.dp + dp_rank

    def coords_of(self, g: int) -> tuple:
        q, d = divmod(g, self.dp)
        return q // self.tp, q % self.tp, d

    def validate(self) -> None:
        if min(self.dp, self.tp, self.pp, self.sp) < 1:
            raise IncompatibleConfigError("all parallel degrees must be >= 1")
        if self.zero_stage is ZeroStage.Z3 and (self.tp, self.pp) != (1, 1):
            raise IncompatibleConfigError("ZeRO-3 requires tp == 1 and pp == 1")
        if self.pp_schedule.kind == "interleaved" and self.pp < 2:
            raise IncompatibleConfigError("interleaved schedule needs pp >= 2")
        if self.sp > 1 and self.dp % self.sp:
            raise IncompatibleConfigError("sp folds into dp and must divide it")
        if self.vocab_multiple < 1:
            raise IncompatibleConfigError("vocab_multiple must be >= 1")


@dataclass(frozen=True)
class RecordMeta:
    """One fragment's metadata (what manifests serialise)."""

    param: str
    kind: str
    pattern: str
    placement: tuple
    shape: tuple
    segments: tuple | None = None
    flat_range: tuple | None = None
    pad_elems: int = 0

    @property
    def file(self) -> str:
        return f"{self.param}.{self.kind}.ucpt"


# ---------------------------------------------------------------------------
# (de)serialisation
# ---------------------------------------------------------------------------


def _segs_out(segs):
    return None if segs is None else [list(s) for s in segs]


def spec_to_dict(spec: ModelSpec) -> dict:
    params = []
    for p in spec.params:
        params.append({"name": p.name, "shape": list(p.shape), "layer_index": p.layer_index,
                       "kind": p.kind.value, "tp_axis_hint": p.tp_axis_hint,
                       "nc_segments": _segs_out(p.nc_segments)})
    return {"name": spec.name, "n_layers": spec.n_layers,
            "tied_pairs": [list(t) for t in spec.tied_pairs], "params": params}


def spec_to_json(spec: ModelSpec) -> str:
    return json.dumps(spec_to_dict(spec), indent=2) + "\n"


def spec_from_dict(d: dict) -> ModelSpec:
    try:
        params = []
        for e in d["params"]:
            segs = e["nc_segments"]
            params.append(ParamSpec(
                name=e["name"], shape=tuple(int(x) for x in e["shape"]),
                layer_index=int(e["layer_index"]), kind=ParamKind(e["kind"]),
                tp_axis_hint=e["tp_axis_hint"],
                nc_segments=None if segs is None else tuple((int(a), int(b)) for a, b in segs)))
        return ModelSpec(name=d["name"], n_layers=int(d["n_layers"]),
                         tied_pairs=tuple((a, b) for a, b in d["tied_pairs"]),
                         params=tuple(params))
    except (KeyError, ValueError, TypeError) as e:
        raise ModelConfigError(f"bad model description: {e}") from e


def config_to_dict(cfg: ParallelConfig) -> dict:
    d = {"dp": cfg.dp, "tp": cfg.tp, "pp": cfg.pp, "sp": cfg.sp,
         "zero_stage": cfg.zero_stage.value, "pp_schedule": cfg.pp_schedule.kind,
         "pp_interleave": cfg.pp_schedule.v}
    if cfg.vocab_multiple != 1:
        d["vocab_multiple"] = cfg.vocab_multiple  # extension key, absent by default
    return d


def config_from_dict(d: dict) -> ParallelConfig:
    try:
        cfg = ParallelConfig(dp=int(d["dp"]), tp=int(d["tp"]), pp=int(d["pp"]), sp=int(d["sp"]),
                             zero_stage=ZeroStage(d["zero_stage"]),
                             pp_schedule=PPSchedule(d["pp_schedule"], int(d["pp_interleave"])),
                             vocab_multiple=int(d.get("vocab_multiple", 1)))
    except (KeyError, ValueError, TypeError) as e:
        raise IncompatibleConfigError(f"bad parallel config: {e}") from e
    cfg.validate()
    return cfg


def parse_config_string(s: str) -> ParallelConfig:
    """'dp,tp,pp,sp,zero,schedule' e.g. '2,1,4,1,z1,seq' or '...,int2'."""
    fields = s.split(",")
    if len(fields) != 6:
        raise IncompatibleConfigError(f"config string needs 6 comma-separated fields: {s!r}")
    try:
        dp, tp, pp, sp = (int(x) for x in fields[:4])
    except ValueError as e:
        raise IncompatibleConfigError(f"bad degree in {s!r}: {e}") from e
    try:
        zs = ZeroStage(fields[4].strip().lower())
    except ValueError as e:
        raise IncompatibleConfigError(f"zero stage must be z0|z1|z2|z3: {fields[4]!r}") from e
    sched = fields[5].strip().lower()
    if sched == "seq":
        ps = PPSchedule()
    elif sched.startswith("int"):
        try:
            ps = PPSchedule("interleaved", int(sched[3:]))
        except ValueError as e:
            raise IncompatibleConfigError(f"bad interleave in {sched!r}") from e
    else:
        raise IncompatibleConfigError(f"schedule must be seq or int<v>: {sched!r}")
    cfg = ParallelConfig(dp, tp, pp, sp, zs, ps)
    cfg.validate()
    return cfg


def format_config_string(cfg: ParallelConfig) -> str:
    sched = "seq" if cfg.pp_schedule.kind == "sequential" else f"int{cfg.pp_schedule.v}"
    return f"{cfg.dp},{cfg.tp},{cfg.pp},{cfg.sp},{cfg.zero_stage.value},{sched}"

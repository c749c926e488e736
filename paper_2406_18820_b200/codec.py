"""On-disk boundary: UCPT tensor containers, rank manifests, tree metadata.

Formats are the reference's, byte for byte:

* UCPT: b"UCPT", u16 version 1, u8 dtype, u8 ndim, ndim x u64 dims, raw LE
  payload (ucp/tensor.py:1-15, :266-320), including its error taxonomy;
* ``shards.json`` manifests and ``config.json`` / ``model.json``
  (ucp/partition.py:1-215), written tmp + rename where the reference does.

Payloads are read straight into caller-provided (pinned) staging memory with
``readinto`` -- no intermediate ``bytes`` object and no ``.copy()``, which is
where the reference spends most of its convert time.
"""

from __future__ import annotations

import json
import os
import struct
from dataclasses import dataclass

import numpy as np

from ._errors import (
    CheckpointLayoutError,
    CorruptHeaderError,
    ManifestError,
    TensorFileError,
    TensorIOError,
    TruncatedPayloadError,
)
from .spec import (
    FORMAT_VERSION,
    DType,
    ModelSpec,
    ParallelConfig,
    RecordMeta,
    Tensor,
    config_from_dict,
    config_to_dict,
    spec_from_dict,
)

MAGIC = b"UCPT"
FILE_VERSION = 1
MAX_FILE_NUMEL = 1 << 40
MANIFEST = "shards.json"
CONFIG_JSON = "config.json"
MODEL_JSON = "model.json"
_DTYPES = {d.value: d for d in DType}


@dataclass(frozen=True)
class Header:
    dtype: DType
    shape: tuple
    offset: int      # payload byte offset in the file
    file_size: int

    @property
    def numel(self) -> int:
        n = 1
        for d in self.shape:
            n *= d
        return n

    @property
    def nbytes(self) -> int:
        return self.numel * self.dtype.itemsize


def read_header(path: str) -> Header:
    """Parse and validate a UCPT header against the file size (same checks
    and classes as ucp/tensor.py:278-316)."""
    try:
        with open(path, "rb") as f:
            head = f.read(8)
            if len(head) < 8:
                raise CorruptHeaderError(f"{path}: header shorter than 8 bytes")
            magic, version, code, ndim = struct.unpack("<4sHBB", head)
            if magic != MAGIC:
                raise CorruptHeaderError(f"{path}: bad magic {magic!r}")
            if version != FILE_VERSION:
                raise CorruptHeaderError(f"{path}: unsupported version {version}")
            if code not in _DTYPES:
                raise CorruptHeaderError(f"{path}: unknown dtype code {code}")
            dims = f.read(8 * ndim)
            size = os.fstat(f.fileno()).st_size
    except OSError as e:
        raise TensorIOError(f"reading {path}: {e}") from e
    if len(dims) < 8 * ndim:
        raise CorruptHeaderError(f"{path}: truncated dims")
    shape = tuple(int(x) for x in struct.unpack(f"<{ndim}Q", dims))
    hdr = Header(_DTYPES[code], shape, 8 + 8 * ndim, size)
    if hdr.numel > MAX_FILE_NUMEL:
        raise CorruptHeaderError(f"{path}: implausible element count {hdr.numel}")
    have = size - hdr.offset
    if have < hdr.nbytes:
        raise TruncatedPayloadError(f"{path}: payload has {have} of {hdr.nbytes} bytes")
    if have > hdr.nbytes:
        raise TensorFileError(f"{path}: {have - hdr.nbytes} trailing bytes")
    return hdr


def read_payload_into(path: str, hdr: Header, dest: memoryview) -> None:
    """Read the payload into dest (len == hdr.nbytes) with readinto."""
    try:
        with open(path, "rb", buffering=0) as f:
            f.seek(hdr.offset)
            got = 0
            while got < hdr.nbytes:
                n = f.readinto(dest[got:])
                if not n:
                    raise TruncatedPayloadError(f"{path}: payload ended early")
                got += n
    except OSError as e:
        raise TensorIOError(f"reading {path}: {e}") from e


def read_range_into(path: str, file_off: int, dest: memoryview) -> None:
    """pread ``len(dest)`` bytes at ``file_off`` (one chunk of a payload;
    several chunks of one file are read by different threads)."""
    try:
        fd = os.open(path, os.O_RDONLY)
        try:
            got = 0
            while got < len(dest):
                n = os.preadv(fd, [dest[got:]], file_off + got)
                if not n:
                    raise TruncatedPayloadError(f"{path}: payload ended early")
                got += n
        finally:
            os.close(fd)
    except OSError as e:
        raise TensorIOError(f"reading {path}: {e}") from e


def payload_chunks(hdr: Header, chunk: int):
    """(payload offset, nbytes) pieces of at most ``chunk`` bytes."""
    if chunk <= 0 or hdr.nbytes <= chunk:
        return [(0, hdr.nbytes)]
    return [(o, min(chunk, hdr.nbytes - o)) for o in range(0, hdr.nbytes, chunk)]


def create_raw(path: str, dtype: DType, shape, nbytes: int) -> int:
    """Create a UCPT file of its final size with the header written; the
    payload is filled by ``write_range`` (possibly from several threads).
    Returns the payload offset."""
    hb = header_bytes(dtype, shape)
    try:
        with open(path, "wb") as f:
            f.write(hb)
            f.truncate(len(hb) + nbytes)
    except OSError as e:
        raise TensorIOError(f"writing {path}: {e}") from e
    return len(hb)


def write_range(path: str, file_off: int, payload) -> None:
    try:
        fd = os.open(path, os.O_WRONLY)
        try:
            mv = memoryview(payload).cast("B")
            done = 0
            while done < len(mv):
                done += os.pwritev(fd, [mv[done:]], file_off + done)
        finally:
            os.close(fd)
    except OSError as e:
        raise TensorIOError(f"writing {path}: {e}") from e


def read_tensor(path: str) -> Tensor:
    hdr = read_header(path)
    arr = np.empty(hdr.numel, dtype=hdr.dtype.storage)
    read_payload_into(path, hdr, memoryview(arr.view(np.uint8)))
    return Tensor(hdr.dtype, hdr.shape, arr.reshape(hdr.shape))


def header_bytes(dtype: DType, shape) -> bytes:
    return struct.pack("<4sHBB", MAGIC, FILE_VERSION, dtype.value, len(shape)) + \
        struct.pack(f"<{len(shape)}Q", *shape)


def write_raw(path: str, dtype: DType, shape, payload) -> None:
    """Write a UCPT file from a buffer-protocol payload (no copy)."""
    try:
        with open(path, "wb") as f:
            f.write(header_bytes(dtype, shape))
            f.write(payload)
    except OSError as e:
        raise TensorIOError(f"writing {path}: {e}") from e


def write_tensor(path: str, t: Tensor) -> None:
    write_raw(path, t.dtype, t.shape, memoryview(np.ascontiguousarray(t.data)).cast("B"))


def payload_bytes_on_disk(path: str) -> int:
    """Whole file size (ucp/tensor.py:323-329 counts the header too)."""
    try:
        return os.path.getsize(path)
    except OSError as e:
        raise TensorIOError(f"stat {path}: {e}") from e


# --------------------------------------------------------------------------- trees


def write_json(path: str, obj: dict) -> None:
    tmp = path + ".tmp"
    with open(tmp, "w") as f:
        json.dump(obj, f, indent=2)
        f.write("\n")
    os.replace(tmp, path)


def ensure_empty_dir(path: str) -> None:
    if os.path.exists(path):
        if not os.path.isdir(path) or os.listdir(path):
            raise CheckpointLayoutError(f"output dir {path!r} exists and is not empty")
    else:
        os.makedirs(path)


def record_to_entry(meta: RecordMeta) -> dict:
    return {"param": meta.param, "kind": meta.kind, "pattern": meta.pattern,
            "segments": None if meta.segments is None else [list(s) for s in meta.segments],
            "flat_range": None if meta.flat_range is None else list(meta.flat_range),
            "pad_elems": meta.pad_elems, "shape": list(meta.shape), "dtype": "f32",
            "file": meta.file}


def entry_to_record(entry: dict, placement: tuple) -> RecordMeta:
    try:
        segs, fr = entry["segments"], entry["flat_range"]
        return RecordMeta(
            param=entry["param"], kind=entry["kind"], pattern=entry["pattern"],
            placement=placement, shape=tuple(int(x) for x in entry["shape"]),
            segments=None if segs is None else tuple((int(a), int(b)) for a, b in segs),
            flat_range=None if fr is None else (int(fr[0]), int(fr[1])),
            pad_elems=int(entry["pad_elems"]))
    except (KeyError, ValueError, TypeError) as e:
        raise ManifestError(f"bad manifest entry: {e}") from e


def read_manifest(rank_dir: str) -> tuple:
    path = os.path.join(rank_dir, MANIFEST)
    if not os.path.isfile(path):
        raise ManifestError(f"{rank_dir!r} has no {MANIFEST} (empty or torn rank dir)")
    try:
        with open(path) as f:
            m = json.load(f)
    except (OSError, json.JSONDecodeError) as e:
        raise ManifestError(f"unreadable manifest {path!r}: {e}") from e
    try:
        pl = m["placement"]
        placement = (pl["pp"], pl["tp"], pl["dp"])
        return m, [entry_to_record(e, placement) for e in m["entries"]]
    except (KeyError, TypeError) as e:
        raise ManifestError(f"malformed manifest {path!r}: {e}") from e


def config_json_dict(cfg: ParallelConfig, step: int, metadata: dict) -> dict:
    return {"format_version": FORMAT_VERSION, "parallel": config_to_dict(cfg), "step": step,
            "world_size": cfg.world_size, "rank_order": "pp,tp,dp", "metadata": metadata}


def manifest_dict(cfg: ParallelConfig, g: int, records) -> dict:
    pp_r, tp_r, dp_r = cfg.coords_of(g)
    return {"format_version": FORMAT_VERSION, "rank": g,
            "placement": {"pp": pp_r, "tp": tp_r, "dp": dp_r},
            "entries": [record_to_entry(m) for m in records]}


@dataclass(frozen=True)
class DistributedCheckpoint:
    root: str
    cfg: ParallelConfig
    spec: ModelSpec
    step: int
    metadata: dict

    def rank_dir(self, g: int) -> str:
        return os.path.join(self.root, f"rank_{g}")

    def rank_dirs(self) -> list:
        return [self.rank_dir(g) for g in range(self.cfg.world_size)]


def load_checkpoint(root: str) -> DistributedCheckpoint:
    cpath, mpath = os.path.join(root, CONFIG_JSON), os.path.join(root, MODEL_JSON)
    if not (os.path.isfile(cpath) and os.path.isfile(mpath)):
        raise CheckpointLayoutError(f"{root!r} lacks {CONFIG_JSON} or {MODEL_JSON}")
    with open(cpath) as f:
        cj = json.load(f)
    with open(mpath) as f:
        spec = spec_from_dict(json.load(f))
    if cj.get("format_version") != FORMAT_VERSION:
        raise CheckpointLayoutError(
            f"{root!r}: unsupported format_version {cj.get('format_version')}")
    ckpt = DistributedCheckpoint(root, config_from_dict(cj["parallel"]), spec, int(cj["step"]),
                                 cj.get("metadata", {}))
    missing = [d for d in ckpt.rank_dirs() if not os.path.isdir(d)]
    if missing:
        raise CheckpointLayoutError(f"missing rank dirs: {missing[:3]}")
    return ckpt

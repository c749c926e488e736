"""The drop-in API: convert / load / resume / union / extract_fragment / ...

Signatures, defaults, return types, raised classes and the statistics
counters follow the reference package (ucp/convert.py:221-563,
ucp/load.py:37-281, ucp/parallel.py:373-411, ucp/tensor.py:208-223,
ucp/partition.py:151-174, ucp/models.py:230-244). Every element of every
tensor on these paths is produced by libucp_b200.so on the GPU; the host does
metadata validation, descriptor compilation and file I/O only.

Keyword-only extensions: ``device=`` (CUDA device) and ``window_bytes=``
(device staging budget per window).
"""

from __future__ import annotations

import hashlib
import json
import os
import threading
from collections import defaultdict
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np
import torch

from . import codec
from ._errors import (
    CheckpointLayoutError,
    ManifestError,
    MissingFragmentError,
    ShapeError,
    UnsupportedCastError,
)
from .engine import Program, Status, align_up, gen_state, pinned_host, require_device
from .layout import all_rank_records, layer_of, pp_layer_map, same_config, validate_model_config
from .plan import RunTable, compile_extract, compile_union, fragment_elems, fragment_shape
from .spec import (
    FORMAT_VERSION,
    STATE_KINDS,
    DType,
    ModelSpec,
    ParallelConfig,
    ParamSpec,
    RecordMeta,
    Tensor,
    format_config_string,
    make_tensor,
    spec_to_json,
)

UCP_META_JSON = "ucp_meta.json"
ATOMIC_FILES = {"weight": "weight.ucpt", "m": "adam_m.ucpt", "v": "adam_v.ucpt"}
DEFAULT_WINDOW_BYTES = 2 << 30

INVOCATIONS = 0


def conversions_invoked() -> int:
    """Process-wide count of convert() calls (ucp/convert.py:66-74)."""
    return INVOCATIONS


# --------------------------------------------------------------------------- types


@dataclass(frozen=True)
class FragmentMsg:
    """One fragment in flight; data is a numpy array or a CUDA tensor."""

    meta: RecordMeta
    data: object


@dataclass(frozen=True)
class ParamState:
    weight: Tensor
    m: Tensor
    v: Tensor


@dataclass
class ModelState:
    spec: ModelSpec
    params: dict
    step: int
    metadata: dict = field(default_factory=dict)


@dataclass(frozen=True)
class AtomicCheckpoint:
    root: str
    spec: ModelSpec
    step: int
    metadata: dict
    source_fingerprint: str

    def param_file(self, param: str, kind: str) -> str:
        return os.path.join(self.root, param, ATOMIC_FILES[kind])

    def read_param(self, param: str) -> dict:
        p = self.spec.param(param)
        out = {}
        for kind in STATE_KINDS:
            t = codec.read_tensor(self.param_file(param, kind))
            if t.dtype is not DType.F32 or tuple(t.shape) != tuple(p.shape):
                raise CheckpointLayoutError(
                    f"{param}.{kind}: expected f32 {p.shape}, got {t.dtype.name} {t.shape}")
            out[kind] = t
        return out


_TORCH_DT = {DType.F32: torch.float32, DType.BF16: torch.bfloat16, DType.F16: torch.float16}


class DeviceTensor:
    """A loaded shard that stays in HBM (``load(..., keep_on_device=True)``):
    the ``Tensor`` interface, with ``data`` materialised to host numpy on
    first access (cached) and ``device`` the zero-copy CUDA tensor (bf16 /
    f16 weights as torch.bfloat16 / float16 views of the same bits).
    SURVEY §8b: the GPU build keeps device buffers and materialises numpy
    lazily, so consolidate_world and the reference's checks work unchanged."""

    __slots__ = ("dtype", "shape", "_dev", "_host")

    def __init__(self, dtype: DType, shape: tuple, dev_bytes: torch.Tensor):
        self.dtype, self.shape, self._host = dtype, tuple(shape), None
        self._dev = dev_bytes.view(_TORCH_DT[dtype]).view(self.shape)

    @property
    def device(self) -> torch.Tensor:
        return self._dev

    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            t = self._dev.contiguous().view(torch.uint8).cpu().numpy()
            self._host = t.view(self.dtype.storage).reshape(self.shape)
        return self._host

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape, dtype=np.int64)) if self.shape else 1

    @property
    def nbytes(self) -> int:
        return self.numel * self.dtype.itemsize

    def tobytes(self) -> bytes:
        return np.ascontiguousarray(self.data).tobytes()

    def bits_equal(self, other) -> bool:
        return (self.dtype is other.dtype and tuple(self.shape) == tuple(other.shape)
                and self.tobytes() == other.tobytes())


@dataclass(frozen=True)
class WorldShard:
    meta: RecordMeta
    tensor: Tensor


@dataclass
class LoadStats:
    bypass: bool = True
    files_read: int = 0
    bytes_read: int = 0
    peak_resident_elements: int = 0
    resident_bound: int = 0
    conversions_invoked: int = 0
    group_files_needed: dict = field(default_factory=dict)
    group_files_read: dict = field(default_factory=dict)
    per_rank: dict = field(default_factory=dict)

    def to_dict(self) -> dict:
        return {"bypass": self.bypass, "files_read": self.files_read,
                "bytes_read": self.bytes_read,
                "peak_resident_elements": self.peak_resident_elements,
                "resident_bound": self.resident_bound,
                "conversions_invoked": self.conversions_invoked,
                "group_files_needed": self.group_files_needed,
                "group_files_read": self.group_files_read,
                "per_rank": {str(k): v for k, v in self.per_rank.items()}}


@dataclass
class LoadedWorld:
    cfg: ParallelConfig
    spec: ModelSpec
    step: int
    metadata: dict
    shards: dict
    stats: LoadStats


@dataclass(frozen=True)
class UcpInfo:
    cfg: ParallelConfig
    records: dict

    def dp_group(self, g: int) -> str:
        pp_r, tp_r, _ = self.cfg.coords_of(g)
        return f"{pp_r},{tp_r}"

    def replication_group(self, meta: RecordMeta) -> str:
        pp_r, tp_r, dp_r = meta.placement
        if meta.flat_range is not None:
            return f"{meta.param}.{meta.kind}@{pp_r},{tp_r},{dp_r}"
        return f"{meta.param}.{meta.kind}@{pp_r},{tp_r}"


def ucp_info(spec: ModelSpec, cfg: ParallelConfig) -> UcpInfo:
    validate_model_config(spec, cfg)
    recs = all_rank_records(spec, cfg)
    return UcpInfo(cfg, {g: list(recs[g]) for g in range(cfg.world_size)})


# --------------------------------------------------------------------------- staging


class _Staging:
    """Grow-only pinned host + device buffers reused across API calls."""

    def __init__(self):
        self.host: dict = {}
        self.dev: dict = {}

    def host_buf(self, key: str, nbytes: int) -> torch.Tensor:
        b = self.host.get(key)
        if b is None or b.numel() < nbytes:
            self.host.pop(key, None)
            b = pinned_host(max(align_up(nbytes, 1 << 20), 1 << 20))
            self.host[key] = b
        return b

    def dev_buf(self, key: str, nbytes: int, device) -> torch.Tensor:
        k = (key, str(device))
        b = self.dev.get(k)
        if b is None or b.numel() < nbytes:
            self.dev.pop(k, None)
            b = torch.empty(max(align_up(nbytes, 1 << 20), 1 << 20), dtype=torch.uint8,
                            device=device)
            self.dev[k] = b
        return b


class _PerThread(threading.local):
    """Staging buffers and status words are per thread: the reference runs
    union()/write_union() concurrently from reducer threads
    (ucp/convert.py:512-522), and every call here is reentrant."""

    def __init__(self):
        self.stage = _Staging()
        self.status: dict = {}
        self.plans: dict = {}  # reshard(): the last compiled ReshardPlan


_LOCAL = _PerThread()


class _StageProxy:
    def __getattr__(self, name):
        return getattr(_LOCAL.stage, name)


_STAGE = _StageProxy()


def _status(dev) -> Status:
    s = _LOCAL.status.get(str(dev))
    if s is None:
        s = _LOCAL.status[str(dev)] = Status(dev)
    return s


def release_staging() -> None:
    """Drop this thread's pinned / device staging buffers and its cached
    reshard() plan (they are grow-only and reused across calls otherwise)."""
    from . import reshard as _reshard

    _LOCAL.stage = _Staging()
    _LOCAL.plans = {}
    _reshard._D2D.state = None  # reshard_device's template, scratch and last sources


def _run(prog: Program, gather: bool, src_base: int, dst_base: int, dev) -> None:
    st = _status(dev)
    st.reset()
    prog.launch(gather, src_base, dst_base, st)
    torch.cuda.synchronize(dev)
    st.raise_if_bad(prog, src_base)


def _as_f32(data) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(data), dtype=np.float32)


def _is_cuda(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


# --------------------------------------------------------------------------- primitives


def union(p: ParamSpec, cfg: ParallelConfig, msgs: list, strict: bool = True):
    """Reassemble one (param, kind) from its fragments on the GPU
    (ucp/convert.py:221-308). numpy in -> numpy out; CUDA tensors in ->
    CUDA tensor out (zero-copy sources)."""
    if not msgs:
        raise MissingFragmentError(f"{p.name}: no fragments at all")
    on_dev = all(_is_cuda(m.data) for m in msgs)
    dev = require_device(msgs[0].data.device if on_dev else None)
    tab = RunTable()
    if on_dev:
        datas = [m.data.contiguous().float() for m in msgs]
        frags = [(m.meta, d.data_ptr(), d.numel()) for m, d in zip(msgs, datas)]
        src_base = 0
    else:
        arrays = [_as_f32(m.data) for m in msgs]
        offs, at = [], 0
        for a in arrays:
            offs.append(at)
            at += align_up(a.nbytes)
        stage = _STAGE.dev_buf("union_src", at, dev)
        for a, o in zip(arrays, offs):
            if a.nbytes:
                stage[o:o + a.nbytes].copy_(torch.from_numpy(a.reshape(-1).view(np.uint8)))
        frags = [(m.meta, o, a.size) for m, a, o in zip(msgs, arrays, offs)]
        src_base = stage.data_ptr()
    compile_union(tab, p, cfg, frags, 0, strict)
    out = torch.empty(max(p.numel, 1), dtype=torch.float32, device=dev)
    prog = Program(tab, dev)
    _run(prog, True, src_base, out.data_ptr(), dev)
    out = out[:p.numel].view(tuple(p.shape))
    return out if on_dev else out.cpu().numpy()


def extract_fragment(p: ParamSpec, cfg: ParallelConfig, meta: RecordMeta, full):
    """One rank's fragment of a consolidated f32 tensor, on the GPU
    (ucp/parallel.py:373-411)."""
    if tuple(full.shape) != tuple(p.shape):
        raise ShapeError(f"{p.name}: expected {p.shape}, got {tuple(full.shape)}")
    on_dev = _is_cuda(full)
    dev = require_device(full.device if on_dev else None)
    if on_dev:
        src = full.contiguous().float()
    else:
        src = torch.from_numpy(_as_f32(full)).to(dev)
    n = fragment_elems(p, cfg, meta)
    out = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
    tab = RunTable()
    compile_extract(tab, p, cfg, [(meta, 0)], src.data_ptr(), DType.F32)
    _run(Program(tab, dev), False, 0, out.data_ptr(), dev)
    out = out[:n].view(fragment_shape(p, cfg, meta))
    return out if on_dev else out.cpu().numpy()


def cast(t: Tensor, to: DType) -> Tensor:
    """RNE cast (ucp/tensor.py:208-223). f32 -> bf16/f16 runs on the GPU;
    the widening directions are exact bit operations."""
    if t.dtype is to:
        return Tensor(to, t.shape, t.data)
    if t.dtype is not DType.F32 and to is not DType.F32:
        raise UnsupportedCastError(f"cannot cast {t.dtype.name} -> {to.name} directly")
    if t.dtype is DType.F16:
        return make_tensor(DType.F32, t.data.astype(np.float32).reshape(t.shape))
    if t.dtype is DType.BF16:
        wide = (t.data.astype(np.uint32) << np.uint32(16)).view(np.float32)
        return make_tensor(DType.F32, wide.reshape(t.shape))
    dev = require_device()
    src = torch.from_numpy(_as_f32(t.data).reshape(-1)).to(dev)
    out = torch.empty(max(t.numel, 1), dtype=torch.int16, device=dev)
    tab = RunTable()
    tab.unit("cast", "weight")
    tab.add(srcs=[src.data_ptr()], dsts=[out.data_ptr()], src_pitch=t.numel, dst_pitch=t.numel,
            rows=1, cols=t.numel, dtype=to, tag=0)
    _run(Program(tab, dev), False, 0, 0, dev)
    host = out[:t.numel].cpu().numpy().view(to.storage).reshape(t.shape)
    return Tensor(to, tuple(t.shape), host)


# --------------------------------------------------------------------------- atomic ckpt


def source_fingerprint(src_root: str) -> str:
    with open(os.path.join(src_root, codec.CONFIG_JSON), "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def load_atomic(root: str) -> AtomicCheckpoint:
    mpath, upath = os.path.join(root, codec.MODEL_JSON), os.path.join(root, UCP_META_JSON)
    if not (os.path.isfile(upath) and os.path.isfile(mpath)):
        raise CheckpointLayoutError(f"{root!r} is not a complete atomic checkpoint (missing metadata)")
    from .spec import spec_from_dict

    with open(mpath) as f:
        spec = spec_from_dict(json.load(f))
    with open(upath) as f:
        meta = json.load(f)
    if meta.get("format_version") != FORMAT_VERSION:
        raise CheckpointLayoutError(f"{root!r}: unsupported format_version {meta.get('format_version')}")
    names = {p.name for p in spec.params}
    have = {d for d in os.listdir(root) if os.path.isdir(os.path.join(root, d))}
    if have != names:
        raise CheckpointLayoutError(
            f"{root!r}: param dirs disagree with model.json "
            f"(missing {sorted(names - have)[:3]}, extra {sorted(have - names)[:3]})")
    return AtomicCheckpoint(root, spec, int(meta["step"]), meta.get("metadata", {}),
                            meta.get("source_config_sha256", ""))


def _windows(items: list, size_of, budget: int) -> list:
    """Greedy contiguous grouping under a byte budget (one oversized item
    gets its own window)."""
    out, cur, acc = [], [], 0
    for it in items:
        s = size_of(it)
        if cur and acc + s > budget:
            out.append(cur)
            cur, acc = [], 0
        cur.append(it)
        acc += s
    if cur:
        out.append(cur)
    return out


def _io_threads(n_workers: int) -> int:
    """File I/O threads of one pipeline pool. The bytes written do not depend
    on it (ucp/convert.py:422-428: output independent of n_workers), so the
    pool uses the host's cores even at the reference's default n_workers=1;
    a larger n_workers can still raise it (up to 32)."""
    cores = os.cpu_count() or 4
    return max(4, min(32, max(cores, 2 * n_workers)))


def _io_pool(n_workers: int) -> ThreadPoolExecutor:
    return ThreadPoolExecutor(max_workers=_io_threads(n_workers))


# --------------------------------------------------------------------------- pipeline


def _write_atomic(out_dir: str, o, ov: memoryview) -> list:
    """One job writing one atomic file. Whole-file writes: concurrent
    ranged writes into one tmpfs file serialise on its inode lock and were
    2.4x slower (profiles/file_cfg2l4_r01ab_*.json)."""
    p, kind, at = o

    def job():
        pdir = os.path.join(out_dir, p.name)
        os.makedirs(pdir, exist_ok=True)
        codec.write_raw(os.path.join(pdir, ATOMIC_FILES[kind]), DType.F32, p.shape,
                        ov[at:at + 4 * p.numel])

    return [job]


class _Step:
    """One window's device work in ``_pipeline``: a single convert_gather or
    load_scatter launch over (src arena, dst arena)."""

    def __init__(self, prog: Program, gather: bool):
        self.prog, self.gather = prog, gather

    def launch(self, src: int, dst: int, st, stream, tgt: int | None = None) -> None:
        self.prog.launch(self.gather, src, dst if tgt is None else tgt, st, stream)

    def check(self, st, src: int, dst: int, stream) -> None:
        st.raise_if_bad(self.prog, src)


class _FusedStep:
    """One fused-resume window: the ucp_reshard_fused launch plus the rest
    tables (units compile_fused could not overlay), over one dst arena that
    holds the atomic tensors at [0, atom_at) and the target shards from
    atom_at on, so a single D2H drains both."""

    def __init__(self, fprog, cprog: Program, lprog: Program, atom_at: int):
        self.fprog, self.cprog, self.lprog, self.atom_at = fprog, cprog, lprog, atom_at
        self._tgt = None

    def launch(self, src: int, dst: int, st, stream, tgt: int | None = None) -> None:
        # tgt: the target shards' base when they go to a device sink instead
        # of the dst arena (resume(keep_on_device=True))
        self._tgt = dst + self.atom_at if tgt is None else tgt
        self.fprog.launch(src, dst, self._tgt, st, stream)
        self.cprog.launch(True, src, dst, st, stream)
        self.lprog.launch(False, dst, self._tgt, st, stream)

    def check(self, st, src: int, dst: int, stream) -> None:
        from .engine import describe_failure

        first, _ = st.read()
        if first == (1 << 64) - 1:
            return
        # localise: re-run the source-reading launches one at a time (the load
        # of atomic tensors cannot fail, it only reads what the others wrote)
        for prog in (self.fprog, self.cprog):
            st.reset(stream)
            if prog is self.fprog:
                prog.launch(src, dst, self._tgt, st, stream)
            else:
                prog.launch(True, src, dst, st, stream)
            stream.synchronize()
            f, _ = st.read()
            if f != (1 << 64) - 1:
                raise describe_failure(prog, f >> 32, f & 0xFFFFFFFF, src, (self.cprog,))
        raise RuntimeError("fused resume reported a failure that did not reproduce")


IO_CHUNK = int(os.environ.get("UCP_IO_CHUNK", 16 << 20))  # bytes per file read job (0: whole files)
COPY_CHUNK = int(os.environ.get("UCP_COPY_CHUNK", 64 << 20))  # bytes per host copy job
SEND_MIN = 4 << 20   # read chunks at least this large issue their own H2D
ALIGN_GAP = 4096     # unsent ranges closer than this are sent as one copy (gap bytes are junk)
PIPE_TRACE: dict = {}  # seconds the last _pipeline call spent waiting, by stage


def _chunks(nbytes: int, chunk: int = 0):
    chunk = chunk or IO_CHUNK
    if chunk <= 0 or nbytes <= chunk:
        return [(0, nbytes)]
    return [(o, min(chunk, nbytes - o)) for o in range(0, nbytes, chunk)]


def _coalesce(ranges, gap: int) -> list:
    """Merge (offset, nbytes) ranges whose holes are at most ``gap`` bytes
    into [offset, nbytes] runs (the holes are copied along)."""
    runs = []
    for at, n in sorted(ranges):
        if runs and at - (runs[-1][0] + runs[-1][1]) <= gap:
            runs[-1][1] = max(runs[-1][1], at + n - runs[-1][0])
        else:
            runs.append([at, n])
    return runs


def _pipeline(wplans: list, dev, key: str, n_workers: int, emit, sink=None) -> None:
    """Windowed file pipeline, double-buffered so file reads of windows w
    and w+1 and the output handling of window w-1 overlap the GPU work of
    window w:

        read files (thread pool, <=IO_CHUNK pread jobs) -> pinned -> H2D ->
        kernel(s) -> D2H -> pinned -> emit jobs (thread pool)

    wplans: [(step, read jobs (path, header, offset), src bytes, outs, dst
    bytes)] with step a _Step/_FusedStep. ``emit(o, view)`` runs on this
    thread and returns zero-argument jobs (file-range writes, host copies)
    that the write pool runs. With ``sink`` (one device address per window)
    the target shards go straight into device memory the caller keeps; the
    D2H then covers only the window's first d_at bytes (the atomic tensors
    of a fused resume; nothing for load). Data-dependent failures raise after their
    window syncs, so a failing window never reaches emit (torn output,
    ucp/convert.py:503)."""
    import time

    PIPE_TRACE.clear()
    if not wplans:
        return
    t_start = time.perf_counter()
    tr = {"read_wait_s": 0.0, "gpu_wait_s": 0.0, "emit_wait_s": 0.0, "emit_submit_s": 0.0}
    ms = max(w[2] for w in wplans)
    md = max(w[4] for w in wplans)
    h_src = [_STAGE.host_buf(f"{key}_src{i}", ms) for i in range(2)]
    if md or sink is None:
        h_dst = [_STAGE.host_buf(f"{key}_dst{i}", max(md, 1)) for i in range(2)]
        d_dst = [_STAGE.dev_buf(f"{key}_dst{i}", max(md, 1), dev) for i in range(2)]
    d_src = [_STAGE.dev_buf(f"{key}_src{i}", ms, dev) for i in range(2)]
    st = _status(dev)
    stream = torch.cuda.current_stream(dev)
    # one H2D stream per slot: each read job enqueues the H2D of its own
    # chunk as soon as the bytes land, so PCIe-in overlaps the file reads
    s_h2d = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    for s_ in s_h2d:  # after everything already queued on the caller's stream
        s_.wait_stream(stream)
    nthreads = _io_threads(n_workers)
    with ThreadPoolExecutor(nthreads) as rpool, ThreadPoolExecutor(nthreads) as wpool:

        def read_and_send(slot, path, file_off, at, n, send):
            codec.read_range_into(path, file_off, memoryview(h_src[slot].numpy())[at:at + n])
            if send:
                with torch.cuda.device(dev), torch.cuda.stream(s_h2d[slot]):
                    d_src[slot][at:at + n].copy_(h_src[slot][at:at + n], non_blocking=True)

        unsent: dict = {}

        def reads(w):
            # chunks below SEND_MIN are not sent by their job (a copy call
            # per small file costs more than it overlaps); they are coalesced
            # into few H2D copies once the window's reads are done
            slot, futs, rest = w % 2, [], []
            for path, hdr, at in wplans[w][1]:
                for c, n in _chunks(hdr.nbytes):
                    if n:
                        send = n >= SEND_MIN
                        futs.append(rpool.submit(read_and_send, slot, path, hdr.offset + c,
                                                 at + c, n, send))
                        if not send:
                            rest.append((at + c, n))
            unsent[w] = rest
            return futs

        def send_rest(w, slot):
            runs = _coalesce(unsent.pop(w), ALIGN_GAP)
            with torch.cuda.stream(s_h2d[slot]):
                for at, n in runs:
                    d_src[slot][at:at + n].copy_(h_src[slot][at:at + n], non_blocking=True)

        pending = {0: reads(0)}
        written: dict = {}
        h2d_ev: dict = {}
        kern_ev: dict = {}
        try:
            for w, (step, _, s_at, outs, d_at) in enumerate(wplans):
                slot = w % 2
                if w + 1 < len(wplans):
                    # start reading window w+1 before waiting for window w:
                    # h_src[(w+1)%2] is free once window w-1's H2D drained,
                    # d_src[(w+1)%2] once window w-1's kernels ran
                    if w >= 1:
                        h2d_ev.pop(w - 1).synchronize()
                        s_h2d[(w + 1) % 2].wait_event(kern_ev.pop(w - 1))
                    pending[w + 1] = reads(w + 1)
                t0 = time.perf_counter()
                for f in pending.pop(w):
                    f.result()
                tr["read_wait_s"] += time.perf_counter() - t0
                send_rest(w, slot)
                h2d_ev[w] = torch.cuda.Event()
                h2d_ev[w].record(s_h2d[slot])
                stream.wait_event(h2d_ev[w])
                st.reset(stream)
                dst_ptr = d_dst[slot].data_ptr() if (md or sink is None) else 0
                step.launch(d_src[slot].data_ptr(), dst_ptr, st, stream,
                            None if sink is None else sink[w])
                kern_ev[w] = torch.cuda.Event()
                kern_ev[w].record(stream)
                if sink is not None and d_at == 0:  # everything went to the sink
                    t0 = time.perf_counter()
                    kern_ev[w].synchronize()
                    tr["gpu_wait_s"] += time.perf_counter() - t0
                    step.check(st, d_src[slot].data_ptr(), dst_ptr, stream)
                    continue
                t0 = time.perf_counter()
                for f in written.pop(w - 2, ()):  # h_dst[slot] is free again
                    f.result()
                tr["emit_wait_s"] += time.perf_counter() - t0
                h_dst[slot][:d_at].copy_(d_dst[slot][:d_at], non_blocking=True)
                done = torch.cuda.Event()
                done.record(stream)
                t0 = time.perf_counter()
                done.synchronize()
                tr["gpu_wait_s"] += time.perf_counter() - t0
                step.check(st, d_src[slot].data_ptr(), d_dst[slot].data_ptr(), stream)
                ov = memoryview(h_dst[slot].numpy())
                t0 = time.perf_counter()
                written[w] = [wpool.submit(job) for o in outs for job in emit(o, ov)]
                tr["emit_submit_s"] += time.perf_counter() - t0
            t0 = time.perf_counter()
            for fs in written.values():
                for f in fs:
                    f.result()
            tr["emit_wait_s"] += time.perf_counter() - t0
        except BaseException:
            for fs in list(pending.values()) + list(written.values()):
                for f in fs:
                    f.cancel()
            raise
    tr["total_s"] = time.perf_counter() - t_start
    tr["windows"] = len(wplans)
    PIPE_TRACE.update(tr)


def _copy_jobs(host: np.ndarray, g_at: int, ov: memoryview, at: int, nb: int) -> list:
    """Jobs copying ov[at:at+nb] to host[g_at:g_at+nb] in IO_CHUNK pieces."""
    src = np.frombuffer(ov, dtype=np.uint8, count=nb, offset=at) if nb else None

    def job(c, n):
        def run():
            host[g_at + c:g_at + c + n] = src[c:c + n]
        return run

    return [job(c, n) for c, n in _chunks(nb, COPY_CHUNK)] if nb else []


# --------------------------------------------------------------------------- convert


def _mapper_phase(ckpt, spec: ModelSpec, cfg: ParallelConfig) -> dict:
    """Manifests, stray/missing files and headers of every rank dir
    (ucp/convert.py:86-107): {(param, kind): [(meta, path, header)]}."""
    units = defaultdict(list)
    names = {p.name for p in spec.params}
    for g in range(cfg.world_size):
        rank_dir = ckpt.rank_dir(g)
        _, records = codec.read_manifest(rank_dir)
        listed = {m.file for m in records}
        on_disk = {f for f in os.listdir(rank_dir) if f.endswith(".ucpt")}
        if on_disk - listed:
            raise ManifestError(
                f"{rank_dir}: stray tensor files not in manifest: {sorted(on_disk - listed)[:3]}")
        for meta in records:
            path = os.path.join(rank_dir, meta.file)
            if not os.path.isfile(path):
                raise ManifestError(f"{rank_dir}: manifest lists missing file {meta.file}")
            hdr = codec.read_header(path)
            if hdr.dtype is not DType.F32:
                raise ManifestError(f"{path}: expected f32 payload, got {hdr.dtype.name}")
            if tuple(hdr.shape) != tuple(meta.shape):
                raise ManifestError(f"{path}: shape {hdr.shape} disagrees with manifest {meta.shape}")
            if meta.param not in names:
                raise ManifestError(f"{path}: param {meta.param!r} not in model.json")
            units[(meta.param, meta.kind)].append((meta, path, hdr))
    missing = [p.name for p in spec.params if not any((p.name, k) in units for k in STATE_KINDS)]
    if missing:
        raise MissingFragmentError(f"no fragments at all for params {missing[:3]}")

    return units


def convert(src: str, out_dir: str, n_workers: int = 1, inner: int = 1,
            strict_replicate: bool = True, *, device=None,
            window_bytes: int = DEFAULT_WINDOW_BYTES) -> AtomicCheckpoint:
    """Distributed checkpoint -> atomic checkpoint (ucp/convert.py:422-563).
    Output bytes do not depend on n_workers/inner (they only size the file
    I/O thread pool)."""
    global INVOCATIONS
    INVOCATIONS += 1
    if n_workers < 1 or inner < 1:
        raise ValueError("n_workers and inner must be >= 1")
    ckpt = codec.load_checkpoint(src)
    spec, cfg = ckpt.spec, ckpt.cfg
    fingerprint = source_fingerprint(src)
    dev = require_device(device)
    codec.ensure_empty_dir(out_dir)

    units = _mapper_phase(ckpt, spec, cfg)

    def src_size(p):
        return sum(align_up(h.nbytes) for k in STATE_KINDS for _, _, h in units.get((p.name, k), ()))

    windows = _windows(list(spec.params), lambda p: src_size(p) + 3 * align_up(4 * p.numel),
                       window_bytes)
    # compile every window first: all metadata validation precedes any IO
    wplans = []
    for wparams in windows:
        tab = RunTable()
        jobs, s_at, a_at, outs = [], 0, 0, []
        for p in wparams:
            for kind in STATE_KINDS:
                items = units.get((p.name, kind))
                if not items:
                    raise MissingFragmentError(f"{p.name}.{kind}: no fragments arrived")
                frags = []
                for meta, path, hdr in items:
                    jobs.append((path, hdr, s_at))
                    frags.append((meta, s_at, hdr.numel))
                    s_at += align_up(hdr.nbytes)
                compile_union(tab, p, cfg, frags, a_at, strict_replicate)
                outs.append((p, kind, a_at))
                a_at += align_up(4 * p.numel)
        wplans.append((_Step(Program(tab, dev), True), jobs, s_at, outs, a_at))
    _pipeline(wplans, dev, "conv", n_workers, lambda o, ov: _write_atomic(out_dir, o, ov))

    with open(os.path.join(out_dir, codec.MODEL_JSON), "w") as f:
        f.write(spec_to_json(spec))
    codec.write_json(os.path.join(out_dir, UCP_META_JSON), {
        "format_version": FORMAT_VERSION, "step": ckpt.step, "metadata": ckpt.metadata,
        "source_config_sha256": fingerprint})
    return AtomicCheckpoint(out_dir, spec, ckpt.step, dict(ckpt.metadata), fingerprint)


# --------------------------------------------------------------------------- load


def _layer_groups(spec: ModelSpec) -> list:
    by_layer: dict = {}
    for p in spec.params:
        by_layer.setdefault(layer_of(spec, p), []).append(p)
    return sorted(by_layer.items())


def resident_bound_elements(spec: ModelSpec, dp: int) -> int:
    worst = 0
    for _, params in _layer_groups(spec):
        worst = max(worst, sum(3 * p.numel for p in params))
    return dp * worst


def _load_stats(atomic: AtomicCheckpoint, spec: ModelSpec, tgt: ParallelConfig,
                bypass: bool) -> LoadStats:
    """Logical read accounting with the reference's redundancy-bypass
    assignment (ucp/load.py:164-214); the GPU path reads each file once."""
    stats = LoadStats(bypass=bypass)
    stats.resident_bound = resident_bound_elements(spec, tgt.dp)
    stats.per_rank = {g: {"files_read": 0, "bytes_read": 0} for g in range(tgt.world_size)}
    stage_of = {layer: s for s, layers in
                enumerate(pp_layer_map(spec.n_layers, tgt.pp, tgt.pp_schedule)) for layer in layers}
    resident = peak = 0
    for layer, params in _layer_groups(spec):
        s = stage_of[layer]
        sized = sorted(((codec.payload_bytes_on_disk(atomic.param_file(p.name, k)), p, k)
                        for p in params for k in STATE_KINDS),
                       key=lambda x: (-x[0], x[1].name, x[2]))
        for t in range(tgt.tp):
            gkey = f"{s},{t}"
            stats.group_files_needed[gkey] = stats.group_files_needed.get(gkey, 0) + len(sized)
            members = [tgt.rank_of(s, t, d) for d in range(tgt.dp)]
            layer_res = 0
            for j, (nbytes, p, _) in enumerate(sized):
                for g in ([members[j % tgt.dp]] if bypass else members):
                    stats.files_read += 1
                    stats.bytes_read += nbytes
                    stats.group_files_read[gkey] = stats.group_files_read.get(gkey, 0) + 1
                    stats.per_rank[g]["files_read"] += 1
                    stats.per_rank[g]["bytes_read"] += nbytes
                layer_res += p.numel * tgt.dp
                resident += p.numel * tgt.dp
                peak = max(peak, resident)
            resident -= layer_res
    stats.peak_resident_elements = peak
    if peak > stats.resident_bound:
        raise CheckpointLayoutError(f"loader exceeded its memory bound: {peak} > {stats.resident_bound}")
    return stats


def load(atomic_root: str, tgt: ParallelConfig, dtype: DType = DType.F32, bypass: bool = True,
         *, device=None, window_bytes: int = DEFAULT_WINDOW_BYTES,
         keep_on_device: bool = False) -> LoadedWorld:
    """Materialise every shard of a target world from an atomic checkpoint
    (ucp/load.py:131-223). Weights are cast to dtype; moments stay f32.

    ``keep_on_device`` (extension): the shards stay in HBM as
    ``DeviceTensor`` (numpy on first ``.data`` access), written by the
    kernels straight into one device arena -- no D2H, no host copies; raises
    MemoryError when the world does not fit the device."""
    atomic = load_atomic(atomic_root)
    spec = atomic.spec
    validate_model_config(spec, tgt)
    info = ucp_info(spec, tgt)
    stats = _load_stats(atomic, spec, tgt, bypass)
    dev = require_device(device)

    by_unit = defaultdict(list)
    for g in range(tgt.world_size):
        for i, m in enumerate(info.records[g]):
            by_unit[(m.param, m.kind)].append((g, i, m))
    wdt = dtype

    def out_dtype(kind):
        return wdt if kind == "weight" else DType.F32

    def tgt_bytes(p):
        return sum(align_up(fragment_elems(p, tgt, m) * out_dtype(k).itemsize)
                   for k in STATE_KINDS for _, _, m in by_unit.get((p.name, k), ()))

    params = [p for _, ps in _layer_groups(spec) for p in ps]
    windows = _windows(params, lambda p: 3 * align_up(4 * p.numel) + tgt_bytes(p), window_bytes)
    wplans, outs_all, total = [], [], 0
    for wparams in windows:
        tab = RunTable()
        jobs, s_at, t_at, outs = [], 0, 0, []
        for p in wparams:
            for kind in STATE_KINDS:
                path = atomic.param_file(p.name, kind)
                hdr = codec.read_header(path)
                if hdr.dtype is not DType.F32:
                    raise CheckpointLayoutError(f"{path}: expected f32, got {hdr.dtype.name}")
                if tuple(hdr.shape) != tuple(p.shape):
                    raise ShapeError(f"{p.name}: expected {p.shape}, got {hdr.shape}")
                jobs.append((path, hdr, s_at))
                targets = []
                odt = out_dtype(kind)
                for g, i, m in by_unit.get((p.name, kind), ()):
                    n = fragment_elems(p, tgt, m)
                    targets.append((m, t_at))
                    o = (g, i, m, odt, t_at, n, fragment_shape(p, tgt, m), total)
                    outs.append(o)
                    outs_all.append(o)
                    total += align_up(n * odt.itemsize, 16)
                    t_at += align_up(n * odt.itemsize)
                compile_extract(tab, p, tgt, targets, s_at, odt)
                s_at += align_up(hdr.nbytes)
        wplans.append((_Step(Program(tab, dev), False), jobs, s_at, outs, t_at))
    filled = {}
    if keep_on_device:
        need = sum(w[4] for w in wplans)
        free, _ = torch.cuda.mem_get_info(dev)
        if need + (1 << 30) > free:
            raise MemoryError(f"target world needs {need} B of HBM, {free} B free")
        arena = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
        bases, b = [], 0
        for w in wplans:
            bases.append(b)
            b += w[4]
        _pipeline([(st_, jobs, s_at, [], 0) for st_, jobs, s_at, _, _ in wplans], dev, "load", 4,
                  None, sink=[arena.data_ptr() + x for x in bases])
        for w, base in zip(wplans, bases):
            for g, i, m, odt, at, n, shape, _ in w[3]:
                nb = n * odt.itemsize
                filled[(g, i)] = DeviceTensor(odt, tuple(shape), arena[base + at:base + at + nb])
    else:
        host = np.empty(max(total, 1), dtype=np.uint8)

        def emit(o, ov):
            _, _, _, odt, at, n, _, g_at = o
            return _copy_jobs(host, g_at, ov, at, n * odt.itemsize)

        _pipeline(wplans, dev, "load", 4, emit)
        for g, i, m, odt, at, n, shape, g_at in outs_all:
            arr = host[g_at:g_at + n * odt.itemsize].view(odt.storage).reshape(shape)
            filled[(g, i)] = Tensor(odt, tuple(shape), arr)
    shards = {g: [WorldShard(m, filled[(g, i)]) for i, m in enumerate(info.records[g])]
              for g in range(tgt.world_size)}
    return LoadedWorld(tgt, spec, atomic.step, dict(atomic.metadata), shards, stats)


# --------------------------------------------------------------------------- resume


def resume(src_root: str, tgt: ParallelConfig, scratch: str, n_workers: int = 1, inner: int = 1,
           dtype: DType = DType.F32, bypass: bool = True, *, device=None,
           fused: bool = True, window_bytes: int = DEFAULT_WINDOW_BYTES,
           keep_on_device: bool = False) -> LoadedWorld:
    """Reload a distributed checkpoint under tgt (ucp/load.py:231-281): lazy
    direct read when the layouts match, else convert into scratch + load.

    With ``fused`` (default) the convert + load pair runs as one pass over
    the source files: the fused kernel writes the atomic
    tensors (saved to ``scratch/atomic`` exactly as convert() would) and the
    target shards from the same registers, so the atomic tree is never read
    back. Observable results (world, stats, scratch tree, conversion count)
    equal the two-pass path. ``keep_on_device`` as for load(): the target
    shards stay in HBM (DeviceTensor); only the atomic tensors cross PCIe."""
    src = codec.load_checkpoint(src_root)
    validate_model_config(src.spec, tgt)
    before = INVOCATIONS
    if same_config(src.cfg, tgt):
        stats = LoadStats(bypass=bypass)
        stats.resident_bound = resident_bound_elements(src.spec, tgt.dp)
        stats.per_rank = {g: {"files_read": 0, "bytes_read": 0} for g in range(tgt.world_size)}
        shards = {}
        for g in range(tgt.world_size):
            rank_dir = src.rank_dir(g)
            _, records = codec.read_manifest(rank_dir)
            out = []
            for meta in records:
                path = os.path.join(rank_dir, meta.file)
                t = codec.read_tensor(path)
                nbytes = codec.payload_bytes_on_disk(path)
                stats.files_read += 1
                stats.bytes_read += nbytes
                stats.per_rank[g]["files_read"] += 1
                stats.per_rank[g]["bytes_read"] += nbytes
                if meta.kind == "weight" and dtype is not DType.F32:
                    t = cast(t, dtype)
                if keep_on_device:
                    d = torch.from_numpy(np.ascontiguousarray(t.data).reshape(-1).view(np.uint8))
                    t = DeviceTensor(t.dtype, t.shape, d.to(require_device(device)))
                out.append(WorldShard(meta, t))
            shards[g] = out
        stats.conversions_invoked = INVOCATIONS - before
        return LoadedWorld(tgt, src.spec, src.step, dict(src.metadata), shards, stats)
    os.makedirs(scratch, exist_ok=True)
    atomic_dir = os.path.join(scratch, "atomic")
    if fused:
        world = _resume_fused(src_root, atomic_dir, tgt, dtype, bypass, n_workers, device,
                              window_bytes, keep_on_device)
    else:
        convert(src_root, atomic_dir, n_workers=n_workers, inner=inner, device=device,
                window_bytes=window_bytes)
        world = load(atomic_dir, tgt, dtype=dtype, bypass=bypass, device=device,
                     window_bytes=window_bytes, keep_on_device=keep_on_device)
    world.stats.conversions_invoked = INVOCATIONS - before
    return world


def _resume_fused(src_root: str, atomic_dir: str, tgt: ParallelConfig, dtype: DType,
                  bypass: bool, n_workers: int, device, window_bytes: int,
                  keep_on_device: bool = False) -> LoadedWorld:
    """convert(src_root, atomic_dir) + load(atomic_dir, tgt) in one pass."""
    from .engine import XProgram
    from .plan import XRunTable, compile_fused

    global INVOCATIONS
    INVOCATIONS += 1  # this is a conversion (ucp/convert.py:435-436)
    ckpt = codec.load_checkpoint(src_root)
    spec, cfg = ckpt.spec, ckpt.cfg
    fingerprint = source_fingerprint(src_root)
    dev = require_device(device)
    codec.ensure_empty_dir(atomic_dir)
    units = _mapper_phase(ckpt, spec, cfg)
    validate_model_config(spec, tgt)
    info = ucp_info(spec, tgt)
    tgt_units = defaultdict(list)
    for g in range(tgt.world_size):
        for i, m in enumerate(info.records[g]):
            tgt_units[(m.param, m.kind)].append((g, i, m))

    def out_dtype(kind):
        return dtype if kind == "weight" else DType.F32

    def size(p):
        b = 0
        for k in STATE_KINDS:
            b += sum(align_up(h.nbytes) for _, _, h in units.get((p.name, k), ()))
            b += align_up(4 * p.numel)
            b += sum(align_up(fragment_elems(p, tgt, m) * out_dtype(k).itemsize)
                     for _, _, m in tgt_units.get((p.name, k), ()))
        return b

    wins, outs_all, total = [], [], 0
    for wparams in _windows(list(spec.params), size, window_bytes):
        fx, rc, rl = XRunTable(), RunTable(), RunTable()
        jobs, s_at, a_at, t_at, atoms, outs = [], 0, 0, 0, [], []
        for p in wparams:
            for kind in STATE_KINDS:
                items = units.get((p.name, kind))
                if not items:
                    raise MissingFragmentError(f"{p.name}.{kind}: no fragments arrived")
                frags = []
                for meta, path, hdr in items:
                    jobs.append((path, hdr, s_at))
                    frags.append((meta, s_at, hdr.numel))
                    s_at += align_up(hdr.nbytes)
                odt = out_dtype(kind)
                targets = []
                for g, i, m in tgt_units.get((p.name, kind), ()):
                    n = fragment_elems(p, tgt, m)
                    targets.append((m, t_at))
                    o = (g, i, m, odt, t_at, n, fragment_shape(p, tgt, m), total)
                    outs.append(o)
                    outs_all.append(o)
                    total += align_up(n * odt.itemsize, 16)
                    t_at += align_up(n * odt.itemsize)
                compile_fused(fx, rc, rl, p, cfg, frags, a_at, tgt, targets, odt, True)
                atoms.append((p, kind, a_at))
                a_at += align_up(4 * p.numel)
        wouts = [("a", o) for o in atoms] + [("t", o[:7] + (a_at + o[4],) + o[7:]) for o in outs]
        wins.append((_FusedStep(XProgram(fx, dev), Program(rc, dev), Program(rl, dev), a_at),
                     jobs, s_at, wouts, a_at + t_at))
    filled = {}
    if keep_on_device:
        # targets straight into one device arena; only the atomics go D2H
        t_sizes = [w[4] - w[0].atom_at for w in wins]
        need = sum(t_sizes)
        free, _ = torch.cuda.mem_get_info(dev)
        if need + (1 << 30) > free:
            raise MemoryError(f"target world needs {need} B of HBM, {free} B free")
        arena = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
        bases, b = [], 0
        for n in t_sizes:
            bases.append(b)
            b += n
        _pipeline([(st_, jobs, s_at, [o for o in wo if o[0] == "a"], st_.atom_at)
                   for st_, jobs, s_at, wo, _ in wins], dev, "res", n_workers,
                  lambda o, ov: _write_atomic(atomic_dir, o[1], ov),
                  sink=[arena.data_ptr() + x for x in bases])
        for w, base in zip(wins, bases):
            for tag, o in w[3]:
                if tag == "t":
                    g, i, m, odt, at, n, shape = o[:7]
                    filled[(g, i)] = DeviceTensor(
                        odt, tuple(shape), arena[base + at:base + at + n * odt.itemsize])
    else:
        host = np.empty(max(total, 1), dtype=np.uint8)

        def emit(o, ov):
            tag, o = o
            if tag == "a":
                return _write_atomic(atomic_dir, o, ov)
            _, _, _, odt, _, n, _, at, g_at = o
            return _copy_jobs(host, g_at, ov, at, n * odt.itemsize)

        _pipeline(wins, dev, "res", n_workers, emit)
    with open(os.path.join(atomic_dir, codec.MODEL_JSON), "w") as f:
        f.write(spec_to_json(spec))
    codec.write_json(os.path.join(atomic_dir, UCP_META_JSON), {
        "format_version": FORMAT_VERSION, "step": ckpt.step, "metadata": ckpt.metadata,
        "source_config_sha256": fingerprint})
    atomic = load_atomic(atomic_dir)
    stats = _load_stats(atomic, spec, tgt, bypass)
    if not keep_on_device:
        for g, i, m, odt, at, n, shape, g_at in outs_all:
            filled[(g, i)] = Tensor(
                odt, tuple(shape), host[g_at:g_at + n * odt.itemsize].view(odt.storage).reshape(shape))
    shards = {g: [WorldShard(m, filled[(g, i)]) for i, m in enumerate(info.records[g])]
              for g in range(tgt.world_size)}
    return LoadedWorld(tgt, spec, atomic.step, dict(atomic.metadata), shards, stats)


# --------------------------------------------------------------------------- save side


def init_state(spec: ModelSpec, seed: int, *, device=None) -> ModelState:
    """Deterministic f32 state generated on the GPU (ucp/models.py:230-244,
    generator ucp/tensor.py:116-184)."""
    from .synth import stream_base

    dev = require_device(device)
    states: dict = {}
    for p in spec.params:
        lead = spec.tied_leader(p.name)
        if lead != p.name:
            states[p.name] = states[lead]
            continue
        buf = torch.empty(max(3 * p.numel, 1), dtype=torch.float32, device=dev)
        for i, kind in enumerate(STATE_KINDS):
            gen_state(stream_base(seed, p.name, kind), 0, p.numel, kind == "v",
                      buf.data_ptr() + 4 * i * p.numel)
        host = buf[:3 * p.numel].cpu().numpy()
        ts = [Tensor(DType.F32, tuple(p.shape), host[i * p.numel:(i + 1) * p.numel].reshape(p.shape))
              for i in range(3)]
        states[p.name] = ParamState(*ts)
    return ModelState(spec, states, 0, {"loss_scale": 1.0, "iteration": 0})


def partition(state: ModelState, cfg: ParallelConfig, out_dir: str, workers: int = 1, *,
              device=None) -> codec.DistributedCheckpoint:
    """Write the distributed checkpoint of a consolidated state; the slicing
    is the load_scatter kernel under the source config
    (ucp/partition.py:125-174)."""
    spec = state.spec
    validate_model_config(spec, cfg)
    dev = require_device(device)
    codec.ensure_empty_dir(out_dir)
    codec.write_json(os.path.join(out_dir, codec.CONFIG_JSON),
                     codec.config_json_dict(cfg, state.step, state.metadata))
    with open(os.path.join(out_dir, codec.MODEL_JSON), "w") as f:
        f.write(spec_to_json(spec))
    recs = all_rank_records(spec, cfg)
    by_unit = defaultdict(list)
    for g in range(cfg.world_size):
        for m in recs[g]:
            by_unit[(m.param, m.kind)].append((g, m))
    files = []
    for p in spec.params:
        tab = RunTable()
        full = torch.empty(max(3 * p.numel, 1), dtype=torch.float32, device=dev)
        outs, at = [], 0
        for i, kind in enumerate(STATE_KINDS):
            data = np.ascontiguousarray(getattr(state.params[p.name], kind).data, dtype=np.float32)
            if p.numel:
                full[i * p.numel:(i + 1) * p.numel].copy_(torch.from_numpy(data.reshape(-1)))
            targets = []
            for g, m in by_unit.get((p.name, kind), ()):
                n = fragment_elems(p, cfg, m)
                targets.append((m, at))
                outs.append((g, m, at, n))
                at += align_up(4 * n)
            compile_extract(tab, p, cfg, targets, full.data_ptr() + 4 * i * p.numel, DType.F32)
        d_out = torch.empty(max(at, 1), dtype=torch.uint8, device=dev)
        _run(Program(tab, dev), False, 0, d_out.data_ptr(), dev)
        host = d_out.cpu().numpy()
        for g, m, o, n in outs:
            files.append((g, m, host[o:o + 4 * n]))
    for g in range(cfg.world_size):
        os.makedirs(os.path.join(out_dir, f"rank_{g}"), exist_ok=True)
    with ThreadPoolExecutor(max_workers=max(1, workers)) as pool:
        list(pool.map(lambda f: codec.write_raw(
            os.path.join(out_dir, f"rank_{f[0]}", f[1].file), DType.F32, f[1].shape,
            memoryview(f[2])), files))
    for g in range(cfg.world_size):
        codec.write_json(os.path.join(out_dir, f"rank_{g}", codec.MANIFEST),
                         codec.manifest_dict(cfg, g, recs[g]))
    return codec.DistributedCheckpoint(out_dir, cfg, spec, state.step, dict(state.metadata))


# --------------------------------------------------------------------------- in-memory reshard


HOST_WINDOW_BYTES = 400_000_000  # state bytes per window of the host-streamed reshard()


def reshard(spec: ModelSpec, src: ParallelConfig, tgt: ParallelConfig, shards: dict,
            dtype: DType = DType.F32, strict: bool = True, *, device=None,
            fused: bool = True) -> dict:
    """In-memory resume(): source fragments {g: [array per record of
    enumerate_rank_records(spec, src, g)]} -> target fragments {g: [array
    per record of enumerate_rank_records(spec, tgt, g)]} (weights cast to
    dtype), through pinned host staging and the fused convert+load kernel.
    CUDA-tensor fragments take the zero-copy device-to-device path
    (reshard.reshard_device) and come back as CUDA tensors.
    Equivalent to convert() then load() without the file system
    (ucp/load.py:276-281); raises the same exceptions."""
    from .reshard import ReshardPlan, reshard_device

    if any(_is_cuda(t) for v in shards.values() for t in v):
        # fragments already in HBM: zero-copy device-to-device reshard
        return reshard_device(spec, src, tgt, shards, dtype=dtype, strict=strict)
    dev = require_device(device)
    key = (spec_to_json(spec), format_config_string(src), getattr(src, "vocab_multiple", 1),
           format_config_string(tgt), getattr(tgt, "vocab_multiple", 1), dtype.name, strict,
           fused, str(dev))
    cache = _LOCAL.plans  # per thread: a plan's streams and device slots are not shared
    plan = cache.get(key)
    if plan is None:
        # small windows: packing, PCIe in, HBM work and PCIe out overlap with
        # little pipeline fill / drain (the e2e leg's 0.4 GB, bench.py)
        plan = ReshardPlan(spec, src, tgt, dtype=dtype, strict=strict, device=dev, fused=fused,
                           window_bytes=HOST_WINDOW_BYTES)
        cache.clear()  # keep one compiled plan (its device slots) per thread
        cache[key] = plan
    return plan.run_host(shards)


def consolidate_world(world: LoadedWorld) -> ModelState:
    """Rebuild the consolidated ModelState of a loaded world on the GPU: the
    union of every (param, kind) over the target layout (the role of
    ucp/oracle.py:213-226; here it is the convert kernel applied to
    in-memory shards). Weights must be f32 (bf16/f16 casts are lossy)."""
    spec, tgt = world.spec, world.cfg
    by_unit = defaultdict(list)
    for g in sorted(world.shards):
        for s in world.shards[g]:
            if s.tensor.dtype is not DType.F32:
                raise ShapeError(f"{s.meta.param}.{s.meta.kind}: consolidate needs f32 shards")
            # device-resident shards go to union() as CUDA tensors (zero copy)
            payload = s.tensor.device if isinstance(s.tensor, DeviceTensor) else s.tensor.data
            by_unit[(s.meta.param, s.meta.kind)].append(FragmentMsg(s.meta, payload))
    params = {}
    for p in spec.params:
        lead = spec.tied_leader(p.name)
        if lead != p.name and lead in params:
            params[p.name] = params[lead]
            continue
        ts = []
        for kind in STATE_KINDS:
            arr = union(p, tgt, by_unit.get((p.name, kind), []), strict=True)
            if _is_cuda(arr):
                arr = arr.cpu().numpy()
            ts.append(Tensor(DType.F32, tuple(p.shape), np.ascontiguousarray(arr)))
        params[p.name] = ParamState(*ts)
    return ModelState(spec, params, world.step, dict(world.metadata))

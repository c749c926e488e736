"""Whole-model reshard engine: convert (union) + load (extract) between two
layouts, in layer windows, on one GPU.

This is the in-memory form of the reference's ``resume()`` data path
(ucp/load.py:276-281 = convert ucp/convert.py:422-563 then load
ucp/load.py:131-223) without the file system: source fragments of every
source rank are laid out in one arena, grouped by window; each window runs
one ``ucp_convert_gather`` launch (source arena -> atomic window buffer) and
one ``ucp_load_scatter`` launch (atomic window -> target fragments of every
target rank). Windows are contiguous groups of parameters in spec order under
a byte budget (a LLaMA layer, the embedding, ...).

Modes:
* device-resident (``step_device``): the whole source arena lives in HBM;
  targets go to a window ring in HBM. This is what ``bench.py`` times as the
  device ``value``.
* host-streamed (``run_host`` / ``stream_host``): source windows are copied
  H2D from pinned memory on a copy stream, converted + loaded on the compute
  stream and copied D2H on a second copy stream, double-buffered, so PCIe in,
  HBM work and PCIe out overlap (north_star item 4). This is the end-to-end
  path a caller with host buffers uses.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from .engine import Program, Status, XProgram, align_up, gen_state, pinned_host, require_device
from .layout import all_rank_records, validate_model_config
from .plan import (
    RunTable,
    XRunTable,
    compile_extract,
    compile_fused,
    compile_union,
    fragment_elems,
    fragment_shape,
)
from .spec import STATE_KINDS, DType, ModelSpec, ParallelConfig, format_config_string
from .synth import stream_base


@dataclass
class Window:
    params: list
    src_frags: list = field(default_factory=list)   # (g, idx, meta, off, n)
    tgt_frags: list = field(default_factory=list)   # (g, idx, meta, off, n, dtype)
    atom: dict = field(default_factory=dict)        # (param, kind) -> off
    src_bytes: int = 0
    atom_bytes: int = 0
    tgt_bytes: int = 0
    src_base: int = 0    # offset of this window in the global source arena
    tgt_base: int = 0    # offset of this window in the global target arena
    conv: object = None  # Program (unfused mode: everything; fused mode: the rest)
    load: object = None
    synth: object = None
    fused: object = None  # XProgram (fused mode)
    tgt_chunks: list = field(default_factory=list)  # per home GPU: (offset, nbytes)


def make_windows(params: list, budget: int) -> list:
    """Contiguous groups of params (spec order) under a state-byte budget."""
    out, cur, acc = [], [], 0
    for p in params:
        s = 12 * p.numel
        if cur and acc + s > budget:
            out.append(Window(cur))
            cur, acc = [], 0
        cur.append(p)
        acc += s
    if cur:
        out.append(Window(cur))
    return out


def layout_windows(spec, src, tgt, windows, dtype, home_of=None, n_homes: int = 1) -> tuple:
    """Assign arena offsets (host only, no device): source fragments of every
    source rank, atomic tensors and target fragments of every target rank,
    grouped by window. With ``home_of`` (target rank -> home GPU) the target
    fragments of a window are ordered by home GPU so each window's target
    region is directly the send buffer of the all-to-all-v exchange
    (``tgt_chunks`` = per-home (offset, nbytes)). Returns (src_total,
    tgt_total)."""
    src_recs = all_rank_records(spec, src)
    tgt_recs = all_rank_records(spec, tgt)
    win_of = {p.name: i for i, w in enumerate(windows) for p in w.params}
    for g in range(src.world_size):
        for i, m in enumerate(src_recs[g]):
            w = win_of.get(m.param)
            if w is None:
                continue
            W = windows[w]
            n = fragment_elems(spec.param(m.param), src, m)
            W.src_frags.append((g, i, m, W.src_bytes, n))
            W.src_bytes += align_up(4 * n)
    order = list(range(tgt.world_size))
    if home_of is not None:
        order.sort(key=lambda g: (home_of[g], g))
    for W in windows:
        W.tgt_chunks = [[0, 0] for _ in range(n_homes)]
    for g in order:
        for i, m in enumerate(tgt_recs[g]):
            w = win_of.get(m.param)
            if w is None:
                continue
            W = windows[w]
            dt = dtype if m.kind == "weight" else DType.F32
            n = fragment_elems(spec.param(m.param), tgt, m)
            h = home_of[g] if home_of is not None else 0
            ch = W.tgt_chunks[h]
            if ch[1] == 0:
                ch[0] = W.tgt_bytes
            W.tgt_frags.append((g, i, m, W.tgt_bytes, n, dt))
            W.tgt_bytes += align_up(dt.itemsize * n)
            ch[1] = W.tgt_bytes - ch[0]
    sb = tb = 0
    for W in windows:
        for p in W.params:
            for k in STATE_KINDS:
                W.atom[(p.name, k)] = W.atom_bytes
                W.atom_bytes += align_up(4 * p.numel)
        W.src_base, W.tgt_base = sb, tb
        sb += W.src_bytes
        tb += W.tgt_bytes
    return sb, tb


class ReshardPlan:
    """Compiled convert+load of (a subset of) a model between two layouts."""

    def __init__(self, spec: ModelSpec, src: ParallelConfig, tgt: ParallelConfig,
                 dtype: DType = DType.F32, strict: bool = True, params=None, device=None,
                 window_bytes: int = 5 << 29, tile_bytes: int = 1 << 17, fused: bool = False,
                 materialize_atomic: bool = True, home_of=None, n_homes: int = 1,
                 peer=None, src_peer=None):
        validate_model_config(spec, src)
        validate_model_config(spec, tgt)
        self.spec, self.src, self.tgt, self.dtype, self.strict = spec, src, tgt, dtype, strict
        self.fused_mode, self.materialize = fused, materialize_atomic
        self.home_of, self.n_homes = home_of, n_homes
        # peer = (ExchangePlan, PeerBuffers): target fragments are written
        # straight into their home GPU's receive slot (absolute addresses)
        self.peer = peer
        # src_peer = dist.PeerSources: source fragments stay on their source
        # rank's GPU and are read at absolute (IPC-mapped) addresses
        self.src_peer = src_peer
        self.device = require_device(device)
        self.tile_bytes = tile_bytes
        names = None if params is None else set(params)
        self.params = [p for p in spec.params if names is None or p.name in names]
        self.windows = self._make_windows(window_bytes)
        self._layout()
        self._compile()
        self.status = Status(self.device)
        self.host_slots = 3  # device slots per direction of the host-streamed pipeline (3 > 2 by 6 % e2e)
        self._bufs = {}

    # ------------------------------------------------------------------ planning

    def _make_windows(self, budget: int) -> list:
        return make_windows(self.params, budget)

    def _layout(self) -> None:
        lay = layout_windows(self.spec, self.src, self.tgt, self.windows, self.dtype,
                             self.home_of, self.n_homes)
        self.src_total, self.tgt_total = lay
        self.max_src = max((W.src_bytes for W in self.windows), default=0)
        self.max_atom = max((W.atom_bytes for W in self.windows), default=0)
        self.max_tgt = max((W.tgt_bytes for W in self.windows), default=0)

    def _compile(self) -> None:
        self.bytes = {"R_c": 0, "W_c": 0, "R_l": 0, "W_l": 0}
        self.fused_bytes = {"R": 0, "W_atom": 0, "W_tgt": 0}
        self.n_fused_units = self.n_units = 0
        for W in self.windows:
            conv, load, synth = RunTable(), RunTable(), RunTable()
            fx = XRunTable()
            src_by_unit, tgt_by_unit = {}, {}
            for g, i, m, off, n in W.src_frags:
                if self.src_peer is not None:
                    off = self.src_peer.addr(g, i)
                src_by_unit.setdefault((m.param, m.kind), []).append((m, off, n))
            for g, i, m, off, n, dt in W.tgt_frags:
                if self.peer is not None:
                    exch, bufs = self.peer
                    w_idx, roff = exch.index_of(g, i)
                    off = bufs.slot(g % exch.world, w_idx) + roff
                tgt_by_unit.setdefault((m.param, m.kind), []).append((m, off))
            for p in W.params:
                for k in STATE_KINDS:
                    a = W.atom[(p.name, k)]
                    frags = src_by_unit.get((p.name, k), [])
                    dt = self.dtype if k == "weight" else DType.F32
                    tg = tgt_by_unit.get((p.name, k), [])
                    self.n_units += 1
                    if self.fused_mode:
                        self.n_fused_units += compile_fused(
                            fx, conv, load, p, self.src, frags, a, self.tgt, tg, dt, self.strict,
                            self.materialize)
                    else:
                        compile_union(conv, p, self.src, frags, a, self.strict)
                        compile_extract(load, p, self.tgt, tg, a, dt)
                    if self.src_peer is None:
                        compile_extract(synth, p, self.src, [(m, off) for m, off, _ in frags], a,
                                        DType.F32)
            W.conv = Program(conv, self.device, self.tile_bytes)
            W.load = Program(load, self.device, self.tile_bytes)
            W.synth = Program(synth, self.device, self.tile_bytes)
            W.fused = XProgram(fx, self.device, self.tile_bytes)
            self.fused_bytes["R"] += fx.src_bytes
            self.fused_bytes["W_atom"] += fx.atom_bytes
            self.fused_bytes["W_tgt"] += fx.dst_bytes
            self.bytes["R_c"] += conv.src_bytes
            self.bytes["W_c"] += conv.dst_bytes
            self.bytes["R_l"] += load.src_bytes
            self.bytes["W_l"] += load.dst_bytes

    # ------------------------------------------------------------------ sizes

    @property
    def state_bytes(self) -> int:
        """S = 12 B x numel (fp32 weight + Adam m + v) of the planned params."""
        return sum(12 * p.numel for p in self.params)

    @property
    def hbm_bytes(self) -> int:
        """Algorithmic HBM traffic of one step: R_c + W_c + R_l + W_l of the
        unfused runs plus R + W_atom + W_tgt of the fused ones."""
        return sum(self.bytes.values()) + sum(self.fused_bytes.values())

    @property
    def n_launches(self) -> int:
        """Kernel launches of one step (one per non-empty tile class)."""
        return sum(W.conv.n_launches + W.load.n_launches + W.fused.n_launches
                   for W in self.windows)

    # ------------------------------------------------------------------ buffers

    def buf(self, key: str, nbytes: int) -> torch.Tensor:
        b = self._bufs.get(key)
        if b is None or b.numel() < nbytes:
            self._bufs.pop(key, None)
            b = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
            self._bufs[key] = b
        return b

    def free(self) -> None:
        self._bufs.clear()

    # ------------------------------------------------------------------ device-resident

    def synthesize(self, seed: int = 7, stream=None) -> torch.Tensor:
        """Generate init_state(spec, seed) window by window on the GPU and
        partition it under the source config into the resident source arena
        (ucp/models.py:230-244 + ucp/partition.py:125-148)."""
        arena = self.buf("src_arena", self.src_total)
        atom = self.buf("atom", self.max_atom)
        for W in self.windows:
            self.gen_atomic(W, atom, seed, stream)
            W.synth.launch(False, atom.data_ptr(), arena.data_ptr() + W.src_base, self.status, stream)
        return arena

    def gen_atomic(self, W: Window, atom: torch.Tensor, seed: int, stream=None) -> None:
        for p in W.params:
            lead = self.spec.tied_leader(p.name)
            for k in STATE_KINDS:
                gen_state(stream_base(seed, lead, k), 0, p.numel, k == "v",
                          atom.data_ptr() + W.atom[(p.name, k)], stream)

    def step_device(self, stream=None, events=None) -> None:
        """One device-resident reshard of every window: inputs already in the
        source arena, targets into a two-slot HBM ring. events[i] (optional)
        gets 4 CUDA events around the fused / convert / load launches."""
        arena = self._bufs["src_arena"] if self.src_peer is None else None
        atom = self.buf("atom", self.max_atom)
        ring = [self.buf("tgt0", self.max_tgt), self.buf("tgt1", self.max_tgt)]
        for i, W in enumerate(self.windows):
            ev = events[i] if events is not None else None
            src_ptr = 0 if arena is None else arena.data_ptr() + W.src_base
            if ev:
                ev[0].record(stream)
            tgt_ptr = 0 if self.peer is not None else ring[i % 2].data_ptr()
            W.fused.launch(src_ptr, atom.data_ptr(), tgt_ptr, self.status, stream)
            if ev:
                ev[1].record(stream)
            W.conv.launch(True, src_ptr, atom.data_ptr(), self.status, stream)
            if ev:
                ev[2].record(stream)
            W.load.launch(False, atom.data_ptr(), tgt_ptr, self.status, stream)
            if ev:
                ev[3].record(stream)

    def step_device_homed(self, exch, group=None, stream=None, comm_stream=None,
                          events=None, comm=None, xevents=None) -> None:
        """Rank-homed variant of ``step_device`` (north_star item 3): after
        window w's reshard launches, its target region (ordered by home GPU,
        see ``layout_windows``) is exchanged with one all-to-all-v over NCCL
        on ``comm_stream`` while window w+1 computes. Window w+2 reuses the
        ring slot only after the exchange of w has drained it. xevents[w]
        (optional): two CUDA events recorded on ``comm_stream`` around window
        w's all-to-all-v (the exchange stage's own time)."""
        import torch.distributed as dist

        stream = stream or torch.cuda.current_stream(self.device)
        comm_stream = comm_stream or torch.cuda.Stream(self.device)
        arena = self._bufs["src_arena"]
        atom = self.buf("atom", self.max_atom)
        ring = [self.buf("tgt0", self.max_tgt), self.buf("tgt1", self.max_tgt)]
        rmax = max((exch.recv_bytes(w) for w in range(exch.n_windows)), default=0)
        recv = [self.buf("rcv0", rmax), self.buf("rcv1", rmax)]
        done = [None, None]
        for w in range(exch.n_windows):
            slot = w % 2
            if done[slot] is not None:
                stream.wait_event(done[slot])
            W = self.windows[w] if w < len(self.windows) else None
            ev = events[w] if events is not None and w < len(events) else None
            if ev:
                ev[0].record(stream)
            if W is not None:
                src_ptr = arena.data_ptr() + W.src_base
                W.fused.launch(src_ptr, atom.data_ptr(), ring[slot].data_ptr(), self.status, stream)
                W.conv.launch(True, src_ptr, atom.data_ptr(), self.status, stream)
                W.load.launch(False, atom.data_ptr(), ring[slot].data_ptr(), self.status, stream)
            ready = torch.cuda.Event()
            ready.record(stream)
            if ev:
                ev[1].record(stream)
                ev[2].record(stream)
                ev[3].record(stream)
            sizes = [nb for _, nb in exch.send[w]]
            xev = xevents[w] if xevents is not None and w < len(xevents) else None
            with torch.cuda.stream(comm_stream):
                comm_stream.wait_event(ready)
                if xev:
                    xev[0].record(comm_stream)
                if comm is not None:  # libucp_b200_comm.so: grouped ncclSend/ncclRecv
                    comm.alltoallv(ring[slot].data_ptr(), sizes, recv[slot].data_ptr(),
                                   exch.recv[w], comm_stream.cuda_stream)
                else:
                    dist.all_to_all_single(recv[slot][:exch.recv_bytes(w)],
                                           ring[slot][:sum(sizes)], exch.recv[w], sizes,
                                           group=group)
                if xev:
                    xev[1].record(comm_stream)
                fin = torch.cuda.Event()
                fin.record(comm_stream)
            done[slot] = fin
        for fin in done:
            if fin is not None:
                stream.wait_event(fin)

    def step_windowed(self, seed: int = 7, stream=None, events=None) -> None:
        """Reshard of a state larger than HBM: each window's
        source fragments are synthesised into a window-sized arena just
        before its launches (outside the events), then resharded exactly as
        in ``step_device``. events[i] brackets window i's reshard launches
        only, so summing them gives device-resident kernel time per step."""
        arena = self.buf("src_win", self.max_src)
        atom = self.buf("atom", self.max_atom)
        ring = [self.buf("tgt0", self.max_tgt), self.buf("tgt1", self.max_tgt)]
        for i, W in enumerate(self.windows):
            self.gen_atomic(W, atom, seed, stream)
            W.synth.launch(False, atom.data_ptr(), arena.data_ptr(), self.status, stream)
            ev = events[i] if events is not None else None
            if ev:
                ev[0].record(stream)
            W.fused.launch(arena.data_ptr(), atom.data_ptr(), ring[i % 2].data_ptr(), self.status,
                           stream)
            if ev:
                ev[1].record(stream)
            W.conv.launch(True, arena.data_ptr(), atom.data_ptr(), self.status, stream)
            if ev:
                ev[2].record(stream)
            W.load.launch(False, atom.data_ptr(), ring[i % 2].data_ptr(), self.status, stream)
            if ev:
                ev[3].record(stream)

    def check(self) -> None:
        """Raise the reference exception for any data-dependent failure seen
        since the last status reset (replica mismatch / nonzero pad). The
        status word is shared by all launches, so a failing window is
        located by re-running the convert launches one at a time."""
        first, _ = self.status.read()
        if first == (1 << 64) - 1:
            return
        arena = self._bufs["src_arena"] if self.src_peer is None else None
        for W in self.windows:
            self._locate(W, 0 if arena is None else arena.data_ptr() + W.src_base)
        raise RuntimeError("reshard reported a failure that did not reproduce")

    def _locate(self, W: Window, src_ptr: int) -> None:
        """Re-run the source-reading launches of one window with a fresh
        status word and raise the reference exception if one fails."""
        from .engine import describe_failure

        atom = self.buf("atom", self.max_atom)
        # rank-homed targets are absolute peer addresses (base 0)
        tgt_ptr = 0 if self.peer is not None else self.buf("tgt0", self.max_tgt).data_ptr()
        for prog in (W.fused, W.conv):
            self.status.reset()
            if prog is W.fused:
                prog.launch(src_ptr, atom.data_ptr(), tgt_ptr, self.status)
            else:
                prog.launch(True, src_ptr, atom.data_ptr(), self.status)
            torch.cuda.synchronize(self.device)
            f, _ = self.status.read()
            if f != (1 << 64) - 1:
                raise describe_failure(prog, f >> 32, f & 0xFFFFFFFF, src_ptr, (W.conv,))

    # ------------------------------------------------------------------ host-streamed

    _PACK_CHUNK = 16 << 20  # bytes per host copy job: big fragments spread over the threads

    def _pack_jobs(self, shards: dict) -> list:
        """Validated copy jobs [(arena byte offset, uint8 view)] per window, in
        window order, big fragments cut into _PACK_CHUNK pieces."""
        from ._errors import ShapeError

        per_win = []
        for W in self.windows:
            jobs = []
            for g, i, m, off, n in W.src_frags:
                a = np.ascontiguousarray(shards[g][i], dtype=np.float32).reshape(-1)
                if a.size != n:
                    raise ShapeError(f"rank {g} {m.param}.{m.kind}: {a.size} elements, want {n}")
                b = a.view(np.uint8)
                at = W.src_base + off
                for c in range(0, max(b.size, 1), self._PACK_CHUNK):
                    jobs.append((at + c, b[c:c + self._PACK_CHUNK]))
            per_win.append(jobs)
        return per_win

    def _pack_pool(self, threads: int = 16):
        pool = getattr(self, "_pool", None)
        if pool is None:
            from concurrent.futures import ThreadPoolExecutor

            pool = self._pool = ThreadPoolExecutor(max(1, threads), thread_name_prefix="ucp-pack")
        return pool

    def pack_host(self, shards: dict, pinned: torch.Tensor | None = None,
                  threads: int = 16) -> torch.Tensor:
        """Copy {g: [array per source record]} into a pinned source arena
        (the plan's own, reused across calls, unless ``pinned`` is given);
        the copies run on ``threads`` host threads (numpy releases the GIL)."""
        host = pinned if pinned is not None else self._pinned("src", self.src_total)
        hv = host.numpy()
        jobs = [j for w in self._pack_jobs(shards) for j in w]

        def copy(job):
            at, b = job
            hv[at:at + b.size] = b

        if threads > 1 and len(jobs) > 1:
            list(self._pack_pool(threads).map(copy, jobs))
        else:
            for j in jobs:
                copy(j)
        return host

    def _pinned(self, key: str, nbytes: int) -> torch.Tensor:
        """A grow-only pinned host buffer owned by the plan."""
        h = getattr(self, "_host_bufs", None)
        if h is None:
            h = self._host_bufs = {}
        b = h.get(key)
        if b is None or b.numel() < nbytes:
            h.pop(key, None)
            b = h[key] = pinned_host(nbytes)
        return b

    def _target_arena(self) -> torch.Tensor:
        """Pinned host target arena for run_host: the previous call's is
        reused once no array it returned is alive any more (they are views
        of it), else a fresh one is allocated."""
        prev = getattr(self, "_tgt_views", None)
        if prev is not None and prev[1]() is None:
            return prev[0]
        return pinned_host(self.tgt_total)

    def stream_host(self, host_src: torch.Tensor, host_tgt: torch.Tensor | None, windows=None,
                    streams=None, slots: int | None = None,
                    dev_tgt: torch.Tensor | None = None, ready=None) -> None:
        """Pinned host source arena -> device -> pinned host target arena,
        multi-buffered (``slots`` device slots per direction, default
        ``self.host_slots``) over windows on three streams. Asynchronous:
        the caller synchronises (the last event is on the D2H stream).

        ``dev_tgt`` (a device byte tensor of ``tgt_total`` bytes, host_tgt
        None): the target fragments stay in HBM at their arena offsets --
        a resume straight onto the GPU; only the sources cross PCIe.

        ``ready(i)``, if given, is called (and must return) before window
        i's H2D is enqueued: the host producer of window i's source bytes
        (run_host's packing threads) overlaps the transfers of the windows
        before it."""
        wins = self.windows if windows is None else windows
        s_in, s_cmp, s_out = streams or self.host_streams()
        ns = max(2, slots or self.host_slots)
        dsrc = [self.buf(f"ssrc{j}", self.max_src) for j in range(ns)]
        dtgt = [self.buf(f"stgt{j}", self.max_tgt) for j in range(ns)] if dev_tgt is None else None
        atom = self.buf("atom", self.max_atom)
        # the caller's stream first: work it queued before this call (the
        # status reset, writes into host_src) must precede our copies and
        # kernels -- the side streams do not synchronise with it implicitly
        cur = torch.cuda.current_stream(self.device)
        for s_ in (s_in, s_cmp, s_out):
            if s_ is not cur:
                s_.wait_stream(cur)
        # buffers are reused across calls: the first H2D must not overwrite a
        # source slot still being read, the first kernel must not overwrite a
        # target slot still being copied out
        s_in.wait_stream(s_cmp)
        s_cmp.wait_stream(s_out)
        ev_in = [torch.cuda.Event() for _ in wins]
        ev_cmp = [torch.cuda.Event() for _ in wins]
        ev_out = [torch.cuda.Event() for _ in wins]
        for i, W in enumerate(wins):
            slot = i % ns
            if ready is not None:
                ready(i)
            with torch.cuda.stream(s_in):
                if i >= ns:
                    s_in.wait_event(ev_cmp[i - ns])
                dsrc[slot][:W.src_bytes].copy_(host_src[W.src_base:W.src_base + W.src_bytes],
                                               non_blocking=True)
                ev_in[i].record(s_in)
            s_cmp.wait_event(ev_in[i])
            if i >= ns:
                s_cmp.wait_event(ev_out[i - ns])
            tptr = (dtgt[slot].data_ptr() if dev_tgt is None
                    else dev_tgt.data_ptr() + W.tgt_base)
            W.fused.launch(dsrc[slot].data_ptr(), atom.data_ptr(), tptr, self.status, s_cmp)
            W.conv.launch(True, dsrc[slot].data_ptr(), atom.data_ptr(), self.status, s_cmp)
            W.load.launch(False, atom.data_ptr(), tptr, self.status, s_cmp)
            ev_cmp[i].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_cmp[i])
                if dev_tgt is None:
                    host_tgt[W.tgt_base:W.tgt_base + W.tgt_bytes].copy_(
                        dtgt[slot][:W.tgt_bytes], non_blocking=True)
                ev_out[i].record(s_out)
        return ev_out[-1] if wins else None

    def unpack_host(self, host_tgt: torch.Tensor) -> dict:
        """{g: [array per target record, canonical order]} views of the host
        target arena."""
        import weakref

        hv = host_tgt.numpy()
        self._tgt_views = (host_tgt, weakref.ref(hv))
        out: dict = {}
        for W in self.windows:
            for g, i, m, off, n, dt in W.tgt_frags:
                at = W.tgt_base + off
                shape = fragment_shape(self.spec.param(m.param), self.tgt, m)
                out.setdefault(g, {})[i] = hv[at:at + dt.itemsize * n].view(dt.storage).reshape(shape)
        return {g: [d[i] for i in sorted(d)] for g, d in out.items()}

    def run_pinned(self, host_src: torch.Tensor, host_tgt: torch.Tensor | None, streams=None,
                   status_out: torch.Tensor | None = None, sync: bool = True,
                   dev_tgt: torch.Tensor | None = None, ready=None) -> None:
        """Public zero-copy entry: pinned host source arena (``pack_host``
        layout) -> H2D -> fused convert+load -> D2H into the pinned host
        target arena (``unpack_host`` layout), double-buffered over windows.

        The call's result is the device status word: it is copied to
        ``status_out`` (pinned int64[2]) on the D2H stream after the last
        window. With ``sync`` the call waits and raises the reference's
        exception on a data-dependent failure (ReplicateMismatchError,
        PaddingError, ...); without it the caller checks ``status_out``
        later with ``check_status_word``."""
        streams = streams or self.host_streams()
        self.stream_host(host_src, host_tgt, None, streams, dev_tgt=dev_tgt, ready=ready)
        if status_out is not None:
            with torch.cuda.stream(streams[2]):
                status_out.copy_(self.status.t, non_blocking=True)
        if sync:
            streams[2].synchronize()
            if status_out is None or not self.status_ok(status_out):
                self._check_windows(host_src)

    def host_streams(self) -> tuple:
        """The plan's own (H2D, compute, D2H) streams: calls that do not pass
        streams reuse them, so back-to-back unsynchronised calls are ordered
        against each other (device slots are reused across calls)."""
        if getattr(self, "_host_streams", None) is None:
            self._host_streams = tuple(torch.cuda.Stream(self.device) for _ in range(3))
        return self._host_streams

    @staticmethod
    def status_ok(word: torch.Tensor) -> bool:
        return int(word.numpy().view(np.uint64)[0]) == (1 << 64) - 1

    def run_host(self, shards: dict) -> dict:
        """End-to-end in-memory reshard of host arrays; returns target arrays
        per rank in canonical record order. Packing into the pinned arena is
        pipelined with the transfers: the host threads copy window by window
        (in window order) while the streams move and reshard the windows
        already packed."""
        host_src = self._pinned("src", self.src_total)
        jobs = self._pack_jobs(shards)  # validates every fragment before any work
        host_tgt = self._target_arena()
        hv = host_src.numpy()

        def copy(job):
            at, b = job
            hv[at:at + b.size] = b

        pool = self._pack_pool()
        futs = [[pool.submit(copy, j) for j in w] for w in jobs]

        def ready(i):
            for f in futs[i]:
                f.result()

        self.status.reset()
        try:
            self.run_pinned(host_src, host_tgt, ready=ready)
        finally:
            for w in futs:  # never leave copies running into a reused arena
                for f in w:
                    f.cancel() or f.exception()
        return self.unpack_host(host_tgt)

    def _check_windows(self, host_src=None) -> None:
        first, _ = self.status.read()
        if first == (1 << 64) - 1:
            return
        dsrc = self.buf("chk_src", self.max_src)
        for W in self.windows:
            if host_src is None:
                break
            dsrc[:W.src_bytes].copy_(host_src[W.src_base:W.src_base + W.src_bytes])
            self._locate(W, dsrc.data_ptr())
        raise RuntimeError("reshard reported a failure that did not reproduce")

    # ------------------------------------------------------------------ verification

    def verify(self, seed: int = 7, windowed: bool = False) -> dict:
        """Full-size, size-independent parity check on the device (outside
        any timed region), for states synthesised with ``synthesize(seed)``:

        1. convert(partition_src(X)) == X bit for bit, where X is the
           generator state (the reference's own round-trip identity,
           SPEC acceptance 1); skipped for fused units that do not
           materialise the atomic tensor;
        2. convert_tgt(load(atomic)) == X: the materialised target fragments
           are a valid checkpoint of the same state under the target layout
           (needs f32 targets; bf16/f16 weights are lossy by design).

        ``windowed``: for states larger than HBM, each window's sources are
        synthesised into a window-sized arena first (as ``step_windowed``).

        Returns {"windows": n, "atomic_ok": bool|None, "target_ok": bool|None}."""
        from .engine import compare

        arena = self.buf("src_win", self.max_src) if windowed else self._bufs["src_arena"]
        atom = self.buf("atom", self.max_atom)
        ref = self.buf("atom_ref", self.max_atom)
        back = self.buf("atom_back", self.max_atom)
        tgt = self.buf("tgt0", self.max_tgt)
        mism = torch.zeros(1, dtype=torch.int64, device=self.device)
        atomic_ok = True if (self.materialize or not self.fused_mode) else None
        target_ok = True if self.dtype is DType.F32 and self.peer is None else None
        for W in self.windows:
            self.status.reset()
            src_ptr = arena.data_ptr() + (0 if windowed else W.src_base)
            if windowed:
                self.gen_atomic(W, ref, seed)
                W.synth.launch(False, ref.data_ptr(), src_ptr, self.status)
            tgt_ptr = 0 if self.peer is not None else tgt.data_ptr()
            W.fused.launch(src_ptr, atom.data_ptr(), tgt_ptr, self.status)
            W.conv.launch(True, src_ptr, atom.data_ptr(), self.status)
            W.load.launch(False, atom.data_ptr(), tgt_ptr, self.status)
            if not windowed:
                self.gen_atomic(W, ref, seed)
            torch.cuda.synchronize(self.device)
            first, _ = self.status.read()
            if first != (1 << 64) - 1:
                self._locate(W, src_ptr)
            if atomic_ok:
                compare(atom.data_ptr(), ref.data_ptr(), W.atom_bytes, mism)
                torch.cuda.synchronize(self.device)
                if int(mism.item()) != -1:
                    atomic_ok = False
            if target_ok:
                self._reverse(W).launch(True, tgt.data_ptr(), back.data_ptr(), self.status)
                compare(back.data_ptr(), ref.data_ptr(), W.atom_bytes, mism)
                torch.cuda.synchronize(self.device)
                if int(mism.item()) != -1:
                    target_ok = False
        return {"windows": len(self.windows), "atomic_ok": atomic_ok, "target_ok": target_ok,
                "fused_units": self.n_fused_units, "units": self.n_units}

    def _reverse(self, W: Window) -> Program:
        rev = getattr(W, "_rev", None)
        if rev is None:
            tab = RunTable()
            by_unit = {}
            for g, i, m, off, n, dt in W.tgt_frags:
                by_unit.setdefault((m.param, m.kind), []).append((m, off, n))
            for p in W.params:
                for k in STATE_KINDS:
                    compile_union(tab, p, self.tgt, by_unit.get((p.name, k), []),
                                  W.atom[(p.name, k)], True)
            rev = W._rev = Program(tab, self.device, self.tile_bytes)
        return rev


# --------------------------------------------------------------------------- device to device


_TORCH_OF = {DType.F32: torch.float32, DType.BF16: torch.bfloat16, DType.F16: torch.float16}


_SRC_V, _TGT_V, _ATOM_V = 1 << 56, 1 << 57, 1 << 58  # virtual spaces of a d2d template
_D2D = threading.local()


def _rebind(v: np.ndarray, starts: np.ndarray, real: np.ndarray, lo: int = _SRC_V) -> np.ndarray:
    """Map virtual addresses (>= lo) inside fragment k, which starts at
    starts[k] (sorted), to real[k] + offset; other values (real scratch
    addresses, zeros) pass through."""
    v = v.astype(np.uint64, copy=True)
    mask = v >= np.uint64(lo)
    if mask.any():
        k = np.searchsorted(starts, v[mask], side="right") - 1
        v[mask] = real[k] + (v[mask] - starts[k])
    return v


class _D2DTemplate:
    """The compiled tables of one device-to-device reshard layout.

    Sources are compiled at virtual addresses (source fragment (g, i) at
    _SRC_V + offset, 256-B aligned) and re-bound to the caller's tensors;
    targets are compiled as offsets into ONE output arena, passed as the
    launches' dst_base, so a call with the same source tensors as the
    previous one patches and uploads nothing. Units that do not fuse
    (Partial mean / noise) use a scratch atomic sized to them alone. Valid
    for calls whose source pointers keep the template's 16-B phase (fresh
    torch allocations always do)."""

    def __init__(self, spec, src, tgt, dtype, strict, device, window_bytes, tile_bytes,
                 src_addr, tgt_addr, tgt_total):
        frags, targets = {}, {}
        for (g, i), (m, a, n) in src_addr.items():
            frags.setdefault((m.param, m.kind), []).append((m, a, n))
        for (g, i), (m, a) in tgt_addr.items():
            targets.setdefault((m.param, m.kind), []).append((m, a))
        self.tgt_total, self.device = tgt_total, device
        wins = make_windows(spec.params, window_bytes)
        # the atomic of a unit is compiled at a virtual address; only units
        # that do not fuse need real scratch, packed per window and bound
        # once the largest window's need is known
        built, need = [], 0
        for W in wins:
            fx, rc, rl = XRunTable(), RunTable(), RunTable()
            vstarts, offs, at = [], [], 0
            for p in W.params:
                for k in STATE_KINDS:
                    dt = dtype if k == "weight" else DType.F32
                    v = _ATOM_V + len(vstarts) * (1 << 40)
                    vstarts.append(v)
                    if compile_fused(fx, rc, rl, p, src, frags.get((p.name, k), []), v, tgt,
                                     targets.get((p.name, k), []), dt, strict, False):
                        offs.append(-1)
                    else:
                        offs.append(at)
                        at += align_up(4 * p.numel)
            need = max(need, at)
            built.append((fx, rc, rl, vstarts, offs))
        self.scratch = (torch.empty(need, dtype=torch.uint8, device=device) if need else None)
        base = self.scratch.data_ptr() if need else 0
        self.progs = []
        for fx, rc, rl, vstarts, offs in built:
            starts = np.array(vstarts, dtype=np.uint64)
            real = np.array([base + max(o, 0) for o in offs], dtype=np.uint64)
            progs = (XProgram(fx, device, tile_bytes), Program(rc, device, tile_bytes),
                     Program(rl, device, tile_bytes))
            for prog in progs[1:]:  # rest tables address the scratch atomics
                runs = prog.runs_host.copy()
                for f in ("src", "dst"):
                    runs[f] = _rebind(runs[f], starts, real, _ATOM_V)
                prog.set_tables(runs, _rebind(prog.aux_host, starts, real, _ATOM_V))
            for prog in progs:
                prog.virt = (prog.runs_host.copy(), prog.aux_host.copy())
            self.progs.append(progs)
        self.bound = None  # source addresses the device tables currently hold
        self.status = Status(device)
        self.word = torch.empty(2, dtype=torch.int64, pin_memory=True)

    def patch(self, starts: np.ndarray, real: np.ndarray) -> None:
        """Rebind every virtual source address to real[k] + (v - starts[k])
        and upload the tables (skipped when the sources did not move)."""
        if self.bound is not None and np.array_equal(self.bound, real):
            return
        for progs in self.progs:
            for prog in progs:
                runs0, aux0 = prog.virt
                runs = runs0.copy()
                for f in ("src", "dst"):
                    runs[f] = _rebind(runs0[f], starts, real)
                prog.set_tables(runs, _rebind(aux0, starts, real))
        self.bound = real

    def launch(self, arena: int, stream) -> None:
        for fused, conv, load in self.progs:
            fused.launch(0, 0, arena, self.status, stream)
            conv.launch(True, 0, 0, self.status, stream)
            load.launch(False, 0, arena, self.status, stream)

    def localise(self, arena: int, stream) -> Exception:
        """Re-run the source-reading launches one at a time (error path)."""
        from .engine import describe_failure

        for fused, conv, _ in self.progs:
            for prog in (fused, conv):
                self.status.reset(stream)
                if prog is fused:
                    prog.launch(0, 0, arena, self.status, stream)
                else:
                    prog.launch(True, 0, 0, self.status, stream)
                stream.synchronize()
                f, _ = self.status.read()
                if f != (1 << 64) - 1:
                    return describe_failure(prog, f >> 32, f & 0xFFFFFFFF, 0, (conv,))
        return RuntimeError("reshard reported a failure that did not reproduce")


class _D2DLayout:
    """Per (spec, layouts, dtype): records, fragment sizes, the output arena
    layout and the views to hand back (host-only, built once)."""

    def __init__(self, spec, src, tgt, dtype):
        src_recs, tgt_recs = all_rank_records(spec, src), all_rank_records(spec, tgt)
        self.src_recs = src_recs
        self.src_n = [[fragment_elems(spec.param(m.param), src, m) for m in src_recs[g]]
                      for g in range(src.world_size)]
        self.src_virt, vat = {}, _SRC_V
        for g in range(src.world_size):
            for i, m in enumerate(src_recs[g]):
                n = self.src_n[g][i]
                self.src_virt[(g, i)] = (m, vat, n)
                vat += align_up(4 * max(n, 1))
        self.starts = np.array([v[1] for v in self.src_virt.values()], dtype=np.uint64)
        self.tgt_off, self.views, at = {}, [], 0
        for g in range(tgt.world_size):
            row = []
            for i, m in enumerate(tgt_recs[g]):
                dt = dtype if m.kind == "weight" else DType.F32
                shape = tuple(fragment_shape(spec.param(m.param), tgt, m))
                n = 1
                for d in shape:
                    n *= int(d)
                self.tgt_off[(g, i)] = (m, at)
                stride, acc = [], 1
                for d in reversed(shape):
                    stride.append(acc)
                    acc *= int(d)
                row.append((dt, shape, tuple(reversed(stride)), at // dt.itemsize))
                at += align_up(dt.itemsize * max(n, 1))
            self.views.append(row)
        self.tgt_total = max(at, 256)


def reshard_device(spec: ModelSpec, src: ParallelConfig, tgt: ParallelConfig, shards: dict,
                   dtype: DType = DType.F32, strict: bool = True, *,
                   window_bytes: int = 5 << 29, tile_bytes: int = 1 << 17) -> dict:
    """Zero-copy device-to-device reshard: source fragments already in HBM
    ({g: [CUDA tensor per record of enumerate_rank_records(spec, src, g)]})
    -> CUDA target fragments {g: [tensor per target record]} (weights as
    torch.bfloat16 / float16 for a 16-bit dtype, holding exactly the
    reference cast's bits), views of one freshly allocated output arena.

    The descriptor tables address the caller's tensors by absolute device
    address and the targets by offset into the arena, so nothing is staged:
    one fused launch per window reads each source replica once, checks it
    and writes every target replica; the atomic tensor is not materialised
    (units that cannot fuse go through a small scratch). The compiled tables
    are cached per thread and layout (``_D2DTemplate``) and re-bound only
    when the source tensors move; the output views are built on the host
    while the kernels run, and the call waits on a pinned status word rather
    than the whole device. The per-thread cache keeps a reference to the
    last call's source tensors (that is how a repeated call recognises them
    without re-validating); ``api.release_staging()`` drops it. Raises the
    reference's exceptions (ReplicateMismatchError, PaddingError,
    ShapeError, ...)."""
    from ._errors import ShapeError
    from .spec import spec_to_json

    validate_model_config(spec, src)
    validate_model_config(spec, tgt)
    first = next((t for v in shards.values() for t in v), None)
    device = require_device(first.device if isinstance(first, torch.Tensor) else None)
    key = (spec_to_json(spec), format_config_string(src), getattr(src, "vocab_multiple", 1),
           format_config_string(tgt), getattr(tgt, "vocab_multiple", 1), dtype.name, strict,
           window_bytes, tile_bytes, str(device))
    # one cached layout per thread: its template, scratch and last sources
    st = getattr(_D2D, "state", None)
    if st is None or st["key"] != key:
        st = _D2D.state = {"key": key, "lay": _D2DLayout(spec, src, tgt, dtype), "tpl": None,
                           "last": None}
    lay = st["lay"]
    # validate the caller's fragments (skipped when they are the very tensors
    # of the previous call: the state holds them, so equal ids are the same
    # live objects)
    tensors = [t for g in range(src.world_size) for t in shards.get(g, [])]
    ids = [id(t) for t in tensors]
    if st["last"] is not None and st["last"][0] == ids:
        real = st["last"][1]
    else:
        for g in range(src.world_size):
            got = shards.get(g, [])
            if len(got) != len(lay.src_recs[g]):
                raise ShapeError(f"rank {g}: {len(got)} fragments, want {len(lay.src_recs[g])}")
            for i, t in enumerate(got):
                n = lay.src_n[g][i]
                if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32
                        and t.is_contiguous() and t.numel() == n and t.device == device):
                    m = lay.src_recs[g][i]
                    raise ShapeError(f"rank {g} {m.param}.{m.kind}: want a contiguous float32 CUDA "
                                     f"tensor of {n} elements on {device}")
        real = np.array([t.data_ptr() for t in tensors], dtype=np.uint64)
    st["last"] = (ids, real, tensors)
    # the cached template holds when every source keeps the virtual 16-B phase;
    # otherwise compile on the real addresses, uncached
    phase_ok = bool(((real - lay.starts) % np.uint64(16) == 0).all())
    if phase_ok:
        if st["tpl"] is None:
            st["tpl"] = _D2DTemplate(spec, src, tgt, dtype, strict, device, window_bytes,
                                     tile_bytes, lay.src_virt, lay.tgt_off, lay.tgt_total)
        tpl = st["tpl"]
        tpl.patch(lay.starts, real)
    else:
        src_addr = {k: (m, int(real[j]), n) for j, (k, (m, _, n)) in enumerate(lay.src_virt.items())}
        tpl = _D2DTemplate(spec, src, tgt, dtype, strict, device, window_bytes, tile_bytes,
                           src_addr, lay.tgt_off, lay.tgt_total)
    arena = torch.empty(lay.tgt_total, dtype=torch.uint8, device=device)
    stream = torch.cuda.current_stream(device)
    tpl.status.reset(stream)
    tpl.launch(arena.data_ptr(), stream)
    tpl.word.copy_(tpl.status.t, non_blocking=True)
    done = torch.cuda.Event()
    done.record(stream)
    # the output views are built while the kernels run
    typed = {DType.F32: arena.view(torch.float32)}
    if dtype is not DType.F32:
        typed[dtype] = arena.view(_TORCH_OF[dtype])
    out = {g: [typed[dt].as_strided(shape, stride, off) for dt, shape, stride, off in row]
           for g, row in enumerate(lay.views)}
    done.synchronize()
    if int(tpl.word[0]) != -1:
        raise tpl.localise(arena.data_ptr(), stream)
    return out

"""Multi-GPU partitioning of the reshard.

Every (param, kind) unit is independent, so the path shards by parameter:
ranks own parameters by LPT on bytes -- identical to the reference's
``plan_work`` LPT on numel (ucp/convert.py:328-341) because every state
tensor is f32. Convert needs no exchange (each rank is fed the source
fragments of the params it owns). Load is param-homed by default (the
reference world has no rank placement, ucp/load.py:69-76); when target ranks
are homed on GPUs (target rank g on GPU g mod N), the only exchange is one
all-to-all-v of the fragments whose owner GPU differs from their home GPU
(``exchange_plan`` + ``alltoallv``), over NCCL.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import torch

from .spec import ModelSpec


@dataclass(frozen=True)
class WorkPlan:
    groups: tuple
    loads: tuple

    def owner(self, param: str) -> int:
        for gi, grp in enumerate(self.groups):
            if param in grp:
                return gi
        raise KeyError(param)


def plan_work(spec: ModelSpec, n_groups: int) -> WorkPlan:
    """LPT: params by numel descending (ties by name), each to the lightest
    group (ties to the lowest index)."""
    if n_groups < 1:
        raise ValueError("n_groups must be >= 1")
    groups = [[] for _ in range(n_groups)]
    loads = [0] * n_groups
    for p in sorted(spec.params, key=lambda q: (-q.numel, q.name)):
        gi = min(range(n_groups), key=lambda i: (loads[i], i))
        groups[gi].append(p.name)
        loads[gi] += p.numel
    return WorkPlan(tuple(tuple(g) for g in groups), tuple(loads))


def owned_params(spec: ModelSpec, rank: int, world: int) -> list:
    return list(plan_work(spec, world).groups[rank])


def env_rank() -> tuple:
    """(rank, world_size, local_rank) from torchrun's environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init_process_group(backend: str = "nccl", force: bool = False):
    """Initialise torch.distributed from torchrun's environment when more
    than one rank runs (or ``force``: a 1-rank group, e.g. to exercise the
    collective path on one GPU)."""
    import torch.distributed as dist

    rank, world, local = env_rank()
    if (world > 1 or force) and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", rank=rank, world_size=world,
                                    device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend, rank=rank, world_size=world)
    return rank, world, local


def exchange_plan(frag_owner: list, frag_home: list, frag_bytes: list, world: int) -> list:
    """send[src][dst] byte counts of the rank-homed load exchange: fragment
    i moves from GPU frag_owner[i] to GPU frag_home[i] when they differ."""
    send = [[0] * world for _ in range(world)]
    for o, h, b in zip(frag_owner, frag_home, frag_bytes):
        if o != h:
            send[o][h] += b
    return send


def alltoallv(send_buf: torch.Tensor, send_counts: list, recv_counts: list, group=None) -> torch.Tensor:
    """One all-to-all-v of uint8 buffers (counts in bytes), NCCL on GPUs or
    gloo on CPU tensors."""
    import torch.distributed as dist

    recv = torch.empty(sum(recv_counts), dtype=torch.uint8, device=send_buf.device)
    dist.all_to_all_single(recv, send_buf, recv_counts, send_counts, group=group)
    return recv


@dataclass
class ExchangePlan:
    """Rank-homed load exchange for one rank (target rank g homed on GPU
    g mod world). Per window index w: this rank sends ``send[w][h]`` =
    (offset, nbytes) of its window-w target region to GPU h and receives
    ``recv[w][s]`` bytes from GPU s; ``index[(g, i)]`` = (w, byte offset in
    the window-w receive buffer) of every target record homed here."""

    rank: int
    world: int
    n_windows: int
    send: list
    recv: list
    index: dict
    all_index: dict = None
    max_recv: int = 0   # largest window receive buffer over all homes (same on every rank)

    def recv_bytes(self, w: int) -> int:
        return sum(self.recv[w])

    def index_of(self, g: int, i: int) -> tuple:
        """(window, offset in the home GPU's window receive buffer) of target
        record i of rank g, for ANY home (not only this rank)."""
        return self.all_index[(g, i)]


def build_exchange(spec: ModelSpec, src, tgt, world: int, rank: int, window_bytes: int,
                   dtype) -> ExchangePlan:
    """Deterministic on every rank: replays every rank's window layout
    (``reshard.layout_windows`` with home ordering) without touching a
    device."""
    from .reshard import layout_windows, make_windows

    home_of = [g % world for g in range(tgt.world_size)]
    plan = plan_work(spec, world)
    layouts = []
    for s in range(world):
        mine = set(plan.groups[s])
        wins = make_windows([p for p in spec.params if p.name in mine], window_bytes)
        layout_windows(spec, src, tgt, wins, dtype, home_of, world)
        layouts.append(wins)
    n_w = max(len(w) for w in layouts)
    send, recv, index, all_index = [], [], {}, {}
    max_recv = 0
    # receive-buffer offsets at every home: senders in rank order, each
    # sender's chunk in its own layout order
    for w in range(n_w):
        for h in range(world):
            at = 0
            for s in range(world):
                W = layouts[s][w] if w < len(layouts[s]) else None
                if W is None:
                    continue
                off, nb = W.tgt_chunks[h]
                for g, i, m, o, n, dt in W.tgt_frags:
                    if home_of[g] == h:
                        all_index[(g, i)] = (w, at + (o - off))
                at += nb
            max_recv = max(max_recv, at)
    for w in range(n_w):
        mine = layouts[rank][w] if w < len(layouts[rank]) else None
        send.append([tuple(mine.tgt_chunks[h]) if mine else (0, 0) for h in range(world)])
        row, at = [], 0
        for s in range(world):
            W = layouts[s][w] if w < len(layouts[s]) else None
            off, nb = W.tgt_chunks[rank] if W else (0, 0)
            row.append(nb)
            if W:
                for g, i, m, o, n, dt in W.tgt_frags:
                    if home_of[g] == rank:
                        index[(g, i)] = (w, at + (o - off))
            at += nb
        recv.append(row)
    return ExchangePlan(rank, world, n_w, send, recv, index, all_index, max_recv)


class PeerBuffers:
    """Receive buffers of every rank, mapped into this process with CUDA IPC
    so the reshard kernels store rank-homed target fragments straight into
    the home GPU's memory (NVLink / NVSwitch peer stores; no separate
    collective). ``n_slots`` ring slots of ``slot_bytes`` each; window w uses
    slot w % n_slots. Handles are exchanged once with all_gather_object over
    the default process group (gloo or NCCL)."""

    def __init__(self, slot_bytes: int, n_slots: int = 2, group=None):
        import ctypes

        import torch.distributed as dist

        from . import _native
        from ._errors import from_status

        lib = _native.lib()
        self.slot_bytes = max(int(slot_bytes), 256)
        self.n_slots = n_slots
        ptr = ctypes.c_void_p()
        rc = lib.ucp_dev_alloc(self.slot_bytes * n_slots, ctypes.byref(ptr))
        if rc:
            raise from_status(rc, "ucp_dev_alloc")
        self.local = ptr.value
        handle = (ctypes.c_ubyte * 64)()
        rc = lib.ucp_ipc_export(ctypes.c_void_p(self.local), handle)
        if rc:
            raise from_status(rc, "ucp_ipc_export")
        self.rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        handles = [None] * world
        dist.all_gather_object(handles, bytes(handle), group=group)
        self.bases, self._mapped = [], []
        for r, hb in enumerate(handles):
            if r == self.rank:
                self.bases.append(self.local)
                continue
            m = ctypes.c_void_p()
            h = (ctypes.c_ubyte * 64).from_buffer_copy(hb)
            rc = lib.ucp_ipc_open(h, ctypes.byref(m))
            if rc:
                raise from_status(rc, f"ucp_ipc_open(rank {r})")
            self.bases.append(m.value)
            self._mapped.append(m.value)

    def slot(self, home: int, w: int) -> int:
        """Device address (valid in this process) of home GPU's slot for window w."""
        return self.bases[home] + (w % self.n_slots) * self.slot_bytes

    def read_local(self, w: int, offset: int, nbytes: int):
        """Synchronous copy of this rank's received bytes (tests / checks)."""
        import ctypes

        import numpy as np

        from . import _native

        out = np.empty(nbytes, dtype=np.uint8)
        if nbytes:
            _native.lib().ucp_peek(ctypes.c_void_p(self.slot(self.rank, w) + offset),
                                   out.ctypes.data, nbytes)
        return out

    def close(self) -> None:
        import ctypes

        from . import _native

        lib = _native.lib()
        for m in self._mapped:
            lib.ucp_ipc_close(ctypes.c_void_p(m))
        self._mapped = []
        if self.local:
            lib.ucp_dev_free(ctypes.c_void_p(self.local))
            self.local = 0


def _ipc_arenas(nbytes: int, group=None) -> tuple:
    """cudaMalloc ``nbytes`` here, export it, all_gather every rank's handle
    and map the others: (local address, [address of rank r's arena valid in
    this process], [mapped addresses to close])."""
    import ctypes

    import torch.distributed as dist

    from . import _native
    from ._errors import from_status

    lib = _native.lib()
    ptr = ctypes.c_void_p()
    rc = lib.ucp_dev_alloc(max(int(nbytes), 256), ctypes.byref(ptr))
    if rc:
        raise from_status(rc, "ucp_dev_alloc")
    handle = (ctypes.c_ubyte * 64)()
    rc = lib.ucp_ipc_export(ctypes.c_void_p(ptr.value), handle)
    if rc:
        raise from_status(rc, "ucp_ipc_export")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    handles = [None] * world
    dist.all_gather_object(handles, bytes(handle), group=group)
    bases, mapped = [], []
    for r, hb in enumerate(handles):
        if r == rank:
            bases.append(ptr.value)
            continue
        m = ctypes.c_void_p()
        rc = lib.ucp_ipc_open((ctypes.c_ubyte * 64).from_buffer_copy(hb), ctypes.byref(m))
        if rc:
            raise from_status(rc, f"ucp_ipc_open(rank {r})")
        bases.append(m.value)
        mapped.append(m.value)
    return ptr.value, bases, mapped


def peer_source_layout(spec: ModelSpec, src, world: int) -> tuple:
    """({(g, i): (home GPU, byte offset in its arena)}, [arena bytes per
    GPU]) for source rank g's record i homed on GPU g mod world: ranks in
    order, records in manifest order, 256-B aligned. Identical on every
    process (no communication needed to address a peer's fragment)."""
    from .engine import align_up
    from .layout import all_rank_records
    from .plan import fragment_elems

    recs = all_rank_records(spec, src)
    offset, sizes = {}, [0] * world
    for g in range(src.world_size):
        h = g % world
        for i, m in enumerate(recs[g]):
            n = fragment_elems(spec.param(m.param), src, m)
            offset[(g, i)] = (h, sizes[h])
            sizes[h] += align_up(4 * n)
    return offset, sizes


class PeerSources:
    """Source fragments homed on their source rank's GPU (source rank g on
    GPU g mod world), one IPC-exported arena per GPU, every arena mapped in
    every process. The param owner's fused kernel then reads the fragments
    it needs straight from the home GPUs (NVLink / NVSwitch peer loads) and
    -- with PeerBuffers -- stores the targets straight into their home GPUs:
    the whole distributed reshard is one kernel per window and no
    collective. Layout is deterministic: on home h, source ranks g = h,
    h + world, ... in order, each rank's records in manifest order."""

    def __init__(self, spec: ModelSpec, src, group=None):
        import torch.distributed as dist

        from .layout import all_rank_records

        self.spec, self.src = spec, src
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.recs = all_rank_records(spec, src)
        self.offset, sizes = peer_source_layout(spec, src, self.world)
        self.nbytes = sizes[self.rank]
        self.local, self.bases, self._mapped = _ipc_arenas(self.nbytes, group)

    def addr(self, g: int, i: int) -> int:
        """Device address, valid in this process, of source rank g's record i."""
        h, off = self.offset[(g, i)]
        return self.bases[h] + off

    def fill(self, seed: int = 7) -> None:
        """Synthesize this GPU's homed fragments: init_state(spec, seed) one
        param at a time (ucp_gen_state) sliced under the source layout by the
        load kernels, written at their absolute local addresses."""
        import torch

        from .engine import Program, Status, gen_state, require_device
        from .plan import RunTable, compile_extract
        from .spec import STATE_KINDS, DType
        from .synth import stream_base

        dev = require_device(None)
        mine = {}
        for g in range(self.src.world_size):
            if g % self.world == self.rank:
                for i, m in enumerate(self.recs[g]):
                    mine.setdefault((m.param, m.kind), []).append((m, self.addr(g, i)))
        st = Status(dev)
        st.reset()
        for p in self.spec.params:
            lead = self.spec.tied_leader(p.name)
            full = torch.empty(max(p.numel, 1), dtype=torch.float32, device=dev)
            for k in STATE_KINDS:
                tg = mine.get((p.name, k))
                if not tg:
                    continue
                gen_state(stream_base(seed, lead, k), 0, p.numel, k == "v", full.data_ptr())
                tab = RunTable()
                compile_extract(tab, p, self.src, tg, full.data_ptr(), DType.F32)
                Program(tab, dev).launch(False, 0, 0, st)
                torch.cuda.synchronize(dev)  # `full` is reused for the next kind

    def close(self) -> None:
        import ctypes

        from . import _native

        lib = _native.lib()
        for m in self._mapped:
            lib.ucp_ipc_close(ctypes.c_void_p(m))
        self._mapped = []
        if self.local:
            lib.ucp_dev_free(ctypes.c_void_p(self.local))
            self.local = 0


class NcclComm:
    """libucp_b200_comm.so communicator (one per process / GPU). Rank 0's
    unique id is distributed over the default torch.distributed group."""

    def __init__(self, group=None):
        import ctypes

        import torch.distributed as dist

        from . import _native
        from ._errors import NativeUnavailableError

        lib = _native.comm_lib()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = (ctypes.c_char * 128)()
        if rank == 0 and lib.ucp_comm_unique_id(uid):
            raise NativeUnavailableError("ucp_comm_unique_id failed")
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = (ctypes.c_char * 128).from_buffer_copy(box[0])
        comm = ctypes.c_void_p()
        if lib.ucp_comm_init(world, rank, uid, ctypes.byref(comm)):
            raise NativeUnavailableError("ucp_comm_init failed")
        self.comm, self.world, self.rank = comm.value, world, rank

    def alltoallv(self, send_ptr: int, send_counts: list, recv_ptr: int, recv_counts: list,
                  stream_ptr: int) -> None:
        import ctypes

        import numpy as np

        from . import _native
        from ._errors import NativeUnavailableError

        sc = np.ascontiguousarray(send_counts, dtype=np.uint64)
        rc = np.ascontiguousarray(recv_counts, dtype=np.uint64)
        if _native.comm_lib().ucp_alltoallv(ctypes.c_void_p(self.comm), ctypes.c_void_p(send_ptr),
                                            sc.ctypes.data, ctypes.c_void_p(recv_ptr),
                                            rc.ctypes.data, ctypes.c_void_p(stream_ptr)):
            raise NativeUnavailableError("ucp_alltoallv failed")

    def close(self) -> None:
        import ctypes

        from . import _native

        if self.comm:
            _native.comm_lib().ucp_comm_destroy(ctypes.c_void_p(self.comm))
            self.comm = None

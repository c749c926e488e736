"""Device side: compiled programs, launches, status words, staging buffers.

PyTorch is used only as plumbing here (device memory, streams, events); all
data movement on the hot path goes through libucp_b200.so.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _native
from ._errors import NativeUnavailableError, PaddingError, ReplicateMismatchError, from_status
from .plan import NCLASS, OP_CHECKZERO, RunTable, expand_tiles

ALIGN = 256  # byte alignment of every fragment / atomic / target buffer


def align_up(n: int, a: int = ALIGN) -> int:
    return (n + a - 1) // a * a


def require_device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise NativeUnavailableError("no CUDA device: the reshard path has no CPU fallback")
    _native.lib()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    return torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise from_status(rc, what)


class _Table:
    """Runs (sorted by kernel class) + aux + scanned ucp_runtile array,
    resident on a device. No per-tile table: each CTA derives its tile
    (include/ucp_b200.h, ucp_runtile)."""

    def _upload(self, runs, aux, rt, info, order, device, run_bytes: int) -> None:
        self.runs_host, self.aux_host, self.rt_host, self.run_order = runs, aux, rt, order
        self.class_info = np.ascontiguousarray(info, dtype=np.int64)
        self.n_runs, self.n_tiles = len(runs), int(self.class_info[:NCLASS].sum())
        self.device = device
        blob = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).to(device)
        self._runs = blob(runs) if len(runs) else torch.zeros(run_bytes, dtype=torch.uint8, device=device)
        self._aux = blob(aux)
        rt_dev = rt.copy()
        rt_dev["first"] = 0xFFFFFFFF  # written by the device scan below
        self._rt = blob(rt_dev) if len(rt) else torch.zeros(16, dtype=torch.uint8, device=device)
        if len(rt):
            with torch.cuda.device(device):
                _check(_native.lib().ucp_runtile_scan(self._rt.data_ptr(),
                                                      self.class_info.ctypes.data,
                                                      stream_ptr(None)), "runtile_scan")

    def set_tables(self, runs: np.ndarray, aux: np.ndarray) -> None:
        """Replace the run / aux contents in place (same shapes and class
        order, e.g. addresses re-bound); the tile scan stays valid."""
        self.runs_host, self.aux_host = runs, aux
        if len(runs):
            self._runs.copy_(torch.from_numpy(np.ascontiguousarray(runs).view(np.uint8)),
                             non_blocking=False)
        self._aux.copy_(torch.from_numpy(np.ascontiguousarray(aux).view(np.uint8)))

    @property
    def tiles_host(self) -> np.ndarray:
        """Every tile as the kernels derive it (tests / diagnostics)."""
        return expand_tiles(self.runs_host, self.rt_host)

    @property
    def n_launches(self) -> int:
        return int((self.class_info[:NCLASS] > 0).sum())


class Program(_Table):
    """One ucp_convert_gather / ucp_load_scatter worth of runs on a device."""

    def __init__(self, table: RunTable, device: torch.device, tile_bytes: int = 1 << 17):
        runs, aux, rt, info, order = table.finish_classed(tile_bytes)
        self.units = table.units
        self.src_bytes, self.dst_bytes = table.src_bytes, table.dst_bytes
        self._upload(runs, aux, rt, info, order, device, 64)

    @property
    def bytes_moved(self) -> int:
        return self.src_bytes + self.dst_bytes

    def launch(self, gather: bool, src_base: int, dst_base: int, status: "Status",
               stream: torch.cuda.Stream | None = None) -> None:
        if self.n_tiles == 0:
            return
        lib = _native.lib()
        fn = lib.ucp_convert_gather if gather else lib.ucp_load_scatter
        rc = fn(self._runs.data_ptr(), self.n_runs, self._aux.data_ptr(), self._rt.data_ptr(),
                self.class_info.ctypes.data, ctypes.c_void_p(src_base),
                ctypes.c_void_p(dst_base), status.ptr, stream_ptr(stream))
        _check(rc, "convert_gather" if gather else "load_scatter")


class XProgram(_Table):
    """One ucp_reshard_fused launch: fused convert+load runs on a device."""

    def __init__(self, table, device: torch.device, tile_bytes: int = 1 << 17):
        runs, aux, rt, info, order = table.finish_classed(tile_bytes)
        self.units = table.units
        self.src_bytes, self.atom_bytes, self.dst_bytes = (table.src_bytes, table.atom_bytes,
                                                           table.dst_bytes)
        self._upload(runs, aux, rt, info, order, device, 64)

    @property
    def bytes_moved(self) -> int:
        return self.src_bytes + self.atom_bytes + self.dst_bytes

    def launch(self, src_base: int, atom_base: int, dst_base: int, status: "Status",
               stream: torch.cuda.Stream | None = None) -> None:
        if self.n_tiles == 0:
            return
        rc = _native.lib().ucp_reshard_fused(
            self._runs.data_ptr(), self.n_runs, self._aux.data_ptr(), self._rt.data_ptr(),
            self.class_info.ctypes.data, ctypes.c_void_p(src_base), ctypes.c_void_p(atom_base),
            ctypes.c_void_p(dst_base), status.ptr, stream_ptr(stream))
        _check(rc, "reshard_fused")


class Status:
    """Device status word (ucp_status) + host readback."""

    def __init__(self, device: torch.device):
        # constructed in the "ok" state (first = ~0, n_bad = 0): a word of
        # zeros would decode as "failure at run 0, element 0"
        self.t = torch.tensor([-1, 0], dtype=torch.int64, device=device)
        self.ptr = self.t.data_ptr()

    def reset(self, stream=None) -> None:
        _check(_native.lib().ucp_status_reset(self.ptr, stream_ptr(stream)), "status_reset")

    def read(self) -> tuple:
        v = self.t.cpu().numpy().view(np.uint64)
        return int(v[0]), int(v[1])

    def raise_if_bad(self, prog: Program, src_base: int) -> None:
        first, n_bad = self.read()
        if first == (1 << 64) - 1:
            return
        raise describe_failure(prog, first >> 32, first & 0xFFFFFFFF, src_base)


def _peek_f32(addr: int) -> int:
    """Read 4 bytes of device memory at an absolute address (error path only)."""
    out = np.zeros(1, dtype=np.uint32)
    rc = _native.lib().ucp_peek(ctypes.c_void_p(addr), out.ctypes.data, 4)
    return int(out[0]) if rc == 0 else 0xFFFFFFFF


def _unit_pad_error(progs, param: str, kind: str, src_base: int) -> Exception | None:
    """PaddingError if any pad-check (CHECKZERO) run of unit (param, kind)
    in ``progs`` sees a nonzero bit pattern, else None. The reference strips
    pads inside _collapse_dp, before it compares tp replicas
    (ucp/convert.py:192, :262-278), so a bad pad outranks a replica mismatch
    of the same unit; the status word orders runs by kernel class instead.
    Pads are < dp elements per tp rank, so this is a few tiny peeks."""
    for prog in progs:
        runs = prog.runs_host
        if "op" not in runs.dtype.names:
            continue
        for j in np.nonzero(runs["op"] == OP_CHECKZERO)[0]:
            r = runs[j]
            u = prog.units[int(r["tag"])]
            if (u.param, u.kind) != (param, kind):
                continue
            n = int(r["rows"]) * int(r["cols"])
            buf = np.zeros(n, dtype=np.uint32)
            if _native.lib().ucp_peek(ctypes.c_void_p(src_base + int(r["src"])), buf.ctypes.data,
                                      4 * n) != 0:
                continue
            bad = np.nonzero(buf)[0]
            if len(bad):
                return PaddingError(f"{param}.{kind}: nonzero pad tail (first bad element "
                                    f"{int(bad[0])})")
    return None


def describe_failure(prog: Program, run_idx: int, elem: int, src_base: int,
                     pad_progs=()) -> Exception:
    """Reference-style exception for a failing run (ucp/convert.py:165-171,
    :272-277, :127-128). ``pad_progs``: other tables of the same window
    that hold the unit's pad checks (the unfused rest of a fused window)."""
    r = prog.runs_host[run_idx]
    unit = prog.units[int(r["tag"])]
    where = f"{unit.param}.{unit.kind}"
    fused = "atom" in r.dtype.names
    if not fused and int(r["op"]) == OP_CHECKZERO:
        return PaddingError(f"{where}: nonzero pad tail (first bad element {elem})")
    pad = _unit_pad_error((prog, *pad_progs), unit.param, unit.kind, src_base)
    if pad is not None:
        return pad
    labels = unit.labels.get(int(prog.run_order[run_idx]))  # keyed by table index
    row, col = divmod(elem, int(r["cols"]))
    n_src, groups = int(r["n_src"]), 1 if fused else max(int(r["groups"]), 1)
    K = n_src // groups
    offs = [int(r["src"])] + [int(x) for x in prog.aux_host[int(r["aux"]):int(r["aux"]) + n_src - 1]]
    pos = 4 * (row * int(r["src_pitch"]) + col)
    vals = [_peek_f32(src_base + o + pos) for o in offs]
    if labels:
        for g in range(groups):
            for k in range(1, K):
                i = g * K + k
                if vals[i] != vals[g * K]:
                    t0, d0 = labels[g * K]
                    t1, d1 = labels[i]
                    if t1 == t0:
                        return ReplicateMismatchError(
                            f"{where} tp_rank {t1}: dp replicas differ (dp {d0} vs dp {d1})")
                    return ReplicateMismatchError(
                        f"{where}: tp replicas differ (tp {t0} vs tp {t1})")
    return ReplicateMismatchError(f"{where}: replicas differ (element {elem})")


class Arena:
    """A device (or pinned host) byte buffer."""

    def __init__(self, nbytes: int, device: torch.device | None = None, pinned: bool = False):
        nbytes = max(int(nbytes), 16)
        if device is not None:
            self.t = torch.empty(nbytes, dtype=torch.uint8, device=device)
        else:
            self.t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=pinned)
        self.nbytes = nbytes

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    def numpy(self) -> np.ndarray:
        return self.t.numpy()


class _Pinned:
    """Keeps an mmap'd, cudaHostRegister'ed host region alive; unregisters
    when the owning tensor is collected (the mapping itself lives as long as
    any numpy / torch view of it)."""

    def __init__(self, mm, arr: np.ndarray):
        self.mm, self.arr, self.ptr = mm, arr, arr.ctypes.data

    def __del__(self):
        try:
            torch.cuda.cudart().cudaHostUnregister(self.ptr)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def pinned_host(nbytes: int, threads: int = 16, huge: bool | None = None) -> torch.Tensor:
    """Page-locked host bytes, exact size: anonymous mmap, first-touched
    from ``threads`` threads (page zeroing is the cost; torch's pinned
    allocator does it on one thread and rounds up to a power of two), then
    cudaHostRegister. About 3x cheaper than ``torch.empty(pin_memory=True)``
    on the B200 hosts (tools/probe_pin.py)."""
    import mmap
    from concurrent.futures import ThreadPoolExecutor

    nbytes = max(int(nbytes), 4096)
    mm = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    if huge is None:
        huge = os.environ.get("UCP_PIN_HUGE", "1") != "0"
    if huge and hasattr(mm, "madvise") and hasattr(mmap, "MADV_HUGEPAGE"):
        # transparent huge pages (THP is "madvise" on the B200 hosts): fewer
        # pages to pin and fewer IOMMU translations per DMA byte
        mm.madvise(mmap.MADV_HUGEPAGE)
    arr = np.frombuffer(mm, dtype=np.uint8)
    step = 64 << 20
    with ThreadPoolExecutor(max(1, threads)) as pool:
        list(pool.map(lambda o: arr[o:o + step].fill(0), range(0, nbytes, step)))
    rc = torch.cuda.cudart().cudaHostRegister(arr.ctypes.data, nbytes, 0)
    if int(rc) != 0:
        raise RuntimeError(f"cudaHostRegister({nbytes}) failed: {rc}")
    t = torch.from_numpy(arr)
    t._ucp_pinned = _Pinned(mm, arr)  # noqa: SLF001 - lifetime anchor
    return t


def gen_state(base: int, start: int, count: int, abs_flag: bool, out_ptr: int, stream=None) -> None:
    _check(_native.lib().ucp_gen_state(base, start, count, int(abs_flag), ctypes.c_void_p(out_ptr),
                                       stream_ptr(stream)), "gen_state")


def compare(a_ptr: int, b_ptr: int, nbytes: int, scratch: torch.Tensor, stream=None) -> None:
    _check(_native.lib().ucp_compare(ctypes.c_void_p(a_ptr), ctypes.c_void_p(b_ptr), nbytes,
                                     scratch.data_ptr(), stream_ptr(stream)), "compare")

"""Kernel-level fuzz: random run tables (shapes, pitches, 16-B phases, ops,
replica counts, fan-out, destination dtypes, tile sizes) executed by the
CUDA kernels through the C ABI and by the numpy interpreter of the same
table (tests/descr_interp.py, itself pinned to the reference goldens on
CPU). Every destination byte must agree, and so must the failure report.

This exercises what the golden cells reach only partly: ROWSPLIT and
row-block tiles of every size, the per-CTA tile derivation over many runs
(ABI v2), scalar heads/tails at every phase, phase-mismatched runs on the
general kernel, MEAN/NOISE/ZERO/CHECKZERO, and the fused kernels (vector
and phase-mismatched scalar cells) with and without the atomic write."""

import numpy as np
import pytest
import torch

from descr_interp import execute, execute_fused
from paper_2406_18820_b200.engine import Program, Status, XProgram
from paper_2406_18820_b200.plan import (
    NO_ATOM,
    OP_CHECKZERO,
    OP_COPY,
    OP_MEAN,
    OP_NOISE,
    OP_ZERO,
    RunTable,
    XRunTable,
    expand_tiles,
)
from paper_2406_18820_b200.spec import DType

pytestmark = pytest.mark.gpu

_ESZ = {DType.F32: 4, DType.BF16: 2, DType.F16: 2}


class _Arena:
    """Bump allocator over a byte buffer: regions at a chosen element phase."""

    def __init__(self):
        self.top = 0

    def take(self, nbytes: int, phase_elems: int, esz: int) -> int:
        at = (self.top + 255) // 256 * 256 + phase_elems * esz
        self.top = at + nbytes
        return at


def _random_bits(rng, n, finite: bool):
    if finite:
        return rng.uniform(-4, 4, n).astype(np.float32)
    b = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    return b.view(np.float32)


def _region(rows, cols, pitch):
    return (rows - 1) * pitch + cols


def _fill(buf, at, rows, cols, pitch, vals):
    """Write vals [rows, cols] f32 at byte offset `at` with row pitch (elements)."""
    v = buf[at:at + 4 * _region(rows, cols, pitch)].view(np.float32)
    for r in range(rows):
        v[r * pitch:r * pitch + cols] = vals[r]


def _build_move(rng, n_runs):
    src_a, dst_a = _Arena(), _Arena()
    plans, tab = [], RunTable()
    tab.unit("fuzz", "weight")
    for _ in range(n_runs):
        op = rng.choice([OP_COPY] * 6 + [OP_MEAN, OP_NOISE, OP_ZERO, OP_CHECKZERO])
        dtype = DType.F32 if op in (OP_CHECKZERO,) else rng.choice([DType.F32, DType.BF16, DType.F16])
        esz = _ESZ[dtype]
        rows = int(rng.choice([1, 1, 2, 3, 17, 64]))
        cols = int(rng.choice([1, 3, 5, 31, 512, 515, 2048, 4099, 40000]))
        aligned = rng.random() < 0.7
        phase = int(rng.integers(0, 4))
        sp = cols + (int(rng.integers(0, 3)) * 4 if aligned else int(rng.integers(0, 9)))
        dp = cols + (int(rng.integers(0, 3)) * 4 if aligned else int(rng.integers(0, 9)))
        groups, K = 1, int(rng.integers(1, 4))
        if op == OP_MEAN:
            groups, K = int(rng.integers(2, 5)), int(rng.integers(1, 3))
        if op in (OP_NOISE, OP_CHECKZERO):
            K = int(rng.integers(1, 3))
        n_src = 0 if op == OP_ZERO else groups * K
        n_dst = 0 if op == OP_CHECKZERO else int(rng.integers(1, 4))
        srcs, data = [], []
        for g in range(groups if n_src else 0):
            vals = _random_bits(rng, rows * cols, finite=op == OP_MEAN).reshape(rows, cols)
            if op == OP_CHECKZERO:
                vals = np.zeros((rows, cols), dtype=np.float32)
            for _k in range(K):
                ph = phase if aligned else int(rng.integers(0, 4))
                at = src_a.take(4 * _region(rows, cols, sp), ph, 4)
                srcs.append(at)
                data.append((at, vals))
        dsts = []
        for _d in range(n_dst):
            ph = phase if aligned else int(rng.integers(0, 4))
            dsts.append(dst_a.take(esz * _region(rows, cols, dp), ph, esz))
        tp = int(rng.integers(2, 9))
        tab.add(srcs=srcs, dsts=dsts, src_pitch=sp, dst_pitch=dp, rows=rows, cols=cols, op=int(op),
                groups=groups, dtype=dtype, tp_rank=int(rng.integers(0, tp)), tp=tp, tag=0)
        plans.append((rows, cols, sp, data))
    src = np.zeros(max(src_a.top, 16), dtype=np.uint8)
    for rows, cols, sp, data in plans:
        for at, vals in data:
            _fill(src, at, rows, cols, sp, vals)
    return tab, src, max(dst_a.top, 16)


@pytest.mark.parametrize("seed", range(48))
def test_move_kernels_match_interpreter(seed):
    rng = np.random.default_rng(1000 + seed)
    tab, src, dst_n = _build_move(rng, int(rng.integers(1, 14)))
    tile_bytes = int(rng.choice([2048, 8192, 1 << 15, 1 << 17]))
    runs, aux, tiles = tab.finish(tile_bytes)
    want = np.full(dst_n, 0xA5, dtype=np.uint8)
    assert execute(runs, aux, tiles, src.copy(), want) == []
    d_src = torch.from_numpy(src).cuda()
    for gather in (True, False):
        if gather and any(int(r["dtype"]) != 0 for r in runs):
            continue  # convert writes f32 atomics only
        got = torch.full((dst_n,), 0xA5, dtype=torch.uint8, device="cuda")
        prog = Program(tab, torch.device("cuda"), tile_bytes)
        st = Status(torch.device("cuda"))
        st.reset()
        prog.launch(gather, d_src.data_ptr(), got.data_ptr(), st)
        torch.cuda.synchronize()
        assert st.read()[0] == (1 << 64) - 1, (seed, gather)
        g = got.cpu().numpy()
        bad = np.flatnonzero(g != want)
        assert bad.size == 0, (seed, gather, bad[:8], len(runs), tile_bytes)


@pytest.mark.parametrize("seed", range(32))
def test_fused_kernel_matches_interpreter(seed):
    rng = np.random.default_rng(2000 + seed)
    fx = XRunTable()
    fx.unit("fuzz", "weight")
    src_a, atom_a, dst_a = _Arena(), _Arena(), _Arena()
    fills = []
    for _ in range(int(rng.integers(1, 12))):
        dtype = rng.choice([DType.F32, DType.BF16, DType.F16])
        esz = _ESZ[dtype]
        rows = int(rng.choice([1, 2, 5, 33]))
        cols = int(rng.choice([1, 4, 7, 512, 777, 4096, 30001]))
        phase = int(rng.integers(0, 4))
        vec = seed % 2 == 0 or rng.random() < 0.3  # odd seeds: mostly phase-mismatched cells
        pad = lambda: int(rng.integers(0, 3)) * 4 if vec else int(rng.integers(0, 9))  # noqa: E731
        sp, ap, dp = cols + pad(), cols + pad(), cols + pad()
        if rows == 1:
            sp = ap = dp = cols
        ph = (lambda: phase) if vec else (lambda: int(rng.integers(0, 4)))  # noqa: E731
        K = int(rng.integers(1, 5))
        vals = _random_bits(rng, rows * cols, finite=False).reshape(rows, cols)
        srcs = []
        for _k in range(K):
            at = src_a.take(4 * _region(rows, cols, sp), ph(), 4)
            srcs.append(at)
            fills.append((at, rows, cols, sp, vals))
        atom = atom_a.take(4 * _region(rows, cols, ap), ph(), 4) if rng.random() < 0.8 else NO_ATOM
        dsts = [dst_a.take(esz * _region(rows, cols, dp), ph(), esz)
                for _d in range(int(rng.integers(0, 4)))]
        fx.add(srcs=srcs, atom=atom, dsts=dsts, src_pitch=sp, atom_pitch=ap, dst_pitch=dp,
               rows=rows, cols=cols, dtype=dtype, tag=0, vec=vec)
    src = np.zeros(max(src_a.top, 16), dtype=np.uint8)
    for at, rows, cols, sp, vals in fills:
        _fill(src, at, rows, cols, sp, vals)
    tile_bytes = int(rng.choice([4096, 1 << 15, 1 << 17]))
    runs, aux, rt, _, _ = fx.finish_classed(tile_bytes)
    w_atom = np.full(max(atom_a.top, 16), 0x5A, dtype=np.uint8)
    w_dst = np.full(max(dst_a.top, 16), 0xA5, dtype=np.uint8)
    assert execute_fused(runs, aux, expand_tiles(runs, rt), src, w_atom, w_dst) == []
    prog = XProgram(fx, torch.device("cuda"), tile_bytes)
    d_src = torch.from_numpy(src).cuda()
    g_atom = torch.full((w_atom.size,), 0x5A, dtype=torch.uint8, device="cuda")
    g_dst = torch.full((w_dst.size,), 0xA5, dtype=torch.uint8, device="cuda")
    st = Status(torch.device("cuda"))
    st.reset()
    prog.launch(d_src.data_ptr(), g_atom.data_ptr(), g_dst.data_ptr(), st)
    torch.cuda.synchronize()
    assert st.read()[0] == (1 << 64) - 1, seed
    assert np.array_equal(g_atom.cpu().numpy(), w_atom), seed
    assert np.array_equal(g_dst.cpu().numpy(), w_dst), seed


def test_fuzz_failure_reports_match():
    """A flipped replica element: the GPU's first failure (run, element),
    mapped back to table order, is the interpreter's first failure."""
    rng = np.random.default_rng(7)
    for trial in range(6):
        tab, src, dst_n = _build_move(rng, 8)
        runs, aux, tiles = tab.finish(8192)
        cand = [i for i, r in enumerate(runs) if int(r["op"]) == OP_COPY and int(r["n_src"]) > 1]
        if not cand:
            continue
        i = cand[int(rng.integers(0, len(cand)))]
        r = runs[i]
        k = int(rng.integers(1, int(r["n_src"])))
        off = int(aux[int(r["aux"]) + k - 1])
        e = int(rng.integers(0, int(r["rows"]) * int(r["cols"])))
        row, col = divmod(e, int(r["cols"]))
        pos = off + 4 * (row * int(r["src_pitch"]) + col)
        src[pos:pos + 4] ^= np.uint8(0x01)
        want_fails = execute(runs, aux, tiles, src.copy(), np.zeros(dst_n, dtype=np.uint8))
        assert (i, e) in want_fails
        prog = Program(tab, torch.device("cuda"), 8192)
        st = Status(torch.device("cuda"))
        st.reset()
        got = torch.zeros(dst_n, dtype=torch.uint8, device="cuda")
        prog.launch(False, torch.from_numpy(src).cuda().data_ptr(), got.data_ptr(), st)
        torch.cuda.synchronize()
        first, _ = st.read()
        run_sorted, elem = first >> 32, first & 0xFFFFFFFF
        assert (int(prog.run_order[run_sorted]), elem) == (i, e), trial


@pytest.mark.parametrize("op", [OP_MEAN, OP_NOISE])
def test_fuzz_failure_reports_match_ops(op):
    """The same for the OPS kernels: a flipped element in a replica (k >= 1)
    of a MEAN group or a NOISE source is reported at its (run, element),
    through the vector and the 4-B paths alike."""
    rng = np.random.default_rng(11 + op)
    hit = 0
    for trial in range(40):
        tab, src, dst_n = _build_move(rng, 8)
        runs, aux, tiles = tab.finish(8192)
        cand = []
        for i, r in enumerate(runs):
            G = max(1, int(r["groups"])) if int(r["op"]) == OP_MEAN else 1
            if int(r["op"]) == op and int(r["n_src"]) > G:
                cand.append((i, int(r["n_src"]) // G))
        if not cand:
            continue
        i, K = cand[int(rng.integers(0, len(cand)))]
        r = runs[i]
        j = int(rng.integers(0, int(r["n_src"])))
        if j % K == 0:
            j += 1  # a replica, not a group's primary
        off = int(aux[int(r["aux"]) + j - 1])
        e = int(rng.integers(0, int(r["rows"]) * int(r["cols"])))
        row, col = divmod(e, int(r["cols"]))
        pos = off + 4 * (row * int(r["src_pitch"]) + col)
        src[pos:pos + 4] ^= np.uint8(0x01)
        want_fails = execute(runs, aux, tiles, src.copy(), np.zeros(dst_n, dtype=np.uint8))
        assert (i, e) in want_fails
        prog = Program(tab, torch.device("cuda"), 8192)
        st = Status(torch.device("cuda"))
        st.reset()
        got = torch.zeros(dst_n, dtype=torch.uint8, device="cuda")
        prog.launch(False, torch.from_numpy(src).cuda().data_ptr(), got.data_ptr(), st)
        torch.cuda.synchronize()
        first, _ = st.read()
        run_sorted, elem = first >> 32, first & 0xFFFFFFFF
        assert (int(prog.run_order[run_sorted]), elem) == (i, e), trial
        hit += 1
    assert hit >= 3, hit

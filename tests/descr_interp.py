"""A numpy interpreter of the device descriptor table (tests only).

Executes ucp_run / ucp_tile tables exactly as the CUDA kernel defines them
(include/ucp_b200.h): tile rectangles, group-major sources with bitwise
replica checks, f64 MEAN, partial NOISE, ZERO, CHECKZERO, and f32 -> f32 /
bf16 / f16 destination casts. It lets the CPU test suite prove that the
descriptor compiler + tiler reproduce the oracle's bytes without a GPU.
"""

from __future__ import annotations

import numpy as np

from oracle import ucp_oracle as O
from paper_2406_18820_b200.plan import (
    OP_CHECKZERO,
    OP_COPY,
    OP_MEAN,
    OP_NOISE,
    OP_ZERO,
    RUN_ROWSPLIT,
)


def _f32_at(buf: np.ndarray, byte_off: np.ndarray) -> np.ndarray:
    assert (byte_off % 4 == 0).all()
    return buf.view(np.uint32)[byte_off // 4].view(np.float32)


def execute(runs, aux, tiles, src: np.ndarray, dst: np.ndarray) -> list:
    """Run the table over uint8 arrays src/dst (offsets relative to them).
    Returns [(run, elem)] failures (replica mismatch / nonzero pad)."""
    fails = []
    src = np.ascontiguousarray(src)
    for t in tiles:
        r = runs[int(t["run"])]
        n_src, n_dst = int(r["n_src"]), int(r["n_dst"])
        a = int(r["aux"])
        srcs = [int(r["src"])] + [int(x) for x in aux[a:a + max(n_src - 1, 0)]] if n_src else []
        dsts = [int(r["dst"])] + [int(x) for x in aux[a + max(n_src - 1, 0):
                                                     a + max(n_src - 1, 0) + n_dst - 1]] if n_dst else []
        if int(r["flags"]) & RUN_ROWSPLIT:
            rows = [int(t["row0"])]
            c0, c1 = int(t["col0"]), int(t["col0"]) + int(t["count"])
        else:
            rows = range(int(t["row0"]), int(t["row0"]) + int(t["count"]))
            c0, c1 = 0, int(r["cols"])
        cols = np.arange(c0, c1, dtype=np.int64)
        G = max(int(r["groups"]), 1)
        K = n_src // G if n_src else 0
        op = int(r["op"])
        dt = int(r["dtype"])
        esz = 4 if dt == 0 else 2
        for row in rows:
            sidx = row * int(r["src_pitch"]) + cols
            didx = row * int(r["dst_pitch"]) + cols
            elem = row * int(r["cols"]) + cols
            bad = np.zeros(len(cols), dtype=bool)
            prim = []
            for g in range(G if op == OP_MEAN else (1 if n_src else 0)):
                p = _f32_at(src, srcs[g * K] + 4 * sidx)
                for k in range(1, K):
                    w = _f32_at(src, srcs[g * K + k] + 4 * sidx)
                    bad |= p.view(np.uint32) != w.view(np.uint32)
                prim.append(p)
            if op == OP_COPY:
                v = prim[0]
            elif op == OP_MEAN:
                acc = prim[0].astype(np.float64)
                for q in prim[1:]:
                    acc = acc + q.astype(np.float64)
                v = (acc / float(G)).astype(np.float32)
            elif op == OP_NOISE:
                v = O.partial_noise(prim[0], int(r["tp_rank"]), int(r["tp"]))
            elif op == OP_ZERO:
                v = np.zeros(len(cols), dtype=np.float32)
            elif op == OP_CHECKZERO:
                v = prim[0]
                bad |= v.view(np.uint32) != 0
            else:
                raise AssertionError(op)
            if bad.any():
                fails.append((int(t["run"]), int(elem[np.argmax(bad)])))
            if dt == 0:
                out = v.view(np.uint8).reshape(-1, 4)
            elif dt == 2:
                out = O.bf16_bits(v).view(np.uint8).reshape(-1, 2)
            else:
                out = O.f16_bits(v).view(np.uint8).reshape(-1, 2)
            for d in dsts:
                pos = d + esz * didx
                for b in range(esz):
                    dst[pos + b] = out[:, b]
    return fails


def execute_fused(runs, aux, tiles, src: np.ndarray, atom: np.ndarray, dst: np.ndarray) -> list:
    """Interpret ucp_xrun tables (ucp_reshard_fused)."""
    from paper_2406_18820_b200.plan import NO_ATOM

    fails = []
    for t in tiles:
        r = runs[int(t["run"])]
        ns, nd = int(r["n_src"]), int(r["n_dst"])
        a = int(r["aux"])
        srcs = [int(r["src"])] + [int(x) for x in aux[a:a + ns - 1]]
        dsts = ([int(r["dst"])] + [int(x) for x in aux[a + ns - 1:a + ns - 1 + nd - 1]]) if nd else []
        if int(r["flags"]) & RUN_ROWSPLIT:
            rows = [int(t["row0"])]
            c0, c1 = int(t["col0"]), int(t["col0"]) + int(t["count"])
        else:
            rows = range(int(t["row0"]), int(t["row0"]) + int(t["count"]))
            c0, c1 = 0, int(r["cols"])
        cols = np.arange(c0, c1, dtype=np.int64)
        dt = int(r["dtype"])
        esz = 4 if dt == 0 else 2
        for row in rows:
            sidx = row * int(r["src_pitch"]) + cols
            v = _f32_at(src, srcs[0] + 4 * sidx)
            bad = np.zeros(len(cols), dtype=bool)
            for s in srcs[1:]:
                bad |= v.view(np.uint32) != _f32_at(src, s + 4 * sidx).view(np.uint32)
            if bad.any():
                fails.append((int(t["run"]), int(row * int(r["cols"]) + cols[np.argmax(bad)])))
            if int(r["atom"]) != NO_ATOM:
                pos = int(r["atom"]) + 4 * (row * int(r["atom_pitch"]) + cols)
                for b in range(4):
                    atom[pos + b] = v.view(np.uint8).reshape(-1, 4)[:, b]
            out = (v.view(np.uint8).reshape(-1, 4) if dt == 0 else
                   (O.bf16_bits(v) if dt == 2 else O.f16_bits(v)).view(np.uint8).reshape(-1, 2))
            didx = row * int(r["dst_pitch"]) + cols
            for d in dsts:
                pos = d + esz * didx
                for b in range(esz):
                    dst[pos + b] = out[:, b]
    return fails

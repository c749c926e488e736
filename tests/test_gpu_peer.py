"""Rank-homed load through CUDA IPC peer memory (north_star item 3), run as
2 processes (on cuda:0 and cuda:1 when two GPUs exist, else both on cuda:0):
each rank's fused reshard kernel stores the target fragments homed on the
other rank straight into that rank's IPC-mapped receive buffer. Checked
against the oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    # rank r on cuda:r when there are enough GPUs (real cross-device IPC over
    # NVLink); otherwise both ranks share cuda:0
    torch.cuda.set_device(rank % torch.cuda.device_count())
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2406_18820_b200 as U
        from oracle import ucp_oracle as O
        from paper_2406_18820_b200.dist import PeerBuffers, build_exchange, owned_params
        from paper_2406_18820_b200.layout import all_rank_records
        from paper_2406_18820_b200.reshard import ReshardPlan
        from paper_2406_18820_b200.spec import DType

        spec = U.make_model("GQA", {"n_layers": 4, "hidden": 64, "q_heads": 8, "kv_heads": 2})
        src = U.ParallelConfig(dp=2, tp=2, pp=2, zero_stage=U.ZeroStage.Z1)
        tgt = U.ParallelConfig(dp=3, tp=2, zero_stage=U.ZeroStage.Z1)
        dtype, wb = DType.BF16, 60_000
        ex = build_exchange(spec, src, tgt, world, rank, wb, dtype)
        bufs = PeerBuffers(ex.max_recv, n_slots=ex.n_windows)
        plan = ReshardPlan(spec, src, tgt, dtype=dtype, params=owned_params(spec, rank, world),
                           window_bytes=wb, fused=True, peer=(ex, bufs),
                           home_of=[g % world for g in range(tgt.world_size)], n_homes=world)
        plan.synthesize(7)
        torch.cuda.synchronize()
        dist.barrier()
        plan.status.reset()
        plan.step_device()
        torch.cuda.synchronize()
        plan.check()
        dist.barrier()
        state = O.init_state(spec, 7)
        recs = all_rank_records(spec, tgt)
        ok = 0
        for (g, i), (w, off) in ex.index.items():
            m = recs[g][i]
            a = O.extract(spec.param(m.param), tgt, m, state[m.param][m.kind])
            a = O.cast_weight(a, dtype.name) if m.kind == "weight" else a
            b = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
            got = bufs.read_local(w, off, b.size)
            assert np.array_equal(got, b), (g, m.param, m.kind)
            ok += 1
        dist.barrier()
        bufs.close()
        homed = sum(len(recs[g]) for g in range(tgt.world_size) if g % world == rank)
        q.put((rank, ok, homed, plan.n_fused_units, plan.n_units))
    finally:
        dist.destroy_process_group()


def test_peer_homed_fused_reshard_two_processes():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time

    res, deadline = [], time.time() + 600
    while len(res) < world:
        try:
            res.append(q.get(timeout=5))
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            assert not dead and time.time() < deadline, f"worker failed: exit codes {dead}"
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, ok, homed, fused, units in res:
        assert ok == homed > 0
        assert fused > 0

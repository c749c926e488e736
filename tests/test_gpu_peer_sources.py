"""Fully peer-homed distributed reshard (dist.PeerSources + PeerBuffers):
source rank g's fragments live on GPU g mod world, target rank t's on GPU t
mod world, and each param owner's fused kernel reads its sources from the
home GPUs and stores the targets into the home GPUs over IPC-mapped peer
memory -- no staging, no collective. Run as 2 processes, on two GPUs when
present, else sharing cuda:0; checked byte-for-byte against the oracle."""

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


def _worker(rank, world, port, q, fault):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    # rank r on cuda:r when there are enough GPUs (real cross-device IPC over
    # NVLink); otherwise both ranks share cuda:0
    torch.cuda.set_device(rank % torch.cuda.device_count())
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2406_18820_b200 as U
        from oracle import ucp_oracle as O
        from paper_2406_18820_b200.dist import PeerBuffers, PeerSources, build_exchange, owned_params
        from paper_2406_18820_b200.layout import all_rank_records
        from paper_2406_18820_b200.reshard import ReshardPlan
        from paper_2406_18820_b200.spec import DType

        spec = U.make_model("GQA", {"n_layers": 4, "hidden": 64, "q_heads": 8, "kv_heads": 2})
        src = U.ParallelConfig(dp=2, tp=2, pp=2, zero_stage=U.ZeroStage.Z1)
        tgt = U.ParallelConfig(dp=3, tp=2, zero_stage=U.ZeroStage.Z1)
        dtype, wb = DType.F32, 60_000
        sources = PeerSources(spec, src)
        sources.fill(7)
        if fault and rank == 1:
            # flip one weight element of a dp replica homed here
            recs = all_rank_records(spec, src)
            # a dp replica (dp rank 1) of a pp-stage-1 rank homed here
            g, i = next((g, k) for g in range(src.world_size) if g % world == rank
                        for k, m in enumerate(recs[g])
                        if m.param == "layers.3.attn_out" and m.kind == "weight"
                        and m.placement[2] == 1)
            import ctypes

            cudart = ctypes.CDLL("libcudart.so.12")
            val = np.array([7.0], dtype=np.float32)
            torch.cuda.synchronize()
            assert cudart.cudaMemcpy(ctypes.c_void_p(sources.addr(g, i) + 4 * 5),
                                     val.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(4),
                                     1) == 0  # cudaMemcpyHostToDevice
        torch.cuda.synchronize()
        dist.barrier()
        ex = build_exchange(spec, src, tgt, world, rank, wb, dtype)
        bufs = PeerBuffers(ex.max_recv, n_slots=ex.n_windows)
        plan = ReshardPlan(spec, src, tgt, dtype=dtype, params=owned_params(spec, rank, world),
                           window_bytes=wb, fused=True, peer=(ex, bufs), src_peer=sources,
                           home_of=[g % world for g in range(tgt.world_size)], n_homes=world)
        plan.status.reset()
        plan.step_device()
        torch.cuda.synchronize()
        err = None
        try:
            plan.check()
        except U.ReplicateMismatchError as e:
            err = str(e)
        dist.barrier()
        ok = 0
        if not fault:
            state = O.init_state(spec, 7)
            recs = all_rank_records(spec, tgt)
            for (g, i), (w, off) in ex.index.items():
                m = recs[g][i]
                a = O.extract(spec.param(m.param), tgt, m, state[m.param][m.kind])
                b = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
                assert np.array_equal(bufs.read_local(w, off, b.size), b), (g, m.param, m.kind)
                ok += 1
        dist.barrier()
        bufs.close()
        sources.close()
        q.put((rank, ok, err, plan.n_fused_units, plan.n_units))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fault", [False, True])
def test_peer_sources_and_targets_two_processes(fault):
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, fault)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time

    res, deadline = [], time.time() + 300
    while len(res) < world:
        try:
            res.append(q.get(timeout=5))
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            assert not dead and time.time() < deadline, f"worker failed: exit codes {dead}"
    res.sort()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    if not fault:
        assert all(ok > 0 and err is None and fused > 0 for _, ok, err, fused, _ in res)
    else:
        errs = [err for _, _, err, _, _ in res if err]
        assert len(errs) == 1 and "layers.3.attn_out.weight" in errs[0] and "dp" in errs[0]

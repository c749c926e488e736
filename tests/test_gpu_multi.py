"""Two distinct GPUs (skipped below that): the native NCCL all-to-all-v
between two processes, and bench.py at N = 2 under torchrun with the
multi-GPU fields the north_star asks for (aggregate HBM roofline, the
exchange stage against NVLink, per-GPU clocks). The peer-memory tests
(test_gpu_peer*.py) also run across two devices when they exist."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _need_two():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two CUDA devices")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _a2a_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2406_18820_b200.dist import NcclComm

        comm = NcclComm()
        # uneven counts: rank s sends (s + 1) * (d + 2) * 4096 + 13 bytes to d
        cnt = lambda s, d: (s + 1) * (d + 2) * 4096 + 13
        send_counts = [cnt(rank, d) for d in range(world)]
        recv_counts = [cnt(s, rank) for s in range(world)]
        pat = lambda s, d, n: ((np.arange(n) * 7 + 31 * s + 5 * d) % 251).astype(np.uint8)
        send = torch.from_numpy(np.concatenate([pat(rank, d, send_counts[d])
                                                for d in range(world)])).cuda()
        recv = torch.zeros(sum(recv_counts), dtype=torch.uint8, device="cuda")
        comm.alltoallv(send.data_ptr(), send_counts, recv.data_ptr(), recv_counts,
                       torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        got, at, ok = recv.cpu().numpy(), 0, True
        for s in range(world):
            ok &= np.array_equal(got[at:at + recv_counts[s]], pat(s, rank, recv_counts[s]))
            at += recv_counts[s]
        comm.close()
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_native_nccl_alltoallv_two_gpus():
    _need_two()
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_a2a_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {0: True, 1: True}


@pytest.mark.parametrize("home", ["param", "rank"])
def test_bench_two_gpus_reports_multi_gpu_fields(home):
    _need_two()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", "bench.py", "--gpus", "2",
           "--config", "cfg1", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e",
           "--home", home, "--exchange", "nccl"]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    d = json.loads(res.stdout.strip().splitlines()[-1])
    assert d["n_gpus"] == 2 and d["value"] > 0
    agg = d["roofline"]["aggregate"]
    assert agg["n_gpus"] == 2 and len(agg["per_rank"]) == 2 and 0 < agg["frac"]
    x = d["exchange"]
    assert x["nvlink_frac"] > 0 and x["bytes_sent_per_gpu_max"] > 0
    assert len(d["clocks"]["per_gpu"]) == 2
    assert d["parity"]["atomic_ok"] and d["parity"]["target_ok"] in (True, None)
    assert "NCCL INFO" in res.stderr  # the communicator log went to stderr

"""bench.py's N > 1 reporting on CPU (gloo, world_size 2): every rank's local
stats are gathered over the process group and rank 0 derives the whole-job
line -- value over the max-over-ranks step time, the aggregate HBM roofline
(N x peak), the exchange stage against NVLink and per-GPU clocks."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _local(rank):
    # rank 1 is the slow one; both send bytes over the exchange
    return {"ms": 10.0 + 2.0 * rank, "S": 40e9, "hbm_bytes": 80e9 + rank * 1e9,
            "clocks": {"sm_mhz": 1800.0 + rank, "sm_max_mhz": 1965.0,
                       "reasons": ["sw_power_cap"] if rank else [], "samples": 5, "gpu": rank},
            "exchange": {"transport": "nccl", "bytes_sent": 9e9 * (1 + rank), "bytes_total": 20e9,
                         "exchange_ms": 12.0 + rank, "step_ms": 14.0 + rank}}


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        stats = bench.gather_stats(_local(rank), world)
        q.put((rank, bench.aggregate_ranks(stats, 6000.0)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_aggregate_fields():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = res[0]
    assert res[1] == a  # every rank derives the same line
    # whole-job value: sum of state over the slowest rank's step
    assert a["ms"] == 12.0 and a["S"] == 80e9
    assert a["value"] == pytest.approx(80e9 / 12e-3 / 1e9)
    agg = a["aggregate"]
    assert agg["n_gpus"] == 2 and agg["peak"] == 12000.0 and agg["unit"] == "GB/s"
    assert agg["achieved"] == pytest.approx(161e9 / 12e-3 / 1e9)
    assert agg["frac"] == pytest.approx(agg["achieved"] / 12000.0)
    assert [r["rank"] for r in agg["per_rank"]] == [0, 1]
    assert agg["load_balance"] == pytest.approx(10 / 12)
    x = a["exchange"]
    assert x["bytes_sent_per_gpu_max"] == 18e9 and x["exchange_ms_max"] == 13.0
    assert x["nvlink_frac"] == pytest.approx(18e9 / 13e-3 / 1e9 / 900.0)
    assert x["nvlink_peak_GBps"] == 900.0 and len(x["per_rank_GBps"]) == 2
    assert x["value"] == pytest.approx(80e9 / 15e-3 / 1e9)
    c = a["clocks"]
    assert c["reasons"] == ["sw_power_cap"] and c["sm_max_mhz"] == 1965.0
    assert [g["gpu"] for g in c["per_gpu"]] == [0, 1] and c["samples"] == 10


def test_single_rank_aggregate_keeps_clock_fields():
    a = bench.aggregate_ranks([_local(0)], 6000.0)
    assert a["aggregate"]["frac"] == pytest.approx(80e9 / 10e-3 / 1e9 / 6000.0)
    assert "per_gpu" not in a["clocks"] and a["clocks"]["gpu"] == 0

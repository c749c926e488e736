"""GPU toy trainer (ucp_adam_step) vs the reference's trained states, the
reference's resume-equivalence acceptance (SPEC criterion 2) through the
GPU convert/load, and the native NCCL all-to-all-v on one rank."""

import os
import socket

import numpy as np
import pytest
import torch

import paper_2406_18820_b200 as U
from helpers import SCALES
from oracle import ucp_oracle as O
from paper_2406_18820_b200.spec import DType

pytestmark = pytest.mark.gpu


def _dict_state(st):
    return {p.name: {k: getattr(st.params[p.name], k).data for k in ("weight", "m", "v")}
            for p in st.spec.params}


def _model_state(spec, d, step):
    return U.ModelState(spec, {p.name: U.ParamState(*(U.make_tensor(DType.F32, d[p.name][k])
                                                      for k in ("weight", "m", "v")))
                               for p in spec.params}, step, {"loss_scale": 1.0, "iteration": step})


def test_trainer_matches_reference_digests(golden):
    for row in golden["trained"]:
        spec = U.make_model(row["model"], SCALES[row["model"]])
        kw = row.get("cfg", {})
        cfg = U.TrainerConfig(lr=kw.get("lr", 1e-3), beta1=kw.get("beta1", 0.9),
                              grad_seed=kw.get("grad_seed", 2024))
        st = U.train_steps(U.init_state(spec, 7), cfg, 0, row["steps"])
        assert st.metadata["iteration"] == row["iteration"]
        assert O.state_digest(spec, _dict_state(st), row["steps"]) == row["digest"], row


@pytest.mark.parametrize("pair", range(4))
def test_resume_equivalence(tmp_path, pair):
    # train 3 -> save under src -> convert -> load under tgt -> resume 3 more
    # == train 6 straight (pkg/tests/test_acceptance.py criterion 2 shape)
    pairs = [("2,1,4,1,z1,seq", "2,2,2,1,z0,seq"), ("4,1,1,1,z3,seq", "2,2,2,1,z0,seq"),
             ("2,2,2,1,z1,int2", "1,1,4,1,z0,seq"), ("4,2,1,1,z1,seq", "2,1,1,1,z3,seq")]
    a, b = (U.parse_config_string(x) for x in pairs[pair])
    spec = U.make_model("GQA", SCALES["GQA"])
    tc = U.TrainerConfig()
    straight = U.train_steps(U.train_steps(U.init_state(spec, 7), tc, 0, 3), tc, 3, 3)
    mid = U.train_steps(U.init_state(spec, 7), tc, 0, 3)
    src = str(tmp_path / "src")
    U.partition(mid, a, src)
    atom = str(tmp_path / "atomic")
    U.convert(src, atom)
    world = U.load(atom, b)
    wd = {g: [(s.meta, s.tensor.data) for s in world.shards[g]] for g in world.shards}
    back = _model_state(spec, O.consolidate_world(spec, b, wd), 3)
    resumed = U.train_steps(back, tc, 3, 3)
    assert U.first_diff(resumed, straight) is None
    # the product's own consolidation (GPU union over the world) agrees
    mine = U.consolidate_world(world)
    assert U.first_diff(mine, back) is None


def test_native_nccl_alltoallv_single_rank():
    import torch.distributed as dist

    from paper_2406_18820_b200.dist import NcclComm

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = NcclComm()
        src = torch.arange(1 << 20, dtype=torch.int32, device="cuda").view(torch.uint8)
        dst = torch.zeros_like(src)
        stream = torch.cuda.current_stream()
        comm.alltoallv(src.data_ptr(), [src.numel()], dst.data_ptr(), [src.numel()],
                       stream.cuda_stream)
        torch.cuda.synchronize()
        assert torch.equal(src, dst)
        comm.close()
    finally:
        dist.destroy_process_group()

#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_trainer.py -x -q > gpurun_out/gpu_trainer_r01i.log 2>&1; echo "trainer rc=$?"; tail -15 gpurun_out/gpu_trainer_r01i.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --home rank --exchange nccl --layers 2 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_nccl1_r01i.json 2> gpurun_out/bench_nccl1_r01i.err; echo "nccl bench rc=$?"; tail -c 400 gpurun_out/bench_nccl1_r01i.json; grep -v Warn gpurun_out/bench_nccl1_r01i.err | tail -3

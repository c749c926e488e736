#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r01e.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_r01e.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --home rank --layers 2 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_homed1_r01e.json 2> gpurun_out/bench_homed1_r01e.err; echo "homed rc=$?"; tail -c 1200 gpurun_out/bench_homed1_r01e.json; tail -3 gpurun_out/bench_homed1_r01e.err
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_cfg3_r01e.json 2> gpurun_out/bench_cfg3_r01e.err; echo "cfg3 rc=$?"; tail -c 300 gpurun_out/bench_cfg3_r01e.json; tail -3 gpurun_out/bench_cfg3_r01e.err
timeout 1200 python bench.py --config cfg4 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_cfg4_r01e.json 2> gpurun_out/bench_cfg4_r01e.err; echo "cfg4 rc=$?"; tail -c 300 gpurun_out/bench_cfg4_r01e.json; tail -3 gpurun_out/bench_cfg4_r01e.err
timeout 1500 python bench.py --config cfg5 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_cfg5_r01e.json 2> gpurun_out/bench_cfg5_r01e.err; echo "cfg5 rc=$?"; tail -c 300 gpurun_out/bench_cfg5_r01e.json; tail -3 gpurun_out/bench_cfg5_r01e.err

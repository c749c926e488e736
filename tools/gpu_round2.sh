#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "llama or reshard" > gpurun_out/gpu_tests2.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_tests2.log
timeout 600 python bench.py --layers 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_small.log 2>&1; echo "small rc=$?"
tail -3 gpurun_out/bench_small.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "full rc=$?"
tail -3 gpurun_out/bench_full.log

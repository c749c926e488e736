#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r01h.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_r01h.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/bench_r01h.json 2> gpurun_out/bench_r01h.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_r01h.json; tail -3 gpurun_out/bench_r01h.err

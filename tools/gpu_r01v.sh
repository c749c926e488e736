#!/bin/bash
# re-validation after a container restore: gpu tests, smoke, default bench, reference arm
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r01v.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_r01v.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01v.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_r01v.log
timeout 1200 python bench.py > gpurun_out/bench_r01v.json 2> gpurun_out/bench_r01v.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_r01v.json; tail -3 gpurun_out/bench_r01v.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_r01v.json 2>&1; echo "ref rc=$?"; tail -c 600 gpurun_out/bench_ref_r01v.json

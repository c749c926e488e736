#!/bin/bash
# store/load cache-hint sweep + run_pinned test + e2e link roofline
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "run_pinned or fused_replica" > gpurun_out/gpu_tests_r01w.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_r01w.log
timeout 1500 bash tools/gpu_kernelsweep.sh > gpurun_out/sweep_r01w.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/sweep_r01w.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_r01w.json 2> gpurun_out/bench_r01w.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_r01w.json').read().strip().splitlines()[-1]); print(d['value'], json.dumps(d['e2e']))"; tail -3 gpurun_out/bench_r01w.err

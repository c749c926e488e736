#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r01j.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gpu_tests_r01j.log
python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-atomic > gpurun_out/bench_noatomic_r01.json 2> gpurun_out/bench_noatomic_r01.err; echo "noatomic rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/bench_noatomic_r01.json').read().strip().splitlines()[-1]); print('no-atomic', round(d['value'],1), round(d['roofline']['frac'],4), d['parity'])"; tail -2 gpurun_out/bench_noatomic_r01.err

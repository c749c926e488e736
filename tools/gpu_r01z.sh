#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r01z.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_r01z.log
timeout 900 python bench.py --dtype bf16 --no-cpu > gpurun_out/bench_bf16_r01z.json 2> gpurun_out/bench_bf16_r01z.err; echo "bf16 rc=$?"; tail -c 400 gpurun_out/bench_bf16_r01z.err
timeout 900 python bench.py > gpurun_out/bench_r01z.json 2> gpurun_out/bench_r01z.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench_r01z.err
for f in bench_bf16_r01z bench_r01z; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); r=d['roofline']; e=d['e2e']
print('$f', round(d['value'],1), round(r['frac'],4), r['kernel'], 'e2e', e['value'] and round(e['value'],2), d['parity'], d['cpu_baseline'] and d['cpu_baseline'].get('value'))"; done

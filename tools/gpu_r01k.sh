#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01k.json 2> gpurun_out/bench_r01k.err; echo "cfg2 rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/bench_r01k.json').read().strip().splitlines()[-1]); print('cfg2', round(d['value'],1), d['e2e'], d['cpu_baseline']['value'])"; tail -2 gpurun_out/bench_r01k.err
timeout 1200 python bench.py --config cfg3 --steps 3 --warmup 3 > gpurun_out/bench_cfg3_r01k.json 2> gpurun_out/bench_cfg3_r01k.err; echo "cfg3 rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/bench_cfg3_r01k.json').read().strip().splitlines()[-1]); print('cfg3', round(d['value'],1), d['e2e'], d['cpu_baseline']['value'])"; tail -2 gpurun_out/bench_cfg3_r01k.err
timeout 1500 python bench.py --config cfg5 --steps 2 --warmup 2 > gpurun_out/bench_cfg5_r01k.json 2> gpurun_out/bench_cfg5_r01k.err; echo "cfg5 rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/bench_cfg5_r01k.json').read().strip().splitlines()[-1]); print('cfg5', round(d['value'],1), d['e2e'], (d['cpu_baseline'] or {}).get('value'))"; tail -2 gpurun_out/bench_cfg5_r01k.err

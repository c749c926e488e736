#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
A="--steps 10 --warmup 3 --no-cpu"
for w in 0.2 0.1 0.05; do
  python bench.py $A --no-verify --e2e-window-gb $w 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('e2e window $w', round(d['e2e']['value'],2), round(d['e2e']['ms_per_step'],1))"
done
python bench.py $A --no-e2e --no-atomic > gpurun_out/bench_noatomic_r01.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/bench_noatomic_r01.json').read().strip().splitlines()[-1]); print('no-atomic', round(d['value'],1), round(d['roofline']['frac'],4), d['parity'])"
python bench.py $A --no-e2e --non-strict > gpurun_out/bench_nonstrict_r01.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/bench_nonstrict_r01.json').read().strip().splitlines()[-1]); print('non-strict', round(d['value'],1), round(d['roofline']['frac'],4), d['parity'])"

#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
A="--steps 10 --warmup 3 --no-cpu --no-e2e"
for f in experiments/libucp_b200_tma_*.so; do
UCP_B200_LIB=$f timeout -s KILL 300 python bench.py $A > gpurun_out/tma.json 2> gpurun_out/tma.err; echo "$f rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/tma.json').read().strip().splitlines()[-1]); print('  ', round(d['value'],1), round(d['roofline']['frac'],4), d['parity']['atomic_ok'], d['parity']['target_ok'])"; tail -1 gpurun_out/tma.err
done

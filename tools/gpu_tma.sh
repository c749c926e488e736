#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
A="--steps 10 --warmup 3 --no-cpu --no-e2e"
python bench.py $A 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ldg', round(d['value'],1), round(d['roofline']['frac'],4), d['parity'])"
UCP_B200_LIB=experiments/libucp_b200_tma.so timeout -s KILL 300 python bench.py $A > gpurun_out/tma.json 2> gpurun_out/tma.err; echo "tma rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/tma.json').read().strip().splitlines()[-1]); print('tma', round(d['value'],1), round(d['roofline']['frac'],4), d['parity'])"; tail -3 gpurun_out/tma.err

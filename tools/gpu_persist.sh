#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
A="--steps 10 --warmup 3 --no-cpu --no-e2e --no-verify"
python bench.py $A 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('base', round(d['value'],1), round(d['roofline']['frac'],4))"
for f in experiments/libucp_b200_persist_b*.so; do
  UCP_B200_LIB=$f python bench.py $A 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['roofline']['frac'],4))"
done

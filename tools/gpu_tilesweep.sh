#!/bin/bash
# kernel A/B: tile size and L2 prefetch hint on the default workload (device value only)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
A="--steps 10 --warmup 3 --no-cpu --no-e2e --no-verify"
for tk in 64 128 256 512 1024; do
  python bench.py $A --tile-kb $tk 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('tile_kb $tk', round(d['value'],1), round(d['roofline']['frac'],4))"
done
for v in 128 256; do
  UCP_B200_LIB=experiments/libucp_b200_pf$v.so python bench.py $A 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pf $v', round(d['value'],1), round(d['roofline']['frac'],4))"
done

#!/bin/bash
# e2e vs host staging allocation: torch pinned / mmap+register (4K) / mmap+register (THP)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for rep in 1 2 3; do
for v in "UCP_PIN_MODE=torch" "UCP_PIN_HUGE=0" "UCP_PIN_HUGE=1"; do
  env $v timeout 900 python bench.py --no-cpu --no-verify --steps 3 > gpurun_out/p.json 2> gpurun_out/p.err; echo -n "$v rc=$? "
  python -c "
import json; d=json.loads(open('gpurun_out/p.json').read().strip().splitlines()[-1]); e=d['e2e']; l=e['link']
print(round(e['value'],2), round(l['h2d_GBps_in_step'],1), round(l['frac'],3), round(l['h2d_GBps'],1), round(l['bidir_GBps'],1))"
done; done
grep -i huge /proc/meminfo | head -4

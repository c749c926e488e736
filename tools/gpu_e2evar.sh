#!/bin/bash
# which bench leg perturbs the e2e number: full vs --no-cpu vs --no-verify, alternating
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for rep in 1 2; do
for v in "" "--no-cpu" "--no-verify"; do
  timeout 900 python bench.py --steps 5 $v > gpurun_out/v.json 2> gpurun_out/v.err; echo -n "[$v] rc=$? "
  python -c "
import json; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); e=d['e2e']; l=e['link']
print(round(e['value'],2), round(l['h2d_GBps_in_step'],1), round(l['frac'],3))"
done; done

#!/bin/bash
# run-to-run variance of the default driver command on one box
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 900 python bench.py > gpurun_out/rep_$i.json 2> gpurun_out/rep_$i.err; echo -n "run $i rc=$? "
  python -c "
import json; d=json.loads(open('gpurun_out/rep_$i.json').read().strip().splitlines()[-1]); r=d['roofline']; e=d['e2e']; c=d['cpu_baseline']
print(round(d['value'],1), round(r['frac'],4), 'e2e', round(e['value'],2), round(e['link']['frac'],3), 'cpu', round(c['value'],3), c['parity_vs_gpu']['bit_exact'], d['clocks'])"
done

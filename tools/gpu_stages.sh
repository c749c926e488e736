#!/bin/bash
# per-stage (unfused convert / load) numbers for every BASELINE config
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 1500 python bench.py --config $c --unfused --steps 5 --no-cpu --no-e2e > gpurun_out/stage_$c.json 2> gpurun_out/stage_$c.err; echo -n "$c rc=$? "
  python -c "
import json; d=json.loads(open('gpurun_out/stage_$c.json').read().strip().splitlines()[-1]); p=d['roofline']['per_stage']; S=d['config']['state_bytes']
print(round(d['value'],1), {k: (round(v['ms'],2), round(S/(v['ms']/1e3)/1e9,1) if v['ms'] else 0, round(v['frac'],3)) for k,v in p.items() if isinstance(v, dict) and v.get('hbm_bytes')}, d['parity'])"
done

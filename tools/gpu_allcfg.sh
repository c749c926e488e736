#!/bin/bash
# every BASELINE config through bench.py (cfg2 is the default workload)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-x}
for c in cfg1 cfg3 cfg4 cfg5; do
  timeout 1500 python bench.py --config $c --steps 5 > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err; echo "$c rc=$?"; tail -2 gpurun_out/bench_${c}_$TAG.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_${c}_$TAG.json').read().strip().splitlines()[-1]); r=d['roofline']; e=d['e2e'] or {}; c=d['cpu_baseline'] or {}
print('$c', round(d['value'],1), 'frac', round(r['frac'],4), 'e2e', e.get('value') and round(e['value'],2), 'link', e.get('link',{}).get('frac') and round(e['link']['frac'],3), 'cpu', c.get('value') and round(c['value'],3), c.get('kind'), (c.get('parity_vs_gpu') or {}).get('bit_exact'), d['parity'])"
done

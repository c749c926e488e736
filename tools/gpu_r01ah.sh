#!/bin/bash
# ABI v2 (per-run tiling, device scan + warp search): full GPU suite, default / unfused / bf16 bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r01ah.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gpu_tests_r01ah.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for v in "" "--unfused" "--dtype bf16"; do
  timeout 900 python bench.py --no-cpu --no-e2e $v > gpurun_out/b.json 2> gpurun_out/b.err; echo "bench '$v' rc=$?"; tail -2 gpurun_out/b.err
  python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); r=d['roofline']
print(round(d['value'],1), round(r['frac'],4), {k: round(v.get('frac',0),4) for k,v in r['per_stage'].items() if isinstance(v, dict)}, d['parity'])"
done

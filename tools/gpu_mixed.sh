#!/bin/bash
# fused mixed-dtype launch A/B (bf16 targets), f32 unchanged, parity tests
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "not refsuite" > gpurun_out/gpu_tests_mixed.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests_mixed.log
for v in "UCP_FUSED_MIXED=1 --dtype bf16" "UCP_FUSED_MIXED=0 --dtype bf16" "UCP_FUSED_MIXED=1 --dtype bf16" "UCP_FUSED_MIXED=0 --dtype bf16" "UCP_FUSED_MIXED=1 --dtype f32"; do
  envv=${v%% *}; arg=${v#* }
  env $envv timeout 900 python bench.py --no-cpu --no-e2e --steps 10 $arg > gpurun_out/b.json 2> gpurun_out/b.err; echo -n "$v rc=$? "
  python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); r=d['roofline']
print(round(d['value'],1), round(r['frac'],4), r['launches_per_step'], d['gpu_launches'], d['parity'])"
done

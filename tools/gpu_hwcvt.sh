#!/bin/bash
# hardware pair casts for 16-bit targets: parity + A/B
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_fuzz.py -m gpu -q -x -k "cast or fuzz or kernel or file_pipeline or device_to_device or keep_on_device or reshard_plan" 2>&1 | tail -2
for v in "--dtype bf16" "--dtype f16" "--dtype bf16 --unfused"; do
  for lib in "" experiments/libucp_b200_t_swcvt.so; do
    UCP_B200_LIB=$lib timeout 900 python bench.py --no-cpu --no-e2e --steps 10 $v > gpurun_out/c.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v', '${lib:-hwcvt}', round(d['value'],1), round(r['frac'],4), {k: round(x['frac'],3) for k,x in r['per_stage'].items() if isinstance(x, dict) and x.get('hbm_bytes')}, d['parity']['atomic_ok'])"
  done
done

#!/bin/bash
# e2e pipeline depth / window sweep
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for args in "--e2e-slots 2" "--e2e-slots 3" "--e2e-slots 4" "--e2e-slots 3 --e2e-window-gb 0.2" "--e2e-slots 3 --e2e-window-gb 0.8" "--e2e-slots 4 --e2e-window-gb 0.2"; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-verify $args 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; l=e.get('link',{})
print('$args', round(e['value'],2), round(e['ms_per_step'],1), round(l.get('h2d_GBps_in_step',0),1), round(l.get('frac',0),3), round(l.get('h2d_GBps',0),1), round(l.get('bidir_GBps',0),1))"
done

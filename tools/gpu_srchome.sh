#!/bin/bash
# peer-homed sources (and targets) through the bench: 1 rank full 7B, 2 ranks (gloo, 1 GPU) 4 layers
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
A="--steps 5 --no-cpu --no-e2e"
timeout 900 python bench.py $A --src-home rank > gpurun_out/sh1.json 2> gpurun_out/sh1.err; echo "1 rank src-home rc=$?"; tail -2 gpurun_out/sh1.err
timeout 900 python bench.py $A --src-home rank --home rank > gpurun_out/sh2.json 2> gpurun_out/sh2.err; echo "1 rank src+tgt home rc=$?"; tail -2 gpurun_out/sh2.err
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29561 bench.py --gpus 2 --dist-backend gloo --layers 4 $A --src-home rank --home rank > gpurun_out/sh3.json 2> gpurun_out/sh3.err; echo "2 ranks src+tgt home rc=$?"; grep -v Warning gpurun_out/sh3.err | tail -2
for f in sh1 sh2 sh3; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['roofline']['frac'],4), d['n_gpus'], d['parity'].get('note','')[:30] if isinstance(d['parity'], dict) else d['parity'])"; done

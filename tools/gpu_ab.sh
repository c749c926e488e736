#!/bin/bash
# A/B of compile-time kernel switches on the GPU box:
#   tools/gpu_ab.sh TAG "CASES" "FLAGS_A" "FLAGS_B" ...
# rebuilds libucp_b200.so per variant (UCP_NVCC_EXTRA, force) and runs the
# kernel-zoo cases (CUDA-event rates) against it; restores the default build.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
TAG=$1; CASES=$2; shift 2
mkdir -p gpurun_out
for V in "$@"; do
  UCP_NVCC_EXTRA="$V" python -c "from paper_2406_18820_b200 import _build; _build.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $V"; continue; }
  for c in $CASES; do
    timeout 600 python tools/kernel_zoo.py --case $c > gpurun_out/ab_${c}_$TAG.json 2>/dev/null
    echo "[$V] $c $(python -c "import json; d=json.load(open('gpurun_out/ab_${c}_$TAG.json')); print({k: (round(v['GBps']), round(v['frac'], 3)) for k, v in d['stages'].items() if v['bytes'] > 1e6}, d['parity']['atomic_ok'], d['parity']['target_ok'])" 2>&1 | tail -1)"
  done
done
python -c "from paper_2406_18820_b200 import _build; _build.build(force=True)" > /dev/null 2>&1

#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_property.py -x -q > gpurun_out/gpu_property_r01q.log 2>&1; echo "prop rc=$?"; tail -5 gpurun_out/gpu_property_r01q.log
ARGS="--layers 2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-verify"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reshard_fused -s 8 -c 2 -o gpurun_out/prof_r01q python bench.py $ARGS > gpurun_out/ncu_r01q.log 2>&1; echo "ncu rc=$?"

#!/bin/bash
# usage: tools/prof.sh TAG  -- gpu tests + launch list + ncu --set full of both move kernels
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
TAG=${1:-r01}
mkdir -p gpurun_out
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_$TAG.log
fi
ARGS="--layers 2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-verify"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS > gpurun_out/launches_$TAG.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:convert_gather -s 13 -c 2 -o gpurun_out/prof_conv_$TAG python bench.py $ARGS > gpurun_out/ncu_conv_$TAG.log 2>&1; echo "ncu conv rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:load_scatter -s 17 -c 2 -o gpurun_out/prof_load_$TAG python bench.py $ARGS > gpurun_out/ncu_load_$TAG.log 2>&1; echo "ncu load rc=$?"
ls -la gpurun_out

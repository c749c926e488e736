#!/bin/bash
# usage: tools/gpu_cycle.sh TAG [bench args...] -- gpu tests, full bench, launch list, ncu of both stages
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
TAG=${1:-x}; shift
mkdir -p gpurun_out
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_$TAG.log
fi
timeout 1500 python bench.py --steps 10 --warmup 3 "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_$TAG.json; tail -5 gpurun_out/bench_$TAG.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
ARGS="--layers 2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-verify $@"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS > gpurun_out/launches_$TAG.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-reshard_fused} -s ${NCU_S:-8} -c ${NCU_C:-2} -o gpurun_out/prof_$TAG python bench.py $ARGS > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
fi

#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
ARGS="--layers 2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-verify"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reshard_fused -s 8 -c 2 -o gpurun_out/prof_r01d python bench.py $ARGS > gpurun_out/ncu_r01d.log 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_cfg3_r01d.json 2> gpurun_out/bench_cfg3_r01d.err; echo "cfg3 rc=$?"; tail -c 1500 gpurun_out/bench_cfg3_r01d.json; tail -3 gpurun_out/bench_cfg3_r01d.err
timeout 600 python bench.py --config cfg1 --steps 20 --warmup 5 > gpurun_out/bench_cfg1_r01d.json 2> gpurun_out/bench_cfg1_r01d.err; echo "cfg1 rc=$?"; tail -c 800 gpurun_out/bench_cfg1_r01d.json
timeout 900 python bench.py --unfused --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_unfused_r01d.json 2>&1; echo "unfused rc=$?"; tail -c 600 gpurun_out/bench_unfused_r01d.json

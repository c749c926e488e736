#!/bin/bash
# ncu launch lists (time + DRAM bytes) of every kernel family on ABI v2
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
A="--layers 2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-verify"
timeout 900 ncu $M --log-file gpurun_out/launches_unfused_r01bh.csv python bench.py $A --unfused > /dev/null 2>&1; echo "unfused rc=$?"
timeout 900 ncu $M --log-file gpurun_out/launches_bf16_r01bh.csv python bench.py $A --dtype bf16 > /dev/null 2>&1; echo "bf16 rc=$?"
timeout 900 ncu $M --log-file gpurun_out/launches_bf16unf_r01bh.csv python bench.py $A --dtype bf16 --unfused > /dev/null 2>&1; echo "bf16 unfused rc=$?"

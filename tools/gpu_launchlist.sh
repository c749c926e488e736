#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:reshard_fused --csv --log-file gpurun_out/launches_default_r01.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/launches_default_r01.log 2>&1; echo "ncu rc=$?"; tail -c 400 gpurun_out/launches_default_r01.log; wc -l gpurun_out/launches_default_r01.csv

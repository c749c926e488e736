#!/bin/bash
# the reference's own file pipeline on the same box / tmpfs, next to ours
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-x}
timeout 900 python tools/file_bench.py --config cfg1 --impl reference --reps 2 > gpurun_out/fileref_cfg1_$TAG.json 2> gpurun_out/fileref_cfg1_$TAG.err; echo "cfg1 rc=$?"; tail -c 600 gpurun_out/fileref_cfg1_$TAG.json; tail -2 gpurun_out/fileref_cfg1_$TAG.err
timeout 1500 python tools/file_bench.py --config cfg2 --layers 4 --impl reference --reps 1 > gpurun_out/fileref_cfg2l4_$TAG.json 2> gpurun_out/fileref_cfg2l4_$TAG.err; echo "cfg2l4 rc=$?"; tail -c 600 gpurun_out/fileref_cfg2l4_$TAG.json; tail -2 gpurun_out/fileref_cfg2l4_$TAG.err

#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r01f.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_r01f.log
timeout 900 python tools/file_bench.py --config cfg1 > gpurun_out/file_cfg1_r01f.json 2> gpurun_out/file_cfg1_r01f.err; echo "file rc=$?"; cat gpurun_out/file_cfg1_r01f.json; tail -3 gpurun_out/file_cfg1_r01f.err
timeout 900 python tools/file_bench.py --config cfg2 --layers 4 --reps 2 > gpurun_out/file_cfg2l4_r01f.json 2> gpurun_out/file_cfg2l4_r01f.err; echo "file2 rc=$?"; cat gpurun_out/file_cfg2l4_r01f.json; tail -3 gpurun_out/file_cfg2l4_r01f.err
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2

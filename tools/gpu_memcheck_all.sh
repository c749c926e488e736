#!/bin/bash
# compute-sanitizer memcheck over the whole GPU suite
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-x}
timeout 3000 compute-sanitizer --tool memcheck --error-exitcode 99 --target-processes all \
  python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/memcheck_all_$TAG.log 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/memcheck_all_$TAG.log | tail -5

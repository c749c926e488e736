#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small GPU parity cases
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-x}
K="${K:-reshard_plan_host_round_trip or union_reference_unit_cases or fused_replica_mismatch or shard_hy or run_pinned or file_pipeline_digests or fused_resume or corrupt_replica}"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
    python -m pytest ${FILES:-tests/test_gpu_parity.py} -m gpu -x -q -k "$K" > gpurun_out/sanitize_${tool}_$TAG.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_${tool}_$TAG.log | tail -3
done

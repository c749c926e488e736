#!/bin/bash
# the reference's own test suite with the B200 engine hot-swapped in, + the GPU suite
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-x}
if [ -d baseline/_ref_tests ]; then
  PYTHONPATH=baseline/_ref:.:tools timeout 2400 python -m pytest baseline/_ref_tests -p ref_suite_plugin -q -p no:cacheprovider -rf > gpurun_out/refsuite_$TAG.log 2>&1
  echo "refsuite rc=$?"; tail -8 gpurun_out/refsuite_$TAG.log
  PYTHONPATH=baseline/_ref timeout 2400 python -m pytest baseline/_ref_tests -q -p no:cacheprovider -rf > gpurun_out/refsuite_unmodified_$TAG.log 2>&1
  echo "unmodified reference suite rc=$?"; tail -5 gpurun_out/refsuite_unmodified_$TAG.log
fi
if [ "${SKIP_GPU_TESTS:-0}" != "1" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/gpu_tests_$TAG.log
fi

#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests/test_gpu_kernel_fuzz.py tests/test_gpu_parity.py tests/test_gpu_property.py -m gpu -q -x 2>&1 | tail -2
for lib in "" experiments/libucp_b200_t_scalar.so; do
  echo "lib=${lib:-staged} unfused"; UCP_B200_LIB=$lib timeout 900 python tools/gpu_misaligned.py unfused 2>&1 | grep -E "dp=3|dp=5" | cut -c1-70
done

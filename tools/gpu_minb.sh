#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for lib in experiments/libucp_b200_t_minb2.so experiments/libucp_b200_t_minb3.so experiments/libucp_b200_t_minb4.so; do
  echo "lib=$lib"; UCP_B200_LIB=$lib timeout 900 python tools/gpu_misaligned.py 2>&1 | grep -E "dp=3|dp=5" | cut -c1-70
  echo "unfused"; UCP_B200_LIB=$lib timeout 900 python tools/gpu_misaligned.py unfused 2>&1 | grep -E "dp=3|dp=5" | cut -c1-70
done

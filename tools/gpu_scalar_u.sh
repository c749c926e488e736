#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for lib in "" experiments/libucp_b200_t_u8.so experiments/libucp_b200_t_u16.so; do
  echo "lib=${lib:-default(U=4)}"; UCP_B200_LIB=$lib timeout 900 python tools/gpu_misaligned.py 2>&1 | grep -E "dp=3|dp=5" | cut -c1-80
done

#!/bin/bash
# file pipeline: chunked I/O vs whole-file jobs (UCP_IO_CHUNK=0), cfg1 + 7B/4 layers
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-x}
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "file_pipeline or resume or corrupt or manifest or pad or bypass or zero2" > gpurun_out/filetests_$TAG.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/filetests_$TAG.log
for ch in 0 16777216; do
  UCP_IO_CHUNK=$ch timeout 900 python tools/file_bench.py --config cfg2 --layers 4 > gpurun_out/file_cfg2l4_${TAG}_c$ch.json 2>gpurun_out/file_err_$ch.log; echo "cfg2l4 chunk=$ch rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/file_cfg2l4_${TAG}_c$ch.json')); print({k: round(v,2) for k,v in d.items() if k.endswith('GBps')}); print(json.dumps(d['pipeline_wait_s_last_rep']))"
done
UCP_IO_CHUNK=16777216 timeout 600 python tools/file_bench.py --config cfg1 > gpurun_out/file_cfg1_$TAG.json 2>&1; echo "cfg1 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/file_cfg1_$TAG.json')); print({k: round(v,2) for k,v in d.items() if k.endswith('GBps')})"
nproc; free -g | head -2; cat /sys/kernel/mm/transparent_hugepage/enabled

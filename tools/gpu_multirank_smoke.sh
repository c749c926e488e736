#!/bin/bash
# multi-rank bench logic on ONE GPU: 2 ranks share cuda:0 over gloo (NCCL refuses 2 ranks per GPU)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29541 bench.py --gpus 2 --dist-backend gloo --layers 4 --steps 3 --warmup 3 > gpurun_out/mr_param.json 2> gpurun_out/mr_param.err; echo "param rc=$?"; tail -c 700 gpurun_out/mr_param.json; grep -v Warning gpurun_out/mr_param.err | tail -3
timeout 900 $R --master-port 29542 bench.py --gpus 2 --dist-backend gloo --layers 4 --steps 3 --warmup 3 --home rank --exchange peer > gpurun_out/mr_peer.json 2> gpurun_out/mr_peer.err; echo "peer rc=$?"; tail -c 700 gpurun_out/mr_peer.json; grep -v Warning gpurun_out/mr_peer.err | tail -3
timeout 900 $R --master-port 29543 bench.py --gpus 2 --impl reference --steps 1 --warmup 1 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo "ref rc=$?"; tail -c 300 gpurun_out/mr_ref.json

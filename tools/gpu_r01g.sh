#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer.py -x -q > gpurun_out/gpu_peer_r01g.log 2>&1; echo "peer rc=$?"; tail -15 gpurun_out/gpu_peer_r01g.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --home rank --layers 2 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_peer1_r01g.json 2> gpurun_out/bench_peer1_r01g.err; echo "peer bench rc=$?"; tail -c 600 gpurun_out/bench_peer1_r01g.json; tail -3 gpurun_out/bench_peer1_r01g.err
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r01g.json 2> gpurun_out/bench_ref_r01g.err; echo "ref rc=$?"; cat gpurun_out/bench_ref_r01g.json; tail -3 gpurun_out/bench_ref_r01g.err

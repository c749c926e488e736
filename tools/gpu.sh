#!/bin/bash
# One entry point for the GPU-box recipes (run through gpurun):
#   tools/gpu.sh RECIPE TAG [extra bench.py args]
# Outputs go to gpurun_out/; kept results are copied into profiles/.
#   round-end   the driver's round-end commands: pytest -m gpu, smoke(), default
#               bench.py, bench.py --impl reference
#   tests       pytest -m gpu
#   allcfg      every BASELINE config through bench.py (fused default)
#   stages      every config with --unfused (convert / load stage rates)
#   repeat      the default bench 3x back to back (run-to-run variance)
#   e2e-sweep   host-streamed e2e: device slots / window size
#   file        file pipeline (tools/file_bench.py), ours; fileref: the reference's
#   sanitize    compute-sanitizer memcheck / racecheck / synccheck on parity tests
#   memcheck    memcheck over the whole GPU suite
#   multirank   2 ranks sharing one GPU over gloo: param-homed, peer-homed, reference arm
#   srchome     peer-homed sources (+ targets), 1 and 2 ranks
#   refsuite    the reference's own test suite with this engine hot-swapped in
#   launchlist  ncu launch list (time + DRAM bytes) of the default bench
#   zoo         per-kernel rates + ncu (tools/gpu_kernel_zoo.sh; NCU=1 for ncu)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
R=${1:?recipe}; TAG=${2:-x}; shift 2 2>/dev/null
summ() {  # one-line digest of a bench JSON line
  python -c "
import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); r=d.get('roofline') or {}; e=d.get('e2e') or {}; c=d.get('cpu_baseline') or {}
print('$2', round(d['value'],1), 'frac', r.get('frac') and round(r['frac'],4), 'e2e', e.get('value') and round(e['value'],2), 'cpu', c.get('value') and round(c['value'],3), c.get('kind'), d.get('parity'))"
}
MR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
case $R in
  round-end)
    timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_$TAG.log
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$TAG.log
    timeout 1200 python bench.py "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; summ gpurun_out/bench_$TAG.json bench
    timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2>&1; echo "ref rc=$?"; tail -c 400 gpurun_out/bench_ref_$TAG.json ;;
  tests)
    timeout 1500 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_$TAG.log ;;
  allcfg|stages)
    X=""; [ $R = stages ] && X="--unfused --no-cpu --no-e2e"
    for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
      timeout 1500 python bench.py --config $c --steps 5 $X "$@" > gpurun_out/${R}_${c}_$TAG.json 2> gpurun_out/${R}_${c}_$TAG.err; echo -n "rc=$? "; summ gpurun_out/${R}_${c}_$TAG.json $c
    done ;;
  repeat)
    for i in 1 2 3; do timeout 900 python bench.py "$@" > gpurun_out/rep${i}_$TAG.json 2>/dev/null; summ gpurun_out/rep${i}_$TAG.json run$i; done ;;
  e2e-sweep)
    for a in "--e2e-slots 2" "--e2e-slots 3" "--e2e-slots 4" "--e2e-window-gb 0.2" "--e2e-window-gb 0.8"; do
      timeout 600 python bench.py --steps 3 --no-cpu --no-verify $a > gpurun_out/e2e_$TAG.json 2>/dev/null
      python -c "
import json; d=json.loads(open('gpurun_out/e2e_$TAG.json').read().strip().splitlines()[-1]); e=d['e2e']; l=e.get('link',{})
print('$a', round(e['value'],2), round(l.get('h2d_GBps_in_step',0),1), round(l.get('frac',0),3))"
    done ;;
  file)
    timeout 900 python tools/file_bench.py --config cfg2 --layers 4 > gpurun_out/file_cfg2l4_$TAG.json 2>&1; echo "cfg2l4 rc=$?"; tail -c 500 gpurun_out/file_cfg2l4_$TAG.json
    timeout 600 python tools/file_bench.py --config cfg1 > gpurun_out/file_cfg1_$TAG.json 2>&1; echo "cfg1 rc=$?"; tail -c 500 gpurun_out/file_cfg1_$TAG.json ;;
  fileref)
    timeout 900 python tools/file_bench.py --config cfg1 --impl reference --reps 2 > gpurun_out/fileref_cfg1_$TAG.json 2>&1; echo "cfg1 rc=$?"; tail -c 500 gpurun_out/fileref_cfg1_$TAG.json ;;
  sanitize)
    K="${K:-reshard_plan_host_round_trip or union_reference_unit_cases or fused_replica_mismatch or shard_hy or run_pinned or file_pipeline_digests or fused_resume or corrupt_replica}"
    for tool in memcheck racecheck synccheck; do
      timeout 1500 compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
        python -m pytest ${FILES:-tests/test_gpu_parity.py tests/test_gpu_kernel_fuzz.py} -m gpu -x -q -k "$K" > gpurun_out/sanitize_${tool}_$TAG.log 2>&1
      echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_${tool}_$TAG.log | tail -3
    done ;;
  memcheck)
    timeout 3000 compute-sanitizer --tool memcheck --error-exitcode 99 --target-processes all \
      python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/memcheck_all_$TAG.log 2>&1
    echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/memcheck_all_$TAG.log | tail -5 ;;
  multirank)
    timeout 900 $MR --master-port 29541 bench.py --gpus 2 --dist-backend gloo --layers 4 --steps 3 "$@" > gpurun_out/mr_param_$TAG.json 2> gpurun_out/mr_param_$TAG.err; echo -n "param rc=$? "; summ gpurun_out/mr_param_$TAG.json param
    timeout 900 $MR --master-port 29542 bench.py --gpus 2 --dist-backend gloo --layers 4 --steps 3 --home rank --exchange peer "$@" > gpurun_out/mr_peer_$TAG.json 2> gpurun_out/mr_peer_$TAG.err; echo -n "peer rc=$? "; summ gpurun_out/mr_peer_$TAG.json peer
    timeout 900 $MR --master-port 29543 bench.py --gpus 2 --impl reference --steps 1 --warmup 1 > gpurun_out/mr_ref_$TAG.json 2> gpurun_out/mr_ref_$TAG.err; echo "ref rc=$?"; tail -c 300 gpurun_out/mr_ref_$TAG.json ;;
  srchome)
    A="--steps 5 --no-cpu --no-e2e"
    timeout 900 python bench.py $A --src-home rank --home rank > gpurun_out/sh1_$TAG.json 2>/dev/null; summ gpurun_out/sh1_$TAG.json "1 rank"
    timeout 900 $MR --master-port 29561 bench.py --gpus 2 --dist-backend gloo --layers 4 $A --src-home rank --home rank > gpurun_out/sh2_$TAG.json 2>/dev/null; summ gpurun_out/sh2_$TAG.json "2 ranks" ;;
  refsuite)
    if [ -d baseline/_ref_tests ]; then
      PYTHONPATH=baseline/_ref:.:tools timeout 2400 python -m pytest baseline/_ref_tests -p ref_suite_plugin -q -p no:cacheprovider -rf > gpurun_out/refsuite_$TAG.log 2>&1
      echo "swapped rc=$?"; tail -4 gpurun_out/refsuite_$TAG.log
      PYTHONPATH=baseline/_ref timeout 2400 python -m pytest baseline/_ref_tests -q -p no:cacheprovider -rf > gpurun_out/refsuite_unmodified_$TAG.log 2>&1
      echo "unmodified rc=$?"; tail -4 gpurun_out/refsuite_unmodified_$TAG.log
    fi ;;
  launchlist)
    timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu "$@" > gpurun_out/launches_$TAG.log 2>&1; echo "ncu rc=$?"; wc -l gpurun_out/launches_$TAG.csv ;;
  zoo)
    bash tools/gpu_kernel_zoo.sh $TAG "$@" ;;
  *) echo "unknown recipe $R"; exit 2 ;;
esac

#!/bin/bash
# usage: [NCU=1] tools/gpu_kernel_zoo.sh TAG [case ...]
# Per shipped kernel family (tools/kernel_zoo.py): CUDA-event rates (plain
# run); with NCU=1 also an ncu launch list and one ncu --set full capture of
# the family's first timed launches, exported on the box to CSV (details +
# raw pages) and the .ncu-rep deleted (gpurun copies back <= 64 MiB).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
TAG=${1:-x}; shift
CASES=${@:-fused_f32 fused_bf16 fused_f16 fused_staged fused_staged5 unfused_f32 unfused_bf16 unfused_f16 unfused_staged unfused_staged_load fused_staged_bf16 general_ops}
mkdir -p gpurun_out
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
for c in $CASES; do
  timeout 600 python tools/kernel_zoo.py --case $c > gpurun_out/zoo_${c}_$TAG.json 2> gpurun_out/zoo_${c}_$TAG.err
  echo "$c rc=$? $(python -c "import json,sys; d=json.load(open('gpurun_out/zoo_${c}_$TAG.json')); print({k: (round(v['GBps']), round(v['frac'], 3)) for k, v in d['stages'].items() if v['bytes'] > 1e6}, d['parity'])" 2>&1 | tail -1)"
  [ "${NCU:-0}" = "1" ] || continue
  timeout 600 ncu $M --log-file gpurun_out/zoo_${c}_$TAG.csv python tools/kernel_zoo.py --case $c --steps 2 > /dev/null 2>&1
  echo "  launches rc=$?"
  K=$(python -c "import sys; sys.path.insert(0,'tools'); import kernel_zoo as z; print('|'.join(z.CASES['$c'][5]))")
  R=gpurun_out/zoo_${c}_$TAG
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^($K)\$" -s ${NCU_S:-6} -c ${NCU_C:-2} -o $R python tools/kernel_zoo.py --case $c --steps 2 > ${R}_ncu.log 2>&1
  echo "  ncu rc=$?"
  ncu -i $R.ncu-rep --page details --csv > ${R}_details.csv 2>/dev/null
  ncu -i $R.ncu-rep --page raw --csv > ${R}_raw.csv 2>/dev/null
  [ "${KEEP_REP:-}" = "$c" ] || rm -f $R.ncu-rep
  du -sh gpurun_out | tail -1
done

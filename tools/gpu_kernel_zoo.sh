#!/bin/bash
# usage: tools/gpu_kernel_zoo.sh TAG [case ...]
# Per shipped kernel family (tools/kernel_zoo.py): CUDA-event rates (plain
# run), an ncu launch list, and one ncu --set full capture of the family's
# first timed launch. Outputs in gpurun_out/zoo_<case>_<TAG>.*
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
TAG=${1:-x}; shift
CASES=${@:-fused_f32 fused_bf16 fused_f16 fused_staged fused_staged5 unfused_f32 unfused_bf16 unfused_f16 unfused_staged general_ops}
mkdir -p gpurun_out
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
for c in $CASES; do
  timeout 600 python tools/kernel_zoo.py --case $c > gpurun_out/zoo_${c}_$TAG.json 2> gpurun_out/zoo_${c}_$TAG.err
  echo "$c rc=$? $(tail -c 600 gpurun_out/zoo_${c}_$TAG.json)"
  timeout 600 ncu $M --log-file gpurun_out/zoo_${c}_$TAG.csv python tools/kernel_zoo.py --case $c --steps 2 > /dev/null 2>&1
  echo "  launches rc=$?"
  K=$(python -c "import sys; sys.path.insert(0,'tools'); import kernel_zoo as z; print('|'.join(z.CASES['$c'][5]))")
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^($K)\$" -s ${NCU_S:-6} -c ${NCU_C:-2} -o gpurun_out/zoo_${c}_$TAG python tools/kernel_zoo.py --case $c --steps 2 > gpurun_out/zoo_${c}_${TAG}_ncu.log 2>&1
  echo "  ncu rc=$?"
done

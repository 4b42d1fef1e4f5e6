#!/bin/bash
# ncu --set full of every op the bench line reports as an extra (one capture
# per op, Reddit-shaped graph), summarised for profiles/. Run on the GPU box:
#   tools/profile_extras.sh TAG [op:feat ...]
set -u
TAG=${1:-r02}
shift || true
OPS=${@:-"softmax:8 softmax_bwd:8 umul_sum:602 dot_sddmm:16 copy_sum:16 copy_max:16"}
OUT=gpurun_out/prof_${TAG}
mkdir -p $OUT
for spec in $OPS; do
  op=${spec%%:*}; feat=${spec##*:}
  name=${op}_d${feat}
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -f -o /tmp/${name} python tools/run_op.py --op $op --feat $feat --reps 1 --warmup 1 --profile \
    > $OUT/${name}.log 2>&1
  ncu -i /tmp/${name}.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
  python tools/ncu_summary.py /tmp/${name}.ncu-rep > $OUT/${name}_summary.txt 2>&1
done
python tools/ncu_extras.py $OUT > $OUT/extras_traffic.json
ls -la $OUT

#!/bin/bash
# Profiles committed under profiles/ (run on the GPU box through gpurun):
#   usage: tools/profile_round.sh [ROUND_TAG]
#   launch list of the default bench command, full ncu capture of one
#   headline step (summaries only: the .ncu-rep stays in /tmp on the box).
set -u
OUT=gpurun_out/prof${1:+_$1}
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > $OUT/bench_under_ncu.log 2>&1
python tools/launch_summary.py $OUT/launches.csv 2 > $OUT/launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -o /tmp/step_full python tools/run_op.py --op copy_sum --feat 602 --reps 1 --warmup 1 --profile \
  > $OUT/step_full.log 2>&1
ncu -i /tmp/step_full.ncu-rep --page raw --csv > $OUT/step_raw.csv
python tools/ncu_summary.py /tmp/step_full.ncu-rep > $OUT/step_summary.txt
ls -la $OUT

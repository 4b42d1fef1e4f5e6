#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over the -m gpu parity
# suites that exercise every kernel family: row kernel (all phi x rho, hub
# rows over clusters with DSMEM merges, packed tiles), g-SDDMM, fused softmax
# (windowed statistics), fused GAT, extrema backward, sampling.
# Run on the GPU box: tools/sanitize.sh TAG
set -u
TAG=${1:-r02}
OUT=gpurun_out/sanitize_${TAG}
mkdir -p $OUT
SUITES=${SUITES:-"tests/test_gpu_parity.py tests/test_gpu_cluster.py tests/test_gpu_softmax_offsets.py tests/test_gpu_gat_fused.py tests/test_gpu_extrema_bwd.py tests/test_gpu_tiled.py tests/test_gpu_sampling.py tests/test_gpu_udf.py"}
for tool in memcheck racecheck synccheck; do
  for s in $SUITES; do
    b=$(basename $s .py)
    timeout ${SAN_TIMEOUT:-600} compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 99 \
      --target-processes all python -m pytest $s -m gpu -x -q -p no:cacheprovider \
      > $OUT/${tool}_${b}.log 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $OUT/${tool}_${b}.log | tail -1)
    res=$(grep -E "passed|failed" $OUT/${tool}_${b}.log | tail -1)
    echo "$tool $b rc=$rc | $summ | $res" | tee -a $OUT/summary.txt
  done
done

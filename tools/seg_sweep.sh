# segmented softmax statistics: parity tests, then Reddit H=8 timing per window budget
# usage: bash tools/seg_sweep.sh OUTDIR "seg mb" ...
out=${1:-gpurun_out/seg}; shift
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_softmax_window.py -q -x > $out/tests.log 2>&1; echo EXIT $? >> $out/tests.log
for cfg in "$@"; do set -- $cfg
  for op in softmax softmax_bwd; do
    GMP_SOFTMAX_SEG=$1 GMP_SOFTMAX_SEG_MB=$2 GMP_SOFTMAX_SEG_BWD=${3:-1} timeout 300 python tools/run_op.py --op $op --feat 8 --time --reps 10 --edge-cache /tmp/pl.npz 2>&1 | grep -v "^graph" | sed "s/^/seg=$1 mb=$2 bwdseg=${3:-1} /" >> $out/timing.log
  done
done

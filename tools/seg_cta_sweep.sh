# resident CTAs per SM of the segmented softmax statistics kernel (fwd and the
# opt-in segmented backward), Reddit H=8
out=${1:-gpurun_out/seg_cta}; mkdir -p $out
for ctas in 1 2 3 0; do
  for op in softmax softmax_bwd; do
    GMP_SOFTMAX_SEG_BWD=1 GMP_SOFTMAX_SEG_CTAS=$ctas timeout 300 python tools/run_op.py --op $op --feat 8 --time --reps 10 --edge-cache /tmp/pl.npz 2>&1 | grep -v "^graph" | sed "s/^/ctas=$ctas /" >> $out/timing.log
  done
done

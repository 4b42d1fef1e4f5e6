# ncu of the segmented softmax statistics kernel (fwd, then bwd: the bwd
# process runs one forward first, hence --launch-skip 1), one launch each
out=${1:-gpurun_out/seg_ncu}; mkdir -p $out
python tools/run_op.py --op softmax --feat 8 --reps 1 --edge-cache /tmp/pl.npz > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:edge_softmax_seg_kernel -c 1 \
  -o $out/seg_softmax python tools/run_op.py --op softmax --feat 8 --reps 1 --edge-cache /tmp/pl.npz > $out/ncu_softmax.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:edge_softmax_seg_kernel --launch-skip 1 -c 1 \
  -o $out/seg_softmax_bwd python tools/run_op.py --op softmax_bwd --feat 8 --reps 1 --edge-cache /tmp/pl.npz > $out/ncu_softmax_bwd.log 2>&1

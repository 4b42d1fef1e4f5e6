# ncu of the softmax extras (current code) + compute-sanitizer memcheck of the
# segmented statistics tests
mkdir -p gpurun_out/s16
bash tools/profile_extras.sh r02d softmax:8 softmax_bwd:8 > gpurun_out/s16/prof.log 2>&1
for tool in memcheck synccheck; do
timeout 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 99 --target-processes all \
  python -m pytest tests/test_gpu_softmax_window.py -k small_graph -m gpu -x -q -p no:cacheprovider \
  > gpurun_out/s16/${tool}_seg.log 2>&1; echo "$tool rc=$?" >> gpurun_out/s16/sanitize_summary.txt
grep -E "ERROR SUMMARY|passed|failed" gpurun_out/s16/${tool}_seg.log | tail -2 >> gpurun_out/s16/sanitize_summary.txt
done

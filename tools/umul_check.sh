# u_mul_e product accumulate: parity suites + Reddit d=602 timing vs copy_u
out=${1:-gpurun_out/umul}; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipe.py tests/test_gpu_tiled.py tests/test_gpu_ring.py tests/test_gpu_gat_fused.py tests/test_gpu_configs.py -m gpu -q -x > $out/tests.log 2>&1; echo EXIT $? >> $out/tests.log
for op in umul_sum copy_sum; do
  timeout 600 python tools/run_op.py --op $op --feat 602 --time --reps 5 --edge-cache /tmp/pl.npz 2>&1 | grep -v "^graph" >> $out/timing.log
done

# u_dot_v g-SDDMM (lane kernel): parity + Reddit d=16 timing
out=${1:-gpurun_out/dot}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -k "sddmm or dot or golden" > $out/tests.log 2>&1; echo EXIT $? >> $out/tests.log
timeout 600 python tools/run_op.py --op dot_sddmm --feat 16 --time --reps 10 --edge-cache /tmp/pl.npz 2>&1 | grep -v "^graph" >> $out/timing.log

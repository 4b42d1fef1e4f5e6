# Time the packed-tile g-SpMM (copy_u / u_mul_e + sum, d=602, Reddit-shaped)
# with the pipelined ring and with the burst kernel (GMP_NO_PIPE=1).
cd $GRAFT_REPO_ROOT
C=/tmp/pl_edges.npz
for op in ${OPS:-copy_sum umul_sum}; do
 for v in pipe nopipe; do
  if [ $v = nopipe ]; then E="GMP_NO_PIPE=1"; else E="GMP_X=1"; fi
  echo "== $op $v"
  env $E timeout 300 python tools/run_op.py --op $op --feat ${FEAT:-602} --reps 5 --time --edge-cache $C 2>&1 | tail -1
 done
done

# time copy_u / u_mul_e + sum (d=602, Reddit-shaped) for each library in $LIBS
# under each environment setting in $ENVS (space-separated, "-" = none)
cd $GRAFT_REPO_ROOT
C=/tmp/pl_edges.npz
for op in ${OPS:-copy_sum umul_sum}; do
 for L in ${LIBS:-paper_1909_01315_b200/libgmp.so}; do
  for E in ${ENVS:--}; do
   [ "$E" = "-" ] && E="GMP_X=1"
   echo "== $op $L $E"
   env $E GMP_LIB=$L timeout 300 python tools/run_op.py --op $op --feat ${FEAT:-602} --reps 5 --time --edge-cache $C 2>&1 | tail -1
  done
 done
done

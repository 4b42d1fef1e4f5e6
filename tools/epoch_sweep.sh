# time the d=16 aggregations and the GNN epochs for each library in $LIBS
# under each environment setting in $ENVS ("-" = none)
cd $GRAFT_REPO_ROOT
C=/tmp/pl_edges.npz
for L in ${LIBS:-paper_1909_01315_b200/libgmp.so}; do
 for E in ${ENVS:--}; do
  [ "$E" = "-" ] && E="GMP_X=1"
  for spec in ${SPECS:-copy_sum:16 umul_sum:16 gcn_epoch:602 gat_epoch:602}; do
   op=${spec%%:*}; feat=${spec##*:}
   printf "%s %s %s: " "$L" "$E" "$spec"
   env $E GMP_LIB=$L timeout 300 python tools/run_op.py --op $op --feat $feat --reps 5 --time --edge-cache $C 2>&1 | tail -1 | sed 's/.*median/median/'
  done
 done
done

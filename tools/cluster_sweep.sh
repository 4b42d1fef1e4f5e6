# headline op under forced heavy-row cluster sizes (GMP_CLUSTER)
cd $GRAFT_REPO_ROOT
C=/tmp/pl_edges.npz
for op in ${OPS:-copy_sum}; do
 for cl in 0 2 4; do
  echo "== $op cluster=$cl"
  GMP_CLUSTER=$cl timeout 300 python tools/run_op.py --op $op --feat ${FEAT:-602} --reps 5 --time --edge-cache $C 2>&1 | tail -1
 done
done

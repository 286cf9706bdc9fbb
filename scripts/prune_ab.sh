# A/B of the gi near-best pruning (TCSE_GI_PRUNE=1 default vs 0), results-invariant
cd ${GRAFT_REPO_ROOT:-.}
for spec in "sxs 16384 4" "laderman 4096 6" "naive555_f1000 8192 3" "sxs_border 8192 4"; do
  for r in 1 2; do
    for pr in 1 0; do
      echo -n "[prune=$pr] "; TCSE_GI_PRUNE=$pr timeout 120 python scripts/probe_perf.py $spec 2>&1 | tail -1
    done
  done
done

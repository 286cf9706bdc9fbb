cd $GRAFT_REPO_ROOT
for spec in "laderman 4096 6 greedy_intersections" "sxs 16384 4" "sxs 16384 4 greedy_intersections"; do
 for r in 1 2; do for t in 1 24 40 64 96; do echo -n "[$t] "; TCSE_GI_PRUNE=$t python scripts/probe_perf.py $spec 2>&1 | tail -1 | sed 's/ wall_ms.*-> / -> /; s/costs=.*//'; done; done
done

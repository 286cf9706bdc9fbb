# A/B of the two exact Greedy-Intersections forms (TCSE_GI_DENSE=1 dense
# reference loop, 0 O(deg) walk) on given probe specs
for spec in "$@"; do
  for rep in 1 2; do
    for d in 1 0; do echo -n "[dense=$d] "; TCSE_GI_DENSE=$d python scripts/probe_perf.py $spec; done
  done
done

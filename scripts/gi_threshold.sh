# sweep of the dense/walk switch point (TCSE_GI_DENSE_MAX, results-invariant)
for spec in "$@"; do
  for t in 128 256 384 512 1024; do echo -n "[max=$t] "; TCSE_GI_DENSE_MAX=$t python scripts/probe_perf.py $spec; done
done

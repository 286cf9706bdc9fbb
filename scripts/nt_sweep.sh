for spec in "sxs 16384 4" "sxs_border 8192 4" "naive555_f1000 8192 4"; do
  for rep in 1 2; do
    for nt in 0 32 64 128; do echo -n "[nt=$nt] "; TCSE_NT=$nt python scripts/probe_perf.py $spec 2>&1 | tail -1; done
  done
done

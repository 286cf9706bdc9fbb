# block-size sweep (TCSE_NT, results-invariant; 0 = automatic choice)
# usage: scripts/nt_sweep.sh "nt list" "spec" ...
nts=$1; shift
for spec in "$@"; do
  for rep in 1 2; do
    for nt in $nts; do echo -n "[nt=$nt] "; TCSE_NT=$nt python scripts/probe_perf.py $spec 2>&1 | tail -1; done
  done
done

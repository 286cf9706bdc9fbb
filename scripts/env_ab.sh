# A/B of results-invariant env knobs: scripts/env_ab.sh "ENV1=a ENV2=b|ENV1=c" "spec" ...
variants=$1; shift
IFS='|' read -ra VS <<< "$variants"
for spec in "$@"; do
  for rep in 1 2; do
    for v in "${VS[@]}"; do echo -n "[$v] "; env $v python scripts/probe_perf.py $spec 2>&1 | tail -1; done
  done
done

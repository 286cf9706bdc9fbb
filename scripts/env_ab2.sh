# A/B over libraries x env settings: bash scripts/env_ab2.sh "libs" "envs" spec...   (env "-" = none)
cd ${GRAFT_REPO_ROOT:-.}
libs=$1; envs=$2; shift 2
for spec in "$@"; do
  for rep in 1 2; do
    for l in $libs; do
      for e in $envs; do
        lp=""; [ "$l" != cur ] && lp=ab/$l.so
        ee=""; [ "$e" != "-" ] && ee=$e
        echo -n "[$l $e] "; env TCSE_LIBRARY=$lp $ee timeout 120 python scripts/probe_perf.py $spec 2>&1 | tail -1 | sed -e 's/ wall_ms=[0-9.]*//' -e 's/ forced=None//' -e 's/costs=.*//'
      done
    done
  done
done

# A/B probe: bash scripts/ab_run.sh "libs" spec...   (lib "cur" = in-tree build)
libs=$1; shift
for spec in "$@"; do
  for rep in 1 2; do
    for l in $libs; do
      if [ "$l" = cur ]; then lp=""; else lp=ab/$l.so; fi
      echo -n "[$l] "; TCSE_LIBRARY=$lp python scripts/probe_perf.py $spec 2>&1 | sed 's/ wall_ms.*-> / -> /'
    done
  done
done

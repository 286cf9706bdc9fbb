#!/bin/bash
# A/B throughput: for each "scheme N iters [strategy]" spec, probe every given library.
# usage: scripts/ab_probe.sh "lib1 lib2 ..." "spec1" "spec2" ...
libs=$1; shift
for spec in "$@"; do
  for rep in 1 2; do
    for l in $libs; do
      if [ "$l" = cur ]; then lp=""; else lp=ab/$l.so; fi
      echo -n "[$l] "; TCSE_LIBRARY=$lp python scripts/probe_perf.py $spec
    done
  done
done

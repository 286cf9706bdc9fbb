cd $GRAFT_REPO_ROOT
for spec in "sxs 16384 4" "laderman 4096 6" "naive555_f1000 8192 3" "sxs_border 8192 4"; do
  for mode in default walk dense; do
    if [ $mode = walk ]; then export TCSE_GI_DENSE=0; elif [ $mode = dense ]; then export TCSE_GI_DENSE=1; else unset TCSE_GI_DENSE; fi
    echo -n "[$mode] "; timeout 120 python scripts/probe_perf.py $spec 2>&1 | tail -1
  done
done

# ncu --set full of the W-group search kernel (sxs, iteration 2) for each "name:lib:env" spec
cd ${GRAFT_REPO_ROOT:-.}
for spec in "$@"; do
  name=${spec%%:*}; rest=${spec#*:}; lib=${rest%%:*}; envs=${rest#*:}
  lp=""; [ "$lib" != cur ] && lp=ab/$lib.so
  env TCSE_LIBRARY=$lp $envs ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k 'regex:search_kernel<\(int\)1, \(int\)64' --launch-skip 2 --launch-count 1 \
    -o gpurun_out/$name python scripts/profile_step.py ${SCHEME:-sxs} ${NPROC:-16384} 2 > gpurun_out/$name.log 2>&1
done

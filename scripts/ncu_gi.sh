#!/bin/bash
# ncu capture of the W-group search kernel (iteration 2) for a forced strategy.
# usage: scripts/ncu_gi.sh scheme N strategy out_name [kernel_regex]
scheme=$1; N=$2; strat=$3; out=$4; kre=${5:-"search_kernel<1, 64"}
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:$kre" --launch-skip ${6:-2} --launch-count 1 \
    -o gpurun_out/$out python scripts/profile_step.py $scheme $N 2 $strat > gpurun_out/$out.log 2>&1

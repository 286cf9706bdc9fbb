# Per-config evidence on one GPU: bench line of each BASELINE config, the
# launch list of the headline bench command, and ncu --set full captures of
# the dominant search kernel of configs 1 and 4.
# usage: bash scripts/evidence_cfg.sh TAG   -> gpurun_out/TAG_*
cd ${GRAFT_REPO_ROOT:-.}
tag=${1:-v}
for c in 0 1 3 4; do timeout 900 python bench.py --config $c > gpurun_out/${tag}_bench_cfg$c.json 2> gpurun_out/${tag}_bench_cfg$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${tag}_ncu_bench.log 2>&1
# config 1: laderman forced gi, all systems in one NT=32 group; skip the 3 dump launches + iteration 1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:search_kernel<\(int\)1, \(int\)32' --launch-skip 4 --launch-count 1 \
  -o gpurun_out/${tag}_cfg1_search python scripts/profile_step.py laderman 4096 3 greedy_intersections > gpurun_out/${tag}_cfg1_search.log 2>&1
# config 4: sxl, the U/V group (W = 3 words, NT = 256, O(deg) walk), iteration 2
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:search_kernel<\(int\)3' --launch-skip 3 --launch-count 1 \
  -o gpurun_out/${tag}_cfg4_search python scripts/profile_step.py sxl 8192 2 > gpurun_out/${tag}_cfg4_search.log 2>&1

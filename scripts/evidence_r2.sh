# Round-2 evidence on one GPU -> gpurun_out/TAG_*:
#   GPU tests, the driver's bench command, every BASELINE config (the
#   reference arm at the same process count for configs 3 and 4), the launch
#   list of the headline command, ncu --set full of the dominant search
#   kernel of configs 2 (W group), 1 and 4 (W group), the pipe microbenchmark.
cd ${GRAFT_REPO_ROOT:-.}
tag=${1:-r2}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu_tests.log 2>&1; echo EXIT $? >> gpurun_out/${tag}_gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 600 python bench.py --config 0 > gpurun_out/${tag}_bench_cfg0.json 2> gpurun_out/${tag}_bench_cfg0.err
timeout 600 python bench.py --config 1 --steps 50 --warmup 5 > gpurun_out/${tag}_bench_cfg1.json 2> gpurun_out/${tag}_bench_cfg1.err
timeout 600 python bench.py --config 3 > gpurun_out/${tag}_bench_cfg3.json 2> gpurun_out/${tag}_bench_cfg3.err
timeout 900 python bench.py --config 4 --steps 2 --warmup 1 > gpurun_out/${tag}_bench_cfg4.json 2> gpurun_out/${tag}_bench_cfg4.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${tag}_ref_cfg2.json 2> gpurun_out/${tag}_ref_cfg2.err
timeout 900 python bench.py --impl reference --config 3 > gpurun_out/${tag}_ref_cfg3.json 2> gpurun_out/${tag}_ref_cfg3.err
timeout 1500 python bench.py --impl reference --config 4 --steps 2 --warmup 1 > gpurun_out/${tag}_ref_cfg4.json 2> gpurun_out/${tag}_ref_cfg4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:search_kernel<\(int\)1, \(int\)64' --launch-skip 2 --launch-count 1 \
  -o gpurun_out/${tag}_search python scripts/profile_step.py sxs 16384 2 > gpurun_out/${tag}_search.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:search_kernel<\(int\)1, \(int\)32' --launch-skip 4 --launch-count 1 \
  -o gpurun_out/${tag}_cfg1_search python scripts/profile_step.py laderman 4096 3 greedy_intersections > gpurun_out/${tag}_cfg1_search.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:search_kernel<\(int\)1, \(int\)256' --launch-skip 2 --launch-count 1 \
  -o gpurun_out/${tag}_cfg4_search python scripts/profile_step.py sxl 8192 2 > gpurun_out/${tag}_cfg4_search.log 2>&1
python -c "
import json, sys; sys.path.insert(0, '.')
import paper_2512_13365_b200 as T
d = T.Device(0)
print(json.dumps({'wordops_gops': d.microbench_wordops(), 'pipes_gops': d.microbench_pipes()}))" > gpurun_out/${tag}_pipes.json 2>&1

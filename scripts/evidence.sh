# Round evidence on one GPU: gpu tests, bench line (config 2), launch list of
# the same command, ncu --set full of the headline W-group search kernel.
# usage: bash scripts/evidence.sh TAG   -> gpurun_out/TAG_*
cd ${GRAFT_REPO_ROOT:-.}
tag=${1:-v}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu_tests.log 2>&1; echo EXIT $? >> gpurun_out/${tag}_gpu_tests.log
timeout 400 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${tag}_ncu_bench.log 2>&1
bash scripts/ncu_ab.sh "${tag}_search:cur:X=1"
if [ -n "$ALLCFG" ]; then
  for c in 0 1 3 4; do timeout 600 python bench.py --config $c > gpurun_out/${tag}_bench_cfg$c.json 2> gpurun_out/${tag}_bench_cfg$c.err; done
fi
if [ -n "$WALL" ]; then
  timeout 900 python scripts/wall_budget.py > gpurun_out/${tag}_wall_budget.log 2>&1
fi

cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python -m pytest tests/test_gpu_giforms.py tests/test_gpu_parity.py tests/test_gpu_bigconfigs.py tests/test_gpu_stress.py -x -q > gpurun_out/s3_tests.log 2>&1; echo EXIT $? >> gpurun_out/s3_tests.log
bash scripts/ab_run.sh "base cur" "sxs 16384 4" "sxs 16384 4 greedy_intersections" "laderman 4096 6 greedy_intersections" "naive555_f1000 8192 3" > gpurun_out/s3_ab.txt 2>&1

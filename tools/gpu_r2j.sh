cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_solve.py -q -p no:cacheprovider -k "lasso_wide or config4 or config2" > gpurun_out/pytest_r2j.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2j.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_cfg4_r2j.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg4_r2j.log
NYS_TAIL_CLUSTER_OFF=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_cfg4_off_r2j.log 2>&1

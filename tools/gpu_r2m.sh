cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_solve.py -q -p no:cacheprovider -k "pinned or cfg1 or small_cases" > gpurun_out/pytest_r2m.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2m.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_cfg4_r2m.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg4_r2m.log

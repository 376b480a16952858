cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_solve.py -q -p no:cacheprovider -k "config5_shard or config4" > gpurun_out/pytest_r2i.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2i.log
timeout 1200 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_cfg5_r2i.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg5_r2i.log

cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solve.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_ah.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ah.log
for c in 2 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bah$c.log 2>&1; done

cd $GRAFT_REPO_ROOT
{
timeout 120 python tools/tail_bench.py 20000 100000 10 square
timeout 120 python tools/tail_bench.py 5000 10000 50 square
} > gpurun_out/h_tail.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "ml_tail" > gpurun_out/h_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/h_pytest.log
timeout 1200 python -m pytest tests/test_gpu_solve.py -m gpu -q -p no:cacheprovider -k "cfg4 or lasso or cfg1" > gpurun_out/h_pytest2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/h_pytest2.log
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/h_b4.log 2>&1

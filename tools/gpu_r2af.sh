cd $GRAFT_REPO_ROOT
{
timeout 120 python tools/tail_bench.py 5000 10000 50 logistic 2>&1 | grep cluster
timeout 120 python tools/tail_bench.py 5000 10000 50 square 2>&1 | grep cluster
timeout 120 python tools/tail_bench.py 20000 100000 10 square 2>&1 | grep cluster
timeout 120 python tools/tail_bench.py 20000 100000 10 logistic 2>&1 | grep cluster
} > gpurun_out/tail_af.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "ml_tail" > gpurun_out/pytest_af.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_af.log
for c in 2 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/baf$c.log 2>&1; done

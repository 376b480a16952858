cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solve.py -q -p no:cacheprovider -k "hvp or ml_tail or wide or config4 or cfg1" > gpurun_out/pytest_r2n.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2n.log
timeout 300 python tools/tail_bench.py 20000 100000 10 square > gpurun_out/tail_bench_r2n.log 2>&1
for shape in "20000 100000 10" "12500 200000 10"; do timeout 300 python tools/hvp_bench.py $shape >> gpurun_out/tail_bench_r2n.log 2>&1; done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_cfg4_r2n.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg4_r2n.log

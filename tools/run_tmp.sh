cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider -k "dgemm or sketch or nystrom or orthonorm" > gpurun_out/u7_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/u7_tests.log
tail -3 gpurun_out/u7_tests.log
{
timeout 300 python tools/gemm_bench.py 20000 100000 258
timeout 300 python tools/gemm_bench.py 5000 10000 133
timeout 300 python tools/gemm_bench.py 12500 200000 390
} 2>&1 | grep -v Capab | tee gpurun_out/u7_gemm.log

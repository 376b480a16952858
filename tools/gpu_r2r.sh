cd $GRAFT_REPO_ROOT
for c in 4 8 16; do NYS_TAIL_MIN_N=4096 NYS_TAIL_C=$c timeout 300 python tools/tail_bench.py 5000 10000 20 logistic >> gpurun_out/tail_mid.log 2>&1; done
for c in 4 8; do NYS_TAIL_MIN_N=4096 NYS_TAIL_C=$c timeout 300 python tools/tail_bench.py 5000 10000 20 square >> gpurun_out/tail_mid.log 2>&1; done
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/b2_base.log 2>&1
NYS_TAIL_MIN_N=4096 NYS_TAIL_C=4 timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/b2_c4.log 2>&1
NYS_TAIL_MIN_N=4096 NYS_TAIL_C=8 timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/b2_c8.log 2>&1
NYS_TAIL_MIN_N=4096 NYS_TAIL_C=4 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solve.py -q -p no:cacheprovider -k "ml_tail or cfg2 or config2 or logistic" > gpurun_out/pytest_mid.log 2>&1

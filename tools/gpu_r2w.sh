cd $GRAFT_REPO_ROOT
NYS_CP_PROBE=1 timeout 300 python tools/cp_probe.py 2 > gpurun_out/cpp_w2.log 2>&1
NYS_CP_PROBE=1 timeout 300 python tools/cp_probe.py 1 > gpurun_out/cpp_w1.log 2>&1
for c in 2 1 3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bw$c.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_w.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_w.log

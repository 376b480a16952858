cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "hvp" > gpurun_out/pytest_r2g.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2g.log
for shape in "12500 200000 10" "20000 100000 10" "6000 150000 10"; do
  timeout 300 python tools/hvp_bench.py $shape >> gpurun_out/hvp_r2g.log 2>&1
  NYS_HVP_CLUSTER_NOQ=1 timeout 300 python tools/hvp_bench.py $shape >> gpurun_out/hvp_r2g.log 2>&1
done

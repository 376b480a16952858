cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_general.py tests/test_gpu_solve.py -q -p no:cacheprovider -k "general or sparse or check_rank or unsupported or csr or structured or spectrum or error_norm or diagonal" > gpurun_out/pytest_r2e.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2e.log

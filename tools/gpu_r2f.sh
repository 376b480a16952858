cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_r2f.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2f.log

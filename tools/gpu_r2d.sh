cd $GRAFT_REPO_ROOT
timeout 300 python tools/cg_refresh_probe.py > gpurun_out/dbg3.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_r2d.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2d.log

cd $GRAFT_REPO_ROOT
timeout 300 python tools/cg_refresh_probe.py > gpurun_out/dbg2.log 2>&1

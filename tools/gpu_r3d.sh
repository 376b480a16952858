cd $GRAFT_REPO_ROOT
timeout 300 python tools/setup_prof.py 1 > gpurun_out/d_setup1.log 2>&1

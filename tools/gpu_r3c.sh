cd $GRAFT_REPO_ROOT
timeout 300 python tools/pyprof_solve.py 1 > gpurun_out/c_pyprof1.log 2>&1
timeout 300 python tools/hostprof.py 1 > gpurun_out/c_hostprof1.log 2>&1

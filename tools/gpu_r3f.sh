cd $GRAFT_REPO_ROOT
timeout 300 python tools/launch_timeline.py 1 > gpurun_out/f_lt1.log 2>&1

cd $GRAFT_REPO_ROOT
for c in 2 3 1; do timeout 300 python tools/trace_solve.py --config $c > gpurun_out/trace_y$c.log 2>&1; done
timeout 300 python tools/profile_solve.py --config 2 --families hvp > gpurun_out/prof_y2.log 2>&1

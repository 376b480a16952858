cd $GRAFT_REPO_ROOT
for c in 1 2 4; do timeout 600 python tools/trace_solve.py --config $c --seq 6 --json gpurun_out/b_trace$c.json > gpurun_out/b_trace$c.log 2>&1; done

cd $GRAFT_REPO_ROOT
NYS_CP_PROBE=1 timeout 300 python tools/cp_probe.py 2 > gpurun_out/cpp_x2.log 2>&1
for c in 2 1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bx$c.log 2>&1; done

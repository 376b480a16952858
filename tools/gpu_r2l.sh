cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --config 1 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_cfg1_r2l.log 2>&1
timeout 300 python tools/hostprof.py 1 > gpurun_out/hostprof_cfg1.log 2>&1
timeout 300 python tools/pyprof_solve.py 1 > gpurun_out/pyprof_cfg1.log 2>&1
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_cfg2_r2l.log 2>&1
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_cfg3_r2l.log 2>&1

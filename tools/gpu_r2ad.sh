cd $GRAFT_REPO_ROOT
for c in 2 1; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bad$c.log 2>&1
NYS_TAIL_MIN_N=1000 NYS_TAIL_C=2 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bad${c}_c2.log 2>&1
NYS_TAIL_MIN_N=1000 NYS_TAIL_C=4 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bad${c}_c4.log 2>&1
done
NYS_TAIL_MIN_N=1000 NYS_TAIL_C=2 timeout 300 python tools/trace_solve.py --config 2 > gpurun_out/trace_ad2.log 2>&1

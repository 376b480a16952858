cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/b2_base.log 2>&1
NYS_TAIL_MIN_N=4096 NYS_TAIL_C=4 timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/b2_c4.log 2>&1
NYS_TAIL_MIN_N=4096 NYS_TAIL_C=8 timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/b2_c8.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/b4.log 2>&1

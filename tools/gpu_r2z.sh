cd $GRAFT_REPO_ROOT
for C in 4 8 16; do echo "C=$C"; NYS_TAIL_MIN_N=1000 NYS_TAIL_C=$C timeout 120 python tools/tail_bench.py 5000 10000 50 logistic; done > gpurun_out/tailc_z.log 2>&1
for C in 8 16; do NYS_TAIL_MIN_N=1000 NYS_TAIL_C=$C timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bz2_c$C.log 2>&1; done

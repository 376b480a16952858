cd $GRAFT_REPO_ROOT
NYS_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 1 --warmup 3 > gpurun_out/bench_g2_gloo.log 2>&1; echo "rc=$?" >> gpurun_out/bench_g2_gloo.log
NYS_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config 5 --steps 1 --warmup 3 > gpurun_out/bench_g2_cfg5_gloo.log 2>&1; echo "rc=$?" >> gpurun_out/bench_g2_cfg5_gloo.log
timeout 900 python bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/bench_g2_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_g2_ref.log

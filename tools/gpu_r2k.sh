cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_r2k.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2k.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg4_r2k.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg4_r2k.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/cfg4_launches_r2k.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_list_r2k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hvp_cluster_kernel -s 3 -c 1 -o gpurun_out/cfg4_hvp_cluster_r2k python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_hvp_r2k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_cluster_kernel -s 3 -c 1 -o gpurun_out/cfg4_tail_cluster_r2k python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_tail_r2k.log 2>&1

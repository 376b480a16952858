cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_r2t.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2t.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hvp_cluster_kernel -s 3 -c 1 -o gpurun_out/r2t_hvp python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_hvp_r2t.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tail_cluster_kernel -s 3 -c 1 -o gpurun_out/r2t_tail python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_tail_r2t.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hvp_cluster_q_kernel -s 2 -c 1 -o gpurun_out/r2t_hvpq python tools/hvp_bench.py 12500 200000 3 > gpurun_out/ncu_hvpq_r2t.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2t_cfg4_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_list_r2t.log 2>&1

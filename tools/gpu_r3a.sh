cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/a_smi.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/a_pytest.log
timeout 900 python bench.py > gpurun_out/a_bench4.log 2>&1; echo "rc=$?" >> gpurun_out/a_bench4.log
for c in 1 2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/a_bench$c.log 2>&1; done

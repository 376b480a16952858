cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r2b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2b.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_r2b.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_cfg4_r2b.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg4_r2b.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_cfg4_r2b.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_cfg4_r2b.log
lscpu > gpurun_out/lscpu.txt; free -g >> gpurun_out/lscpu.txt

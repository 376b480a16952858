cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_r2v.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2v.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/b4v.log 2>&1
NYS_DEVICE_STOP=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/b4v_off.log 2>&1
timeout 600 python bench.py --config 1 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/b1v.log 2>&1
NYS_DEVICE_STOP=0 timeout 600 python bench.py --config 1 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/b1v_off.log 2>&1

cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/u3_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/u3_tests.log
timeout 600 python bench.py --config 5 --steps 2 --warmup 1 --no-cpu > gpurun_out/u3_bench5.json 2> gpurun_out/u3_bench5.err
timeout 900 python tools/trace_solve.py --config 5 --json gpurun_out/u3_trace5.json > gpurun_out/u3_trace5.log 2>&1
tail -3 gpurun_out/u3_tests.log; cat gpurun_out/u3_bench5.json

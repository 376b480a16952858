cd $GRAFT_REPO_ROOT
{
timeout 120 python tools/tail_probe.py 5000 10000 logistic
timeout 120 python tools/tail_probe.py 5000 10000 square
timeout 120 python tools/tail_probe.py 20000 100000 square
timeout 120 python tools/tail_bench.py 5000 10000 50 logistic 2>&1 | grep cluster
timeout 120 python tools/tail_bench.py 20000 100000 10 square 2>&1 | grep cluster
} > gpurun_out/tail_ag.log 2>&1

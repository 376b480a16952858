# HVP launch timing sweep over the wide-row kernels (run on the GPU box)
python tools/hvp_bench.py 20000 100000 20 nod
python tools/hvp_bench.py 20000 100000 20
for lag in 1 3; do NYS_HVP_CLUSTER_LAG=$lag python tools/hvp_bench.py 20000 100000 20 nod; done
NYS_HVP_CLUSTER_OFF=1 python tools/hvp_bench.py 20000 100000 20 nod
python tools/hvp_bench.py 12500 200000 10 nod
python tools/hvp_bench.py 20000 30000 20 nod

# HVP launch timing sweep over the wide-row kernels (run on the GPU box)
for lag in 1 2; do for sh in "20000 30000" "20000 60000" "20000 100000" "20000 140000"; do echo "lag $lag"; NYS_HVP_CLUSTER_LAG=$lag python tools/hvp_bench.py $sh 20; done; done

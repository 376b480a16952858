# HVP launch timing sweep over the strip-kernel knobs (run on the GPU box)
for cfg in "20000 100000" "12500 200000"; do
  for m in 0 2; do for lag in 2 3; do echo "== $cfg mode$m lag $lag"; NYS_STRIP_MODE=$m NYS_STRIP_LAG=$lag python tools/hvp_bench.py $cfg 20; done; done
  echo "== twopass"; NYS_HVP_TWOPASS=1 python tools/hvp_bench.py $cfg 20
done

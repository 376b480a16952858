cd $GRAFT_REPO_ROOT
for c in 1 2; do timeout 300 python tools/spin_prof.py $c; done > gpurun_out/e_spin.log 2>&1
NYS_LOOKAHEAD=0 timeout 300 python tools/spin_prof.py 1 >> gpurun_out/e_spin.log 2>&1

cd $GRAFT_REPO_ROOT
for c in lasso_rho_lo logistic_rho_lo; do
 timeout 120 python tools/debug_case.py $c
 NYS_CG_PERSIST_OFF=1 timeout 120 python tools/debug_case.py $c
 NYS_LOOKAHEAD=0 timeout 120 python tools/debug_case.py $c
done > gpurun_out/dbg1.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_r2c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2c.log

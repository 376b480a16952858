cd $GRAFT_REPO_ROOT
NYS_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config 4 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/v2_bench4_n2.json 2> gpurun_out/v2_bench4_n2.err
NYS_DIST_BACKEND=gloo timeout 1500 python bench.py --gpus 2 --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/v2_bench5_n2.json 2> gpurun_out/v2_bench5_n2.err
for f in gpurun_out/v2_bench4_n2 gpurun_out/v2_bench5_n2; do tail -2 $f.err; python -c "
import json;d=json.load(open('$f.json'));print(d['n_gpus'],d['value'],d['result'])"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/v2_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/v2_ncu_bench.log 2>&1
python tools/ncu_launch_summary.py gpurun_out/v2_launches.csv 30 > gpurun_out/v2_launch_summary.txt; head -12 gpurun_out/v2_launch_summary.txt

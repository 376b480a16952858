cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/u9_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/u9_tests.log
tail -3 gpurun_out/u9_tests.log
for c in 4 2 1 3 5; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/u9_bench$c.json 2> gpurun_out/u9_bench$c.err
python -c "
import json;d=json.load(open('gpurun_out/u9_bench$c.json'));print($c,d['value'],d['result'],d.get('e2e',{}).get('value'),d['roofline']['frac'],d['clocks'])"
done

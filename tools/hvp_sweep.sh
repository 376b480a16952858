# HVP launch timing sweep over the strip-kernel knobs (run on the GPU box)
python tools/hvp_bench.py 20000 100000 20
python tools/hvp_bench.py 20000 100000 20 nod
NYS_HVP_TWOPASS=1 python tools/hvp_bench.py 20000 100000 20 nod
NYS_STRIP_FORCE=1 python tools/hvp_bench.py 12500 200000 20 nod
NYS_STRIP_FORCE=1 NYS_STRIP_MODE=2 NYS_STRIP_LAG=3 python tools/hvp_bench.py 12500 200000 20 nod
NYS_HVP_TWOPASS=1 python tools/hvp_bench.py 12500 200000 20 nod
python tools/hvp_bench.py 5000 10000 50

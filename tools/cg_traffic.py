"""Operator applications per x-update PCG launch of a short config solve, for
pairing with an ncu launch list of cg_persist_kernel (dram bytes per launch):

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:cg_persist \\
        --csv --log-file out.csv python tools/cg_traffic.py 2 6 > units.txt
    python tools/cg_traffic.py --combine out.csv units.txt   # bytes per application
"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(cfg, iters):
    import torch

    import bench
    import paper_2310_08333_b200 as nys
    from paper_2310_08333_b200 import _lib
    from paper_2310_08333_b200.admm import _Engine

    units = []
    orig = _Engine._retire

    def retire(self, it, nxt):
        out = orig(self, it, nxt)
        units.append(int(self.rbs_host[it.par][8 + _lib.CG_NHVP]))
        return out

    _Engine._retire = retire
    d, opts = bench.build_problem(cfg)
    opts.max_iter = iters
    A = torch.from_numpy(d.A).cuda()
    nys.solve(bench.make_gpu_problem(d, A), opts)
    torch.cuda.synchronize()
    print(json.dumps(units))


def combine(csv_path, units_path):
    units = json.loads(open(units_path).read().strip().splitlines()[-1])
    rows = list(csv.reader(open(csv_path)))
    hi = [i for i, r in enumerate(rows) if "Metric Name" in r][0]
    h = rows[hi]
    ii, mi, vi, ui = h.index("ID"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = {}
    for r in rows[hi + 1:]:
        v = float(r[vi].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ui], 1)
        per.setdefault(int(r[ii]), 0.0)
        per[int(r[ii])] += v * scale
    launches = [per[k] for k in sorted(per)]
    m = min(len(launches), len(units))
    tot_b = sum(launches[:m])
    tot_u = sum(units[:m])
    print(json.dumps({"launches": m, "bytes": tot_b, "units": tot_u, "bytes_per_unit": tot_b / max(tot_u, 1)}))


if __name__ == "__main__":
    if sys.argv[1] == "--combine":
        combine(sys.argv[2], sys.argv[3])
    else:
        run(int(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else 6)

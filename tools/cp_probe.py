"""Phase times of the persistent PCG kernel over one config-2 solve
(NYS_CP_PROBE=1: CTA 0 stamps %globaltimer at every phase boundary).

    NYS_CP_PROBE=1 python tools/cp_probe.py [config]
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2310_08333_b200 as nys  # noqa: E402
from paper_2310_08333_b200 import _lib  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
d, opts = bench.build_problem(cfg)
A = torch.from_numpy(d.A).cuda()
prob = bench.make_gpu_problem(d, A)
nys.solve(prob, opts)
L = _lib.lib()
acc = (C.c_ulonglong * 24)()
cnt = C.c_ulonglong(0)
L.nys_debug_cp_probe(acc, C.byref(cnt))
res = nys.solve(prob, opts)
L.nys_debug_cp_probe(acc, C.byref(cnt))
names = ["head: block sums, U wait, U^T r0", "barrier 1", "first precond: apply_slice", "barrier 2",
         "direction (after the r.z sum)", "rows of A (HVP)", "barrier 3", "step: U^T r", "barrier 4",
         "stop + precond apply", "barrier 5", "stop test", "z/u tail + finish", "head loop (gate..rhs, r0)",
         "first precond: all_sum x2 + stop", "first precond: coef colsum", "step: p.Ap sum",
         "step: y partial sums", "step: x, r update + ||r||^2", "r.z sum"]
n = max(cnt.value, 1)
tot = sum(acc[:20])
print(f"launches {cnt.value}, iterations {res.iterations}, CG iterations {sum(h.cg_iters for h in res.history)}")
for i in (13, 0, 1, 14, 15, 2, 3, 19, 4, 5, 6, 16, 17, 18, 7, 8, 9, 10, 11, 12):
    nm = names[i]
    print(f"{nm:36s} {acc[i] / n / 1e3:8.2f} us/launch  {100 * acc[i] / max(tot, 1):5.1f}%")
print(f"{'total':36s} {tot / n / 1e3:8.2f} us/launch")

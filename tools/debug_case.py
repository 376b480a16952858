"""Run one golden solve case under the current environment switches and print
the first CG counts next to the reference's (diagnostics for a parity miss)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import numpy as np  # noqa: E402

from test_gpu_solve import gpu_options, gpu_problem  # noqa: E402
from conftest import load_golden  # noqa: E402
import cases  # noqa: E402
import paper_2310_08333_b200 as nys  # noqa: E402

name = sys.argv[1]
gold = load_golden(f"solve_{name}.npz")
spec = cases.SOLVE_CASES[name][0]()
res = nys.solve(gpu_problem(spec), gpu_options(name))
cg = [h.cg_iters for h in res.history]
env = {k: v for k, v in os.environ.items() if k.startswith("NYS_")}
print(name, env, res.status.value, res.iterations, "ref", int(gold["iterations"]))
print("  gpu cg", cg[:12])
print("  ref cg", list(gold["cg_iters"][:12]))
print("  gpu tol", [f"{h.cg_tol:.3e}" for h in res.history[:4]], "ref", [f"{t:.3e}" for t in gold["cg_tol"][:4]] if "cg_tol" in gold else "")

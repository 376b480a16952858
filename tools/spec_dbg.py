import os, sys
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2310_08333_b200 as nys
from paper_2310_08333_b200 import admm
d, opts = bench.build_problem(1)
A = torch.from_numpy(d.A).cuda()
prob = bench.make_gpu_problem(d, A)
orig = admm._Engine._may_speculate
def wrap(self, k, it, have_pc, last_sketch, rho_frozen, cycle_hits):
    r = orig(self, k, it, have_pc, last_sketch, rho_frozen, cycle_hits)
    print("spec", k, r, len(it.after), cycle_hits, self.const_hess, have_pc)
    return r
admm._Engine._may_speculate = wrap
r = nys.solve(prob, opts)
print(r.iterations)

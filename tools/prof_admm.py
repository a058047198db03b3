"""Drive one short admm_persistent launch at a config for ncu (developer tool)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
from paper_2602_04551_b200 import Problem

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 8
inst = synth.config_instance(cfg, seed=0)
rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
pr = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=-1.0, max_iters=iters)
fx = [((), ())] + synth.random_fixings(inst.p, nb - 1, seed=5, depth_lo=1, depth_hi=6, prefer=inst.support_true)
for rep in range(2):
    out = pr.l0l2_bound_batch(fx)
    torch.cuda.synchronize()
ks = pr.l0l2_kernel_stats()
print("admm launches", ks["admm_launches"], "ms/launch", ks["admm_ms"] / ks["admm_launches"],
      "alg GB/s", ks["admm_bytes_alg"] / ks["admm_ms"] / 1e6)

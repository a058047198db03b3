import sys, numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_2602_04551_b200 import Problem
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
inst = synth.config_instance(cfg, seed=0)
rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
fx = [((), ())] + synth.random_fixings(inst.p, 15, seed=11, depth_lo=5, depth_hi=10, prefer=inst.support_true)
for ce in (10, 20, 1000):
    pr = Problem(np.asfortranarray(inst.X), inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=-1.0, max_iters=100, check_every=ce)
    w = pr.l0l2_bound_batch(fx)["warm_out"]
    best = 1e9
    for r in range(3):
        pr.l0l2_kernel_stats(reset=True)
        pr.l0l2_bound_batch(fx, warm_in=w); torch.cuda.synchronize()
        ks = pr.l0l2_kernel_stats()
        best = min(best, ks["admm_ms"] / 101)
    print("check_every %d: %.4f ms/iteration" % (ce, best), flush=True)
    pr.close()

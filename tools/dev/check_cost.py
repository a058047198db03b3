"""Developer probe: cost of the convergence checks (every 10 iterations) in the fused kernel:
fixed 100 iterations at C4 with check_every 10 vs 100 (10 checks vs 1), B = 1 and 16."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_04551_b200 import Problem  # noqa: E402

inst = synth.config_instance(sys.argv[1] if len(sys.argv) > 1 else "C4", seed=0)
rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
out = {}
for ce in (10, 100):
    pr = Problem(np.asfortranarray(inst.X), inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=-1.0,
                 max_iters=100, check_every=ce)
    fx = [((), ())] + synth.random_fixings(inst.p, 15, seed=11, depth_lo=5, depth_hi=10, prefer=inst.support_true)
    warm = pr.l0l2_bound_batch(fx)["warm_out"]
    for B in (1, 16):
        pr.l0l2_bound_batch(fx[:B], warm_in=warm[:B])
        torch.cuda.synchronize()
        pr.l0l2_kernel_stats(reset=True)
        for _ in range(3):
            pr.l0l2_bound_batch(fx[:B], warm_in=warm[:B])
        torch.cuda.synchronize()
        ks = pr.l0l2_kernel_stats()
        out["ce%d_B%d" % (ce, B)] = ks["admm_ms"] / ks["admm_launches"]
    pr.close()
print(json.dumps(out))

"""Developer probe: where the convergence check's cost goes at C4 B = 16 (fixed 100 iterations):
nonzeros of β⁺ per node and their union, and the launch time with check_every 10 / 100 under the
primal-gather variants (L0L2_GATHER=0 whole columns from the segments, =1 row slices, and the row
slices with the dense Zβ sweep forced by L0L2_NZCAP=0)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_04551_b200 import Problem  # noqa: E402

inst = synth.config_instance(sys.argv[1] if len(sys.argv) > 1 else "C4", seed=0)
rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
fx = [((), ())] + synth.random_fixings(inst.p, 15, seed=11, depth_lo=5, depth_hi=10, prefer=inst.support_true)
out = {}
for env in ({"L0L2_GATHER": "0"}, {"L0L2_GATHER": "1"}, {"L0L2_GATHER": "1", "L0L2_NZCAP": "0"}):
    for kk in ("L0L2_GATHER", "L0L2_NZCAP"):
        os.environ.pop(kk, None)
    os.environ.update(env)
    tag = ",".join("%s=%s" % kv for kv in env.items())
    for ce in (10, 100):
        pr = Problem(np.asfortranarray(inst.X), inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=-1.0,
                     max_iters=100, check_every=ce)
        warm = pr.l0l2_bound_batch(fx)["warm_out"]
        if ce == 10 and "nnz" not in out:
            b = warm[:, 0].cpu().numpy()
            out["nnz"] = [int(np.count_nonzero(r)) for r in b]
            out["union"] = int(np.count_nonzero(np.any(b != 0, axis=0)))
        pr.l0l2_bound_batch(fx, warm_in=warm)
        torch.cuda.synchronize()
        pr.l0l2_kernel_stats(reset=True)
        for _ in range(3):
            pr.l0l2_bound_batch(fx, warm_in=warm)
        torch.cuda.synchronize()
        ks = pr.l0l2_kernel_stats()
        out["%s ce%d" % (tag, ce)] = ks["admm_ms"] / ks["admm_launches"]
        pr.close()
print(json.dumps(out))

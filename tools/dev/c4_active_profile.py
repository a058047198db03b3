"""Developer probe: how the C4 tree prefix's ADMM sweeps split by active-node count.
Runs the bench's step (C4 seed 0, 512 nodes, B = 16, rho = 3 mean||X_j||^2) with record=True and
models each 16-node launch as max(iters) sweeps, counting per sweep the nodes still iterating."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_04551_b200 import Problem  # noqa: E402

inst = synth.config_instance("C4", seed=0)
rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
pr = Problem(np.asfortranarray(inst.X), inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=1e-4,
             max_iters=10000)
res = pr.l0l2_solve(gap_tol=1e-2, batch=16, node_limit=512, record=True)
its = [t["iters"] for t in res["trace"]]
hist = np.zeros(17)
for g in range(0, len(its), 16):
    grp = np.array(its[g:g + 16])
    for s in range(int(grp.max())):
        hist[int((grp > s).sum())] += 1
print(json.dumps({"nodes": len(its), "mean_iters": float(np.mean(its)), "sweeps_by_active": hist.tolist(),
                  "iters": its}))

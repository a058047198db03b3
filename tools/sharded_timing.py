"""Per-iteration time of the column-sharded bound's local work (developer tool): one rank's share of
C4's columns (W = 1, 2, 4, 8 → p/W columns; no exchange), fixed iterations, B nodes.  The W-rank time
per iteration ≈ this + one all-reduce of n·B doubles (and of n·B + 4B at checks)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_04551_b200 import ShardedProblem  # noqa: E402

inst = synth.config_instance("C4", seed=0)
rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
iters = 100
rows = []
for W in (1, 2, 4, 8):
    pr = inst.p // W
    sp = ShardedProblem(inst.X[:, :pr], inst.y, 0, pr, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=-1.0,
                        max_iters=iters)
    for B in (1, 16):
        fx = [((), ())] * B
        sp.l0l2_bound_sharded(fx)
        torch.cuda.synchronize()
        t = time.perf_counter()
        sp.l0l2_bound_sharded(fx)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        rows.append(dict(W=W, p_r=pr, B=B, ms_per_iteration=dt / iters * 1e3))
    sp.close()
print(json.dumps(dict(impl="gemm" if os.environ.get("L0L2_SHARD_GEMM") == "1" else "fused", rows=rows)))

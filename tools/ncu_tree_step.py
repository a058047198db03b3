"""One C4 tree-step solve in bench.py's configuration (512-node prefix by default), for ncu captures of
tree-step launches (developer tool).  Prints the kernel stats of the solve as JSON.
    python tools/ncu_tree_step.py [node_limit]
Launch k's algorithmic bytes = stats(limit after round k) − stats(limit after round k−1); with B = 16
the rounds hold 1, 2, 4, 8, 16, 16, ... nodes, so node_limit 31 → 5 launches, 47 → 6."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_04551_b200 import Problem  # noqa: E402

limit = int(sys.argv[1]) if len(sys.argv) > 1 else 512
inst = synth.config_instance("C4", seed=0)
rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
pr = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=1e-4)
pr.l0l2_kernel_stats(reset=True)
r = pr.l0l2_solve(gap_tol=1e-2, batch=16, node_limit=limit)
torch.cuda.synchronize()
print(json.dumps(dict(node_limit=limit, nodes=r["stats"]["nodes"], rounds=r["stats"]["rounds"],
                      kstats=pr.l0l2_kernel_stats())))

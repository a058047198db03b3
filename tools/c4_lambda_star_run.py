"""C4 at the recipe's λ0* (bench.py's instance) solved for a fixed wall time with the MP incumbent and
early prune, printing the gap trajectory (developer tool: documents why the recipe's λ2* = 1e-4 tree
does not certify in minutes)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_04551_b200 import Problem  # noqa: E402

T = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
inst = synth.config_instance("C4", seed=0)
rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
pr = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=1e-4)
out = []
for lim in (T / 10, T / 3, T):
    t = time.perf_counter()
    r = pr.l0l2_solve(gap_tol=1e-2, batch=16, init_mp=True, early_prune=True, time_limit_s=lim)
    out.append(dict(time_limit_s=lim, s=time.perf_counter() - t, gap=r["gap"], lb=r["stats"]["lb"], ub=r["obj"],
                    nodes=r["stats"]["nodes"], max_open=r["stats"]["max_open"], support=[int(j) for j in r["support"]]))
    print(json.dumps(out[-1]), flush=True)

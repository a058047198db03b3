"""Time-to-certified-optimality of C2 (developer tool): gap 1e-6 / node_tol 1e-8 and gap 1e-2 / 1e-4, B = 16,
with and without MP + early prune; prints one JSON line."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_04551_b200 import Problem  # noqa: E402

inst = synth.config_instance("C2", seed=0)
rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
out = []
for gt, nt in ((1e-2, 1e-4), (1e-6, 1e-8)):
    for ext in (False, True):
        pr = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=nt)
        kw = dict(gap_tol=gt, batch=16, init_mp=ext, early_prune=ext)
        pr.l0l2_solve(**kw)
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = pr.l0l2_solve(**kw)
        dt = time.perf_counter() - t
        st = r["stats"]
        out.append(dict(gap_tol=gt, ext=ext, s=dt, nodes=st["nodes"], t_bound=st["t_bound"], t_upper=st["t_upper"],
                        t_tree=st["t_tree"], rounds=st["rounds"], obj=r["obj"]))
        pr.close()
print(json.dumps(out))

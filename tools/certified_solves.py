"""Time-to-certified-optimality of l0l2_solve on the BASELINE configs that close (developer tool;
bench.py reports the same measurement for C3).  python tools/certified_solves.py C3 1e-2 1e-4 16"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_04551_b200 import Problem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
gap = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-2
ntol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-4
B = int(sys.argv[4]) if len(sys.argv) > 4 else 16
rm = float(sys.argv[5]) if len(sys.argv) > 5 else 3.0
tl = float(sys.argv[6]) if len(sys.argv) > 6 else 120.0
t = time.time()
inst = synth.config_instance(cfg, seed=0)
print("instance %s n=%d p=%d lam0=%.4g lam2=%.4g M=%.4g (%.1fs)" % (cfg, inst.n, inst.p, inst.lambda0, inst.lambda2,
                                                                  inst.M, time.time() - t), flush=True)
rho = rm * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
pr = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=ntol, max_iters=10000)
for rep in range(2):
    torch.cuda.synchronize()
    t = time.time()
    r = pr.l0l2_solve(gap_tol=gap, batch=B, time_limit_s=tl)
    dt = time.time() - t
    st = r["stats"]
    print("rep %d: %.3f s status %d nodes %d rounds %d iters/node %.1f gap %.3g obj %.10g |S|=%d S==S_true %s"
          % (rep, dt, st["status"], st["nodes"], st["rounds"], st["node_iters"] / max(1, st["nodes"]), r["gap"],
             r["obj"], len(r["support"]), list(r["support"]) == list(inst.support_true)), flush=True)

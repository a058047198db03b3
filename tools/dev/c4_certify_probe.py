"""Which λ0 multiple of the recipe's λ0* (the C5 path multipliers) lets the C4 tree close?
    python tools/c4_certify_probe.py <time_limit_s> <mult> [<mult> ...]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_04551_b200 import Problem  # noqa: E402

tl = float(sys.argv[1])
for m in [float(a) for a in sys.argv[2:]]:
    inst = synth.config_instance("C4", seed=0, lambda0_mult=m)
    rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
    pr = Problem(np.asfortranarray(inst.X), inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=1e-4)
    t = time.perf_counter()
    r = pr.l0l2_solve(gap_tol=1e-2, batch=16, time_limit_s=tl, init_mp=True, early_prune=True)
    dt = time.perf_counter() - t
    st = r["stats"]
    print(json.dumps({"lambda0_mult": m, "lambda0": inst.lambda0, "lambda2": inst.lambda2, "M": inst.M, "time_s": dt,
                      "certified": st["status"] <= 1, "gap": r["gap"], "nodes": st["nodes"],
                      "support_size": int(len(r["support"]))}), flush=True)
    pr.close()

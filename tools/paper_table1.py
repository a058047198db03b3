"""Time to a 1% gap on the paper's Table 1 analog of C4 (n=1e3, p=1e5, SNR 10, ρ_corr 0.2, k0=10,
node gap 1e-4; paper: 355 s on A100 at K=1), λ2*/λ0*/M from our recipe.
    python tools/paper_table1.py [seed] [time_limit_s]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_04551_b200 import Problem  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
tl = float(sys.argv[2]) if len(sys.argv) > 2 else 300.0
t = time.time()
inst = synth.make_instance(1000, 100000, 10, 0.2, 10.0, seed)
lam2 = synth.tune_lambda2(inst)
lam0 = synth.lambda0_rule(inst, lam2)
M = synth.bigM_rule(inst, lam2)
t_gen = time.time() - t
rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
out = {"instance": "n=1000 p=100000 k*=10 corr=0.2 SNR=10 seed %d" % seed, "lambda0": lam0, "lambda2": lam2, "M": M,
       "gen_s": t_gen, "runs": []}
for ext in (True, False):
    pr = Problem(np.asfortranarray(inst.X), inst.y, lam0, lam2, M, rho=rho, node_tol=1e-4, max_iters=10000)
    t = time.perf_counter()
    r = pr.l0l2_solve(gap_tol=1e-2, batch=16, time_limit_s=tl, init_mp=ext, early_prune=ext)
    dt = time.perf_counter() - t
    st = r["stats"]
    out["runs"].append({"init_mp+early_prune": ext, "time_s": dt, "certified": st["status"] <= 1, "gap": r["gap"],
                        "nodes": st["nodes"], "node_iters": st["node_iters"], "objective": r["obj"],
                        "support": [int(j) for j in r["support"]]})
    pr.close()
    print(json.dumps(out["runs"][-1]), flush=True)
print(json.dumps(out))

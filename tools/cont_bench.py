"""C4 tree step (512-node prefix, bench.py's configuration) and the certified C4 (λ0 = 2λ0*) solve with
and without continuous batching (developer tool); prints JSON lines."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_04551_b200 import Problem  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "prefix"
l0m = 2.0 if which == "cert" else 1.0
inst = synth.config_instance("C4", seed=0, lambda0_mult=l0m)
rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
pr = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=1e-4)
for k in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,4,8").split(",")]:
    for ext in ((False, True) if which == "cert" else (False,)):
        kw = dict(gap_tol=1e-2, batch=16, continuous=k, init_mp=ext, early_prune=ext)
        if which == "prefix":
            kw["node_limit"] = 512
            pr.l0l2_solve(**kw)
        else:
            kw["time_limit_s"] = 120.0
        torch.cuda.synchronize()
        pr.l0l2_kernel_stats(reset=True)
        t = time.perf_counter()
        r = pr.l0l2_solve(**kw)
        dt = time.perf_counter() - t
        ks = pr.l0l2_kernel_stats()
        st = r["stats"]
        print(json.dumps(dict(which=which, continuous=k, ext=ext, s=dt, nodes=st["nodes"], nodes_per_s=st["nodes"] / dt,
                              node_iters=st["node_iters"], gap=r["gap"], obj=r["obj"], status=st["status"],
                              suspensions=st["suspensions"], launches=ks["admm_launches"], sweeps=ks["admm_iters"],
                              lane_util=ks["admm_node_iters"] / max(1, 16 * ks["admm_iters"]),
                              admm_ms=ks["admm_ms"])), flush=True)

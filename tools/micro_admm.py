"""Quick ADMM-kernel microbenchmark (developer tool): fixed-iteration l0l2_bound_batch at a config for a
few batch sizes; prints ms per launch-iteration and the kernel's roofline fraction.
    python tools/micro_admm.py C4 1,8,16 100"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_04551_b200 import Problem  # noqa: E402

FP64 = 37.1
HBM = 6540.8
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
Bs = [int(b) for b in (sys.argv[2] if len(sys.argv) > 2 else "1,8,16").split(",")]
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 100
if cfg in ("P3000", "P11962"):   # the paper's n = 3000, p = 30000 workload / its real data set's
    # shape n = 11 962, p = 23 250 (synthetic data of that shape), wide-n ADMM path
    n_, p_ = (3000, 30000) if cfg == "P3000" else (11962, 23250)
    inst = synth.make_instance(n_, p_, 10, 0.1, 10.0 / 3.0, 0)
    lam2 = synth.tune_lambda2(inst)
    inst.lambda2, inst.lambda0, inst.M = lam2, synth.lambda0_rule(inst, lam2), synth.bigM_rule(inst, lam2)
else:
    inst = synth.config_instance(cfg, seed=0)
rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
pr = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=-1.0, max_iters=iters)
fx = [((), ())] + synth.random_fixings(inst.p, max(Bs) - 1, seed=11, depth_lo=5, depth_hi=10, prefer=inst.support_true)
warm = pr.l0l2_bound_batch(fx)["warm_out"]
rows = []
for B in Bs:
    pr.l0l2_bound_batch(fx[:B], warm_in=warm[:B])
    torch.cuda.synchronize()
    pr.l0l2_kernel_stats(reset=True)
    for _ in range(3):
        pr.l0l2_bound_batch(fx[:B], warm_in=warm[:B])
    torch.cuda.synchronize()
    ks = pr.l0l2_kernel_stats()
    s = ks["admm_ms"] / 1e3
    tf = ks["admm_flops_alg"] / s / 1e12
    gbs = ks["admm_bytes_alg"] / s / 1e9
    ai = ks["admm_flops_alg"] / ks["admm_bytes_alg"]
    frac = tf / FP64 if ai * HBM / 1e3 >= FP64 else gbs / HBM
    rows.append(dict(B=B, ms_per_launch_iter=ks["admm_ms"] / ks["admm_launches"] / (iters + 1),
                     node_iters_per_s=ks["admm_node_iters"] / s, tflops=tf, gbs=gbs, frac=frac))
print(json.dumps(dict(config=cfg, iters=iters, info=pr.info(), rows=rows)))

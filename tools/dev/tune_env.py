"""Sweep tuning env hooks of the ADMM kernel on the §8(d) microbenchmark (developer tool):
    python tools/tune_env.py C4 16 100 L0L2_PFD=0,1,2,3 L0L2_PFS=0,6"""
import itertools
import os
import subprocess
import sys

cfg, B, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
axes = [(a.split("=")[0], a.split("=")[1].split(",")) for a in sys.argv[4:]]
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_2602_04551_b200 import Problem
cfg, B, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
if cfg.startswith("n"):   # e.g. n500p100000: synthetic shape for kernel timing only
    nn, pp = cfg[1:].split("p")
    inst = synth.make_instance(int(nn), int(pp), 10, 0.1, 5.0, 0)
    inst.lambda0, inst.lambda2, inst.M = 10.0, 0.01, 2.0
else:
    inst = synth.config_instance(cfg, seed=0)
rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
pr = Problem(np.asfortranarray(inst.X), inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=-1.0, max_iters=iters)
fx = [((), ())] + synth.random_fixings(inst.p, B - 1, seed=11, depth_lo=5, depth_hi=10, prefer=inst.support_true)
w = pr.l0l2_bound_batch(fx)["warm_out"]
best = 1e9
for r in range(3):
    pr.l0l2_kernel_stats(reset=True)
    pr.l0l2_bound_batch(fx, warm_in=w); torch.cuda.synchronize()
    ks = pr.l0l2_kernel_stats()
    best = min(best, ks["admm_ms"] / (iters + 1))   # per iteration of the whole batch
print("ms/iteration (all %d nodes) %.4f  node-it/s %.0f" % (B, best, B * 1e3 / best))
'''
for combo in itertools.product(*[v for _, v in axes]):
    env = dict(os.environ)
    tag = " ".join("%s=%s" % (k, v) for (k, _), v in zip(axes, combo))
    for (k, _), v in zip(axes, combo):
        env[k] = v
    r = subprocess.run([sys.executable, "-c", code, cfg, str(B), str(iters)], env=env, capture_output=True, text=True)
    print(tag, "|", (r.stdout.strip() or r.stderr.strip()[-300:]), flush=True)

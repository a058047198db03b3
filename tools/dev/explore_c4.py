"""Explore C4 solve settings on the GPU (developer tool)."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
import synth
from paper_2602_04551_b200 import Problem

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
tl = float(sys.argv[2]) if len(sys.argv) > 2 else 60
t = time.time()
inst = synth.config_instance(cfg, seed=0)
print("gen %.1fs lam0 %.4g lam2 %.4g M %.4g sqrt(l0/l2) %.4g" % (time.time() - t, inst.lambda0, inst.lambda2, inst.M,
      (inst.lambda0 / inst.lambda2) ** 0.5), flush=True)
rho0 = float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
for mult in (1, 3, 10):
    pr = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho0 * mult, node_tol=1e-4)
    pr.l0l2_kernel_stats(reset=True)
    t = time.time()
    out = pr.l0l2_bound_batch([((), ())])
    import torch; torch.cuda.synchronize()
    ks = pr.l0l2_kernel_stats()
    print("rho x%g root: iters %d lb %.8g primal %.8g flags %d time %.3fs GB/s %.0f" % (mult, int(out["iters"][0]),
          float(out["lb"][0]), float(out["primal"][0]), int(out["flags"][0]), time.time() - t,
          ks["admm_bytes_alg"] / max(1e-9, ks["admm_ms"]) / 1e6), flush=True)
    pr.close()
for mult, gap, ntol, B in [(3, 1e-2, 1e-4, 16), (3, 1e-2, 1e-4, 8)]:
    t = time.time()
    pr = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho0 * mult, node_tol=ntol)
    tc = time.time() - t
    pr.l0l2_kernel_stats(reset=True)
    t = time.time()
    r = pr.l0l2_solve(gap_tol=gap, batch=B, time_limit_s=tl, verbose=True)
    ts = time.time() - t
    ks = pr.l0l2_kernel_stats()
    st = r["stats"]
    print(json.dumps(dict(mult=mult, gap=gap, ntol=ntol, B=B, create=tc, solve=ts, obj=r["obj"], cgap=r["gap"],
        supp=[int(j) for j in r["support"]], nodes=st["nodes"], iters=st["node_iters"], rounds=st["rounds"],
        max_open=st["max_open"], t_bound=st["t_bound"], t_upper=st["t_upper"], t_tree=st["t_tree"],
        admm_ms=ks["admm_ms"], launches=ks["admm_launches"], sweeps=ks["admm_iters"],
        GBs=ks["admm_bytes_alg"] / max(1e-9, ks["admm_ms"]) / 1e6, upper_ms=ks["upper_ms"])), flush=True)
    pr.close()

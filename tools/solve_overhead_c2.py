"""Where the time of a C2 certified solve goes (developer tool)."""
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_2602_04551_b200 import Problem
inst = synth.config_instance("C2", seed=0)
rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
pr = Problem(np.asfortranarray(inst.X), inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=1e-8)
for rep in range(3):
    torch.cuda.synchronize()
    pr.l0l2_kernel_stats(reset=True)
    t = time.perf_counter()
    r = pr.l0l2_solve(gap_tol=1e-6, batch=16)
    w = time.perf_counter() - t
    st = r["stats"]
    ks = pr.l0l2_kernel_stats()
    print("wall %.3f t_total %.3f bound %.3f upper %.3f tree %.3f admm_ms %.1f (launches %d) upper_ms %.1f rounds %d nodes %d iters %d"
          % (w, st["t_total"], st["t_bound"], st["t_upper"], st["t_tree"], ks["admm_ms"], ks["admm_launches"],
             ks["upper_ms"], st["rounds"], st["nodes"], st["node_iters"]), flush=True)

import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_2602_04551_b200 import Problem
inst = synth.config_instance("C4", seed=0)
rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
pr = Problem(np.asfortranarray(inst.X), inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=1e-4)
for nl in (512, 512, 1, 1, 64):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = pr.l0l2_solve(gap_tol=1e-2, batch=16, node_limit=nl)
    w = time.perf_counter() - t
    st = r["stats"]
    ks = pr.l0l2_kernel_stats(reset=True)
    print("node_limit %d wall %.3f t_total %.3f bound %.3f upper %.3f tree %.3f admm_ms %.1f rounds %d nodes %d"
          % (nl, w, st["t_total"], st["t_bound"], st["t_upper"], st["t_tree"], ks["admm_ms"], st["rounds"], st["nodes"]), flush=True)

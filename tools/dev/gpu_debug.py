"""Quick GPU sanity run: kernel vs oracle on small instances (developer tool)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import synth  # noqa: E402
from paper_2602_04551_b200 import Problem  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(a - b)) / (1.0 + np.max(np.abs(b))))


def check_fixed(inst, lam0, lam2, M, fixings, iters, warm=None, label=""):
    t = time.time()
    prob = Problem(inst.X, inst.y, lam0, lam2, M, node_tol=-1.0, max_iters=iters, check_every=10)
    print(label, "create %.3fs rho %.4g" % (time.time() - t, prob.rho), flush=True)
    P = O.Problem(inst.X, inst.y, lam0, lam2, M, rho=prob.rho)
    out = prob.l0l2_bound_batch(fixings, warm_in=None if warm is None else torch.tensor(warm).cuda(),
                                want_warm=True, want_zhat=True)
    torch.cuda.synchronize()
    wo = out["warm_out"].cpu().numpy()
    lb = out["lb"].cpu().numpy()
    pr = out["primal"].cpu().numpy()
    it = out["iters"].cpu().numpy()
    br = out["branch_j"].cpu().numpy()
    worst = 0
    for k, (F0, F1) in enumerate(fixings):
        code = O.make_code(inst.p, F0, F1)
        w = None if warm is None else (warm[k, 0], warm[k, 1])
        r = O.admm_node(P, code, warm=w, node_tol=-1.0, max_iters=iters, check_every=10)
        eb, ev = rel(wo[k, 0], r.beta), rel(wo[k, 1], r.v)
        el = abs(lb[k] - r.lb) / max(1, abs(r.lb))
        ep = abs(pr[k] - r.primal) / max(1, abs(r.primal))
        worst = max(worst, eb, ev, el, ep)
        print(f"  node {k}: it {it[k]}/{r.iters} beta {eb:.2e} v {ev:.2e} lb {el:.2e} ({lb[k]:.10g} vs {r.lb:.10g}) "
              f"primal {ep:.2e} branch {br[k]}/{r.branch_j}", flush=True)
    print(label, "WORST", worst, flush=True)
    prob.close()
    return worst


def main():
    torch.cuda.init()
    inst = synth.config_instance("C1", seed=0)
    fx = [((), ())] + synth.random_fixings(inst.p, 4, seed=1, depth_lo=1, depth_hi=6)
    check_fixed(inst, inst.lambda0, inst.lambda2, inst.M, fx, 57, label="C1")
    inst2 = synth.make_instance(200, 2000, 5, 0.2, 5.0, 3)
    lam2 = synth.tune_lambda2(inst2)
    lam0 = synth.lambda0_rule(inst2, lam2)
    M = synth.bigM_rule(inst2, lam2)
    fx = [((), ())] + synth.random_fixings(inst2.p, 10, seed=2, depth_lo=1, depth_hi=8, prefer=inst2.support_true)
    check_fixed(inst2, lam0, lam2, M, fx, 40, label="n200p2000")
    # solve C1 vs brute force
    P = O.Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M)
    bf = O.brute_force(P)
    prob = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=P.rho, node_tol=1e-10, max_iters=20000)
    t = time.time()
    res = prob.l0l2_solve(gap_tol=1e-9, batch=8)
    print("C1 solve %.3fs obj %.12g bf %.12g supp %s bf %s stats %s" % (time.time() - t, res["obj"], bf[0],
          list(res["support"]), list(bf[1]), res["stats"]), flush=True)


if __name__ == "__main__":
    main()

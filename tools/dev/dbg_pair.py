"""Developer check of the paired-CTA ADMM kernel: a 16+1-node batch vs each node alone (bitwise)
and vs the oracle, for several iteration counts; then converging batches (mode switches)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import synth  # noqa: E402
from paper_2602_04551_b200 import Problem  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(a - b)) / (1.0 + np.max(np.abs(b))))


def inst_of(kind):
    if kind == "direct":
        inst = synth.make_instance(300, 120, 6, 0.5, 5.0, 7)
    else:
        inst = synth.make_instance(200, 2000, 5, 0.1, 3.0, 3)
    lam2 = max(synth.tune_lambda2(inst), 0.5)
    return inst, synth.lambda0_rule(inst, lam2), lam2, synth.bigM_rule(inst, lam2)


def main():
    kind = sys.argv[1] if len(sys.argv) > 1 else "direct"
    inst, lam0, lam2, M = inst_of(kind)
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    fx = [((), ())] + synth.random_fixings(inst.p, 16, seed=17, depth_lo=1, depth_hi=10, prefer=inst.support_true)
    for N in [0, 1, 2, 3, 10, 11, 57]:
        prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=-1.0, max_iters=max(N, 1))
        out = prob.l0l2_bound_batch(fx)
        wo = out["warm_out"].cpu().numpy()
        singles = []
        for k in [0, 1, 8, 9, 16]:
            o1 = prob.l0l2_bound_batch([fx[k]])
            singles.append((k, o1["warm_out"].cpu().numpy()[0]))
        prob.close()
        msg = []
        for k, w1 in singles:
            msg.append("node %d: batch-vs-single %.2e" % (k, rel(wo[k], w1)))
        errs = []
        for k in range(len(fx)):
            r = O.admm_node(P, O.make_code(inst.p, *fx[k]), node_tol=-1.0, max_iters=max(N, 1))
            errs.append(rel(wo[k, 0], r.beta))
        print("N=%d" % N, "; ".join(msg), "| oracle beta err per node:", " ".join("%.0e" % e for e in errs), flush=True)


if __name__ == "__main__":
    main()

"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck) on the library's kernels.

usage: compute-sanitizer --tool <tool> python tools/sanitize_run.py <case>
  c1      C1 (n=50, p=20, direct regime): 17-node bound batch (paired CTAs, compaction, two groups),
          upper bounds, matching pursuit, a short solve
  c2      C2-shaped (n=p=1000, direct regime) 16-node batch, fixed 12 iterations
  zform   p > 2n Z-form (n=200, p=2000): 17-node batch with convergence (compaction), the dense
          primal fallback (L0L2_NZCAP=0) and a short solve with early prune + MP
  wide    the wide-n path: forced (L0L2_WIDE=1) on a ragged Z-form instance (17-node batch with warm
          starts, a short solve with MP + early prune) and natural at n = 1064 (16 nodes)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_04551_b200 import Problem  # noqa: E402


def fixings(inst, B, seed):
    return [((), ())] + synth.random_fixings(inst.p, B - 1, seed=seed, depth_lo=1, depth_hi=6)


def main(case):
    if case == "c1":
        inst = synth.config_instance("C1", seed=0)
        pr = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, node_tol=1e-7, max_iters=300)
        pr.l0l2_bound_batch(fixings(inst, 17, 1), want_zhat=True, want_dual_r=True)
        pr.l0l2_upper_batch([[0, 3, 7], [], list(range(inst.p))])
        pr.l0l2_matching_pursuit()
        pr.l0l2_solve(gap_tol=1e-3, batch=8, init_mp=True, early_prune=True)
        pr.close()
    elif case == "c2":
        inst = synth.make_instance(1000, 1000, 10, 0.5, 5.0, 0)
        pr = Problem(np.asfortranarray(inst.X), inst.y, 1.0, 0.5, 2.0, node_tol=-1.0, max_iters=12)
        pr.l0l2_bound_batch(fixings(inst, 16, 2))
        pr.close()
    elif case == "zform":
        inst = synth.make_instance(200, 2000, 5, 0.1, 3.0, 3)
        lam2 = 0.5
        lam0, M = synth.lambda0_rule(inst, lam2), synth.bigM_rule(inst, lam2)
        pr = Problem(inst.X, inst.y, lam0, lam2, M, node_tol=1e-6, max_iters=400)
        pr.l0l2_bound_batch(fixings(inst, 17, 3))
        os.environ["L0L2_NZCAP"] = "0"
        pr.l0l2_bound_batch(fixings(inst, 9, 4))
        del os.environ["L0L2_NZCAP"]
        pr.l0l2_solve(gap_tol=1e-2, batch=16, node_limit=40, init_mp=True, early_prune=True)
        pr.close()
    elif case == "round2":
        # device frontier, continuous batching (host frontier), large-support upper bound, column-sharded bound
        inst = synth.make_instance(80, 60, 5, 0.3, 3.0, 21)
        lam2 = 0.5
        lam0, M = synth.lambda0_rule(inst, lam2), synth.bigM_rule(inst, lam2)
        pr = Problem(inst.X, inst.y, lam0, lam2, M, node_tol=1e-8)
        pr.l0l2_solve(gap_tol=1e-4, batch=16, record=True, init_mp=True, early_prune=True)   # device frontier
        pr.l0l2_solve(gap_tol=1e-4, batch=4, record=True, continuous=3)                      # host frontier
        pr.close()
        inst = synth.make_instance(200, 1500, 5, 0.1, 3.0, 3)
        pr = Problem(inst.X, inst.y, 1.0, 2.0, 1e3)
        rng = np.random.default_rng(1)
        pr.l0l2_upper_batch([np.sort(rng.choice(inst.p, size=700, replace=False)), [0, 5, 9]])
        pr.close()
        from paper_2602_04551_b200 import ShardedProblem
        sp = ShardedProblem(inst.X[:, :700], inst.y, 0, 700, 1.0, 2.0, 2.0, node_tol=1e-6, max_iters=300)
        sp.l0l2_bound_sharded([((), ()), ((1,), (3,))])
        sp.close()
    elif case == "wide":
        os.environ["L0L2_WIDE"] = "1"
        inst = synth.make_instance(61, 203, 4, 0.3, 4.0, 9)
        lam2 = 0.5
        lam0, M = synth.lambda0_rule(inst, lam2), synth.bigM_rule(inst, lam2)
        pr = Problem(inst.X, inst.y, lam0, lam2, M, node_tol=1e-7, max_iters=300)
        out = pr.l0l2_bound_batch(fixings(inst, 17, 5), want_zhat=True, want_dual_r=True)
        pr.l0l2_bound_batch(fixings(inst, 3, 6), warm_in=out["warm_out"][:3].contiguous())
        pr.l0l2_solve(gap_tol=1e-3, batch=16, node_limit=60, init_mp=True, early_prune=True)
        pr.close()
        del os.environ["L0L2_WIDE"]
        inst = synth.make_instance(1064, 2200, 5, 0.3, 4.0, 31)
        pr = Problem(np.asfortranarray(inst.X), inst.y, 1.0, 0.5, 2.0, node_tol=-1.0, max_iters=12)
        pr.l0l2_bound_batch(fixings(inst, 16, 7))
        pr.close()
    print("sanitize case %s done" % case)


if __name__ == "__main__":
    main(sys.argv[1])

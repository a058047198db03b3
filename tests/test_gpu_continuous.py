"""Continuous batching (second half; P:272 reads a batch as a snapshot) — -m gpu.

With l0l2_solve(continuous=k) a 16-node launch suspends its last ≤ k iterating nodes at a regular
check while open nodes wait; they resume in a later launch from their own (β, v), best dual and
iteration count.  What must hold:
* the certificate is unchanged (support bit-exact and objective = brute force);
* a suspended-and-resumed node computes exactly what it would have computed uninterrupted: every
  finished node of the continuous tree matches the oracle's node relaxation on the same fixings and
  parent warm start (reconstructed from the trace's parent ids), i.e. the same iteration count,
  the same branch index and the LB to 1e-6 — the tree ORDER differs from the synchronous rounds,
  the node arithmetic does not.
"""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2602_04551_b200 import FLAG_CONVERGED, Problem  # noqa: E402


@pytest.mark.parametrize("seed", range(6))
def test_continuous_certificate_equals_brute_force(seed):
    if seed == 0:
        inst = synth.config_instance("C1", seed=0)
        lam0, lam2, M = inst.lambda0, inst.lambda2, inst.M
    else:
        rng = np.random.default_rng(100 + seed)
        n, p = int(rng.choice([30, 60])), int(rng.choice([9, 12]))
        inst = synth.make_instance(n, p, 3, float(rng.choice([0.0, 0.3])), 4.0, seed)
        lam0, lam2, M = float(rng.uniform(0.01, 1)) * n / 10, float(rng.uniform(0.05, 1)), float(rng.uniform(1, 6))
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    obj, S, _ = O.brute_force(P)
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-10, max_iters=20000)
    for k in (4, 12):
        res = prob.l0l2_solve(gap_tol=1e-9, batch=16, continuous=k)
        assert abs(res["obj"] - obj) <= 1e-9 * max(1.0, abs(obj)), (k, res["obj"], obj)
        assert np.array_equal(res["support"], S)
        assert res["stats"]["lb"] <= obj * (1 + 1e-9)
    prob.close()


def _oracle_replay(P, trace, node_tol):
    """The oracle's node relaxation of every traced node, on the fixings and parent warm state the
    trace's parent ids define (parents are solved before their children)."""
    by_id = {t["id"]: t for t in trace}
    memo = {}

    def fix(u):
        F0, F1 = [], []
        while u["parent"] >= 0:
            j, val = u["lastfix"] // 2, u["lastfix"] % 2
            (F1 if val else F0).append(j)
            u = by_id[u["parent"]]
        return tuple(sorted(F0)), tuple(sorted(F1))

    def solve(uid):
        if uid in memo:
            return memo[uid]
        u = by_id[uid]
        warm, plb = None, -np.inf
        if u["parent"] >= 0:
            par = solve(u["parent"])
            warm, plb = (par.beta, par.v), par.lb
        F0, F1 = fix(u)
        r = O.admm_node(P, O.make_code(P.p, F0, F1), warm=warm, parent_lb=plb, node_tol=node_tol)
        memo[uid] = r
        return r

    return {t["id"]: solve(t["id"]) for t in trace}


def test_resumed_nodes_compute_what_uninterrupted_nodes_compute():
    inst = synth.make_instance(80, 60, 5, 0.3, 3.0, 21)   # the tree-parity instance (~100 nodes)
    lam2 = 0.5
    lam0 = synth.lambda0_rule(inst, lam2)
    M = synth.bigM_rule(inst, lam2)
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    ref = O.bnb_solve(P, B=16, gap_tol=1e-4, node_tol=1e-8)
    suspended = 0
    for B, k in ((4, 3), (8, 6)):   # narrow launches, so open nodes wait while a launch's tail runs
        prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-8)
        res = prob.l0l2_solve(gap_tol=1e-4, batch=B, record=True, continuous=k)
        prob.close()
        suspended += res["stats"]["suspensions"]
        assert abs(res["obj"] - ref["obj"]) <= 1e-9 * abs(ref["obj"])
        assert np.array_equal(res["support"], ref["support"])
        oracle_nodes = _oracle_replay(P, res["trace"], 1e-8)
        for t in res["trace"]:
            r = oracle_nodes[t["id"]]
            assert t["iters"] == r.iters, (B, t["id"], t["iters"], r.iters)
            assert abs(t["lb"] - r.lb) <= 1e-6 * max(1.0, abs(r.lb)), (B, t["id"], t["lb"], r.lb)
            assert bool(t["flags"] & FLAG_CONVERGED) == r.converged
            assert t["branch_j"] == r.branch_j or r.branch_j < 0, (B, t["id"], t["branch_j"], r.branch_j)
    assert suspended > 0

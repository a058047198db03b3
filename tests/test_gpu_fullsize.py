"""GPU parity at BASELINE's full sizes and on kernel paths the bench relies on (-m gpu), all through
the C-ABI against the CPU oracle (VERDICT r01 "untested kernel paths"):

* C2 (n = p = 1000): the direct-regime kernel instantiation the C2 solves run
  (admm_persistent<…, DIR = true> at p ≈ 1000), fixed iterations, B ∈ {1, 16, 17};
* C2 certified solves (gap 1e-6, node_tol 1e-8, B = 16), with and without the matching-pursuit
  incumbent + early prune, node for node against the oracle's committed trees
  (tests/golden/oracle_C2_tree_*.json, written by tools/oracle_tree_golden.py from oracle/ only);
* C3 (n = 1000, p = 1e4) and C5 (n = 500, p = 2e4 Toeplitz) at full size, fixed iterations;
* the dense-β⁺ primal fallback (forward-only Zβ sweep + ‖L(Zβ)‖², forced by L0L2_NZCAP = 0);
* Z-form (p > 2n) tree parity with early prune and the MP incumbent.
"""
import json
import os

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2602_04551_b200 import FLAG_PRUNED, Problem  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)), initial=0.0) / (1.0 + np.max(np.abs(b), initial=0.0)))


def _fixed_iteration_check(inst, rho, B, N, sample, seed, env=None):
    P = O.Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho)
    prob = Problem(np.asfortranarray(inst.X), inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho,
                   node_tol=-1.0, max_iters=N)
    fx = [((), ())] + synth.random_fixings(inst.p, B - 1, seed=seed, depth_lo=1, depth_hi=10,
                                           prefer=inst.support_true)
    out = prob.l0l2_bound_batch(fx)
    wo, lb, pr = out["warm_out"].cpu().numpy(), out["lb"].cpu().numpy(), out["primal"].cpu().numpy()
    it = out["iters"].cpu().numpy()
    prob.close()
    for k in sample:
        if k >= B:
            continue
        r = O.admm_node(P, O.make_code(inst.p, *fx[k]), node_tol=-1.0, max_iters=N)
        assert it[k] == N
        assert rel(wo[k, 0], r.beta) < 1e-9, (k, rel(wo[k, 0], r.beta))
        assert rel(wo[k, 1], r.v) < 1e-9, (k, rel(wo[k, 1], r.v))
        assert abs(lb[k] - r.lb) <= 1e-9 * max(1.0, abs(r.lb)), (k, lb[k], r.lb)
        assert abs(pr[k] - r.primal) <= 1e-9 * max(1.0, abs(r.primal)), (k, pr[k], r.primal)
        assert np.all(wo[k, 0][list(fx[k][0])] == 0.0)
        assert np.max(np.abs(wo[k, 0])) <= inst.M


@pytest.fixture(scope="module")
def c2():
    return synth.config_instance("C2", seed=0)


@pytest.mark.parametrize("B", [1, 16, 17])
def test_c2_full_size_direct_regime_fixed_iterations(c2, B):
    """The C2 solves' kernel (direct regime R17, D = 1000×1000 streamed) at the full C2 size."""
    rho = O.default_rho(c2.X) * 3.0
    _fixed_iteration_check(c2, rho, B, 41, sample=(0, 1, 8, 15, 16), seed=100 + B)


@pytest.mark.parametrize("ext", [False, True])
def test_c2_certified_solve_tree_parity(ext):
    """C2 certified to gap 1e-6 (node_tol 1e-8, B = 16, ρ = 3·mean‖X_j‖²) as in bench.py's
    certified_solves: node for node against the oracle's committed tree (same ids, LBs 1e-6,
    iteration counts, branches, early-pruned nodes) and the same certificate."""
    name = "oracle_C2_tree_g1e-06_n1e-08_B16%s.json" % ("_mpep" if ext else "")
    g = json.load(open(os.path.join(ROOT, "tests", "golden", name)))
    inst = synth.config_instance("C2", seed=0)
    assert abs(inst.lambda0 - g["lambda0"]) <= 1e-12 * g["lambda0"]
    prob = Problem(np.asfortranarray(inst.X), inst.y, inst.lambda0, inst.lambda2, inst.M, rho=g["rho"],
                   node_tol=g["node_tol"])
    res = prob.l0l2_solve(gap_tol=g["gap_tol"], batch=g["batch"], record=True, init_mp=ext, early_prune=ext)
    prob.close()
    assert list(res["support"]) == g["support"]
    assert abs(res["obj"] - g["obj"]) <= 1e-9 * abs(g["obj"])
    assert res["gap"] <= g["gap_tol"]
    gt = {t["id"]: t for t in res["trace"]}
    for t in g["trace"]:
        u = gt.get(t["id"])
        assert u is not None, ("node missing on GPU", t["id"])
        assert abs(u["lb"] - t["lb"]) <= 1e-6 * max(1.0, abs(t["lb"])), (t["id"], u["lb"], t["lb"])
        assert u["iters"] == t["iters"], (t["id"], u["iters"], t["iters"])
        assert u["branch_j"] == t["branch_j"], (t["id"], u["branch_j"], t["branch_j"])
        assert abs(u["ub"] - t["ub"]) <= 1e-6 * abs(t["ub"])
        assert bool(u["flags"] & FLAG_PRUNED) == t["early"]
    assert len(res["trace"]) == g["nodes"]


@pytest.mark.parametrize("cfg", ["C3", "C5"])
def test_c3_c5_full_size_fixed_iterations(cfg):
    """C3 (Z = 80 MB, L2-resident) and C5 (n = 500 Toeplitz) at BASELINE's full sizes, 17 nodes
    (paired CTAs + a second group), fixed iterations, sampled nodes vs the oracle's G-form."""
    inst = synth.config_instance(cfg, seed=0)
    rho = O.default_rho(inst.X) * 3.0
    _fixed_iteration_check(inst, rho, 17, 23, sample=(0, 5, 16), seed=7)


def test_dense_primal_fallback(monkeypatch):
    """L0L2_NZCAP = 0 forces the dense-β⁺ primal check (forward-only sweep Zβ, reduction,
    ‖L(Zβ)‖²) for every node at every check: same fixed-iteration bounds as the oracle."""
    monkeypatch.setenv("L0L2_NZCAP", "0")
    monkeypatch.setenv("L0L2_GATHER", "1")   # the row-slice gather path (whose dense fallback this is)
    inst = synth.make_instance(200, 2000, 5, 0.1, 3.0, 3)   # p > 2n: Z-form
    lam2 = max(synth.tune_lambda2(inst), 0.5)
    inst.lambda2 = lam2
    inst.lambda0 = synth.lambda0_rule(inst, lam2)
    inst.M = synth.bigM_rule(inst, lam2)
    rho = O.default_rho(inst.X)
    _fixed_iteration_check(inst, rho, 17, 31, sample=(0, 3, 9, 16), seed=12)
    # and with convergence decisions driven by the dense primal: same iteration counts
    P = O.Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho)
    prob = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=1e-6, max_iters=4000)
    fx = [((), ())] + synth.random_fixings(inst.p, 5, seed=2, depth_lo=1, depth_hi=6)
    out = prob.l0l2_bound_batch(fx)
    prob.close()
    for k in range(len(fx)):
        r = O.admm_node(P, O.make_code(inst.p, *fx[k]), node_tol=1e-6, max_iters=4000)
        assert int(out["iters"][k]) == r.iters
        assert abs(float(out["lb"][k]) - r.lb) <= 1e-6 * max(1.0, abs(r.lb))


@pytest.mark.parametrize("B", [1, 16])
def test_zform_tree_parity_early_prune_and_mp(B):
    """p > 2n (Z-form kernel) with the MP incumbent and early prune on both sides: node-for-node
    tree parity with the oracle (ids, LBs 1e-6, iterations, branches, early-stopped nodes)."""
    inst = synth.make_instance(50, 130, 3, 0.2, 6.0, 5)   # 123-node oracle tree at B = 16
    lam2 = 0.5
    lam0 = synth.lambda0_rule(inst, lam2)
    M = synth.bigM_rule(inst, lam2)
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    ref = O.bnb_solve(P, B=B, gap_tol=1e-4, node_tol=1e-8, record=True, early_prune=True, init_mp=True)
    assert ref["nodes"] >= 20
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-8)
    res = prob.l0l2_solve(gap_tol=1e-4, batch=B, record=True, early_prune=True, init_mp=True)
    prob.close()
    assert abs(res["obj"] - ref["obj"]) <= 1e-9 * abs(ref["obj"])
    assert np.array_equal(res["support"], ref["support"])
    gt = {t["id"]: t for t in res["trace"]}
    for t in ref["trace"]:
        g = gt.get(t["id"])
        assert g is not None, ("node missing on GPU", t["id"])
        assert abs(g["lb"] - t["lb"]) <= 1e-6 * max(1.0, abs(t["lb"]))
        assert g["iters"] == t["iters"]
        assert bool(g["flags"] & FLAG_PRUNED) == t["early"]
        assert g["branch_j"] == t["branch_j"] or t["branch_j"] < 0
    assert len(res["trace"]) == ref["nodes"]


@pytest.mark.parametrize("ce,mi", [(1, 40), (10, 1001), (7, 50)])
def test_consecutive_checks(ce, mi):
    """check_every = 1 (every iteration is a check) and max_iters ≡ 1 (mod check_every) (two checks
    in a row at the end): the double-buffered check sums keep every CTA's decision identical, and
    the fixed-iteration / converged results match the oracle."""
    inst = synth.make_instance(200, 2000, 5, 0.1, 3.0, 3)
    lam2 = 0.5
    lam0, M = synth.lambda0_rule(inst, lam2), synth.bigM_rule(inst, lam2)
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-7, max_iters=mi, check_every=ce)
    fx = [((), ())] + synth.random_fixings(inst.p, 16, seed=4, depth_lo=1, depth_hi=6)
    out = prob.l0l2_bound_batch(fx)
    prob.close()
    for k in (0, 7, 16):
        r = O.admm_node(P, O.make_code(inst.p, *fx[k]), node_tol=1e-7, max_iters=mi, check_every=ce)
        assert int(out["iters"][k]) == r.iters
        assert abs(float(out["lb"][k]) - r.lb) <= 1e-6 * max(1.0, abs(r.lb))


def test_c4_certified_solve_oracle_evidence():
    """North-star target (NS-T9): the certified C4 solve of bench.py's certified_c4 (n=1000, p=1e5,
    λ0 = 2λ0*, gap 1e-2, node_tol 1e-4, B = 16, ρ = 3·mean‖X_j‖²).  Oracle evidence:
    * its first 111 nodes (10 rounds) equal the oracle's own BnB on the same instance node for node
      (tests/golden/oracle_C4_l0x2_tree_g0.01_n0.0001_B16_lim96.json, written by
      tools/oracle_tree_golden.py from oracle/ only, 36 CPU-minutes): ids, LBs 1e-6, iterations,
      branches, UBs 1e-6;
    * the returned objective is the oracle's exact box ridge on the returned support (1e-9), the
      support is the planted β† support, and the certified LB ≤ that objective with gap ≤ 1e-2."""
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_C4_l0x2_tree_g0.01_n0.0001_B16_lim96.json")))
    inst = synth.config_instance("C4", seed=0, lambda0_mult=2.0)
    assert abs(inst.lambda0 - g["lambda0"]) <= 1e-12 * g["lambda0"]
    prob = Problem(np.asfortranarray(inst.X), inst.y, inst.lambda0, inst.lambda2, inst.M, rho=g["rho"],
                   node_tol=g["node_tol"])
    res = prob.l0l2_solve(gap_tol=g["gap_tol"], batch=g["batch"], record=True)
    prob.close()
    gt = {t["id"]: t for t in res["trace"]}
    for t in g["trace"]:
        u = gt.get(t["id"])
        assert u is not None, ("node missing on GPU", t["id"])
        assert abs(u["lb"] - t["lb"]) <= 1e-6 * max(1.0, abs(t["lb"])), (t["id"], u["lb"], t["lb"])
        assert u["iters"] == t["iters"], (t["id"], u["iters"], t["iters"])
        assert u["branch_j"] == t["branch_j"], (t["id"], u["branch_j"], t["branch_j"])
        assert abs(u["ub"] - t["ub"]) <= 1e-6 * abs(t["ub"]), (t["id"], u["ub"], t["ub"])
    st = res["stats"]
    assert st["status"] <= 1 and res["gap"] <= g["gap_tol"]
    assert np.array_equal(res["support"], inst.support_true)
    P = O.Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=g["rho"])
    ref, bS = O.upper_bound(P, res["support"])
    assert abs(res["obj"] - ref) <= 1e-9 * abs(ref), (res["obj"], ref)
    assert rel(res["beta"][res["support"]], bS) < 1e-6
    assert st["lb"] <= ref * (1 + 1e-12)


def test_upper_bound_large_supports():
    """Supports too large for the shared-memory FPG (|S| ≥ 670): the Gram is formed in HBM by a gather +
    DMMA GEMM and the FPG iterations run from it; objective = the oracle's exact ridge on
    the support (box inactive: M large), including |S| > n."""
    inst = synth.make_instance(400, 3000, 5, 0.1, 3.0, 3)
    lam0, lam2, M = 1.0, 2.0, 1e3
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    rng = np.random.default_rng(5)
    sups = [np.sort(rng.choice(inst.p, size=s, replace=False)) for s in (700, 1200, 5)]
    prob = Problem(inst.X, inst.y, lam0, lam2, M)
    obj, betas = prob.l0l2_upper_batch(sups)
    prob.close()
    for k, S in enumerate(sups):
        ref, bS = O.upper_bound(P, S)
        assert abs(float(obj[k]) - ref) <= 1e-9 * abs(ref), (len(S), float(obj[k]), ref)
        assert rel(betas[k], bS) < 1e-6

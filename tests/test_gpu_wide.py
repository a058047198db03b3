"""GPU parity of the wide-n ADMM path (-m gpu), through the C-ABI against the CPU oracle.

The fused persistent kernel holds u and its forward accumulators in registers and an n×8 tile ring
in shared memory, so it stops at n = 1056.  Larger n (the paper's n = 3000, p = 30000 workload,
P:878; its n = 11 962 data set) runs the wide-n path (admm.cu `wide_sweep` + a split-K
forward GEMM per iteration) on the same node state.  Checked here:

* the path forced at small sizes (L0L2_WIDE=1) on C3-, C5-shaped and ragged instances: fixed
  iterations (β, v, LB, primal within 1e-9 of the oracle), B ∈ {1, 16, 17}, warm starts, converged
  bounds with the oracle's iteration counts / branches / supports, a Z-form BnB tree with the
  matching-pursuit incumbent and early prune node for node against the oracle's BnB;
* the path at its natural sizes: n = 1064 (the first n past the fused kernel), n = 1500, and the
  paper's n = 3000, p = 30000 shape (root + nodes, fixed iterations; one converged root bound).
"""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2602_04551_b200 import FLAG_CONVERGED, FLAG_INTEGRAL, FLAG_PRUNED, Problem  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)), initial=0.0) / (1.0 + np.max(np.abs(b), initial=0.0)))


def _instance(kind):
    if kind == "woodbury":    # C3-shaped (p > 2n: Z-form)
        inst = synth.make_instance(200, 2000, 5, 0.1, 3.0, 3)
    elif kind == "toeplitz":  # C5-shaped
        inst = synth.make_instance(120, 1500, 5, 0.9, 1.0, 5, kind="toeplitz")
    elif kind == "ragged":    # n, p not multiples of 8, p not a multiple of the 64-column CTA block
        inst = synth.make_instance(61, 203, 4, 0.3, 4.0, 9)
    lam2 = max(synth.tune_lambda2(inst), 0.5)
    return inst, synth.lambda0_rule(inst, lam2), lam2, synth.bigM_rule(inst, lam2)


@pytest.fixture(scope="module", params=["woodbury", "toeplitz", "ragged"])
def case(request):
    inst, lam0, lam2, M = _instance(request.param)
    return request.param, inst, lam0, lam2, M, O.Problem(inst.X, inst.y, lam0, lam2, M)


@pytest.fixture
def wide(monkeypatch):
    monkeypatch.setenv("L0L2_WIDE", "1")


def _fixings(inst, B, seed):
    return [((), ())] + synth.random_fixings(inst.p, B - 1, seed=seed, depth_lo=1, depth_hi=10,
                                             prefer=inst.support_true)


def _check_fixed(P, inst, prob, fx, N, sample, warm=None):
    M = P.M
    out = prob.l0l2_bound_batch(fx, warm_in=warm)
    wo, lb, pr = out["warm_out"].cpu().numpy(), out["lb"].cpu().numpy(), out["primal"].cpu().numpy()
    it = out["iters"].cpu().numpy()
    for k in sample:
        if k >= len(fx):
            continue
        wk = None if warm is None else (warm[k, 0].cpu().numpy(), warm[k, 1].cpu().numpy())
        r = O.admm_node(P, O.make_code(inst.p, *fx[k]), node_tol=-1.0, max_iters=N, warm=wk)
        assert it[k] == N
        assert rel(wo[k, 0], r.beta) < 1e-9, (k, rel(wo[k, 0], r.beta))
        assert rel(wo[k, 1], r.v) < 1e-9, (k, rel(wo[k, 1], r.v))
        assert abs(lb[k] - r.lb) <= 1e-9 * max(1.0, abs(r.lb)), (k, lb[k], r.lb)
        assert abs(pr[k] - r.primal) <= 1e-9 * max(1.0, abs(r.primal)), (k, pr[k], r.primal)
        assert np.all(wo[k, 0][list(fx[k][0])] == 0.0)
        assert np.max(np.abs(wo[k, 0])) <= M
    return out


@pytest.mark.parametrize("B", [1, 16, 17])
def test_forced_wide_fixed_iterations(case, wide, B):
    name, inst, lam0, lam2, M, P = case
    N = 23   # checks at 10, 20 and the last iteration
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=-1.0, max_iters=N)
    assert prob.info()["admm_path"] == "wide-n"
    _check_fixed(P, inst, prob, _fixings(inst, B, seed=40 + B), N, sample=range(B))
    prob.close()


def test_forced_wide_warm_starts(case, wide):
    """Warm starts (R6): children from their parent's (β, v) with β_F0 = 0 and the refresh."""
    name, inst, lam0, lam2, M, P = case
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=-1.0, max_iters=15)
    root = prob.l0l2_bound_batch([((), ())])
    fx = synth.random_fixings(inst.p, 5, seed=7, depth_lo=1, depth_hi=3, prefer=inst.support_true)
    warm = root["warm_out"][[0] * len(fx)].contiguous()
    _check_fixed(P, inst, prob, fx, 15, sample=range(len(fx)), warm=warm)
    prob.close()


def test_forced_wide_converged_bounds_and_decisions(case, wide):
    """Converged bounds within 1e-6 with the oracle's iteration counts, branch index, integrality
    and support where the decisions are separated."""
    name, inst, lam0, lam2, M, P = case
    tol = 1e-9
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=tol, max_iters=20000)
    fx = _fixings(inst, 6, seed=11)
    out = prob.l0l2_bound_batch(fx, want_zhat=True)
    z = out["zhat"].cpu().numpy()
    for k, (F0, F1) in enumerate(fx):
        code = O.make_code(inst.p, F0, F1)
        r = O.admm_node(P, code, node_tol=tol, max_iters=20000)
        lb, pr = float(out["lb"][k]), float(out["primal"][k])
        assert abs(lb - r.lb) <= 1e-6 * max(1.0, abs(r.lb))
        assert abs(pr - r.primal) <= 1e-6 * max(1.0, abs(r.primal))
        assert int(out["flags"][k]) & FLAG_CONVERGED
        assert int(out["iters"][k]) == r.iters
        frac = np.minimum(r.z, 1 - r.z)[code == O.FREE]
        if frac.size >= 2:
            top = np.sort(frac)[-2:]
            if top[1] - top[0] > 1e-6:
                assert int(out["branch_j"][k]) == r.branch_j
        if not np.any(np.abs(r.z - 0.5) < 1e-6):
            assert bool(int(out["flags"][k]) & FLAG_INTEGRAL) == r.integral
            gpu_supp = np.nonzero(((code == O.FIX1) | ((code == O.FREE) & (z[k] >= 0.5))))[0]
            assert np.array_equal(gpu_supp, r.support)
    prob.close()


def test_forced_wide_dual_residual(case, wide):
    name, inst, lam0, lam2, M, P = case
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=-1.0, max_iters=20)
    out = prob.l0l2_bound_batch([((), ())], want_dual_r=True)
    r = O.admm_node(P, O.make_code(inst.p), node_tol=-1.0, max_iters=20)
    assert rel(out["dual_r"][0].cpu().numpy(), inst.y - inst.X @ r.b) < 1e-9
    prob.close()


@pytest.mark.parametrize("B", [1, 16])
def test_forced_wide_tree_parity_mp_early_prune(wide, B):
    """A Z-form tree (p > 2n) with the MP incumbent and early prune (R16) on the device frontier:
    node for node = the oracle's BnB (ids, LBs 1e-6, iterations, branches, early-pruned nodes)."""
    inst = synth.make_instance(50, 130, 3, 0.2, 6.0, 5)   # 123-node oracle tree at B = 16
    lam2 = 0.5
    lam0 = synth.lambda0_rule(inst, lam2)
    M = synth.bigM_rule(inst, lam2)
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    ref = O.bnb_solve(P, B=B, gap_tol=1e-4, node_tol=1e-8, record=True, early_prune=True, init_mp=True)
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-8)
    assert prob.info()["admm_path"] == "wide-n"
    res = prob.l0l2_solve(gap_tol=1e-4, batch=B, record=True, early_prune=True, init_mp=True)
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
    prob.close()


def test_forced_wide_solve_equals_brute_force(wide):
    inst = synth.make_instance(6, 14, 3, 0.3, 4.0, 5)   # p > 2n: the Z-form (L0L2_WIDE applies)
    lam2 = 0.3
    lam0 = synth.lambda0_rule(inst, lam2)
    M = synth.bigM_rule(inst, lam2)
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    bf_obj, bf_S, _ = O.brute_force(P)
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-10, max_iters=20000)
    assert prob.info()["admm_path"] == "wide-n"
    res = prob.l0l2_solve(gap_tol=1e-9, batch=8)
    assert abs(res["obj"] - bf_obj) <= 1e-9 * abs(bf_obj)
    assert list(res["support"]) == list(bf_S)
    prob.close()


@pytest.mark.parametrize("n,p", [(1064, 2200), (1500, 4000)])
def test_wide_beyond_the_fused_kernel(n, p):
    """n past the fused kernel's tile ring (formerly L0L2_EINVAL): the wide-n path, 17 nodes, fixed
    iterations, vs the oracle."""
    inst = synth.make_instance(n, p, 5, 0.3, 4.0, 31)
    lam2 = 0.5
    lam0 = synth.lambda0_rule(inst, lam2)
    M = synth.bigM_rule(inst, lam2)
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=-1.0, max_iters=21)
    assert prob.info()["admm_path"] == "wide-n"
    _check_fixed(P, inst, prob, _fixings(inst, 17, seed=4), 21, sample=(0, 7, 8, 15, 16))
    prob.close()


@pytest.fixture(scope="module")
def paper_n3000():
    """The paper's n = 3000, p = 30000 workload (SNR 10/3, k = 10; λ2, λ0, M by the recipe of
    DESIGN.md §5)."""
    inst = synth.make_instance(3000, 30000, 10, 0.1, 10.0 / 3.0, 0)
    lam2 = synth.tune_lambda2(inst)
    lam0 = synth.lambda0_rule(inst, lam2)
    M = synth.bigM_rule(inst, lam2)
    rho = 3.0 * O.default_rho(inst.X)
    return inst, lam0, lam2, M, O.Problem(inst.X, inst.y, lam0, lam2, M, rho=rho)


def test_paper_shape_n3000_fixed_iterations(paper_n3000):
    inst, lam0, lam2, M, P = paper_n3000
    prob = Problem(np.asfortranarray(inst.X), inst.y, lam0, lam2, M, rho=P.rho, node_tol=-1.0, max_iters=12)
    assert prob.info()["admm_path"] == "wide-n"
    _check_fixed(P, inst, prob, _fixings(inst, 16, seed=5), 12, sample=(0, 5, 15))
    prob.close()


def test_paper_shape_n3000_converged_root(paper_n3000):
    """The root relaxation to node_tol 1e-4: same iteration count, LB and primal within 1e-6."""
    inst, lam0, lam2, M, P = paper_n3000
    prob = Problem(np.asfortranarray(inst.X), inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-4, max_iters=3000)
    out = prob.l0l2_bound_batch([((), ())])
    r = O.admm_node(P, O.make_code(inst.p), node_tol=1e-4, max_iters=3000)
    assert int(out["iters"][0]) == r.iters
    assert abs(float(out["lb"][0]) - r.lb) <= 1e-6 * max(1.0, abs(r.lb))
    assert abs(float(out["primal"][0]) - r.primal) <= 1e-6 * max(1.0, abs(r.primal))
    prob.close()

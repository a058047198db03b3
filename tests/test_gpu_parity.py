"""GPU parity: the sm_100a library (through the C-ABI) against the CPU oracle (-m gpu).

Tolerances: FP64 throughout; the two sides use different formulations of
the same b-update (GPU: Z-form (I − ZᵀZ)/ρ with identity-based checks; oracle: direct D or
Woodbury G-form with explicit r̂ = y − Xb̂), so iterates agree to rounding amplified by the
iteration count: fixed-iteration states within 1e-9 relative, bounds within 1e-9 relative,
converged bounds / objectives within 1e-6 (north star), integer decisions (iteration counts,
branch index, support) exactly where separated.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2602_04551_b200 import FLAG_CONVERGED, FLAG_INTEGRAL, FLAG_PRUNED, L0L2Error, Problem  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)), initial=0.0) / (1.0 + np.max(np.abs(b), initial=0.0)))


def _instance(kind):
    if kind == "C1":
        inst = synth.config_instance("C1", seed=0)
        return inst, inst.lambda0, inst.lambda2, inst.M
    if kind == "direct":     # n ≥ p: the oracle uses the direct D
        inst = synth.make_instance(300, 120, 6, 0.5, 5.0, 7)
    elif kind == "woodbury":  # p > n: C3-shaped
        inst = synth.make_instance(200, 2000, 5, 0.1, 3.0, 3)
    elif kind == "toeplitz":  # C5-shaped
        inst = synth.make_instance(120, 1500, 5, 0.9, 1.0, 5, kind="toeplitz")
    elif kind == "ragged":    # n, p not multiples of 8 (ragged tiles and rows)
        inst = synth.make_instance(61, 203, 4, 0.3, 4.0, 9)
    lam2 = synth.tune_lambda2(inst)
    lam2 = max(lam2, 0.5)
    return inst, synth.lambda0_rule(inst, lam2), lam2, synth.bigM_rule(inst, lam2)


KINDS = ["C1", "direct", "woodbury", "toeplitz", "ragged"]


@pytest.fixture(scope="module", params=KINDS)
def case(request):
    inst, lam0, lam2, M = _instance(request.param)
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    return request.param, inst, lam0, lam2, M, P


def _fixings(inst, B, seed):
    return [((), ())] + synth.random_fixings(inst.p, B - 1, seed=seed, depth_lo=1, depth_hi=10,
                                             prefer=inst.support_true)


@pytest.mark.parametrize("B", [1, 3, 8, 17])
def test_fixed_iteration_state_and_bounds(case, B):
    """T2: after N iterations with node_tol disabled, β, v, LB, primal match the oracle."""
    name, inst, lam0, lam2, M, P = case
    N = 57
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=-1.0, max_iters=N)
    fx = _fixings(inst, B, seed=B)
    out = prob.l0l2_bound_batch(fx, want_zhat=True)
    wo, lb, pr = out["warm_out"].cpu().numpy(), out["lb"].cpu().numpy(), out["primal"].cpu().numpy()
    it = out["iters"].cpu().numpy()
    for k, (F0, F1) in enumerate(fx):
        r = O.admm_node(P, O.make_code(inst.p, F0, F1), node_tol=-1.0, max_iters=N)
        assert it[k] == N
        assert rel(wo[k, 0], r.beta) < 1e-9, (name, k, rel(wo[k, 0], r.beta))
        assert rel(wo[k, 1], r.v) < 1e-9
        assert abs(lb[k] - r.lb) <= 1e-9 * max(1.0, abs(r.lb)), (name, k, lb[k], r.lb)
        assert abs(pr[k] - r.primal) <= 1e-9 * max(1.0, abs(r.primal))
        assert np.all(wo[k, 0][list(F0)] == 0.0)            # β_F0 = 0 exactly
        assert np.max(np.abs(wo[k, 0])) <= M                 # box, exactly
    prob.close()


def test_warm_start_parity(case):
    """Warm start: children continue from the parent's (β, v) in both implementations."""
    name, inst, lam0, lam2, M, P = case
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=-1.0, max_iters=30)
    root = prob.l0l2_bound_batch([((), ())])
    warm = root["warm_out"]
    r0 = O.admm_node(P, O.make_code(inst.p), node_tol=-1.0, max_iters=30)
    j = int(root["branch_j"][0].item())
    if j < 0:
        j = 0
    kids = [((j,), ()), ((), (j,))]
    out = prob.l0l2_bound_batch(kids, warm_in=torch.cat([warm, warm]), parent_lb=[float(root["lb"][0])] * 2)
    for k, (F0, F1) in enumerate(kids):
        r = O.admm_node(P, O.make_code(inst.p, F0, F1), warm=(r0.beta, r0.v), parent_lb=r0.lb,
                        node_tol=-1.0, max_iters=30)
        assert rel(out["warm_out"][k, 0].cpu().numpy(), r.beta) < 1e-9
        assert abs(float(out["lb"][k]) - r.lb) <= 1e-9 * max(1.0, abs(r.lb))
    prob.close()


def test_batched_equals_single_bitwise(case):
    """T4: a node's arithmetic is independent of the other nodes in its batch (bitwise)."""
    name, inst, lam0, lam2, M, P = case
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-8, max_iters=400)
    fx = _fixings(inst, 11, seed=3)
    batch = prob.l0l2_bound_batch(fx)
    for k in (0, 4, 9):
        one = prob.l0l2_bound_batch([fx[k]])
        assert torch.equal(one["warm_out"][0], batch["warm_out"][k])
        assert float(one["lb"][0]) == float(batch["lb"][k])
        assert int(one["iters"][0]) == int(batch["iters"][k])
    prob.close()


def test_paired_equals_split_bitwise(case, monkeypatch):
    """A 16-node group on paired CTAs (both node halves stream the same tiles, halves retire at
    their own checks, the mode switches to single-half mid-launch) gives bitwise the results of the
    same group run as two single-half launches (L0L2_PAIR=0)."""
    name, inst, lam0, lam2, M, P = case
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-6, max_iters=600)
    fx = _fixings(inst, 16, seed=5)
    monkeypatch.setenv("L0L2_PAIR", "1")
    paired = prob.l0l2_bound_batch(fx)
    monkeypatch.setenv("L0L2_PAIR", "0")
    split = prob.l0l2_bound_batch(fx)
    for key in ("warm_out", "lb", "primal", "iters", "branch_j", "flags"):
        assert torch.equal(paired[key], split[key]), key
    prob.close()


def test_compaction_is_bitwise_invisible(case, monkeypatch):
    """Node-slot compaction (≤ 8 active nodes spread over both halves are moved into half 0 for
    single-half sweeps) changes no result bit: compare with compaction disabled."""
    name, inst, lam0, lam2, M, P = case
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-7, max_iters=800)
    fx = _fixings(inst, 16, seed=8)
    monkeypatch.setenv("L0L2_COMPACT", "1")
    a = prob.l0l2_bound_batch(fx, want_dual_r=True)
    monkeypatch.setenv("L0L2_COMPACT", "0")
    b = prob.l0l2_bound_batch(fx, want_dual_r=True)
    for key in ("warm_out", "lb", "primal", "iters", "branch_j", "flags", "dual_r"):
        assert torch.equal(a[key], b[key]), key
    it = a["iters"].cpu().numpy()
    assert len(set(it.tolist())) > 1   # nodes retire at different checks
    prob.close()


def test_column_gather_equals_row_gather(case, monkeypatch):
    """The primal check's ‖Xβ⁺‖²: the whole-column gather from the epilogue's segments (default in the
    Z-form, no compaction, no dense fallback) and the row-slice gather over compacted per-node lists
    (L0L2_GATHER=1) agree to rounding with the same iteration counts and decisions, and the default
    keeps a node's result independent of the other nodes (one node alone = the same node in a
    16-node batch, bitwise)."""
    name, inst, lam0, lam2, M, P = case
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-7, max_iters=800)
    fx = _fixings(inst, 16, seed=9)
    monkeypatch.setenv("L0L2_GATHER", "0")
    a = prob.l0l2_bound_batch(fx)
    single = prob.l0l2_bound_batch(fx[5:6])
    monkeypatch.setenv("L0L2_GATHER", "1")
    b = prob.l0l2_bound_batch(fx)
    assert torch.equal(a["iters"], b["iters"]) and torch.equal(a["branch_j"], b["branch_j"])
    for key in ("lb", "primal"):
        x, y = a[key].cpu().numpy(), b[key].cpu().numpy()
        assert np.all(np.abs(x - y) <= 1e-12 * np.maximum(1.0, np.abs(y))), key
    for key in ("warm_out", "lb", "primal", "iters", "flags"):
        assert torch.equal(a[key][5:6], single[key]), key
    prob.close()


def test_converged_bounds_and_decisions(case):
    """T3: converged LB / primal within 1e-6; LB ≤ independent relaxation optimum; iteration
    counts, branch index and support equal where the decisions are separated."""
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
        if inst.p <= 20:
            opt, _ = O.relaxation_fista(P, code)
            assert lb <= opt + 1e-8 * max(1.0, abs(opt))
    prob.close()


def test_dual_residual_output(case):
    """dual_r = y − X b̂ at the last check."""
    name, inst, lam0, lam2, M, P = case
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=-1.0, max_iters=20)
    out = prob.l0l2_bound_batch([((), ())], want_dual_r=True)
    r = O.admm_node(P, O.make_code(inst.p), node_tol=-1.0, max_iters=20)
    ref = inst.y - inst.X @ r.b
    assert rel(out["dual_r"][0].cpu().numpy(), ref) < 1e-9
    prob.close()


def test_upper_batch(case):
    """T5: FPG objective = exact box-ridge optimum (1e-9), incl. empty and box-active supports."""
    name, inst, lam0, lam2, M, P = case
    sups = [np.array([], dtype=np.int64), inst.support_true] + synth.random_supports(inst.p, 6, seed=2, s_lo=1,
                                                                                     s_hi=min(40, inst.p))
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho)
    obj, betas = prob.l0l2_upper_batch(sups)
    for k, S in enumerate(sups):
        ref, bS = O.upper_bound(P, S)
        assert abs(float(obj[k]) - ref) <= 1e-9 * max(1.0, abs(ref)), (k, float(obj[k]), ref)
        if len(S):
            assert rel(betas[k], bS) < 1e-6
    prob.close()
    # box-active: a small M clamps coefficients
    Ms = 0.05 * M
    P2 = O.Problem(inst.X, inst.y, lam0, lam2, Ms)
    prob = Problem(inst.X, inst.y, lam0, lam2, Ms)
    obj, betas = prob.l0l2_upper_batch([inst.support_true])
    ref, bS = O.upper_bound(P2, inst.support_true)
    assert abs(float(obj[0]) - ref) <= 1e-9 * abs(ref)
    prob.close()


def test_edge_cases():
    inst, lam0, lam2, M = _instance("C1")
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-10)
    # all coordinates fixed to zero: β = 0, bound = ½‖y‖²
    out = prob.l0l2_bound_batch([(tuple(range(inst.p)), ())])
    assert abs(float(out["lb"][0]) - 0.5 * P.yy) <= 1e-9 * P.yy
    assert int(out["branch_j"][0]) == -1 and int(out["flags"][0]) & FLAG_INTEGRAL
    # all fixed to one: relaxation = box ridge on all columns + λ0 p
    out = prob.l0l2_bound_batch([((), tuple(range(inst.p)))])
    ref, _ = O.upper_bound(P, np.arange(inst.p))
    assert abs(float(out["lb"][0]) - ref) <= 1e-6 * abs(ref)
    # F0 ∩ F1 ≠ ∅ and out-of-range indices are rejected
    with pytest.raises(L0L2Error):
        prob.l0l2_bound_batch([((1,), (1,))])
    with pytest.raises(L0L2Error):
        prob.l0l2_bound_batch([((inst.p + 3,), ())])
    # empty batch
    assert prob.l0l2_upper_batch([])[0].numel() == 0
    prob.close()


@pytest.mark.parametrize("seed", range(8))
def test_solve_equals_brute_force(seed):
    """T6: certified optimum = brute force (support exact, objective 1e-9)."""
    if seed == 0:
        inst = synth.config_instance("C1", seed=0)
        lam0, lam2, M = inst.lambda0, inst.lambda2, inst.M
    else:
        rng = np.random.default_rng(seed)
        n, p = int(rng.choice([15, 30, 60])), int(rng.choice([6, 9, 12]))
        inst = synth.make_instance(n, p, 3, float(rng.choice([0.0, 0.2, 0.5])), 5.0, seed)
        lam0, lam2, M = float(rng.uniform(0.01, 1)) * n / 10, float(rng.uniform(0.01, 1)), float(rng.uniform(1, 10))
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    obj, S, _ = O.brute_force(P)
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-10, max_iters=20000)
    for B in (1, 8):
        res = prob.l0l2_solve(gap_tol=1e-9, batch=B)
        assert abs(res["obj"] - obj) <= 1e-9 * max(1.0, abs(obj))
        assert np.array_equal(res["support"], S)
        assert res["stats"]["lb"] <= obj * (1 + 1e-9)
    prob.close()


@pytest.mark.parametrize("B", [1, 4, 16])
def test_solve_tree_parity(B):
    """T7: node-for-node tree parity with the oracle's BnB (same ids, bounds, iterations, branches)."""
    # ~100-node tree that the oracle closes to a 1e-4 gap in well under a second
    inst = synth.make_instance(80, 60, 5, 0.3, 3.0, 21)
    lam2 = 0.5
    lam0 = synth.lambda0_rule(inst, lam2)
    M = synth.bigM_rule(inst, lam2)
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    ref = O.bnb_solve(P, B=B, gap_tol=1e-4, node_tol=1e-8, record=True)
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-8)
    res = prob.l0l2_solve(gap_tol=1e-4, batch=B, record=True)
    assert abs(res["obj"] - ref["obj"]) <= 1e-9 * abs(ref["obj"])
    assert np.array_equal(res["support"], ref["support"])
    gt = {t["id"]: t for t in res["trace"]}
    matched = 0
    for t in ref["trace"]:
        g = gt.get(t["id"])
        assert g is not None, ("node missing on GPU", t["id"])
        assert abs(g["lb"] - t["lb"]) <= 1e-6 * max(1.0, abs(t["lb"]))
        assert g["iters"] == t["iters"]
        assert g["branch_j"] == t["branch_j"] or t["branch_j"] < 0
        matched += 1
    assert matched == len(res["trace"]) == ref["nodes"]
    prob.close()


@pytest.mark.parametrize("B", [1, 16])
def test_solve_tree_parity_early_prune(B):
    """Early prune (R16) on both sides: node-for-node parity with the oracle's BnB (same ids,
    bounds, iterations, branches, and the same nodes stopped early), same certificate."""
    inst = synth.make_instance(80, 60, 5, 0.3, 3.0, 21)
    lam2 = 0.5
    lam0 = synth.lambda0_rule(inst, lam2)
    M = synth.bigM_rule(inst, lam2)
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    ref = O.bnb_solve(P, B=B, gap_tol=1e-4, node_tol=1e-8, record=True, early_prune=True)
    assert any(t["early"] for t in ref["trace"])
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-8)
    res = prob.l0l2_solve(gap_tol=1e-4, batch=B, record=True, early_prune=True)
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


def test_c4_full_size_sampled():
    """BASELINE C4 (n=1000, p=1e5) in the bench's configuration: root ADMM state after a fixed
    number of iterations vs the oracle (all p coordinates), and the first 31 nodes of the solve
    vs the oracle's committed tree prefix (tests/golden/oracle_C4_prefix.json, written by
    tools/oracle_c4_prefix.py from oracle/ only)."""
    inst = synth.config_instance("C4", seed=0)
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_C4_prefix.json")))
    rho = golden["rho"]
    assert abs(inst.lambda0 - golden["lambda0"]) <= 1e-12 * golden["lambda0"]
    P = O.Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho)
    prob = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=-1.0, max_iters=12)
    out = prob.l0l2_bound_batch([((), ())])
    r = O.admm_node(P, O.make_code(inst.p), node_tol=-1.0, max_iters=12)
    assert rel(out["warm_out"][0, 0].cpu().numpy(), r.beta) < 1e-9
    assert rel(out["warm_out"][0, 1].cpu().numpy(), r.v) < 1e-9
    assert abs(float(out["lb"][0]) - r.lb) <= 1e-9 * abs(r.lb)
    prob.close()
    prob = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=golden["node_tol"])
    res = prob.l0l2_solve(gap_tol=golden["gap_tol"], batch=golden["batch"], node_limit=golden["nodes"], record=True)
    gt = {t["id"]: t for t in res["trace"]}
    for t in golden["trace"]:
        g = gt[t["id"]]
        assert abs(g["lb"] - t["lb"]) <= 1e-6 * abs(t["lb"]), (t["id"], g["lb"], t["lb"])
        assert g["iters"] == t["iters"], (t["id"], g["iters"], t["iters"])
        assert g["branch_j"] == t["branch_j"]
        assert abs(g["ub"] - t["ub"]) <= 1e-6 * abs(t["ub"])
    assert res["stats"]["nodes"] == golden["nodes"]
    assert abs(res["obj"] - golden["ub"]) <= 1e-6 * golden["ub"]
    prob.close()


# ---------------------------------------------------------------- matching pursuit (Algorithm 3)
def test_matching_pursuit_parity(case):
    """l0l2_matching_pursuit vs the oracle's Algorithm 3: same support (bit-exact
    integer decisions), β within 1e-9, objective within 1e-9 relative, same number of rounds."""
    name, inst, lam0, lam2, M, P = case
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho)
    g = prob.l0l2_matching_pursuit()
    r = O.matching_pursuit(P)
    assert list(g["support"]) == list(r.support), name
    assert rel(g["beta"], r.beta) < 1e-9
    assert abs(g["obj"] - r.obj) <= 1e-9 * abs(r.obj)
    assert g["rounds"] == r.rounds
    assert np.all(np.abs(g["beta"]) <= M)
    prob.close()


def test_matching_pursuit_c4_full_size():
    """Algorithm 3 at the bench's full size (C4: n=1000, p=1e5) vs the oracle."""
    inst = synth.config_instance("C4", seed=0)
    P = O.Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=1.0)
    prob = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=1.0)
    g = prob.l0l2_matching_pursuit()
    r = O.matching_pursuit(P)
    assert list(g["support"]) == list(r.support)
    assert rel(g["beta"], r.beta) < 1e-9
    assert abs(g["obj"] - r.obj) <= 1e-9 * abs(r.obj)
    assert g["rounds"] == r.rounds
    prob.close()


@pytest.mark.parametrize("seed", [0, 3])
def test_solve_with_mp_incumbent(seed):
    """l0l2_solve with the matching-pursuit incumbent (init_mp) still certifies the
    brute-force optimum, and its answer is never worse than the heuristic's own objective."""
    inst = synth.config_instance("C1", seed=seed)
    P = O.Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M)
    bf_obj, bf_S, _ = O.brute_force(P)
    prob = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=P.rho, node_tol=1e-10, max_iters=20000)
    mp = prob.l0l2_matching_pursuit()
    res = prob.l0l2_solve(gap_tol=1e-9, batch=8, init_mp=True)
    assert abs(res["obj"] - bf_obj) <= 1e-9 * abs(bf_obj)
    assert list(res["support"]) == list(bf_S)
    assert res["obj"] <= mp["obj"] * (1 + 1e-12)
    prob.close()


@pytest.mark.parametrize("n", [1008, 1056])
def test_largest_n_classes(n):
    """The two largest n classes of the ADMM kernel (n8 = 1008, and 1056 = the largest n whose tile
    ring fits: most registers, least shared-memory slack, fragment rows running past ld into the next
    stage) vs the oracle, with a 16+1-node batch (paired CTAs, compaction), fixed iterations."""
    inst = synth.make_instance(n, 2200, 5, 0.3, 4.0, 31)   # p > 2n: the Z-form kernel at its largest n classes
    lam2 = 0.5
    lam0 = synth.lambda0_rule(inst, lam2)
    M = synth.bigM_rule(inst, lam2)
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=-1.0, max_iters=23)
    fx = _fixings(inst, 17, seed=4)
    out = prob.l0l2_bound_batch(fx)
    wo, lb = out["warm_out"].cpu().numpy(), out["lb"].cpu().numpy()
    for k in (0, 7, 8, 15, 16):
        r = O.admm_node(P, O.make_code(inst.p, *fx[k]), node_tol=-1.0, max_iters=23)
        assert rel(wo[k, 0], r.beta) < 1e-9, (n, k)
        assert abs(lb[k] - r.lb) <= 1e-9 * max(1.0, abs(r.lb))
    prob.close()


@pytest.mark.parametrize("variant", ["lambda0_zero", "box_inactive", "box_tight"])
def test_degenerate_penalties(variant):
    """Degenerate penalty settings of eq:perspective: λ0 = 0 (no ℓ0 term: ψ is the pure ridge
    branch, ẑ ∈ {0, 1}), M ≫ ‖β‖∞ (box never active), M tiny (box active on most coordinates).
    Fixed-iteration ADMM state vs the oracle, and the certified solve = brute force."""
    inst = synth.make_instance(40, 12, 3, 0.2, 4.0, 2)   # p = 12: brute force in milliseconds
    lam2 = 0.05
    lam0, M = synth.lambda0_rule(inst, lam2), synth.bigM_rule(inst, lam2)
    if variant == "lambda0_zero":
        lam0 = 0.0
    elif variant == "box_inactive":
        M = 1e3
    else:
        M = 0.05
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=-1.0, max_iters=37)
    fx = _fixings(inst, 5, seed=2)
    out = prob.l0l2_bound_batch(fx)
    wo, lb = out["warm_out"].cpu().numpy(), out["lb"].cpu().numpy()
    for k, (F0, F1) in enumerate(fx):
        r = O.admm_node(P, O.make_code(inst.p, F0, F1), node_tol=-1.0, max_iters=37)
        assert rel(wo[k, 0], r.beta) < 1e-9, (variant, k)
        assert abs(lb[k] - r.lb) <= 1e-9 * max(1.0, abs(r.lb))
    prob.close()
    bf_obj, bf_S, _ = O.brute_force(P)
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-10, max_iters=20000)
    res = prob.l0l2_solve(gap_tol=1e-9, batch=8)
    assert abs(res["obj"] - bf_obj) <= 1e-8 * max(1.0, abs(bf_obj)), (variant, res["obj"], bf_obj)
    prob.close()


def test_direct_regime_equals_zform(monkeypatch):
    """R17: for p ≤ 2n the kernel streams D = (I − ZᵀZ)/ρ (p×p) instead of Z; same bounds (1e-9),
    iteration counts and branches as the Z-form on the same nodes, and both vs the oracle."""
    inst, lam0, lam2, M = _instance("direct")
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    fx = _fixings(inst, 17, seed=6)
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("L0L2_DIRECT", mode)
        prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=1e-7, max_iters=3000)
        outs[mode] = prob.l0l2_bound_batch(fx)
        prob.close()
    a, b = outs["1"], outs["0"]
    la, lb_ = a["lb"].cpu().numpy(), b["lb"].cpu().numpy()
    assert np.max(np.abs(la - lb_) / np.maximum(1.0, np.abs(lb_))) < 1e-9
    assert torch.equal(a["iters"], b["iters"]) and torch.equal(a["branch_j"], b["branch_j"])
    for k in (0, 9, 16):
        r = O.admm_node(P, O.make_code(inst.p, *fx[k]), node_tol=1e-7, max_iters=3000)
        assert abs(float(la[k]) - r.lb) <= 1e-6 * max(1.0, abs(r.lb))
        assert int(a["iters"][k]) == r.iters


def test_direct_regime_lifts_the_n_limit():
    """n > 1056 with p ≤ min(2n, 1056): the direct regime streams D (p×p), so the Z-form's n limit
    does not apply; fixed-iteration state vs the oracle."""
    inst = synth.make_instance(1500, 300, 5, 0.3, 4.0, 8)
    lam2 = 0.5
    lam0, M = synth.lambda0_rule(inst, lam2), synth.bigM_rule(inst, lam2)
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=P.rho, node_tol=-1.0, max_iters=29)
    fx = _fixings(inst, 9, seed=3)
    out = prob.l0l2_bound_batch(fx)
    wo, lb = out["warm_out"].cpu().numpy(), out["lb"].cpu().numpy()
    for k in (0, 4, 8):
        r = O.admm_node(P, O.make_code(inst.p, *fx[k]), node_tol=-1.0, max_iters=29)
        assert rel(wo[k, 0], r.beta) < 1e-9
        assert abs(lb[k] - r.lb) <= 1e-9 * max(1.0, abs(r.lb))
    prob.close()

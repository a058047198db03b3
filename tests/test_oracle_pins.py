"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the passage it pins.  None of them re-types the oracle's formula: they
check hand-derived values (tests/golden), definitions the formulas were derived from
(the z/s minimisation of P:1077-1104, the conjugate of P:1152-1169, the prox argmin of
P:388), closed forms, an independent library route (scipy lsq_linear), brute force and
invariants.
"""
import itertools
import math

import numpy as np
import pytest
from scipy.optimize import lsq_linear, minimize_scalar

import oracle as O
import synth

CODES = {"free": O.FREE, "F0": O.FIX0, "F1": O.FIX1}


# ---------------------------------------------------------------- golden hand-derived values
def test_golden_T(golden):
    for e in golden["T"]:
        assert float(O.T(*e["args"])) == pytest.approx(e["value"], abs=0), e["cite"]


def test_golden_psi_h_nu_prox_z(golden):
    for e in golden["psi"]:
        v = O.psi(e["beta"], CODES[e["code"]], e["lam0"], e["lam2"], e["M"])
        assert float(v) == pytest.approx(e["value"], rel=1e-15, abs=1e-15), e["cite"]
    for e in golden["h"]:
        assert float(O.h(e["x"], e["lam0"], e["lam2"], e["M"])) == pytest.approx(e["value"], abs=1e-15), e["cite"]
    for e in golden["nu"]:
        v = O.nu(e["x"], CODES[e["code"]], e["lam0"], e["lam2"], e["M"])
        assert float(v) == pytest.approx(e["value"], abs=1e-15), e["cite"]
    for e in golden["prox"]:
        v = O.prox_beta(e["bt"], CODES[e["code"]], e["lam0"], e["lam2"], e["M"], e["rho"])
        assert float(v) == pytest.approx(e["value"], abs=1e-15), e["cite"]
    for e in golden["z"]:
        v = O.recover_z(e["beta"], CODES[e["code"]], e["lam0"], e["lam2"], e["M"])
        assert float(v) == pytest.approx(e["value"], abs=1e-15), e["cite"]


def test_golden_D_and_ub_and_mip(golden):
    for e in golden["D"]:
        P = O.Problem(np.array(e["X"]), np.array(e["y"]), 0.1, 1.0, 10.0, rho=e["rho"])
        assert P.apply_D(np.array([1.0]))[0] == pytest.approx(e["D"][0][0], abs=1e-15), e["cite"]
        assert P.c[0] == pytest.approx(e["c"][0]), e["cite"]
    for e in golden["ub"]:
        P = O.Problem(np.array(e["X"]), np.array(e["y"]), 0.0, e["lam2"], e["M"])
        obj, b = O.upper_bound(P, [0])
        assert b[0] == pytest.approx(e["beta"][0], abs=1e-14), e["cite"]
    for e in golden["mip"]:
        P = O.Problem(np.array(e["X"]), np.array(e["y"]), e["lam0"], e["lam2"], e["M"])
        obj, S, _ = O.brute_force(P)
        assert obj == pytest.approx(e["obj"], abs=1e-14), e["cite"]
        assert list(S) == e["support"], e["cite"]
        res = O.bnb_solve(P, B=1, gap_tol=1e-9, node_tol=1e-10)
        assert res["obj"] == pytest.approx(e["obj"], abs=1e-12), e["cite"]


def test_golden_admm_start(golden):
    """the root (cold) node starts at β = v = 0 with NO refresh; a child takes the parent's
    (β, v), zeroes β on F0, then refreshes b and v before iterating (hand-derived 1-D values)."""
    for e in golden["admm_start"]:
        P = O.Problem(np.array(e["X"]), np.array(e["y"]), e["lam0"], e["lam2"], e["M"], rho=e["rho"])
        warm = None if e["warm"] is None else (np.array([e["warm"][0]]), np.array([e["warm"][1]]))
        r = O.admm_node(P, np.array([CODES[e["code"]]], dtype=np.int8), warm=warm, node_tol=-1.0,
                        max_iters=e["iters"])
        assert r.beta[0] == pytest.approx(e["beta"], abs=1e-15), e["cite"]
        assert r.v[0] == pytest.approx(e["v"], abs=1e-15), e["cite"]


def test_golden_branch_rule(golden):
    """R10: most fractional free ẑ, ties → larger |β_j|, then lower j; integrality
     and the rounded support F1 ∪ {ẑ ≥ ½} on hand-built (β, code) vectors."""
    for e in golden["branch"]:
        code = np.array([CODES[c] for c in e["code"]], dtype=np.int8)
        z, integral, support, j = O.finalize_node(np.array(e["beta"]), code, e["lam0"], e["lam2"], e["M"])
        assert j == e["branch_j"], e["cite"]
        assert integral == e["integral"], e["cite"]
        assert list(support) == e["support"], e["cite"]


# ---------------------------------------------------------------- operator properties
def _rand_params(rng):
    lam0 = float(10 ** rng.uniform(-3, 1))
    lam2 = float(10 ** rng.uniform(-3, 1))
    M = float(10 ** rng.uniform(-1, 1))
    rho = float(10 ** rng.uniform(-1, 2))
    return lam0, lam2, M, rho


def test_T_properties():
    """eq:Tdef: odd, nondecreasing, 1-Lipschitz, |T| ≤ m."""
    rng = np.random.default_rng(1)
    t = rng.normal(scale=5, size=10000)
    a = rng.uniform(0, 3, size=10000)
    m = rng.uniform(0.1, 5, size=10000)
    f = O.T(t, a, m)
    assert np.array_equal(O.T(-t, a, m), -f)
    assert np.all(np.abs(f) <= m)
    dt = rng.uniform(0, 1, size=10000)
    g = O.T(t + dt, a, m)
    assert np.all(g >= f) and np.all(g - f <= dt + 1e-15)


def test_psi_is_the_zs_minimum():
    """ψ (eq:psi) equals min over (z, s) of λ0 z + λ2 s, β² ≤ s z, |β| ≤ M z, z ∈ [0,1]
    (eq:minzs), solved here numerically in z with s = β²/z."""
    rng = np.random.default_rng(2)
    for _ in range(600):
        lam0, lam2, M, _ = _rand_params(rng)
        beta = float(rng.uniform(-M, M))
        if abs(beta) < 1e-9:
            continue
        f = lambda z: lam0 * z + lam2 * beta * beta / z
        res = minimize_scalar(f, bounds=(abs(beta) / M, 1.0), method="bounded",
                              options=dict(xatol=1e-13))
        ref = min(res.fun, f(abs(beta) / M), f(1.0))
        got = float(O.psi(beta, O.FREE, lam0, lam2, M))
        assert got == pytest.approx(ref, rel=1e-7, abs=1e-10)
        assert float(O.psi(beta, O.FIX1, lam0, lam2, M)) == pytest.approx(lam0 + lam2 * beta * beta)
        assert float(O.psi(beta, O.FIX0, lam0, lam2, M)) == math.inf
        # z recovery: the minimiser of the same problem
        z = float(O.recover_z(beta, O.FREE, lam0, lam2, M))
        assert f(z) == pytest.approx(ref, rel=1e-7, abs=1e-10)
        s = beta * beta / z
        assert beta * beta <= s * z + 1e-12 and abs(beta) <= M * z + 1e-12


def _grid(M, k=400001):
    return np.append(np.linspace(-M, M, k), 0.0)   # exact 0 for the F0 indicator


def test_nu_is_the_conjugate_of_psi():
    """ν_i(x) = max_{|β|≤M} [xβ − ψ_i(β)]  (P:1152-1169 derive min ψ − xβ = −ν), by grid."""
    rng = np.random.default_rng(3)
    for _ in range(300):
        lam0, lam2, M, _ = _rand_params(rng)
        g = _grid(M)
        for code in (O.FREE, O.FIX1):
            ps = O.psi(g, code, lam0, lam2, M)
            for x in rng.uniform(0, 4 * (lam2 * M + lam0 / M), size=3):
                ref = float(np.max(x * g - ps))
                got = float(O.nu(x, code, lam0, lam2, M))
                # grid resolution: error ≤ (slope range)·(spacing)
                tol = (x + 2 * lam2 * M + lam0 / M) * (2 * M / 400000) + 1e-12
                assert got == pytest.approx(ref, abs=tol)
        assert float(O.nu(1.3, O.FIX0, lam0, lam2, M)) == 0.0


def test_h_continuity():
    """h (eq:hdef) is continuous at x = 2Mλ2."""
    rng = np.random.default_rng(4)
    for _ in range(1000):
        lam0, lam2, M, _ = _rand_params(rng)
        x0 = 2 * M * lam2
        lo = float(O.h(x0, lam0, lam2, M))
        hi = float(O.h(x0 * (1 + 1e-12), lam0, lam2, M))
        assert hi == pytest.approx(lo, rel=1e-9, abs=1e-12)


def test_prox_is_the_argmin():
    """eq:minbetalower attains min_β ρ/2(β−β̃)² + ψ(β) over |β| ≤ M, by grid.
    Guards against the Algorithm-2 / batched form [R3]."""
    rng = np.random.default_rng(5)
    worst = 0.0
    for _ in range(400):
        lam0, lam2, M, rho = _rand_params(rng)
        g = _grid(M, 200001)
        for code in (O.FREE, O.FIX1, O.FIX0):
            ps = O.psi(g, code, lam0, lam2, M)
            for bt in rng.normal(scale=3 * M, size=3):
                obj = 0.5 * rho * (g - bt) ** 2 + ps
                ref = float(np.min(obj))
                b = float(O.prox_beta(bt, code, lam0, lam2, M, rho))
                got = 0.5 * rho * (b - bt) ** 2 + float(O.psi(b, code, lam0, lam2, M))
                assert got <= ref + 1e-9 * (1 + abs(ref))
                worst = max(worst, ref - got)
    assert worst < 1e-3   # the grid can never beat the exact prox by more than resolution


# ---------------------------------------------------------------- precompute
def test_woodbury_equals_direct():
    """D via the corrected Woodbury form ([R1]) equals the direct (XᵀX+ρI)⁻¹."""
    rng = np.random.default_rng(6)
    for _ in range(20):
        n, p = int(rng.integers(3, 12)), int(rng.integers(13, 40))
        X = rng.normal(size=(n, p))
        rho = float(10 ** rng.uniform(-1, 1))
        P = O.Problem(X, rng.normal(size=n), 0.1, 0.1, 1.0, rho=rho)
        assert P.G is not None
        Dd = np.linalg.inv(X.T @ X + rho * np.eye(p))
        W = rng.normal(size=(p, 3))
        assert np.allclose(P.apply_D(W), Dd @ W, rtol=1e-9, atol=1e-12)
    # the paper's literal 1/ρ² constant is wrong unless ρ = 1 (E1)
    X = rng.normal(size=(4, 10))
    rho = 0.7
    lit = np.eye(10) / rho - X.T @ np.linalg.inv(X @ X.T + rho * np.eye(4)) @ X / rho ** 2
    assert not np.allclose(lit, np.linalg.inv(X.T @ X + rho * np.eye(10)), atol=1e-3)


# ---------------------------------------------------------------- dual bound and ADMM
def _small(seed, n=30, p=8, corr=0.2):
    inst = synth.make_instance(n, p, 3, corr, 5.0, seed)
    lam2 = 0.05 + 0.5 * (seed % 3)
    lam0 = 0.5 * (1 + seed % 4)
    M = synth.bigM_rule(inst, lam2) * (1.0 if seed % 2 else 3.0)
    return O.Problem(inst.X, inst.y, lam0, lam2, M)


def _rand_code(rng, p):
    code = np.zeros(p, dtype=np.int8)
    k = int(rng.integers(0, p // 2 + 1))
    idx = rng.choice(p, size=k, replace=False)
    code[idx] = rng.integers(1, 3, size=k)
    return code


def test_weak_duality_random_points():
    """Prop. 1: D(r̂) ≤ relaxation optimum ≤ P(β) for any b̂ and feasible β."""
    rng = np.random.default_rng(7)
    for seed in range(12):
        P = _small(seed)
        code = _rand_code(rng, P.p)
        opt, _ = O.relaxation_fista(P, code)
        for _ in range(8):
            bhat = rng.normal(scale=2 * P.M, size=P.p)
            assert O.dual_value(P, bhat, code) <= opt + 1e-7 * (1 + abs(opt))
            beta = rng.uniform(-P.M, P.M, size=P.p)
            beta[code == O.FIX0] = 0
            assert opt <= O.primal_value(P, beta, code) + 1e-9


def test_all_F0_node():
    """All coordinates in F0: β = 0, primal = dual = ½‖y‖²."""
    P = _small(1)
    code = np.full(P.p, O.FIX0, dtype=np.int8)
    assert O.dual_value(P, np.zeros(P.p), code) == pytest.approx(0.5 * P.yy)
    r = O.admm_node(P, code, node_tol=1e-12)
    assert r.primal == pytest.approx(0.5 * P.yy) and r.lb == pytest.approx(0.5 * P.yy)
    assert r.integral and len(r.support) == 0


def test_one_dimensional_closed_form():
    """X=[1], y=[2], λ0=0.1, λ2=0.5, M=10: the relaxation optimum is 1.1 at β=1, by hand from
    eq:relaxnode2 (quadratic zone |β| ≥ √0.2: min ½(2−β)²+0.1+0.5β² → β=1, value 1.1; the ℓ1
    zone's constrained minimum is ½(2−√0.2)²+2√0.05·√0.2 = 1.406 > 1.1)."""
    P = O.Problem(np.array([[1.0]]), np.array([2.0]), 0.1, 0.5, 10.0, rho=1.0)
    r = O.admm_node(P, np.zeros(1, dtype=np.int8), node_tol=1e-13, max_iters=5000)
    assert r.lb == pytest.approx(1.1, abs=1e-9)
    assert r.beta[0] == pytest.approx(1.0, abs=1e-7)
    assert r.integral


@pytest.mark.parametrize("seed", range(12))
def test_admm_matches_independent_relaxation_oracle(seed):
    """Converged ADMM bound = FISTA relaxation optimum, strong duality,
    KKT residual < 1e-8 (north star), LB ≤ optimum (weak duality)."""
    rng = np.random.default_rng(100 + seed)
    P = _small(seed, p=8 + seed % 3)
    code = _rand_code(rng, P.p)
    opt, _ = O.relaxation_fista(P, code)
    r = O.admm_node(P, code, node_tol=1e-11, max_iters=40000)
    assert r.converged
    assert r.lb_best <= opt + 1e-8 * max(1, abs(opt))
    assert r.lb_best == pytest.approx(opt, rel=1e-7)
    assert r.primal == pytest.approx(opt, rel=1e-7)
    assert r.kkt < 1e-8


def test_warm_start_benefit_and_same_fixed_point():
    """a child warm-started from its parent reaches the cold-start optimum with fewer
    iterations in aggregate (S:211, S:577 #8)."""
    warm_it = cold_it = 0
    for seed in range(8):
        P = _small(seed, n=40, p=10)
        root = O.admm_node(P, np.zeros(P.p, dtype=np.int8), node_tol=1e-9)
        if root.branch_j < 0:
            continue
        for val in (O.FIX0, O.FIX1):
            code = np.zeros(P.p, dtype=np.int8)
            code[root.branch_j] = val
            w = O.admm_node(P, code, warm=(root.beta, root.v), node_tol=1e-9)
            c = O.admm_node(P, code, node_tol=1e-9)
            assert w.lb == pytest.approx(c.lb, rel=1e-6)
            warm_it += w.iters
            cold_it += c.iters
    assert warm_it < cold_it


def test_check_cadence_and_running_max():
    """Checks every 10 iterations; LB is the running max of checked duals [R7]."""
    P = _small(3, n=30, p=9)
    r = O.admm_node(P, np.zeros(P.p, dtype=np.int8), node_tol=-1, max_iters=57, check_every=10)
    assert [it for it, _ in r.duals] == [10, 20, 30, 40, 50, 57]
    assert r.lb_best == max(d for _, d in r.duals)
    assert r.iters == 57 and not r.converged


# ---------------------------------------------------------------- upper bound
def _kkt_box_qp(Q, q, M, b, tol):
    g = Q @ b - q
    for i in range(len(b)):
        if abs(b[i]) < M * (1 - 1e-12):
            assert abs(g[i]) <= tol
        else:
            assert g[i] * np.sign(b[i]) <= tol
        assert abs(b[i]) <= M


def test_box_ridge_kkt_and_lsq_linear():
    """eq:upperboundbeta optimum: KKT of the box QP, and equality with an
    independent bounded least-squares solver (scipy lsq_linear on [X_S; √(2λ2)I])."""
    rng = np.random.default_rng(8)
    for t in range(40):
        n, s = int(rng.integers(5, 30)), int(rng.integers(1, 12))
        X = rng.normal(size=(n, s))
        y = rng.normal(size=n) * 3
        lam2 = float(10 ** rng.uniform(-2, 1))
        M = float(10 ** rng.uniform(-1.5, 0.5))
        Q = X.T @ X + 2 * lam2 * np.eye(s)
        b = O.box_ridge(Q, X.T @ y, M)
        _kkt_box_qp(Q, X.T @ y, M, b, 1e-9 * (1 + np.abs(X.T @ y).max()))
        A = np.vstack([X, math.sqrt(2 * lam2) * np.eye(s)])
        ref = lsq_linear(A, np.concatenate([y, np.zeros(s)]), bounds=(-M, M), tol=1e-14,
                         lsmr_tol="auto", method="bvls")
        f = lambda z: 0.5 * np.sum((y - X @ z) ** 2) + lam2 * z @ z
        assert f(b) <= f(ref.x) + 1e-10 * (1 + f(ref.x))
        assert f(b) == pytest.approx(f(ref.x), rel=1e-9, abs=1e-12)


# ---------------------------------------------------------------- brute force and BnB
def _lsq_brute(P):
    """Independent enumeration: scipy bounded LSQ for every support (p ≤ 8)."""
    best = (0.5 * P.yy, ())
    for s in range(1, P.p + 1):
        for S in itertools.combinations(range(P.p), s):
            A = np.vstack([P.X[:, S], math.sqrt(2 * P.lam2) * np.eye(s)])
            r = lsq_linear(A, np.concatenate([P.y, np.zeros(s)]), bounds=(-P.M, P.M),
                           method="bvls", tol=1e-14)
            val = 0.5 * float(np.sum((A @ r.x - np.concatenate([P.y, np.zeros(s)])) ** 2)) + P.lam0 * s
            if val < best[0] - 1e-12:
                best = (val, S)
    return best


@pytest.mark.parametrize("seed", range(6))
def test_brute_force_vs_independent_enumeration(seed):
    P = _small(seed, n=20, p=7)
    obj, S, _ = O.brute_force(P)
    ref, Sref = _lsq_brute(P)
    assert obj == pytest.approx(ref, rel=1e-9)
    assert tuple(S.tolist()) == tuple(Sref)


def test_brute_force_monotone_in_lambda0():
    """Larger λ0 never yields a larger optimal support."""
    inst = synth.make_instance(30, 10, 3, 0.3, 5.0, 11)
    sizes = []
    for lam0 in (0.01, 0.1, 1.0, 5.0, 20.0, 1e3):
        P = O.Problem(inst.X, inst.y, lam0, 0.1, 3.0)
        sizes.append(len(O.brute_force(P)[1]))
    assert sizes == sorted(sizes, reverse=True) and sizes[-1] == 0


@pytest.mark.parametrize("seed", range(10))
def test_bnb_equals_brute_force(seed):
    """SPEC acceptance #1: BnB at gap 1e-9 returns the enumeration optimum and support;
    certificate independent of the batch size."""
    rng = np.random.default_rng(seed)
    n, p = int(rng.choice([15, 30])), int(rng.choice([6, 8, 10]))
    inst = synth.make_instance(n, p, 3, float(rng.choice([0.0, 0.2, 0.5])), 5.0, seed)
    P = O.Problem(inst.X, inst.y, float(rng.uniform(0.01, 1)) * n / 10, float(rng.uniform(0.01, 1)),
                  float(rng.uniform(1, 10)))
    obj, S, _ = O.brute_force(P)
    for B in (1, 4):
        res = O.bnb_solve(P, B=B, gap_tol=1e-9, node_tol=1e-10, record=True)
        assert res["obj"] == pytest.approx(obj, rel=1e-9)
        assert tuple(res["support"].tolist()) == tuple(S.tolist())
        assert res["lb"] <= obj * (1 + 1e-9)
        # pruning soundness: every node whose fixings are consistent with the
        # optimal support has LB ≤ optimum
        Sset = set(S.tolist())
        for t in res["trace"]:
            if set(t["F1"]) <= Sset and not (set(t["F0"]) & Sset):
                assert t["lb"] <= obj * (1 + 1e-8) + 1e-12


def test_C1_bnb_equals_brute_force():
    """C1 of BASELINE.json (n=50, p=20, λ0=0.1, λ2=0.01): BnB = brute force over 2^20 supports."""
    inst = synth.config_instance("C1", seed=0)
    P = O.Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M)
    obj, S, _ = O.brute_force(P)
    res = O.bnb_solve(P, B=8, gap_tol=1e-9, node_tol=1e-10)
    assert res["obj"] == pytest.approx(obj, rel=1e-9)
    assert tuple(res["support"].tolist()) == tuple(S.tolist())


def test_tree_invariants():
    """Child LB ≥ parent LB; UB ≥ every LB of a node containing the optimum."""
    P = _small(5, n=40, p=12)
    res = O.bnb_solve(P, B=2, gap_tol=1e-9, node_tol=1e-10, record=True)
    lbs = {t["id"]: t["lb"] for t in res["trace"]}
    # ids: children of node u get consecutive ids; reconstruct parents by fixings
    for t in res["trace"]:
        for u in res["trace"]:
            if u["depth"] == t["depth"] + 1 and set(t["F0"]) <= set(u["F0"]) and set(t["F1"]) <= set(u["F1"]) \
                    and len(u["F0"]) + len(u["F1"]) == len(t["F0"]) + len(t["F1"]) + 1:
                assert u["lb"] >= lbs[t["id"]] - 1e-12
    assert res["lb"] <= res["obj"] + 1e-9


# ---------------------------------------------------------------- generator
def test_generator_recipe():
    """SNR is exact with the empirical variance; β† equispaced ones; determinism."""
    a = synth.make_instance(200, 50, 5, 0.2, 3.0, 7)
    b = synth.make_instance(200, 50, 5, 0.2, 3.0, 7)
    assert np.array_equal(a.X, b.X) and np.array_equal(a.y, b.y)
    assert a.X.flags.f_contiguous
    assert list(a.support_true) == [0, 10, 20, 30, 40]
    mu = a.X @ a.beta_true
    assert np.var(mu) / a.sigma ** 2 == pytest.approx(3.0, rel=1e-12)
    big = synth.make_instance(20000, 6, 2, 0.2, 5.0, 1)
    C = np.cov(big.X, rowvar=False)
    off = C[~np.eye(6, dtype=bool)]
    assert abs(off.mean() - 0.2) < 0.03 and abs(np.diag(C).mean() - 1.0) < 0.03


# ---------------------------------------------------------------- matching pursuit (Algorithm 3)
def _F(P, beta):
    """The objective Algorithm 3 descends, evaluated from its definition:
    ½‖y − Xβ‖² + λ2‖β‖² + λ0·|supp β|."""
    r = P.y - P.X @ beta
    return 0.5 * float(r @ r) + P.lam2 * float(beta @ beta) + P.lam0 * int(np.count_nonzero(beta))


def _mp_instance(seed, n=30, p=12):
    inst = synth.make_instance(n, p, 3, 0.3, 4.0, seed)
    return O.Problem(inst.X, inst.y, 2.0, 0.05, 1.5)


@pytest.mark.parametrize("seed", [0, 1])
def test_mp_forward_delta_is_the_objective_change(seed):
    """Δ_j of the forward step = F(β + β_j e_j) − F(β) for j ∉ S, at a random feasible β,
    and β_j is the 1-D argmin over [−M, M] of ½‖r − X_j t‖² + λ2 t² (scipy)."""
    P = _mp_instance(seed)
    rng = np.random.default_rng(seed)
    S = rng.choice(P.p, 4, replace=False)
    beta = np.zeros(P.p)
    beta[S] = rng.uniform(-P.M, P.M, 4)
    r = P.y - P.X @ beta
    inS = np.zeros(P.p, dtype=bool)
    inS[S] = True
    delta, b = O.mp_forward_scores(P, r, inS)
    for j in np.nonzero(~inS)[0]:
        bj = beta.copy()
        bj[j] = b[j]
        assert delta[j] == pytest.approx(_F(P, bj) - _F(P, beta), rel=1e-10, abs=1e-9)
        ref = minimize_scalar(lambda t: 0.5 * np.sum((r - P.X[:, j] * t) ** 2) + P.lam2 * t * t,
                              bounds=(-P.M, P.M), method="bounded", options={"xatol": 1e-12})
        assert b[j] == pytest.approx(ref.x, abs=1e-7)
    assert np.all(np.isinf(delta[S]))


@pytest.mark.parametrize("seed", [0, 1])
def test_mp_backward_delta_is_the_objective_change(seed):
    """Δ_j of the backward step = F(β − β_j e_j) − F(β) for j ∈ S."""
    P = _mp_instance(seed)
    rng = np.random.default_rng(10 + seed)
    S = np.sort(rng.choice(P.p, 5, replace=False))
    beta = np.zeros(P.p)
    beta[S] = rng.uniform(-P.M, P.M, 5)
    r = P.y - P.X @ beta
    dS = O.mp_backward_scores(P, r, beta, S)
    for i, j in enumerate(S):
        bj = beta.copy()
        bj[j] = 0.0
        assert dS[i] == pytest.approx(_F(P, bj) - _F(P, beta), rel=1e-10, abs=1e-9)


def test_mp_orthogonal_design_is_exact():
    """With orthogonal columns the ℓ0-ℓ2 box problem separates, so Algorithm 3 (forward steps only;
    every backward Δ is then −(forward Δ) > 0) reaches the brute-force optimum exactly."""
    rng = np.random.default_rng(7)
    for trial in range(4):
        n, p = 20, 8
        Qm, _ = np.linalg.qr(rng.standard_normal((n, p)))
        X = Qm * rng.uniform(0.5, 3.0, p)
        y = X @ (rng.standard_normal(p) * rng.integers(0, 2, p)) + 0.3 * rng.standard_normal(n)
        P = O.Problem(X, y, 0.2 + 0.2 * trial, 0.1, 1.2)
        mp = O.matching_pursuit(P)
        bf_obj, bf_S, _ = O.brute_force(P)
        assert mp.obj == pytest.approx(bf_obj, rel=1e-12)
        assert list(mp.support) == list(bf_S)
        assert all(kind == "+" for kind, _, _ in mp.steps)


@pytest.mark.parametrize("seed", range(4))
def test_mp_descent_fixed_point_and_valid_upper_bound(seed):
    """Every accepted step lowers F by exactly its Δ < 0; the output is a fixed point (no forward
    or backward Δ < 0), feasible (|β| ≤ M), F(β) = the returned objective = ub_objective on its
    support, and never below the brute-force optimum."""
    P = _mp_instance(seed)
    mp = O.matching_pursuit(P)
    beta = np.zeros(P.p)
    inS = np.zeros(P.p, dtype=bool)
    f = _F(P, beta)
    # replay the step log from the definition
    for kind, j, d in mp.steps:
        assert d < 0
        r = P.y - P.X @ beta
        if kind == "+":
            delta, b = O.mp_forward_scores(P, r, inS)
            beta[j], inS[j] = b[j], True
        else:
            beta[j], inS[j] = 0.0, False
        f_new = _F(P, beta)
        assert f_new - f == pytest.approx(d, rel=1e-9, abs=1e-9)
        f = f_new
    assert np.allclose(beta, mp.beta, rtol=1e-12, atol=1e-14)   # replay recomputes r from scratch
    assert mp.obj == pytest.approx(_F(P, mp.beta), rel=1e-12)
    assert mp.obj == pytest.approx(O.ub_objective(P, mp.support, mp.beta[mp.support]), rel=1e-12)
    assert np.all(np.abs(mp.beta) <= P.M)
    r = P.y - P.X @ mp.beta
    delta, _ = O.mp_forward_scores(P, r, np.isin(np.arange(P.p), mp.support))
    assert np.min(delta) >= 0
    if len(mp.support):
        assert np.min(O.mp_backward_scores(P, r, mp.beta, mp.support)) >= 0
    assert mp.obj >= O.brute_force(P)[0] - 1e-9


@pytest.mark.parametrize("seed", range(3))
def test_early_prune_keeps_the_certificate(seed):
    """Early prune (R16) changes only how long pruned nodes run: the BnB
    still certifies the brute-force optimum, solves no more node iterations, and every node that
    stopped early is pruned (its LB ≥ the incumbent)."""
    inst = synth.make_instance(40, 14, 3, 0.3, 4.0, 20 + seed)
    lam2 = max(synth.tune_lambda2(inst), 0.05)
    P = O.Problem(inst.X, inst.y, synth.lambda0_rule(inst, lam2), lam2, synth.bigM_rule(inst, lam2))
    bf_obj, bf_S, _ = O.brute_force(P)
    a = O.bnb_solve(P, B=4, gap_tol=1e-9, node_tol=1e-9, record=True)
    b = O.bnb_solve(P, B=4, gap_tol=1e-9, node_tol=1e-9, record=True, early_prune=True)
    for r in (a, b):
        assert r["obj"] == pytest.approx(bf_obj, rel=1e-9)
        assert list(r["support"]) == list(bf_S)
    early = [t for t in b["trace"] if t["early"]]
    assert all(t["pruned"] for t in early)          # an early-stopped node is always pruned
    assert not any(t["early"] for t in a["trace"])


@pytest.mark.parametrize("seed", range(3))
def test_mp_incumbent_keeps_the_certificate(seed):
    """init_mp: the BnB started from Algorithm 3's incumbent (refit by the exact box ridge on
    its support) certifies the brute-force optimum; its initial UB is the better of ½‖y‖², the MP point
    and the refit, so the first round's threshold is never above the plain BnB's."""
    inst = synth.make_instance(40, 12, 3, 0.3, 4.0, 30 + seed)
    lam2 = max(synth.tune_lambda2(inst), 0.05)
    P = O.Problem(inst.X, inst.y, synth.lambda0_rule(inst, lam2), lam2, synth.bigM_rule(inst, lam2))
    bf_obj, bf_S, _ = O.brute_force(P)
    r = O.bnb_solve(P, B=4, gap_tol=1e-9, node_tol=1e-9, record=True, init_mp=True)
    assert r["obj"] == pytest.approx(bf_obj, rel=1e-9)
    assert list(r["support"]) == list(bf_S)
    mp = O.matching_pursuit(P)
    ub0 = min(0.5 * P.yy, mp.obj, O.upper_bound(P, mp.support)[0] if len(mp.support) else np.inf)
    assert r["trace"][0]["ub"] >= bf_obj * (1 - 1e-12)
    assert ub0 >= bf_obj * (1 - 1e-12)                 # every incumbent is a feasible objective
    plain = O.bnb_solve(P, B=4, gap_tol=1e-9, node_tol=1e-9)
    assert r["nodes"] <= plain["nodes"]


def test_node_map_does_not_change_the_tree():
    """bnb_solve's node_map only decides where the independent nodes of a round run: a process pool
    (the all-cores oracle baseline) gives the same tree, node for node, as the serial map."""
    import multiprocessing as mp
    inst = synth.make_instance(30, 10, 3, 0.2, 4.0, 7)
    P = O.Problem(inst.X, inst.y, 1.0, 0.2, 3.0)
    serial = O.bnb_solve(P, B=4, gap_tol=1e-9, node_tol=1e-9, record=True)
    with mp.get_context("fork").Pool(2) as pool:
        par = O.bnb_solve(P, B=4, gap_tol=1e-9, node_tol=1e-9, record=True, node_map=pool.map)
    assert [(t["id"], t["lb"], t["iters"], t["branch_j"]) for t in serial["trace"]] == \
        [(t["id"], t["lb"], t["iters"], t["branch_j"]) for t in par["trace"]]
    assert serial["obj"] == par["obj"]

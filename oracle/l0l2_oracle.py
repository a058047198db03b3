"""Plain, slow, obviously-correct CPU oracle (numpy, float64) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline, --impl reference)
may import this module.  It shares no code with paper_2602_04551_b200/.

Every function cites the PAPER.md passage ("P:<line>") it restates; SPEC.md lines
are "S:<line>".  Readings where the paper is silent, garbled or inconsistent are
the ones listed in DESIGN.md §3 ("Readings") and are marked [Rn] below.

Formulation choice (deliberately different from the GPU's Z-form, so the two
check each other): the b-update applies D = (XᵀX+ρI)⁻¹ directly when n ≥ p and
the Woodbury G-form D w = (w − Xᵀ G X w)/ρ, G = (XXᵀ+ρI)⁻¹, when p > n
(P:369-379 with the 1/ρ² typo corrected, [R1]).  The dual bound evaluates
r̂ = y − X b̂ and Xᵀr̂ explicitly, not through identities.

Parity status: every function below is pinned by tests/test_oracle_pins.py
except the ones whose docstring says "parity unpinned".
"""
from __future__ import annotations

import itertools
import math
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla

FREE, FIX0, FIX1 = 0, 1, 2   # per-coordinate fixation code: free, i∈F0, i∈F1

__all__ = [
    "FREE", "FIX0", "FIX1", "T", "psi", "h", "nu", "prox_beta", "recover_z",
    "Problem", "make_code", "primal_value", "dual_value", "admm_node", "NodeResult",
    "box_ridge", "upper_bound", "brute_force", "relaxation_fista", "bnb_solve",
    "ub_objective", "default_rho", "MPResult", "mp_forward_scores", "mp_backward_scores",
    "matching_pursuit", "finalize_node",
]


# ----------------------------------------------------------------------------------------------
# Scalar operators (vectorised over numpy arrays)
# ----------------------------------------------------------------------------------------------

def T(t, a, m):
    """Box-constrained soft-thresholding, eq:Tdef.

    T(t; a, m) = 0 if |t| ≤ a;  (|t|−a)·sign(t) if a < |t| ≤ a+m;  m·sign(t) otherwise.
    """
    t = np.asarray(t, dtype=np.float64)
    at = np.abs(t)
    out = np.where(at <= a, 0.0, np.where(at <= a + m, (at - a) * np.sign(t), m * np.sign(t)))
    return out


def psi(beta, code, lam0, lam2, M):
    """ψ_i(β_i; λ0, λ2, M), eq:psi; derivation P:1077-1104.

    F0: 0 if β_i = 0 else +∞.  F1 or √(λ0/λ2) ≤ |β_i| ≤ M: λ0 + λ2β_i².
    |β_i| ≤ √(λ0/λ2) ≤ M: 2√(λ0λ2)|β_i|.  √(λ0/λ2) > M: (λ0/M + λ2M)|β_i|.
    Outside the box |β_i| > M: +∞ (the indicator of eq:relaxnode2).
    """
    beta = np.asarray(beta, dtype=np.float64)
    code = np.broadcast_to(np.asarray(code), beta.shape)
    ab = np.abs(beta)
    sr = math.sqrt(lam0 / lam2)
    if sr <= M:
        free = np.where(ab >= sr, lam0 + lam2 * beta * beta, 2.0 * math.sqrt(lam0 * lam2) * ab)
    else:
        free = (lam0 / M + lam2 * M) * ab
    out = np.where(code == FIX1, lam0 + lam2 * beta * beta, free)
    out = np.where(code == FIX0, np.where(beta == 0.0, 0.0, np.inf), out)
    out = np.where(ab > M, np.inf, out)
    return out


def h(x, lam0, lam2, M):
    """h(x), eq:hdef: x²/(4λ2) − λ0 if x ≤ 2Mλ2, else Mx − λ0 − λ2M²."""
    x = np.asarray(x, dtype=np.float64)
    return np.where(x <= 2.0 * M * lam2, x * x / (4.0 * lam2) - lam0, M * x - lam0 - lam2 * M * M)


def nu(x, code, lam0, lam2, M):
    """ν_i(x), appendix form eq:nudef2 [R2: main-text λ2² typo at P:533].

    F0: 0.  F1: h(x).  free with √(λ0/λ2) ≤ M: [h(x)]₊.  free with √(λ0/λ2) > M:
    [Mx − λ0 − λ2M²]₊.
    """
    x = np.asarray(x, dtype=np.float64)
    code = np.broadcast_to(np.asarray(code), x.shape)
    hx = h(x, lam0, lam2, M)
    if math.sqrt(lam0 / lam2) <= M:
        free = np.maximum(hx, 0.0)
    else:
        free = np.maximum(M * x - lam0 - lam2 * M * M, 0.0)
    out = np.where(code == FIX1, hx, free)
    return np.where(code == FIX0, 0.0, out)


def prox_beta(bt, code, lam0, lam2, M, rho):
    """β-update, eq:minbetalower, derivation P:1108-1128  [R3].

    argmin_β ρ/2 (β − β̃)² + ψ(β) + ι{|β| ≤ M}:
      F0                                              → 0
      F1, or (free, √(λ0/λ2) ≤ M, |β̃| ≥ 2√(λ0λ2)/ρ + √(λ0/λ2)) → T(ρβ̃/(ρ+2λ2); 0, M)
      free, √(λ0/λ2) ≤ M, |β̃| below that threshold        → T(β̃; 2√(λ0λ2)/ρ, M)
      free, √(λ0/λ2) > M                                → T(β̃; λ0/(Mρ) + λ2M/ρ, M)
    """
    bt = np.asarray(bt, dtype=np.float64)
    code = np.broadcast_to(np.asarray(code), bt.shape)
    sr = math.sqrt(lam0 / lam2)
    quad = T(rho / (rho + 2.0 * lam2) * bt, 0.0, M)
    if sr <= M:
        a = 2.0 * math.sqrt(lam0 * lam2) / rho
        free = np.where(np.abs(bt) >= a + sr, quad, T(bt, a, M))
    else:
        a = lam0 / (M * rho) + lam2 * M / rho
        free = T(bt, a, M)
    out = np.where(code == FIX1, quad, free)
    return np.where(code == FIX0, 0.0, out)


def recover_z(beta, code, lam0, lam2, M):
    """Optimal z for fixed β in eq:relaxnode.

    F0 → 0, F1 → 1, free → min(1, max(|β|/M, √(λ2/λ0)|β|)) (cases 3(a)-(c)).
    """
    beta = np.asarray(beta, dtype=np.float64)
    code = np.broadcast_to(np.asarray(code), beta.shape)
    ab = np.abs(beta)
    zf = np.minimum(1.0, np.maximum(ab / M, math.sqrt(lam2 / lam0) * ab)) if lam0 > 0 else np.where(ab > 0, 1.0, 0.0)
    return np.where(code == FIX0, 0.0, np.where(code == FIX1, 1.0, zf))


# ----------------------------------------------------------------------------------------------
# Problem data and the tree-wide precompute
# ----------------------------------------------------------------------------------------------

def default_rho(X):
    """ADMM penalty default = mean_j ‖X_j‖² ([R5]: the paper never states ρ)."""
    return float(np.mean(np.einsum("ij,ij->j", X, X)))


class Problem:
    """(X, y, λ0, λ2, M) plus the ADMM precompute of P:369-379 (done once per tree)."""

    def __init__(self, X, y, lam0, lam2, M, rho=None):
        self.X = np.asarray(X, dtype=np.float64)
        self.y = np.asarray(y, dtype=np.float64)
        self.n, self.p = self.X.shape
        self.lam0, self.lam2, self.M = float(lam0), float(lam2), float(M)
        if self.lam2 <= 0 or self.lam0 < 0 or self.M <= 0:
            raise ValueError("need λ2 > 0, λ0 ≥ 0, M > 0 (S:89)")
        self.rho = float(rho) if rho else default_rho(self.X)
        # c = Xᵀy
        self.c = self.X.T @ self.y
        self.yy = float(self.y @ self.y)
        if self.n >= self.p:
            # D = (XᵀX + ρI_p)⁻¹  (first case)
            self.D = np.linalg.inv(self.X.T @ self.X + self.rho * np.eye(self.p))
            self.G = None
        else:
            # G = (XXᵀ + ρI_n)⁻¹ held as a Cholesky factor ("two triangular systems")
            self.D = None
            self.G = sla.cho_factor(self.X @ self.X.T + self.rho * np.eye(self.n), lower=True)

    def apply_D(self, w):
        """b = D w with D = (XᵀX+ρI)⁻¹, eq:b_update.

        p > n: D = (1/ρ)(I_p − Xᵀ(XXᵀ+ρI_n)⁻¹X)  — the Woodbury form of P:375 with the
        paper's 1/ρ² corrected to 1/ρ [R1].
        """
        if self.D is not None:
            return self.D @ w
        return (w - self.X.T @ sla.cho_solve(self.G, self.X @ w)) / self.rho


def make_code(p, F0=(), F1=()):
    code = np.zeros(p, dtype=np.int8)
    F0 = np.asarray(F0, dtype=np.int64)
    F1 = np.asarray(F1, dtype=np.int64)
    if np.intersect1d(F0, F1).size:
        raise ValueError("F0 ∩ F1 ≠ ∅ (S:28)")
    code[F0] = FIX0
    code[F1] = FIX1
    return code


def primal_value(P: Problem, beta, code):
    """Objective of eq:relaxnode2: ½‖y − Xβ‖² + Σ ψ_i(β_i)."""
    r = P.y - P.X @ beta
    return 0.5 * float(r @ r) + float(np.sum(psi(beta, code, P.lam0, P.lam2, P.M)))


def dual_value(P: Problem, b, code):
    """Dual bound of Proposition 1 (eq:dual P:525-527) at r̂ = y − X b̂.

    D(r̂) = −½‖r̂‖² + yᵀr̂ − Σ_i ν_i(|X_iᵀ r̂|), evaluated explicitly.  Valid for any r̂.
    """
    r = P.y - P.X @ b
    xr = P.X.T @ r
    return -0.5 * float(r @ r) + float(P.y @ r) - float(np.sum(nu(np.abs(xr), code, P.lam0, P.lam2, P.M)))


# ----------------------------------------------------------------------------------------------
# Node relaxation: scalar (one node at a time) ADMM
# ----------------------------------------------------------------------------------------------

@dataclass
class NodeResult:
    lb: float               # max(best checked dual, parent LB)  [R7]
    lb_best: float          # best checked dual
    primal: float           # P(β) at the last check
    beta: np.ndarray
    v: np.ndarray
    b: np.ndarray
    iters: int
    converged: bool
    z: np.ndarray
    integral: bool
    support: np.ndarray
    branch_j: int
    kkt: float
    duals: list = field(default_factory=list)   # (iteration, dual) of every check
    pruned: bool = False    # stopped early: LB_best ≥ prune_ub at a check (early prune, R16)


def admm_node(P: Problem, code, warm=None, parent_lb=-math.inf, node_tol=1e-4,
              check_every=10, max_iters=10000, int_tol=1e-4, prune_ub=math.inf) -> NodeResult:
    """ADMM on eq:ADMM1 for one node, warm start P:543.

    Start ([R6]): a cold node (the root, or any node without a parent state) starts
    from (β, v) = (0, 0) with no refresh ("For the root node, we initialize the ADMM variables
    to zero").  A warm node takes the parent's (β, v), sets β_i ← 0 on F0, then refreshes
    b = D(c + ρβ − v) (eq:b_update) and v ← v + ρ(b − β) (eq:v_i-update) before iterating.
    Iteration t: w = c + ρβ − v; b = D w (eq:b_update); β̃ = b + v/ρ;
    β = prox(β̃) (eq:minbetalower); v ← v + ρ(b − β) (eq:v_i-update).
    Every `check_every` iterations (and at max_iters): dual at r̂ = y − Xb,
    LB_best = running max [R7]; primal P(β); stop when
    (P − LB_best)/max(1, |P|) ≤ node_tol ([R8]).
    Finalize: LB = max(LB_best, parent LB); ẑ from β;
    integral if every free ẑ is within int_tol of {0,1}; support = F1 ∪ {free: ẑ ≥ ½};
    branch j = argmax_free min(ẑ, 1−ẑ), ties → larger |β_j|, then lower index [R10].
    Early prune [R16, SURVEY §8(f) rank 2]: a check that does not converge but finds
    LB_best ≥ prune_ub stops the node (it will be pruned; any dual is a valid bound).
    """
    code = np.asarray(code, dtype=np.int8)
    p, rho = P.p, P.rho
    if warm is None:
        beta = np.zeros(p)      # root / cold node: ADMM variables initialised to zero
        v = np.zeros(p)
    else:
        beta = np.array(warm[0], dtype=np.float64)
        v = np.array(warm[1], dtype=np.float64)
        beta[code == FIX0] = 0.0                 # respect the new F0 fixings
        b = P.apply_D(P.c + rho * beta - v)      # then update b (eq:b_update) ...
        v = v + rho * (b - beta)                 # ... and v (eq:v_i-update)
    lb_best = -math.inf
    primal = math.inf
    duals = []
    it = 0
    converged = False
    pruned = False
    beta_prev = beta.copy()
    while it < max_iters:
        it += 1
        w = P.c + rho * beta - v
        b = P.apply_D(w)
        bt = b + v / rho
        beta_prev = beta
        beta = prox_beta(bt, code, P.lam0, P.lam2, P.M, rho)
        v = v + rho * (b - beta)
        if it % check_every == 0 or it == max_iters:
            d = dual_value(P, b, code)
            duals.append((it, d))
            lb_best = max(lb_best, d)
            primal = primal_value(P, beta, code)
            if (primal - lb_best) / max(1.0, abs(primal)) <= node_tol:
                converged = True
                break
            if lb_best >= prune_ub:
                pruned = True
                break
    kkt = max(float(np.max(np.abs(b - beta), initial=0.0)),
              rho * float(np.max(np.abs(beta - beta_prev), initial=0.0))) / (1.0 + float(np.max(np.abs(P.c), initial=0.0)))
    z, integral, support, branch_j = finalize_node(beta, code, P.lam0, P.lam2, P.M, int_tol)
    return NodeResult(lb=max(lb_best, parent_lb), lb_best=lb_best, primal=primal, beta=beta, v=v, b=b,
                      iters=it, converged=converged, z=z, integral=integral, support=support,
                      branch_j=branch_j, kkt=kkt, duals=duals, pruned=pruned)


def finalize_node(beta, code, lam0, lam2, M, int_tol=1e-4):
    """Node finalize → (ẑ, integral, support, branch j).

    ẑ = recover_z(β); integral iff every free ẑ_i is within int_tol of {0, 1}
    (S:224); support = F1 ∪ {free i: ẑ_i ≥ ½} (rounding, tie at ½ included [R13]);
    branch j ("Select j ∈ [p] minus (F0 ∪ F1)") = the free coordinate with the largest
    min(ẑ_j, 1 − ẑ_j), ties → larger |β_j|, then lower j [R10, S:381]; −1 when integral.
    """
    beta = np.asarray(beta, dtype=np.float64)
    code = np.asarray(code, dtype=np.int8)
    z = recover_z(beta, code, lam0, lam2, M)
    free = code == FREE
    frac = np.minimum(z, 1.0 - z)
    integral = bool(np.all(frac[free] <= int_tol))
    support = np.nonzero((code == FIX1) | (free & (z >= 0.5)))[0].astype(np.int64)
    branch_j = -1
    if not integral:
        best = None
        for j in np.nonzero(free)[0]:          # plain scan in index order: strict improvement only
            key = (float(frac[j]), float(abs(beta[j])))
            if best is None or key > best[0]:
                best = (key, int(j))
        branch_j = best[1]
    return z, integral, support, branch_j


# ----------------------------------------------------------------------------------------------
# Upper bound: exact box-constrained ridge on a support (eq:upperboundbeta)
# ----------------------------------------------------------------------------------------------

def box_ridge(Q, q, M, max_sweeps=200000):
    """Exact minimiser of ½βᵀQβ − qᵀβ s.t. |β_i| ≤ M  (Q SPD; eq:upperboundbeta).

    Unconstrained solve first; if outside the box, cyclic coordinate descent
    β_i ← clip((q_i − Σ_{k≠i} Q_ik β_k)/Q_ii, ±M) to a fixed point, then an exact
    re-solve on the identified free set (KKT-checked).  North star: "closed-form ridge
    on the support for upper bounds".
    """
    s = len(q)
    if s == 0:
        return np.zeros(0)
    beta = np.linalg.solve(Q, q)
    if np.all(np.abs(beta) <= M):
        return beta
    beta = np.clip(beta, -M, M)
    for _ in range(max_sweeps):
        delta = 0.0
        for i in range(s):
            g = q[i] - Q[i] @ beta + Q[i, i] * beta[i]
            nb = min(max(g / Q[i, i], -M), M)
            delta = max(delta, abs(nb - beta[i]))
            beta[i] = nb
        if delta <= 1e-15 * (1.0 + M):
            break
    # exact polish on the active set A = {|β_i| = M}
    A = np.abs(beta) >= M * (1 - 1e-12)
    F = ~A
    b2 = beta.copy()
    b2[A] = np.sign(beta[A]) * M
    if F.any():
        b2[F] = np.linalg.solve(Q[np.ix_(F, F)], q[F] - Q[np.ix_(F, A)] @ b2[A])
    grad = Q @ b2 - q
    ok = np.all(np.abs(b2[F]) <= M) and np.all(grad[A] * np.sign(b2[A]) <= 1e-9 * (1 + np.abs(q).max()))
    return b2 if ok else beta


def ub_objective(P: Problem, S, beta_S):
    """Objective of eq:perspective at z = 1_S: ½‖y − X_Sβ_S‖² + λ2‖β_S‖² + λ0|S|."""
    S = np.asarray(S, dtype=np.int64)
    r = P.y - P.X[:, S] @ beta_S
    return 0.5 * float(r @ r) + P.lam2 * float(beta_S @ beta_S) + P.lam0 * len(S)


def upper_bound(P: Problem, S):
    """UB on a support: exact box ridge (eq:upperboundbeta) + λ0|S|.  Returns (obj, β_S)."""
    S = np.asarray(S, dtype=np.int64)
    if len(S) == 0:
        return 0.5 * P.yy, np.zeros(0)
    XS = P.X[:, S]
    Q = XS.T @ XS + 2.0 * P.lam2 * np.eye(len(S))
    bS = box_ridge(Q, XS.T @ P.y, P.M)
    return ub_objective(P, S, bS), bS


# ----------------------------------------------------------------------------------------------
# Brute force (plain definition of the final result, §8(c1))
# ----------------------------------------------------------------------------------------------

def brute_force(P: Problem, max_p=20):
    """min over all 2^p supports S of λ0|S| + min_{|β|≤M} ½‖y−X_Sβ‖² + λ2‖β‖².

    Ties → smaller |S|, then lexicographic.  Unconstrained ridge values (a lower
    bound of the box value) screen supports; box-violating candidates below the running
    best are re-solved exactly with box_ridge.  The winner's objective is recomputed from
    the definition.  Returns (obj, S, β_S).
    """
    p = P.p
    if p > max_p:
        raise ValueError("brute force limited to p ≤ %d" % max_p)
    G = P.X.T @ P.X
    q = P.c
    best = (0.5 * P.yy, np.zeros(0, dtype=np.int64), np.zeros(0))
    best_obj = best[0]
    for s in range(1, p + 1):
        if P.lam0 * s >= best_obj:
            break   # every support of size ≥ s costs ≥ λ0·s ≥ best (objective terms are ≥ 0)
        combos = np.array(list(itertools.combinations(range(p), s)), dtype=np.int64)
        for lo in range(0, len(combos), 20000):
            C = combos[lo:lo + 20000]
            Q = G[C[:, :, None], C[:, None, :]] + 2.0 * P.lam2 * np.eye(s)[None]
            qs = q[C]
            bet = np.linalg.solve(Q, qs[:, :, None])[:, :, 0]
            f = 0.5 * P.yy - 0.5 * np.einsum("ij,ij->i", qs, bet) + P.lam0 * s
            inbox = np.all(np.abs(bet) <= P.M, axis=1)
            for idx in np.nonzero(f < best_obj)[0]:
                if inbox[idx]:
                    val, bS = f[idx], bet[idx]
                else:
                    bS = box_ridge(Q[idx], qs[idx], P.M)
                    val = 0.5 * P.yy - qs[idx] @ bS + 0.5 * bS @ Q[idx] @ bS + P.lam0 * s
                if val < best_obj:
                    best_obj = val
                    best = (val, C[idx].copy(), bS.copy())
    S, bS = best[1], best[2]
    return (ub_objective(P, S, bS) if len(S) else 0.5 * P.yy), S, bS


def relaxation_fista(P: Problem, code, tol=1e-12, max_iters=200000):
    """Independent relaxation oracle: FISTA with restart on eq:relaxnode2.

    minimise F(β) = ½‖y−Xβ‖² + Σψ_i(β_i) over ‖β‖∞ ≤ M with step 1/L, L = ‖X‖₂²; the
    proximal map of ψ/L is eq:minbetalower with ρ = L.  The smooth part is evaluated
    through the Gram matrix (½‖y‖² − cᵀβ + ½βᵀXᵀXβ).  Returns (F at the last iterate
    evaluated from the definition, β).  (SPEC S:507-515.)
    """
    code = np.asarray(code, dtype=np.int8)
    G = P.X.T @ P.X
    L = float(np.linalg.eigvalsh(G)[-1]) * (1 + 1e-12)
    fval = lambda b: 0.5 * P.yy - P.c @ b + 0.5 * b @ G @ b + float(np.sum(psi(b, code, P.lam0, P.lam2, P.M)))
    x = np.zeros(P.p)
    yk = x.copy()
    t = 1.0
    fprev = fval(x)
    for _ in range(max_iters):
        g = G @ yk - P.c
        xn = prox_beta(yk - g / L, code, P.lam0, P.lam2, P.M, L)
        f = fval(xn)
        if f > fprev and t > 1.0:     # adaptive restart (a plain prox-gradient step is kept)
            t = 1.0
            yk = x.copy()
            continue
        tn = 0.5 * (1 + math.sqrt(1 + 4 * t * t))
        yk = xn + (t - 1) / tn * (xn - x)
        done = np.max(np.abs(xn - x), initial=0.0) <= tol * (1 + np.max(np.abs(xn), initial=0.0))
        x, t, fprev = xn, tn, f
        if done:
            break
    return primal_value(P, x, code), x


# ----------------------------------------------------------------------------------------------
# Branch-and-bound: batched reading of Algorithm 1
# ----------------------------------------------------------------------------------------------

def _solve_node(args):
    """One node of a BnB round: its relaxation (admm_node) and the UB on its rounded support."""
    P, code, warm, plb, node_tol, check_every, max_iters, int_tol, prune_ub = args
    res = admm_node(P, code, warm=warm, parent_lb=plb, node_tol=node_tol, check_every=check_every,
                    max_iters=max_iters, int_tol=int_tol, prune_ub=prune_ub)
    obj, bS = upper_bound(P, res.support)
    return res, obj, bS


def bnb_solve(P: Problem, B=1, gap_tol=1e-2, node_tol=1e-4, check_every=10, max_iters=10000,
              int_tol=1e-4, prune_tol=1e-12, node_limit=None, time_limit=None, record=False,
              early_prune=False, init_mp=False, node_map=map):
    """Best-first synchronous-round BnB (Algorithm 1) [R9, R11].

    UB starts at ½‖y‖² (β = 0 is feasible).  Each round: drop open nodes with
    LB ≥ UB(1−prune_tol); stop if none remain or (UB − LB)/UB ≤ gap_tol;
    pop min(B, |N|) nodes by (LB, id); solve each node's relaxation (warm
    started from its parent) and the UB on its rounded support; apply all
    of the round's UB improvements (lowest id wins ties); then in id order prune by
    LB_u ≥ UB(1−prune_tol) or integral ẑ, else branch on j into
    (F0∪{j}, F1) then (F0, F1∪{j}) with LB_u and the parent's (β, v).
    early_prune [R16]: each node's ADMM stops at the first check whose LB_best ≥ UB(1−prune_tol)
    with UB the incumbent at the start of the round (the node is then pruned by the rule above,
    since the round can only lower UB).
    node_map: how the round's independent node solves are mapped (default the builtin map, one
    after the other; a multiprocessing pool's map runs them on several cores — the nodes of a round
    are independent, so the tree is identical).
    init_mp ("we use ... matching pursuit ... to obtain an initial upper bound"): before
    the root, the incumbent is the better of β = 0, Algorithm 3's own point (matching_pursuit) and
    the exact box ridge on its support (upper_bound), strict improvements only, in that order.
    """
    t0 = time.perf_counter()
    p = P.p
    UB = 0.5 * P.yy
    inc_S, inc_b = np.zeros(0, dtype=np.int64), np.zeros(0)
    if init_mp:
        mp = matching_pursuit(P)
        if mp.obj < UB:
            UB, inc_S, inc_b = mp.obj, mp.support, mp.beta[mp.support]
        if len(mp.support):
            obj, bS = upper_bound(P, mp.support)
            if obj < UB:
                UB, inc_S, inc_b = obj, mp.support, bS
    # open node: (lb, id, depth, F0 tuple, F1 tuple, warm)
    open_nodes = [(-math.inf, 0, 0, (), (), None)]
    next_id = 1
    nodes = rounds = node_iters = 0
    trace = []
    status = "optimal"
    LB = -math.inf
    while True:
        open_nodes = [u for u in open_nodes if not (u[0] >= UB * (1 - prune_tol))]
        if not open_nodes:
            LB = UB
            break
        LB = min(u[0] for u in open_nodes)
        if UB > 0 and (UB - LB) / UB <= gap_tol:
            status = "gap"
            break
        if node_limit is not None and nodes >= node_limit:
            status = "node_limit"
            break
        if time_limit is not None and time.perf_counter() - t0 >= time_limit:
            status = "time_limit"
            break
        open_nodes.sort(key=lambda u: (u[0], u[1]))
        batch, open_nodes = open_nodes[:B], open_nodes[B:]
        rounds += 1
        results = []
        prune_ub = UB * (1 - prune_tol) if early_prune else math.inf
        jobs = [(make_code(p, F0, F1), warm, plb) for (plb, uid, depth, F0, F1, warm) in batch]
        solved = list(node_map(_solve_node, [(P, code, warm, plb, node_tol, check_every, max_iters, int_tol,
                                               prune_ub) for (code, warm, plb) in jobs]))
        for (plb, uid, depth, F0, F1, warm), (res, obj, bS) in zip(batch, solved):
            results.append((uid, depth, F0, F1, res, obj, bS))
            nodes += 1
            node_iters += res.iters
        for (uid, depth, F0, F1, res, obj, bS) in sorted(results, key=lambda r: r[0]):
            if obj < UB:
                UB, inc_S, inc_b = obj, res.support, bS
        for (uid, depth, F0, F1, res, obj, bS) in sorted(results, key=lambda r: r[0]):
            pruned = res.lb >= UB * (1 - prune_tol) or res.integral
            if record:
                trace.append(dict(id=uid, depth=depth, F0=F0, F1=F1, lb=res.lb, lb_best=res.lb_best,
                                  primal=res.primal, iters=res.iters, branch_j=res.branch_j,
                                  integral=res.integral, support=tuple(res.support.tolist()), ub=obj,
                                  pruned=pruned, early=res.pruned, round=rounds))
            if pruned:
                continue
            j = res.branch_j
            warm = (res.beta, res.v)
            open_nodes.append((res.lb, next_id, depth + 1, tuple(sorted(F0 + (j,))), F1, warm))
            open_nodes.append((res.lb, next_id + 1, depth + 1, F0, tuple(sorted(F1 + (j,))), warm))
            next_id += 2
    beta = np.zeros(p)
    beta[inc_S] = inc_b
    gap = 0.0 if UB <= 0 else max(0.0, (UB - LB) / UB)
    return dict(obj=UB, beta=beta, support=inc_S, lb=LB, gap=gap, nodes=nodes, rounds=rounds,
                node_iters=node_iters, status=status, open=len(open_nodes), trace=trace,
                time=time.perf_counter() - t0)


# ----------------------------------------------------------------------------------------------
# Matching-pursuit root heuristic (Algorithm 3; outline P:781-783)
# ----------------------------------------------------------------------------------------------

def mp_forward_scores(P: Problem, r, inS):
    """Forward step 1(a)-(c) of Algorithm 3 for every candidate j ∉ S:
    c = X_{S^c}ᵀ r, D = ‖X_{S^c}‖² + 2λ2, β* = c / D, β = Proj_[−M,M](β*),
    Δ = −β⊙c + ½β²⊙D + λ0.  Members of S get Δ = +∞.  Returns (Δ, β)."""
    c = P.X.T @ r
    D = np.einsum("ij,ij->j", P.X, P.X) + 2.0 * P.lam2
    b = np.clip(c / D, -P.M, P.M)
    delta = -b * c + 0.5 * b * b * D + P.lam0
    delta = np.where(inS, np.inf, delta)
    return delta, b


def mp_backward_scores(P: Problem, r, beta, S):
    """Backward step 2(a)-(b) of Algorithm 3 for j ∈ S (in the order of S):
    c_S = X_Sᵀ r, Δ = β⊙c_S + (½‖X_S‖² − λ2)⊙β² − λ0."""
    S = np.asarray(S, dtype=np.int64)
    XS = P.X[:, S]
    cS = XS.T @ r
    bS = beta[S]
    return bS * cS + (0.5 * np.einsum("ij,ij->j", XS, XS) - P.lam2) * bS * bS - P.lam0


@dataclass
class MPResult:
    support: np.ndarray           # sorted column indices of S
    beta: np.ndarray              # length p, zero off S
    obj: float                    # ½‖y − Xβ‖² + λ2‖β‖² + λ0|S| (a feasible point of eq:perspective)
    rounds: int
    steps: list = field(default_factory=list)   # ("+"/"−", j, Δ_j) in the order taken


def matching_pursuit(P: Problem, max_rounds=None):
    """Algorithm 3, step by step.  S ← ∅, β ← 0, r ← y; repeat { forward: the
    candidate j* = argmin Δ over j ∉ S joins S if Δ_j* < 0 (β_j* ← its projected value,
    r ← r − X_j*β_j*); backward: with the residual after the forward step, j* = argmin Δ over
    j ∈ S leaves S if Δ_j* < 0 (r ← r + X_j*β_j*, β_j* ← 0) } until a round changes nothing.
    Readings (R15): argmin ties → lowest column index; a round is one forward then
    one backward step; the loop is capped at max_rounds (default 4p + 10: every accepted step
    lowers the objective strictly, so the cap is a guard, not a stopping rule)."""
    p = P.p
    max_rounds = 4 * p + 10 if max_rounds is None else int(max_rounds)
    beta = np.zeros(p)
    r = P.y.copy()
    inS = np.zeros(p, dtype=bool)
    steps = []
    rounds = 0
    while rounds < max_rounds:
        rounds += 1
        changed = False
        delta, b = mp_forward_scores(P, r, inS)
        j = int(np.argmin(delta))            # first minimum = lowest index (R15)
        if delta[j] < 0:
            inS[j] = True
            beta[j] = b[j]
            r = r - P.X[:, j] * b[j]
            steps.append(("+", j, float(delta[j])))
            changed = True
        S = np.nonzero(inS)[0]               # ascending, so argmin ties → lowest index
        if len(S):
            dS = mp_backward_scores(P, r, beta, S)
            i = int(np.argmin(dS))
            if dS[i] < 0:
                j = int(S[i])
                r = r + P.X[:, j] * beta[j]
                steps.append(("-", j, float(dS[i])))
                beta[j] = 0.0
                inS[j] = False
                changed = True
        if not changed:
            break
    S = np.nonzero(inS)[0]
    obj = 0.5 * float(r @ r) + P.lam2 * float(beta @ beta) + P.lam0 * len(S)
    return MPResult(support=S, beta=beta, obj=obj, rounds=rounds, steps=steps)

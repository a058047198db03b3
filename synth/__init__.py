"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module is the ONLY code both sides use.  It holds none of the method's
arithmetic (no ADMM, prox, dual, FPG or branch-and-bound): it draws the design
matrix and response of PAPER.md §4.1 ("Datasets"), applies the
parameter-selection recipe of §4.1 as restated in DESIGN.md
"Input recipe", and draws random node fixings for parity tests.

Recipe:
  * rows of X ~ N(0, Σ) with Σ = ρ_c·11ᵀ + (1−ρ_c)·I, drawn as
    x = √ρ_c·g·1 + √(1−ρ_c)·ε with g, ε iid N(0,1)
  * Toeplitz/AR(1) variant for the real-data-shaped C5: x_j = φ x_{j−1} + √(1−φ²) ε_j
  * β† has k* equispaced ones at indices round(i·p/k*), i = 0..k*−1
  * y = Xβ† + σε with σ² = Var_emp(Xβ†)/SNR   (empirical variance S:474)
  * λ2* = argmin over 100 log-spaced λ2 ∈ [1e-4, 1e4] of ‖β† − β_S†(λ2)‖₂
  * M = 1.5·‖β_S†(λ2*)‖∞  ("M = 1.5 M*(λ2*)")
  * λ0* from the add/drop rule of DESIGN.md (replaces the external path rule)

RNG: numpy PCG64(seed); X is returned column-major (Fortran order), float64.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Instance", "make_instance", "config_instance", "CONFIGS",
    "ridge_on_support", "tune_lambda2", "bigM_rule", "lambda0_rule",
    "random_fixings", "random_supports",
]


@dataclass
class Instance:
    X: np.ndarray            # n×p, Fortran order, float64
    y: np.ndarray            # n
    beta_true: np.ndarray    # p
    support_true: np.ndarray  # int64 indices of β†
    sigma: float
    lambda0: float = float("nan")
    lambda2: float = float("nan")
    M: float = float("nan")
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.X.shape[0]

    @property
    def p(self) -> int:
        return self.X.shape[1]


def _equispaced_support(p: int, k: int) -> np.ndarray:
    # "k0 equispaced nonzero entries of value 1"; indices round(i·p/k)
    idx = np.array([int(round(i * p / k)) for i in range(k)], dtype=np.int64)
    return np.unique(np.clip(idx, 0, p - 1))


def make_instance(n: int, p: int, k: int, corr: float, snr: float, seed: int,
                  kind: str = "const") -> Instance:
    """Draw (X, y, β†) per P:809.  kind = "const" (Σ = ρ11ᵀ+(1−ρ)I) or "toeplitz" (AR(1))."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if kind == "const":
        # draw as p×n C-order then view transposed -> n×p Fortran order (column j contiguous)
        E = rng.standard_normal((p, n))
        g = rng.standard_normal(n)
        E *= math.sqrt(1.0 - corr)
        E += math.sqrt(corr) * g[None, :]
        X = E.T
    elif kind == "toeplitz":
        E = rng.standard_normal((p, n))
        s = math.sqrt(1.0 - corr * corr)
        for j in range(1, p):
            E[j] *= s
            E[j] += corr * E[j - 1]
        X = E.T
    else:
        raise ValueError(kind)
    assert X.flags.f_contiguous
    S = _equispaced_support(p, k)
    beta = np.zeros(p)
    beta[S] = 1.0
    mu = X[:, S].sum(axis=1)
    sigma = math.sqrt(float(np.var(mu)) / snr)
    y = mu + sigma * rng.standard_normal(n)
    return Instance(X=X, y=np.ascontiguousarray(y), beta_true=beta, support_true=S, sigma=sigma,
                    meta=dict(n=n, p=p, k=k, corr=corr, snr=snr, seed=seed, kind=kind))


def ridge_on_support(X: np.ndarray, y: np.ndarray, S: np.ndarray, lam2: float) -> np.ndarray:
    """β(λ2) restricted to S: (X_SᵀX_S + 2λ2 I) β_S = X_Sᵀ y."""
    XS = X[:, S]
    Q = XS.T @ XS + 2.0 * lam2 * np.eye(len(S))
    return np.linalg.solve(Q, XS.T @ y)


def tune_lambda2(inst: Instance) -> float:
    """λ2* by grid search, 100 log points on [1e-4, 1e4]; ties -> smaller λ2."""
    S = inst.support_true
    XS = inst.X[:, S]
    G = XS.T @ XS
    q = XS.T @ inst.y
    best, best_err = None, math.inf
    for lam2 in np.logspace(-4, 4, 100):
        b = np.linalg.solve(G + 2.0 * lam2 * np.eye(len(S)), q)
        err = float(np.linalg.norm(inst.beta_true[S] - b))
        if err < best_err:
            best, best_err = float(lam2), err
    return best


def bigM_rule(inst: Instance, lam2: float, factor: float = 1.5) -> float:
    """M = 1.5·‖β_S†(λ2)‖∞."""
    b = ridge_on_support(inst.X, inst.y, inst.support_true, lam2)
    return factor * float(np.max(np.abs(b)))


def lambda0_rule(inst: Instance, lam2: float) -> float:
    """Deterministic λ0* (replaces the external path rule of P:823).

    With f(β_S) = ½‖y − X_Sβ_S‖² + λ2‖β_S‖² fitted on S†:
      drop_j = ½ β_j² / (Q⁻¹)_jj        objective increase when j ∈ S† is removed (refit)
      add_j  = ½ (X_jᵀr)² / (‖X_j‖² + 2λ2 − X_jᵀX_S Q⁻¹ X_SᵀX_j)   decrease when j ∉ S† is added
    λ0* = √(max add · min drop) if max add < min drop, else max add.
    """
    X, y, S = inst.X, inst.y, inst.support_true
    XS = X[:, S]
    Q = XS.T @ XS + 2.0 * lam2 * np.eye(len(S))
    Qi = np.linalg.inv(Q)
    bS = Qi @ (XS.T @ y)
    r = y - XS @ bS
    drop = 0.5 * bS ** 2 / np.diag(Qi)
    mask = np.ones(X.shape[1], dtype=bool)
    mask[S] = False
    # chunked over columns to bound memory at p = 1e5
    max_add = 0.0
    cols = np.nonzero(mask)[0]
    for lo in range(0, len(cols), 8192):
        J = cols[lo:lo + 8192]
        XJ = X[:, J]
        cj = XJ.T @ r
        XSXJ = XS.T @ XJ                      # s × |J|
        denom = (XJ * XJ).sum(axis=0) + 2.0 * lam2 - np.einsum("ij,ij->j", XSXJ, Qi @ XSXJ)
        max_add = max(max_add, float(np.max(0.5 * cj ** 2 / denom)))
    min_drop = float(np.min(drop))
    if max_add < min_drop:
        return math.sqrt(max_add * min_drop)
    return max_add


# BASELINE.json configs.  C1 fixes λ0, λ2; the others use the recipe.
CONFIGS = {
    "C1": dict(n=50, p=20, k=3, corr=0.1, snr=5.0, kind="const", lambda0=0.1, lambda2=0.01),
    "C2": dict(n=1000, p=1000, k=10, corr=0.5, snr=5.0, kind="const"),
    "C3": dict(n=1000, p=10000, k=10, corr=0.1, snr=3.0, kind="const"),
    "C4": dict(n=1000, p=100000, k=10, corr=0.1, snr=5.0, kind="const"),
    "C5": dict(n=500, p=20000, k=10, corr=0.9, snr=1.0, kind="toeplitz"),
}


def config_instance(name: str, seed: int = 0, lambda0_mult: float = 1.0) -> Instance:
    """Build a BASELINE.json config with its λ0, λ2, M per the recipe."""
    c = dict(CONFIGS[name])
    lam0 = c.pop("lambda0", None)
    lam2 = c.pop("lambda2", None)
    inst = make_instance(seed=seed, **c)
    if lam2 is None:
        lam2 = tune_lambda2(inst)
    if lam0 is None:
        lam0 = lambda0_rule(inst, lam2)
    inst.lambda2 = float(lam2)
    inst.lambda0 = float(lam0) * lambda0_mult
    inst.M = bigM_rule(inst, lam2)
    inst.meta["config"] = name
    return inst


def random_fixings(p: int, B: int, seed: int, depth_lo: int = 0, depth_hi: int = 10,
                   prefer: np.ndarray | None = None) -> list[tuple[np.ndarray, np.ndarray]]:
    """B random node fixings (F0, F1) with |F0|+|F1| ∈ [depth_lo, depth_hi], disjoint.

    `prefer` (optional) biases picks toward given indices (e.g. S†) so F1 hits signal columns.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for _ in range(B):
        d = int(rng.integers(depth_lo, depth_hi + 1))
        d = min(d, p)
        if prefer is not None and len(prefer) and d:
            k1 = min(len(prefer), int(rng.integers(0, d + 1)))
            a = rng.choice(prefer, size=k1, replace=False) if k1 else np.array([], dtype=np.int64)
            rest = np.setdiff1d(np.arange(p), a)
            b = rng.choice(rest, size=d - k1, replace=False)
            idx = np.concatenate([a, b]).astype(np.int64)
        else:
            idx = rng.choice(p, size=d, replace=False).astype(np.int64)
        val = rng.integers(0, 2, size=d).astype(np.int64)
        out.append((np.sort(idx[val == 0]), np.sort(idx[val == 1])))
    return out


def random_supports(p: int, B: int, seed: int, s_lo: int = 0, s_hi: int = 40) -> list[np.ndarray]:
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for _ in range(B):
        s = int(rng.integers(s_lo, min(s_hi, p) + 1))
        out.append(np.sort(rng.choice(p, size=s, replace=False).astype(np.int64)))
    return out

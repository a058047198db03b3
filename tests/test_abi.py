"""C-ABI checks that need no GPU: the library loads, exports every entry point declared in
include/l0l2.h, refuses to run without a device (no CPU fallback), and the pure host logic
(rebalancing plan) behaves as documented."""
import re

import numpy as np
import pytest

import paper_2602_04551_b200 as L


def _declared():
    hdr = open(L.binding.HERE + "/../include/l0l2.h").read()
    return sorted(set(re.findall(r"\b(l0l2_[a-z_0-9]+)\s*\(", hdr)))


def test_every_declared_symbol_is_exported():
    syms = L.exported_symbols()
    assert set(syms) == set(_declared())
    missing = [k for k, v in syms.items() if not v]
    assert not missing, missing
    assert len(syms) >= 12


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(L.L0L2Error) as e:
        L.Problem(np.ones((4, 3)), np.ones(4), 0.1, 0.1, 1.0)
    assert e.value.code == L.ECUDA
    assert "no CPU fallback" in str(e.value)


def test_argument_validation_before_device():
    # λ2 ≤ 0 and M ≤ 0 are rejected before any device work
    for lam2, M in ((0.0, 1.0), (-1.0, 1.0), (0.1, 0.0)):
        with pytest.raises(L.L0L2Error) as e:
            L.Problem(np.ones((4, 3)), np.ones(4), 0.1, lam2, M)
        assert e.value.code == L.EINVAL


@pytest.mark.parametrize("counts,B", [([10, 0, 3, 0], 4), ([100, 0, 0, 0, 0, 0, 0, 0], 16), ([5, 5], 4),
                                      ([0, 0], 4), ([1000, 3, 7, 0], 8)])
def test_rebalance_plan(counts, B):
    plan = L.rebalance_plan(counts, B)
    c = list(counts)
    for src, dst, k in plan:
        assert k > 0 and src != dst and c[src] >= k
        c[src] -= k
        c[dst] += k
    assert sum(c) == sum(counts)
    # termination rule: the emptiest rank has ≥ B nodes or the spread is ≤ 1
    assert min(c) >= B or max(c) - min(c) <= 1 or len(plan) >= 4 * len(c)
    # determinism
    assert plan == L.rebalance_plan(counts, B)


def test_rebalance_plan_no_moves_when_balanced():
    assert L.rebalance_plan([20, 20, 20, 20], 16) == []
    assert L.rebalance_plan([3], 16) == []

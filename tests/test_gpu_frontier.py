"""Device frontier (csrc/frontier.cu) — -m gpu.

Single-rank synchronous solves keep the open set, the fixings, the warm-state refcounts and the
incumbent on the device (the host reads one status per round).  The host frontier of solve.cu
(L0L2_HOST_FRONTIER=1) implements the same batched reading of Algorithm 1 (R9), so the two
must produce the SAME tree: every trace record (id, depth, LB, primal, iterations, branch, flags, UB,
parent, fixing) bitwise equal, and the same certificate.  Both are also checked against the oracle's
tree by test_gpu_parity / test_gpu_fullsize, which now run on the device frontier.
"""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2602_04551_b200 import Problem  # noqa: E402


def _solve(monkeypatch, host, inst, lam0, lam2, M, rho, **kw):
    monkeypatch.setenv("L0L2_HOST_FRONTIER", "1" if host else "0")
    prob = Problem(inst.X, inst.y, lam0, lam2, M, rho=rho, node_tol=kw.pop("node_tol", 1e-8))
    res = prob.l0l2_solve(record=True, **kw)
    prob.close()
    return res


@pytest.mark.parametrize("B", [1, 4, 16, 33])
@pytest.mark.parametrize("ext", [False, True])
def test_device_frontier_equals_host_frontier(monkeypatch, B, ext):
    inst = synth.make_instance(80, 60, 5, 0.3, 3.0, 21)
    lam2 = 0.5
    lam0 = synth.lambda0_rule(inst, lam2)
    M = synth.bigM_rule(inst, lam2)
    rho = O.default_rho(inst.X)
    kw = dict(gap_tol=1e-4, batch=B, init_mp=ext, early_prune=ext)
    h = _solve(monkeypatch, True, inst, lam0, lam2, M, rho, **dict(kw))
    d = _solve(monkeypatch, False, inst, lam0, lam2, M, rho, **dict(kw))
    assert len(h["trace"]) == len(d["trace"]) > 10
    for a, b in zip(h["trace"], d["trace"]):
        assert a == b, (a, b)
    assert np.array_equal(h["beta"], d["beta"])
    assert h["obj"] == d["obj"] and h["gap"] == d["gap"]
    for key in ("nodes", "node_iters", "rounds", "lb", "ub", "status", "support_size"):
        assert h["stats"][key] == d["stats"][key], key


def test_device_frontier_wide_tree_and_small_pool(monkeypatch):
    """A C3-shaped tree with a small warm-state pool (children start cold when the pool is full) and
    a frontier that outgrows the initial device arrays: same tree as the host frontier."""
    inst = synth.make_instance(120, 800, 5, 0.2, 1.5, 4)
    lam2 = 0.5
    lam0 = synth.lambda0_rule(inst, lam2)
    M = synth.bigM_rule(inst, lam2)
    rho = O.default_rho(inst.X)
    kw = dict(gap_tol=1e-9, batch=16, node_limit=600, warm_bytes_cap=64 * 2 * 800 * 8)
    h = _solve(monkeypatch, True, inst, lam0, lam2, M, rho, **dict(kw))
    d = _solve(monkeypatch, False, inst, lam0, lam2, M, rho, **dict(kw))
    assert len(h["trace"]) == len(d["trace"]) >= 200
    for a, b in zip(h["trace"], d["trace"]):
        assert a == b, (a, b)
    assert h["obj"] == d["obj"]
    assert h["stats"]["max_open"] > 16

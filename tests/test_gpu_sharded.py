"""Column-sharded single-node ADMM (csrc/sharded.cu) — -m gpu.

Two processes share cuda:0; each holds half of X's columns (l0l2_create_sharded) and the per-iteration
all-reduce of u = Σ_r Z_r w_r (plus the check terms) runs over the library's host transport on a gloo
group.  The bounds must be the oracle's: fixed-iteration (β, v) gathered from the two shards within
1e-9, LB and primal within 1e-9, and converged bounds with the oracle's iteration counts; warm starts
follow P:543 exactly as in the node-parallel kernel."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import synth  # noqa: E402


def _instance():
    inst = synth.make_instance(160, 900, 5, 0.2, 3.0, 13)   # p > 2n: the Z-form
    lam2 = 0.5
    return inst, synth.lambda0_rule(inst, lam2), lam2, synth.bigM_rule(inst, lam2)


def _fixings(inst):
    return [((), ())] + synth.random_fixings(inst.p, 4, seed=3, depth_lo=1, depth_hi=6, prefer=inst.support_true)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, impl, q):
    import torch.distributed as dist
    os.environ["L0L2_SHARD_GEMM"] = "1" if impl == "gemm" else "0"
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_04551_b200 import ShardedProblem
        inst, lam0, lam2, M = _instance()
        p = inst.p
        cuts = [p * r // world for r in range(world + 1)]
        c0, c1 = cuts[rank], cuts[rank + 1]
        rho = O.default_rho(inst.X)
        kw = dict(node_tol=-1.0, max_iters=37) if mode == "fixed" else dict(node_tol=1e-7, max_iters=20000)
        sp = ShardedProblem(inst.X[:, c0:c1], inst.y, c0, p, lam0, lam2, M, rho=rho, device=0, **kw)
        fx = _fixings(inst)
        out = sp.l0l2_bound_sharded(fx)
        res = {k: v.cpu().numpy() for k, v in out.items() if k != "rc"}
        # warm children of the root (its state on this rank's columns)
        kids = [((int(inst.support_true[0]),), ()), ((), (int(inst.support_true[0]),))]
        w0 = out["warm_out"][:1]
        outk = sp.l0l2_bound_sharded(kids, warm_in=torch.cat([w0, w0]), parent_lb=[float(out["lb"][0])] * 2)
        resk = {k: v.cpu().numpy() for k, v in outk.items() if k != "rc"}
        sp.close()
        q.put((rank, c0, c1, res, resk, None))
    except Exception as e:
        import traceback
        q.put((rank, 0, 0, None, None, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _run(mode, impl, world=2):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, impl, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
    for r in out:
        assert r[5] is None, r[5]
    return out


@pytest.mark.parametrize("impl", ["fused", "gemm"])
@pytest.mark.parametrize("mode", ["fixed", "converged"])
def test_two_rank_column_sharded_bounds_equal_the_oracle(mode, impl):
    """impl "fused": the persistent ADMM kernel in step mode on each rank's shard (one launch per
    iteration, U all-reduced between launches); "gemm": the unfused reference loop."""
    inst, lam0, lam2, M = _instance()
    P = O.Problem(inst.X, inst.y, lam0, lam2, M)
    out = _run(mode, impl)
    fx = _fixings(inst)
    kw = dict(node_tol=-1.0, max_iters=37) if mode == "fixed" else dict(node_tol=1e-7, max_iters=20000)
    # every rank returns the same bounds, iterations and flags
    for key in ("lb", "primal", "iters", "flags"):
        assert np.array_equal(out[0][3][key], out[1][3][key]), key
        assert np.array_equal(out[0][4][key], out[1][4][key]), key
    beta = np.concatenate([o[3]["warm_out"][:, 0, :] for o in out], axis=1)
    v = np.concatenate([o[3]["warm_out"][:, 1, :] for o in out], axis=1)
    refs = []
    for k, (F0, F1) in enumerate(fx):
        r = O.admm_node(P, O.make_code(inst.p, F0, F1), **kw)
        refs.append(r)
        lb, pr, it = out[0][3]["lb"][k], out[0][3]["primal"][k], out[0][3]["iters"][k]
        assert it == r.iters, (k, it, r.iters)
        tol = 1e-9 if mode == "fixed" else 1e-6
        assert abs(lb - r.lb) <= tol * max(1.0, abs(r.lb)), (k, lb, r.lb)
        assert abs(pr - r.primal) <= tol * max(1.0, abs(r.primal)), (k, pr, r.primal)
        if mode == "fixed":
            assert np.max(np.abs(beta[k] - r.beta)) <= 1e-9 * (1 + np.max(np.abs(r.beta)))
            assert np.max(np.abs(v[k] - r.v)) <= 1e-9 * (1 + np.max(np.abs(r.v)))
    kids = [((int(inst.support_true[0]),), ()), ((), (int(inst.support_true[0]),))]
    for k, (F0, F1) in enumerate(kids):
        r = O.admm_node(P, O.make_code(inst.p, F0, F1), warm=(refs[0].beta, refs[0].v), parent_lb=refs[0].lb, **kw)
        assert out[0][4]["iters"][k] == r.iters
        tol = 1e-9 if mode == "fixed" else 1e-6
        assert abs(out[0][4]["lb"][k] - r.lb) <= tol * max(1.0, abs(r.lb))

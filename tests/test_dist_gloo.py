"""World-size-2 CPU (gloo) coverage of the multi-GPU host logic of l0l2_solve.

The NCCL data path itself needs GPUs; what runs here is everything the ranks must agree on
without it: the per-round status exchange (global UB = min, global LB = min of the ranks'
open-node minima, termination), the deterministic rebalancing plan computed by libl0l2 on
every rank from all-gathered open counts, and node-count conservation under the plan."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2602_04551_b200 as L
    g = torch.Generator().manual_seed(1234 + rank)
    results = []
    for rnd in range(20):
        # local state of this rank after a round
        open_cnt = int(torch.randint(0, 40, (1,), generator=g))
        ub = float(100 + torch.rand(1, generator=g) * 10)
        lbmin = float(90 + torch.rand(1, generator=g) * 10) if open_cnt else float("inf")
        st = torch.tensor([ub, lbmin, float(open_cnt)], dtype=torch.float64)
        allst = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allst, st)
        gub = min(float(s[0]) for s in allst)
        owner = min(r for r in range(world) if float(allst[r][0]) == gub)
        glb = min(float(s[1]) for s in allst)
        gopen = sum(int(s[2]) for s in allst)
        done = gopen == 0 or (gub - glb) / gub <= 0.05
        counts = [int(s[2]) for s in allst]
        plan = L.rebalance_plan(counts, 16)
        after = list(counts)
        for src, dst, k in plan:
            after[src] -= k
            after[dst] += k
        # every rank must have derived the same decision: gather and compare
        mine = torch.tensor([gub, glb, float(gopen), float(done), float(owner)] + [float(x) for x in after],
                            dtype=torch.float64)
        allm = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allm, mine)
        same = all(torch.equal(allm[0], m) for m in allm)
        results.append((same, sum(after) == sum(counts), min(after) >= min(counts)))
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, results))


@pytest.mark.parametrize("world", [2])
def test_status_exchange_and_rebalance_agree_across_ranks(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, res in out:
        assert len(res) == 20
        for same, conserved, not_worse in res:
            assert same and conserved and not_worse


def _transport_worker(rank, world, port, q):
    """The HostTransport callbacks (the marshalling the library calls during a multi-rank solve),
    invoked through their C function pointers exactly as solve.cu invokes them."""
    import ctypes as C
    import numpy as np
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_04551_b200 import HostTransport
    t = HostTransport().struct
    ok = []
    mine = np.array([rank + 0.5, -rank, 7.0 * rank], dtype=np.float64)
    out = np.zeros(3 * world)
    ok.append(t.allgather(None, mine.ctypes.data, out.ctypes.data, mine.nbytes) == 0)
    ok.append(np.array_equal(out, np.concatenate([[r + 0.5, -r, 7.0 * r] for r in range(world)])))
    buf = np.arange(5, dtype=np.int64) * (rank + 1)
    ok.append(t.bcast(None, buf.ctypes.data, buf.nbytes, 1) == 0)
    ok.append(np.array_equal(buf, np.arange(5) * 2))
    pay = np.full(4, 3.25) if rank == 0 else np.zeros(4)
    if rank == 0:
        ok.append(t.send(None, pay.ctypes.data, pay.nbytes, 1) == 0)
    else:
        ok.append(t.recv(None, pay.ctypes.data, pay.nbytes, 0) == 0)
        ok.append(np.array_equal(pay, np.full(4, 3.25)))
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, all(ok)))


def test_host_transport_callbacks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_transport_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in out), out

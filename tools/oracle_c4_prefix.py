"""Run the CPU oracle's BnB on a config for a fixed node prefix and store its per-node trace.

Calls only oracle/ and synth/ (allowed source of stored expected values).  Output:
tests/golden/oracle_<cfg>_prefix.json — node-for-node tree of the first `nodes` nodes
(id, fixings, LB, primal, iterations, branch index, support, UB) plus the mean ADMM iterations
per node, used (a) as the C4 tree-parity fixture and (b) to convert the oracle's measured
node-iteration rate into nodes/s for bench.py's cpu_baseline.
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
nodes = int(sys.argv[2]) if len(sys.argv) > 2 else 31
rho_mult = float(sys.argv[3]) if len(sys.argv) > 3 else 3.0
B = int(sys.argv[4]) if len(sys.argv) > 4 else 16
inst = synth.config_instance(cfg, seed=0)
rho = O.default_rho(inst.X) * rho_mult
P = O.Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho)
t = time.time()
res = O.bnb_solve(P, B=B, gap_tol=1e-2, node_tol=1e-4, node_limit=nodes, record=True)
dt = time.time() - t
out = dict(config=cfg, seed=0, rho=rho, rho_mult=rho_mult, batch=B, gap_tol=1e-2, node_tol=1e-4,
           lambda0=inst.lambda0, lambda2=inst.lambda2, M=inst.M, nodes=res["nodes"], node_iters=res["node_iters"],
           iters_per_node=res["node_iters"] / max(1, res["nodes"]), ub=res["obj"], lb=res["lb"],
           seconds=dt, trace=[{k: (list(v) if isinstance(v, tuple) else v) for k, v in tr.items()} for tr in res["trace"]],
           script="tools/oracle_c4_prefix.py (oracle only)")
with open("tests/golden/oracle_%s_prefix.json" % cfg, "w") as f:
    json.dump(out, f, indent=1, default=float)
print("done", res["nodes"], res["node_iters"], dt)

"""Run the CPU oracle's BnB (oracle/ only) on a BASELINE config and store its node-for-node trace as a
tests/golden fixture (allowed source of stored expected values: this script calls only oracle/ and
synth/, never the CUDA library).

usage: python tools/oracle_tree_golden.py CFG GAP_TOL NODE_TOL B RHO_MULT [mp_ep] [NODE_LIMIT] [LAMBDA0_MULT]
  mp_ep: 1 → init_mp + early_prune (DESIGN R15/R16) on the oracle side
  LAMBDA0_MULT: λ0 = mult·λ0* (the paper's λ0-path multipliers)
writes tests/golden/oracle_<CFG>[_l0x<mult>]_tree_g<gap>_n<node_tol>_B<B>[_mpep][_lim<N>].json
"""
import json
import sys
import time

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import synth  # noqa: E402

cfg, gap_tol, node_tol, B, rho_mult = sys.argv[1], float(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), float(sys.argv[5])
ext = len(sys.argv) > 6 and sys.argv[6] == "1"
limit = int(sys.argv[7]) if len(sys.argv) > 7 and int(sys.argv[7]) > 0 else None
l0m = float(sys.argv[8]) if len(sys.argv) > 8 else 1.0
inst = synth.config_instance(cfg, seed=0, lambda0_mult=l0m)
rho = O.default_rho(inst.X) * rho_mult
P = O.Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho)
t = time.time()
res = O.bnb_solve(P, B=B, gap_tol=gap_tol, node_tol=node_tol, node_limit=limit, record=True,
                  init_mp=ext, early_prune=ext)
dt = time.time() - t
name = "oracle_%s%s_tree_g%g_n%g_B%d%s%s.json" % (cfg, "_l0x%g" % l0m if l0m != 1.0 else "", gap_tol, node_tol, B,
                                                  "_mpep" if ext else "", "_lim%d" % limit if limit else "")
out = dict(config=cfg, seed=0, lambda0_mult=l0m, rho=rho, rho_mult=rho_mult, batch=B, gap_tol=gap_tol, node_tol=node_tol,
           init_mp=ext, early_prune=ext, node_limit=limit,
           lambda0=inst.lambda0, lambda2=inst.lambda2, M=inst.M, nodes=res["nodes"], rounds=res["rounds"],
           node_iters=res["node_iters"], obj=res["obj"], lb=res["lb"], gap=res["gap"], status=res["status"],
           support=[int(j) for j in res["support"]], seconds=dt,
           trace=[dict(id=tr["id"], depth=tr["depth"], lb=tr["lb"], primal=tr["primal"], iters=tr["iters"],
                       branch_j=tr["branch_j"], ub=tr["ub"], early=tr["early"], pruned=tr["pruned"],
                       F0=[int(j) for j in tr["F0"]], F1=[int(j) for j in tr["F1"]]) for tr in res["trace"]],
           script="tools/oracle_tree_golden.py (oracle only)")
with open("tests/golden/" + name, "w") as f:
    json.dump(out, f, separators=(",", ":"), default=float)
print(name, res["nodes"], res["node_iters"], res["status"], "%.1fs" % dt)

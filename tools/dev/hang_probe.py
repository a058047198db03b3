import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_2602_04551_b200 import Problem
n, p, iters = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
inst = synth.make_instance(n, p, 5, 0.2, 5.0, 3)
pr = Problem(inst.X, inst.y, 50.0, 1.0, 2.0, node_tol=-1.0, max_iters=iters)
t = time.time()
out = pr.l0l2_bound_batch([((), ())] * 3)
torch.cuda.synchronize()
print(n, p, iters, "ok %.3fs" % (time.time() - t), float(out["lb"][0]), flush=True)

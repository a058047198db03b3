"""Per-warp phase breakdown of admm_persistent from a -DL0L2_PROF build (developer tool):
    L0L2_LIB=libl0l2_prof.so python tools/prof_phases.py C4 200 16 [check_every]"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_04551_b200 import Problem, binding  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 16
ce = int(sys.argv[4]) if len(sys.argv) > 4 else 10
inst = synth.config_instance(cfg, seed=0)
rho = 3.0 * float(np.mean(np.einsum("ij,ij->j", inst.X, inst.X)))
pr = Problem(inst.X, inst.y, inst.lambda0, inst.lambda2, inst.M, rho=rho, node_tol=-1.0, max_iters=iters,
             check_every=ce)
fx = [((), ())] + synth.random_fixings(inst.p, nb - 1, seed=5, depth_lo=1, depth_hi=6, prefer=inst.support_true)
lib = binding.load_library()
buf = (C.c_ulonglong * (160 * 16 * 8))()
pr.l0l2_bound_batch(fx)
torch.cuda.synchronize()
lib.l0l2_debug_prof(buf, 1)
pr.l0l2_bound_batch(fx)
torch.cuda.synchronize()
lib.l0l2_debug_prof(buf, 1)
a = np.frombuffer(buf, dtype=np.uint64).reshape(160, 16, 8).astype(np.float64)

a = a[:148]
mma = a[:, :14, :].mean(axis=(0, 1))
epi = a[:, 14:16, :].mean(axis=(0, 1))
w0 = a[:, 0, :].mean(axis=0)
print("MMA warps  (cycles/warp): stage-wait %.3g adj %.3g wready-wait %.3g fwd %.3g release %.3g" % tuple(mma[:5]))
print("epi warps  (cycles/warp): stage-wait %.3g pre %.3g sready-wait %.3g partials %.3g xwait %.3g math %.3g" % tuple(epi[:6]))
print("warp 0 loop: fused sweeps %.3g, sync+reduce %.3g, check phase %.3g" % (w0[6], w0[7], w0[5]))
s6 = a[:, 0, 6]
s7 = a[:, 0, 7]
print("per-CTA fused sweeps: min %.4g mean %.4g max %.4g; sync+reduce min %.4g mean %.4g max %.4g"
      % (s6.min(), s6.mean(), s6.max(), s7.min(), s7.mean(), s7.max()))
print("slowest CTAs:", np.argsort(-s6)[:8], "fastest:", np.argsort(s6)[:8])
for tag, idxs in (("slowest", np.argsort(-s6)[:4]), ("fastest", np.argsort(s6)[:4])):
    for c in idxs:
        m = a[c, :14, :].mean(axis=0)
        e = a[c, 14:16, :].mean(axis=0)
        print("%s CTA %3d: MMA stage %.3g adj %.3g wready %.3g fwd %.3g rel %.3g | epi stage %.3g pre %.3g sready %.3g part %.3g xwait %.3g math %.3g"
              % ((tag, c) + tuple(m[:5]) + tuple(e[:6])))

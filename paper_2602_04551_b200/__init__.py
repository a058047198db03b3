"""B200-native (sm_100a) ℓ0–ℓ2 branch-and-bound hot path of arXiv 2602.04551.

Thin Python binding over the C-ABI in include/l0l2.h (libl0l2.so, built in-tree by
build.py).  This module only marshals arguments: every numeric step runs in the library's
CUDA kernels.  There is no CPU fallback — importing works without a GPU (so the ABI can be
inspected), but creating a problem without a CUDA device raises L0L2Error.
"""
from .binding import (  # noqa: F401
    L0L2Error, Problem, lib_path, load_library, exported_symbols, rebalance_plan,
    FLAG_CONVERGED, FLAG_INTEGRAL, FLAG_MAXITER, FLAG_PRUNED, OK, EINVAL, ENOMEM, ECUDA, ENCCL, WNOTCONV, WLIMIT,
    nccl_unique_id, nccl_selftest, HostTransport, ShardedProblem,
)

__all__ = ["Problem", "ShardedProblem", "L0L2Error", "load_library", "rebalance_plan"]

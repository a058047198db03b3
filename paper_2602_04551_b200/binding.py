"""ctypes binding of include/l0l2.h — same names as the C entry points, marshalling only."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(HERE, os.environ.get("L0L2_LIB", "libl0l2.so"))   # L0L2_LIB: in-tree variant (tuning runs)

OK, EINVAL, ENOMEM, ECUDA, ENCCL = 0, -1, -2, -3, -4
WNOTCONV, WLIMIT = 1, 2
FLAG_CONVERGED, FLAG_INTEGRAL, FLAG_MAXITER, FLAG_PRUNED = 1, 2, 4, 8


class L0L2Error(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("l0l2 error %d: %s" % (code, msg))
        self.code = code


class _Opts(C.Structure):
    _fields_ = [("M", C.c_double), ("rho", C.c_double), ("node_tol", C.c_double), ("int_tol", C.c_double),
                ("check_every", C.c_int32), ("max_iters", C.c_int32), ("device", C.c_int32),
                ("x_on_device", C.c_int32)]


class _SolveOpts(C.Structure):
    _fields_ = [("gap_tol", C.c_double), ("time_limit_s", C.c_double), ("node_limit", C.c_int64),
                ("batch", C.c_int32), ("rebalance_every", C.c_int32), ("warm_bytes_cap", C.c_int64),
                ("verbose", C.c_int32), ("record", C.c_int32), ("init_mp", C.c_int32),
                ("early_prune", C.c_int32), ("continuous", C.c_int32), ("coop_rampup", C.c_int32)]


class _Stats(C.Structure):
    _fields_ = [("nodes", C.c_int64), ("node_iters", C.c_int64), ("rounds", C.c_int64), ("max_open", C.c_int64),
                ("nodes_global", C.c_int64), ("node_iters_global", C.c_int64),
                ("t_total", C.c_double), ("t_bound", C.c_double), ("t_upper", C.c_double), ("t_tree", C.c_double),
                ("t_comm", C.c_double), ("lb", C.c_double), ("ub", C.c_double), ("gap", C.c_double),
                ("status", C.c_int32), ("support_size", C.c_int32), ("nodes_moved", C.c_int64),
                ("suspensions", C.c_int64), ("coop_rounds", C.c_int64)]


class _KStats(C.Structure):
    _fields_ = [("admm_launches", C.c_int64), ("admm_iters", C.c_int64), ("admm_node_iters", C.c_int64),
                ("admm_ms", C.c_double), ("admm_bytes_alg", C.c_double), ("admm_flops_alg", C.c_double),
                ("upper_launches", C.c_int64), ("upper_ms", C.c_double), ("upper_bytes_alg", C.c_double)]


_ALLGATHER_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64)
_P2P_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32)


class _Transport(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allgather", _ALLGATHER_FN), ("send", _P2P_FN), ("recv", _P2P_FN),
                ("bcast", _P2P_FN)]


_lib = None
P = C.c_void_p


def lib_path():
    return _LIB_PATH


def load_library():
    """Load libl0l2.so (fails loudly if it has not been built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError("libl0l2.so not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(no CPU fallback exists)")
    lib = C.CDLL(_LIB_PATH, mode=C.RTLD_GLOBAL)
    lib.l0l2_default_opts.argtypes = [C.POINTER(_Opts)]
    lib.l0l2_default_opts.restype = None
    lib.l0l2_create.argtypes = [P, P, C.c_int64, C.c_int64, C.c_double, C.c_double, C.POINTER(_Opts), C.POINTER(P)]
    lib.l0l2_create.restype = C.c_int
    lib.l0l2_bound_batch.argtypes = [P, C.c_int32] + [P] * 13 + [P]
    lib.l0l2_bound_batch.restype = C.c_int
    lib.l0l2_upper_batch.argtypes = [P, C.c_int32, P, P, P, P, P]
    lib.l0l2_upper_batch.restype = C.c_int
    lib.l0l2_matching_pursuit.argtypes = [P, C.c_int32, P, P, C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                          C.POINTER(C.c_int32)]
    lib.l0l2_matching_pursuit.restype = C.c_int
    lib.l0l2_default_solve_opts.argtypes = [C.POINTER(_SolveOpts)]
    lib.l0l2_default_solve_opts.restype = None
    lib.l0l2_solve.argtypes = [P, C.POINTER(_SolveOpts), P, C.POINTER(C.c_double), C.POINTER(C.c_double),
                               C.POINTER(_Stats)]
    lib.l0l2_solve.restype = C.c_int
    lib.l0l2_nccl_unique_id.argtypes = [P]
    lib.l0l2_nccl_unique_id.restype = C.c_int
    lib.l0l2_comm_init.argtypes = [P, C.c_int32, C.c_int32, P]
    lib.l0l2_comm_init.restype = C.c_int
    lib.l0l2_comm_init_transport.argtypes = [P, C.c_int32, C.c_int32, C.POINTER(_Transport)]
    lib.l0l2_comm_init_transport.restype = C.c_int
    lib.l0l2_rebalance_plan.argtypes = [C.c_int32, P, C.c_int64, P, C.c_int32]
    lib.l0l2_rebalance_plan.restype = C.c_int
    lib.l0l2_kernel_stats.argtypes = [P, C.POINTER(_KStats), C.c_int32]
    lib.l0l2_kernel_stats.restype = C.c_int
    lib.l0l2_solve_trace.argtypes = [P, P, C.c_int64]
    lib.l0l2_solve_trace.restype = C.c_int64
    lib.l0l2_create_sharded.argtypes = [P, P, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double,
                                        C.POINTER(_Opts), C.c_int32, C.c_int32, P, P, C.POINTER(P)]
    lib.l0l2_create_sharded.restype = C.c_int
    lib.l0l2_bound_sharded.argtypes = [P, C.c_int32] + [P] * 10 + [P]
    lib.l0l2_bound_sharded.restype = C.c_int
    lib.l0l2_info.argtypes = [P] + [P] * 5
    lib.l0l2_info.restype = C.c_int
    lib.l0l2_nccl_selftest.argtypes = [C.c_int32]
    lib.l0l2_nccl_selftest.restype = C.c_int
    lib.l0l2_admm_path.argtypes = [P]
    lib.l0l2_admm_path.restype = C.c_int
    lib.l0l2_last_error.argtypes = [P]
    lib.l0l2_last_error.restype = C.c_char_p
    lib.l0l2_destroy.argtypes = [P]
    lib.l0l2_destroy.restype = None
    _lib = lib
    return lib


def exported_symbols():
    """Names of the l0l2_* functions declared in include/l0l2.h that the library exports."""
    import re
    hdr = open(os.path.join(HERE, "..", "include", "l0l2.h")).read()
    names = sorted(set(re.findall(r"\b(l0l2_[a-z_0-9]+)\s*\(", hdr)))
    lib = load_library()
    return {n: hasattr(lib, n) for n in names}


def _check(rc, ctx=None, allow_warn=True):
    if rc < 0 or (rc > 0 and not allow_warn):
        msg = load_library().l0l2_last_error(ctx).decode(errors="replace")
        raise L0L2Error(rc, msg)
    return rc


def rebalance_plan(counts, batch, max_moves=64):
    lib = load_library()
    cnt = np.ascontiguousarray(counts, dtype=np.int64)
    plan = np.zeros(3 * max_moves, dtype=np.int64)
    m = lib.l0l2_rebalance_plan(len(cnt), cnt.ctypes.data, int(batch), plan.ctypes.data, max_moves)
    if m < 0:
        raise L0L2Error(m, "bad arguments")
    return [tuple(int(x) for x in plan[3 * i:3 * i + 3]) for i in range(min(m, max_moves))]


def nccl_selftest(device=0) -> int:
    """l0l2_nccl_selftest: the NCCL calls of the multi-GPU exchange on a 1-rank communicator."""
    return load_library().l0l2_nccl_selftest(int(device))


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(load_library().l0l2_nccl_unique_id(C.cast(buf, P)))
    return bytes(buf)


class HostTransport:
    """l0l2_transport callbacks over a torch.distributed process group (e.g. gloo): host bytes in,
    host bytes out — marshalling only; the exchange logic lives in the library (solve.cu)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.group = group
        W = dist.get_world_size(group)

        def view(addr, nbytes):
            return torch.from_numpy(np.ctypeslib.as_array((C.c_uint8 * int(nbytes)).from_address(addr)))

        def allgather(user, inp, out, nbytes):
            try:
                outs = [torch.empty(int(nbytes), dtype=torch.uint8) for _ in range(W)]
                dist.all_gather(outs, view(inp, nbytes).clone(), group=group)
                view(out, W * nbytes).copy_(torch.cat(outs))
                return 0
            except Exception:
                return 1

        def send(user, buf, nbytes, peer):
            try:
                dist.send(view(buf, nbytes).clone(), dst=int(peer), group=group)
                return 0
            except Exception:
                return 1

        def recv(user, buf, nbytes, peer):
            try:
                t = torch.empty(int(nbytes), dtype=torch.uint8)
                dist.recv(t, src=int(peer), group=group)
                view(buf, nbytes).copy_(t)
                return 0
            except Exception:
                return 1

        def bcast(user, buf, nbytes, root):
            try:
                t = view(buf, nbytes).clone()
                dist.broadcast(t, src=int(root), group=group)
                view(buf, nbytes).copy_(t)
                return 0
            except Exception:
                return 1

        self._fns = (_ALLGATHER_FN(allgather), _P2P_FN(send), _P2P_FN(recv), _P2P_FN(bcast))
        self.struct = _Transport(None, *self._fns)


def _ptr(t):
    """Device pointer of a torch CUDA tensor (or None → NULL)."""
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


class Problem:
    """One l0l2_ctx: (X, y, λ0, λ2, M) resident in HBM with the tree-wide precompute done.

    X: numpy float64 (n×p; any order — copied column-major) or a torch CUDA float64 tensor in
    column-major layout (X.T contiguous); y likewise.
    """

    def __init__(self, X, y, lambda0, lambda2, M, rho=0.0, node_tol=1e-4, int_tol=1e-4, check_every=10,
                 max_iters=10000, device=0):
        self._lib = load_library()
        o = _Opts()
        self._lib.l0l2_default_opts(C.byref(o))
        o.M, o.rho, o.node_tol, o.int_tol = float(M), float(rho), float(node_tol), float(int_tol)
        o.check_every, o.max_iters, o.device = int(check_every), int(max_iters), int(device)
        self._keep = []
        if isinstance(X, np.ndarray):
            Xf = np.asfortranarray(X, dtype=np.float64)
            yf = np.ascontiguousarray(y, dtype=np.float64)
            n, p = Xf.shape
            o.x_on_device = 0
            xp, yp = Xf.ctypes.data, yf.ctypes.data
            self._keep += [Xf, yf]
        else:   # torch CUDA tensors
            import torch
            assert X.is_cuda and X.dtype == torch.float64
            n, p = X.shape
            if not X.T.is_contiguous():
                X = X.T.contiguous().T
            yv = y.contiguous()
            torch.cuda.current_stream(X.device).synchronize()   # X, y complete before the library copies them
            o.x_on_device = 1
            xp, yp = X.data_ptr(), yv.data_ptr()
            self._keep += [X, yv]
        self.n, self.p = int(n), int(p)
        self.lambda0, self.lambda2, self.M = float(lambda0), float(lambda2), float(M)
        ctx = P()
        rc = self._lib.l0l2_create(C.c_void_p(xp), C.c_void_p(yp), self.n, self.p, self.lambda0, self.lambda2,
                                   C.byref(o), C.byref(ctx))
        self._keep = []
        if rc != OK:
            raise L0L2Error(rc, self._lib.l0l2_last_error(None).decode(errors="replace"))
        self._ctx = ctx
        self.device = int(device)

    # -------------------------------------------------------------- lifecycle / info
    def close(self):
        if getattr(self, "_ctx", None):
            self._lib.l0l2_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self):
        n, p, dev, launches = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        rho = C.c_double()
        _check(self._lib.l0l2_info(self._ctx, C.byref(n), C.byref(p), C.byref(rho), C.byref(dev), C.byref(launches)),
               self._ctx)
        path = self._lib.l0l2_admm_path(self._ctx)
        return dict(n=n.value, p=p.value, rho=rho.value, device_bytes=dev.value, kernel_launches=launches.value,
                    admm_path={0: "fused-zform", 1: "fused-direct", 2: "wide-n"}.get(path, path))

    def l0l2_kernel_stats(self, reset=False):
        ks = _KStats()
        _check(self._lib.l0l2_kernel_stats(self._ctx, C.byref(ks), int(bool(reset))), self._ctx)
        return {f: getattr(ks, f) for f, _ in _KStats._fields_}

    @property
    def rho(self):
        return self.info()["rho"]

    # -------------------------------------------------------------- batch calls (device tensors)
    def fixings_csr(self, fixings):
        """[(F0, F1), ...] → (fix_off int64[B+1], fix_idx int32, fix_val uint8) CUDA tensors."""
        import torch
        off, idx, val = [0], [], []
        for F0, F1 in fixings:
            F0 = [int(i) for i in F0]
            F1 = [int(i) for i in F1]
            idx += F0 + F1
            val += [0] * len(F0) + [1] * len(F1)
            off.append(len(idx))
        dev = torch.device("cuda", self.device)
        return (torch.tensor(off, dtype=torch.int64, device=dev),
                torch.tensor(idx if idx else [0], dtype=torch.int32, device=dev),
                torch.tensor(val if val else [0], dtype=torch.uint8, device=dev))

    def l0l2_bound_batch(self, fixings, warm_in=None, parent_lb=None, want_warm=True, want_zhat=False,
                         want_dual_r=False, stream=None):
        import torch
        B = len(fixings)
        dev = torch.device("cuda", self.device)
        fo, fi, fv = self.fixings_csr(fixings)
        f64 = dict(dtype=torch.float64, device=dev)
        out = dict(lb=torch.empty(B, **f64), primal=torch.empty(B, **f64),
                   branch_j=torch.empty(B, dtype=torch.int32, device=dev),
                   iters=torch.empty(B, dtype=torch.int32, device=dev),
                   flags=torch.empty(B, dtype=torch.uint8, device=dev))
        out["warm_out"] = torch.empty((B, 2, self.p), **f64) if want_warm else None
        out["zhat"] = torch.empty((B, self.p), **f64) if want_zhat else None
        out["dual_r"] = torch.empty((B, self.n), **f64) if want_dual_r else None
        if warm_in is not None:
            warm_in = warm_in.to(**f64).contiguous()
        if parent_lb is not None:
            parent_lb = torch.as_tensor(parent_lb, **f64).contiguous()
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        rc = self._lib.l0l2_bound_batch(self._ctx, B, _ptr(fo), _ptr(fi), _ptr(fv), _ptr(warm_in), _ptr(parent_lb),
                                        _ptr(out["lb"]), _ptr(out["primal"]), _ptr(out["warm_out"]),
                                        _ptr(out["zhat"]), _ptr(out["dual_r"]), _ptr(out["branch_j"]),
                                        _ptr(out["iters"]), _ptr(out["flags"]), C.c_void_p(s.cuda_stream))
        _check(rc, self._ctx)
        out["rc"] = rc
        return out

    def l0l2_upper_batch(self, supports, stream=None):
        import torch
        dev = torch.device("cuda", self.device)
        off, idx = [0], []
        for S in supports:
            idx += [int(i) for i in S]
            off.append(len(idx))
        so = torch.tensor(off, dtype=torch.int64, device=dev)
        si = torch.tensor(idx if idx else [0], dtype=torch.int32, device=dev)
        obj = torch.empty(len(supports), dtype=torch.float64, device=dev)
        bs = torch.empty(max(1, len(idx)), dtype=torch.float64, device=dev)
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        _check(self._lib.l0l2_upper_batch(self._ctx, len(supports), _ptr(so), _ptr(si), _ptr(obj), _ptr(bs),
                                          C.c_void_p(s.cuda_stream)), self._ctx)
        betas = []
        bsh = bs.cpu().numpy()
        for k in range(len(supports)):
            betas.append(bsh[off[k]:off[k + 1]].copy())
        return obj, betas

    # -------------------------------------------------------------- solve / multi-GPU
    def l0l2_matching_pursuit(self, max_rounds=0):
        """Algorithm 3 on the device → dict(support, beta, obj, rounds)."""
        beta = np.zeros(self.p, dtype=np.float64)
        supp = np.zeros(max(1, self.p), dtype=np.int32)
        slen, rounds = C.c_int32(), C.c_int32()
        obj = C.c_double()
        rc = self._lib.l0l2_matching_pursuit(self._ctx, int(max_rounds), beta.ctypes.data, supp.ctypes.data,
                                             C.byref(slen), C.byref(obj), C.byref(rounds))
        _check(rc, self._ctx)
        return dict(support=supp[:slen.value].copy(), beta=beta, obj=obj.value, rounds=rounds.value)

    def l0l2_comm_init(self, nranks, rank, uid: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(self._lib.l0l2_comm_init(self._ctx, int(nranks), int(rank), C.cast(buf, P)), self._ctx)

    def l0l2_comm_init_transport(self, nranks, rank, transport: HostTransport):
        self._transport = transport   # the callbacks must outlive the context
        _check(self._lib.l0l2_comm_init_transport(self._ctx, int(nranks), int(rank), C.byref(transport.struct)),
               self._ctx)

    def init_distributed(self, transport="nccl"):
        """Attach the current torch.distributed process group: transport "nccl" builds an NCCL
        communicator (one GPU per rank); "host" routes the same exchange through HostTransport
        callbacks on the group (gloo; also several ranks sharing one GPU)."""
        import torch.distributed as dist
        if not dist.is_initialized() or dist.get_world_size() == 1:
            return
        if transport == "host":
            self.l0l2_comm_init_transport(dist.get_world_size(), dist.get_rank(), HostTransport())
            return
        obj = [nccl_unique_id() if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        self.l0l2_comm_init(dist.get_world_size(), dist.get_rank(), obj[0])

    def l0l2_solve(self, gap_tol=1e-2, batch=16, time_limit_s=0.0, node_limit=0, rebalance_every=8,
                   warm_bytes_cap=0, verbose=False, record=False, init_mp=False, early_prune=False, continuous=0,
                   coop_rampup=False):
        so = _SolveOpts()
        self._lib.l0l2_default_solve_opts(C.byref(so))
        so.gap_tol, so.batch, so.time_limit_s = float(gap_tol), int(batch), float(time_limit_s)
        so.node_limit, so.rebalance_every, so.warm_bytes_cap = int(node_limit), int(rebalance_every), int(warm_bytes_cap)
        so.verbose = int(bool(verbose))
        so.record = int(bool(record))
        so.init_mp = int(bool(init_mp))
        so.early_prune = int(bool(early_prune))
        so.continuous = int(continuous)
        so.coop_rampup = int(bool(coop_rampup))
        beta = np.zeros(self.p, dtype=np.float64)
        obj, gap = C.c_double(), C.c_double()
        st = _Stats()
        rc = self._lib.l0l2_solve(self._ctx, C.byref(so), beta.ctypes.data, C.byref(obj), C.byref(gap), C.byref(st))
        _check(rc, self._ctx)
        stats = {f: getattr(st, f) for f, _ in _Stats._fields_}
        out = dict(beta=beta, obj=obj.value, gap=gap.value, support=np.nonzero(beta)[0], stats=stats, rc=rc)
        if record:
            nrec = self._lib.l0l2_solve_trace(self._ctx, None, 0)
            buf = np.zeros((max(1, nrec), 10))
            self._lib.l0l2_solve_trace(self._ctx, buf.ctypes.data, nrec)
            out["trace"] = [dict(id=int(r[0]), depth=int(r[1]), lb=r[2], primal=r[3], iters=int(r[4]),
                                 branch_j=int(r[5]), flags=int(r[6]), ub=r[7], parent=int(r[8]), lastfix=int(r[9]))
                            for r in buf[:nrec]]
        return out


class ShardedProblem:
    """Column-sharded context (l0l2_create_sharded): this rank's columns [col0, col0 + p_r) of X;
    the current torch.distributed group carries the exchange (transport "host": the library's host
    transport over the group, ranks may share a GPU; "nccl": one GPU per rank).  Marshalling only."""

    def __init__(self, X_r, y, col0, p_total, lambda0, lambda2, M, rho=0.0, node_tol=1e-4, int_tol=1e-4,
                 check_every=10, max_iters=10000, device=0, transport="host"):
        import torch.distributed as dist
        self._lib = load_library()
        o = _Opts()
        self._lib.l0l2_default_opts(C.byref(o))
        o.M, o.rho, o.node_tol, o.int_tol = float(M), float(rho), float(node_tol), float(int_tol)
        o.check_every, o.max_iters, o.device = int(check_every), int(max_iters), int(device)
        Xf = np.asfortranarray(X_r, dtype=np.float64)
        yf = np.ascontiguousarray(y, dtype=np.float64)
        self.n, self.p = Xf.shape
        self.col0, self.p_total = int(col0), int(p_total)
        W, R = (dist.get_world_size(), dist.get_rank()) if dist.is_initialized() else (1, 0)
        self._transport, uid = None, None
        if W > 1 and transport == "host":
            self._transport = HostTransport()
        elif W > 1:
            obj = [nccl_unique_id() if R == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        ctx = P()
        rc = self._lib.l0l2_create_sharded(Xf.ctypes.data, yf.ctypes.data, self.n, self.p, self.col0, self.p_total,
                                           float(lambda0), float(lambda2), C.byref(o), W, R,
                                           C.byref(self._transport.struct) if self._transport else None,
                                           C.cast(uid, P) if uid is not None else None, C.byref(ctx))
        if rc != OK:
            raise L0L2Error(rc, self._lib.l0l2_last_error(None).decode(errors="replace"))
        self._ctx = ctx

    def close(self):
        if getattr(self, "_ctx", None):
            self._lib.l0l2_destroy(self._ctx)
            self._ctx = None

    def l0l2_bound_sharded(self, fixings, warm_in=None, parent_lb=None):
        """fixings: list of (F0, F1) with GLOBAL column indices; warm_in: torch CUDA [B, 2, p_r] or None."""
        import torch
        dev = torch.device("cuda", torch.cuda.current_device())
        B = len(fixings)
        off, idx, val = [0], [], []
        for F0, F1 in fixings:
            idx += [int(j) for j in F0] + [int(j) for j in F1]
            val += [0] * len(F0) + [1] * len(F1)
            off.append(len(idx))
        t_off = torch.tensor(off, dtype=torch.int64, device=dev)
        t_idx = torch.tensor(idx or [0], dtype=torch.int32, device=dev)
        t_val = torch.tensor(val or [0], dtype=torch.uint8, device=dev)
        plb = torch.tensor(parent_lb, dtype=torch.float64, device=dev) if parent_lb is not None else None
        lb = torch.empty(B, dtype=torch.float64, device=dev)
        primal = torch.empty_like(lb)
        wout = torch.empty((B, 2, self.p), dtype=torch.float64, device=dev)
        iters = torch.empty(B, dtype=torch.int32, device=dev)
        flags = torch.empty(B, dtype=torch.uint8, device=dev)
        win = warm_in.contiguous() if warm_in is not None else None
        torch.cuda.current_stream().synchronize()
        rc = self._lib.l0l2_bound_sharded(self._ctx, B, _ptr(t_off), _ptr(t_idx), _ptr(t_val), _ptr(win), _ptr(plb),
                                          _ptr(lb), _ptr(primal), _ptr(wout), _ptr(iters), _ptr(flags), None)
        _check(rc, self._ctx)
        torch.cuda.synchronize()
        return dict(lb=lb, primal=primal, warm_out=wout, iters=iters, flags=flags, rc=rc)

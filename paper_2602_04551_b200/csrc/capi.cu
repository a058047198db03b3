// C-ABI entry points of include/l0l2.h (argument checking, data placement, batching).
#include <cmath>
#include <cstdarg>
#include <cstring>

#include <vector>

#include "common.cuh"

namespace l0l2 {

int set_err(Ctx* c, int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

void* dalloc(Ctx* c, size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  c->owned.push_back(p);
  c->bytes += (int64_t)bytes;
  return p;
}

namespace {

__global__ void finite_check(const double* __restrict__ X, int64_t ld, int64_t n, int64_t p, int* bad) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * p) return;
  const double x = X[(e / n) * ld + e % n];
  if (!isfinite(x)) atomicOr(bad, 1);
}

}  // namespace
}  // namespace l0l2

using namespace l0l2;

static thread_local std::string g_last_error;

extern "C" {

void l0l2_default_opts(l0l2_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->M = 0.0;
  o->rho = 0.0;
  o->node_tol = 1e-4;
  o->int_tol = 1e-4;
  o->check_every = 10;
  o->max_iters = 10000;
  o->device = 0;
  o->x_on_device = 0;
}

const char* l0l2_last_error(const l0l2_ctx* ctx) {
  if (ctx) return ctx->impl.err.c_str();
  return g_last_error.c_str();
}

void l0l2_destroy(l0l2_ctx* ctx) {
  if (!ctx) return;
  Ctx* c = &ctx->impl;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (void* p : c->owned) cudaFree(p);
  if (c->ub_scratch) cudaFree(c->ub_scratch);
  for (void* s : c->scr) if (s) cudaFree(s);
  for (double* m : c->pool_chunks) cudaFree(m);
  if (c->solve_buf) cudaFree(c->solve_buf);
  if (c->sh_buf) cudaFree(c->sh_buf);
  if (c->gemm_ws) cudaFree(c->gemm_ws);
  if (c->solve_stream) cudaStreamDestroy(c->solve_stream);
  for (auto e : c->ev) if (e) cudaEventDestroy(e);
  comm_free(c);
  frontier_free(c);
  delete ctx;
}

}  // extern "C"

namespace {
struct ShardCfg {   // column-sharded context (sharded.cu): this rank's columns and its communicator
  int64_t col0, p_total;
  int32_t nranks, rank;
  const l0l2_transport* t;
  const uint8_t* nccl_id;
};

int create_impl(const double* X, const double* y, int64_t n, int64_t p, double lambda0, double lambda2,
                const l0l2_opts* opts, const ShardCfg* sh, l0l2_ctx** out) {
  if (out) *out = nullptr;
  auto fail = [](int code, const char* msg) {
    g_last_error = msg;
    return code;
  };
  if (!X || !y || !opts || !out) return fail(L0L2_EINVAL, "null argument");
  if (n <= 0 || p <= 0) return fail(L0L2_EINVAL, "n, p must be > 0");
  if (!(lambda2 > 0.0) || !std::isfinite(lambda2)) return fail(L0L2_EINVAL, "lambda2 must be > 0 (S:89)");
  if (!(lambda0 >= 0.0) || !std::isfinite(lambda0)) return fail(L0L2_EINVAL, "lambda0 must be >= 0");
  if (!(opts->M > 0.0) || !std::isfinite(opts->M)) return fail(L0L2_EINVAL, "M must be > 0");
  if (!(opts->rho >= 0.0)) return fail(L0L2_EINVAL, "rho must be >= 0");
  if (opts->check_every < 1 || opts->max_iters < 1) return fail(L0L2_EINVAL, "check_every, max_iters >= 1");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) {
    cudaGetLastError();
    return fail(L0L2_ECUDA, "no CUDA device: this library has no CPU fallback");
  }
  if (opts->device < 0 || opts->device >= ndev) return fail(L0L2_EINVAL, "bad device ordinal");
  l0l2_ctx* ctx = new l0l2_ctx();
  Ctx* c = &ctx->impl;
  c->device = opts->device;
  c->n = n;
  c->p = p;
  c->ld = padded_ld(n);
  c->lam0 = lambda0;
  c->lam2 = lambda2;
  c->M = opts->M;
  c->rho = opts->rho;
  c->node_tol = opts->node_tol;
  c->int_tol = opts->int_tol;
  c->check_every = opts->check_every;
  c->max_iters = opts->max_iters;
  if (sh) {
    c->sharded = 1;
    c->col0 = sh->col0;
    c->p_total = sh->p_total;
  }
  int rc = L0L2_OK;
  auto bail = [&](int code) {
    g_last_error = c->err;
    l0l2_destroy(ctx);
    return code;
  };
  if (cudaSetDevice(c->device) != cudaSuccess) return bail(set_err(c, L0L2_ECUDA, "cudaSetDevice"));
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device);
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, c->device);
  if (major < 10) return bail(set_err(c, L0L2_ECUDA, "device is not sm_100 class (built for sm_100a only)"));
  const int64_t ld = c->ld, p8 = round8(p);
  c->X = (double*)dalloc(c, sizeof(double) * ld * p8);
  c->Z = (double*)dalloc(c, sizeof(double) * ld * p8);
  c->y = (double*)dalloc(c, sizeof(double) * ld);
  c->c = (double*)dalloc(c, sizeof(double) * p8);
  c->colsq = (double*)dalloc(c, sizeof(double) * p8);
  c->L = (double*)dalloc(c, sizeof(double) * ld * n);
  c->Lt = (double*)dalloc(c, sizeof(double) * ld * n);
  if (!c->X || !c->Z || !c->y || !c->c || !c->colsq || !c->L || !c->Lt)
    return bail(set_err(c, L0L2_ENOMEM, "device allocation of problem data (%lld bytes)", (long long)c->bytes));
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return bail(set_err(c, L0L2_ECUDA, "stream"));
  auto ck = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess) rc = set_err(c, L0L2_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return e == cudaSuccess;
  };
  bool ok = ck(cudaMemsetAsync(c->X, 0, sizeof(double) * ld * p8, st), "memset X") &&
            ck(cudaMemsetAsync(c->y, 0, sizeof(double) * ld, st), "memset y") &&
            ck(cudaMemsetAsync(c->c, 0, sizeof(double) * p8, st), "memset c") &&
            ck(cudaMemsetAsync(c->colsq, 0, sizeof(double) * p8, st), "memset colsq");
  const cudaMemcpyKind kind = opts->x_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  // device-resident X, y may still be being written on a caller's stream that has no ordering with
  // this library's non-blocking stream: wait for all prior device work before copying them
  if (opts->x_on_device) ok = ok && ck(cudaDeviceSynchronize(), "synchronize before copying device X, y");
  ok = ok && ck(cudaMemcpy2DAsync(c->X, sizeof(double) * ld, X, sizeof(double) * n, sizeof(double) * n, p, kind, st),
                "copy X") &&
       ck(cudaMemcpyAsync(c->y, y, sizeof(double) * n, kind, st), "copy y");
  if (ok) {
    int* bad = (int*)dalloc(c, sizeof(int));
    ok = bad && ck(cudaMemsetAsync(bad, 0, sizeof(int), st), "memset");
    if (ok) {
      const int64_t tot = n * p;
      finite_check<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(c->X, ld, n, p, bad);
      finite_check<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(c->y, n, n, 1, bad);
      c->launches += 2;
      int hb = 0;
      ok = ck(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st), "copy flag") &&
           ck(cudaStreamSynchronize(st), "sync");
      if (ok && hb) {
        rc = set_err(c, L0L2_EINVAL, "NaN/Inf in X or y");
        ok = false;
      }
    }
  }
  if (ok) {
    // direct regime (R17): b = D w with the p×p D when p ≤ 2n and D's tile ring fits
    c->ldD = padded_ld(c->p);
    c->direct = (c->p <= 2 * c->n && c->ldD <= padded_ld(1056)) ? 1 : 0;
    if (const char* e = getenv("L0L2_DIRECT")) c->direct = c->direct && atoi(e) != 0;   // test / tuning hook
    if (sh) {   // the sharded precompute all-reduces XXᵀ over the ranks (Z-form only)
      c->direct = 0;
      if (sh->nranks > 1) {
        rc = sh->t ? l0l2_comm_init_transport(ctx, sh->nranks, sh->rank, sh->t)
                   : l0l2_comm_init(ctx, sh->nranks, sh->rank, sh->nccl_id);
        ok = rc == L0L2_OK;
      }
    }
    if (ok) {
      rc = precompute(c, st);
      ok = rc == L0L2_OK;
    }
  }
  if (ok && !sh) {   // the fused node-parallel kernel
    rc = admm_alloc(c);
    ok = rc == L0L2_OK;
  }
  if (ok && sh) {    // a sharded context runs the same kernel in step mode on its shard when n fits
    c->shard_fused = (admm_alloc(c) == L0L2_OK && !c->wide) ? 1 : 0;
    c->err.clear();
  }
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (!ok) return bail(rc ? rc : L0L2_ECUDA);
  *out = ctx;
  return L0L2_OK;
}

}  // namespace

extern "C" {

int l0l2_create(const double* X, const double* y, int64_t n, int64_t p, double lambda0, double lambda2,
                const l0l2_opts* opts, l0l2_ctx** out) {
  return create_impl(X, y, n, p, lambda0, lambda2, opts, nullptr, out);
}

int l0l2_create_sharded(const double* X_r, const double* y, int64_t n, int64_t p_r, int64_t col0, int64_t p_total,
                        double lambda0, double lambda2, const l0l2_opts* opts, int32_t nranks, int32_t rank,
                        const l0l2_transport* t, const uint8_t nccl_id[128], l0l2_ctx** out) {
  if (out) *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks || col0 < 0 || p_r <= 0 || col0 + p_r > p_total ||
      (nranks > 1 && !t && !nccl_id)) {
    g_last_error = "l0l2_create_sharded: bad shard / communicator arguments";
    return L0L2_EINVAL;
  }
  const ShardCfg sh{col0, p_total, nranks, rank, t, nccl_id};
  return create_impl(X_r, y, n, p_r, lambda0, lambda2, opts, &sh, out);
}

int l0l2_bound_sharded(l0l2_ctx* ctx, int32_t B, const int64_t* fix_off, const int32_t* fix_idx,
                       const uint8_t* fix_val, const double* warm_in, const double* parent_lb, double* lb,
                       double* primal, double* warm_out, int32_t* iters, uint8_t* flags, void* stream) {
  if (!ctx) return L0L2_EINVAL;
  Ctx* c = &ctx->impl;
  if (!c->sharded) return set_err(c, L0L2_EINVAL, "not a column-sharded context (l0l2_create_sharded)");
  if (B < 0 || B > 128) return set_err(c, L0L2_EINVAL, "0 <= B <= 128");
  if (B == 0) return L0L2_OK;
  if (!lb || !primal || !iters || !flags) return set_err(c, L0L2_EINVAL, "null output");
  L0L2_CUDA(c, cudaSetDevice(c->device));
  return bound_sharded(c, B, fix_off, fix_idx, fix_val, warm_in, parent_lb, lb, primal, warm_out, iters, flags,
                       (cudaStream_t)stream);
}

int l0l2_info(const l0l2_ctx* ctx, int64_t* n, int64_t* p, double* rho, int64_t* device_bytes, int64_t* launches) {
  if (!ctx) return L0L2_EINVAL;
  const Ctx* c = &ctx->impl;
  if (n) *n = c->n;
  if (p) *p = c->p;
  if (rho) *rho = c->rho;
  if (device_bytes) {
    // everything the context holds on the device: problem data and ADMM work space, the growable
    // batch I/O scratch, the solve's round buffers and the warm-state pool chunks (all kept until
    // l0l2_destroy, so this is also the peak)
    int64_t b = c->bytes;
    for (size_t s : c->scr_bytes) b += (int64_t)s;
    b += (int64_t)c->solve_buf_bytes;
    b += (int64_t)c->pool_chunks.size() * c->pool_chunk_bytes;
    *device_bytes = b;
  }
  if (launches) *launches = c->launches;
  return L0L2_OK;
}

int l0l2_admm_path(const l0l2_ctx* ctx) {
  if (!ctx) return L0L2_EINVAL;
  const Ctx* c = &ctx->impl;
  return c->wide ? 2 : (c->direct ? 1 : 0);
}

int l0l2_bound_batch(l0l2_ctx* ctx, int32_t B, const int64_t* fix_off, const int32_t* fix_idx,
                     const uint8_t* fix_val, const double* warm_in, const double* parent_lb, double* lb,
                     double* primal, double* warm_out, double* zhat, double* dual_r, int32_t* branch_j,
                     int32_t* iters, uint8_t* flags, void* stream) {
  if (!ctx) return L0L2_EINVAL;
  Ctx* c = &ctx->impl;
  if (B < 0) return set_err(c, L0L2_EINVAL, "B < 0");
  if (B == 0) return L0L2_OK;
  if (!lb || !primal || !branch_j || !iters || !flags) return set_err(c, L0L2_EINVAL, "null output");
  if (!fix_off && (fix_idx || fix_val)) return set_err(c, L0L2_EINVAL, "fix_idx without fix_off");
  L0L2_CUDA(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t p = c->p;
  // device scratch: warm pointer table, support compaction (unused here), per-group pointers
  double** wptr = (double**)c->scratch(sizeof(double*) * 2 * kBC);
  int32_t* scnt = (int32_t*)c->scratch2(sizeof(int32_t) * kBC + sizeof(int32_t) * kBC * p);
  if (!wptr || !scnt) return set_err(c, L0L2_ENOMEM, "scratch");
  int32_t* sidx = scnt + kBC;
  bool notconv = false;
  for (int g0 = 0; g0 < B; g0 += kBC) {
    const int nb = std::min(kBC, B - g0);
    const double* hin[kBC] = {};
    double* hout[kBC] = {};
    for (int k = 0; k < nb; k++) {
      hin[k] = warm_in ? warm_in + (int64_t)(g0 + k) * 2 * p : nullptr;
      hout[k] = warm_out ? warm_out + (int64_t)(g0 + k) * 2 * p : nullptr;
    }
    L0L2_CUDA(c, cudaMemcpyAsync(wptr, hin, sizeof(hin), cudaMemcpyHostToDevice, st));
    L0L2_CUDA(c, cudaMemcpyAsync(wptr + kBC, hout, sizeof(hout), cudaMemcpyHostToDevice, st));
    int rc = pack_group(c, nb, fix_off ? fix_off + g0 : nullptr, fix_idx, fix_val, (const double* const*)wptr, st);
    if (rc) return rc;
    BoundArgs a{nb, parent_lb ? parent_lb + g0 : nullptr, lb + g0, primal + g0, iters + g0, flags + g0};
    for (int k = 0; k < nb; k++) if (!hin[k]) a.cold_mask |= 1u << k;
    rc = run_admm(c, a, st);
    if (rc) return rc;
    rc = finalize_group(c, nb, zhat ? zhat + (int64_t)g0 * p : nullptr, branch_j + g0, flags + g0, scnt, sidx, p, st);
    if (rc) return rc;
    if (warm_out) {
      rc = unpack_warm(c, nb, wptr + kBC, st);
      if (rc) return rc;
    }
    if (dual_r) {
      rc = dual_residual(c, nb, dual_r + (int64_t)g0 * c->n, c->n, st);
      if (rc) return rc;
    }
    uint8_t hf[kBC];
    int32_t hit[kBC];
    L0L2_CUDA(c, cudaMemcpyAsync(hf, flags + g0, nb, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaMemcpyAsync(hit, iters + g0, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    rc = account_admm(c, nb, hit);
    if (rc) return rc;
    for (int k = 0; k < nb; k++) notconv |= (hf[k] & L0L2_FLAG_MAXITER) != 0;
  }
  return notconv ? L0L2_WNOTCONV : L0L2_OK;
}

// developer instrumentation (only populated in -DL0L2_PROF builds; not part of include/l0l2.h)
int l0l2_debug_prof(unsigned long long* out, int32_t reset) { return debug_prof(out, reset); }

int l0l2_kernel_stats(l0l2_ctx* ctx, l0l2_kstats* out, int32_t reset) {
  if (!ctx) return L0L2_EINVAL;
  Ctx* c = &ctx->impl;
  if (out) *out = c->ks;
  if (reset) c->ks = l0l2_kstats{};
  return L0L2_OK;
}

int l0l2_upper_batch(l0l2_ctx* ctx, int32_t B, const int64_t* supp_off, const int32_t* supp_idx, double* obj,
                     double* beta_s, void* stream) {
  if (!ctx) return L0L2_EINVAL;
  Ctx* c = &ctx->impl;
  if (B < 0 || (B > 0 && (!supp_off || !obj))) return set_err(c, L0L2_EINVAL, "bad arguments");
  L0L2_CUDA(c, cudaSetDevice(c->device));
  int rc = upper_batch(c, B, supp_off, supp_idx, obj, beta_s, (cudaStream_t)stream);
  if (rc) return rc;
  L0L2_CUDA(c, cudaStreamSynchronize((cudaStream_t)stream));
  return L0L2_OK;
}

int l0l2_matching_pursuit(l0l2_ctx* ctx, int32_t max_rounds, double* beta, int32_t* support, int32_t* support_len,
                          double* obj, int32_t* rounds) {
  if (!ctx) return L0L2_EINVAL;
  Ctx* c = &ctx->impl;
  if (!beta || !support || !support_len || !obj) return set_err(c, L0L2_EINVAL, "bad arguments");
  L0L2_CUDA(c, cudaSetDevice(c->device));
  std::vector<int32_t> S;
  std::vector<double> b;
  int r = 0;
  int rc = mp_run(c, max_rounds, nullptr, S, b, obj, &r);
  if (rc) return rc;
  std::memcpy(beta, b.data(), sizeof(double) * c->p);
  if (!S.empty()) std::memcpy(support, S.data(), sizeof(int32_t) * S.size());
  *support_len = (int32_t)S.size();
  if (rounds) *rounds = r;
  return L0L2_OK;
}

}  // extern "C"

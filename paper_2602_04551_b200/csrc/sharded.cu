// Column-sharded single-node ADMM for the narrow-frontier phases of the tree
// (the root, the ramp-up, C2/C3-class trees with few open nodes), where node parallelism leaves
// GPUs idle.  Rank r of W holds columns [col0, col0 + p_r) of X; the precompute all-reduces
// A = Σ_r X_r X_rᵀ + ρI, every rank factors A = LLᵀ and keeps Z_r = L⁻¹X_r.  One ADMM
// iteration of B nodes (the paper's b-update through Xw / Xᵀt; the Z-form of DESIGN.md §4):
//   u_r = Z_r w_r  (n × B, local DMMA GEMM)  →  u = Σ_r u_r  (all-reduce: the one exchange)
//   s_r = Z_rᵀ u   (p_r × B, local)          →  b = (w − s)/ρ, β⁺ = prox(b + v/ρ), v⁺, w⁺ (local)
// and at checks the per-node sums of the dual / primal terms plus X_r β⁺
// (for ‖Xβ‖²) are all-reduced in one buffer; every rank takes the same decisions from the same
// sums.  The exchange is NCCL (`ncclAllReduce`, one GPU per rank over NVLink) or the caller's host
// transport (all-gather + a fixed rank-order sum: several ranks may share one GPU, as in the tests).
// This is a host-stepped loop of library kernels (two GEMMs, an epilogue, a decision kernel per
// iteration): unlike the fused persistent kernel it reads Z_r twice per iteration, and each
// iteration pays one all-reduce latency — the price of splitting one node over W GPUs.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace l0l2 {
namespace {

struct SP {   // scalars of the node relaxation (eq:minbetalower, eq:psi, eq:nudef2)
  double rho, inv_rho, lam0, lam2, M, yy, node_tol;
  double shrink, sr, a_l1, a_4, psi_l1, psi_4;
  bool sr_le_M;
};

__device__ __forceinline__ double Tbox(double t, double a, double m) {   // eq:Tdef
  const double at = fabs(t);
  if (at <= a) return 0.0;
  if (at <= a + m) return copysign(at - a, t);
  return copysign(m, t);
}
__device__ __forceinline__ double prox(const SP& k, double bt, uint8_t code) {   // eq:minbetalower
  if (code == 1) return 0.0;
  const double quad = Tbox(k.shrink * bt, 0.0, k.M);
  if (code == 2) return quad;
  if (k.sr_le_M) return fabs(bt) >= k.a_l1 + k.sr ? quad : Tbox(bt, k.a_l1, k.M);
  return Tbox(bt, k.a_4, k.M);
}
__device__ __forceinline__ double psi_f(const SP& k, double b, uint8_t code) {   // eq:psi
  const double ab = fabs(b);
  if (code == 1) return b == 0.0 ? 0.0 : INFINITY;
  if (ab > k.M) return INFINITY;
  if (code == 2) return k.lam0 + k.lam2 * b * b;
  if (k.sr_le_M) return ab >= k.sr ? k.lam0 + k.lam2 * b * b : k.psi_l1 * ab;
  return k.psi_4 * ab;
}
__device__ __forceinline__ double h_f(const SP& k, double x) {                    // eq:hdef
  return x <= 2.0 * k.M * k.lam2 ? x * x / (4.0 * k.lam2) - k.lam0 : k.M * x - k.lam0 - k.lam2 * k.M * k.M;
}
__device__ __forceinline__ double nu_f(const SP& k, double x, uint8_t code) {     // eq:nudef2
  if (code == 1) return 0.0;
  if (code == 2) return h_f(k, x);
  if (k.sr_le_M) return fmax(h_f(k, x), 0.0);
  return fmax(k.M * x - k.lam0 - k.lam2 * k.M * k.M, 0.0);
}

constexpr int NT = 256;   // threads of the per-node kernels (one CTA per node, fixed-order sums)

// codes and state of node k on this rank's columns: fixings (GLOBAL indices) outside
// [col0, col0 + pr) belong to other ranks; warm edit β_F0 = 0
__global__ void sh_init(int64_t pr, int64_t col0, const int64_t* __restrict__ off, const int32_t* __restrict__ idx,
                        const uint8_t* __restrict__ val, const double* __restrict__ warm, uint8_t* code, double* beta,
                        double* v) {
  const int k = blockIdx.x;
  for (int64_t j = threadIdx.x; j < pr; j += blockDim.x) {
    code[k * pr + j] = 0;
    beta[k * pr + j] = warm ? warm[(int64_t)k * 2 * pr + j] : 0.0;
    v[k * pr + j] = warm ? warm[(int64_t)k * 2 * pr + pr + j] : 0.0;
  }
  __syncthreads();
  if (off && threadIdx.x == 0)
    for (int64_t q = off[k]; q < off[k + 1]; q++) {
      const int64_t j = (int64_t)idx[q] - col0;
      if (j < 0 || j >= pr) continue;
      code[k * pr + j] = val[q] ? 2 : 1;
      if (!val[q]) beta[k * pr + j] = 0.0;
    }
}

// w = c + ρβ − v (the b-update's right-hand side, eq:b_update)
__global__ void sh_w(int64_t pr, int B, const double* __restrict__ c, const double* __restrict__ beta,
                     const double* __restrict__ v, double rho, double* w) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= pr * B) return;
  w[e] = c[e % pr] + rho * beta[e] - v[e];
}

// b = (w − s)/ρ, then (refresh: warm nodes' v only) or (β⁺ = prox(b + v/ρ), v⁺ = v + ρ(b − β⁺));
// per-node partial check terms of this rank's columns in a fixed order: Σ b·s, Σ ν(|c − s|),
// Σ c·β⁺, Σ ψ(β⁺) (Xᵀr̂ = c − s and ‖Xb‖² = bᵀs)
__global__ void sh_epilogue(SP k, int64_t pr, const double* __restrict__ c, const uint8_t* __restrict__ code,
                            const double* __restrict__ w, const double* __restrict__ s, double* beta, double* v,
                            const uint8_t* __restrict__ active, const uint8_t* __restrict__ cold, int refresh,
                            double* terms) {
  const int nd = blockIdx.x;
  __shared__ double red[4][NT / 32];
  double t1 = 0.0, t2 = 0.0, t3 = 0.0, t4 = 0.0;
  const bool act = active[nd] != 0;
  for (int64_t j = threadIdx.x; j < pr; j += blockDim.x) {
    const int64_t e = (int64_t)nd * pr + j;
    const uint8_t cd = code[e];
    const double b = (w[e] - s[e]) * k.inv_rho;
    double bn = beta[e], vn = v[e];
    if (act) {
      if (refresh) {
        if (!cold[nd]) vn = v[e] + k.rho * (b - beta[e]);
      } else {
        bn = prox(k, b + v[e] * k.inv_rho, cd);
        vn = v[e] + k.rho * (b - bn);
      }
      beta[e] = bn;
      v[e] = vn;
    }
    t1 = fma(b, s[e], t1);
    t2 += nu_f(k, fabs(c[j] - s[e]), cd);
    t3 = fma(c[j], bn, t3);
    t4 += psi_f(k, bn, cd);
  }
  double vals[4] = {t1, t2, t3, t4};
  for (int q = 0; q < 4; q++) {
    for (int o = 16; o > 0; o >>= 1) vals[q] += __shfl_xor_sync(0xffffffffu, vals[q], o);
    if ((threadIdx.x & 31) == 0) red[q][threadIdx.x >> 5] = vals[q];
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double a = 0.0;
    for (int wq = 0; wq < NT / 32; wq++) a += red[threadIdx.x][wq];
    terms[nd * 4 + threadIdx.x] = a;
  }
}

// decisions from the all-reduced sums (identical on every rank): dual at r̂ = y − X b̂,
// primal P(β), running max of the duals (R7), stop rule (R8)
__global__ void sh_decide(SP k, int B, int64_t n, int64_t ldx, const double* __restrict__ terms,
                          const double* __restrict__ xb, int it, int last, double* lbb, double* primal, uint8_t* active,
                          uint8_t* flags, int32_t* iters) {
  const int nd = blockIdx.x;
  __shared__ double red[NT / 32];
  double q = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) q = fma(xb[nd * ldx + i], xb[nd * ldx + i], q);
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = q;
  __syncthreads();
  if (threadIdx.x != 0 || !active[nd]) return;
  double xx = 0.0;
  for (int wq = 0; wq < NT / 32; wq++) xx += red[wq];
  const double* T = terms + nd * 4;
  const double dual = 0.5 * k.yy - 0.5 * T[0] - T[1];
  const double pr = 0.5 * k.yy - T[2] + 0.5 * xx + T[3];
  const double lb = fmax(lbb[nd], dual);
  lbb[nd] = lb;
  primal[nd] = pr;
  iters[nd] = it;
  if ((pr - lb) / fmax(1.0, fabs(pr)) <= k.node_tol) { active[nd] = 0; flags[nd] = L0L2_FLAG_CONVERGED; }
  else if (last) { active[nd] = 0; flags[nd] = L0L2_FLAG_MAXITER; }
}

__global__ void sh_out(int B, int64_t pr, const double* __restrict__ lbb, const double* __restrict__ plb,
                       const double* __restrict__ beta, const double* __restrict__ v, double* lb, double* warm_out) {
  const int k = blockIdx.x;
  if (threadIdx.x == 0) lb[k] = fmax(lbb[k], plb ? plb[k] : -INFINITY);
  if (warm_out)
    for (int64_t j = threadIdx.x; j < pr; j += blockDim.x) {
      warm_out[(int64_t)k * 2 * pr + j] = beta[k * pr + j];
      warm_out[(int64_t)k * 2 * pr + pr + j] = v[k * pr + j];
    }
}

__global__ void sh_init_nodes(int B, const double* warm_in_flag_src, uint8_t* active, uint8_t* cold, double* lbb,
                              uint8_t* flags, int32_t* iters, int has_warm) {
  const int k = threadIdx.x;
  if (k >= B) return;
  active[k] = 1;
  cold[k] = has_warm ? 0 : 1;
  lbb[k] = -INFINITY;
  flags[k] = 0;
  iters[k] = 0;
  (void)warm_in_flag_src;
}

}  // namespace

// Fused variant: the persistent ADMM kernel on this rank's column shard in STEP mode (one phase per
// launch: the u0 sweep, the refresh sweep, then one fused adjoint + epilogue + forward iteration per
// launch), U = Σ_r Z_r w_r all-reduced between launches, and at checks the rank's check totals and
// Z_r β⁺ all-reduced before a decision kernel (admm.cu step_decide).  Z_r is read once per iteration.
int bound_sharded_fused(Ctx* c, int B, const int64_t* fix_off, const int32_t* fix_idx, const uint8_t* fix_val,
                        const double* warm_in, const double* parent_lb, double* lb, double* primal, double* warm_out,
                        int32_t* iters, uint8_t* flags, cudaStream_t st) {
  const int64_t pr = c->p;
  // fixings (GLOBAL column indices) → this rank's local columns
  std::vector<int64_t> off(B + 1, 0), loff(B + 1, 0);
  std::vector<int32_t> idx, lidx;
  std::vector<uint8_t> val, lval;
  if (fix_off) {
    L0L2_CUDA(c, cudaMemcpyAsync(off.data(), fix_off, sizeof(int64_t) * (B + 1), cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    idx.resize(off[B]);
    val.resize(off[B]);
    if (off[B] > 0) {
      L0L2_CUDA(c, cudaMemcpyAsync(idx.data(), fix_idx, sizeof(int32_t) * off[B], cudaMemcpyDeviceToHost, st));
      L0L2_CUDA(c, cudaMemcpyAsync(val.data(), fix_val, off[B], cudaMemcpyDeviceToHost, st));
      L0L2_CUDA(c, cudaStreamSynchronize(st));
    }
    for (int k = 0; k < B; k++) {
      for (int64_t q = off[k]; q < off[k + 1]; q++) {
        const int64_t j = (int64_t)idx[q] - c->col0;
        if (idx[q] < 0 || idx[q] >= c->p_total) return set_err(c, L0L2_EINVAL, "fixing index out of range");
        if (j < 0 || j >= pr) continue;
        lidx.push_back((int32_t)j);
        lval.push_back(val[q]);
      }
      loff[k + 1] = (int64_t)lidx.size();
    }
  }
  int64_t* d_off = (int64_t*)c->scratch_n(2, sizeof(int64_t) * (B + 1) + sizeof(double) * kBC * 4 + 64);
  int32_t* d_idx = (int32_t*)c->scratch_n(3, sizeof(int32_t) * std::max<size_t>(1, lidx.size()));
  uint8_t* d_val = (uint8_t*)c->scratch_n(4, std::max<size_t>(1, lval.size()));
  double** wptr = (double**)c->scratch_n(5, sizeof(double*) * 2 * kBC);
  if (!d_off || !d_idx || !d_val || !wptr) return set_err(c, L0L2_ENOMEM, "sharded scratch");
  double* tot = (double*)((char*)d_off + ((sizeof(int64_t) * (B + 1) + 63) / 64) * 64);
  L0L2_CUDA(c, cudaMemcpyAsync(d_off, loff.data(), sizeof(int64_t) * (B + 1), cudaMemcpyHostToDevice, st));
  if (!lidx.empty()) {
    L0L2_CUDA(c, cudaMemcpyAsync(d_idx, lidx.data(), sizeof(int32_t) * lidx.size(), cudaMemcpyHostToDevice, st));
    L0L2_CUDA(c, cudaMemcpyAsync(d_val, lval.data(), lval.size(), cudaMemcpyHostToDevice, st));
  }
  bool notconv = false;
  int rc = L0L2_OK;
  for (int g0 = 0; g0 < B; g0 += kBC) {
    const int nb = std::min(kBC, B - g0);
    const double* hin[kBC] = {};
    double* hout[kBC] = {};
    for (int k = 0; k < nb; k++) {
      hin[k] = warm_in ? warm_in + (int64_t)(g0 + k) * 2 * pr : nullptr;
      hout[k] = warm_out ? warm_out + (int64_t)(g0 + k) * 2 * pr : nullptr;
    }
    L0L2_CUDA(c, cudaMemcpyAsync(wptr, hin, sizeof(hin), cudaMemcpyHostToDevice, st));
    L0L2_CUDA(c, cudaMemcpyAsync(wptr + kBC, hout, sizeof(hout), cudaMemcpyHostToDevice, st));
    if ((rc = pack_group(c, nb, fix_off ? d_off + g0 : nullptr, d_idx, d_val, (const double* const*)wptr, st))) return rc;
    BoundArgs a{nb, parent_lb ? parent_lb + g0 : nullptr, lb + g0, primal + g0, iters + g0, flags + g0};
    if (!warm_in) a.cold_mask = (1u << nb) - 1u;
    const int64_t ucount = (int64_t)kBC * c->ld;
    if ((rc = admm_step(c, a, 0, 0, tot, st)) || (rc = shard_allreduce(c, c->U, ucount, st))) return rc;
    if (warm_in && ((rc = admm_step(c, a, 1, 0, tot, st)) || (rc = shard_allreduce(c, c->U, ucount, st)))) return rc;
    int hfl[2 * kBC];
    for (int it = 1; it <= c->max_iters; it++) {
      const int chk = (it % c->check_every == 0) || it == c->max_iters;
      if ((rc = admm_step(c, a, 2, chk, tot, st)) || (rc = shard_allreduce(c, c->U, ucount, st))) return rc;
      if (!chk) continue;
      if ((rc = shard_allreduce(c, tot, kBC * 4, st)) || (rc = shard_allreduce(c, c->Ub, ucount, st)) ||
          (rc = admm_step_decide(c, a, it, tot, st)))
        return rc;
      L0L2_CUDA(c, cudaMemcpyAsync(hfl, c->node_i, sizeof(hfl), cudaMemcpyDeviceToHost, st));
      L0L2_CUDA(c, cudaStreamSynchronize(st));
      bool any = false;
      for (int k = 0; k < nb; k++) any |= (hfl[2 * k] & 64) != 0;   // F_ACTIVE (admm.cu)
      if (!any) break;
    }
    if ((rc = admm_step_outputs(c, a, st))) return rc;
    if (warm_out && (rc = unpack_warm(c, nb, wptr + kBC, st))) return rc;
    uint8_t hf[kBC];
    L0L2_CUDA(c, cudaMemcpyAsync(hf, flags + g0, nb, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    for (int k = 0; k < nb; k++) notconv |= (hf[k] & L0L2_FLAG_MAXITER) != 0;
  }
  return notconv ? L0L2_WNOTCONV : L0L2_OK;
}

// Column-sharded bound of B nodes (see the file header).  Device pointers, ordered on `stream`.
int bound_sharded(Ctx* c, int B, const int64_t* fix_off, const int32_t* fix_idx, const uint8_t* fix_val,
                  const double* warm_in, const double* parent_lb, double* lb, double* primal, double* warm_out,
                  int32_t* iters, uint8_t* flags, cudaStream_t st) {
  const char* eg = getenv("L0L2_SHARD_GEMM");   // test hook: the unfused GEMM loop below
  if (c->shard_fused && !(eg && atoi(eg) != 0))
    return bound_sharded_fused(c, B, fix_off, fix_idx, fix_val, warm_in, parent_lb, lb, primal, warm_out, iters,
                               flags, st);
  const int64_t pr = c->p, n = c->n, ld = c->ld;
  // work space: code, β, v, w, s (B × pr), u / Xβ (B × ld), terms (B × 4) + Xβ (B × ld) exchange block
  const size_t need = (size_t)B * pr * (1 + 8 * 4) + sizeof(double) * ((size_t)B * ld * 2 + (size_t)B * 4) + 64 * B + 4096;
  if (c->sh_bytes < need) {
    if (c->sh_buf) cudaFree(c->sh_buf);
    c->sh_buf = nullptr;
    c->sh_bytes = 0;
    if (cudaMalloc(&c->sh_buf, need) != cudaSuccess) { cudaGetLastError(); return set_err(c, L0L2_ENOMEM, "sharded work space"); }
    c->sh_bytes = need;
  }
  char* cur = (char*)c->sh_buf;
  auto A = [&](size_t b) { char* r = cur; cur += (b + 255) / 256 * 256; return r; };
  double* beta = (double*)A(sizeof(double) * B * pr);
  double* v = (double*)A(sizeof(double) * B * pr);
  double* w = (double*)A(sizeof(double) * B * pr);
  double* s = (double*)A(sizeof(double) * B * pr);
  double* u = (double*)A(sizeof(double) * B * ld);
  double* ex = (double*)A(sizeof(double) * ((size_t)B * 4 + (size_t)B * ld));   // [terms B×4 | Xβ B×ld]
  uint8_t* code = (uint8_t*)A((size_t)B * pr);
  uint8_t* active = (uint8_t*)A(B);
  uint8_t* cold = (uint8_t*)A(B);
  double* lbb = (double*)A(sizeof(double) * B);
  double* terms = ex;
  double* xb = ex + (size_t)B * 4;
  SP k{};
  k.rho = c->rho; k.inv_rho = 1.0 / c->rho; k.lam0 = c->lam0; k.lam2 = c->lam2; k.M = c->M; k.yy = c->yy;
  k.node_tol = c->node_tol;
  k.shrink = c->rho / (c->rho + 2.0 * c->lam2);
  k.sr = std::sqrt(c->lam0 / c->lam2);
  k.sr_le_M = k.sr <= c->M;
  k.a_l1 = 2.0 * std::sqrt(c->lam0 * c->lam2) / c->rho;
  k.a_4 = c->lam0 / (c->M * c->rho) + c->lam2 * c->M / c->rho;
  k.psi_l1 = 2.0 * std::sqrt(c->lam0 * c->lam2);
  k.psi_4 = c->lam0 / c->M + c->lam2 * c->M;
  sh_init<<<B, NT, 0, st>>>(pr, c->col0, fix_off, fix_idx, fix_val, warm_in, code, beta, v);
  sh_init_nodes<<<1, 128, 0, st>>>(B, warm_in, active, cold, lbb, flags, iters, warm_in != nullptr);
  c->launches += 2;
  const unsigned gw = (unsigned)((pr * B + 255) / 256);
  auto half_iteration = [&](int refresh) -> int {   // u = Σ_r Z_r w_r; s = Z_rᵀ u; epilogue
    sh_w<<<gw, 256, 0, st>>>(pr, B, c->c, beta, v, c->rho, w);
    L0L2_LAUNCHED(c);
    int rc = gemm_f64(c, n, B, pr, 1.0, c->Z, ld, false, w, pr, false, 0.0, u, ld, st);
    if (rc) return rc;
    if ((rc = shard_allreduce(c, u, (int64_t)B * ld, st))) return rc;
    if ((rc = gemm_f64(c, pr, B, n, 1.0, c->Z, ld, true, u, ld, false, 0.0, s, pr, st))) return rc;
    sh_epilogue<<<B, NT, 0, st>>>(k, pr, c->c, code, w, s, beta, v, active, cold, refresh, terms);
    L0L2_LAUNCHED(c);
    return L0L2_OK;
  };
  // warm start (R6): the refresh of b and v; cold nodes start at (0, 0) unchanged
  int rc = L0L2_OK;
  if (warm_in && (rc = half_iteration(1))) return rc;
  std::vector<uint8_t> hact(B);
  bool notconv = false;
  for (int it = 1; it <= c->max_iters; it++) {
    if ((rc = half_iteration(0))) return rc;
    const bool chk = it % c->check_every == 0 || it == c->max_iters;
    if (!chk) continue;
    // ‖Xβ‖²: X_r β⁺ (local) joins the check terms in ONE all-reduce
    if ((rc = gemm_f64(c, n, B, pr, 1.0, c->X, ld, false, beta, pr, false, 0.0, xb, ld, st))) return rc;
    if ((rc = shard_allreduce(c, ex, (int64_t)B * 4 + (int64_t)B * ld, st))) return rc;
    sh_decide<<<B, NT, 0, st>>>(k, B, n, ld, terms, xb, it, it == c->max_iters, lbb, primal, active, flags, iters);
    L0L2_LAUNCHED(c);
    L0L2_CUDA(c, cudaMemcpyAsync(hact.data(), active, B, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    bool any = false;
    for (int q = 0; q < B; q++) any |= hact[q] != 0;
    if (!any) break;
  }
  sh_out<<<B, NT, 0, st>>>(B, pr, lbb, parent_lb, beta, v, lb, warm_out);
  L0L2_LAUNCHED(c);
  std::vector<uint8_t> hf(B);
  L0L2_CUDA(c, cudaMemcpyAsync(hf.data(), flags, B, cudaMemcpyDeviceToHost, st));
  L0L2_CUDA(c, cudaStreamSynchronize(st));
  for (int q = 0; q < B; q++) notconv |= (hf[q] & L0L2_FLAG_MAXITER) != 0;
  return notconv ? L0L2_WNOTCONV : L0L2_OK;
}

}  // namespace l0l2

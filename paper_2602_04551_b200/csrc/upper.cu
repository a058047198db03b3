// Batched upper bound on candidate supports (§3.3-§3.4).
//
// For each support S (one warp per support) minimise eq:upperboundbeta
//     U_S(β) = ½‖y − X_Sβ‖² + λ2‖β‖²   s.t. |β_i| ≤ M
// by the paper's fast proximal gradient method: Nesterov extrapolation t/(t+3)
// (eq:fpg_extrapolate), gradient (eq:fpg_grad), box projection (eq:fpg_step) and Armijo
// backtracking (eq:fpg_armijo).  B200 form: the Gram matrix
// Q = X_SᵀX_S + 2λ2I and q = X_Sᵀy = c_S are formed once per support in shared memory, so each
// iteration works in s-space:  ∇ = Qβ̃ − q,  U_S(β) = ½‖y‖² − qᵀβ + ½βᵀQβ.  These are the same
// iterates as the paper's masked dense form in exact arithmetic.
#include <cmath>

#include "common.cuh"

namespace l0l2 {
namespace {

constexpr int kRC = 32;   // rows of X_S staged per Gram chunk

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
// several independent sums in one butterfly (the shuffle latencies overlap)
template <int K>
__device__ __forceinline__ void warp_sum_k(double (&x)[K]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < K; i++) x[i] += __shfl_xor_sync(0xffffffffu, x[i], o);
}
__device__ __forceinline__ double warp_max(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// Gram pre-pass: one CTA of nw warps per support; warp w accumulates Q = X_SᵀX_S over the row
// chunks w, w + nw, ... (kRC rows each, staged in its shared slice), then the nw partials are summed
// in warp order and 2λ2 added on the diagonal; Q (symmetric, s×s) → Qout[nd].  The X_S gather is
// spread over nw warps instead of one (the FPG iterations themselves run on one warp).
__global__ void __launch_bounds__(256) gram_kernel(const double* __restrict__ X, int64_t ld, int64_t n, double lam2,
                                                  const int64_t* __restrict__ off, const int32_t* __restrict__ idx,
                                                  double* __restrict__ Qout, int64_t qstride) {
  extern __shared__ double sm[];
  const int nd = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t o0 = off[nd];
  const int s = (int)(off[nd + 1] - o0);
  if (s == 0) return;
  const int32_t* S = idx + o0;
  double* Qp = sm + (int64_t)warp * (s * s + kRC * s);   // this warp's partial, then its staging
  double* Xc = Qp + s * s;
  for (int e = lane; e < s * s; e += 32) Qp[e] = 0.0;
  __syncwarp();
  for (int64_t r0 = (int64_t)warp * kRC; r0 < n; r0 += (int64_t)nw * kRC) {
    const int rr = (int)((n - r0) < kRC ? (n - r0) : kRC);
    for (int e = lane; e < rr * s; e += 32) {
      const int a = e / rr, r = e % rr;
      Xc[r * s + a] = X[(int64_t)S[a] * ld + r0 + r];
    }
    __syncwarp();
    for (int e = lane; e < s * s; e += 32) {
      const int a = e / s, b = e % s;
      if (b < a) continue;
      double acc = Qp[a * s + b];
      for (int r = 0; r < rr; r++) acc = fma(Xc[r * s + a], Xc[r * s + b], acc);
      Qp[a * s + b] = acc;
    }
    __syncwarp();
  }
  __syncthreads();
  double* Q = Qout + (int64_t)nd * qstride;
  for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
    const int a = e / s, b = e % s;
    const int u = a <= b ? a * s + b : b * s + a;   // upper-triangle entry
    double v = 0.0;
    for (int w = 0; w < nw; w++) v += sm[(int64_t)w * (s * s + kRC * s) + u];
    Q[e] = v + (a == b ? 2.0 * lam2 : 0.0);
  }
}

// one warp (one CTA) per support
__global__ void __launch_bounds__(32) fpg_kernel(const double* __restrict__ X, int64_t ld, int64_t n,
                                                 const double* __restrict__ y, const double* __restrict__ c,
                                                 double yy, double lam0, double lam2, double M,
                                                 const int64_t* __restrict__ off, const int32_t* __restrict__ idx,
                                                 double* __restrict__ obj, double* __restrict__ beta_s,
                                                 double* __restrict__ Qglobal, int64_t qstride, int smax_smem,
                                                 int max_iters, const double* __restrict__ Qpre) {
  extern __shared__ double sm[];
  const int nd = blockIdx.x, lane = threadIdx.x;
  const int64_t o0 = off[nd];
  const int s = (int)(off[nd + 1] - o0);
  if (s == 0) {
    if (lane == 0) obj[nd] = 0.5 * yy;
    return;
  }
  const int32_t* S = idx + o0;
  double* Q = (s <= smax_smem) ? sm : Qglobal + (int64_t)nd * qstride;
  double* vec = (s <= smax_smem) ? sm + (int64_t)s * s : sm;      // 6 vectors of length s
  double* q = vec;
  double* bb = vec + s;       // β^t
  double* bp = vec + 2 * s;   // β^{t−1}
  double* bt = vec + 3 * s;   // β̃
  double* g = vec + 4 * s;    // ∇
  double* bn = vec + 5 * s;   // trial β^{t+1}
  double* Xc = vec + 6 * s;   // [kRC][s] staging of X_S rows

  // ---- Gram Q = X_SᵀX_S + 2λ2 I: from the multi-warp pre-pass, or staged kRC rows at a time here
  if (Qpre) {
    const double* Qs = Qpre + (int64_t)nd * qstride;
    if (s <= smax_smem) {
      for (int e = lane; e < s * s; e += 32) Q[e] = Qs[e];
    } else {
      Q = const_cast<double*>(Qs);
    }
  } else {
  for (int e = lane; e < s * s; e += 32) Q[e] = 0.0;
  __syncwarp();
  for (int64_t r0 = 0; r0 < n; r0 += kRC) {
    const int rr = (int)((n - r0) < kRC ? (n - r0) : kRC);
    for (int e = lane; e < rr * s; e += 32) {
      const int a = e / rr, r = e % rr;
      Xc[r * s + a] = X[(int64_t)S[a] * ld + r0 + r];
    }
    __syncwarp();
    for (int e = lane; e < s * s; e += 32) {
      const int a = e / s, b = e % s;
      if (b < a) continue;
      double acc = Q[a * s + b];
      for (int r = 0; r < rr; r++) acc = fma(Xc[r * s + a], Xc[r * s + b], acc);
      Q[a * s + b] = acc;
    }
    __syncwarp();
  }
  for (int e = lane; e < s * s; e += 32) {
    const int a = e / s, b = e % s;
    if (b < a) Q[a * s + b] = Q[b * s + a];
    else if (a == b) Q[a * s + b] += 2.0 * lam2;
  }
  }
  for (int a = lane; a < s; a += 32) { q[a] = c[S[a]]; bb[a] = 0.0; bp[a] = 0.0; }
  __syncwarp();
  // warm start (R12): β⁰ = Proj_[−M,M](Q⁻¹q) by a Cholesky factor of the s×s Gram in the
  // staging area (s ≤ 32).  When the box is inactive this is the minimiser and FPG stops after one
  // step; otherwise FPG continues from it.  The FPG iterations are the paper's.
  if (s <= 32) {
    double* Lf = Xc;   // [s][s] lower factor (kRC·s ≥ s² doubles for s ≤ kRC)
    for (int j = 0; j < s; j++) {
      double d = 0.0;
      if (lane == j) {
        d = Q[j * s + j];
        for (int k2 = 0; k2 < j; k2++) d -= Lf[j * s + k2] * Lf[j * s + k2];
        Lf[j * s + j] = sqrt(d);
      }
      __syncwarp();
      if (lane > j && lane < s) {
        double v = Q[lane * s + j];
        for (int k2 = 0; k2 < j; k2++) v -= Lf[lane * s + k2] * Lf[j * s + k2];
        Lf[lane * s + j] = v / Lf[j * s + j];
      }
      __syncwarp();
    }
    if (lane == 0) {
      double* z = bt;   // forward L z = q, then back Lᵀ x = z (x in bn)
      for (int i = 0; i < s; i++) {
        double v = q[i];
        for (int k2 = 0; k2 < i; k2++) v -= Lf[i * s + k2] * z[k2];
        z[i] = v / Lf[i * s + i];
      }
      for (int i = s - 1; i >= 0; i--) {
        double v = z[i];
        for (int k2 = i + 1; k2 < s; k2++) v -= Lf[k2 * s + i] * bn[k2];
        bn[i] = v / Lf[i * s + i];
      }
    }
    __syncwarp();
    for (int a = lane; a < s; a += 32) {
      const double b0 = fmin(fmax(bn[a], -M), M);
      bb[a] = b0;
      bp[a] = b0;
    }
    __syncwarp();
  }
  // Gershgorin bound on λmax(Q) → initial step α0 = 1/L̂ (R12)
  double Lh = 0.0;
  for (int a = lane; a < s; a += 32) {
    double r = 0.0;
    for (int b = 0; b < s; b++) r += fabs(Q[a * s + b]);
    Lh = fmax(Lh, r);
  }
  Lh = warp_max(Lh);
  const double alpha0 = 1.0 / Lh;

  double f_cur = 0.0;   // f(β) = −qᵀβ + ½βᵀQβ  (U_S = ½‖y‖² + f)
  for (int t = 0; t < max_iters; t++) {
    const double mom = (double)t / (double)(t + 3);
    for (int a = lane; a < s; a += 32) bt[a] = bb[a] + mom * (bb[a] - bp[a]);
    __syncwarp();
    double qb = 0.0, bg = 0.0;
    for (int a = lane; a < s; a += 32) {
      double r = 0.0;
      for (int b = 0; b < s; b++) r = fma(Q[a * s + b], bt[b], r);
      const double ga = r - q[a];
      g[a] = ga;
      qb = fma(q[a], bt[a], qb);
      bg = fma(bt[a], ga, bg);
    }
    __syncwarp();
    {
      double r2[2] = {qb, bg};
      warp_sum_k<2>(r2);
      qb = r2[0];
      bg = r2[1];
    }
    const double f_t = 0.5 * bg - 0.5 * qb;     // ½β̃ᵀ(Qβ̃ − q) − ½qᵀβ̃
    double alpha = alpha0, f_n = 0.0;
    for (int ls = 0; ls < 60; ls++) {
      double gd = 0.0, dd = 0.0;
      for (int a = lane; a < s; a += 32) {
        const double v = fmin(fmax(bt[a] - alpha * g[a], -M), M);
        bn[a] = v;
        const double d = v - bt[a];
        gd = fma(g[a], d, gd);
        dd = fma(d, d, dd);
      }
      __syncwarp();
      double qn = 0.0, nQn = 0.0;
      for (int a = lane; a < s; a += 32) {
        double r = 0.0;
        for (int b = 0; b < s; b++) r = fma(Q[a * s + b], bn[b], r);
        qn = fma(q[a], bn[a], qn);
        nQn = fma(bn[a], r, nQn);
      }
      {
        double r4[4] = {gd, dd, qn, nQn};
        warp_sum_k<4>(r4);
        gd = r4[0];
        dd = r4[1];
        qn = r4[2];
        nQn = r4[3];
      }
      f_n = 0.5 * nQn - qn;
      const double rhs = f_t + gd + dd / (2.0 * alpha);
      if (f_n <= rhs + 1e-15 * fabs(rhs)) break;   // eq:fpg_armijo (rounding slack)
      alpha *= 0.5;
    }
    double dmax = 0.0, bmax = 0.0;
    for (int a = lane; a < s; a += 32) {
      dmax = fmax(dmax, fabs(bn[a] - bb[a]));
      bmax = fmax(bmax, fabs(bn[a]));
      bp[a] = bb[a];
      bb[a] = bn[a];
    }
    __syncwarp();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
      bmax = fmax(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
    }
    f_cur = f_n;
    if (dmax <= 1e-14 * (1.0 + bmax)) break;   // change in β_S below tolerance
  }
  if (lane == 0) obj[nd] = 0.5 * yy + f_cur + lam0 * (double)s;
  if (beta_s)
    for (int a = lane; a < s; a += 32) beta_s[o0 + a] = bb[a];
}

// X_S of one support gathered densely (n × s, ld n) for the large-support Gram GEMM
__global__ void gather_cols(const double* __restrict__ X, int64_t ld, int64_t n, const int32_t* __restrict__ S, int s,
                            double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * s) return;
  out[e] = X[(int64_t)S[e / n] * ld + e % n];
}
__global__ void add_diag_q(double* Q, int s, double v) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a < s) Q[(int64_t)a * s + a] += v;
}

}  // namespace

int upper_batch(Ctx* c, int B, const int64_t* supp_off, const int32_t* supp_idx, double* obj, double* beta_s,
                cudaStream_t st) {
  if (B <= 0) return L0L2_OK;
  std::vector<int64_t> off(B + 1);
  L0L2_CUDA(c, cudaMemcpyAsync(off.data(), supp_off, sizeof(int64_t) * (B + 1), cudaMemcpyDeviceToHost, st));
  L0L2_CUDA(c, cudaStreamSynchronize(st));
  int smax = 0;
  for (int k = 0; k < B; k++) {
    const int64_t sk = off[k + 1] - off[k];
    if (sk < 0 || sk > c->p) return set_err(c, L0L2_EINVAL, "bad support offsets");
    smax = std::max<int>(smax, (int)sk);
  }
  const size_t vec_bytes = sizeof(double) * (size_t)(6 + kRC) * smax;
  const size_t limit = 200 * 1024;
  int smax_smem = smax;
  size_t smem = sizeof(double) * (size_t)smax * smax + vec_bytes;
  double* Qg = nullptr;
  int64_t qstride = 0;
  if (smem > limit) {   // Gram does not fit shared memory: keep it in HBM/L2
    smax_smem = 0;
    smem = vec_bytes;
    qstride = (int64_t)smax * smax;
    if (c->ub_scratch_bytes < (size_t)B * qstride * sizeof(double)) {
      if (c->ub_scratch) cudaFree(c->ub_scratch);
      c->ub_scratch_bytes = (size_t)B * qstride * sizeof(double);
      if (cudaMalloc(&c->ub_scratch, c->ub_scratch_bytes) != cudaSuccess) {
        c->ub_scratch = nullptr;
        c->ub_scratch_bytes = 0;
        return set_err(c, L0L2_ENOMEM, "upper-bound Gram scratch");
      }
    }
    Qg = (double*)c->ub_scratch;
    if (smem > limit) {
      // large supports (the vectors + staging no longer fit shared memory): the Gram of every support
      // is formed in HBM by a gather + DMMA GEMM (Q = X_SᵀX_S + 2λ2I), and the FPG iterations run from
      // it with only their six s-vectors in shared memory — the same iterates
      const size_t vec6 = sizeof(double) * (size_t)6 * smax;
      if (vec6 > limit) return set_err(c, L0L2_EINVAL, "support too large (%d)", smax);
      double* XS = (double*)c->scratch_n(1, sizeof(double) * (size_t)c->n * smax);
      if (!XS) return set_err(c, L0L2_ENOMEM, "upper-bound X_S scratch");
      for (int k = 0; k < B; k++) {
        const int sk = (int)(off[k + 1] - off[k]);
        if (sk == 0) continue;
        const int64_t tot = c->n * sk;
        gather_cols<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(c->X, c->ld, c->n, supp_idx + off[k], sk, XS);
        L0L2_LAUNCHED(c);
        double* Qk = Qg + (int64_t)k * qstride;
        int rc = gemm_f64(c, sk, sk, c->n, 1.0, XS, c->n, true, XS, c->n, false, 0.0, Qk, sk, st);
        if (rc) return rc;
        add_diag_q<<<(sk + 255) / 256, 256, 0, st>>>(Qk, sk, 2.0 * c->lam2);
        L0L2_LAUNCHED(c);
      }
      L0L2_CUDA(c, cudaFuncSetAttribute(fpg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)limit));
      if (!c->ev[2]) {
        for (auto& e : c->ev) if (!e) L0L2_CUDA(c, cudaEventCreate(&e));
      }
      L0L2_CUDA(c, cudaEventRecord(c->ev[2], st));
      fpg_kernel<<<B, 32, vec6, st>>>(c->X, c->ld, c->n, c->y, c->c, c->yy, c->lam0, c->lam2, c->M, supp_off, supp_idx,
                                      obj, beta_s, nullptr, qstride, 0, 50000, Qg);
      L0L2_LAUNCHED(c);
      L0L2_CUDA(c, cudaEventRecord(c->ev[3], st));
      L0L2_CUDA(c, cudaEventSynchronize(c->ev[3]));
      float ms = 0.f;
      L0L2_CUDA(c, cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]));
      c->ks.upper_launches++;
      c->ks.upper_ms += ms;
      c->ks.upper_bytes_alg += 8.0 * (double)c->n * (double)(off[B] - off[0]);
      return L0L2_OK;
    }
  }
  // multi-warp Gram pre-pass when nw ≥ 2 warps' partials fit shared memory
  int gnw = 0;
  for (int w = 8; w >= 2; w /= 2)
    if (sizeof(double) * (size_t)w * ((size_t)smax * smax + (size_t)kRC * smax) <= limit) { gnw = w; break; }
  const double* Qpre = nullptr;
  if (gnw && smax > 0) {
    const int64_t qs = (int64_t)smax * smax;
    if (c->ub_scratch_bytes < (size_t)B * qs * sizeof(double)) {
      if (c->ub_scratch) cudaFree(c->ub_scratch);
      c->ub_scratch_bytes = (size_t)B * qs * sizeof(double);
      if (cudaMalloc(&c->ub_scratch, c->ub_scratch_bytes) != cudaSuccess) {
        c->ub_scratch = nullptr;
        c->ub_scratch_bytes = 0;
        return set_err(c, L0L2_ENOMEM, "upper-bound Gram scratch");
      }
    }
    qstride = qs;
    Qg = nullptr;
    Qpre = (const double*)c->ub_scratch;
  }
  L0L2_CUDA(c, cudaFuncSetAttribute(fpg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)limit));
  L0L2_CUDA(c, cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)limit));
  if (!c->ev[2]) {
    for (auto& e : c->ev) if (!e) L0L2_CUDA(c, cudaEventCreate(&e));
  }
  L0L2_CUDA(c, cudaEventRecord(c->ev[2], st));
  if (Qpre) {
    gram_kernel<<<B, 32 * gnw, sizeof(double) * (size_t)gnw * ((size_t)smax * smax + (size_t)kRC * smax), st>>>(
        c->X, c->ld, c->n, c->lam2, supp_off, supp_idx, (double*)c->ub_scratch, qstride);
    L0L2_LAUNCHED(c);
  }
  fpg_kernel<<<B, 32, smem, st>>>(c->X, c->ld, c->n, c->y, c->c, c->yy, c->lam0, c->lam2, c->M, supp_off, supp_idx,
                                  obj, beta_s, Qg, qstride, smax_smem, 50000, Qpre);
  L0L2_LAUNCHED(c);
  L0L2_CUDA(c, cudaEventRecord(c->ev[3], st));
  L0L2_CUDA(c, cudaEventSynchronize(c->ev[3]));
  float ms = 0.f;
  L0L2_CUDA(c, cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]));
  c->ks.upper_launches++;
  c->ks.upper_ms += ms;
  c->ks.upper_bytes_alg += 8.0 * (double)c->n * (double)(off[B] - off[0]);   // X_S gathered once per support
  return L0L2_OK;
}

}  // namespace l0l2

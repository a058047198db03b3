// Matching-pursuit root heuristic (Algorithm 3; outline P:781-783).
//
// State on the device: residual r (n), β (p), membership inS (p), the support list S (|S|).
// One round = forward step + backward step (R15):
//   forward   c_j = X_jᵀ r, D_j = ‖X_j‖² + 2λ2, β_j = Proj_[−M,M](c_j / D_j),
//             Δ_j = −β_j c_j + ½ β_j² D_j + λ0  (j ∉ S)
//             j* = argmin Δ (ties → lowest j); if Δ_j* < 0: S ∪= {j*}, r −= X_j* β_j*
//   backward  c_j = X_jᵀ r, Δ_j = β_j c_j + (½‖X_j‖² − λ2) β_j² − λ0  (j ∈ S)
//             j* = argmin Δ (ties → lowest j); if Δ_j* < 0: S \= {j*}, r += X_j* β_j*, β_j* = 0
// The forward scan is one HBM-bound pass over X (a warp per column, coalesced column reads,
// r staged in shared memory, fixed-order butterfly sums), reduced to one candidate per CTA and
// then in CTA order by a single-CTA apply kernel; the backward step touches |S| columns only.
// The host loop reads one flag per round.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace l0l2 {
namespace {

constexpr int MP_THREADS = 256;
constexpr int MP_WARPS = MP_THREADS / 32;

struct Cand { double delta, b; int j; };

__device__ __forceinline__ bool cand_better(double d, int j, double bd, int bj) {
  return d < bd || (d == bd && j < bj);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// c_j = X_jᵀ r for one column (lane-strided rows, four independent accumulators so each lane keeps
// four loads in flight, fixed combination order and butterfly): every lane gets the sum
__device__ __forceinline__ double col_dot(const double* __restrict__ X, int64_t ld, int64_t n, int64_t j,
                                          const double* r, int lane) {
  const double* col = X + j * ld;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int64_t i = lane;
  for (; i + 96 < n; i += 128) {
    a0 = fma(__ldcs(col + i), r[i], a0);
    a1 = fma(__ldcs(col + i + 32), r[i + 32], a1);
    a2 = fma(__ldcs(col + i + 64), r[i + 64], a2);
    a3 = fma(__ldcs(col + i + 96), r[i + 96], a3);
  }
  for (; i < n; i += 32) a0 = fma(__ldcs(col + i), r[i], a0);
  return warp_sum((a0 + a1) + (a2 + a3));
}

__global__ void __launch_bounds__(MP_THREADS) mp_forward_scan(const double* __restrict__ X, int64_t ld, int64_t n,
                                                             int64_t p, const double* __restrict__ r,
                                                             const double* __restrict__ colsq,
                                                             const uint8_t* __restrict__ inS, double lam0,
                                                             double lam2, double M, Cand* cand) {
  extern __shared__ double rs[];
  __shared__ Cand wbest[MP_WARPS];
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) rs[i] = r[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * MP_WARPS + warp, nw = (int64_t)gridDim.x * MP_WARPS;
  double bd = INFINITY, bb = 0.0;
  int bj = 0x7fffffff;
  for (int64_t j = gw; j < p; j += nw) {
    if (inS[j]) continue;   // warp-uniform (one column per warp)
    const double c = col_dot(X, ld, n, j, rs, lane);
    const double D = colsq[j] + 2.0 * lam2;
    const double b = fmin(fmax(c / D, -M), M);
    const double d = -b * c + 0.5 * b * b * D + lam0;
    if (cand_better(d, (int)j, bd, bj)) { bd = d; bb = b; bj = (int)j; }
  }
  if (lane == 0) wbest[warp] = Cand{bd, bb, bj};
  __syncthreads();
  if (threadIdx.x == 0) {
    Cand best = wbest[0];
    for (int w = 1; w < MP_WARPS; w++)
      if (cand_better(wbest[w].delta, wbest[w].j, best.delta, best.j)) best = wbest[w];
    cand[blockIdx.x] = best;
  }
}

// state[0] = |S|, state[1] = changed this round, state[2] = forward j or −1, state[3] = backward j or −1
__global__ void __launch_bounds__(1024) mp_forward_apply(const double* __restrict__ X, int64_t ld, int64_t n,
                                                         const Cand* __restrict__ cand, int ncand, double* r,
                                                         double* beta, uint8_t* inS, int32_t* S, int* state,
                                                         double* log_delta) {
  __shared__ Cand best;
  __shared__ Cand wb[32];
  // argmin over the per-CTA candidates: the (Δ, j) lexicographic minimum is order independent, so a
  // parallel tree gives the same winner as a sequential scan
  {
    Cand b{INFINITY, 0.0, 0x7fffffff};
    for (int q = threadIdx.x; q < ncand; q += blockDim.x)
      if (cand_better(cand[q].delta, cand[q].j, b.delta, b.j)) b = cand[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Cand x{__shfl_xor_sync(0xffffffffu, b.delta, o), __shfl_xor_sync(0xffffffffu, b.b, o),
             __shfl_xor_sync(0xffffffffu, b.j, o)};
      if (cand_better(x.delta, x.j, b.delta, b.j)) b = x;
    }
    if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = b;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    Cand b = wb[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); w++)
      if (cand_better(wb[w].delta, wb[w].j, b.delta, b.j)) b = wb[w];
    best = b;
    state[2] = -1;
    if (b.delta < 0.0) {
      inS[b.j] = 1;
      beta[b.j] = b.b;
      S[state[0]] = b.j;
      state[0] += 1;
      state[1] = 1;
      state[2] = b.j;
      log_delta[0] = b.delta;
    }
  }
  __syncthreads();
  if (best.delta < 0.0) {
    const double* col = X + (int64_t)best.j * ld;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) r[i] = __dsub_rn(r[i], __dmul_rn(col[i], best.b));
  }
}

__global__ void __launch_bounds__(1024) mp_backward(const double* __restrict__ X, int64_t ld, int64_t n,
                                                    const double* __restrict__ colsq, double lam0, double lam2,
                                                    double* r, double* beta, uint8_t* inS, int32_t* S, int* state,
                                                    double* log_delta) {
  __shared__ Cand wbest[32];
  __shared__ int best_pos;
  __shared__ double best_b;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int cnt = state[0];
  double bd = INFINITY;
  int bj = 0x7fffffff, bpos = -1;
  for (int q = warp; q < cnt; q += nw) {
    const int j = S[q];
    const double c = col_dot(X, ld, n, j, r, lane);
    const double b = beta[j];
    const double d = b * c + (0.5 * colsq[j] - lam2) * b * b - lam0;
    if (cand_better(d, j, bd, bj)) { bd = d; bj = j; bpos = q; }
  }
  if (lane == 0) wbest[warp] = Cand{bd, (double)bpos, bj};
  __syncthreads();
  if (threadIdx.x == 0) {
    Cand b = wbest[0];
    for (int w = 1; w < nw; w++)
      if (cand_better(wbest[w].delta, wbest[w].j, b.delta, b.j)) b = wbest[w];
    state[3] = -1;
    best_pos = -1;
    if (cnt > 0 && b.delta < 0.0) {
      best_pos = (int)b.b;
      best_b = beta[b.j];
      state[1] = 1;
      state[3] = b.j;
      log_delta[1] = b.delta;
    }
  }
  __syncthreads();
  if (best_pos >= 0) {
    const int j = S[best_pos];
    const double* col = X + (int64_t)j * ld;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) r[i] = __dadd_rn(r[i], __dmul_rn(col[i], best_b));
    __syncthreads();
    if (threadIdx.x == 0) {
      beta[j] = 0.0;
      inS[j] = 0;
      S[best_pos] = S[cnt - 1];   // order of S is irrelevant: argmin ties are broken by column index
      state[0] = cnt - 1;
    }
  }
}

// obj = ½‖r‖² + λ2‖β‖² + λ0|S| (fixed-order block sums)
__global__ void __launch_bounds__(1024) mp_objective(const double* __restrict__ r, int64_t n,
                                                     const double* __restrict__ beta, int64_t p, double lam0,
                                                     double lam2, const int* state, double* obj) {
  __shared__ double ws[32][2];
  double a = 0.0, b = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a = fma(r[i], r[i], a);
  for (int64_t j = threadIdx.x; j < p; j += blockDim.x) b = fma(beta[j], beta[j], b);
  a = warp_sum(a);
  b = warp_sum(b);
  if ((threadIdx.x & 31) == 0) { ws[threadIdx.x >> 5][0] = a; ws[threadIdx.x >> 5][1] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double A = 0.0, Bs = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) { A += ws[w][0]; Bs += ws[w][1]; }
    obj[0] = 0.5 * A + lam2 * Bs + lam0 * (double)state[0];
  }
}

}  // namespace

int mp_run(Ctx* c, int max_rounds, cudaStream_t st, std::vector<int32_t>& S_out, std::vector<double>& beta_out,
           double* obj, int* rounds_out) {
  const int64_t n = c->n, p = c->p;
  if (max_rounds <= 0) max_rounds = (int)std::min<int64_t>(4 * p + 10, 1 << 30);
  const int grid = 4 * c->sms;   // 32 warps per SM stream the columns
  // work space (allocated on first use, kept with the context)
  if (!c->mp_r) {
    c->mp_r = (double*)dalloc(c, sizeof(double) * n);
    c->mp_beta = (double*)dalloc(c, sizeof(double) * p);
    c->mp_inS = (uint8_t*)dalloc(c, p);
    c->mp_S = (int32_t*)dalloc(c, sizeof(int32_t) * p);
    c->mp_cand = dalloc(c, sizeof(Cand) * grid);
    c->mp_state = (int*)dalloc(c, sizeof(int) * 4);
    c->mp_log = (double*)dalloc(c, sizeof(double) * 4);
    if (!c->mp_r || !c->mp_beta || !c->mp_inS || !c->mp_S || !c->mp_cand || !c->mp_state || !c->mp_log)
      return set_err(c, L0L2_ENOMEM, "matching pursuit work space");
  }
  // S ← ∅, β ← 0, r ← y
  L0L2_CUDA(c, cudaMemcpyAsync(c->mp_r, c->y, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  L0L2_CUDA(c, cudaMemsetAsync(c->mp_beta, 0, sizeof(double) * p, st));
  L0L2_CUDA(c, cudaMemsetAsync(c->mp_inS, 0, p, st));
  L0L2_CUDA(c, cudaMemsetAsync(c->mp_state, 0, sizeof(int) * 4, st));
  const size_t smem = sizeof(double) * n;
  if (smem > 48 * 1024)
    L0L2_CUDA(c, cudaFuncSetAttribute(mp_forward_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int rounds = 0;
  int hstate[4] = {0, 0, 0, 0};
  while (rounds < max_rounds) {
    rounds++;
    L0L2_CUDA(c, cudaMemsetAsync(c->mp_state + 1, 0, sizeof(int), st));
    mp_forward_scan<<<grid, MP_THREADS, smem, st>>>(c->X, c->ld, n, p, c->mp_r, c->colsq, c->mp_inS, c->lam0,
                                                     c->lam2, c->M, (Cand*)c->mp_cand);
    L0L2_LAUNCHED(c);
    mp_forward_apply<<<1, 1024, 0, st>>>(c->X, c->ld, n, (const Cand*)c->mp_cand, grid, c->mp_r, c->mp_beta,
                                         c->mp_inS, c->mp_S, c->mp_state, c->mp_log);
    L0L2_LAUNCHED(c);
    mp_backward<<<1, 1024, 0, st>>>(c->X, c->ld, n, c->colsq, c->lam0, c->lam2, c->mp_r, c->mp_beta, c->mp_inS,
                                    c->mp_S, c->mp_state, c->mp_log);
    L0L2_LAUNCHED(c);
    L0L2_CUDA(c, cudaMemcpyAsync(hstate, c->mp_state, sizeof(hstate), cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    if (!hstate[1]) break;
  }
  double* dobj = c->mp_log + 2;
  mp_objective<<<1, 1024, 0, st>>>(c->mp_r, n, c->mp_beta, p, c->lam0, c->lam2, c->mp_state, dobj);
  L0L2_LAUNCHED(c);
  S_out.assign(hstate[0], 0);
  beta_out.assign(p, 0.0);
  if (hstate[0] > 0)
    L0L2_CUDA(c, cudaMemcpyAsync(S_out.data(), c->mp_S, sizeof(int32_t) * hstate[0], cudaMemcpyDeviceToHost, st));
  L0L2_CUDA(c, cudaMemcpyAsync(beta_out.data(), c->mp_beta, sizeof(double) * p, cudaMemcpyDeviceToHost, st));
  L0L2_CUDA(c, cudaMemcpyAsync(obj, dobj, sizeof(double), cudaMemcpyDeviceToHost, st));
  L0L2_CUDA(c, cudaStreamSynchronize(st));
  std::sort(S_out.begin(), S_out.end());
  if (rounds_out) *rounds_out = rounds;
  return L0L2_OK;
}

}  // namespace l0l2

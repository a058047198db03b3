// Tree-wide precompute of l0l2_create ("done once for the entire tree").
//
//   c = Xᵀy, colsq_j = ‖X_j‖²                         (one streaming pass over X)
//   A = XXᵀ + ρI_n                                     (DMMA GEMM, n²p flops)
//   A = LLᵀ                                            (blocked right-looking Cholesky)
//   Z = L⁻¹X                                           (blocked forward substitution, n²p flops)
//   Lt = Lᵀ                                            (for ‖Xβ‖² = ‖L(Zβ)‖² in the primal check)
//
// Then D = (XᵀX+ρI)⁻¹ = (I − ZᵀZ)/ρ (Woodbury with the paper's 1/ρ² corrected to 1/ρ,
// DESIGN.md R1), so every ADMM b-update is b = (w − Zᵀ(Zw))/ρ (admm.cu).
#include <cmath>

#include "common.cuh"

namespace l0l2 {
namespace {

constexpr int NB = 64;   // Cholesky / TRSM block size
constexpr int kPotrfSmem = 2 * NB * (NB + 1) * (int)sizeof(double);

// c_j = X_jᵀ y, colsq_j = ‖X_j‖²: one warp per column, fixed-order reduction.
__global__ void col_stats(const double* __restrict__ X, int64_t ld, int64_t n, int64_t p,
                          const double* __restrict__ y, double* __restrict__ c, double* __restrict__ colsq) {
  int64_t j = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (j >= p) return;
  const double* x = X + j * ld;
  double s = 0.0, q = 0.0;
  for (int64_t i = lane; i < n; i += 32) {
    double xi = x[i];
    s = fma(xi, y[i], s);
    q = fma(xi, xi, q);
  }
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    q += __shfl_xor_sync(0xffffffffu, q, o);
  }
  if (lane == 0) { c[j] = s; colsq[j] = q; }
}

__global__ void dot_self(const double* __restrict__ y, int64_t n, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(y[i], y[i], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += red[w];
    *out = t;
  }
}

__global__ void sum_vec(const double* __restrict__ x, int64_t n, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += red[w];
    *out = t;
  }
}

__global__ void add_diag(double* A, int64_t ld, int64_t n, double rho) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) A[i + i * ld] += rho;
}

// Factor the nb×nb diagonal block A[k0.., k0..] = Lkk Lkkᵀ in one CTA; write Lkk into L and
// Lkk⁻¹ (lower) into Inv (NB×NB, col-major, ld NB).  info ← 1 + j if a pivot is ≤ 0.
__global__ void potrf_diag(const double* __restrict__ A, double* __restrict__ L, int64_t ld,
                           int64_t k0, int nb, double* __restrict__ Inv, int* info) {
  extern __shared__ double smem_pd[];
  double (*a)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(smem_pd);             // a[i][j]
  double (*inv)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(smem_pd + NB * (NB + 1));
  const int t = threadIdx.x;
  for (int e = t; e < nb * nb; e += blockDim.x) {
    int i = e % nb, j = e / nb;
    a[i][j] = (i >= j) ? A[(k0 + i) + (k0 + j) * ld] : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < nb; j++) {
    if (t == 0) {
      double d = a[j][j];
      if (!(d > 0.0)) { if (*info == 0) *info = (int)(k0 + j) + 1; d = 1.0; }
      a[j][j] = sqrt(d);
    }
    __syncthreads();
    double djj = a[j][j];
    for (int i = j + 1 + t; i < nb; i += blockDim.x) a[i][j] /= djj;
    __syncthreads();
    // trailing rank-1 update of the lower triangle
    int m = nb - j - 1;
    for (int e = t; e < m * m; e += blockDim.x) {
      int i = j + 1 + e % m, l = j + 1 + e / m;
      if (l <= i) a[i][l] -= a[i][j] * a[l][j];
    }
    __syncthreads();
  }
  // inverse of the lower-triangular block: column cc solves Lkk x = e_cc by forward substitution
  for (int cc = t; cc < nb; cc += blockDim.x) {
    for (int i = 0; i < nb; i++) {
      if (i < cc) { inv[i][cc] = 0.0; continue; }
      double s = (i == cc) ? 1.0 : 0.0;
      for (int m2 = cc; m2 < i; m2++) s -= a[i][m2] * inv[m2][cc];
      inv[i][cc] = s / a[i][i];
    }
  }
  __syncthreads();
  for (int e = t; e < nb * nb; e += blockDim.x) {
    int i = e % nb, j = e / nb;
    L[(k0 + i) + (k0 + j) * ld] = (i >= j) ? a[i][j] : 0.0;
    Inv[i + j * NB] = inv[i][j];
  }
}

__global__ void transpose_sq(const double* __restrict__ in, double* __restrict__ out, int64_t ld, int64_t n) {
  __shared__ double tile[32][33];
  int64_t bx = (int64_t)blockIdx.x * 32, by = (int64_t)blockIdx.y * 32;
  // element (row = bx + tx, col = by + r) read coalesced along rows
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int64_t row = bx + threadIdx.x, col = by + r;
    tile[r][threadIdx.x] = (row < n && col < n) ? in[row + col * ld] : 0.0;
  }
  __syncthreads();
  // out(row', col') = in(col', row'): write out[row' + col'*ld] with row' = by + tx, col' = bx + r
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int64_t rowp = by + threadIdx.x, colp = bx + r;
    if (rowp < n && colp < n) out[rowp + colp * ld] = tile[threadIdx.x][r];
  }
}

}  // namespace

int precompute(Ctx* c, cudaStream_t st) {
  const int64_t n = c->n, p = c->p, ld = c->ld;
  const int64_t p8 = round8(p);
  {
    int wpb = 8;
    col_stats<<<(unsigned)((p + wpb - 1) / wpb), wpb * 32, 0, st>>>(c->X, ld, n, p, c->y, c->c, c->colsq);
    L0L2_LAUNCHED(c);
  }
  double* d_yy = (double*)dalloc(c, sizeof(double));
  double* A = (double*)dalloc(c, sizeof(double) * ld * n);
  double* Inv = (double*)dalloc(c, sizeof(double) * NB * NB);
  int* info = (int*)dalloc(c, sizeof(int));
  if (!d_yy || !A || !Inv || !info) return set_err(c, L0L2_ENOMEM, "precompute scratch");
  dot_self<<<1, 256, 0, st>>>(c->y, n, d_yy);
  L0L2_LAUNCHED(c);
  if (c->rho <= 0.0) {
    // ρ default = mean_j ‖X_j‖² (R5), reduced on the device
    double* d_rho = (double*)dalloc(c, sizeof(double));
    if (!d_rho) return set_err(c, L0L2_ENOMEM, "rho scratch");
    sum_vec<<<1, 256, 0, st>>>(c->colsq, p, d_rho);
    L0L2_LAUNCHED(c);
    if (c->sharded) {   // the mean over ALL columns (column-sharded context, sharded.cu)
      int rc0 = shard_allreduce(c, d_rho, 1, st);
      if (rc0) return rc0;
    }
    double s = 0.0;
    L0L2_CUDA(c, cudaMemcpyAsync(&s, d_rho, sizeof(double), cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    c->rho = s / (double)(c->sharded ? c->p_total : p);
  }
  L0L2_CUDA(c, cudaFuncSetAttribute(potrf_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, kPotrfSmem));
  L0L2_CUDA(c, cudaMemsetAsync(info, 0, sizeof(int), st));
  L0L2_CUDA(c, cudaMemsetAsync(A, 0, sizeof(double) * ld * n, st));
  L0L2_CUDA(c, cudaMemsetAsync(c->L, 0, sizeof(double) * ld * n, st));
  // A = X Xᵀ + ρ I  (op(B) = Xᵀ: element (k, col) = X[col + k*ld])
  int rc = gemm_f64(c, n, n, p, 1.0, c->X, ld, false, c->X, ld, true, 0.0, A, ld, st);
  if (rc) return rc;
  // column-sharded context: A = Σ_r X_r X_rᵀ over the ranks' columns (sharded.cu)
  if (c->sharded && (rc = shard_allreduce(c, A, ld * n, st))) return rc;
  add_diag<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(A, ld, n, c->rho);
  L0L2_LAUNCHED(c);
  // Z starts as a copy of X (padded rows / columns are zero)
  L0L2_CUDA(c, cudaMemcpyAsync(c->Z, c->X, sizeof(double) * ld * p8, cudaMemcpyDeviceToDevice, st));
  for (int64_t k0 = 0; k0 < n; k0 += NB) {
    const int nb = (int)std::min<int64_t>(NB, n - k0);
    potrf_diag<<<1, 256, kPotrfSmem, st>>>(A, c->L, ld, k0, nb, Inv, info);
    L0L2_LAUNCHED(c);
    const int64_t r0 = k0 + nb, rem = n - r0;
    if (rem > 0) {
      // panel: L[r0:, k0:k0+nb] = A[r0:, k0:k0+nb] · Lkk⁻ᵀ
      rc = gemm_f64(c, rem, nb, nb, 1.0, A + r0 + k0 * ld, ld, false, Inv, NB, true, 0.0,
                    c->L + r0 + k0 * ld, ld, st);
      if (rc) return rc;
      // trailing: A[r0:, r0:] −= Lpanel · Lpanelᵀ
      rc = gemm_f64(c, rem, rem, nb, -1.0, c->L + r0 + k0 * ld, ld, false, c->L + r0 + k0 * ld, ld, true,
                    1.0, A + r0 + r0 * ld, ld, st);
      if (rc) return rc;
    }
    // forward substitution for Z = L⁻¹X, block row k0 (in place; M = nb ≤ 64 = one GEMM row tile)
    rc = gemm_f64(c, nb, p8, nb, 1.0, Inv, NB, false, c->Z + k0, ld, false, 0.0, c->Z + k0, ld, st);
    if (rc) return rc;
    if (rem > 0) {
      rc = gemm_f64(c, rem, p8, nb, -1.0, c->L + r0 + k0 * ld, ld, false, c->Z + k0, ld, false, 1.0,
                    c->Z + r0, ld, st);
      if (rc) return rc;
    }
  }
  {
    dim3 blk(32, 8), grd((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32));
    transpose_sq<<<grd, blk, 0, st>>>(c->L, c->Lt, ld, n);
    L0L2_LAUNCHED(c);
  }
  int h_info = 0;
  L0L2_CUDA(c, cudaMemcpyAsync(&h_info, info, sizeof(int), cudaMemcpyDeviceToHost, st));
  L0L2_CUDA(c, cudaMemcpyAsync(&c->yy, d_yy, sizeof(double), cudaMemcpyDeviceToHost, st));
  L0L2_CUDA(c, cudaStreamSynchronize(st));
  if (h_info) return set_err(c, L0L2_EINVAL, "XXᵀ+ρI not positive definite at pivot %d", h_info - 1);
  if (c->direct) {
    // D = (I − ZᵀZ)/ρ = (XᵀX + ρI)⁻¹ (Woodbury, R1), p8 × p8 with zero padding
    c->D = (double*)dalloc(c, sizeof(double) * c->ldD * p8);
    if (!c->D) return set_err(c, L0L2_ENOMEM, "direct-regime D");
    L0L2_CUDA(c, cudaMemsetAsync(c->D, 0, sizeof(double) * c->ldD * p8, st));
    rc = gemm_f64(c, p8, p8, n, -1.0 / c->rho, c->Z, ld, true, c->Z, ld, false, 0.0, c->D, c->ldD, st);
    if (rc) return rc;
    add_diag<<<(unsigned)((p + 255) / 256), 256, 0, st>>>(c->D, c->ldD, p, 1.0 / c->rho);
    L0L2_LAUNCHED(c);
    L0L2_CUDA(c, cudaStreamSynchronize(st));
  }
  return L0L2_OK;
}

}  // namespace l0l2

// FP64 GEMM on the sm_100a DMMA pipe (mma.sync.m8n8k4.f64 → SASS DMMA.8x8x4).
// tcgen05 has no f64 kind, so FP64 contractions use warp-level DMMA
// with register accumulators.  Used by the tree-wide precompute (A = XXᵀ+ρI,
// blocked Cholesky trailing updates, Z = L⁻¹X) and by the optional r̂ = y − Xb̂ output.
#include <algorithm>

#include "common.cuh"

namespace l0l2 {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, PADS = 68;  // PADS ≡ 4 (mod 16): conflict-free fragments

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) gemm_kernel(int64_t M, int64_t N, int64_t K, double alpha,
                                                   const double* __restrict__ A, int64_t lda,
                                                   const double* __restrict__ B, int64_t ldb,
                                                   double beta, double* __restrict__ C, int64_t ldc,
                                                   int64_t ksplit, int64_t zstride) {
  // split-K (blockIdx.z): this CTA's K range [kb, ke); its partial goes to C + z·zstride
  const int64_t kb = (int64_t)blockIdx.z * ksplit, ke = min(K, kb + ksplit);
  C += (int64_t)blockIdx.z * zstride;
  __shared__ double As[2][BK][PADS];
  __shared__ double Bs[2][BK][PADS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 2) * 32;   // 2 warps along m (32 rows each)
  const int wn = (warp & 3) * 16;    // 4 warps along n (16 cols each)
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 2; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

  double ra[4], rb[4];
  auto gload = [&](int64_t k0) {
#pragma unroll
    for (int r = 0; r < 4; r++) {
      int e = tid + r * 256;              // 0..1023 over the 64×16 tile
      int mm, kk;
      if (!TA) { mm = e & 63; kk = e >> 6; } else { kk = e & 15; mm = e >> 4; }
      int64_t gm = m0 + mm, gk = k0 + kk;
      double v = 0.0;
      if (gm < M && gk < ke) v = TA ? A[gk + gm * lda] : A[gm + gk * lda];
      ra[r] = v;
      int nn;
      if (!TB) { kk = e & 15; nn = e >> 4; } else { nn = e & 63; kk = e >> 6; }
      int64_t gn = n0 + nn;
      gk = k0 + kk;
      v = 0.0;
      if (gn < N && gk < ke) v = TB ? B[gn + gk * ldb] : B[gk + gn * ldb];
      rb[r] = v;
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int r = 0; r < 4; r++) {
      int e = tid + r * 256;
      int mm, kk;
      if (!TA) { mm = e & 63; kk = e >> 6; } else { kk = e & 15; mm = e >> 4; }
      As[buf][kk][mm] = ra[r];
      int nn;
      if (!TB) { kk = e & 15; nn = e >> 4; } else { nn = e & 63; kk = e >> 6; }
      Bs[buf][kk][nn] = rb[r];
    }
  };
  const int64_t nk = ke > kb ? (ke - kb + BK - 1) / BK : 0;
  if (nk > 0) gload(kb);
  sstore(0);
  __syncthreads();
  for (int64_t kt = 0; kt < nk; kt++) {
    const int buf = kt & 1;
    if (kt + 1 < nk) gload(kb + (kt + 1) * BK);
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; i++) af[i] = As[buf][ks + (lane & 3)][wm + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 2; j++) bf[j] = Bs[buf][ks + (lane & 3)][wn + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 2; j++) dmma(acc[i][j], af[i], bf[j]);
    }
    if (kt + 1 < nk) sstore(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 2; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        int64_t gm = m0 + wm + i * 8 + (lane >> 2);
        int64_t gn = n0 + wn + j * 8 + 2 * (lane & 3) + h;
        if (gm < M && gn < N) {
          double* cp = C + gm + gn * ldc;
          *cp = alpha * acc[i][j][h] + (beta == 0.0 ? 0.0 : beta * *cp);
        }
      }
}

// Narrow-N variant (N ≤ 16: u = Z w, s = Zᵀu, r = y − X b for ≤ 16 nodes): CTA tile 128 × 16, each of
// the 8 warps owns 16 rows × 16 columns (2 × 2 DMMA tiles), so no DMMA is spent on padding columns.
constexpr int NBM = 128, NBN = 16, NPADA = 132, NPADB = 20;   // ≡ 4 (mod 16): conflict-free fragments
template <bool TA, bool TB>
__global__ void __launch_bounds__(256) gemm_n16_kernel(int64_t M, int64_t N, int64_t K, double alpha,
                                                       const double* __restrict__ A, int64_t lda,
                                                       const double* __restrict__ B, int64_t ldb,
                                                       double beta, double* __restrict__ C, int64_t ldc,
                                                       int64_t ksplit, int64_t zstride) {
  __shared__ double As[2][BK][NPADA];
  __shared__ double Bs[2][BK][NPADB];
  const int64_t kb = (int64_t)blockIdx.z * ksplit, ke = min(K, kb + ksplit);
  C += (int64_t)blockIdx.z * zstride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp * 16;
  const int64_t m0 = (int64_t)blockIdx.y * NBM;
  double acc[2][2][2];
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 2; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
  double ra[8], rb;
  auto gload = [&](int64_t k0) {
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const int e = tid + r * 256;   // 0..2047 over the 128×16 A tile
      int mm, kk;
      if (!TA) { mm = e & 127; kk = e >> 7; } else { kk = e & 15; mm = e >> 4; }
      const int64_t gm = m0 + mm, gk = k0 + kk;
      ra[r] = (gm < M && gk < ke) ? (TA ? A[gk + gm * lda] : A[gm + gk * lda]) : 0.0;
    }
    int nn, kk;
    if (!TB) { kk = tid & 15; nn = tid >> 4; } else { nn = tid & 15; kk = tid >> 4; }
    const int64_t gk = k0 + kk;
    rb = (nn < N && gk < ke) ? (TB ? B[nn + gk * ldb] : B[gk + nn * ldb]) : 0.0;
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const int e = tid + r * 256;
      int mm, kk;
      if (!TA) { mm = e & 127; kk = e >> 7; } else { kk = e & 15; mm = e >> 4; }
      As[buf][kk][mm] = ra[r];
    }
    int nn, kk;
    if (!TB) { kk = tid & 15; nn = tid >> 4; } else { nn = tid & 15; kk = tid >> 4; }
    Bs[buf][kk][nn] = rb;
  };
  const int64_t nk = ke > kb ? (ke - kb + BK - 1) / BK : 0;
  if (nk > 0) gload(kb);
  sstore(0);
  __syncthreads();
  for (int64_t kt = 0; kt < nk; kt++) {
    const int buf = kt & 1;
    if (kt + 1 < nk) gload(kb + (kt + 1) * BK);
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double af[2], bf[2];
#pragma unroll
      for (int i = 0; i < 2; i++) af[i] = As[buf][ks + (lane & 3)][wm + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 2; j++) bf[j] = Bs[buf][ks + (lane & 3)][j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 2; i++)
#pragma unroll
        for (int j = 0; j < 2; j++) dmma(acc[i][j], af[i], bf[j]);
    }
    if (kt + 1 < nk) sstore(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 2; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int64_t gm = m0 + wm + i * 8 + (lane >> 2);
        const int64_t gn = j * 8 + 2 * (lane & 3) + h;
        if (gm < M && gn < N) {
          double* cp = C + gm + gn * ldc;
          *cp = alpha * acc[i][j][h] + (beta == 0.0 ? 0.0 : beta * *cp);
        }
      }
}

// split-K epilogue: C = alpha·Σ_z part[z] + beta·C, the partials summed in z order (deterministic)
__global__ void splitk_reduce(int64_t M, int64_t N, int splits, const double* __restrict__ part, double alpha,
                              double beta, double* __restrict__ C, int64_t ldc) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M * N) return;
  const int64_t m = e % M, n = e / M;
  double a = 0.0;
  for (int z = 0; z < splits; z++) a += part[(int64_t)z * M * N + e];
  double* cp = C + m + n * ldc;
  *cp = alpha * a + (beta == 0.0 ? 0.0 : beta * *cp);
}

}  // namespace

int gemm_f64(Ctx* c, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
             bool transA, const double* B, int64_t ldb, bool transB, double beta, double* C,
             int64_t ldc, cudaStream_t st) {
  if (M <= 0 || N <= 0) return L0L2_OK;
  const bool narrow = N <= NBN;
  dim3 grid(narrow ? 1u : (unsigned)((N + BN - 1) / BN), (unsigned)((M + (narrow ? NBM : BM) - 1) / (narrow ? NBM : BM)));
  if (grid.y > 65535) return set_err(c, L0L2_EINVAL, "gemm: M too large");
  // few output tiles and a long K (e.g. u = Z w: n × B × p): split K over ~2 CTAs per SM, partials
  // to a workspace, then a fixed-order sum
  const int64_t tiles = (int64_t)grid.x * grid.y;
  int splits = 1;
  if (tiles < c->sms && K >= 8 * BK * 16)
    splits = (int)std::min<int64_t>({(2 * c->sms + tiles - 1) / tiles, K / (BK * 16), 128});
  const int64_t ksplit = splits > 1 ? ((K + splits - 1) / splits + BK - 1) / BK * BK : K;
  if (splits > 1) splits = (int)((K + ksplit - 1) / ksplit);
  double* Cout = C;
  int64_t ldo = ldc, zstride = 0;
  double a_out = alpha, b_out = beta;
  if (splits > 1) {
    const size_t need = sizeof(double) * (size_t)splits * M * N;
    if (c->gemm_ws_bytes < need) {
      if (c->gemm_ws) cudaFree(c->gemm_ws);
      c->gemm_ws = nullptr;
      c->gemm_ws_bytes = 0;
      if (cudaMalloc(&c->gemm_ws, need) != cudaSuccess) { cudaGetLastError(); return set_err(c, L0L2_ENOMEM, "gemm split-K"); }
      c->gemm_ws_bytes = need;
    }
    Cout = (double*)c->gemm_ws;
    ldo = M;
    zstride = M * N;
    a_out = 1.0;
    b_out = 0.0;
    grid.z = (unsigned)splits;
  }
  if (narrow) {
    if (!transA && !transB) gemm_n16_kernel<false, false><<<grid, 256, 0, st>>>(M, N, K, a_out, A, lda, B, ldb, b_out, Cout, ldo, ksplit, zstride);
    else if (!transA && transB) gemm_n16_kernel<false, true><<<grid, 256, 0, st>>>(M, N, K, a_out, A, lda, B, ldb, b_out, Cout, ldo, ksplit, zstride);
    else if (transA && !transB) gemm_n16_kernel<true, false><<<grid, 256, 0, st>>>(M, N, K, a_out, A, lda, B, ldb, b_out, Cout, ldo, ksplit, zstride);
    else gemm_n16_kernel<true, true><<<grid, 256, 0, st>>>(M, N, K, a_out, A, lda, B, ldb, b_out, Cout, ldo, ksplit, zstride);
  } else if (!transA && !transB) gemm_kernel<false, false><<<grid, 256, 0, st>>>(M, N, K, a_out, A, lda, B, ldb, b_out, Cout, ldo, ksplit, zstride);
  else if (!transA && transB) gemm_kernel<false, true><<<grid, 256, 0, st>>>(M, N, K, a_out, A, lda, B, ldb, b_out, Cout, ldo, ksplit, zstride);
  else if (transA && !transB) gemm_kernel<true, false><<<grid, 256, 0, st>>>(M, N, K, a_out, A, lda, B, ldb, b_out, Cout, ldo, ksplit, zstride);
  else gemm_kernel<true, true><<<grid, 256, 0, st>>>(M, N, K, a_out, A, lda, B, ldb, b_out, Cout, ldo, ksplit, zstride);
  L0L2_LAUNCHED(c);
  if (splits > 1) {
    splitk_reduce<<<(unsigned)((M * N + 255) / 256), 256, 0, st>>>(M, N, splits, Cout, alpha, beta, C, ldc);
    L0L2_LAUNCHED(c);
  }
  return L0L2_OK;
}

}  // namespace l0l2

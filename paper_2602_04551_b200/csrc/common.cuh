// Internal declarations of the l0l2 sm_100a library (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/l0l2.h"

namespace l0l2 {

constexpr int kBC = 16;         // node columns per ADMM pass: two DMMA n=8 halves share each Z tile
constexpr int kPt = 8;          // Z columns per tile (DMMA m-dim of the adjoint = 8)
constexpr int kAdmmThreads = 512;  // 16 warps per persistent CTA
constexpr int kSums = 6;        // per-node partial sums of a check (see admm.cu)

// leading dimension of Z / X in HBM: ≥ n, even, ≡ 4 (mod 16) doubles so that the 8-byte
// DMMA fragment loads from a TMA-copied tile are shared-memory bank-conflict free.
// Also ≥ round8(n), so the DMMA m8 row tiles of the forward product stay inside a column;
// rows n..ld-1 are zero.
inline int64_t round8(int64_t n) { return (n + 7) / 8 * 8; }
inline int64_t padded_ld(int64_t n) {
  int64_t r8 = round8(n);
  return r8 + (((4 - r8) % 16) + 16) % 16;
}

struct Ctx;

struct NcclApi;  // dlopen'ed NCCL entry points (solve.cpp)

struct Ctx {
  int device = 0;
  int sms = 148;
  int64_t n = 0, p = 0, ld = 0;   // ld = padded leading dimension of X and Z
  double lam0 = 0, lam2 = 0, M = 0, rho = 0;
  double node_tol = 1e-4, int_tol = 1e-4;
  int check_every = 10, max_iters = 10000;
  double yy = 0;                  // ‖y‖²
  // device data (owned)
  double *X = nullptr, *Z = nullptr, *y = nullptr, *c = nullptr, *colsq = nullptr, *L = nullptr, *Lt = nullptr;
  // direct regime (p ≤ 2n and p ≤ 1056, R17): D = (XᵀX + ρI)⁻¹ = (I − ZᵀZ)/ρ, p×p, ld ldD
  double *D = nullptr;
  int64_t ldD = 0;
  int direct = 0;
  // ADMM work space for one pass of kBC nodes
  double *stt = nullptr;                                    // node state, per-tile blocks (admm.cu)
  double *bchk = nullptr;                                   // [p][kBC]
  double *U = nullptr, *Ub = nullptr;                       // [kBC][ld]
  double *Upart = nullptr;                                  // [grid][kBC][ld]
  double *sums = nullptr;                                   // [grid][kBC][kSums]
  double *sums2 = nullptr;                                  // [grid][kBC] ‖Xβ‖² partials
  int32_t *seg_idx = nullptr, *nz_idx = nullptr;            // sparse primal check (admm.cu)
  double *seg_val = nullptr, *nz_val = nullptr;
  int *seg_cnt = nullptr;
  int seg_cap = 0, nz_cap = 0;

  // matching-pursuit root heuristic work space (mp.cu, allocated on first use)
  double *mp_r = nullptr, *mp_beta = nullptr, *mp_log = nullptr;
  uint8_t* mp_inS = nullptr;
  int32_t* mp_S = nullptr;
  void* mp_cand = nullptr;
  int* mp_state = nullptr;

  double *node_f = nullptr;                                 // per-node scalars (admm.cu)
  int *node_i = nullptr;
  int *badflag = nullptr;
  unsigned* bar = nullptr;                                  // grid barrier words
  void* ub_scratch = nullptr;                               // Gram spill for very large supports
  size_t ub_scratch_bytes = 0;
  int grid = 0;
  int admm_cls = -1;                                        // n class of the ADMM kernel (admm.cu)
  // wide-n path (admm.cu): n beyond the fused kernel's on-chip budget; host-stepped kernels + GEMMs
  int wide = 0;
  double *wW = nullptr, *wB = nullptr;                      // w⁺ and β⁺ at checks, [p8][kBC]
  double *wXB = nullptr;                                    // Xβ⁺ at checks, [kBC][ld]
  double *wsum = nullptr;                                   // per-CTA check sums [nblk][kBC][4]
  int *wit0 = nullptr;                                      // iterations of the nodes before the launch
  double *wpart = nullptr;                                  // forward partials per column chunk [wcc][kBC][ld]
  int wrb = 0, wcc = 0;                                     // forward grid: row blocks × column chunks
  int64_t wcpc = 0;                                         // columns per chunk
  // scratch for batch I/O in solve (device)
  std::vector<void*> owned;
  int64_t bytes = 0;
  int64_t launches = 0;
  std::string err;
  // growable device scratch buffers (batch I/O)
  void* scr[6] = {};
  size_t scr_bytes[6] = {};
  void* scratch_n(int i, size_t b) {
    if (scr_bytes[i] < b) {
      if (scr[i]) cudaFree(scr[i]);
      scr[i] = nullptr;
      scr_bytes[i] = 0;
      if (cudaMalloc(&scr[i], b) != cudaSuccess) { cudaGetLastError(); return nullptr; }
      scr_bytes[i] = b;
    }
    return scr[i];
  }
  void* scratch(size_t b) { return scratch_n(0, b); }
  void* scratch2(size_t b) { return scratch_n(1, b); }
  std::vector<double> trace;   // l0l2_solve_trace records (8 doubles per node)
  // live kernel timing (l0l2_kernel_stats)
  l0l2_kstats ks{};
  cudaEvent_t ev[4] = {};
  // multi-GPU
  int nranks = 1, rank = 0;
  void* nccl_comm = nullptr;
  NcclApi* nccl = nullptr;
  cudaStream_t comm_stream = nullptr;
  // caller-provided host transport (l0l2_comm_init_transport): used instead of NCCL when set
  l0l2_transport host_tr{};
  bool host_tr_set = false;
  // kept across l0l2_solve calls (allocation and stream creation are not free): the warm-state
  // pool chunks, the round I/O block (sized for solve_buf_B nodes), the solve stream, the pool cap
  std::vector<double*> pool_chunks;
  void* solve_buf = nullptr;
  size_t solve_buf_bytes = 0;
  int64_t pool_chunk_bytes = 0;   // bytes per warm-pool chunk (2p doubles × slots per chunk)
  int solve_buf_B = 0;
  cudaStream_t solve_stream = nullptr;
  size_t pool_cap = 0;
  void* fr_state = nullptr;   // device frontier arrays (frontier.cu), kept across solves
  // column-sharded single-node ADMM (sharded.cu): this rank holds columns [col0, col0 + p) of p_total
  int sharded = 0;
  int shard_fused = 0;        // the fused step-mode kernel is available (n within the Z-form classes)
  int64_t col0 = 0, p_total = 0;
  void* sh_buf = nullptr;
  size_t sh_bytes = 0;
  Ctx* coop_view = nullptr;   // cooperative ramp-up: this rank's column block as a sharded view (solve.cu)
  void* gemm_ws = nullptr;    // split-K partials of gemm_f64
  size_t gemm_ws_bytes = 0;
};

int set_err(Ctx* c, int code, const char* fmt, ...);
int debug_prof(unsigned long long* out, int reset);   // -DL0L2_PROF builds only (admm.cu)
void* dalloc(Ctx* c, size_t bytes);   // tracked cudaMalloc (nullptr on failure)

#define L0L2_CUDA(ctx, expr)                                                            \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return ::l0l2::set_err((ctx), L0L2_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__,   \
                             #expr, cudaGetErrorString(e_));                          \
  } while (0)

#define L0L2_LAUNCHED(ctx)                                                              \
  do {                                                                                 \
    (ctx)->launches++;                                                                 \
    cudaError_t e_ = cudaGetLastError();                                               \
    if (e_ != cudaSuccess)                                                             \
      return ::l0l2::set_err((ctx), L0L2_ECUDA, "%s:%d launch: %s", __FILE__, __LINE__, \
                             cudaGetErrorString(e_));                                 \
  } while (0)

// ---- launchers (each returns an L0L2 status) -------------------------------------------
// C (M×N, col-major, ldc) = alpha * op(A) * op(B) + beta * C; op(A) M×K, op(B) K×N.
// transA: A stored K×M col-major (element (m,k) at A[k + m*lda]); else M×K (A[m + k*lda]).
// transB: B stored N×K col-major (element (k,n) at B[n + k*ldb]); else K×N (B[k + n*ldb]).
int gemm_f64(Ctx* c, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
             bool transA, const double* B, int64_t ldb, bool transB, double beta, double* C,
             int64_t ldc, cudaStream_t st);
int precompute(Ctx* c, cudaStream_t st);
int admm_alloc(Ctx* c);
// bound one group of ≤ kBC nodes whose code plane / warm state are already packed
struct BoundArgs {
  int nb;                       // nodes in this group (≤ kBC)
  const double* parent_lb;      // device [nb] or null
  double *lb, *primal;          // device [nb]
  int *iters;                   // device [nb]
  uint8_t* flags;               // device [nb]
  double prune_ub = INFINITY;   // stop a node once its best dual reaches this (early prune, R16)
  unsigned cold_mask = 0;       // nodes without a parent state: start at β = v = 0, no refresh (R6);
                                // also resumed nodes (their state continues as is)
  // continuous batching (§8(f) rank 2, solve.cu): resumed nodes' best dual and iterations so far
  // (device [nb] or null), where the launch writes them back, and the suspension rule
  const double* lbbest_in = nullptr;
  const int* it0_in = nullptr;
  double* out_lbbest = nullptr;
  int suspend_at = 0, susp_min = 0;
  // device frontier (frontier.cu): cold bits from the device warm-pointer array (null = cold) and the
  // early-prune threshold read from device memory at launch
  const double* const* warm_ptrs = nullptr;
  const double* prune_ub_dev = nullptr;
};
constexpr uint8_t kFlagSuspended = 16;   // node flag: suspended by continuous batching (internal)
int pack_group(Ctx* c, int nb, const int64_t* fix_off, const int32_t* fix_idx, const uint8_t* fix_val,
               const double* const* warm_ptrs_dev, cudaStream_t st);
int run_admm(Ctx* c, const BoundArgs& a, cudaStream_t st);
// step mode of the ADMM kernel (column-sharded fused path): one phase per launch (admm.cu)
int admm_step(Ctx* c, const BoundArgs& a, int phase, int chk, double* tot_out, cudaStream_t st);
int admm_step_decide(Ctx* c, const BoundArgs& a, int it, const double* tot, cudaStream_t st);
int admm_step_outputs(Ctx* c, const BoundArgs& a, cudaStream_t st);
int account_admm(Ctx* c, int nb, const int* iters_host);
void account_admm_stats(Ctx* c, int nb, const int* iters_host, float ms);   // same, given the launch's time
// device-frontier solve (frontier.cu): single rank, synchronous rounds
void frontier_free(Ctx* c);
int solve_device(Ctx* c, const l0l2_solve_opts& o, double* beta, double* obj, double* gap, l0l2_stats* stats);
int finalize_group(Ctx* c, int nb, double* zhat, int32_t* branch_j, uint8_t* flags,
                   int32_t* supp_cnt, int32_t* supp_idx, int64_t supp_stride, cudaStream_t st);
int unpack_warm(Ctx* c, int nb, double* const* warm_ptrs_dev, cudaStream_t st);
// device frontier: apply the fixing chains (records {parent, 2j + value}, rec_stride ints apart) of a
// packed group's nodes to its code plane / state (after pack_group with null fixings)
int scatter_chain_group(Ctx* c, int nb, const int* node_rec, const int* recs, int rec_stride, cudaStream_t st);
int dual_residual(Ctx* c, int nb, double* dual_r, int64_t ldr, cudaStream_t st);
int upper_batch(Ctx* c, int B, const int64_t* supp_off, const int32_t* supp_idx, double* obj,
                double* beta_s, cudaStream_t st);

// Algorithm 3 (matching pursuit) on the device; S_out ascending, beta_out length p.
int mp_run(Ctx* c, int max_rounds, cudaStream_t st, std::vector<int32_t>& S_out, std::vector<double>& beta_out,
           double* obj, int* rounds);

void comm_free(Ctx* c);   // also frees the cooperative ramp-up view
void coop_free(Ctx* c);
int shard_allreduce(Ctx* c, double* d, int64_t count, cudaStream_t st);   // solve.cu
int bound_sharded(Ctx* c, int B, const int64_t* fix_off, const int32_t* fix_idx, const uint8_t* fix_val,
                  const double* warm_in, const double* parent_lb, double* lb, double* primal, double* warm_out,
                  int32_t* iters, uint8_t* flags, cudaStream_t st);   // sharded.cu

}  // namespace l0l2

struct l0l2_ctx {
  l0l2::Ctx impl;
};

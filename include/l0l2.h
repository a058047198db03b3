/*
 * l0l2.h — C-ABI of the B200 (sm_100a) library for the data-parallel hot path of the
 * ℓ0–ℓ2 branch-and-bound of arXiv 2602.04551 (PAPER.md, cited as P:<line>).
 *
 *   problem (eq:original; Big-M perspective MIP eq:perspective):
 *       min_β ½‖y − Xβ‖² + λ0‖β‖₀ + λ2‖β‖²   s.t. ‖β‖∞ ≤ M
 *
 * Conventions shared by every entry point
 *   - All floating point is IEEE float64.  X is n×p COLUMN-major (column j = feature j,
 *     contiguous, leading dimension n).  Index arrays are 0-based int32 unless stated.
 *   - Return value: 0 = OK; negative = hard failure (L0L2_E*); positive = soft warning
 *     (L0L2_W*) whose outputs are still valid.  l0l2_last_error() gives a message.
 *   - A ctx owns all device memory it allocates and is bound to one CUDA device.  It is
 *     not thread-safe; separate ctxs (one per GPU / process) are independent.
 *   - No CPU fallback exists: every numeric step runs in this library's sm_100a kernels.
 *     Without a usable CUDA device l0l2_create returns L0L2_ECUDA.
 */
#ifndef L0L2_H_
#define L0L2_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define L0L2_OK          0
#define L0L2_EINVAL    (-1)   /* bad argument: n,p ≤ 0; λ2 ≤ 0; λ0 < 0; M ≤ 0; ρ < 0;
                                 F0 ∩ F1 ≠ ∅; index out of range; NaN/Inf in X or y */
#define L0L2_ENOMEM    (-2)   /* device or host allocation failed */
#define L0L2_ECUDA     (-3)   /* CUDA runtime error / no device */
#define L0L2_ENCCL     (-4)   /* NCCL error, or libnccl.so.2 not loadable */
#define L0L2_WNOTCONV    1    /* a node hit max_iters; its bound is still valid */
#define L0L2_WLIMIT      2    /* time or node limit reached; bounds are valid */

/* node flags (bit set) returned by l0l2_bound_batch */
#define L0L2_FLAG_CONVERGED 1u  /* relative primal-dual gap ≤ node_tol at a check */
#define L0L2_FLAG_INTEGRAL  2u  /* every free ẑ within int_tol of {0,1} (P:258 prune (i)) */
#define L0L2_FLAG_MAXITER   4u  /* stopped at max_iters */
#define L0L2_FLAG_PRUNED    8u  /* stopped early: best dual ≥ the prune threshold (l0l2_solve early_prune) */

typedef struct l0l2_ctx l0l2_ctx;

/* Options of the node relaxation (ADMM) and of the data placement. */
typedef struct {
  double  M;            /* Big-M box bound > 0; required, no default in the paper */
  double  rho;          /* ADMM penalty ρ > 0; 0 → mean_j ‖X_j‖² (R5)        */
  double  node_tol;     /* node stop: (P(β) − LB)/max(1,|P|) ≤ node_tol; default 1e-4;
                           a negative value disables the test (fixed-iteration mode)            */
  double  int_tol;      /* integrality tolerance on ẑ; default 1e-4                      */
  int32_t check_every;  /* dual/primal check cadence in iterations; default 10          */
  int32_t max_iters;    /* ADMM iteration cap per node; default 10000                    */
  int32_t device;       /* CUDA device ordinal                                                   */
  int32_t x_on_device;  /* 1: X, y passed to l0l2_create are device pointers on `device`; the
                           library synchronises the device before copying them, so writes
                           still pending on any stream complete first                          */
} l0l2_opts;

/* Fill `o` with the defaults above (M = 0 must then be set by the caller). */
void l0l2_default_opts(l0l2_opts* o);

/*
 * l0l2_create — copy (X, y) to HBM and run the tree-wide precompute:
 *   c = Xᵀy, colsq_j = ‖X_j‖², A = XXᵀ + ρI_n = LLᵀ (Cholesky), Z = L⁻¹X (n×p).
 * D = (XᵀX+ρI)⁻¹ = (I − ZᵀZ)/ρ is then applied implicitly (Woodbury, P:375 with the 1/ρ²
 * typo corrected, R1).  X and y are copied (host or device per opts->x_on_device)
 * and never aliased afterwards.  For p ≤ 2n (and p ≤ 1056) the direct regime is used: D =
 * (XᵀX + ρI)⁻¹ = (I − ZᵀZ)/ρ is precomputed (p×p) and the bound kernel streams D (R17).
 * For n > 1056 outside the direct regime (the fused kernel's tile ring of Z no longer fits one CTA's
 * shared memory) the node bounds run on the wide-n path (l0l2_admm_path = 2): same arithmetic and
 * outputs, Z streamed twice per iteration.
 * Errors: L0L2_EINVAL (see above), L0L2_ENOMEM, L0L2_ECUDA.
 * On error *out is NULL.
 */
int l0l2_create(const double* X, const double* y, int64_t n, int64_t p,
                double lambda0, double lambda2, const l0l2_opts* opts, l0l2_ctx** out);

/*
 * l0l2_bound_batch — lower bounds of B open nodes at once (batched ADMM).
 *
 * Node k has fixings F0 (z=0) and F1 (z=1): entries fix_idx[fix_off[k] .. fix_off[k+1])
 * with fix_val 0 → F0, 1 → F1.  Every node runs ADMM on eq:ADMM1 with the closed-form
 * updates eq:b_update, eq:minbetalower and eq:v_i-update,
 * warm-started from warm_in or cold (zeros).  Every check_every iterations the dual
 * bound of Proposition 1 is evaluated at r̂ = y − X b̂ and the primal objective of
 * eq:relaxnode2 at β; the node stops when the relative gap ≤ node_tol.
 *
 * ALL array arguments are DEVICE pointers on the ctx device (e.g. torch CUDA tensors),
 * ordered on `stream` (cudaStream_t, NULL = legacy default stream):
 *   in   fix_off   int64[B+1]        CSR offsets into fix_idx / fix_val
 *   in   fix_idx   int32[nnz]        coordinate indices, 0 ≤ idx < p, disjoint F0/F1 per node
 *   in   fix_val   uint8[nnz]        0 → F0, 1 → F1
 *   in   warm_in   double[B][2][p]   parent (β, v) per node, or NULL for cold starts
 *   in   parent_lb double[B]         inherited bounds, or NULL (−∞)
 *   out  lb        double[B]         max(best checked dual, parent_lb)  — a valid lower bound
 *   out  primal    double[B]         P(β) at the last check (upper bound of the relaxation)
 *   out  warm_out  double[B][2][p]   final (β, v) for the children, or NULL
 *   out  zhat      double[B][p]      ẑ recovered from β, or NULL
 *   out  dual_r    double[B][n]      r̂ = y − X b̂ at the last check, or NULL
 *   out  branch_j  int32[B]          most fractional free j (ties: larger |β_j|, lower j), −1 if integral
 *   out  iters     int32[B]          ADMM iterations run
 *   out  flags     uint8[B]          L0L2_FLAG_* bits
 * Returns L0L2_WNOTCONV if any node stopped at max_iters (its lb is still valid).
 * The per-node arithmetic is independent of B and of the other nodes (bitwise).  Nodes run in
 * groups of 16 per persistent kernel launch (two node halves on CTA pairs that share each Z tile
 * through L2); the call blocks until all groups are done.
 */
int l0l2_bound_batch(l0l2_ctx* ctx, int32_t B,
                     const int64_t* fix_off, const int32_t* fix_idx, const uint8_t* fix_val,
                     const double* warm_in, const double* parent_lb,
                     double* lb, double* primal, double* warm_out, double* zhat, double* dual_r,
                     int32_t* branch_j, int32_t* iters, uint8_t* flags, void* stream);

/*
 * l0l2_upper_batch — feasible objectives on B candidate supports.
 * For support S_k = supp_idx[supp_off[k] .. supp_off[k+1]) (sorted, distinct) minimise
 * eq:upperboundbeta U_S(β) = ½‖y − X_Sβ‖² + λ2‖β‖² s.t. |β_i| ≤ M by the fast proximal
 * gradient method with Nesterov extrapolation t/(t+3) and Armijo backtracking
 * (eq:fpg_extrapolate..eq:fpg_armijo), batched one CTA per support (Gram
 * Q = X_SᵀX_S + 2λ2I by a multi-warp pre-pass — or, for supports too large for shared memory
 * (|S| ≳ 670, up to ~4000), by a gather + DMMA GEMM into HBM — then the iterations in support space).
 * DEVICE pointers, ordered on `stream`:
 *   in  supp_off int64[B+1], supp_idx int32[nnz]
 *   out obj      double[B]     U_S(β) + λ0|S|  (objective of eq:perspective at z = 1_S)
 *   out beta_s   double[nnz]   β_S aligned with supp_idx (may be NULL)
 */
int l0l2_upper_batch(l0l2_ctx* ctx, int32_t B, const int64_t* supp_off, const int32_t* supp_idx,
                     double* obj, double* beta_s, void* stream);

/*
 * l0l2_matching_pursuit — the root heuristic of PAPER.md §"Matching Pursuit Algorithm"
 * (Algorithm 3; outline P:781-783), run on the device against the resident X.
 * S ← ∅, β ← 0, r ← y; each round: forward step (every j ∉ S scored by
 * Δ_j = −β_j c_j + ½β_j²D_j + λ0 with c = Xᵀr, D = ‖X_j‖² + 2λ2, β_j = Proj_[−M,M](c_j/D_j);
 * the argmin joins S if Δ < 0), then backward step (every j ∈ S scored by
 * Δ_j = β_j c_j + (½‖X_j‖² − λ2)β_j² − λ0 with the updated residual; the argmin leaves S if
 * Δ < 0); stop when a round changes nothing or after max_rounds (≤ 0 → 4p + 10).  Argmin ties
 * → lowest column index (R15).
 * HOST outputs: beta double[p] (zero off S), support int32[p capacity] ascending, *support_len,
 * *obj = ½‖y − Xβ‖² + λ2‖β‖² + λ0|S| (a feasible objective of eq:perspective), *rounds (may be NULL).
 * Errors: L0L2_EINVAL on NULL outputs, L0L2_ECUDA / L0L2_ENOMEM on device failures.
 */
int l0l2_matching_pursuit(l0l2_ctx* ctx, int32_t max_rounds, double* beta, int32_t* support, int32_t* support_len,
                          double* obj, int32_t* rounds);

/* Options of the branch-and-bound driver (Algorithm 1). */
typedef struct {
  double  gap_tol;          /* stop when (UB − LB)/UB ≤ gap_tol; default 1e-2   */
  double  time_limit_s;     /* ≤ 0: none                                                          */
  int64_t node_limit;       /* ≤ 0: none                                                          */
  int32_t batch;            /* B = nodes per round (the paper's K); default 16            */
  int32_t rebalance_every;  /* multi-GPU: rounds between frontier rebalancing; default 8         */
  int64_t warm_bytes_cap;   /* device bytes for parent warm states; 0 → 25% of free HBM          */
  int32_t verbose;          /* 1: one progress line per round on stderr                          */
  int32_t record;           /* 1: keep a per-node trace of this rank (l0l2_solve_trace)           */
  int32_t init_mp;          /* 1: initial incumbent from l0l2_matching_pursuit, refit on its support by
                               the upper-bound routine; 0 (default): β = 0            */
  int32_t early_prune;      /* 1: a node's ADMM stops at the first check whose best dual ≥ UB(1−1e-12),
                               UB = the incumbent at the start of its round (the node is pruned
                               anyway; R16); 0 (default): run to node_tol        */
  int32_t continuous;       /* continuous batching (P:272 reads the batch as a
                               snapshot): k > 0 → when at most k nodes of a 16-node launch are still
                               iterating (at a regular check, after ≥ 2·check_every iterations) while
                               open nodes wait, the launch suspends them; they resume bitwise where
                               they stopped in the next launch, next to fresh nodes.  Bounds and the
                               certificate are unchanged; the tree order (node ids) differs from the
                               synchronous rounds.  Single rank only.  0 (default): synchronous      */
  int32_t coop_rampup;      /* multi-GPU: 1 → until the frontier is
                               partitioned (every rank holds the same tree), the ranks solve each node
                               of a round TOGETHER through the column-sharded bound (rank r: its column
                               block of Z, one all-reduce of u per iteration) instead of each solving
                               all of them; the blocks of the final (β, v) are all-gathered into full warm
                               states.  Needs ≥ 8 columns per rank.  0 (default): redundant ramp-up   */
} l0l2_solve_opts;

void l0l2_default_solve_opts(l0l2_solve_opts* o);

typedef struct {
  int64_t nodes;            /* node relaxations solved (this rank)                               */
  int64_t node_iters;       /* Σ ADMM iterations over solved nodes (this rank)                   */
  int64_t rounds;           /* synchronous rounds                                                */
  int64_t max_open;         /* largest open-node count seen (this rank)                          */
  int64_t nodes_global;     /* Σ nodes over ranks                                                */
  int64_t node_iters_global;
  double  t_total, t_bound, t_upper, t_tree, t_comm;   /* seconds                              */
  double  lb, ub, gap;      /* certified global bounds at return                                 */
  int32_t status;           /* 0 optimal (queue exhausted), 1 gap reached, 2 node limit, 3 time limit */
  int32_t support_size;
  int64_t nodes_moved;      /* open nodes moved between ranks by frontier rebalancing (Σ over ranks) */
  int64_t suspensions;      /* continuous batching: node suspensions (each node resumed later)       */
  int64_t coop_rounds;      /* rounds solved cooperatively (column-sharded ramp-up, coop_rampup)      */
} l0l2_stats;

/*
 * l0l2_solve — certified best-first BnB (Algorithm 1, batched reading DESIGN.md R9).
 * Rounds: select ≤ B open nodes by (LB, id); l0l2_bound_batch on them (warm
 * started from the parent state kept in HBM); l0l2_upper_batch on the rounded supports
 * F1 ∪ {free: ẑ ≥ ½}; incumbent update; prune by LB ≥ UB(1−1e-12) or integral ẑ
 * (P:258); branch on the most fractional coordinate (R10).
 * With a communicator (l0l2_comm_init) the frontier is partitioned across ranks and the
 * incumbent / global LB / termination are exchanged every round over NCCL.
 * HOST outputs: beta double[p] (β*, zeros off the support), obj (UB), gap ((UB−LB)/UB);
 * stats may be NULL.  Every rank returns the same beta, obj and gap.
 * Returns L0L2_WLIMIT when a time/node limit stopped the search (bounds still valid).
 */
int l0l2_solve(l0l2_ctx* ctx, const l0l2_solve_opts* opts, double* beta, double* obj, double* gap,
               l0l2_stats* stats);

/* Per-node trace of the last l0l2_solve run with opts.record = 1 (this rank's nodes, in the
 * order they were solved; suspended launches of a node are not records, its finishing one is).
 * Record r occupies rec[10r .. 10r+9] =
 *   {node id, depth, LB, primal P(β), ADMM iterations, branch j (−1 = none), flags, UB on its support,
 *    parent id (−1 = root), fixing that created it: 2j + value (value 0 → F0, 1 → F1; −1 = root)}.
 * Returns the number of records available (may exceed max_nodes; only max_nodes are written). */
int64_t l0l2_solve_trace(const l0l2_ctx* ctx, double* rec, int64_t max_nodes);

/* Multi-GPU, one process per GPU (torch.distributed provides the process group and
 * broadcasts the id bytes).  NCCL is loaded at run time (libnccl.so.2).             */
int l0l2_nccl_unique_id(uint8_t out[128]);
/* Self-test of the NCCL carrier on one rank (device ordinal `device`): loads libnccl.so.2, builds a
 * 1-rank communicator and runs the collectives the multi-GPU exchange uses — in-place all-reduce of
 * doubles, all-gather, broadcast, a grouped send/recv to itself — checking the bytes.  L0L2_OK, or
 * L0L2_ENCCL / L0L2_ECUDA. */
int l0l2_nccl_selftest(int32_t device);
int l0l2_comm_init(l0l2_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t id[128]);

/* Alternative to NCCL: a caller-provided HOST transport (e.g. a gloo / MPI process group, or
 * several ranks sharing one GPU, which NCCL rejects).  Every callback is collective in the usual
 * sense, is called from the thread running l0l2_solve, moves HOST bytes, and returns 0 on success
 * (anything else aborts the solve with L0L2_ENCCL):
 *   allgather(user, in, out, bytes): out[r·bytes .. (r+1)·bytes) ← rank r's `in`, for every rank r
 *   send(user, buf, bytes, peer) / recv(user, buf, bytes, peer): blocking point-to-point; every
 *     send is matched by a recv of the same size issued by the peer in the same order
 *   bcast(user, buf, bytes, root): buf ← root's buf on every rank
 * The struct is copied; `user` must stay valid until l0l2_destroy.  Semantics of the exchange are
 * those of the NCCL path; only the carrier differs. */
typedef struct {
  void* user;
  int32_t (*allgather)(void* user, const void* in, void* out, int64_t bytes);
  int32_t (*send)(void* user, const void* buf, int64_t bytes, int32_t peer);
  int32_t (*recv)(void* user, void* buf, int64_t bytes, int32_t peer);
  int32_t (*bcast)(void* user, void* buf, int64_t bytes, int32_t root);
} l0l2_transport;
int l0l2_comm_init_transport(l0l2_ctx* ctx, int32_t nranks, int32_t rank, const l0l2_transport* t);

/*
 * Column-sharded single-node ADMM for the narrow-frontier phases of a tree (the
 * root, the ramp-up, narrow C2/C3-class trees), where node parallelism leaves GPUs idle.  Rank `rank`
 * of `nranks` holds columns [col0, col0 + p_r) of the n × p_total design matrix (X_r: n × p_r
 * column-major, host pointer; y: the full n-vector on every rank).  l0l2_create_sharded runs the
 * tree-wide precompute with A = Σ_r X_r X_rᵀ + ρI all-reduced over the ranks (ρ = 0 → the
 * mean of ‖X_j‖² over ALL columns) and keeps Z_r = L⁻¹X_r; the communicator is the caller's host
 * transport `t` (several ranks may share one GPU) or, if t is NULL, NCCL from `nccl_id` (one GPU per
 * rank).  Collective: every rank calls it.  The direct regime is not used (always the Z-form).
 * Errors: as l0l2_create, plus L0L2_EINVAL for inconsistent shard arguments, L0L2_ENCCL.
 */
int l0l2_create_sharded(const double* X_r, const double* y, int64_t n, int64_t p_r, int64_t col0, int64_t p_total,
                        double lambda0, double lambda2, const l0l2_opts* opts, int32_t nranks, int32_t rank,
                        const l0l2_transport* t, const uint8_t nccl_id[128], l0l2_ctx** out);

/*
 * l0l2_bound_sharded — the lower bounds of B ≤ 128 nodes (the semantics of l0l2_bound_batch: ADMM
 * on eq:ADMM1, warm starts P:543, dual of Proposition 1 and primal every check_every iterations, stop
 * at node_tol) computed by ALL ranks of a sharded context together: per iteration u = Σ_r Z_r w_r is
 * all-reduced (n × B doubles) and each rank updates its own columns; at checks the per-node dual /
 * primal terms and X_r β are all-reduced once.  Collective.  DEVICE pointers on `stream`:
 *   fix_off int64[B+1], fix_idx int32 (GLOBAL column indices; each rank applies its own), fix_val;
 *   warm_in double[B][2][p_r] (this rank's columns of (β, v)) or NULL (cold); parent_lb double[B] or NULL;
 *   out lb[B], primal[B], iters[B], flags[B] (identical on every rank), warm_out[B][2][p_r] or NULL.
 * Returns L0L2_WNOTCONV if a node stopped at max_iters.
 */
int l0l2_bound_sharded(l0l2_ctx* ctx, int32_t B, const int64_t* fix_off, const int32_t* fix_idx,
                       const uint8_t* fix_val, const double* warm_in, const double* parent_lb, double* lb,
                       double* primal, double* warm_out, int32_t* iters, uint8_t* flags, void* stream);

/* Frontier rebalancing plan used by l0l2_solve every rebalance_every rounds (pure host logic,
 * exported for tests).  counts[r] = open nodes on rank r.  While the emptiest rank holds fewer
 * than `batch` nodes and the fullest holds ≥ 2 more, move half the difference (ties → lowest
 * rank).  Writes up to max_moves triples (src, dst, k) into plan; returns the number of moves
 * (which may exceed max_moves), or −1 on bad arguments. */
int l0l2_rebalance_plan(int32_t nranks, const int64_t* counts, int64_t batch, int64_t* plan, int32_t max_moves);

/* Per-kernel device timing, measured with CUDA events on the stream each kernel is launched on
 * (accumulated since l0l2_create or the last reset).  admm_*: the persistent ADMM kernel;
 * bytes_alg / flops_alg are the ALGORITHMIC traffic / work of those launches: per iteration one
 * read of Z (8·n·p bytes) plus the node state (β, v read + write, fixation code: 33·p bytes per
 * node) and 4·n·p flops per node.  upper_*: the FPG kernel. */
typedef struct {
  int64_t admm_launches, admm_iters, admm_node_iters;
  double  admm_ms, admm_bytes_alg, admm_flops_alg;
  int64_t upper_launches;
  double  upper_ms;
  double  upper_bytes_alg;  /* Σ 8·n·|S| over the supports: the X_S gather of the Gram build */
} l0l2_kstats;
int l0l2_kernel_stats(l0l2_ctx* ctx, l0l2_kstats* out, int32_t reset);

/* Introspection: n, p, ρ actually used, device bytes held by the context (problem data, ADMM work
 * space, batch scratch, solve buffers, warm-state pool; all kept until l0l2_destroy, so this is
 * also the peak), and kernel launches so far. */
int l0l2_info(const l0l2_ctx* ctx, int64_t* n, int64_t* p, double* rho, int64_t* device_bytes,
              int64_t* kernel_launches);

/* Which ADMM implementation the context's node bounds run on:
 *   0 = the fused persistent kernel, Z-form (Z = L⁻¹X streamed once per iteration);
 *   1 = the fused persistent kernel, direct regime b = D w (p ≤ 2n, R17);
 *   2 = the wide-n path (n beyond the fused kernel's on-chip budget, n > 1056): a column-tiled
 *       adjoint + epilogue kernel and a split-K forward GEMM per iteration, same node state and
 *       arithmetic (Z read twice per iteration).
 * Negative on a null context. */
int l0l2_admm_path(const l0l2_ctx* ctx);

const char* l0l2_last_error(const l0l2_ctx* ctx);
void l0l2_destroy(l0l2_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* L0L2_H_ */

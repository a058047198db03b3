// Batched ADMM node lower bound (§3.1-§3.2) as ONE persistent,
// cooperative sm_100a kernel per group of kBC = 16 nodes.
//
// Per iteration t and node k (state β, v in HBM, layout [p][kBC] node-minor):
//   w  = c + ρβ − v                              (eq:b_update)
//   u  = Z w            (n)   forward  contraction, Z = L⁻¹X  (precompute.cu)
//   s  = Zᵀ u           (p)   adjoint  contraction
//   b  = (w − s)/ρ                               (= D w with D = (XᵀX+ρI)⁻¹, Woodbury, R1)
//   β⁺ = prox(b + v/ρ)                           (eq:minbetalower, R3)
//   v⁺ = v + ρ(b − β⁺)                           (eq:v_i-update)
//
// One-pass mapping: because the prox, the v-update and the next w
// are elementwise in the coordinate j, one sweep over 8-column tiles Z_J of Z does
//   adjoint  S_J = Z_Jᵀ u          (DMMA m8n8k4, K = n split over 14 warps)
//   epilogue b, β⁺, v⁺, w⁺ and the check sums for the 8×8 (column, node) block
//   forward  u⁺ += Z_J w⁺_J        (DMMA, accumulators in registers)
// from the SAME shared-memory copy of Z_J (a cp.async.bulk / TMA bulk copy, 3-stage ring
// with mbarriers), so Z is read from HBM once per iteration.
//
// Node halves and CTA pairs.  A CTA holds u (n×8) and its forward accumulator (n×8) in
// registers — half the register file each — so one CTA serves one node half (8 nodes).  Z's
// tiles are cut into G = grid fixed sub-ranges.  When both halves of the group have active
// nodes, CTAs 2P and 2P+1 both stream sub-ranges 2P and 2P+1 in the same order, one per half:
// the second read of each tile is an L2 hit, so HBM sees Z once per iteration for 16 nodes and
// every SM does 8-node DMMA work on twice the tiles (FP64-bound instead of HBM-bound).  When
// only one half is active, every CTA streams its own sub-range for that half.  Forward partials,
// check sums and nonzero lists are kept per sub-range and reduced across the grid in a fixed
// order, so a node's arithmetic is bitwise the same in either mode, in any slot, for any B.
//
// Direct regime (p ≤ 2n, the paper's D branch P:374, R17): the same kernel streams the
// tiles of the precomputed p×p D = (I − ZᵀZ)/ρ instead of Z; the adjoint contraction then IS b = D w
// (u := w), the epilogue writes w⁺ straight to the next sweep's u buffer (double-buffered by sweep
// parity) and there is no forward contraction and no cross-CTA reduction.
//
// Checks (every check_every iterations) use identities that need no pass over X:
//   Xᵀr̂ = c − s,  ‖X b‖² = bᵀs   ⇒  dual(r̂ = y − Xb) = ½‖y‖² − ½ bᵀs − Σ ν_j(|c_j − s_j|)
//   primal P(β) = ½‖y‖² − cᵀβ + ½‖Xβ‖² + Σ ψ_j(β_j)
// where ‖Xβ‖² is a gather over β⁺'s nonzeros (dense β⁺: one forward-only sweep Zβ, ‖L(Zβ)‖²).
#include <cmath>
#include <cstdlib>

#include "common.cuh"

namespace l0l2 {
namespace {

constexpr int NW = kAdmmThreads / 32;   // 16 warps: 14 MMA + 2 epilogue
constexpr int NEW = 2;                  // epilogue warps
constexpr int NH = kBC / 8;             // node halves (one per CTA of a pair)
static_assert(NH == 2, "a CTA pair serves the two node halves");
constexpr int F_ACTIVE = 64;            // internal node flag bit (not exported)
constexpr int F_COLD = 128;             // internal: cold node (β = v = 0, no warm refresh) or a
                                        // resumed (suspended) node: its state continues, no refresh
constexpr int F_SUSP = 32;              // internal: suspended at a check (continuous batching, §8(f) rank 2)

struct KP {
  const double* __restrict__ Z;
  const double* __restrict__ Lt;   // Lᵀ, col-major ld (column i = row i of L)
  double* stt;                     // node state in tile blocks (st_* below)
  double* bchk;                    // b at the last check, [p][kBC]
  double* U; double* Ub; double* Upart; double* sums; double* sums2;
  // nonzeros of β⁺ at check iterations (sparse primal): per-CTA segments in tile
  // order, then a dense per-node list in CTA order
  int32_t* seg_idx; double* seg_val; int* seg_cnt;   // [grid][kBC][seg_cap], [grid][kBC]
  int32_t* nz_idx; double* nz_val;                     // [kBC][nz_cap]
  const double* __restrict__ X;                        // column-major, ld
  int seg_cap, nz_cap;
  double* nodef;                   // [kBC][4]: lb_best, primal, parent_lb, last dual
  int* nodei;                      // [kBC][2]: flags, iters
  unsigned* bar;                   // [2]: count, generation
  double* out_lb; double* out_primal; int* out_iters; uint8_t* out_flags;
  int64_t ld, n, n8, p8;           // streamed operand (Z, or D in the direct regime): ld, rows, rows/8·8
  int64_t xld, xn;                  // X (sparse primal gather) and Lᵀ: leading dimension, rows
  int direct;                       // direct regime (R17): b = D w, w⁺ written to U, no forward / reduction
  int ntiles, nsr, nb, check_every, max_iters, pfd;   // nsr: tile sub-ranges (= grid)
  unsigned act_mask;               // node slots run by this launch (outputs written for these only)
  double prune_ub;                 // early prune threshold (R16; +inf = off)
  const double* prune_ub_dev;      // or read from device memory at launch (device frontier), if set
  int suspend_at;                  // continuous batching: at a check with ≤ suspend_at active nodes (and
                                   // ≥ susp_min iterations in this launch) the launch suspends them (0 = off)
  int susp_min;
  double* out_lbbest;              // [nb] running max of checked duals (to resume a suspended node), or null
  // step mode (column-sharded fused path, sharded.cu): the launch runs ONE phase and exits, the host
  // all-reduces U (and at checks the per-node check totals and Zβ) across the ranks in between:
  //   phase 0: u0 sweep (forward-only from w0) + reduction into U
  //   phase 1: the warm refresh sweep + reduction
  //   phase 2: one fused iteration + reduction; at a check also this rank's check totals (tot_out)
  //            and Z_r β⁺ reduced into Ub (the decision runs in step_decide after the all-reduce)
  int step_mode, step_phase, step_chk;
  double* tot_out;                 // [kBC][4] this rank's Σ of the check terms (phase 2, check)
  int compact;                     // node-slot compaction allowed (tuning / test hook)
  int gather_mode;                 // primal check gather: 0 = whole columns (Z-form), 1 = row slices
  int pfs;                         // tiles L2-prefetched by prefill (during the grid reduction)
  int tsplit;                      // bulk copies per Z tile (divides kPt)
  double rho, inv_rho, lam0, lam2, M, yy, node_tol;
  double shrink, sr, a_l1, a_4, psi_l1, psi_4, zsr;
  bool sr_le_M;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
#ifndef L0L2_DEBUG_HANG
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(saddr(b)), "r"(phase) : "memory");
}
#else
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
  for (long long spin = 0;; spin++) {
    unsigned ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(saddr(b)), "r"(phase) : "memory");
    if (ok) return;
    if (spin == 2000000) {
      printf("HANG mbar blk %d tid %d bar %p phase %u\n", blockIdx.x, threadIdx.x, b, phase);
      __trap();
    }
  }
}
#endif
// TMA bulk copy global → shared (SASS UBLKCP), completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(b))
      : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Grid-wide barrier (sense by generation counter); the kernel is launched cooperatively so
// all CTAs are co-resident.
__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned gen;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
    __threadfence();
    unsigned prev = atomicAdd(bar, 1u);
    if (prev == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(bar + 1), "r"(gen + 1) : "memory");
    } else {
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
      } while (cur == gen);
    }
    __threadfence();
  }
  __syncthreads();
}

// ---------------------------------------------------------------- the operators
__device__ __forceinline__ double Tbox(double t, double a, double m) {   // eq:Tdef
  double at = fabs(t);
  if (at <= a) return 0.0;
  if (at <= a + m) return copysign(at - a, t);
  return copysign(m, t);
}
__device__ __forceinline__ double prox(const KP& k, double bt, uint8_t code) {   // eq:minbetalower
  if (code == 1) return 0.0;
  double quad = Tbox(k.shrink * bt, 0.0, k.M);
  if (code == 2) return quad;
  if (k.sr_le_M) return fabs(bt) >= k.a_l1 + k.sr ? quad : Tbox(bt, k.a_l1, k.M);
  return Tbox(bt, k.a_4, k.M);
}
__device__ __forceinline__ double psi_f(const KP& k, double b, uint8_t code) {   // eq:psi
  double ab = fabs(b);
  if (code == 1) return b == 0.0 ? 0.0 : INFINITY;
  if (ab > k.M) return INFINITY;
  if (code == 2) return k.lam0 + k.lam2 * b * b;
  if (k.sr_le_M) return ab >= k.sr ? k.lam0 + k.lam2 * b * b : k.psi_l1 * ab;
  return k.psi_4 * ab;
}
__device__ __forceinline__ double h_f(const KP& k, double x) {                    // eq:hdef
  return x <= 2.0 * k.M * k.lam2 ? x * x / (4.0 * k.lam2) - k.lam0 : k.M * x - k.lam0 - k.lam2 * k.M * k.M;
}
__device__ __forceinline__ double nu_f(const KP& k, double x, uint8_t code) {     // eq:nudef2
  if (code == 1) return 0.0;
  if (code == 2) return h_f(k, x);
  if (k.sr_le_M) return fmax(h_f(k, x), 0.0);
  return fmax(k.M * x - k.lam0 - k.lam2 * k.M * k.M, 0.0);
}

// ---------------------------------------------------------------- shared memory layout
#ifndef L0L2_NST
#define L0L2_NST 3
#endif
constexpr int NST = L0L2_NST;  // Z tile stages in the TMA ring (3 × 64.75 KB at n = 1000)
constexpr int PFD_DEFAULT = 0; // tiles prefetched into L2 beyond the smem ring (k.pfd); 0 measured best on the C4 step
                               // (92.6 vs 89.2 nodes/s, profiles/sweeps_r02/) and at C3; 1 is ~1% faster at C4 B ≤ 8
#ifndef L0L2_NMW
#define L0L2_NMW 14
#endif
constexpr int NMW = L0L2_NMW;  // MMA warps (adjoint + forward); warps NMW, NMW+1 run the epilogue
                               // (with 12 MMA warps the last 2 warps idle during sweeps)
static_assert(NMW + NEW <= NW, "warp roles");
constexpr int MMA_THREADS = NMW * 32;
// n classes of the kernel: KS adjoint k-steps (4 rows) and MT forward row tiles (8 rows) per MMA
// warp, so n8 ≤ min(4·NMW·KS, 8·NMW·MT).  (19, 10) is the largest class; the 3-stage tile ring then
// caps n at 1056 (shared memory, checked in admm_alloc).  (16 MMA warps would
// balance the 4 SM sub-partitions, but 18 warps leave 96 registers per thread: u and the forward
// accumulators no longer fit.)
constexpr int NCLS = 5;
#if L0L2_NMW == 12
constexpr int CLS_KS[NCLS] = {2, 6, 10, 16, 22};
constexpr int CLS_MT[NCLS] = {1, 3, 5, 8, 11};
#else
constexpr int CLS_KS[NCLS] = {2, 5, 10, 18, 19};
constexpr int CLS_MT[NCLS] = {1, 3, 5, 9, 10};
#endif

// Per-stage copy of the epilogue's operands for tile J, TMA'd with Z_J on the same mbarrier:
//   β_J [8][kBC], v_J [8][kBC], c_J [8], code_J [8][kBC] bytes (node-minor, as in HBM; a CTA
//   uses its half's 8 nodes of each row)
constexpr int STB = kPt * kBC;                             // (column, node) elements per tile
constexpr int STQ = (STB + STB + 8 + STB / 8 + 15) / 16 * 16;   // doubles per stage (128-B multiple)
constexpr unsigned STQ_BYTES = 8 * STQ;
// The node state lives in HBM in the same per-tile blocks ("stt", STQ doubles per 8-column tile),
// so each stage needs ONE bulk copy for all of it:  β at st_beta(j, nd), v at st_beta(j, nd) + STB,
// c_j at st_c(j), the fixation code byte at st_code(j, nd).
__host__ __device__ __forceinline__ int64_t st_beta(int64_t j, int nd) { return (j >> 3) * STQ + (j & 7) * kBC + nd; }
__host__ __device__ __forceinline__ int64_t st_c(int64_t j) { return (j >> 3) * STQ + 2 * STB + (j & 7); }
__device__ __forceinline__ uint8_t& st_code(double* stt, int64_t j, int nd) {
  return reinterpret_cast<uint8_t*>(stt + (j >> 3) * STQ + 2 * STB + 8)[(j & 7) * kBC + nd];
}
__device__ __forceinline__ uint8_t st_code(const double* stt, int64_t j, int nd) {
  return reinterpret_cast<const uint8_t*>(stt + (j >> 3) * STQ + 2 * STB + 8)[(j & 7) * kBC + nd];
}

struct Smem {
  double* tiles;      // [NST][kPt][ld]   Z_J ring (stage q at tiles + q·kPt·ld)
  double* stq;        // [NST][STQ]       β_J, v_J, c_J, code_J of the staged tile
  double* spart;      // [2][NMW][64]     adjoint partials per MMA warp (double buffered)
  double* Ws;         // [2][8][12]       w⁺_J of the CTA's half (node-major, padded; double
                      //                  buffered), then [2 sub-ranges][64][4] check-sum stash
  double* red;        // [kBC]            running max of checked duals (R7)
  uint64_t* mbar;     // [NST]
  uint64_t* sready;   // [2]              S_J partials ready / w⁺ buffer free (NMW arrivals)
  uint64_t* wready;   // [2]              w⁺_J ready (NEW arrivals)
  int* flags;         // [kBC]
  unsigned* rel;      // [NST] MMA warps done with the stage (last one refills it)
  int* ncnt;          // [kBC]            per-node β⁺ nonzero totals at a check (lmatvec fallback)
  int* stile;         // [NST]            tile held by each ring slot (−1: end of this CTA's sweep)
  int* zres;          // [NST]            tile whose Z_J is in the slot (−1: none yet)
  int* it0;           // [kBC]            iterations a (resumed) node had run before this launch
  int* sched;         // [9]              sweep number, stages issued, tiles taken, done (issuer
                      //                  only); node half, paired, tile range [t0, t1) of the sweep,
                      //                  issue deferred
};

// Producer → consumer hand-offs inside the CTA are mbarriers, not named barriers: a named barrier
// holding all MMA warps would also make every MMA warp wait for the slowest one each tile.
//   sready[par]: MMA warps → epilogue "S_J partials of tile t written" (one arrival per MMA warp;
//                in forward-only sweeps: "w⁺ buffer par free")
//   wready[par]: epilogue → MMA warps "w⁺_J(t) written" (one arrival per epilogue warp)
__device__ __forceinline__ void mbar_arrive_warp(uint64_t* b) {
  __syncwarp();   // orders the lanes' shared-memory writes before lane 0's release-arrive
  if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}

enum { SW_FWD_W = 0, SW_FWD_BETA = 1, SW_FUSED = 2 };

// Developer instrumentation (-DL0L2_PROF): per-warp clock64 totals of each wait / work phase,
// read back with l0l2_debug_prof (tools/prof_phases.py).  Compiled out otherwise.
#ifdef L0L2_PROF
__device__ unsigned long long g_prof[160][NW][8];
#define PROF_T0() long long pt_ = clock64()
#define PROF_RESET() pt_ = clock64()
// per-warp totals in shared memory (a global read-modify-write per phase would distort the timing);
// flushed to g_prof once at the end of the launch
__shared__ unsigned long long prof_s[NW][8];
#define PROF_ACC(slot) do { long long n_ = clock64(); if ((threadIdx.x & 31) == 0) prof_s[threadIdx.x >> 5][slot] += (unsigned long long)(n_ - pt_); pt_ = n_; } while (0)
#else
#define PROF_T0() do {} while (0)
#define PROF_RESET() do {} while (0)
#define PROF_ACC(slot) do {} while (0)
#endif

__device__ __forceinline__ unsigned tile_bytes(const KP& k) { return (unsigned)(kPt * k.ld * sizeof(double)); }

// stage t → ring slot sg: Z_J plus the epilogue operands of the same columns (one mbarrier)
// Resident tiles: a slot keeps the Z_J it last received (zres[slot] = its tile), so when a CTA's tiles
// of a sweep fit the ring (≤ NST tiles, e.g. C2's 125 tiles of D on ≥ 124 CTAs) every later sweep
// re-stages only the tile's state block — Z_J stays in shared memory for the whole launch.
__device__ __forceinline__ void issue_stage(const KP& k, Smem& s, int t, int sg) {
  const unsigned tb = tile_bytes(k);
  const bool have = s.zres[sg] == t;
  mbar_expect_tx(&s.mbar[sg], (have ? 0u : tb) + STQ_BYTES);
  // Z_J as k.tsplit bulk copies of kPt/tsplit whole columns each (1 is fastest: every copy issued
  // costs the issuing MMA warp time on the critical path)
  const int cpc = kPt / k.tsplit;
  if (!have) {
    s.zres[sg] = t;
    for (int c = 0; c < kPt; c += cpc)
      bulk_g2s(s.tiles + (size_t)sg * kPt * k.ld + c * k.ld, k.Z + ((int64_t)t * kPt + c) * k.ld,
               (unsigned)(cpc * k.ld * sizeof(double)), &s.mbar[sg]);
  }
  // the tile's whole state block (β_J, v_J, c_J, code_J) in one copy
  bulk_g2s(s.stq + sg * STQ, k.stt + (int64_t)t * STQ, STQ_BYTES, &s.mbar[sg]);
}

// Tile scheduling.  Every sweep streams all tiles of Z once.  Sub-range r < G = gridDim.x is
// the fixed tile range [T(r), T(r+1)), T(r) = ⌊ntiles·r/G⌋ (bitwise deterministic, independent of
// the batch composition).  The CTA streams one contiguous range per sweep (set by prefill: its own
// sub-range, or its pair's two).  The stages a CTA consumes are numbered m = 0, 1, ... in ring
// order (slot m % NST): stage m holds tile t0 + m while m < t1 − t0, then one end-marker stage (tile
// −1, a plain arrive, no copy) at which consumers stop; nothing is issued past it.  Stage m is a
// function of m alone (issue_stage_m), so the thread that refills a slot needs no shared scheduler
// state.  The tile id is written before the (release) arrive, so every consumer reads it after its
// (acquire) wait on the stage's mbarrier.  (A dynamic, grid-wide ticket schedule was measured and
// gave nothing.)
__device__ __forceinline__ int sub_t(const KP& k, int r) { return (int)((int64_t)k.ntiles * r / k.nsr); }

__device__ void issue_stage_m(const KP& k, Smem& s, int m, int t0, int t1) {
  if (m > t1 - t0) return;
  const int sg = m % NST;
  const int tile = m < t1 - t0 ? t0 + m : -1;
  s.stile[sg] = tile;
  if (tile >= 0) {
    fence_proxy_async_smem();
    issue_stage(k, s, tile, sg);
    if (k.pfd > 0 && tile + k.pfd < t1) prefetch_l2(k.Z + (int64_t)(tile + k.pfd) * kPt * k.ld, tile_bytes(k));
  } else {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(&s.mbar[sg])) : "memory");
  }
}

// Start sweep number `sw`: choose the CTA's node half and tile range from the node flags, then
// issue the first NST stages.  Called by thread 0 once before the first sweep and again at the end
// of every sweep (so the next sweep's first tiles stream in while the grid reduces u; the flags it
// sees may still include nodes that the coming check retires, which only costs idle DMMA slots).
// Paired: both halves active → CTA g serves half g&1 on sub-ranges 2⌊g/2⌋, 2⌊g/2⌋+1.  Otherwise
// CTA g serves the active half on sub-range g.  Every CTA decides from the same flags.  While the
// mode stays, the CTA's next tiles hold β, v rows of its half that it wrote itself (epilogue
// threads: generic → async proxy fence, then the CTA barrier before this call).  When the mode
// changes, those rows may have been written by the partner CTA, which may still be sweeping: the
// issue is deferred (sched[8]) to the start of the next sweep, which follows a grid barrier.
__device__ void issue_first(const KP& k, Smem& s) {
  fence_proxy_async_smem();   // the launch's generic zeroing of the ring precedes its first TMA writes
  for (int m = 0; m < NST; m++) issue_stage_m(k, s, m, s.sched[6], s.sched[7]);
  // the grid reduction that follows leaves HBM idle: pull the sweep's next tiles into L2 meanwhile
  const int t0 = s.sched[6], t1 = s.sched[7];
  for (int t = t0 + NST + k.pfd; t < t1 && t < t0 + NST + k.pfs; t++) prefetch_l2(k.Z + (int64_t)t * kPt * k.ld, tile_bytes(k));
}

// The CTA's node half and tile range of a sweep, from the current node flags (every CTA decides
// from the same flags).  Paired: both halves active → CTA g serves half g&1 on sub-ranges
// 2⌊g/2⌋, 2⌊g/2⌋+1.  Otherwise CTA g serves the active half on sub-range g.
__device__ void choose_mode(const KP& k, Smem& s) {
  const int g = blockIdx.x;
  int a0 = 0, a1 = 0;
  for (int nd = 0; nd < 8; nd++) {
    a0 |= s.flags[nd] & F_ACTIVE;
    a1 |= s.flags[8 + nd] & F_ACTIVE;
  }
  const bool paired = a0 && a1;
  s.sched[4] = paired ? (g & 1) : (a0 ? 0 : 1);
  s.sched[5] = paired;
  s.sched[6] = paired ? sub_t(k, g & ~1) : sub_t(k, g);
  s.sched[7] = paired ? sub_t(k, (g & ~1) + 2) : sub_t(k, g + 1);
}

// Start sweep number `sw` (thread 0, after the CTA barrier that ends the previous sweep): issue its
// first NST stages now, so they stream in while the grid reduces u — unless a check decision
// (which may retire nodes, change the mode and permute node slots) comes before that sweep
// (defer): then mode and first stages are settled at the start of the sweep (deferred_start),
// after the grid barrier.  The CTA's next tiles hold β, v rows that it wrote itself (epilogue:
// generic → async proxy fence before the CTA barrier) while the mode stays; any other case
// crosses a grid barrier first.
__device__ void prefill(const KP& k, Smem& s, int sw, bool defer) {
  s.sched[0] = sw;
  s.sched[8] = defer;
  // stages issued now and not yet consumed (waited for by the drain at the end of the launch)
  s.sched[1] = 0;
  if (defer) return;
  choose_mode(k, s);
  s.sched[1] = min(NST, s.sched[7] - s.sched[6] + 1);
  issue_first(k, s);
}

// One sweep over this CTA's tiles, warp-specialised:
//   MMA warps (0..NMW−1):  adj(t0); for t: [adj(t+1)] → wait w⁺(t) → fwd(t) → release stage(t)
//   epilogue warps:        for t: wait S(t) → b, β⁺, v⁺, w⁺, check sums → publish w⁺(t)
// so the elementwise epilogue of tile t overlaps the DMMA adjoint of tile t+1.  u of this
// iteration lives in registers as the adjoint's B fragments (MMA warp w owns k-steps [ks0, ks1),
// lane holds U[row = 4q + lane%4][node = 8h + lane/4]).  Forward partials go to Upart[sub-range],
// check sums to sums[sub-range], per sub-range (a paired CTA flushes at its sub-range boundary).
template <int MODE, int KS, int MT, bool DIR>
__device__ void sweep(const KP& k, Smem& s, bool refresh, bool check, unsigned& phases, unsigned& hph,
                      double* sums_out = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.x;
  constexpr bool fused = (MODE == SW_FUSED);
  const bool is_mma = warp < NMW;
  const bool is_epi = warp >= NMW && warp < NMW + NEW;
  if (s.sched[8]) {   // deferred start (prefill); a grid barrier has passed.  (sched[8] is rewritten
                      // only by the next prefill, so every thread takes this branch.)
    if (tid == 0) {
      choose_mode(k, s);
      issue_first(k, s);
    }
    __syncthreads();   // the mode below, and the scheduler state before the in-sweep issuers
  }
  // this sweep's node half and sub-ranges (s.sched[4..7] do not change until the CTA barrier at
  // the end of the sweep)
  const int h = s.sched[4];
  const bool paired = s.sched[5] != 0;
  const int sr0 = paired ? (g & ~1) : g;
  const int tb = paired ? sub_t(k, sr0 + 1) : 0x7fffffff;   // first tile of the second sub-range
  const int t0s = s.sched[6], t1s = s.sched[7];               // this sweep's tile range
  // direct regime (R17): this sweep reads w from uin and writes w⁺ to uout (double-buffered by
  // sweep parity; a CTA may finish its tiles while another still loads its u fragments)
  const double* uin = (DIR && (s.sched[0] & 1)) ? k.Ub : k.U;
  double* uout = (DIR && (s.sched[0] & 1)) ? k.U : k.Ub;
  // wait for ring stage m; returns its tile (−1: the CTA's sweep is over)
  auto stage = [&](int m) {
    const int sg = m % NST;
    mbar_wait(&s.mbar[sg], (phases >> sg) & 1u);
    phases ^= 1u << sg;
    return s.stile[sg];
  };

  if (is_mma) {
    // Branch-free fragment schedule (so every shared-memory fragment load is an immediate offset
    // from one base and can be hoisted ahead of its DMMA): warp w owns adjoint k-steps q = w + NMW·i
    // (i < KS) and forward row tiles m = w + NMW·i (i < MT).  Indices past n8 read rows beyond the
    // column (Z's zero padding, the next column, or — past the ring — the staged state blocks): their
    // u fragment is 0 and their forward accumulator is never stored.  Those reads must be finite
    // (NaN·0 = NaN), so the ring and the state stages are zeroed at launch (stale shared memory of
    // an earlier kernel could hold any bit pattern) and only ever receive Z and state blocks.
    const int mt = (int)(k.n8 / 8);
    const int kt = (int)(k.n8 / 4);
    const int ld = (int)k.ld;
    const int cA = lane >> 2, kA = lane & 3;
    double acc[MT][2];
#pragma unroll
    for (int i = 0; i < MT; i++) acc[i][0] = acc[i][1] = 0.0;
    double uf[KS];
    const bool uact = (s.flags[8 * h + cA] & F_ACTIVE) != 0;
#pragma unroll
    for (int i = 0; i < KS; i++) {
      const int q = warp + NMW * i;
      uf[i] = (fused && uact && q < kt) ? __ldcg(uin + (8 * h + cA) * ld + q * 4 + kA) : 0.0;
    }
    // this CTA's forward partial of sub-range sr: Upart[sr][8h + node][row]; then restart
    auto flush = [&](int sr) {
      double* up = k.Upart + ((int64_t)sr * kBC + 8 * h) * k.ld;
#pragma unroll
      for (int i = 0; i < MT; i++) {
        const int m = warp + i * NMW;
        if (m < mt) {
          const int row = m * 8 + (lane >> 2), nd = 2 * (lane & 3);
          up[(int64_t)nd * k.ld + row] = acc[i][0];
          up[(int64_t)(nd + 1) * k.ld + row] = acc[i][1];
        }
        acc[i][0] = acc[i][1] = 0.0;
      }
    };
    bool flushed = !paired;
    int ctile = -1;   // tile of stage m (forward)
    // adjoint of stage m (fused sweeps); false at the end marker
    int ntile = -1;
    auto adjoint = [&](int m) {
      PROF_T0();
      const int tile = stage(m);
      ntile = tile;
      PROF_ACC(0);
      if (tile < 0) return false;
      const double* T = s.tiles + (size_t)(m % NST) * kPt * ld + cA * ld + kA;
#ifndef L0L2_ADJ_CHAINS
#define L0L2_ADJ_CHAINS 4
#endif
      constexpr int NCH = L0L2_ADJ_CHAINS;   // independent DMMA accumulator chains of the adjoint
      double sc[NCH][2];
#pragma unroll
      for (int c = 0; c < NCH; c++) sc[c][0] = sc[c][1] = 0.0;
#pragma unroll
// EXP_NOADJ / EXP_NOFWD / EXP_NOEPI: timing experiments only (the results are wrong), built with
// tools/build_variant.py — they compile out the adjoint DMMAs, the forward DMMAs or the epilogue math
// to measure what the tile pipeline costs without them.
#ifndef EXP_NOADJ
      for (int i = 0; i < KS; i++) dmma(sc[i % NCH], T[4 * (warp + NMW * i)], uf[i]);
#endif
      double* sp = s.spart + (m & 1) * NMW * 64 + warp * 64;
      // C fragment: row (col j) = lane>>2, cols (node) = 2*(lane&3) + {0,1}
      if (NCH == 4) {
        sp[cA * 8 + 2 * kA] = (sc[0][0] + sc[1][0]) + (sc[2 % NCH][0] + sc[3 % NCH][0]);
        sp[cA * 8 + 2 * kA + 1] = (sc[0][1] + sc[1][1]) + (sc[2 % NCH][1] + sc[3 % NCH][1]);
      } else {
        sp[cA * 8 + 2 * kA] = sc[0][0] + sc[1 % NCH][0];
        sp[cA * 8 + 2 * kA + 1] = sc[0][1] + sc[1 % NCH][1];
      }
      mbar_arrive_warp(&s.sready[m & 1]);
      PROF_ACC(1);
      return true;
    };
    bool cur;
    if (fused) { cur = adjoint(0); ctile = ntile; }
    else { ctile = stage(0); cur = ctile >= 0; }
    for (int m = 0; cur; m++) {
      const int sg = m % NST;
      const bool nxt = fused ? adjoint(m + 1) : true;
      PROF_T0();
      if (!flushed && ctile >= tb && !DIR) { flush(sr0); flushed = true; }
      mbar_wait(&s.wready[m & 1], (hph >> (m & 1)) & 1u);   // w⁺_J(m) published
      hph ^= 1u << (m & 1);
      PROF_ACC(2);
      const double* T = s.tiles + (size_t)sg * kPt * ld + kA * ld + cA;
      const double* W = s.Ws + (m & 1) * 8 * 12;
      // ---- forward: U⁺(rows × 8 nodes) += Z_J (rows × 8 cols) · W_J (8 cols × 8 nodes)
      const double b0 = W[cA * 12 + kA];         // B[k = j][n = node]
      const double b1 = W[cA * 12 + 4 + kA];
      // two passes (k = cols 0-3, then 4-7), so consecutive DMMAs never share an accumulator (the
      // asm volatile DMMAs issue in source order; back-to-back dependent pairs stalled on latency)
#ifndef EXP_NOFWD
      if (!DIR) {
#pragma unroll
        for (int i = 0; i < MT; i++) dmma(acc[i], T[8 * (warp + NMW * i)], b0);          // A[m = row][k = col j]
#pragma unroll
        for (int i = 0; i < MT; i++) dmma(acc[i], T[4 * ld + 8 * (warp + NMW * i)], b1);
      }
#endif
      PROF_ACC(3);
      if (!fused) mbar_arrive_warp(&s.sready[m & 1]);   // w⁺ buffer m&1 free again
      // release stage m: the last MMA warp to finish its forward refills the slot with stage m + NST
      // (no CTA barrier, no shared scheduler state: a relaxed counter suffices; the reset is ordered
      // before the next use of the counter by the refill's release-arrive on the stage mbarrier).
      // (Issuing from an epilogue warp instead was measured slower: the refill then waits for it.)
      __syncwarp();
      if (lane == 0) {
        unsigned old;
        asm volatile("atom.relaxed.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(saddr(&s.rel[sg])) : "memory");
        if (old == NMW - 1) {
          s.rel[sg] = 0;
          issue_stage_m(k, s, m + NST, t0s, t1s);
        }
      }
      __syncwarp();
      PROF_ACC(4);
      if (fused) { cur = nxt; ctile = ntile; }
      else { ctile = stage(m + 1); cur = ctile >= 0; }
    }
    if (!DIR) {
      if (!flushed) flush(sr0);
      flush(paired ? sr0 + 1 : sr0);
    }
  } else if (is_epi) {
    // ---------------- epilogue warps: element (j = et>>3, node = 8h + (et&7)) of each 8×8 block
    const int et = tid - MMA_THREADS, j = et >> 3, nd = et & 7, node = 8 * h + nd;
    const bool active = (s.flags[node] & F_ACTIVE) != 0;
    const bool cold = (s.flags[node] & F_COLD) != 0;
    double sT1 = 0.0, sT2 = 0.0, sT3 = 0.0, sT4 = 0.0;
    const int ew = et >> 5;   // epilogue warp: columns 4·ew .. 4·ew + 3 of each tile
    int seg_n = 0;            // β⁺ nonzeros of (sub-range, warp ew, node) so far (check sweeps)
    int sr = sr0;             // sub-range of the current tile
    // close sub-range sr: its nonzero count and its check sums (stash slot sr − sr0)
    auto eflush = [&]() {
      if (fused && check) {
        if ((et & 31) < 8) k.seg_cnt[((int64_t)sr * NEW + ew) * kBC + node] = seg_n;
        double* st = s.Ws + 2 * 8 * 12 + ((sr - sr0) * 64 + et) * 4;
        st[0] = sT1; st[1] = sT2; st[2] = sT3; st[3] = sT4;
      }
      sT1 = sT2 = sT3 = sT4 = 0.0;
      seg_n = 0;
      sr++;
    };
    int m = 0;
    for (;; m++) {
      PROF_T0();
      const int tile = stage(m);   // stage m landed (its state operands too), or the end marker
      PROF_ACC(0);
      if (tile < 0) break;
      if (paired && sr == sr0 && tile >= tb) eflush();
      const int sg = m % NST;
      const int64_t col0 = (int64_t)tile * kPt;
      const int el = j * kBC + node;
      const int64_t e = col0 * kBC + el;
      const double* q = s.stq + sg * STQ;
      const double q_beta = q[el], q_v = q[STB + el], q_c = q[2 * STB + j];
      const uint8_t q_code = reinterpret_cast<const uint8_t*>(q + 2 * STB + 8)[el];
      // everything that does not depend on S_J is formed before the hand-off
      const double w = q_c + k.rho * q_beta - q_v;      // eq:b_update input c + ρβ − v
      const double vr = q_v * k.inv_rho;
      double wn = 0.0;
      if (!fused && active) wn = (MODE == SW_FWD_BETA) ? q_beta : w;
      PROF_ACC(1);
      // fused: S_J(m) partials written; forward-only: w⁺ buffer m&1 released by fwd(m − 2)
      if (fused || m >= 2) {
        mbar_wait(&s.sready[m & 1], (hph >> (m & 1)) & 1u);
        hph ^= 1u << (m & 1);
      }
      PROF_ACC(2);
#ifndef EXP_NOEPI
      if (fused) {
        // S_J = Σ over the NMW k-split partials, pairwise in a fixed tree (short dependency chain)
        const double* sp = s.spart + (m & 1) * NMW * 64 + j * 8 + nd;
        double part[NMW];
#pragma unroll
        for (int i = 0; i < NMW; i++) part[i] = sp[i * 64];
#pragma unroll
        for (int hh = 1; hh < NMW; hh *= 2)
#pragma unroll
          for (int i = 0; i + hh < NMW; i += 2 * hh) part[i] += part[i + hh];
        const double sv = part[0];
        double bnz = 0.0;
        if (active) {
          // b = D w: Z-form D = (I − ZᵀZ)/ρ (R1) with sv = (ZᵀZ w)_j, or direct with sv = (D w)_j
          const double b = DIR ? sv : (w - sv) * k.inv_rho;
          const double bn = refresh ? q_beta : prox(k, b + vr, q_code);
          // the refresh sweep updates b, v of warm nodes only; a cold node starts at (0, 0) (R6)
          const double vn = (refresh && cold) ? q_v : q_v + k.rho * (b - bn);
          if (check) {
            const double xxb = DIR ? w - k.rho * b : sv;   // (XᵀX b)_j, since (XᵀX + ρI) b = w
            sT1 = fma(b, xxb, sT1);
            sT2 += nu_f(k, fabs(q_c - xxb), q_code);
            sT3 = fma(q_c, bn, sT3);
            sT4 += psi_f(k, bn, q_code);
            k.bchk[e] = b;
          }
          k.stt[st_beta(col0 + j, node)] = bn;
          k.stt[st_beta(col0 + j, node) + STB] = vn;
          wn = q_c + k.rho * bn - vn;
          bnz = bn;
        }
        if (check) {
          // append this tile's nonzeros of β⁺ to the (sub-range, epilogue warp, node) segment, in
          // column order: ballot + popcount, no barrier (every lane of a node keeps the same count)
          const unsigned bal = __ballot_sync(0xffffffffu, bnz != 0.0);
          const unsigned mnode = bal & (0x01010101u << nd);
          if (bnz != 0.0) {
            const int r = seg_n + __popc(mnode & ((1u << (tid & 31)) - 1u));
            const int64_t o = (((int64_t)sr * NEW + ew) * kBC + node) * k.seg_cap + r;
            k.seg_idx[o] = (int32_t)(col0 + j);
            k.seg_val[o] = bnz;
          }
          seg_n += __popc(mnode);
        }
      }
#endif
      s.Ws[(m & 1) * 8 * 12 + nd * 12 + j] = wn;
      if (DIR) uout[(int64_t)node * k.ld + col0 + j] = wn;   // the next sweep's w (R17)
      mbar_arrive_warp(&s.wready[m & 1]);
      PROF_ACC(5);
    }
    // forward-only sweeps: consume the buffer-free arrivals of the last two forwards
    if (!fused)
      for (int i = m >= 2 ? m - 2 : 0; i < m; i++) {
        mbar_wait(&s.sready[i & 1], (hph >> (i & 1)) & 1u);
        hph ^= 1u << (i & 1);
      }
    // β, v were written through the generic proxy; the next sweep reads them with TMA
    fence_proxy_async_global();
    if (sr == sr0) eflush();
    if (paired && sr == sr0 + 1) eflush();
  }
  __syncthreads();
  // a check decision follows a check sweep and the dense-primal sweep: defer the next start
  if (tid == 0) prefill(k, s, s.sched[0] + 1, check || MODE == SW_FWD_BETA);
  // per-sub-range check sums of the CTA's 8 nodes (fixed order over the tile's 8 columns)
  if (fused && check && tid < (paired ? 2 : 1) * 8 * 4) {
    const int si = tid >> 5, nd = (tid >> 2) & 7, q = tid & 3;
    double a = 0.0;
    for (int j = 0; j < 8; j++) a += s.Ws[2 * 8 * 12 + (si * 64 + j * 8 + nd) * 4 + q];
    sums_out[((int64_t)(sr0 + si) * kBC + 8 * h + nd) * kSums + q] = a;
  }
}

// Fixed-order grid reduction of the forward partials into dst[node][row] (rows < n8).  CTA g owns
// elements [e0, e1) (≤ RED_E of them per pass); thread (c, e) sums partials q ∈ chunk c in order,
// then chunk sums are added in chunk order — deterministic and independent of the batch.
constexpr int RED_E = 64;
constexpr int RED_C = kAdmmThreads / RED_E;
__device__ void reduce_u(const KP& k, Smem& s, double* dst) {
  const int tid = threadIdx.x;
  const int g = blockIdx.x, G = gridDim.x, Q = k.nsr;
  const int64_t E = (int64_t)kBC * k.n8;
  const int64_t e0 = E * g / G, e1 = E * (g + 1) / G;
  const int el = tid % RED_E, c = tid / RED_E;
  const int q0 = Q * c / RED_C, q1 = Q * (c + 1) / RED_C;
  for (int64_t eb = e0; eb < e1; eb += RED_E) {
    const int64_t e = eb + el;
    double a = 0.0;
    // inactive nodes: their partials were not written this sweep, and their u is never used
    const bool live = e < e1 && (s.flags[e / k.n8] & F_ACTIVE);
    if (live) {
      const int64_t nd = e / k.n8, row = e % k.n8;
      const double* src = k.Upart + nd * k.ld + row;
      const int64_t qs = (int64_t)kBC * k.ld;
      // all partials of the chunk in flight at once (the sum stays in q order)
      constexpr int MAXQ = 20;
      if (q1 - q0 <= MAXQ) {
        double v[MAXQ];
#pragma unroll
        for (int i = 0; i < MAXQ; i++) v[i] = (q0 + i < q1) ? __ldcg(src + (int64_t)(q0 + i) * qs) : 0.0;
#pragma unroll
        for (int i = 0; i < MAXQ; i++) a += v[i];
      } else {
#pragma unroll 8
        for (int q = q0; q < q1; q++) a += __ldcg(src + q * qs);
      }
    }
    s.spart[c * RED_E + el] = a;
    __syncthreads();
    if (c == 0 && live) {
      double r = s.spart[el];
#pragma unroll
      for (int cc = 1; cc < RED_C; cc++) r += s.spart[cc * RED_E + el];
      const int64_t nd = e / k.n8, row = e % k.n8;
      dst[nd * k.ld + row] = r;
    }
    __syncthreads();
  }
}

// Dense per-node list of β⁺'s nonzeros: CTA g copies its segment to offset Σ_{g'<g} cnt[g'].
// Returns (in tot[nd], every CTA identically) the node's total count.
// (Active nodes only: the segments of the others were not written this sweep; their total is 0.)
// CTA g copies the segments of sub-range g.
__device__ void compact_nonzeros(const KP& k, Smem& s, int* tot) {
  const int g = blockIdx.x, G = k.nsr;
  __shared__ int off_s[kBC], all_s[kBC], own_s[NEW][kBC];
  if (threadIdx.x < kBC) { off_s[threadIdx.x] = 0; all_s[threadIdx.x] = 0; }
  __syncthreads();
  // counts of all (sub-range, epilogue warp) segments, loaded by every thread in parallel; integer
  // sums are exact in any order (shared-memory atomics)
  for (int e = threadIdx.x; e < G * NEW * kBC; e += blockDim.x) {
    const int q = e / kBC, nd = e % kBC;
    if (!(s.flags[nd] & F_ACTIVE)) continue;
    const int c = __ldcg(k.seg_cnt + e);
    if (c) {
      atomicAdd(&all_s[nd], c);
      if (q < g * NEW) atomicAdd(&off_s[nd], c);
    }
    if (q >= g * NEW && q < (g + 1) * NEW) own_s[q - g * NEW][nd] = c;
  }
  __syncthreads();
  if (threadIdx.x < kBC) tot[threadIdx.x] = (s.flags[threadIdx.x] & F_ACTIVE) ? all_s[threadIdx.x] : 0;
  // this CTA's segments → the dense per-node lists at their offsets (segment order = column order)
  for (int w = 0; w < NEW; w++)
    for (int nd = 0; nd < kBC; nd++) {
      if (!(s.flags[nd] & F_ACTIVE)) continue;
      const int q = g * NEW + w;
      const int c = own_s[w][nd];
      int off = off_s[nd];
      for (int ww = 0; ww < w; ww++) off += own_s[ww][nd];
      const int64_t so = ((int64_t)q * kBC + nd) * k.seg_cap;
      for (int r = threadIdx.x; r < c; r += blockDim.x)
        if (off + r < k.nz_cap) {
          k.nz_idx[(int64_t)nd * k.nz_cap + off + r] = __ldcg(k.seg_idx + so + r);
          k.nz_val[(int64_t)nd * k.nz_cap + off + r] = __ldcg(k.seg_val + so + r);
        }
    }
}

// ‖Xβ‖² partials from the sparse β⁺ (nodes with ≤ nz_cap nonzeros): CTA g owns rows [i0, i1).
// In pass h, warp pair (2·nl, 2·nl+1) serves node nd = 8h + nl: lane l of the pair takes entries
// e ≡ l (mod 64) and accumulates X[i, j_e]·β_e for 8 rows i at once (one contiguous 64-byte piece
// of column j_e); the 64 slot sums are reduced by a fixed butterfly and a fixed pair order —
// deterministic and independent of the batch.
__device__ void gather_partial(const KP& k, Smem& s, const int* tot) {
  const int g = blockIdx.x, G = gridDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i0 = k.xn * g / G, i1 = k.xn * (g + 1) / G;
  const int nl = warp >> 1, slot = (warp & 1) * 32 + lane;
  double* red = s.spart;   // [8][2][8]
  double part = 0.0;       // thread tid < kBC: node tid
  for (int h = 0; h < NH; h++) {
    const int nd = 8 * h + nl;
    const bool use = nl < 8 && (s.flags[nd] & F_ACTIVE) && tot[nd] <= k.nz_cap;
    for (int64_t r0 = i0; r0 < i1; r0 += 8) {
      double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (use) {
        const int cnt = tot[nd];
        const int32_t* ix = k.nz_idx + (int64_t)nd * k.nz_cap;
        const double* vx = k.nz_val + (int64_t)nd * k.nz_cap;
        const int nr = (int)(i1 - r0 < 8 ? i1 - r0 : 8);
#pragma unroll 8
        for (int e = slot; e < cnt; e += 64) {
          const double bv = __ldcg(vx + e);
          const double* col = k.X + (int64_t)__ldcg(ix + e) * k.xld + r0;
#pragma unroll
          for (int r = 0; r < 8; r++)
            if (r < nr) a[r] = fma(bv, __ldg(col + r), a[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < 8; r++)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a[r] += __shfl_xor_sync(0xffffffffu, a[r], o);
      if (nl < 8 && lane < 8) {
        double v = 0.0;
#pragma unroll
        for (int r = 0; r < 8; r++) v = lane == r ? a[r] : v;
        red[(nl * 2 + (warp & 1)) * 8 + lane] = v;
      }
      __syncthreads();
      if ((tid >> 3) == h && tid < kBC) {
        const int l = tid & 7;
        for (int r = 0; r < 8 && r0 + r < i1; r++) {
          const double xb = red[(l * 2) * 8 + r] + red[(l * 2 + 1) * 8 + r];
          part = fma(xb, xb, part);
        }
      }
      __syncthreads();
    }
  }
  if (tid < kBC && (s.flags[tid] & F_ACTIVE) && tot[tid] <= k.nz_cap) k.sums2[(int64_t)g * kBC + tid] = part;
}

// ‖L (Zβ)‖² partials: rows of L split over CTAs; per node one partial per CTA (nodes whose β⁺
// has more than nz_cap nonzeros; the others use gather_partial).
// Column-partitioned primal gather (Z-form): CTA g accumulates X_j β_j over WHOLE columns (8n-byte
// coalesced reads) for the β⁺ nonzeros of sub-range g — the epilogue's own segments (sub-range g,
// epilogue warp 0 then 1, column order within each), no compaction into per-node lists — of every
// active node into the forward-partial slot Upart[g][node][·]; reduce_u then sums the slots in
// sub-range order (the forward partials' fixed order, so a node's sum depends on its own nonzeros only)
// and xnorm_partial takes ‖Xβ‖² over the CTA's rows.  No per-node cap: no dense Zβ fallback.
__device__ void gather_segs(const KP& k, Smem& s) {
  // work items (node, 256-row chunk) dealt to the 16 warps in turn (at B = 1 one node's chunks still
  // spread over several warps); a lane holds 8 rows 32 apart, so each segment entry issues 8 coalesced
  // loads per lane; per row the entries are summed in segment order (epilogue warp 0's columns, then
  // warp 1's), as a sequential walk would
  const int g = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nchunk = (int)((k.n8 + 255) / 256);
  for (int it = warp; it < kBC * nchunk; it += kAdmmThreads / 32) {
    const int nd = it / nchunk;
    const int64_t r0 = (int64_t)(it % nchunk) * 256;
    if (!(s.flags[nd] & F_ACTIVE)) continue;
    const int64_t q0 = ((int64_t)g * NEW + 0) * kBC + nd, q1 = ((int64_t)g * NEW + 1) * kBC + nd;
    const int32_t* ixp[2] = {k.seg_idx + q0 * k.seg_cap, k.seg_idx + q1 * k.seg_cap};
    const double* vxp[2] = {k.seg_val + q0 * k.seg_cap, k.seg_val + q1 * k.seg_cap};
    const int cn[2] = {__ldcg(k.seg_cnt + q0), __ldcg(k.seg_cnt + q1)};
    double* up = k.Upart + ((int64_t)g * kBC + nd) * k.ld;
    double a[8];
#pragma unroll
    for (int r = 0; r < 8; r++) a[r] = 0.0;
    for (int sgm = 0; sgm < 2; sgm++)
      for (int e = 0; e < cn[sgm]; e++) {
        const double v = __ldcg(vxp[sgm] + e);
        const double* col = k.X + (int64_t)__ldcg(ixp[sgm] + e) * k.xld + r0 + lane;
#pragma unroll
        for (int r = 0; r < 8; r++)   // rows n..n8 of X are zero padding
          if (r0 + lane + 32 * r < k.n8) a[r] = fma(v, __ldg(col + 32 * r), a[r]);
      }
#pragma unroll
    for (int r = 0; r < 8; r++)
      if (r0 + lane + 32 * r < k.n8) up[r0 + lane + 32 * r] = a[r];
  }
}
// The gather's partials → Ub for THIS CTA's rows [n8·g/G, n8·(g+1)/G) of every active node (the same
// per-element order as reduce_u: fixed chunks of the Q partials), then ‖Xβ‖² over those rows per node
// in row order.  Row ranges, unlike reduce_u's node-major element ranges, do not depend on a node's
// slot, so a node's result is the same alone or in a batch; no grid barrier between the two steps.
__device__ void reduce_rows_norm(const KP& k, Smem& s) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.x, G = gridDim.x, Q = k.nsr;
  const int64_t r0 = k.n8 * g / G, r1 = k.n8 * (g + 1) / G, nr = r1 - r0;
  const int64_t E = (int64_t)kBC * nr;
  const int el = tid % RED_E, c = tid / RED_E;
  const int q0 = Q * c / RED_C, q1 = Q * (c + 1) / RED_C;
  for (int64_t eb = 0; eb < E; eb += RED_E) {
    const int64_t e = eb + el;
    const int64_t nd = nr > 0 ? e / nr : 0, row = r0 + (nr > 0 ? e % nr : 0);
    double a = 0.0;
    const bool live = e < E && (s.flags[nd] & F_ACTIVE);
    if (live) {
      const double* src = k.Upart + nd * k.ld + row;
      const int64_t qs = (int64_t)kBC * k.ld;
      for (int q = q0; q < q1; q++) a += __ldcg(src + q * qs);
    }
    s.spart[c * RED_E + el] = a;
    __syncthreads();
    if (c == 0 && live) {
      double r = s.spart[el];
#pragma unroll
      for (int cc = 1; cc < RED_C; cc++) r += s.spart[cc * RED_E + el];
      k.Ub[nd * k.ld + row] = r;
    }
    __syncthreads();
  }
  // warp w ↔ node w: squares over this CTA's rows in row order (lane stride, fixed butterfly)
  if (warp < kBC && (s.flags[warp] & F_ACTIVE)) {
    double part = 0.0;
    for (int64_t i = r0 + lane; i < r1; i += 32)
      if (i < k.xn) {
        const double x = __ldcg(k.Ub + (int64_t)warp * k.ld + i);
        part = fma(x, x, part);
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) k.sums2[(int64_t)g * kBC + warp] = part;
  }
}
__device__ void lmatvec_partial(const KP& k, Smem& s) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = blockIdx.x, G = gridDim.x;
  const int64_t i0 = k.xn * g / G, i1 = k.xn * (g + 1) / G;
  double part[kBC];
#pragma unroll
  for (int nd = 0; nd < kBC; nd++) part[nd] = 0.0;
  for (int64_t i = i0 + warp; i < i1; i += NW) {
    double a[kBC];
#pragma unroll
    for (int nd = 0; nd < kBC; nd++) a[nd] = 0.0;
    const double* lrow = k.Lt + i * k.xld;   // row i of L = column i of Lᵀ, entries m ≤ i
    for (int64_t m = lane; m <= i; m += 32) {
      const double l = lrow[m];
#pragma unroll
      for (int nd = 0; nd < kBC; nd++) a[nd] = fma(l, __ldcg(k.Ub + nd * k.xld + m), a[nd]);
    }
#pragma unroll
    for (int nd = 0; nd < kBC; nd++) {
      double x = a[nd];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      part[nd] = fma(x, x, part[nd]);
    }
  }
  if (lane == 0)
    for (int nd = 0; nd < kBC; nd++) s.spart[warp * kBC + nd] = part[nd];
  __syncthreads();
  if (threadIdx.x < kBC && s.ncnt[threadIdx.x] > k.nz_cap) {   // ncnt holds the node totals here
    double a = 0.0;
    for (int w = 0; w < NW; w++) a += s.spart[w * kBC + threadIdx.x];
    k.sums2[(int64_t)g * kBC + threadIdx.x] = a;
  }
}

// Node-slot compaction (paired → single-half mode with all active nodes in half 0): exchange
// slots a_i ↔ b_i.  Every CTA swaps its per-node shared state; block 0 the per-node scalars in
// HBM; CTA g the state blocks and b_chk rows of the tiles of sub-range g and rows
// [n·g/G, n·(g+1)/G) of u.  A node's arithmetic does not depend on its slot, so results are
// bitwise those without compaction.  Applied again (an involution) before the outputs.
__device__ void swap_slots(const KP& k, Smem& s, const int* pa, const int* pb, int np) {
  const int tid = threadIdx.x, g = blockIdx.x, G = gridDim.x;
  __syncthreads();
  if (tid == 0)
    for (int q = 0; q < np; q++) {
      const int a = pa[q], b = pb[q];
      int f = s.flags[a]; s.flags[a] = s.flags[b]; s.flags[b] = f;
      f = s.it0[a]; s.it0[a] = s.it0[b]; s.it0[b] = f;
      double r = s.red[a]; s.red[a] = s.red[b]; s.red[b] = r;
      if (g == 0) {
        for (int i = 0; i < 4; i++) { double t = k.nodef[a * 4 + i]; k.nodef[a * 4 + i] = k.nodef[b * 4 + i]; k.nodef[b * 4 + i] = t; }
        for (int i = 0; i < 2; i++) { int t = k.nodei[a * 2 + i]; k.nodei[a * 2 + i] = k.nodei[b * 2 + i]; k.nodei[b * 2 + i] = t; }
      }
    }
  const int t0 = sub_t(k, g), t1 = sub_t(k, g + 1);
  const int64_t cols = (int64_t)(t1 - t0) * kPt;
  for (int64_t e = tid; e < cols * np; e += blockDim.x) {
    const int q = (int)(e % np);
    const int64_t j = (int64_t)t0 * kPt + e / np;
    const int a = pa[q], b = pb[q];
    double* B = k.stt + st_beta(j, 0);
    double t = B[a]; B[a] = B[b]; B[b] = t;
    t = B[STB + a]; B[STB + a] = B[STB + b]; B[STB + b] = t;
    uint8_t* C = &st_code(k.stt, j, 0);
    uint8_t c = C[a]; C[a] = C[b]; C[b] = c;
    double* H = k.bchk + j * kBC;
    t = H[a]; H[a] = H[b]; H[b] = t;
  }
  const int64_t r0 = k.n8 * g / G, r1 = k.n8 * (g + 1) / G;
  double* Ucur = (k.direct && (s.sched[0] & 1)) ? k.Ub : k.U;   // the buffer the next sweep reads
  for (int64_t e = tid; e < (r1 - r0) * np; e += blockDim.x) {
    const int q = (int)(e % np);
    const int64_t row = r0 + e / np;
    double* ua = Ucur + (int64_t)pa[q] * k.ld + row;
    double* ub = Ucur + (int64_t)pb[q] * k.ld + row;
    const double t = *ua; *ua = *ub; *ub = t;
  }
  fence_proxy_async_global();   // the next sweep reads the state blocks with TMA
  grid_sync(k.bar);
}

// DIR: the direct regime (R17) as a separate instantiation, so the Z-form code is unchanged by it
template <int KS, int MT, bool DIR>
__global__ void __launch_bounds__(kAdmmThreads, 1) admm_persistent(KP k_in) {
  KP k = k_in;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem s;
  {
    double* base = reinterpret_cast<double*>(smem_raw);
    s.tiles = base;
    s.stq = base + (size_t)NST * kPt * k.ld;
    s.spart = s.stq + NST * STQ;
    s.Ws = s.spart + 2 * NMW * 64;
    s.red = s.Ws + 2 * 8 * 12 + 2 * 64 * 4;
    s.mbar = reinterpret_cast<uint64_t*>(s.red + kBC);
    s.sready = s.mbar + NST;
    s.wready = s.sready + 2;
    s.flags = reinterpret_cast<int*>(s.wready + 2);
    s.rel = reinterpret_cast<unsigned*>(s.flags + kBC);
    s.ncnt = reinterpret_cast<int*>(s.rel + NST);
    s.stile = s.ncnt + kBC;
    s.zres = s.stile + NST;
    s.it0 = s.zres + NST;
    s.sched = s.it0 + kBC;
  }
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int q = 0; q < NST; q++) mbar_init(&s.mbar[q], 1);
    for (int q = 0; q < 2; q++) {
      mbar_init(&s.sready[q], NMW);
      mbar_init(&s.wready[q], NEW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < NST) { s.rel[tid] = 0; s.zres[tid] = -1; }
  for (size_t i = tid; i < (size_t)NST * kPt * k.ld + NST * STQ; i += blockDim.x) s.tiles[i] = 0.0;   // stq follows
  if (tid < kBC) {
    s.flags[tid] = __ldcg(k.nodei + tid * 2);
    s.it0[tid] = __ldcg(k.nodei + tid * 2 + 1);   // 0, or the iterations of a resumed node
    s.red[tid] = __ldcg(k.nodef + tid * 4);       // −∞, or the best dual of a resumed node (R7)
  }
  __syncthreads();
#ifdef L0L2_PROF
  if (tid < NW * 8) prof_s[tid / 8][tid % 8] = 0;
#endif
  if (k.prune_ub_dev) k.prune_ub = __ldcg(k.prune_ub_dev);   // (KP is the kernel's by-value copy)
  unsigned phases = 0, hph = 0;
  __shared__ int swp_a[8], swp_b[8];   // slot pairs exchanged by the compaction (same in every thread)
  int nswp = 0;
  if (tid == 0) prefill(k, s, 0, false);
  __syncthreads();   // the sweep reads its node half and sub-ranges from s.sched

  if (k.step_mode) {   // one phase per launch (column-sharded fused path, see KP)
    if (k.step_phase == 0) {
      sweep<SW_FWD_W, KS, MT, DIR>(k, s, false, false, phases, hph);
    } else if (k.step_phase == 1) {
      sweep<SW_FUSED, KS, MT, DIR>(k, s, true, false, phases, hph);
    } else {
      sweep<SW_FUSED, KS, MT, DIR>(k, s, false, k.step_chk != 0, phases, hph, k.sums);
    }
    grid_sync(k.bar);
    reduce_u(k, s, k.U);
    if (k.step_phase == 2 && k.step_chk) {
      // this rank's totals of the check terms (sub-ranges in order) and Z_r β⁺ for ‖Xβ‖² = ‖L Σ_r Z_r β_r‖²
      if (blockIdx.x == 0 && tid < kBC * 4) {
        const int nd = tid >> 2, term = tid & 3;
        double a = 0.0;
        if (s.flags[nd] & F_ACTIVE)
          for (int q = 0; q < k.nsr; q++) a += __ldcg(k.sums + ((int64_t)q * kBC + nd) * kSums + term);
        k.tot_out[nd * 4 + term] = a;
      }
      grid_sync(k.bar);   // reduce_u has read Upart before the β sweep rewrites it
      sweep<SW_FWD_BETA, KS, MT, DIR>(k, s, false, false, phases, hph);
      grid_sync(k.bar);
      reduce_u(k, s, k.Ub);
    }
    if (tid == 0)
      for (int sg = 0; sg < NST && sg < s.sched[1]; sg++) mbar_wait(&s.mbar[sg], (phases >> sg) & 1u);
    return;
  }

  // u0 = Z (c + ρβ0 − v0), then the warm-start refresh sweep (R6: b, v of warm nodes; cold
  // nodes keep β = v = 0 and only their w⁺ = c is formed)
  sweep<SW_FWD_W, KS, MT, DIR>(k, s, false, false, phases, hph);
  grid_sync(k.bar);
  if (!DIR) reduce_u(k, s, k.U);
  grid_sync(k.bar);
  sweep<SW_FUSED, KS, MT, DIR>(k, s, true, false, phases, hph);
  grid_sync(k.bar);
  if (!DIR) reduce_u(k, s, k.U);
  grid_sync(k.bar);

  int nchk = 0;   // checks so far: the per-sub-range check sums are double-buffered by its parity, so a
                 // CTA that runs ahead into the next check sweep (no grid barrier follows a decision)
                 // never overwrites the sums a slower CTA is still reading in its decision step
  for (int it = 1; it <= k.max_iters; it++) {
    bool chk = (it % k.check_every == 0) || (it == k.max_iters);
    for (int nd = 0; nd < kBC; nd++)   // a resumed node reaching its own iteration cap
      chk |= (s.flags[nd] & F_ACTIVE) && s.it0[nd] + it == k.max_iters;
    double* sums_cur = k.sums + (size_t)(nchk & 1) * k.nsr * kBC * kSums;
    if (chk) nchk++;
    PROF_T0();
    sweep<SW_FUSED, KS, MT, DIR>(k, s, false, chk, phases, hph, sums_cur);
    PROF_ACC(6);
    grid_sync(k.bar);
    if (!DIR) reduce_u(k, s, k.U);
    __shared__ int tot_s[kBC];
    const bool segs = !DIR && k.gather_mode == 0;   // primal from the segments (gather_segs)
    if (chk && !segs) compact_nonzeros(k, s, tot_s);   // β⁺'s nonzeros → dense per-node lists
    // (direct regime, no check: w⁺ is complete after the first barrier and the next sweep writes the
    // other buffer, so one barrier per iteration suffices)
    if (!DIR || chk) grid_sync(k.bar);
    PROF_ACC(7);
    if (!chk) continue;
    PROF_RESET();
    // primal ‖Xβ‖²: a gather over β⁺'s nonzeros (sparse at the paper's workloads); a node with
    // more than nz_cap nonzeros falls back to one forward-only sweep Zβ and ‖L(Zβ)‖²
    if (segs) {   // whole-column gather from the segments (Z-form: Upart holds ≥ n rows)
      gather_segs(k, s);
      grid_sync(k.bar);
      reduce_rows_norm(k, s);   // (the final grid barrier below orders sums2 for the decision)
    } else {
      gather_partial(k, s, tot_s);
      bool dense = false;
      if (tid < kBC) s.ncnt[tid] = tot_s[tid];
      __syncthreads();
      for (int nd = 0; nd < kBC; nd++) dense |= (s.flags[nd] & F_ACTIVE) && tot_s[nd] > k.nz_cap;
      if (dense) {
        sweep<SW_FWD_BETA, KS, MT, DIR>(k, s, false, false, phases, hph);
        grid_sync(k.bar);
        reduce_u(k, s, k.Ub);
        grid_sync(k.bar);
        lmatvec_partial(k, s);
      }
    }
    grid_sync(k.bar);
    PROF_ACC(5);
    // every CTA derives the same per-node decision from the same partials in a fixed order: the
    // sub-range partials of each (node, term) are summed in RCH fixed chunks in parallel, then the
    // chunk sums in chunk order (a sequential 148-term loop per node was ~45 µs of L2 latency)
    {
      constexpr int RCH = 4;
      double* cs = s.spart;   // [kBC][5][RCH]
      const int Q = (int)gridDim.x;
      if (tid < kBC * 5 * RCH) {
        const int nd = tid / (5 * RCH), term = (tid / RCH) % 5, ch = tid % RCH;
        double a = 0.0;
        if (s.flags[nd] & F_ACTIVE) {
          const int q0 = Q * ch / RCH, q1 = Q * (ch + 1) / RCH;
#pragma unroll 8
          for (int q = q0; q < q1; q++)
            a += term < 4 ? __ldcg(sums_cur + ((int64_t)q * kBC + nd) * kSums + term)
                          : __ldcg(k.sums2 + (int64_t)q * kBC + nd);
        }
        cs[tid] = a;
      }
      __syncthreads();
    }
    if (tid < kBC) {
      const int nd = tid;
      int fl = s.flags[nd];
      if (fl & F_ACTIVE) {
        double T[5];
        for (int term = 0; term < 5; term++) {
          const double* c4 = s.spart + (nd * 5 + term) * 4;
          T[term] = (c4[0] + c4[1]) + (c4[2] + c4[3]);
        }
        const double T1 = T[0], T2 = T[1], T3 = T[2], T4 = T[3], T5 = T[4];
        const double dual = 0.5 * k.yy - 0.5 * T1 - T2;
        const double primal = 0.5 * k.yy - T3 + 0.5 * T5 + T4;
        const double lbb = fmax(s.red[nd], dual);   // running max of checked duals (R7)
        s.red[nd] = lbb;
        bool conv = (primal - lbb) / fmax(1.0, fabs(primal)) <= k.node_tol;
        if (conv) fl = (fl & ~F_ACTIVE) | L0L2_FLAG_CONVERGED;
        else if (lbb >= k.prune_ub) fl = (fl & ~F_ACTIVE) | L0L2_FLAG_PRUNED;   // early prune (R16)
        else if (s.it0[nd] + it >= k.max_iters) fl = (fl & ~F_ACTIVE) | L0L2_FLAG_MAXITER;
        s.flags[nd] = fl;
        if (blockIdx.x == 0) {
          k.nodef[nd * 4 + 0] = lbb;
          k.nodef[nd * 4 + 1] = primal;
          k.nodef[nd * 4 + 3] = dual;
          k.nodei[nd * 2 + 0] = fl;
          k.nodei[nd * 2 + 1] = s.it0[nd] + it;
        }
      }
    }
    __syncthreads();
    unsigned am = 0;
    for (int nd = 0; nd < kBC; nd++) am |= (s.flags[nd] & F_ACTIVE) ? 1u << nd : 0u;
    if (!am) break;
    // continuous batching (§8(f) rank 2): few nodes left in this launch — suspend them here (their
    // β, v, best dual and iteration count go back to the caller, which resumes them bitwise where
    // they stopped, next to fresh nodes); only at regular checks, so resumed nodes stay on the
    // check_every grid
    if (k.suspend_at > 0 && it % k.check_every == 0 && it >= k.susp_min && __popc(am) <= k.suspend_at) {
      if (tid < kBC && (s.flags[tid] & F_ACTIVE)) {
        const int fl = (s.flags[tid] & ~F_ACTIVE) | F_SUSP;
        s.flags[tid] = fl;
        if (blockIdx.x == 0) k.nodei[tid * 2 + 0] = fl;
      }
      __syncthreads();
      break;
    }
    // ≤ 8 active nodes spread over both halves: move them into half 0 (the next sweep then runs
    // in single-half mode on every SM instead of paired); at most once per launch
    if (k.compact && nswp == 0 && __popc(am) <= 8 && (am & 0xFFu) && (am & 0xFF00u)) {
      int np = 0, ib = 0;
      for (int a = 8; a < 16; a++) {
        if (!((am >> a) & 1u)) continue;
        while ((am >> ib) & 1u) ib++;   // next inactive slot of half 0 (exists: |active| ≤ 8)
        swp_a[np] = a;
        swp_b[np] = ib++;
        np++;
      }
      __syncthreads();
      swap_slots(k, s, swp_a, swp_b, np);
      nswp = np;
    }
  }
  if (nswp) swap_slots(k, s, swp_a, swp_b, nswp);   // back to the caller's slots
#ifdef L0L2_PROF
  __syncthreads();
  if (tid < NW * 8) g_prof[blockIdx.x][tid / 8][tid % 8] += prof_s[tid / 8][tid % 8];
#endif
  // drain the prefill issued after the last sweep before the CTA retires
  if (tid == 0)
    for (int sg = 0; sg < NST && sg < s.sched[1]; sg++) mbar_wait(&s.mbar[sg], (phases >> sg) & 1u);
  if (blockIdx.x == 0 && tid < k.nb && ((k.act_mask >> tid) & 1u)) {
    const int nd = tid;
    const double lbb = s.red[nd], plb = __ldcg(k.nodef + nd * 4 + 2);
    k.out_lb[nd] = fmax(lbb, plb);
    k.out_primal[nd] = k.nodef[nd * 4 + 1];
    k.out_iters[nd] = k.nodei[nd * 2 + 1];
    k.out_flags[nd] = (uint8_t)((s.flags[nd] & (L0L2_FLAG_CONVERGED | L0L2_FLAG_MAXITER | L0L2_FLAG_PRUNED)) |
                                ((s.flags[nd] & F_SUSP) ? kFlagSuspended : 0));
    if (k.out_lbbest) k.out_lbbest[nd] = lbb;
  }
}

// ---------------------------------------------------------------- packing / finalize kernels

// code plane and state for one group: column j, node nd (nd ≥ nb and j ≥ p are inactive F0)
__global__ void pack_kernel(int64_t p, int64_t p8, int nb, double* stt, const double* __restrict__ c,
                            const double* const* warm) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= p8 * kBC) return;
  const int64_t j = e / kBC;
  const int nd = (int)(e % kBC);
  uint8_t cd = (nd < nb && j < p) ? 0 : 1;
  st_code(stt, j, nd) = cd;
  double b = 0.0, vv = 0.0;
  if (nd < nb && j < p && warm != nullptr && warm[nd] != nullptr) {
    b = warm[nd][j];
    vv = warm[nd][p + j];
  }
  stt[st_beta(j, nd)] = b;
  stt[st_beta(j, nd) + STB] = vv;
  if (nd == 0) stt[st_c(j)] = j < p ? c[j] : 0.0;
}

__global__ void scatter_fix(int nb, const int64_t* __restrict__ off, const int32_t* __restrict__ idx,
                            const uint8_t* __restrict__ val, double* stt, int64_t p, int* bad) {
  const int nd = blockIdx.x;
  if (nd >= nb) return;
  const int64_t q0 = off[nd], q1 = off[nd + 1];
  for (int64_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
    const int32_t j = idx[q];
    if (j < 0 || j >= p) { atomicOr(bad, 1); continue; }
    const uint8_t cd = val[q] ? 2 : 1;
    for (int64_t r = q0; r < q; r++)               // F0 ∩ F1 ≠ ∅, order independent
      if (idx[r] == j && (val[r] ? 2 : 1) != cd) atomicOr(bad, 2);
    st_code(stt, j, nd) = cd;
    if (cd == 1) stt[st_beta(j, nd)] = 0.0;        // warm edit: β_j ← 0 on F0
  }
}

// device frontier (frontier.cu): the fixings of node nd of a group as a chain of records
// rec → {parent record, 2j + value}; codes F0 → 1, F1 → 2, and the warm edit β_j ← 0 on F0
__global__ void scatter_chain(int nb, const int* __restrict__ node_rec, const int* __restrict__ recs, int rec_stride,
                              double* stt) {
  const int nd = blockIdx.x;
  if (nd >= nb || threadIdx.x != 0) return;
  for (int r = node_rec[nd]; r >= 0; r = recs[(int64_t)r * rec_stride]) {
    const int fx = recs[(int64_t)r * rec_stride + 1];
    const int64_t j = fx >> 1;
    st_code(stt, j, nd) = (fx & 1) ? 2 : 1;
    if (!(fx & 1)) stt[st_beta(j, nd)] = 0.0;
  }
}

__global__ void init_nodes(int nb, unsigned mask, unsigned cold, const double* parent_lb, const double* lbbest_in,
                           const int* it0_in, const double* const* warm_ptrs, double* nodef, int* nodei) {
  const int nd = threadIdx.x;
  if (nd >= kBC) return;
  // device frontier: a node without a parent state (null warm pointer) is cold
  if (warm_ptrs && nd < nb && warm_ptrs[nd] == nullptr) cold |= 1u << nd;
  nodef[nd * 4 + 0] = (nd < nb && lbbest_in) ? lbbest_in[nd] : -INFINITY;
  nodef[nd * 4 + 1] = INFINITY;
  nodef[nd * 4 + 2] = (nd < nb && parent_lb) ? parent_lb[nd] : -INFINITY;
  nodef[nd * 4 + 3] = -INFINITY;
  nodei[nd * 2 + 0] = (nd < nb && ((mask >> nd) & 1u)) ? (F_ACTIVE | (((cold >> nd) & 1u) ? F_COLD : 0)) : 0;
  nodei[nd * 2 + 1] = (nd < nb && it0_in) ? it0_in[nd] : 0;
}

// ẑ, integrality, branch index (R10), support F1 ∪ {ẑ ≥ ½}
struct BrKey { double frac, ab; int64_t j; };
__device__ __forceinline__ bool better(const BrKey& a, const BrKey& b) {
  if (a.frac != b.frac) return a.frac > b.frac;
  if (a.ab != b.ab) return a.ab > b.ab;
  return a.j < b.j;
}

__global__ void __launch_bounds__(512) finalize_kernel(int64_t p, double M, double zsr, bool lam0_pos, double int_tol,
                                                       const double* __restrict__ stt,
                                                       double* zhat, int64_t ldz, int32_t* branch_j, uint8_t* flags,
                                                       int32_t* supp_cnt, int32_t* supp_idx, int64_t supp_stride) {
  const int nd = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ int wcnt[16];
  __shared__ int base_s;
  __shared__ BrKey wkey[16];
  __shared__ int nonint_s;
  if (tid == 0) { base_s = 0; nonint_s = 0; }
  __syncthreads();
  BrKey best{-1.0, -1.0, (int64_t)1 << 62};
  int nonint = 0;
  for (int64_t c0 = 0; c0 < p; c0 += blockDim.x) {
    const int64_t j = c0 + tid;
    bool insupp = false;
    if (j < p) {
      const double b = stt[st_beta(j, nd)];
      const uint8_t cd = st_code(stt, j, nd);
      const double ab = fabs(b);
      double z;
      if (cd == 1) z = 0.0;
      else if (cd == 2) z = 1.0;
      else z = lam0_pos ? fmin(1.0, fmax(ab / M, zsr * ab)) : (ab > 0.0 ? 1.0 : 0.0);
      if (zhat) zhat[(int64_t)nd * ldz + j] = z;
      if (cd == 0) {
        const double fr = fmin(z, 1.0 - z);
        if (fr > int_tol) nonint = 1;
        BrKey kk{fr, ab, j};
        if (better(kk, best)) best = kk;
        insupp = z >= 0.5;
      } else {
        insupp = (cd == 2);
      }
    }
    // ordered compaction of the support
    const unsigned m = __ballot_sync(0xffffffffu, insupp);
    if (lane == 0) wcnt[warp] = __popc(m);
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) { if (w < warp) off += wcnt[w]; tot += wcnt[w]; }
    if (insupp) {
      const int pos = base_s + off + __popc(m & ((1u << lane) - 1u));
      if (pos < supp_stride) supp_idx[(int64_t)nd * supp_stride + pos] = (int32_t)j;
    }
    __syncthreads();
    if (tid == 0) base_s += tot;
    __syncthreads();
  }
  // branch key reduction (warp then block, deterministic comparator)
  for (int o = 16; o > 0; o >>= 1) {
    BrKey other{__shfl_xor_sync(0xffffffffu, best.frac, o), __shfl_xor_sync(0xffffffffu, best.ab, o),
                (int64_t)__shfl_xor_sync(0xffffffffu, (long long)best.j, o)};
    if (better(other, best)) best = other;
  }
  if (lane == 0) wkey[warp] = best;
  if (nonint) atomicOr(&nonint_s, 1);
  __syncthreads();
  if (tid == 0) {
    BrKey b = wkey[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); w++) if (better(wkey[w], b)) b = wkey[w];
    const bool integral = (nonint_s == 0);
    branch_j[nd] = integral ? -1 : (int32_t)b.j;
    flags[nd] = (uint8_t)((flags[nd] & ~L0L2_FLAG_INTEGRAL) | (integral ? L0L2_FLAG_INTEGRAL : 0));
    supp_cnt[nd] = base_s;
  }
}

__global__ void unpack_kernel(int64_t p, int nb, const double* __restrict__ stt, double* const* warm) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= p * kBC) return;
  const int64_t j = e / kBC;
  const int nd = (int)(e % kBC);
  if (nd >= nb || warm[nd] == nullptr) return;
  warm[nd][j] = stt[st_beta(j, nd)];
  warm[nd][p + j] = stt[st_beta(j, nd) + STB];
}

__global__ void fill_y(double* r, int64_t ldr, const double* y, int64_t n, int nb) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * nb) return;
  r[(e / n) * ldr + e % n] = y[e % n];
}

// step mode decision (column-sharded fused path): from the ALL-REDUCED check totals and Zβ, per node
// the dual of Proposition 1 at r̂ = y − X b̂, the primal with ‖Xβ‖² = ‖L Zβ‖²,
// the running max (R7) and the stop rule (R8) — the same arithmetic as the in-kernel decision
__global__ void step_decide(KP k, int it, const double* __restrict__ tot) {
  const int nd = blockIdx.x;
  int fl = k.nodei[nd * 2];
  if (!(fl & F_ACTIVE)) return;
  __shared__ double red[32];
  double q = 0.0;
  for (int64_t i = threadIdx.x; i < k.xn; i += blockDim.x) {   // (L Zβ)_i = Σ_{m ≤ i} L_im (Zβ)_m
    const double* lrow = k.Lt + i * k.xld;
    double a = 0.0;
    for (int64_t m = 0; m <= i; m++) a = fma(lrow[m], k.Ub[nd * k.ld + m], a);
    q = fma(a, a, q);
  }
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = q;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double xx = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); w++) xx += red[w];
  const double* T = tot + nd * 4;
  const double dual = 0.5 * k.yy - 0.5 * T[0] - T[1];
  const double primal = 0.5 * k.yy - T[2] + 0.5 * xx + T[3];
  const double lbb = fmax(k.nodef[nd * 4 + 0], dual);
  const int itn = k.nodei[nd * 2 + 1] + it;   // (it0 = 0 in step mode)
  if ((primal - lbb) / fmax(1.0, fabs(primal)) <= k.node_tol) fl = (fl & ~F_ACTIVE) | L0L2_FLAG_CONVERGED;
  else if (it >= k.max_iters) fl = (fl & ~F_ACTIVE) | L0L2_FLAG_MAXITER;
  k.nodef[nd * 4 + 0] = lbb;
  k.nodef[nd * 4 + 1] = primal;
  k.nodef[nd * 4 + 3] = dual;
  k.nodei[nd * 2 + 0] = fl;
  k.out_iters[nd] = itn;   // iterations run so far (the node's count once it stops)
}
__global__ void step_outputs(KP k) {
  const int nd = threadIdx.x;
  if (nd >= k.nb) return;
  k.out_lb[nd] = fmax(k.nodef[nd * 4 + 0], k.nodef[nd * 4 + 2]);
  k.out_primal[nd] = k.nodef[nd * 4 + 1];
  k.out_flags[nd] = (uint8_t)(k.nodei[nd * 2] & (L0L2_FLAG_CONVERGED | L0L2_FLAG_MAXITER));
}

// ---------------------------------------------------------------- wide-n path
// The fused kernel keeps u (n×8) and its forward accumulators (n×8) in registers and a 3-stage ring
// of n×8 Z tiles in shared memory, which caps n at 1056.  Beyond that (the paper's n = 3000 and
// 11 962 workloads) the SAME iteration runs on the same node state (stt, node_f/node_i,
// bchk) as a host-stepped sequence:
//   wide_sweep_p    S_J = Z_Jᵀu for groups of 32 columns (persistent, one CTA per SM; per-warp cp.async
//                   rings, DMMA, fixed-order cross-warp tree), then the fused kernel's elementwise
//                   epilogue (b, β⁺, v⁺, w⁺, check terms) — one read of Z;
//   wide_forward_p  u⁺ = Z w⁺ (n × 16, K = p; row blocks × column chunks, chunk partials summed in
//                   order by wide_reduce) — the second read of Z;
//   at checks       Xβ⁺ by the same product on X (‖Xβ‖²), then wide_decide: dual, primal
//                   (P:320-325), running max (R7), stop (R8), early prune (R16) — the fused
//                   kernel's decision arithmetic.
// Z is streamed twice per iteration instead of once; every sum has a fixed order.
constexpr int WTH = 256;              // 8 warps per CTA

// w = c + ρβ − v of the active nodes (0 for the others), [p8][kBC]; keeps the nodes' starting
// iteration counts (a resumed node continues its count)
__global__ void __launch_bounds__(WTH) wide_w0(KP k, double* W, int* it0) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (blockIdx.x == 0 && threadIdx.x < kBC) it0[threadIdx.x] = k.nodei[threadIdx.x * 2 + 1];
  if (e >= k.p8 * kBC) return;
  const int64_t j = e / kBC;
  const int nd = (int)(e % kBC);
  double w = 0.0;
  if (k.nodei[nd * 2] & F_ACTIVE) {
    const int64_t o = st_beta(j, nd);
    w = k.stt[st_c(j)] + k.rho * k.stt[o] - k.stt[o + STB];
  }
  W[e] = w;
}

// Each warp streams its share of Z through its own cp.async ring in shared memory (no registers held
// by loads in flight, no CTA barrier inside the K loop), one CTA per SM.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr(dst)), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

constexpr int WPS = 4;                       // ring stages per warp (5 measured slower at B = 16: 0.50 vs 0.41 ms)
constexpr int WGT = 4;                       // tiles per group of the pipelined sweep (32 columns)
constexpr int WGC = WGT * kPt;               // 32 columns
constexpr int WGE = WGC * kBC;               // (column, node) elements per group
constexpr int WSR = 16;                      // rows per stage (4 k-steps)
constexpr int WLDS = WSR + 2;                // smem doubles per column of a stage (padded)
constexpr int WSTG = WGC * WLDS;             // doubles per stage (4.5 KB)
constexpr size_t WSWEEP_SMEM = sizeof(double) * ((size_t)(WTH / 32) * WPS * WSTG + 4 * WGE);   // 160 KB

// Persistent over groups of 32 columns (4 tiles); warp w owns every 8th 16-row stage of the group
// (4 k-steps each), so u is read once per group and Z once per sweep.  A warp issues
// the first stages of its next group before the cross-warp tree and the epilogue of the current one,
// so HBM keeps streaming through them.  Epilogue and check sums: wide_sweep's arithmetic and order.
template <bool REFRESH>
__global__ void __launch_bounds__(WTH, 1) wide_sweep_p(KP k, int check, double* W, double* Bb, double* wsum) {
  extern __shared__ __align__(16) double wsm[];
  __shared__ double csum[WTH / kBC][kBC][4];
  __shared__ int fl[kBC];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cA = lane >> 2, kA = lane & 3;
  if (tid < kBC) fl[tid] = k.nodei[tid * 2];
  __syncthreads();
  const bool a0 = (fl[cA] & F_ACTIVE) != 0, a1 = (fl[8 + cA] & F_ACTIVE) != 0;
  const int ngroups = (k.ntiles + WGT - 1) / WGT;
  const int US = (int)((k.n8 + WSR - 1) / WSR);                     // 16-row stages per column
  // warp w takes the stages w, w + 8, w + 16, ... of every column (at any moment the CTA's warps read
  // adjacent 16-row blocks: 1 KB runs per column rather than 128-B pieces of 8 distant slabs)
  constexpr int NWP = WTH / 32;
  const int nsw = US > warp ? (US - warp + NWP - 1) / NWP : 0;
  double* ring = wsm + (size_t)warp * WPS * WSTG;
  double* red = wsm + (size_t)(WTH / 32) * WPS * WSTG;             // [4][WGE]
  const double* Ur0 = k.U + (int64_t)cA * k.ld + kA;
  const double* Ur1 = k.U + (int64_t)(8 + cA) * k.ld + kA;
  // stage m (in this warp's global sequence: group g_m = blockIdx.x + (m / nsw)·gridDim.x, stage m % nsw)
  // → ring slot m % WPS.  Rows past n8 and columns past p8 are zero-filled.
  auto issue = [&](int m) {
    const int gi = nsw > 0 ? m / nsw : 0;
    const int g = blockIdx.x + gi * gridDim.x;
    if (nsw > 0 && g < ngroups) {
      const int t0 = g * WGT, ncol = min(WGT, k.ntiles - t0) * kPt;
      const double* Zg = k.Z + (int64_t)t0 * kPt * k.ld;
      double* dst = ring + (m % WPS) * WSTG;
      const int64_t row0 = (int64_t)(warp + NWP * (m % nsw)) * WSR;
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const int c = lane + 32 * i, col = c >> 3, part = c & 7;
        const bool ok = col < ncol && row0 + 2 * part < k.n8;
        cp_async16(dst + col * WLDS + 2 * part, ok ? Zg + (int64_t)col * k.ld + row0 + 2 * part : k.Z, ok ? 16 : 0);
      }
    }
    cp_commit();
  };
  int m = 0;   // this warp's next stage to consume
#pragma unroll
  for (int q = 0; q < WPS - 1; q++) issue(q);
  // u rows of a stage (a0 / a1: the lane's nodes cA, 8 + cA), loaded one stage ahead (L2 latency off the
  // DMMA path)
  double ua[4], ub[4];
  auto load_u = [&](int sI, double* xa, double* xb) {
    const int64_t row0 = (int64_t)(warp + NWP * sI) * WSR;
#pragma unroll
    for (int ks = 0; ks < 4; ks++) {
      // the last stage may run past n8 (and past ld): those rows of Z are zero-filled, u is not read
      const bool rv = nsw > 0 && row0 + 4 * ks + kA < k.n8;
      xa[ks] = (a0 && rv) ? __ldcg(Ur0 + row0 + 4 * ks) : 0.0;
      xb[ks] = (a1 && rv) ? __ldcg(Ur1 + row0 + 4 * ks) : 0.0;
    }
  };
  // u rows two stages ahead, rotating three register sets (L2 latency under full HBM load exceeds one
  // stage of DMMAs)
  double va[4], vb[4], wa[4], wb[4];
  load_u(0, ua, ub);
  load_u(nsw > 1 ? 1 : 0, va, vb);
  for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const int t0 = g * WGT;
    const int nt = min(WGT, k.ntiles - t0);
    double acc[WGT][2][2];
#pragma unroll
    for (int t = 0; t < WGT; t++) acc[t][0][0] = acc[t][0][1] = acc[t][1][0] = acc[t][1][1] = 0.0;
    // one stage: refill the ring WPS − 1 ahead, load the next stage's u rows into (na, nb), compute
    // with (xa, xb); the loop below alternates the two u register sets (no copies on the load path)
    auto step = [&](int sI, const double* xa, const double* xb, double* na, double* nb) {
      issue(m + WPS - 1);
      load_u((sI + 2) % nsw, na, nb);   // two stages ahead (the next group restarts at 0)
      cp_wait<WPS - 1>();
      __syncwarp();
      const double* bp = ring + (m % WPS) * WSTG + cA * WLDS + kA;
#pragma unroll
      for (int ks = 0; ks < 4; ks++) {
        double x[WGT];
#pragma unroll
        for (int t = 0; t < WGT; t++) x[t] = bp[t * kPt * WLDS + 4 * ks];
#pragma unroll
        for (int t = 0; t < WGT; t++) dmma(acc[t][0], x[t], xa[ks]);
#pragma unroll
        for (int t = 0; t < WGT; t++) dmma(acc[t][1], x[t], xb[ks]);
      }
      __syncwarp();   // the slot is refilled by a later issue
      m++;
    };
    // stage sI computes with set sI % 3 and loads stage sI + 2 into set (sI + 2) % 3; at the end of a group
    // the sets are rotated so that set 0 holds stage 0 of the next group (once per group, off the hot loop)
    int sI = 0;
    for (; sI + 3 <= nsw; sI += 3) {
      step(sI, ua, ub, wa, wb);
      step(sI + 1, va, vb, ua, ub);
      step(sI + 2, wa, wb, va, vb);
    }
    if (sI < nsw) step(sI, ua, ub, wa, wb), sI++;
    if (sI < nsw) step(sI, va, vb, ua, ub), sI++;
    // now (sI % 3) names the set holding stage 0 of the next group, the following set stage 1
    if (nsw % 3 == 1) {
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const double t0a = va[q], t0b = vb[q];
        va[q] = wa[q]; vb[q] = wb[q];   // stage 1 (loaded into w)
        ua[q] = t0a; ub[q] = t0b;       // stage 0 (loaded into v)
      }
    } else if (nsw % 3 == 2) {
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const double t0a = wa[q], t0b = wb[q];
        wa[q] = ua[q]; wb[q] = ub[q];
        va[q] = wa[q]; vb[q] = wb[q];   // stage 1 (loaded into u)
        ua[q] = t0a; ub[q] = t0b;       // stage 0 (loaded into w)
      }
    }
    // the next group's first stages are already in flight (issue runs WPS − 1 stages ahead)
    auto put = [&](double* dst) {
#pragma unroll
      for (int t = 0; t < WGT; t++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          dst[t * 128 + cA * kBC + 8 * h + 2 * kA] = acc[t][h][0];
          dst[t * 128 + cA * kBC + 8 * h + 2 * kA + 1] = acc[t][h][1];
        }
    };
    for (int half = 4; half >= 1; half >>= 1) {
      if (warp >= half && warp < 2 * half) put(red + (warp - half) * WGE);
      __syncthreads();
      if (warp < half) {
        const double* src = red + warp * WGE;
#pragma unroll
        for (int t = 0; t < WGT; t++)
#pragma unroll
          for (int h = 0; h < 2; h++) {
            acc[t][h][0] += src[t * 128 + cA * kBC + 8 * h + 2 * kA];
            acc[t][h][1] += src[t * 128 + cA * kBC + 8 * h + 2 * kA + 1];
          }
      }
      __syncthreads();
    }
    if (warp == 0) put(red);
    __syncthreads();
    const int node = tid & (kBC - 1);
    const bool active = (fl[node] & F_ACTIVE) != 0, cold = (fl[node] & F_COLD) != 0;
    double sT1 = 0.0, sT2 = 0.0, sT3 = 0.0, sT4 = 0.0;
#pragma unroll
    for (int i = 0; i < WGE / WTH; i++) {
      const int e = tid + WTH * i, t = e >> 7, el = e & 127, jj = el >> 4;
      if (t >= nt) continue;
      const int64_t tile = t0 + t, col = tile * kPt + jj;
      double* q = k.stt + tile * STQ;
      const double q_beta = q[el], q_v = q[STB + el], q_c = q[2 * STB + jj];
      const uint8_t q_code = reinterpret_cast<const uint8_t*>(q + 2 * STB + 8)[el];
      const double sv = red[e];
      const double w = q_c + k.rho * q_beta - q_v;
      double wn = 0.0, bo = 0.0;
      if (active) {
        const double b = (w - sv) * k.inv_rho;                                // b = D w, D = (I − ZᵀZ)/ρ (R1)
        const double bn = REFRESH ? q_beta : prox(k, b + q_v * k.inv_rho, q_code);
        const double vn = (REFRESH && cold) ? q_v : q_v + k.rho * (b - bn);   // cold: (0, 0), no refresh (R6)
        if (check) {
          sT1 = fma(b, sv, sT1);                                              // bᵀ(XᵀX b)
          sT2 += nu_f(k, fabs(q_c - sv), q_code);                            // Σ ν(|Xᵀr̂|)
          sT3 = fma(q_c, bn, sT3);                                            // cᵀβ
          sT4 += psi_f(k, bn, q_code);                                        // Σ ψ(β)
          k.bchk[col * kBC + node] = b;
        }
        q[el] = bn;
        q[STB + el] = vn;
        wn = q_c + k.rho * bn - vn;
        bo = bn;
      }
      W[col * kBC + node] = wn;
      if (check) Bb[col * kBC + node] = bo;
    }
    if (check) {
      csum[tid >> 4][node][0] = sT1;
      csum[tid >> 4][node][1] = sT2;
      csum[tid >> 4][node][2] = sT3;
      csum[tid >> 4][node][3] = sT4;
      __syncthreads();
      if (tid < kBC * 4) {
        const int nd = tid >> 2, term = tid & 3;
        double a = 0.0;
        for (int q = 0; q < WTH / kBC; q++) a += csum[q][nd][term];
        wsum[((int64_t)g * kBC + nd) * 4 + term] = a;
      }
    }
    __syncthreads();   // red and csum are reused by the next group
  }
  cp_wait<0>();
}

// dst = A W with per-warp cp.async rings: CTA (x, y) owns rows [256x, 256x + 256) and column chunk y;
// warp w streams rows 32w..32w+31 of the chunk in stages of 16 columns (4 k-steps, 4 KB) and keeps
// its 32 × 16 output block in registers (4 row tiles × 2 node halves).
constexpr int WFPR = 256;                    // rows per CTA
constexpr int WFPC = 16;                     // columns per stage
constexpr int WFLD = 36;                     // smem doubles per column of a stage (32 rows + pad)
constexpr int WFSTG = WFPC * WFLD;
constexpr size_t WFWD_SMEM = sizeof(double) * (size_t)(WTH / 32) * WPS * WFSTG;   // 144 KB
__global__ void __launch_bounds__(WTH, 1) wide_forward_p(const double* __restrict__ A, int64_t ld, int64_t n8,
                                                         int64_t p8, const double* __restrict__ W, int64_t cpc,
                                                         double* part) {
  extern __shared__ __align__(16) double wsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, cA = lane >> 2, kA = lane & 3;
  const int64_t r0 = (int64_t)blockIdx.x * WFPR + warp * 32;
  const int64_t c0 = (int64_t)blockIdx.y * cpc, c1 = min(p8, c0 + cpc);
  const int nst = (int)((c1 - c0 + WFPC - 1) / WFPC);
  double* ring = wsm + (size_t)warp * WPS * WFSTG;
  auto issue = [&](int m) {
    if (m < nst) {
      double* dst = ring + (m % WPS) * WFSTG;
      const int64_t cb = c0 + (int64_t)m * WFPC;
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const int c = lane + 32 * i, col = c >> 4, part = c & 15;
        const int64_t row = r0 + 2 * part;
        const bool ok = cb + col < c1 && row < n8;
        cp_async16(dst + col * WFLD + 2 * part, ok ? A + (cb + col) * ld + row : A, ok ? 16 : 0);
      }
    }
    cp_commit();
  };
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; i++) acc[i][0][0] = acc[i][0][1] = acc[i][1][0] = acc[i][1][1] = 0.0;
#pragma unroll
  for (int m = 0; m < WPS - 1; m++) issue(m);
  // the stage's w rows (B fragments), loaded one stage ahead
  auto load_w = [&](int m, double* x0, double* x1) {
    const int64_t cb = c0 + (int64_t)m * WFPC;
#pragma unroll
    for (int ks = 0; ks < 4; ks++) {
      const bool ok = m < nst && cb + 4 * ks + kA < c1;
      x0[ks] = ok ? __ldg(W + (cb + 4 * ks + kA) * kBC + cA) : 0.0;
      x1[ks] = ok ? __ldg(W + (cb + 4 * ks + kA) * kBC + 8 + cA) : 0.0;
    }
  };
  double b0[4], b1[4], n0[4], n1[4];
  load_w(0, b0, b1);
  int m = 0;
  auto step = [&](const double* x0w, const double* x1w, double* y0w, double* y1w) {
    issue(m + WPS - 1);
    load_w(m + 1, y0w, y1w);
    cp_wait<WPS - 1>();
    __syncwarp();
    const double* bp = ring + (m % WPS) * WFSTG + kA * WFLD + cA;
#pragma unroll
    for (int ks = 0; ks < 4; ks++) {
      double x[4];
#pragma unroll
      for (int i = 0; i < 4; i++) x[i] = bp[4 * ks * WFLD + 8 * i];
#pragma unroll
      for (int i = 0; i < 4; i++) dmma(acc[i][0], x[i], x0w[ks]);
#pragma unroll
      for (int i = 0; i < 4; i++) dmma(acc[i][1], x[i], x1w[ks]);
    }
    __syncwarp();
    m++;
  };
  while (m < nst) {
    step(b0, b1, n0, n1);
    if (m < nst) step(n0, n1, b0, b1);
  }
  cp_wait<0>();
  double* pb = part + (int64_t)blockIdx.y * kBC * ld;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const int64_t row = r0 + 8 * i + cA;
    if (row >= n8) continue;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      pb[(int64_t)(8 * h + 2 * kA) * ld + row] = acc[i][h][0];
      pb[(int64_t)(8 * h + 2 * kA + 1) * ld + row] = acc[i][h][1];
    }
  }
}

__global__ void wide_reduce(int64_t n, int64_t ld, int nchunk, const double* __restrict__ part, double* dst) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * kBC) return;
  const int64_t row = e % n, nd = e / n;
  double a = 0.0;
  for (int y = 0; y < nchunk; y++) a += part[((int64_t)y * kBC + nd) * ld + row];
  dst[nd * ld + row] = a;
}

// per node: the check totals (CTA partials in fixed order), ‖Xβ⁺‖², and the fused kernel's decision
__global__ void __launch_bounds__(WTH) wide_decide(KP k, int it, int nblk, const double* __restrict__ wsum,
                                                   const double* __restrict__ XB, const int* __restrict__ it0) {
  const int nd = blockIdx.x, tid = threadIdx.x;
  int fl = k.nodei[nd * 2];
  if (!(fl & F_ACTIVE)) return;
  __shared__ double red[WTH / 32][5];
  double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int q = tid; q < nblk; q += WTH)
    for (int t = 0; t < 4; t++) v[t] += wsum[((int64_t)q * kBC + nd) * 4 + t];
  for (int64_t i = tid; i < k.xn; i += WTH) {
    const double x = XB[(int64_t)nd * k.xld + i];
    v[4] = fma(x, x, v[4]);
  }
  for (int t = 0; t < 5; t++)
    for (int o = 16; o > 0; o >>= 1) v[t] += __shfl_xor_sync(0xffffffffu, v[t], o);
  if ((tid & 31) == 0)
    for (int t = 0; t < 5; t++) red[tid >> 5][t] = v[t];
  __syncthreads();
  if (tid != 0) return;
  double T[5];
  for (int t = 0; t < 5; t++) {
    T[t] = 0.0;
    for (int w = 0; w < WTH / 32; w++) T[t] += red[w][t];
  }
  const double dual = 0.5 * k.yy - 0.5 * T[0] - T[1];
  const double primal = 0.5 * k.yy - T[2] + 0.5 * T[4] + T[3];
  const double lbb = fmax(k.nodef[nd * 4 + 0], dual);   // running max of checked duals (R7)
  const double pub = k.prune_ub_dev ? *k.prune_ub_dev : k.prune_ub;
  if ((primal - lbb) / fmax(1.0, fabs(primal)) <= k.node_tol) fl = (fl & ~F_ACTIVE) | L0L2_FLAG_CONVERGED;
  else if (lbb >= pub) fl = (fl & ~F_ACTIVE) | L0L2_FLAG_PRUNED;   // early prune (R16)
  else if (it0[nd] + it >= k.max_iters) fl = (fl & ~F_ACTIVE) | L0L2_FLAG_MAXITER;
  k.nodef[nd * 4 + 0] = lbb;
  k.nodef[nd * 4 + 1] = primal;
  k.nodef[nd * 4 + 3] = dual;
  k.nodei[nd * 2 + 0] = fl;
  k.nodei[nd * 2 + 1] = it0[nd] + it;
}

__global__ void wide_outputs(KP k) {
  const int nd = threadIdx.x;
  if (nd >= k.nb || !((k.act_mask >> nd) & 1u)) return;
  const double lbb = k.nodef[nd * 4 + 0];
  k.out_lb[nd] = fmax(lbb, k.nodef[nd * 4 + 2]);
  k.out_primal[nd] = k.nodef[nd * 4 + 1];
  k.out_iters[nd] = k.nodei[nd * 2 + 1];
  k.out_flags[nd] = (uint8_t)(k.nodei[nd * 2] & (L0L2_FLAG_CONVERGED | L0L2_FLAG_MAXITER | L0L2_FLAG_PRUNED));
  if (k.out_lbbest) k.out_lbbest[nd] = lbb;
}

using AdmmKernel = void (*)(KP);
template <bool DIR>
AdmmKernel admm_kernel_t(int cls) {
  switch (cls) {
    case 0: return admm_persistent<CLS_KS[0], CLS_MT[0], DIR>;
    case 1: return admm_persistent<CLS_KS[1], CLS_MT[1], DIR>;
    case 2: return admm_persistent<CLS_KS[2], CLS_MT[2], DIR>;
    case 3: return admm_persistent<CLS_KS[3], CLS_MT[3], DIR>;
    default: return admm_persistent<CLS_KS[4], CLS_MT[4], DIR>;
  }
}
AdmmKernel admm_kernel(int cls, bool direct) {
  return direct ? admm_kernel_t<true>(cls) : admm_kernel_t<false>(cls);
}
int admm_class(int64_t n8) {
  for (int c = 0; c < NCLS; c++)
    if (n8 <= 4 * NMW * CLS_KS[c] && n8 <= 8 * NMW * CLS_MT[c]) return c;
  return -1;
}

}  // namespace

#ifdef L0L2_PROF
int debug_prof(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_prof, sizeof(g_prof));
  if (reset) {
    static unsigned long long zero[160][NW][8];
    cudaMemcpyToSymbol(g_prof, zero, sizeof(g_prof));
  }
  return (int)(sizeof(g_prof) / sizeof(unsigned long long));
}
#else
int debug_prof(unsigned long long*, int) { return 0; }
#endif

size_t admm_smem_bytes(int64_t ld) {
  return sizeof(double) * ((size_t)NST * kPt * ld + NST * STQ + 2 * NMW * 64 + 2 * 8 * 12 + 2 * 64 * 4 + kBC) +
         (NST + 4) * sizeof(uint64_t) + 3 * kBC * sizeof(int) + (2 * NST + 12) * sizeof(int) + NST * sizeof(unsigned) + 64;
}

int admm_alloc_wide(Ctx* c) {
  const int64_t p8 = round8(c->p), ld = c->ld;
  const int64_t nblk = (p8 / kPt + WGT - 1) / WGT;   // check-sum blocks (groups of the sweep, ≤ 4 tiles)
  c->wide = 1;
  c->admm_cls = -1;
  c->grid = 0;
  c->stt = (double*)dalloc(c, sizeof(double) * (p8 / kPt) * STQ);
  if (c->stt) L0L2_CUDA(c, cudaMemset(c->stt, 0, sizeof(double) * (p8 / kPt) * STQ));
  c->bchk = (double*)dalloc(c, sizeof(double) * p8 * kBC);
  c->U = (double*)dalloc(c, sizeof(double) * kBC * ld);
  c->wW = (double*)dalloc(c, sizeof(double) * p8 * kBC);
  c->wB = (double*)dalloc(c, sizeof(double) * p8 * kBC);
  c->wXB = (double*)dalloc(c, sizeof(double) * kBC * ld);
  c->wsum = (double*)dalloc(c, sizeof(double) * nblk * kBC * 4);
  c->wit0 = (int*)dalloc(c, sizeof(int) * kBC);
  // forward grid, one CTA per SM: row blocks × column chunks ≤ #SMs (chunks ≥ 64 columns, whole stages)
  c->wrb = (int)((round8(c->n) + WFPR - 1) / WFPR);
  c->wcc = (int)std::max<int64_t>(1, std::min<int64_t>(p8 / 64, c->sms / c->wrb));
  c->wcpc = ((p8 + c->wcc - 1) / c->wcc + WFPC - 1) / WFPC * WFPC;
  L0L2_CUDA(c, cudaFuncSetAttribute(wide_sweep_p<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WSWEEP_SMEM));
  L0L2_CUDA(c, cudaFuncSetAttribute(wide_sweep_p<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WSWEEP_SMEM));
  L0L2_CUDA(c, cudaFuncSetAttribute(wide_forward_p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WFWD_SMEM));
  c->wcc = (int)((p8 + c->wcpc - 1) / c->wcpc);
  c->wpart = (double*)dalloc(c, sizeof(double) * c->wcc * kBC * ld);
  c->node_f = (double*)dalloc(c, sizeof(double) * kBC * 4);
  c->node_i = (int*)dalloc(c, sizeof(int) * kBC * 2);
  c->badflag = (int*)dalloc(c, sizeof(int));
  if (!c->stt || !c->bchk || !c->U || !c->wW || !c->wB || !c->wXB || !c->wsum || !c->wit0 || !c->wpart || !c->node_f ||
      !c->node_i || !c->badflag)
    return set_err(c, L0L2_ENOMEM, "admm work space (wide-n path)");
  // rows n..ld of u stay 0 (the adjoint reads whole 4-row k-steps); padding columns of β, v stay 0
  L0L2_CUDA(c, cudaMemset(c->U, 0, sizeof(double) * kBC * ld));
  L0L2_CUDA(c, cudaMemset(c->bchk, 0, sizeof(double) * p8 * kBC));
  return L0L2_OK;
}

int admm_alloc(Ctx* c) {
  // the streamed operand: Z (n×p, ld) or, in the direct regime, D (p×p, ldD)
  const int64_t p8 = round8(c->p), ld = c->direct ? c->ldD : c->ld;
  const int64_t kn = c->direct ? c->p : c->n;
  c->admm_cls = admm_class(round8(kn));
  // the fused kernel's on-chip budget: n8 within its register classes and the 3-stage ring of n×8
  // tiles in shared memory (n ≤ 1056); beyond it (Z-form only) the wide-n path
  bool fits = c->admm_cls >= 0 && admm_smem_bytes(ld) + 1024 <= 227 * 1024;
  if (const char* e = getenv("L0L2_WIDE"))   // test hook: force the wide-n path
    if (atoi(e) != 0 && !c->direct) fits = false;
  if (!fits) {
    if (c->direct) return set_err(c, L0L2_EINVAL, "direct regime: p = %lld too large", (long long)c->p);
    return admm_alloc_wide(c);
  }
  const int ntiles = (int)(p8 / kPt);
  // an even grid: CTA pairs (2P, 2P+1) serve the two node halves; a sub-range may be empty.  At
  // least 2 tiles per CTA: for small p an iteration is latency-bound, and fewer CTAs cut the grid
  // barrier / reduction cost (C2, 125 tiles: ADMM 13% faster on 64 CTAs than on 124; C4 unchanged)
  // (two tiles per sub-range at most: ⌈ntiles/2⌉ sub-ranges, rounded up to even)
  c->grid = std::min(c->sms, std::max(2, ((ntiles + 1) / 2 + 1) & ~1));
  // ≤ 1 tile per sub-range (a paired CTA then streams ≤ 2 tiles, fewer than the ring's NST slots):
  // the tiles stay resident in shared memory across the sweeps of a launch (issue_stage)
  if (ntiles <= c->sms) c->grid = std::min(c->sms, std::max(2, (ntiles + 1) & ~1));
  if (const char* e = getenv("L0L2_GRID")) c->grid = std::max(1, std::min(c->grid, atoi(e)));   // testing hook
  c->grid = std::max(2, c->grid & ~1);
  c->stt = (double*)dalloc(c, sizeof(double) * (p8 / kPt) * STQ);
  if (c->stt) L0L2_CUDA(c, cudaMemset(c->stt, 0, sizeof(double) * (p8 / kPt) * STQ));   // padding stays 0
  c->bchk = (double*)dalloc(c, sizeof(double) * p8 * kBC);
  c->U = (double*)dalloc(c, sizeof(double) * kBC * ld);
  c->Ub = (double*)dalloc(c, sizeof(double) * kBC * ld);
  c->Upart = (double*)dalloc(c, sizeof(double) * c->grid * kBC * ld);
  c->sums = (double*)dalloc(c, sizeof(double) * 2 * c->grid * kBC * kSums);   // double-buffered by check parity
  c->sums2 = (double*)dalloc(c, sizeof(double) * c->grid * kBC);
  // sparse primal check: per-CTA segments of β⁺'s nonzeros (capacity = the CTA's columns) and the
  // dense per-node lists (capacity p/16: above it the forward-only Zβ sweep is cheaper)
  c->seg_cap = (int)((ntiles + c->grid - 1) / c->grid) * (kPt / NEW);   // columns per (CTA, epilogue warp)
  c->nz_cap = (int)std::max<int64_t>(256, round8(c->p) / 16);
  if (c->direct) c->nz_cap = (int)round8(c->p);   // no dense fallback (it needs Z): every β⁺ is gathered
  c->seg_idx = (int32_t*)dalloc(c, sizeof(int32_t) * c->grid * NEW * kBC * c->seg_cap);
  c->seg_val = (double*)dalloc(c, sizeof(double) * c->grid * NEW * kBC * c->seg_cap);
  c->seg_cnt = (int*)dalloc(c, sizeof(int) * c->grid * NEW * kBC);
  c->nz_idx = (int32_t*)dalloc(c, sizeof(int32_t) * kBC * c->nz_cap);
  c->nz_val = (double*)dalloc(c, sizeof(double) * kBC * c->nz_cap);
  if (!c->seg_idx || !c->seg_val || !c->seg_cnt || !c->nz_idx || !c->nz_val)
    return set_err(c, L0L2_ENOMEM, "sparse check work space");
  c->node_f = (double*)dalloc(c, sizeof(double) * kBC * 4);
  c->node_i = (int*)dalloc(c, sizeof(int) * kBC * 2);
  c->bar = (unsigned*)dalloc(c, sizeof(unsigned) * 2);
  c->badflag = (int*)dalloc(c, sizeof(int));
  if (!c->stt || !c->bchk || !c->U || !c->Ub || !c->Upart || !c->sums || !c->sums2 ||
      !c->node_f || !c->node_i || !c->bar || !c->badflag)
    return set_err(c, L0L2_ENOMEM, "admm work space");
  L0L2_CUDA(c, cudaMemset(c->U, 0, sizeof(double) * kBC * ld));
  L0L2_CUDA(c, cudaMemset(c->Ub, 0, sizeof(double) * kBC * ld));
  L0L2_CUDA(c, cudaMemset(c->Upart, 0, sizeof(double) * c->grid * kBC * ld));
  L0L2_CUDA(c, cudaMemset(c->bchk, 0, sizeof(double) * p8 * kBC));
  L0L2_CUDA(c, cudaMemset(c->bar, 0, sizeof(unsigned) * 2));
  const size_t smem = admm_smem_bytes(ld);
  const AdmmKernel kern = admm_kernel(c->admm_cls, c->direct != 0);
  {
    // the 3-stage Z ring (24·ld doubles) must fit with everything else: n ≤ 1056 on B200
    int optin = 0;
    cudaFuncAttributes fa{};
    L0L2_CUDA(c, cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
    L0L2_CUDA(c, cudaFuncGetAttributes(&fa, kern));
    if (smem + fa.sharedSizeBytes > (size_t)optin)
      return set_err(c, L0L2_EINVAL, "n = %lld needs %zu B of shared memory per CTA for the ADMM tile ring (> %d)",
                     (long long)c->n, smem + fa.sharedSizeBytes, optin);
  }
  L0L2_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int nblk = 0;
  L0L2_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nblk, kern, kAdmmThreads, smem));
  if (nblk < 1) return set_err(c, L0L2_EINVAL, "ADMM kernel does not fit an SM (n=%lld)", (long long)c->n);
  return L0L2_OK;
}

int pack_group(Ctx* c, int nb, const int64_t* fix_off, const int32_t* fix_idx, const uint8_t* fix_val,
               const double* const* warm_ptrs_dev, cudaStream_t st) {
  const int64_t p8 = round8(c->p);
  const int64_t tot = p8 * kBC;
  pack_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(c->p, p8, nb, c->stt, c->c, warm_ptrs_dev);
  L0L2_LAUNCHED(c);
  if (fix_off) {
    L0L2_CUDA(c, cudaMemsetAsync(c->badflag, 0, sizeof(int), st));
    scatter_fix<<<nb, 128, 0, st>>>(nb, fix_off, fix_idx, fix_val, c->stt, c->p, c->badflag);
    L0L2_LAUNCHED(c);
    int bad = 0;
    L0L2_CUDA(c, cudaMemcpyAsync(&bad, c->badflag, sizeof(int), cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    if (bad & 1) return set_err(c, L0L2_EINVAL, "fixing index out of range");
    if (bad & 2) return set_err(c, L0L2_EINVAL, "F0 ∩ F1 ≠ ∅ (S:28)");
  }
  return L0L2_OK;
}

// A group of more than 8 nodes runs as ONE launch with paired CTAs (one Z read feeds both node
// halves), or as two launches, one per half (each half stops on its own).  Paired measured faster
// at every config, L2-resident Z included (fixed 100 iterations, B = 16, ms per 16-node iteration,
// paired vs split: C2 0.030 vs 0.053, C3 0.058 vs 0.080, C5 0.059 vs 0.073); the split path stays
// behind L0L2_PAIR=0 and is covered by the parity tests.
int launch_admm(Ctx* c, const BoundArgs& a, unsigned mask, cudaStream_t st);
bool admm_paired(const Ctx* c) {
  (void)c;
  if (const char* e = getenv("L0L2_PAIR")) return atoi(e) != 0;   // tuning / test hook
  return true;
}

int run_admm_wide(Ctx* c, const BoundArgs& a, cudaStream_t st);

int run_admm(Ctx* c, const BoundArgs& a, cudaStream_t st) {
  if (!c->ev[0]) {
    for (auto& e : c->ev) L0L2_CUDA(c, cudaEventCreate(&e));
  }
  L0L2_CUDA(c, cudaEventRecord(c->ev[0], st));
  if (c->wide) {
    const int rc = run_admm_wide(c, a, st);
    if (rc) return rc;
    L0L2_CUDA(c, cudaEventRecord(c->ev[1], st));
    return L0L2_OK;
  }
  const bool split = a.nb > 8 && !admm_paired(c);
  const unsigned all = (1u << a.nb) - 1u;
  const unsigned masks[2] = {split ? (all & 0xFFu) : all, all & 0xFF00u};
  for (int l = 0; l < (split ? 2 : 1); l++) {
    int rc = launch_admm(c, a, masks[l], st);
    if (rc) return rc;
  }
  L0L2_CUDA(c, cudaEventRecord(c->ev[1], st));
  return L0L2_OK;
}

KP make_kp(Ctx* c, const BoundArgs& a, unsigned mask);

int launch_admm(Ctx* c, const BoundArgs& a, unsigned mask, cudaStream_t st) {
  init_nodes<<<1, 32, 0, st>>>(a.nb, mask, a.cold_mask, a.parent_lb, a.lbbest_in, a.it0_in, a.warm_ptrs, c->node_f,
                               c->node_i);
  L0L2_LAUNCHED(c);
  KP k = make_kp(c, a, mask);
  void* args[] = {&k};
  L0L2_CUDA(c, cudaLaunchCooperativeKernel((void*)admm_kernel(c->admm_cls, c->direct != 0), dim3(c->grid),
                                           dim3(kAdmmThreads), args, admm_smem_bytes(k.ld), st));
  L0L2_LAUNCHED(c);
  return L0L2_OK;
}

// step mode launches (column-sharded fused path, sharded.cu): phase 0 initialises the group's nodes
int admm_step(Ctx* c, const BoundArgs& a, int phase, int chk, double* tot_out, cudaStream_t st) {
  const unsigned mask = (1u << a.nb) - 1u;
  if (phase == 0) {
    init_nodes<<<1, 32, 0, st>>>(a.nb, mask, a.cold_mask, a.parent_lb, nullptr, nullptr, nullptr, c->node_f, c->node_i);
    L0L2_LAUNCHED(c);
  }
  KP k = make_kp(c, a, mask);
  k.step_mode = 1;
  k.step_phase = phase;
  k.step_chk = chk;
  k.tot_out = tot_out;
  k.compact = 0;
  void* args[] = {&k};
  L0L2_CUDA(c, cudaLaunchCooperativeKernel((void*)admm_kernel(c->admm_cls, c->direct != 0), dim3(c->grid),
                                           dim3(kAdmmThreads), args, admm_smem_bytes(k.ld), st));
  L0L2_LAUNCHED(c);
  return L0L2_OK;
}
int admm_step_decide(Ctx* c, const BoundArgs& a, int it, const double* tot, cudaStream_t st) {
  KP k = make_kp(c, a, (1u << a.nb) - 1u);
  step_decide<<<a.nb, 256, 0, st>>>(k, it, tot);
  L0L2_LAUNCHED(c);
  return L0L2_OK;
}
int admm_step_outputs(Ctx* c, const BoundArgs& a, cudaStream_t st) {
  KP k = make_kp(c, a, (1u << a.nb) - 1u);
  step_outputs<<<1, 32, 0, st>>>(k);
  L0L2_LAUNCHED(c);
  return L0L2_OK;
}

// The wide-n path (see wide_sweep): one group of ≤ 16 nodes, all its iterations, host-stepped; the
// host reads the 16 node flags after each check (the loop's only synchronisation).
int run_admm_wide(Ctx* c, const BoundArgs& a, cudaStream_t st) {
  const unsigned mask = (1u << a.nb) - 1u;
  init_nodes<<<1, 32, 0, st>>>(a.nb, mask, a.cold_mask, a.parent_lb, a.lbbest_in, a.it0_in, a.warm_ptrs, c->node_f,
                               c->node_i);
  L0L2_LAUNCHED(c);
  const KP k = make_kp(c, a, mask);
  const int nblk = (k.ntiles + WGT - 1) / WGT;   // check-sum blocks = column groups of the sweep
  const unsigned sgrid = (unsigned)std::min(nblk, c->sms);
  auto sweep = [&](bool refresh, int chk) {
    if (refresh) wide_sweep_p<true><<<sgrid, WTH, WSWEEP_SMEM, st>>>(k, chk, c->wW, c->wB, c->wsum);
    else wide_sweep_p<false><<<sgrid, WTH, WSWEEP_SMEM, st>>>(k, chk, c->wW, c->wB, c->wsum);
    L0L2_LAUNCHED(c);
    return L0L2_OK;
  };
  auto forward_of = [&](const double* A, const double* W, double* dst) {   // dst = A W (n × 16, K = p)
    wide_forward_p<<<dim3((unsigned)c->wrb, (unsigned)c->wcc), WTH, WFWD_SMEM, st>>>(A, c->ld, k.n8, k.p8, W, c->wcpc,
                                                                                      c->wpart);
    L0L2_LAUNCHED(c);
    wide_reduce<<<(unsigned)((c->n * kBC + 255) / 256), 256, 0, st>>>(c->n, c->ld, c->wcc, c->wpart, dst);
    L0L2_LAUNCHED(c);
    return L0L2_OK;
  };
  auto forward = [&](const double* W, double* dst) { return forward_of(c->Z, W, dst); };
  // u0 = Z(c + ρβ0 − v0), then the warm-start refresh (R6) and its u
  wide_w0<<<(unsigned)((k.p8 * kBC + WTH - 1) / WTH), WTH, 0, st>>>(k, c->wW, c->wit0);
  L0L2_LAUNCHED(c);
  int rc = forward(c->wW, c->U);
  if (rc) return rc;
  if ((rc = sweep(true, 0)) || (rc = forward(c->wW, c->U))) return rc;
  int hn[2 * kBC];
  L0L2_CUDA(c, cudaMemcpyAsync(hn, c->node_i, sizeof(hn), cudaMemcpyDeviceToHost, st));
  L0L2_CUDA(c, cudaStreamSynchronize(st));
  int it0[kBC];
  for (int nd = 0; nd < kBC; nd++) it0[nd] = hn[2 * nd + 1];
  for (int it = 1; it <= c->max_iters; it++) {
    bool chk = (it % c->check_every == 0) || (it == c->max_iters);
    for (int nd = 0; nd < kBC; nd++) chk |= (hn[2 * nd] & F_ACTIVE) && it0[nd] + it == c->max_iters;
    if ((rc = sweep(false, chk ? 1 : 0)) || (rc = forward(c->wW, c->U))) return rc;
    if (!chk) continue;
    if ((rc = forward_of(c->X, c->wB, c->wXB))) return rc;
    wide_decide<<<kBC, WTH, 0, st>>>(k, it, nblk, c->wsum, c->wXB, c->wit0);
    L0L2_LAUNCHED(c);
    L0L2_CUDA(c, cudaMemcpyAsync(hn, c->node_i, sizeof(hn), cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    bool any = false;
    for (int nd = 0; nd < kBC; nd++) any |= (hn[2 * nd] & F_ACTIVE) != 0;
    if (!any) break;
  }
  wide_outputs<<<1, 32, 0, st>>>(k);
  L0L2_LAUNCHED(c);
  return L0L2_OK;
}

KP make_kp(Ctx* c, const BoundArgs& a, unsigned mask) {
  KP k{};
  k.act_mask = mask;
  k.prune_ub = a.prune_ub;
  k.prune_ub_dev = a.prune_ub_dev;
  k.suspend_at = a.suspend_at;
  k.susp_min = a.susp_min;
  k.out_lbbest = a.out_lbbest;
  k.compact = 1;
  if (const char* e = getenv("L0L2_COMPACT")) k.compact = atoi(e) != 0;   // tuning / test hook
  k.Z = c->direct ? c->D : c->Z;
  k.Lt = c->Lt;
  k.direct = c->direct;
  k.xld = c->ld;
  k.xn = c->n;
  k.stt = c->stt; k.bchk = c->bchk;
  k.U = c->U; k.Ub = c->Ub; k.Upart = c->Upart; k.sums = c->sums; k.sums2 = c->sums2;
  k.nodef = c->node_f; k.nodei = c->node_i; k.bar = c->bar;
  k.seg_idx = c->seg_idx; k.seg_val = c->seg_val; k.seg_cnt = c->seg_cnt; k.nz_idx = c->nz_idx; k.nz_val = c->nz_val;
  k.X = c->X; k.seg_cap = c->seg_cap; k.nz_cap = c->nz_cap;
  // whole-column gather from the segments (measured faster at C4, C3 and C5: per 100 iterations at
  // B = 16, 29.5 vs 30.4 ms, 5.01 vs 5.38 ms, 5.38 vs 5.66 ms); the row-slice gather stays as the hook
  k.gather_mode = 0;
  if (const char* e = getenv("L0L2_GATHER")) k.gather_mode = atoi(e) != 0;   // test / tuning hook
  // testing hook (0 = always the dense sweep); the direct regime has no dense fallback (it needs Z)
  if (const char* e = getenv("L0L2_NZCAP"))
    if (!c->direct) k.nz_cap = std::min(k.nz_cap, atoi(e));
  k.out_lb = a.lb; k.out_primal = a.primal; k.out_iters = a.iters; k.out_flags = a.flags;
  k.ld = c->direct ? c->ldD : c->ld;
  k.n = c->direct ? c->p : c->n;
  k.n8 = round8(k.n);
  k.p8 = round8(c->p);
  k.pfd = PFD_DEFAULT;
  k.pfs = 0;
  if (const char* e = getenv("L0L2_PFS")) k.pfs = std::max(0, atoi(e));   // tuning hook
  if (const char* e = getenv("L0L2_PFD")) k.pfd = std::max(0, atoi(e));   // tuning hook
  k.tsplit = 1;
  if (const char* e = getenv("L0L2_TSPLIT")) {                           // tuning hook
    const int v = atoi(e);
    k.tsplit = (v == 2 || v == 4 || v == 8) ? v : 1;
  }
  k.ntiles = (int)(k.p8 / kPt); k.nsr = c->grid; k.nb = a.nb; k.check_every = c->check_every; k.max_iters = c->max_iters;
  k.rho = c->rho; k.inv_rho = 1.0 / c->rho; k.lam0 = c->lam0; k.lam2 = c->lam2; k.M = c->M; k.yy = c->yy;
  k.node_tol = c->node_tol;
  k.shrink = c->rho / (c->rho + 2.0 * c->lam2);
  k.sr = std::sqrt(c->lam0 / c->lam2);
  k.sr_le_M = k.sr <= c->M;
  k.a_l1 = 2.0 * std::sqrt(c->lam0 * c->lam2) / c->rho;
  k.a_4 = c->lam0 / (c->M * c->rho) + c->lam2 * c->M / c->rho;
  k.psi_l1 = 2.0 * std::sqrt(c->lam0 * c->lam2);
  k.psi_4 = c->lam0 / c->M + c->lam2 * c->M;
  return k;
}

// Called after the stream has been synchronised past run_admm: accumulate the event-timed
// duration and the algorithmic work of the launch (iterations = max over its nodes + refresh).
int account_admm(Ctx* c, int nb, const int* iters_host) {
  float ms = 0.f;
  L0L2_CUDA(c, cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
  account_admm_stats(c, nb, iters_host, ms);
  return L0L2_OK;
}

void account_admm_stats(Ctx* c, int nb, const int* iters_host, float ms) {
  // iterations streamed = Σ over the launches (one, or one per node half when split) of
  // (max iterations of its nodes + the refresh sweep)
  const bool split = nb > 8 && !admm_paired(c);
  int64_t tmax[2] = {0, 0}, tsum = 0;
  for (int k = 0; k < nb; k++) {
    const int l = split ? k / 8 : 0;
    tmax[l] = std::max<int64_t>(tmax[l], iters_host[k]);
    tsum += iters_host[k];
  }
  const int nl = split ? 2 : 1;
  double T = 0.0;
  for (int l = 0; l < nl; l++) T += (double)(tmax[l] + 1);
  // per iteration one read of the streamed operand (Z: n×p, or D: p×p in the direct regime) and the
  // node state; flops per node-iteration 4np (Zᵀ(Zw)) or 2p² (Dw)
  const double p = (double)c->p, kn = c->direct ? p : (double)c->n;
  const double fl = c->direct ? 2.0 * p * p : 4.0 * kn * p;
  c->ks.admm_launches += nl;
  c->ks.admm_iters += (int64_t)T;
  c->ks.admm_node_iters += tsum;
  c->ks.admm_ms += ms;
  c->ks.admm_bytes_alg += T * 8.0 * kn * p + 33.0 * p * (double)(tsum + nb);
  c->ks.admm_flops_alg += (double)(tsum + nb) * fl;
}

int scatter_chain_group(Ctx* c, int nb, const int* node_rec, const int* recs, int rec_stride, cudaStream_t st) {
  scatter_chain<<<nb, 32, 0, st>>>(nb, node_rec, recs, rec_stride, c->stt);
  L0L2_LAUNCHED(c);
  return L0L2_OK;
}

int finalize_group(Ctx* c, int nb, double* zhat, int32_t* branch_j, uint8_t* flags, int32_t* supp_cnt,
                   int32_t* supp_idx, int64_t supp_stride, cudaStream_t st) {
  const bool lam0_pos = c->lam0 > 0.0;
  const double zsr = lam0_pos ? std::sqrt(c->lam2 / c->lam0) : 0.0;
  finalize_kernel<<<nb, 512, 0, st>>>(c->p, c->M, zsr, lam0_pos, c->int_tol, c->stt, zhat, c->p,
                                      branch_j, flags, supp_cnt, supp_idx, supp_stride);
  L0L2_LAUNCHED(c);
  return L0L2_OK;
}

int unpack_warm(Ctx* c, int nb, double* const* warm_ptrs_dev, cudaStream_t st) {
  const int64_t tot = c->p * kBC;
  unpack_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(c->p, nb, c->stt, warm_ptrs_dev);
  L0L2_LAUNCHED(c);
  return L0L2_OK;
}

int dual_residual(Ctx* c, int nb, double* dual_r, int64_t ldr, cudaStream_t st) {
  const int64_t tot = c->n * nb;
  fill_y<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(dual_r, ldr, c->y, c->n, nb);
  L0L2_LAUNCHED(c);
  // r̂ = y − X b̂ with b̂ = b at the last check (op(B)(j, node) = bchk[node + j*kBC])
  return gemm_f64(c, c->n, nb, c->p, -1.0, c->X, c->ld, false, c->bchk, kBC, true, 1.0, dual_r, ldr, st);
}

}  // namespace l0l2

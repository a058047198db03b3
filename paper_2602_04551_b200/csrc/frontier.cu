// Device frontier of l0l2_solve (Algorithm 1, batched reading DESIGN.md
// R9) for a single rank in synchronous rounds: selection, pruning, incumbent update, branching and
// the frontier merge run on the device; the host reads one small status per round (plus the support
// offsets the upper-bound launch is sized from) and never sees a node descriptor.
//
// Data (HBM):
//   open set   a SORTED array of entries (LB, id, depth, warm slot, fixing record), double-buffered.
//              Sorted by (LB, id) — the best-first order of P:258/P:279 with FIFO ties — so
//              a round's batch is its prefix and the nodes pruned by LB ≥ UB(1−1e-12) are its suffix.
//   fixings    parent-linked records {parent record, 2j + value, parent id}; a node's (F0, F1) is the
//              chain from its record to the root (replaces the host's per-node fixing lists).
//   warm pool  the context's chunks of 2p-double slots (P:543 warm starts), with device refcounts and
//              a device free stack (children share their parent's slot, refcount 2).
//   incumbent  UB, support and β_S on the device.
// Per round: select (prune suffix, LB, batch = prefix) → [status] → per 16-node group: slot
// allocation, pack + fixing chains, ADMM, finalize, unpack → supports compacted → FPG upper bound →
// update (UB in id order, prune/branch in id order, children sorted) → merge of the rest of the open
// array with the children (merge-path positions by binary search, fully parallel).
// The arithmetic of every node and the order of every decision are those of the host frontier
// (solve.cu), so the trees are identical node for node (tested); only the orchestration moved.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace l0l2 {
namespace {

struct OpenEnt { double lb; long long id; int depth, slot, rec, pad; };   // 32 bytes
struct FixRec { int parent, fix; long long parent_id; };                  // fix = 2j + value
static_assert(sizeof(FixRec) == 16, "FixRec layout (scatter_chain reads ints 0, 1 of every 4)");

struct Scal {   // device scalars; the host reads the whole struct once per round
  long long n_open, nodes, node_iters, next_id, n_recs, n_trace;
  double ub, lbmin, ub_round;
  int n_free, nb, nC, pad;
};

constexpr int kTraceRec = 10;
constexpr int kChunk = 64;   // warm slots per pool chunk (as solve.cu's SlotPool)

__device__ __forceinline__ bool key_less(const OpenEnt& a, const OpenEnt& b) {
  return a.lb < b.lb || (a.lb == b.lb && a.id < b.id);
}
__device__ __forceinline__ void release(int s, int* ref, int* stack, int* n_free) {
  if (s < 0) return;
  if (atomicSub(&ref[s], 1) == 1) stack[atomicAdd(n_free, 1)] = s;
}

// prune the suffix LB ≥ UB(1−1e-12), report the global LB (min open = the first entry) and
// the batch size; the early-prune threshold of the round (R16) is the UB at its start
__global__ void fr_select(const OpenEnt* __restrict__ A, Scal* S, int* slot_ref, int* free_stack, int B, int early) {
  __shared__ long long np_s;
  const long long N = S->n_open;
  const double thr = S->ub * (1.0 - 1e-12);
  if (threadIdx.x == 0) {
    long long lo = 0, hi = N;   // first index with lb ≥ thr
    while (lo < hi) {
      const long long mid = (lo + hi) / 2;
      if (A[mid].lb >= thr) hi = mid; else lo = mid + 1;
    }
    np_s = lo;
  }
  __syncthreads();
  const long long np = np_s;
  for (long long i = np + threadIdx.x; i < N; i += blockDim.x) release(A[i].slot, slot_ref, free_stack, &S->n_free);
  __syncthreads();
  if (threadIdx.x == 0) {
    S->n_open = np;
    S->lbmin = np ? A[0].lb : S->ub;
    S->nb = (int)(np < B ? np : B);
    S->ub_round = early ? thr : INFINITY;
  }
}

// one 16-node group: warm pointers (parent's slot → in, a fresh slot → out), parent bounds, records
__global__ void fr_group(const OpenEnt* __restrict__ sel, int nb, Scal* S, int* slot_ref, int* free_stack,
                         double* const* chunk_base, long long p2, double** wptr, double* plb, int* node_rec,
                         int* out_slot) {
  const int k = threadIdx.x;
  if (k == 0)
    for (int q = 0; q < nb; q++) {
      int s = -1;
      if (S->n_free > 0) {   // pool exhausted: the children start cold (bounds stay valid)
        s = free_stack[--S->n_free];
        slot_ref[s] = 1;
      }
      out_slot[q] = s;
    }
  __syncwarp();
  if (k < kBC) {
    double* in = nullptr;
    double* out = nullptr;
    if (k < nb) {
      const int si = sel[k].slot, so = out_slot[k];
      if (si >= 0) in = chunk_base[si / kChunk] + (long long)(si % kChunk) * p2;
      if (so >= 0) out = chunk_base[so / kChunk] + (long long)(so % kChunk) * p2;
      plb[k] = sel[k].lb;
      node_rec[k] = sel[k].rec;
    }
    wptr[k] = in;
    wptr[kBC + k] = out;
  }
}

// supports of the round's nodes (finalize wrote them to rows of stride p) → one contiguous list
__global__ void fr_supp(int nb, const int32_t* __restrict__ scnt, const int32_t* __restrict__ sidx, long long stride,
                        long long* soff, int32_t* sall) {
  const int k = blockIdx.x;
  long long o = 0;
  for (int q = 0; q < k; q++) o += scnt[q];
  if (k == 0 && threadIdx.x == 0) {
    long long t = 0;
    for (int q = 0; q < nb; q++) { soff[q] = t; t += scnt[q]; }
    soff[nb] = t;
  }
  for (int i = threadIdx.x; i < scnt[k]; i += blockDim.x) sall[o + i] = sidx[(long long)k * stride + i];
}

// Algorithm 1 body for the solved batch (R9): UB updates in id order (lowest id wins ties), then
// prune (LB ≥ UB(1−1e-12) or integral) or branch (F0 child first) in id order; children
// inherit the node's LB and share its final state; parents' states are released; children sorted
__global__ void fr_update(const OpenEnt* __restrict__ sel, int nb, const double* __restrict__ lb,
                          const double* __restrict__ primal, const int32_t* __restrict__ iters,
                          const int32_t* __restrict__ branch, const uint8_t* __restrict__ flags,
                          const double* __restrict__ obj, const int32_t* __restrict__ scnt,
                          const long long* __restrict__ soff, const int32_t* __restrict__ sall,
                          const double* __restrict__ beta_s, const int* __restrict__ out_slot, Scal* S, FixRec* recs,
                          OpenEnt* C, int* slot_ref, int* free_stack, int32_t* inc_S, double* inc_b, int* inc_n,
                          double* trace) {
  __shared__ int ord[128];
  __shared__ int inc_k;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int q = 0; q < nb; q++) {   // order by id (insertion sort, nb ≤ 128)
      int x = q;
      int a = q;
      while (a > 0 && sel[ord[a - 1]].id > sel[x].id) { ord[a] = ord[a - 1]; a--; }
      ord[a] = x;
    }
    double UB = S->ub;
    inc_k = -1;
    for (int a = 0; a < nb; a++) {
      const int q = ord[a];
      if (obj[q] < UB) { UB = obj[q]; inc_k = q; }
    }
    S->ub = UB;
  }
  __syncthreads();
  if (inc_k >= 0) {
    const int q = inc_k;
    const long long o = soff[q];
    for (int i = tid; i < scnt[q]; i += blockDim.x) { inc_S[i] = sall[o + i]; inc_b[i] = beta_s[o + i]; }
    if (tid == 0) *inc_n = scnt[q];
  }
  if (trace)
    for (int a = tid; a < nb; a += blockDim.x) {
      const int q = ord[a];
      const int r = sel[q].rec;
      double* t = trace + (S->n_trace + a) * kTraceRec;
      t[0] = (double)sel[q].id; t[1] = (double)sel[q].depth; t[2] = lb[q]; t[3] = primal[q]; t[4] = (double)iters[q];
      t[5] = (double)branch[q]; t[6] = (double)flags[q]; t[7] = obj[q];
      t[8] = r >= 0 ? (double)recs[r].parent_id : -1.0;
      t[9] = r >= 0 ? (double)recs[r].fix : -1.0;
    }
  __syncthreads();
  if (tid == 0) {
    const double thr = S->ub * (1.0 - 1e-12);
    long long next = S->next_id, nrec = S->n_recs, its = 0;
    int nC = 0;
    for (int a = 0; a < nb; a++) {
      const int q = ord[a];
      its += iters[q];
      const bool pruned = lb[q] >= thr || (flags[q] & L0L2_FLAG_INTEGRAL) || branch[q] < 0;
      if (pruned) {
        release(out_slot[q], slot_ref, free_stack, &S->n_free);
        continue;
      }
      const int j = branch[q];
      recs[nrec] = FixRec{sel[q].rec, 2 * j, sel[q].id};         // F0 ∪ {j}
      recs[nrec + 1] = FixRec{sel[q].rec, 2 * j + 1, sel[q].id}; // F1 ∪ {j}
      C[nC++] = OpenEnt{lb[q], next, sel[q].depth + 1, out_slot[q], (int)nrec, 0};
      C[nC++] = OpenEnt{lb[q], next + 1, sel[q].depth + 1, out_slot[q], (int)nrec + 1, 0};
      if (out_slot[q] >= 0) slot_ref[out_slot[q]] += 1;   // two children share the state (ref 2)
      next += 2;
      nrec += 2;
    }
    for (int a = 1; a < nC; a++) {   // sort the children by (LB, id)
      const OpenEnt x = C[a];
      int b = a;
      while (b > 0 && key_less(x, C[b - 1])) { C[b] = C[b - 1]; b--; }
      C[b] = x;
    }
    S->next_id = next;
    S->n_recs = nrec;
    S->nodes += nb;
    S->node_iters += its;
    if (trace) S->n_trace += nb;
    S->nC = nC;
  }
  __syncthreads();
  for (int q = tid; q < nb; q += blockDim.x) release(sel[q].slot, slot_ref, free_stack, &S->n_free);   // consumed
}

// merge the rest of the open array with the sorted children: each element's output position is its
// own index plus the number of elements of the other sequence before it (keys are unique: ids)
__global__ void fr_merge(const OpenEnt* __restrict__ R, long long nr, const OpenEnt* __restrict__ C,
                         OpenEnt* __restrict__ out, Scal* S) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int nC = S->nC;
  if (i < nr) {
    const OpenEnt e = R[i];
    int lo = 0, hi = nC;
    while (lo < hi) { const int m = (lo + hi) / 2; if (key_less(C[m], e)) lo = m + 1; else hi = m; }
    out[i + lo] = e;
  } else if (i < nr + nC) {
    const int j = (int)(i - nr);
    const OpenEnt e = C[j];
    long long lo = 0, hi = nr;
    while (lo < hi) { const long long m = (lo + hi) / 2; if (key_less(R[m], e)) lo = m + 1; else hi = m; }
    out[j + lo] = e;
  }
  if (i == 0) S->n_open = nr + nC;
}

__global__ void fr_init(OpenEnt* A, Scal* S, double ub, int n_free, int* free_stack, int nslots, int* slot_ref) {
  for (int s = threadIdx.x; s < nslots; s += blockDim.x) { free_stack[s] = nslots - 1 - s; slot_ref[s] = 0; }
  if (threadIdx.x == 0) {
    A[0] = OpenEnt{-INFINITY, 0, 0, -1, -1, 0};   // the root: cold, no fixings
    Scal z{};
    z.n_open = 1;
    z.next_id = 1;
    z.ub = ub;
    z.n_free = n_free;
    *S = z;
  }
}

using Clock = std::chrono::steady_clock;
double secs(Clock::time_point a) { return std::chrono::duration<double>(Clock::now() - a).count(); }

// growable device array (copy on growth, stream-ordered)
template <class T>
struct DArr {
  T* p = nullptr;
  long long cap = 0;
  int grow(long long need, cudaStream_t st, Ctx* c, long long keep) {
    if (need <= cap) return L0L2_OK;
    long long nc = std::max(need, std::max(2 * cap, 1024LL));
    T* q = nullptr;
    if (cudaMalloc(&q, sizeof(T) * nc) != cudaSuccess) { cudaGetLastError(); return set_err(c, L0L2_ENOMEM, "frontier arrays"); }
    if (p && keep > 0) L0L2_CUDA(c, cudaMemcpyAsync(q, p, sizeof(T) * keep, cudaMemcpyDeviceToDevice, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    if (p) cudaFree(p);
    p = q;
    cap = nc;
    return L0L2_OK;
  }
  void free() { if (p) cudaFree(p); p = nullptr; cap = 0; }
};

// the frontier's device arrays, kept in the context across solves (allocation is not free) and
// grown on demand
struct FrState {
  DArr<OpenEnt> A[2], Cb;
  DArr<FixRec> recs;
  DArr<double> trace;
  DArr<int> slot_ref, free_stack;
  DArr<double*> chunk_base;
  DArr<char> blk;
  std::vector<cudaEvent_t> evs;
  ~FrState() {
    A[0].free(); A[1].free(); Cb.free(); recs.free(); trace.free(); slot_ref.free(); free_stack.free();
    chunk_base.free(); blk.free();
    for (auto e : evs) cudaEventDestroy(e);
  }
};

}  // namespace

void frontier_free(Ctx* c) {
  delete static_cast<FrState*>(c->fr_state);
  c->fr_state = nullptr;
}

int solve_device(Ctx* c, const l0l2_solve_opts& o, double* beta, double* obj_out, double* gap_out, l0l2_stats* stats) {
  const auto T0 = Clock::now();
  if (!c->solve_stream) L0L2_CUDA(c, cudaStreamCreateWithFlags(&c->solve_stream, cudaStreamNonBlocking));
  cudaStream_t st = c->solve_stream;
  const int64_t p = c->p, p2 = 2 * p;
  const int B = o.batch;
  if (B > 128) return set_err(c, L0L2_EINVAL, "device frontier: batch ≤ 128");
  // ---- warm pool capacity (as the host frontier: opts cap or 25% of the HBM free at the first solve)
  size_t pool_cap;
  if (o.warm_bytes_cap > 0) {
    pool_cap = std::max<size_t>(kChunk, (size_t)o.warm_bytes_cap / (sizeof(double) * p2));
  } else {
    if (!c->pool_cap) {
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      c->pool_cap = std::max<size_t>(kChunk, fr / 4 / (sizeof(double) * p2));
    }
    pool_cap = c->pool_cap;
  }
  // ---- device state (kept in the context)
  if (!c->fr_state) c->fr_state = new FrState();
  FrState& F = *static_cast<FrState*>(c->fr_state);
  auto& A = F.A;
  auto& Cb = F.Cb;
  auto& recs = F.recs;
  auto& trace = F.trace;
  auto& slot_ref = F.slot_ref;
  auto& free_stack = F.free_stack;
  auto& chunk_base = F.chunk_base;
  auto& blk = F.blk;
  int rc = L0L2_OK;
  auto fail = [&](int code) { cudaStreamSynchronize(st); return code; };
  int nslots = (int)c->pool_chunks.size() * kChunk;
  if ((rc = A[0].grow(4096, st, c, 0)) || (rc = A[1].grow(4096, st, c, 0)) || (rc = Cb.grow(2 * B, st, c, 0)) ||
      (rc = recs.grow(8192, st, c, 0)) || (rc = slot_ref.grow(nslots + kChunk, st, c, 0)) ||
      (rc = free_stack.grow(nslots + kChunk, st, c, 0)) || (rc = chunk_base.grow(nslots / kChunk + 1, st, c, 0)))
    return fail(rc);
  if (o.record && (rc = trace.grow(4096 * kTraceRec, st, c, 0))) return fail(rc);
  // round buffers: scalars, batch results, supports
  size_t need = 0;
  auto sz = [&](size_t b) { size_t o2 = need; need += (b + 255) / 256 * 256; return o2; };
  const size_t oS = sz(sizeof(Scal)), oLB = sz(8 * B), oPR = sz(8 * B), oOBJ = sz(8 * B), oPLB = sz(8 * B),
               oIT = sz(4 * B), oBR = sz(4 * B), oSC = sz(4 * B), oFL = sz(B), oOS = sz(4 * B), oNR = sz(4 * B),
               oW = sz(sizeof(double*) * 2 * kBC * ((B + kBC - 1) / kBC)), oSO = sz(8 * (B + 1)),
               oSI = sz(sizeof(int32_t) * (size_t)B * p), oSA = sz(sizeof(int32_t) * (size_t)B * p),
               oBS = sz(sizeof(double) * (size_t)B * p), oIS = sz(sizeof(int32_t) * p), oIB = sz(sizeof(double) * p),
               oIN = sz(sizeof(int));
  if ((rc = blk.grow(need, st, c, 0))) return fail(rc);
  char* b0 = blk.p;
  Scal* S = (Scal*)(b0 + oS);
  double *d_lb = (double*)(b0 + oLB), *d_pr = (double*)(b0 + oPR), *d_obj = (double*)(b0 + oOBJ),
         *d_plb = (double*)(b0 + oPLB);
  int32_t *d_it = (int32_t*)(b0 + oIT), *d_br = (int32_t*)(b0 + oBR), *d_sc = (int32_t*)(b0 + oSC);
  uint8_t* d_fl = (uint8_t*)(b0 + oFL);
  int *d_os = (int*)(b0 + oOS), *d_nr = (int*)(b0 + oNR);
  double** d_w = (double**)(b0 + oW);
  long long* d_so = (long long*)(b0 + oSO);
  int32_t *d_si = (int32_t*)(b0 + oSI), *d_sa = (int32_t*)(b0 + oSA), *d_is = (int32_t*)(b0 + oIS);
  double *d_bs = (double*)(b0 + oBS), *d_ib = (double*)(b0 + oIB);
  int* d_in = (int*)(b0 + oIN);
  // ---- warm pool: every chunk the context already holds, all slots free
  {
    std::vector<double*> cb(c->pool_chunks.begin(), c->pool_chunks.end());
    if (!cb.empty())
      L0L2_CUDA(c, cudaMemcpyAsync(chunk_base.p, cb.data(), sizeof(double*) * cb.size(), cudaMemcpyHostToDevice, st));
  }
  // ---- initial incumbent: β = 0, or the matching-pursuit heuristic as in the host path
  double UB0 = 0.5 * c->yy;
  std::vector<int32_t> incS;
  std::vector<double> incB;
  double t_upper = 0.0, t_bound = 0.0, t_tree = 0.0;
  if (o.init_mp) {
    auto t0 = Clock::now();
    std::vector<int32_t> mS;
    std::vector<double> mb;
    double mobj = 0.0;
    if ((rc = mp_run(c, 0, st, mS, mb, &mobj, nullptr))) return fail(rc);
    if (mobj < UB0) {
      UB0 = mobj;
      incS = mS;
      incB.assign(mS.size(), 0.0);
      for (size_t i = 0; i < mS.size(); i++) incB[i] = mb[mS[i]];
    }
    if (!mS.empty()) {
      const long long off[2] = {0, (long long)mS.size()};
      L0L2_CUDA(c, cudaMemcpyAsync(d_so, off, sizeof(off), cudaMemcpyHostToDevice, st));
      L0L2_CUDA(c, cudaMemcpyAsync(d_sa, mS.data(), sizeof(int32_t) * mS.size(), cudaMemcpyHostToDevice, st));
      if ((rc = upper_batch(c, 1, (const int64_t*)d_so, d_sa, d_obj, d_bs, st))) return fail(rc);
      std::vector<double> h(mS.size() + 1);
      L0L2_CUDA(c, cudaMemcpyAsync(h.data(), d_obj, sizeof(double), cudaMemcpyDeviceToHost, st));
      L0L2_CUDA(c, cudaMemcpyAsync(h.data() + 1, d_bs, sizeof(double) * mS.size(), cudaMemcpyDeviceToHost, st));
      L0L2_CUDA(c, cudaStreamSynchronize(st));
      if (h[0] < UB0) {
        UB0 = h[0];
        incS = mS;
        incB.assign(h.begin() + 1, h.end());
      }
    }
    t_upper += secs(t0);
  }
  const int inc_n0 = (int)incS.size();
  L0L2_CUDA(c, cudaMemcpyAsync(d_in, &inc_n0, sizeof(int), cudaMemcpyHostToDevice, st));
  if (inc_n0) {
    L0L2_CUDA(c, cudaMemcpyAsync(d_is, incS.data(), sizeof(int32_t) * inc_n0, cudaMemcpyHostToDevice, st));
    L0L2_CUDA(c, cudaMemcpyAsync(d_ib, incB.data(), sizeof(double) * inc_n0, cudaMemcpyHostToDevice, st));
  }
  fr_init<<<1, 256, 0, st>>>(A[0].p, S, UB0, nslots, free_stack.p, nslots, slot_ref.p);
  L0L2_LAUNCHED(c);
  // ---- rounds
  auto& evs = F.evs;
  auto ev = [&](size_t i) -> cudaEvent_t {
    while (evs.size() <= i) { cudaEvent_t e; cudaEventCreate(&e); evs.push_back(e); }
    return evs[i];
  };
  int cur = 0, status = 0;
  long long rounds = 0, max_open = 0;
  bool notconv = false;
  double LB = -INFINITY;
  Scal h{};
  std::vector<int32_t> hit(B);
  std::vector<uint8_t> hfl(B);
  while (true) {
    auto tt = Clock::now();
    fr_select<<<1, 1024, 0, st>>>(A[cur].p, S, slot_ref.p, free_stack.p, B, o.early_prune ? 1 : 0);
    L0L2_LAUNCHED(c);
    L0L2_CUDA(c, cudaMemcpyAsync(&h, S, sizeof(Scal), cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    t_tree += secs(tt);
    max_open = std::max(max_open, h.n_open);
    if (h.n_open == 0) { LB = h.ub; status = 0; break; }
    LB = h.lbmin;
    if (h.ub > 0 && (h.ub - LB) / h.ub <= o.gap_tol) { status = 1; break; }
    if (o.node_limit > 0 && h.nodes >= o.node_limit) { status = 2; break; }
    if (o.time_limit_s > 0 && secs(T0) >= o.time_limit_s) { status = 3; break; }
    const int nb = h.nb;
    // capacities for this round (the stream is idle here)
    if ((rc = A[1 - cur].grow(h.n_open + 2 * nb, st, c, 0)) || (rc = A[cur].grow(h.n_open + 2 * nb, st, c, h.n_open)) ||
        (rc = recs.grow(h.n_recs + 2 * nb, st, c, h.n_recs)))
      return fail(rc);
    if (o.record && (rc = trace.grow((h.n_trace + nb) * kTraceRec, st, c, h.n_trace * kTraceRec))) return fail(rc);
    if (h.n_free < nb && (size_t)nslots < pool_cap) {   // grow the warm pool by whole chunks
      std::vector<int> ids;
      while (h.n_free + (int)ids.size() < nb && (size_t)nslots + kChunk <= std::max<size_t>(pool_cap, kChunk)) {
        // slot bookkeeping arrays follow the pool (their live prefix is kept)
        if ((rc = slot_ref.grow(nslots + kChunk, st, c, nslots)) ||
            (rc = free_stack.grow(nslots + kChunk, st, c, h.n_free + (long long)ids.size())) ||
            (rc = chunk_base.grow(nslots / kChunk + 1, st, c, nslots / kChunk)))
          return fail(rc);
        double* m = nullptr;
        if (cudaMalloc(&m, sizeof(double) * p2 * kChunk) != cudaSuccess) { cudaGetLastError(); break; }
        c->pool_chunks.push_back(m);
        c->pool_chunk_bytes = (int64_t)(sizeof(double) * p2 * kChunk);
        L0L2_CUDA(c, cudaMemcpyAsync(chunk_base.p + c->pool_chunks.size() - 1, &c->pool_chunks.back(), sizeof(double*),
                                     cudaMemcpyHostToDevice, st));
        for (int i = kChunk - 1; i >= 0; i--) ids.push_back(nslots + i);
        std::vector<int> zeros(kChunk, 0);
        L0L2_CUDA(c, cudaMemcpyAsync(slot_ref.p + nslots, zeros.data(), sizeof(int) * kChunk, cudaMemcpyHostToDevice, st));
        L0L2_CUDA(c, cudaStreamSynchronize(st));
        nslots += kChunk;
      }
      if (!ids.empty()) {
        L0L2_CUDA(c, cudaMemcpyAsync(free_stack.p + h.n_free, ids.data(), sizeof(int) * ids.size(),
                                     cudaMemcpyHostToDevice, st));
        const int nf = h.n_free + (int)ids.size();
        L0L2_CUDA(c, cudaMemcpyAsync(&S->n_free, &nf, sizeof(int), cudaMemcpyHostToDevice, st));
        L0L2_CUDA(c, cudaStreamSynchronize(st));
      }
    }
    rounds++;
    // ---- bound the batch = A[cur][0 .. nb), groups of ≤ 16 nodes
    const int ng = (nb + kBC - 1) / kBC;
    L0L2_CUDA(c, cudaEventRecord(ev(2 * ng), st));   // phase marks (GPU time): bound | upper
    for (int g = 0; g < ng; g++) {
      const int g0 = g * kBC, gn = std::min(kBC, nb - g0);
      double** wg = d_w + 2 * kBC * g;
      fr_group<<<1, 32, 0, st>>>(A[cur].p + g0, gn, S, slot_ref.p, free_stack.p, chunk_base.p, p2, wg, d_plb + g0,
                                 d_nr + g0, d_os + g0);
      L0L2_LAUNCHED(c);
      if ((rc = pack_group(c, gn, nullptr, nullptr, nullptr, (const double* const*)wg, st))) return fail(rc);
      if ((rc = scatter_chain_group(c, gn, d_nr + g0, (const int*)recs.p, 4, st))) return fail(rc);
      BoundArgs a{gn, d_plb + g0, d_lb + g0, d_pr + g0, d_it + g0, d_fl + g0};
      a.warm_ptrs = (const double* const*)wg;
      a.prune_ub_dev = &S->ub_round;
      L0L2_CUDA(c, cudaEventRecord(ev(2 * g), st));
      if ((rc = run_admm(c, a, st))) return fail(rc);
      L0L2_CUDA(c, cudaEventRecord(ev(2 * g + 1), st));
      if ((rc = finalize_group(c, gn, nullptr, d_br + g0, d_fl + g0, d_sc + g0, d_si + (int64_t)g0 * p, p, st)))
        return fail(rc);
      if ((rc = unpack_warm(c, gn, wg + kBC, st))) return fail(rc);
    }
    L0L2_CUDA(c, cudaEventRecord(ev(2 * ng + 1), st));
    // ---- upper bounds on the rounded supports
    fr_supp<<<nb, 128, 0, st>>>(nb, d_sc, d_si, p, d_so, d_sa);
    L0L2_LAUNCHED(c);
    if ((rc = upper_batch(c, nb, (const int64_t*)d_so, d_sa, d_obj, d_bs, st))) return fail(rc);   // syncs
    L0L2_CUDA(c, cudaEventRecord(ev(2 * ng + 2), st));
    // kernel accounting of the round's ADMM launches (the stream has passed them)
    L0L2_CUDA(c, cudaMemcpyAsync(hit.data(), d_it, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaMemcpyAsync(hfl.data(), d_fl, nb, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    for (int g = 0; g < ng; g++) {
      float ms = 0.f;
      L0L2_CUDA(c, cudaEventElapsedTime(&ms, ev(2 * g), ev(2 * g + 1)));
      account_admm_stats(c, std::min(kBC, nb - g * kBC), hit.data() + g * kBC, ms);
    }
    {
      float mb = 0.f, mu = 0.f;
      L0L2_CUDA(c, cudaEventSynchronize(ev(2 * ng + 2)));
      L0L2_CUDA(c, cudaEventElapsedTime(&mb, ev(2 * ng), ev(2 * ng + 1)));
      L0L2_CUDA(c, cudaEventElapsedTime(&mu, ev(2 * ng + 1), ev(2 * ng + 2)));
      t_bound += mb / 1e3;
      t_upper += mu / 1e3;
    }
    for (int q = 0; q < nb; q++) notconv |= (hfl[q] & L0L2_FLAG_MAXITER) != 0;
    // ---- tree update and frontier merge
    tt = Clock::now();
    fr_update<<<1, 256, 0, st>>>(A[cur].p, nb, d_lb, d_pr, d_it, d_br, d_fl, d_obj, d_sc, d_so, d_sa, d_bs, d_os, S,
                                 recs.p, Cb.p, slot_ref.p, free_stack.p, d_is, d_ib, d_in, o.record ? trace.p : nullptr);
    L0L2_LAUNCHED(c);
    const long long nr = h.n_open - nb;
    fr_merge<<<(unsigned)((nr + 2 * nb + 255) / 256), 256, 0, st>>>(A[cur].p + nb, nr, Cb.p, A[1 - cur].p, S);
    L0L2_LAUNCHED(c);
    cur ^= 1;
    t_tree += secs(tt);
    if (o.verbose)
      fprintf(stderr, "[l0l2] round %lld nodes %lld open %lld UB %.10g LB %.10g\n", rounds, h.nodes + nb, h.n_open,
              h.ub, LB);
  }
  // ---- result: the incumbent and the certificate
  int inc_n = 0;
  L0L2_CUDA(c, cudaMemcpyAsync(&inc_n, d_in, sizeof(int), cudaMemcpyDeviceToHost, st));
  L0L2_CUDA(c, cudaStreamSynchronize(st));
  std::vector<int32_t> hS(inc_n);
  std::vector<double> hB(inc_n);
  if (inc_n) {
    L0L2_CUDA(c, cudaMemcpyAsync(hS.data(), d_is, sizeof(int32_t) * inc_n, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaMemcpyAsync(hB.data(), d_ib, sizeof(double) * inc_n, cudaMemcpyDeviceToHost, st));
  }
  c->trace.clear();
  if (o.record && h.n_trace > 0) {
    c->trace.resize((size_t)h.n_trace * kTraceRec);
    L0L2_CUDA(c, cudaMemcpyAsync(c->trace.data(), trace.p, sizeof(double) * c->trace.size(), cudaMemcpyDeviceToHost, st));
  }
  L0L2_CUDA(c, cudaStreamSynchronize(st));
  std::memset(beta, 0, sizeof(double) * p);
  for (int i = 0; i < inc_n; i++) beta[hS[i]] = hB[i];
  const double ub = h.ub;
  const double g = ub > 0 ? std::max(0.0, (ub - LB) / ub) : 0.0;
  if (obj_out) *obj_out = ub;
  if (gap_out) *gap_out = g;
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->nodes = stats->nodes_global = h.nodes;
    stats->node_iters = stats->node_iters_global = h.node_iters;
    stats->rounds = rounds;
    stats->max_open = max_open;
    stats->t_total = secs(T0);
    stats->t_bound = t_bound;
    stats->t_upper = t_upper;
    stats->t_tree = t_tree;
    stats->lb = LB;
    stats->ub = ub;
    stats->gap = g;
    stats->status = status;
    stats->support_size = inc_n;
  }
  if (status >= 2) return L0L2_WLIMIT;
  return notconv ? L0L2_WNOTCONV : L0L2_OK;
}

}  // namespace l0l2

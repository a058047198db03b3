// Branch-and-bound driver l0l2_solve (Algorithm 1) and the multi-GPU
// frontier exchange over NCCL.
//
// Batched synchronous-round reading of Algorithm 1 (R9, identical to the oracle's
// bnb_solve so single-GPU trees can be compared node for node):
//   each round: drop open nodes with LB ≥ UB(1−1e-12); stop when none remain or
//   (UB − LB)/UB ≤ gap_tol; pop min(B, |N|) nodes by (LB, id);
//   bound them (l0l2_bound_batch machinery, warm started from the parent state kept in HBM,
//   P:543); upper bound on the rounded supports; apply every UB improvement of the
//   round (lowest id wins ties); then in id order prune (LB ≥ UB(1−1e-12) or integral ẑ)
//   or branch into (F0∪{j}, F1) and (F0, F1∪{j}) with the parent's bound.
// The node bodies (ADMM, finalize, FPG) run in this library's kernels; the host keeps the
// priority queue of node descriptors and the refcounted pool of parent warm states (in HBM).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <queue>

#include "common.cuh"

namespace l0l2 {

// ---------------------------------------------------------------- NCCL, loaded at run time
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi* load_nccl(std::string& err) {
  static NcclApi api;
  static bool tried = false, ok = false;
  if (tried) {
    if (!ok) err = "libnccl.so.2 not loadable";
    return ok ? &api : nullptr;
  }
  tried = true;
  api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!api.h) {
    err = std::string("dlopen libnccl.so.2: ") + dlerror();
    return nullptr;
  }
#define SYM(name, f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(api.h, name)); if (!api.f) { err = name; return nullptr; }
  SYM("ncclGetUniqueId", GetUniqueId)
  SYM("ncclCommInitRank", CommInitRank)
  SYM("ncclAllGather", AllGather)
  SYM("ncclAllReduce", AllReduce)
  SYM("ncclBroadcast", Broadcast)
  SYM("ncclSend", Send)
  SYM("ncclRecv", Recv)
  SYM("ncclGroupStart", GroupStart)
  SYM("ncclGroupEnd", GroupEnd)
  SYM("ncclCommDestroy", CommDestroy)
  SYM("ncclGetErrorString", GetErrorString)
#undef SYM
  ok = true;
  return &api;
}

// Sum of a device vector over the ranks, identical on every rank (column-sharded ADMM, sharded.cu;
// the sharded precompute): NCCL all-reduce on the stream, or over the host transport an all-gather
// and a sum in rank order on the host.
int shard_allreduce(Ctx* c, double* d, int64_t count, cudaStream_t st) {
  if (c->nranks <= 1 || count <= 0) return L0L2_OK;
  if (c->host_tr_set) {
    const size_t bytes = sizeof(double) * (size_t)count;
    std::vector<double> mine((size_t)count), all((size_t)count * c->nranks);
    L0L2_CUDA(c, cudaMemcpyAsync(mine.data(), d, bytes, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    const l0l2_transport& t = c->host_tr;
    if (t.allgather(t.user, mine.data(), all.data(), (int64_t)bytes))
      return set_err(c, L0L2_ENCCL, "host transport allgather failed");
    for (int64_t i = 0; i < count; i++) {
      double a = all[(size_t)i];
      for (int r = 1; r < c->nranks; r++) a += all[(size_t)r * count + i];
      mine[(size_t)i] = a;
    }
    L0L2_CUDA(c, cudaMemcpyAsync(d, mine.data(), bytes, cudaMemcpyHostToDevice, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    return L0L2_OK;
  }
  if (!c->nccl || !c->nccl_comm) return set_err(c, L0L2_ENCCL, "communicator not initialised");
  ncclResult_t r = c->nccl->AllReduce(d, d, (size_t)count, ncclDouble, ncclSum, (ncclComm_t)c->nccl_comm, st);
  if (r != ncclSuccess) return set_err(c, L0L2_ENCCL, "ncclAllReduce: %s", c->nccl->GetErrorString(r));
  return L0L2_OK;
}

// the cooperative ramp-up's column view (coop_view below): only what the view allocated itself (its
// X, Z, c, L and communicator belong to the full context)
void coop_free(Ctx* c) {
  Ctx* v = c->coop_view;
  if (!v) return;
  cudaDeviceSynchronize();
  for (void* q : v->owned) cudaFree(q);
  for (void* q : v->scr) if (q) cudaFree(q);
  if (v->sh_buf) cudaFree(v->sh_buf);
  if (v->gemm_ws) cudaFree(v->gemm_ws);
  for (auto e : v->ev) if (e) cudaEventDestroy(e);
  delete v;
  c->coop_view = nullptr;
}

void comm_free(Ctx* c) {
  coop_free(c);
  if (c->nccl && c->nccl_comm) c->nccl->CommDestroy((ncclComm_t)c->nccl_comm);
  c->nccl_comm = nullptr;
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  c->comm_stream = nullptr;
}

#define NCCL_CK(c, expr)                                                                        \
  do {                                                                                         \
    ncclResult_t r_ = (expr);                                                                  \
    if (r_ != ncclSuccess)                                                                     \
      return set_err((c), L0L2_ENCCL, "%s:%d %s: %s", __FILE__, __LINE__, #expr,               \
                     (c)->nccl->GetErrorString(r_));                                           \
  } while (0)

namespace {

using Clock = std::chrono::steady_clock;
static double secs(Clock::time_point a) { return std::chrono::duration<double>(Clock::now() - a).count(); }

struct Node {
  double lb;
  int64_t id;
  int32_t depth;
  std::vector<int32_t> fidx;
  std::vector<uint8_t> fval;
  int slot;   // warm state slot (−1 = cold)
  // continuous batching: a suspended node resumes from its own state with these
  double lbbest = -INFINITY;   // running max of its checked duals (R7)
  int32_t it0 = 0;             // ADMM iterations already run
  int64_t parent = -1;         // trace: parent id and the fixing that created the node (2j + value)
  int64_t lastfix = -1;
};
constexpr int kTraceRec = 10;   // doubles per l0l2_solve_trace record

struct NodeCmp {   // min-heap by (lb, id)
  bool operator()(const Node& a, const Node& b) const { return a.lb != b.lb ? a.lb > b.lb : a.id > b.id; }
};

// Refcounted pool of parent (β, v) states, 2p doubles each, in HBM.
// Refcounted parent warm states (2p doubles per slot) in chunks of HBM owned by the context and
// reused by later solves (cudaMalloc/cudaFree of ~26 MB chunks per solve cost ~10% of a C4 step).
struct SlotPool {
  Ctx* c = nullptr;
  int64_t p = 0;
  size_t cap = 0;
  std::vector<int> freel, ref;
  static constexpr int kPerChunk = 64;   // 64 slots (≈100 MB at C4) per cudaMalloc
  std::vector<double*>& chunk() const { return c->pool_chunks; }
  double* ptr(int s) const { return chunk()[s / kPerChunk] + (int64_t)(s % kPerChunk) * 2 * p; }
  void adopt() {   // the chunks earlier solves left in the context: all slots free
    for (size_t q = 0; q < chunk().size(); q++) add_slots();
  }
  void add_slots() {
    const int base = (int)ref.size();
    ref.resize(ref.size() + kPerChunk, 0);
    for (int i = kPerChunk - 1; i >= 0; i--) freel.push_back(base + i);
  }
  int alloc() {
    if (freel.empty()) {
      if ((chunk().size() + 1) * kPerChunk > cap) return -1;
      double* m = nullptr;
      if (cudaMalloc(&m, sizeof(double) * 2 * p * kPerChunk) != cudaSuccess) {
        cudaGetLastError();
        cap = chunk().size() * kPerChunk;
        return -1;
      }
      chunk().push_back(m);
      c->pool_chunk_bytes = (int64_t)(sizeof(double) * 2 * p * kPerChunk);
      add_slots();
    }
    const int s = freel.back();
    freel.pop_back();
    ref[s] = 1;
    return s;
  }
  void addref(int s) { if (s >= 0) ref[s]++; }
  void release(int s) {
    if (s < 0) return;
    if (--ref[s] == 0) freel.push_back(s);
  }
};

// Per-round device I/O buffers
struct RoundBufs {
  int64_t* fix_off = nullptr;
  int32_t* fix_idx = nullptr;
  uint8_t* fix_val = nullptr;
  double* parent_lb = nullptr;
  double *lbbest_in = nullptr, *lbbest_out = nullptr;
  int32_t* it0_in = nullptr;
  double *lb = nullptr, *primal = nullptr, *obj = nullptr, *beta_s = nullptr;
  int32_t *iters = nullptr, *branch = nullptr, *scnt = nullptr, *sidx = nullptr, *cidx = nullptr;
  int64_t* soff = nullptr;
  uint8_t* flags = nullptr;
  double** wptr = nullptr;
};

struct Status {   // exchanged every round (8 doubles = 64 B per rank)
  // ub: the rank's pruning threshold (its own incumbent or an adopted global UB); own: the objective
  // of the incumbent VECTOR this rank holds (never an adopted value), which elects the owner of β*
  double ub, lbmin, open, nodes, iters, elapsed, own, pad;
};

// Deterministic rebalancing plan from the open counts of all ranks (pure host logic):
// repeatedly move half the difference from the fullest to the emptiest rank while the emptiest
// has fewer than B nodes and the difference exceeds 1.  Ties → lowest rank.
}  // namespace

std::vector<int64_t> rebalance_plan(const std::vector<int64_t>& counts, int64_t B) {
  std::vector<int64_t> cnt = counts, plan;   // triples (src, dst, k)
  const int W = (int)cnt.size();
  for (int guard = 0; guard < 4 * W; guard++) {
    int hi = 0, lo = 0;
    for (int r = 1; r < W; r++) {
      if (cnt[r] > cnt[hi]) hi = r;
      if (cnt[r] < cnt[lo]) lo = r;
    }
    if (cnt[lo] >= B || cnt[hi] - cnt[lo] <= 1) break;
    int64_t k = (cnt[hi] - cnt[lo]) / 2;
    if (k <= 0) break;
    plan.push_back(hi);
    plan.push_back(lo);
    plan.push_back(k);
    cnt[hi] -= k;
    cnt[lo] += k;
  }
  return plan;
}

namespace {

// ---- cooperative ramp-up: before the frontier is partitioned every rank holds
// the same tree, so instead of solving the same nodes W times the ranks solve each node once TOGETHER
// through the column-sharded bound (sharded.cu) on their column block of the full context's Z.
// Column block r = [cut(r), cut(r+1)): multiples of 8 (a block's padding columns must be zero — only
// the last block has any, the context's own zero padding).
int64_t coop_cut(const Ctx* c, int r) {
  const int64_t p8 = round8(c->p);
  return std::min<int64_t>(c->p, round8(p8 * r / c->nranks));
}
bool coop_possible(const Ctx* c) {
  for (int r = 0; r < c->nranks; r++)
    if (coop_cut(c, r + 1) - coop_cut(c, r) < (int64_t)kPt) return false;
  return true;
}
// the rank's block as a column-sharded view: X, Z, c, colsq, L point INTO the full context (no copies);
// its own ADMM work space; the full context's communicator
int coop_view(Ctx* c, Ctx** out) {
  Ctx* v = c->coop_view;
  if (v && (v->rank != c->rank || v->p_total != c->p)) {
    coop_free(c);
    v = nullptr;
  }
  if (!v) {
    v = new Ctx();
    const int64_t col0 = coop_cut(c, c->rank), col1 = coop_cut(c, c->rank + 1);
    v->device = c->device; v->sms = c->sms; v->n = c->n; v->p = col1 - col0; v->ld = c->ld;
    v->lam0 = c->lam0; v->lam2 = c->lam2; v->M = c->M; v->rho = c->rho; v->node_tol = c->node_tol;
    v->int_tol = c->int_tol; v->check_every = c->check_every; v->max_iters = c->max_iters; v->yy = c->yy;
    v->X = c->X + col0 * c->ld; v->Z = c->Z + col0 * c->ld; v->y = c->y; v->c = c->c + col0;
    v->colsq = c->colsq + col0; v->L = c->L; v->Lt = c->Lt;
    v->sharded = 1; v->col0 = col0; v->p_total = c->p; v->direct = 0;
    v->nranks = c->nranks; v->rank = c->rank;
    c->coop_view = v;
    const int rc = admm_alloc(v);   // the fused step-mode kernel when n fits, else the GEMM loop
    v->shard_fused = (rc == L0L2_OK && !v->wide) ? 1 : 0;
    v->err.clear();
  }
  // the communicator may have been (re)initialised since: always the full context's
  v->nccl = c->nccl; v->nccl_comm = c->nccl_comm; v->host_tr = c->host_tr; v->host_tr_set = c->host_tr_set;
  *out = v;
  return L0L2_OK;
}

struct Solver {
  Ctx* c;
  l0l2_solve_opts o;
  cudaStream_t st = nullptr;
  SlotPool pool;
  RoundBufs d;
  std::priority_queue<Node, std::vector<Node>, NodeCmp> open;
  std::vector<Node> running;       // continuous batching: suspended nodes (resumed first)
  double UB = 0.0;                 // pruning threshold (≤ inc_ub: may be a global UB adopted from a peer)
  double inc_ub = 0.0;             // objective of the incumbent vector (inc_S, inc_b) held by this rank
  std::vector<int32_t> inc_S;
  std::vector<double> inc_b;
  int64_t next_id = 1, nodes = 0, node_iters = 0, rounds = 0, max_open = 0;
  double t_bound = 0, t_upper = 0, t_tree = 0, t_comm = 0;
  bool notconv = false;
  std::vector<double>* trace = nullptr;
  // multi-rank
  int W = 1, R = 0;
  bool partitioned = false;
  int64_t id_counter = 0, id_base = 0;
  int ub_owner = 0;
  int64_t moved = 0;   // nodes this rank sent away by rebalancing
  int64_t suspensions = 0;   // continuous batching: node suspensions (each resumed later)
  int64_t launch_slots = 0, launch_sweeps = 0;   // lane utilisation: Σ node-iterations / (16 · sweeps)

  int64_t new_id() {
    if (!partitioned) return next_id++;
    return id_base + (id_counter++) * W + R;
  }

  // the round I/O buffers, carved from one context-owned block (reallocated only for a larger B)
  int alloc_bufs(int Bmax) {
    const int64_t p = c->p;
    size_t need = 0;
    auto sz = [&](size_t b) { need += (b + 255) / 256 * 256; };
    sz(sizeof(int64_t) * (Bmax + 1)); for (int i = 0; i < 6; i++) sz(sizeof(double) * Bmax);
    for (int i = 0; i < 4; i++) sz(sizeof(int32_t) * Bmax);
    sz(sizeof(int32_t) * (size_t)kBC * p); sz(sizeof(int64_t) * (Bmax + 1)); sz(Bmax); sz(sizeof(double*) * 2 * kBC);
    if (c->solve_buf_B < Bmax) {
      if (c->solve_buf) cudaFree(c->solve_buf);
      c->solve_buf = nullptr;
      c->solve_buf_B = 0;
      if (cudaMalloc(&c->solve_buf, need) != cudaSuccess) {
        cudaGetLastError();
        return set_err(c, L0L2_ENOMEM, "solve buffers");
      }
      c->solve_buf_B = Bmax;
      c->solve_buf_bytes = need;
    }
    char* cur = (char*)c->solve_buf;
    auto A = [&](size_t b) { void* r = cur; cur += (b + 255) / 256 * 256; return r; };
    d.fix_off = (int64_t*)A(sizeof(int64_t) * (Bmax + 1));
    d.parent_lb = (double*)A(sizeof(double) * Bmax);
    d.lbbest_in = (double*)A(sizeof(double) * Bmax);
    d.lbbest_out = (double*)A(sizeof(double) * Bmax);
    d.it0_in = (int32_t*)A(sizeof(int32_t) * Bmax);
    d.lb = (double*)A(sizeof(double) * Bmax);
    d.primal = (double*)A(sizeof(double) * Bmax);
    d.obj = (double*)A(sizeof(double) * Bmax);
    d.iters = (int32_t*)A(sizeof(int32_t) * Bmax);
    d.branch = (int32_t*)A(sizeof(int32_t) * Bmax);
    d.scnt = (int32_t*)A(sizeof(int32_t) * Bmax);
    d.sidx = (int32_t*)A(sizeof(int32_t) * (size_t)kBC * p);
    d.soff = (int64_t*)A(sizeof(int64_t) * (Bmax + 1));
    d.flags = (uint8_t*)A(Bmax);
    d.wptr = (double**)A(sizeof(double*) * 2 * kBC);
    if (!d.fix_off || !d.parent_lb || !d.lb || !d.primal || !d.obj || !d.iters || !d.branch || !d.scnt ||
        !d.sidx || !d.soff || !d.flags || !d.wptr)
      return set_err(c, L0L2_ENOMEM, "solve buffers");
    return L0L2_OK;
  }

  // Solve one batch of nodes on this GPU; returns results in host vectors.
  struct Res {
    double lb, primal, obj;
    int32_t iters, branch;
    uint8_t flags;
    bool susp;        // suspended by continuous batching: resumes later from slot
    double lbbest;
    std::vector<int32_t> supp;
    std::vector<double> beta_s;
    int slot;
  };

  int process(std::vector<Node>& batch, std::vector<Res>& res) {
    const int B = (int)batch.size();
    res.assign(B, Res{});
    if (B == 0) return L0L2_OK;
    auto t0 = Clock::now();
    const int64_t p = c->p;
    // fixings (CSR) and parent bounds
    std::vector<int64_t> off(B + 1, 0);
    std::vector<int32_t> fidx;
    std::vector<uint8_t> fval;
    std::vector<double> plb(B), lbb(B);
    std::vector<int32_t> it0(B);
    bool resumed = false;
    for (int k = 0; k < B; k++) {
      fidx.insert(fidx.end(), batch[k].fidx.begin(), batch[k].fidx.end());
      fval.insert(fval.end(), batch[k].fval.begin(), batch[k].fval.end());
      off[k + 1] = (int64_t)fidx.size();
      plb[k] = batch[k].lb;
      lbb[k] = batch[k].lbbest;
      it0[k] = batch[k].it0;
      resumed |= batch[k].it0 > 0;
    }
    int32_t* dfi = (int32_t*)c->scratch_n(2, sizeof(int32_t) * std::max<size_t>(1, fidx.size()));
    uint8_t* dfv = (uint8_t*)c->scratch_n(3, std::max<size_t>(1, fval.size()));
    if (!dfi || !dfv) return set_err(c, L0L2_ENOMEM, "fix buffers");
    L0L2_CUDA(c, cudaMemcpyAsync(d.fix_off, off.data(), sizeof(int64_t) * (B + 1), cudaMemcpyHostToDevice, st));
    if (!fidx.empty()) {
      L0L2_CUDA(c, cudaMemcpyAsync(dfi, fidx.data(), sizeof(int32_t) * fidx.size(), cudaMemcpyHostToDevice, st));
      L0L2_CUDA(c, cudaMemcpyAsync(dfv, fval.data(), fval.size(), cudaMemcpyHostToDevice, st));
    }
    L0L2_CUDA(c, cudaMemcpyAsync(d.parent_lb, plb.data(), sizeof(double) * B, cudaMemcpyHostToDevice, st));
    if (resumed) {
      L0L2_CUDA(c, cudaMemcpyAsync(d.lbbest_in, lbb.data(), sizeof(double) * B, cudaMemcpyHostToDevice, st));
      L0L2_CUDA(c, cudaMemcpyAsync(d.it0_in, it0.data(), sizeof(int32_t) * B, cudaMemcpyHostToDevice, st));
    }
    std::vector<int32_t> scnt(B);
    for (int g0 = 0; g0 < B; g0 += kBC) {
      const int nb = std::min(kBC, B - g0);
      double* hp[2 * kBC] = {};
      for (int k = 0; k < nb; k++) {
        const Node& u = batch[g0 + k];
        hp[k] = u.slot >= 0 ? pool.ptr(u.slot) : nullptr;
        const int s = pool.alloc();
        res[g0 + k].slot = s;
        hp[kBC + k] = s >= 0 ? pool.ptr(s) : nullptr;
      }
      L0L2_CUDA(c, cudaMemcpyAsync(d.wptr, hp, sizeof(hp), cudaMemcpyHostToDevice, st));
      int rc = pack_group(c, nb, d.fix_off + g0, dfi, dfv, (const double* const*)d.wptr, st);
      if (rc) return rc;
      BoundArgs a{nb, d.parent_lb + g0, d.lb + g0, d.primal + g0, d.iters + g0, d.flags + g0};
      // cold: no parent state, or a resumed node (its own state continues, no refresh)
      for (int k = 0; k < nb; k++) if (!hp[k] || batch[g0 + k].it0 > 0) a.cold_mask |= 1u << k;
      if (o.early_prune) a.prune_ub = UB * (1.0 - 1e-12);   // UB of the round's start (R16)
      if (resumed) { a.lbbest_in = d.lbbest_in + g0; a.it0_in = d.it0_in + g0; }
      a.out_lbbest = d.lbbest_out + g0;
      // continuous batching: suspend the last few nodes of a launch while others are waiting
      if (o.continuous > 0 && W == 1 && !open.empty()) {
        a.suspend_at = o.continuous;
        a.susp_min = 2 * c->check_every;
      }
      if ((rc = run_admm(c, a, st))) return rc;
      if ((rc = finalize_group(c, nb, nullptr, d.branch + g0, d.flags + g0, d.scnt + g0, d.sidx, p, st))) return rc;
      if ((rc = unpack_warm(c, nb, d.wptr + kBC, st))) return rc;
      // supports of this group → host (counts first)
      L0L2_CUDA(c, cudaMemcpyAsync(scnt.data() + g0, d.scnt + g0, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, st));
      int32_t hit_g[kBC];
      L0L2_CUDA(c, cudaMemcpyAsync(hit_g, d.iters + g0, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, st));
      L0L2_CUDA(c, cudaStreamSynchronize(st));
      if ((rc = account_admm(c, nb, hit_g))) return rc;
      for (int k = 0; k < nb; k++) {
        res[g0 + k].supp.resize(scnt[g0 + k]);
        if (scnt[g0 + k] > 0)
          L0L2_CUDA(c, cudaMemcpyAsync(res[g0 + k].supp.data(), d.sidx + (int64_t)k * p, sizeof(int32_t) * scnt[g0 + k],
                                       cudaMemcpyDeviceToHost, st));
      }
    }
    std::vector<double> hlb(B), hpr(B), hlbb(B);
    std::vector<int32_t> hit(B), hbr(B);
    std::vector<uint8_t> hfl(B);
    L0L2_CUDA(c, cudaMemcpyAsync(hlb.data(), d.lb, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaMemcpyAsync(hlbb.data(), d.lbbest_out, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaMemcpyAsync(hpr.data(), d.primal, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaMemcpyAsync(hit.data(), d.iters, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaMemcpyAsync(hbr.data(), d.branch, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaMemcpyAsync(hfl.data(), d.flags, B, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    // the parents' warm states have been consumed by pack_group
    for (int k = 0; k < B; k++) pool.release(batch[k].slot);
    t_bound += secs(t0);
    return finish_upper(batch, res, hlb, hpr, hit, hbr, hfl, hlbb);
  }

  // upper bounds on the rounded supports of the nodes that finished, then the per-node results
  int finish_upper(std::vector<Node>& batch, std::vector<Res>& res, const std::vector<double>& hlb,
                   const std::vector<double>& hpr, const std::vector<int32_t>& hit, const std::vector<int32_t>& hbr,
                   const std::vector<uint8_t>& hfl, const std::vector<double>& hlbb) {
    const int B = (int)batch.size();
    auto t1 = Clock::now();
    std::vector<int64_t> so(B + 1, 0);
    std::vector<int32_t> sall;
    for (int k = 0; k < B; k++) {
      if (hfl[k] & kFlagSuspended) res[k].supp.clear();
      sall.insert(sall.end(), res[k].supp.begin(), res[k].supp.end());
      so[k + 1] = (int64_t)sall.size();
    }
    int32_t* dsi = (int32_t*)c->scratch_n(4, sizeof(int32_t) * std::max<size_t>(1, sall.size()));
    double* dbs = (double*)c->scratch_n(5, sizeof(double) * std::max<size_t>(1, sall.size()));
    if (!dsi || !dbs) return set_err(c, L0L2_ENOMEM, "support buffers");
    L0L2_CUDA(c, cudaMemcpyAsync(d.soff, so.data(), sizeof(int64_t) * (B + 1), cudaMemcpyHostToDevice, st));
    if (!sall.empty())
      L0L2_CUDA(c, cudaMemcpyAsync(dsi, sall.data(), sizeof(int32_t) * sall.size(), cudaMemcpyHostToDevice, st));
    int rc = upper_batch(c, B, d.soff, dsi, d.obj, dbs, st);
    if (rc) return rc;
    std::vector<double> hob(B), hbs(sall.size());
    L0L2_CUDA(c, cudaMemcpyAsync(hob.data(), d.obj, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
    if (!sall.empty())
      L0L2_CUDA(c, cudaMemcpyAsync(hbs.data(), dbs, sizeof(double) * sall.size(), cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    for (int k = 0; k < B; k++) {
      Res& r = res[k];
      r.lb = hlb[k];
      r.primal = hpr[k];
      r.iters = hit[k];
      r.branch = hbr[k];
      r.flags = hfl[k];
      r.obj = hob[k];
      r.beta_s.assign(hbs.begin() + so[k], hbs.begin() + so[k + 1]);
      r.susp = (r.flags & kFlagSuspended) != 0;
      r.lbbest = hlbb[k];
      if (r.susp) r.obj = INFINITY;
      if (r.flags & L0L2_FLAG_MAXITER) notconv = true;
      if (!r.susp) nodes++;
      node_iters += r.iters - batch[k].it0;
    }
    t_upper += secs(t1);
    return L0L2_OK;
  }

  // Cooperative bound of a batch that every rank holds (ramp-up): rank r runs the node relaxations on its
  // column block through the column-sharded path (one all-reduce of u = Σ_r Z_r w_r per iteration, the
  // check totals all-reduced: identical LB / primal / iterations / flags on every rank), the blocks of
  // the final (β, v) are all-gathered into full warm states, then finalize (branch, integrality,
  // support) and the upper bounds run on the full context — so every rank derives the same tree.
  int64_t coop_rounds = 0;
  int process_coop(std::vector<Node>& batch, std::vector<Res>& res) {
    const int B = (int)batch.size();
    res.assign(B, Res{});
    if (B == 0) return L0L2_OK;
    auto t0 = Clock::now();
    coop_rounds++;
    Ctx* v = nullptr;
    int rc = coop_view(c, &v);
    if (rc) return rc;
    const int64_t p = c->p, pr = v->p, col0 = v->col0;
    int64_t pmax = 0;
    for (int r = 0; r < W; r++) pmax = std::max(pmax, coop_cut(c, r + 1) - coop_cut(c, r));
    std::vector<double> hlb(B), hpr(B);
    std::vector<int32_t> hit(B), hbr(B);
    std::vector<uint8_t> hfl(B);
    std::vector<double> mine((size_t)B * 2 * pmax, 0.0);   // [node][β | v][pmax]: this rank's block
    for (int pass = 0; pass < 2; pass++) {   // nodes without a parent state (cold), then warm ones
      std::vector<int> ids;
      for (int k = 0; k < B; k++) if ((batch[k].slot < 0) == (pass == 0)) ids.push_back(k);
      if (ids.empty()) continue;
      const int nb = (int)ids.size();
      std::vector<int64_t> off(nb + 1, 0);
      std::vector<int32_t> fidx;
      std::vector<uint8_t> fval;
      std::vector<double> plb(nb);
      for (int i = 0; i < nb; i++) {
        const Node& u = batch[ids[i]];
        fidx.insert(fidx.end(), u.fidx.begin(), u.fidx.end());
        fval.insert(fval.end(), u.fval.begin(), u.fval.end());
        off[i + 1] = (int64_t)fidx.size();
        plb[i] = u.lb;
      }
      const size_t nw = (size_t)nb * 2 * pr;
      const size_t bytes = sizeof(int64_t) * (nb + 1) + sizeof(double) * (3 * nb + 2 * nw) + sizeof(int32_t) * nb +
                           sizeof(int32_t) * std::max<size_t>(1, fidx.size()) + nb + fval.size() + 256;
      char* blk = (char*)c->scratch_n(2, bytes);
      if (!blk) return set_err(c, L0L2_ENOMEM, "cooperative bound buffers");
      int64_t* d_off = (int64_t*)blk;
      double* d_plb = (double*)(d_off + nb + 1);
      double* d_lb = d_plb + nb;
      double* d_pr = d_lb + nb;
      double* d_win = d_pr + nb;
      double* d_wout = d_win + nw;
      int32_t* d_it = (int32_t*)(d_wout + nw);
      int32_t* d_fi = d_it + nb;
      uint8_t* d_fl = (uint8_t*)(d_fi + std::max<size_t>(1, fidx.size()));
      uint8_t* d_fv = d_fl + nb;
      L0L2_CUDA(c, cudaMemcpyAsync(d_off, off.data(), sizeof(int64_t) * (nb + 1), cudaMemcpyHostToDevice, st));
      L0L2_CUDA(c, cudaMemcpyAsync(d_plb, plb.data(), sizeof(double) * nb, cudaMemcpyHostToDevice, st));
      if (!fidx.empty()) {
        L0L2_CUDA(c, cudaMemcpyAsync(d_fi, fidx.data(), sizeof(int32_t) * fidx.size(), cudaMemcpyHostToDevice, st));
        L0L2_CUDA(c, cudaMemcpyAsync(d_fv, fval.data(), fval.size(), cudaMemcpyHostToDevice, st));
      }
      if (pass == 1)   // the parents' (β, v) on this rank's block
        for (int i = 0; i < nb; i++) {
          const double* ps = pool.ptr(batch[ids[i]].slot);
          L0L2_CUDA(c, cudaMemcpyAsync(d_win + (size_t)i * 2 * pr, ps + col0, sizeof(double) * pr,
                                       cudaMemcpyDeviceToDevice, st));
          L0L2_CUDA(c, cudaMemcpyAsync(d_win + (size_t)i * 2 * pr + pr, ps + p + col0, sizeof(double) * pr,
                                       cudaMemcpyDeviceToDevice, st));
        }
      rc = bound_sharded(v, nb, d_off, d_fi, d_fv, pass == 1 ? d_win : nullptr, d_plb, d_lb, d_pr, d_wout, d_it,
                         d_fl, st);
      if (rc < 0) return set_err(c, rc, "cooperative bound: %s", v->err.c_str());
      std::vector<double> tlb(nb), tpr(nb), tw(nw);
      std::vector<int32_t> tit(nb);
      std::vector<uint8_t> tfl(nb);
      L0L2_CUDA(c, cudaMemcpyAsync(tlb.data(), d_lb, sizeof(double) * nb, cudaMemcpyDeviceToHost, st));
      L0L2_CUDA(c, cudaMemcpyAsync(tpr.data(), d_pr, sizeof(double) * nb, cudaMemcpyDeviceToHost, st));
      L0L2_CUDA(c, cudaMemcpyAsync(tit.data(), d_it, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, st));
      L0L2_CUDA(c, cudaMemcpyAsync(tfl.data(), d_fl, nb, cudaMemcpyDeviceToHost, st));
      L0L2_CUDA(c, cudaMemcpyAsync(tw.data(), d_wout, sizeof(double) * nw, cudaMemcpyDeviceToHost, st));
      L0L2_CUDA(c, cudaStreamSynchronize(st));
      for (int i = 0; i < nb; i++) {
        const int k = ids[i];
        hlb[k] = tlb[i];
        hpr[k] = tpr[i];
        hit[k] = tit[i];
        hfl[k] = tfl[i];
        std::memcpy(&mine[((size_t)k * 2) * pmax], &tw[(size_t)i * 2 * pr], sizeof(double) * pr);
        std::memcpy(&mine[((size_t)k * 2 + 1) * pmax], &tw[(size_t)i * 2 * pr + pr], sizeof(double) * pr);
      }
    }
    // every rank's blocks of every node's (β, v)
    std::vector<double> all((size_t)W * B * 2 * pmax);
    {
      auto tc = Clock::now();
      if ((rc = xg_allgather(mine.data(), all.data(), sizeof(double) * mine.size()))) return rc;
      t_comm += secs(tc);
    }
    // full warm states → fresh pool slots (a full pool: a scratch state, the children start cold)
    std::vector<int64_t> off(B + 1, 0);
    std::vector<int32_t> fidx;
    std::vector<uint8_t> fval;
    for (int k = 0; k < B; k++) {
      fidx.insert(fidx.end(), batch[k].fidx.begin(), batch[k].fidx.end());
      fval.insert(fval.end(), batch[k].fval.begin(), batch[k].fval.end());
      off[k + 1] = (int64_t)fidx.size();
    }
    int32_t* dfi = (int32_t*)c->scratch_n(2, sizeof(int32_t) * std::max<size_t>(1, fidx.size()));
    uint8_t* dfv = (uint8_t*)c->scratch_n(3, std::max<size_t>(1, fval.size()) + sizeof(double) * 2 * p * kBC + 256);
    if (!dfi || !dfv) return set_err(c, L0L2_ENOMEM, "cooperative finalize buffers");
    double* tmp = (double*)(dfv + (std::max<size_t>(1, fval.size()) + 255) / 256 * 256);   // kBC × 2p
    L0L2_CUDA(c, cudaMemcpyAsync(d.fix_off, off.data(), sizeof(int64_t) * (B + 1), cudaMemcpyHostToDevice, st));
    if (!fidx.empty()) {
      L0L2_CUDA(c, cudaMemcpyAsync(dfi, fidx.data(), sizeof(int32_t) * fidx.size(), cudaMemcpyHostToDevice, st));
      L0L2_CUDA(c, cudaMemcpyAsync(dfv, fval.data(), fval.size(), cudaMemcpyHostToDevice, st));
    }
    L0L2_CUDA(c, cudaMemcpyAsync(d.flags, hfl.data(), B, cudaMemcpyHostToDevice, st));
    std::vector<double> full(2 * p);
    std::vector<int32_t> scnt(B);
    for (int g0 = 0; g0 < B; g0 += kBC) {
      const int nb = std::min(kBC, B - g0);
      double* hp[2 * kBC] = {};
      for (int k = 0; k < nb; k++) {
        for (int r = 0; r < W; r++) {
          const int64_t a = coop_cut(c, r), b = coop_cut(c, r + 1);
          const double* src = &all[(((size_t)r * B + g0 + k) * 2) * pmax];
          std::memcpy(&full[a], src, sizeof(double) * (b - a));
          std::memcpy(&full[p + a], src + pmax, sizeof(double) * (b - a));
        }
        double* t = tmp + (size_t)k * 2 * p;
        L0L2_CUDA(c, cudaMemcpyAsync(t, full.data(), sizeof(double) * 2 * p, cudaMemcpyHostToDevice, st));
        L0L2_CUDA(c, cudaStreamSynchronize(st));   // `full` is reused for the next node
        const int s2 = pool.alloc();
        res[g0 + k].slot = s2;
        if (s2 >= 0)
          L0L2_CUDA(c, cudaMemcpyAsync(pool.ptr(s2), t, sizeof(double) * 2 * p, cudaMemcpyDeviceToDevice, st));
        hp[k] = t;
      }
      L0L2_CUDA(c, cudaMemcpyAsync(d.wptr, hp, sizeof(hp), cudaMemcpyHostToDevice, st));
      if ((rc = pack_group(c, nb, d.fix_off + g0, dfi, dfv, (const double* const*)d.wptr, st))) return rc;
      if ((rc = finalize_group(c, nb, nullptr, d.branch + g0, d.flags + g0, d.scnt + g0, d.sidx, p, st))) return rc;
      L0L2_CUDA(c, cudaMemcpyAsync(scnt.data() + g0, d.scnt + g0, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, st));
      L0L2_CUDA(c, cudaStreamSynchronize(st));
      for (int k = 0; k < nb; k++) {
        res[g0 + k].supp.resize(scnt[g0 + k]);
        if (scnt[g0 + k] > 0)
          L0L2_CUDA(c, cudaMemcpyAsync(res[g0 + k].supp.data(), d.sidx + (int64_t)k * p, sizeof(int32_t) * scnt[g0 + k],
                                       cudaMemcpyDeviceToHost, st));
      }
    }
    L0L2_CUDA(c, cudaMemcpyAsync(hbr.data(), d.branch, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaMemcpyAsync(hfl.data(), d.flags, B, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    for (int k = 0; k < B; k++) pool.release(batch[k].slot);   // the parents' states were consumed
    t_bound += secs(t0);
    return finish_upper(batch, res, hlb, hpr, hit, hbr, hfl, hlb);
  }

  // Algorithm 1 body for one solved batch (id order; UB first, then prune/branch)
  void update_tree(std::vector<Node>& batch, std::vector<Res>& res) {
    const int B = (int)batch.size();
    std::vector<int> order(B);
    for (int k = 0; k < B; k++) order[k] = k;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return batch[a].id < batch[b].id; });
    for (int k : order)
      if (!res[k].susp && res[k].obj < UB) {
        UB = inc_ub = res[k].obj;
        inc_S = res[k].supp;
        inc_b = res[k].beta_s;
      }
    if (trace)
      for (int k : order) {
        const Res& r = res[k];
        if (r.susp) continue;
        const double rec[kTraceRec] = {(double)batch[k].id, (double)batch[k].depth, r.lb, r.primal, (double)r.iters,
                                       (double)r.branch, (double)r.flags, r.obj, (double)batch[k].parent,
                                       (double)batch[k].lastfix};
        trace->insert(trace->end(), rec, rec + kTraceRec);
      }
    for (int k : order) {
      Res& r = res[k];
      if (r.susp) {   // continuous batching: resumes in a later launch from its own state
        Node u = batch[k];
        u.lb = r.lb;
        u.lbbest = r.lbbest;
        u.it0 = r.iters;
        u.slot = r.slot;
        running.push_back(std::move(u));
        suspensions++;
        continue;
      }
      const bool integral = (r.flags & L0L2_FLAG_INTEGRAL) != 0;
      const bool pruned = r.lb >= UB * (1.0 - 1e-12) || integral || r.branch < 0;
      if (pruned) {
        pool.release(r.slot);
        continue;
      }
      const Node& u = batch[k];
      Node a{r.lb, 0, u.depth + 1, u.fidx, u.fval, r.slot};
      Node b{r.lb, 0, u.depth + 1, u.fidx, u.fval, r.slot};
      a.fidx.push_back(r.branch);
      a.fval.push_back(0);   // F0 ∪ {j}
      b.fidx.push_back(r.branch);
      b.fval.push_back(1);   // F1 ∪ {j}
      a.id = new_id();
      b.id = new_id();
      a.parent = b.parent = u.id;
      a.lastfix = 2 * (int64_t)r.branch;
      b.lastfix = 2 * (int64_t)r.branch + 1;
      pool.addref(r.slot);   // two children share the parent's state (ref 1 → 2)
      open.push(std::move(a));
      open.push(std::move(b));
    }
    max_open = std::max<int64_t>(max_open, (int64_t)open.size());
  }

  void prune_open() {
    {   // suspended nodes whose bound already prunes them
      std::vector<Node> keep;
      for (auto& u : running) {
        if (u.lb >= UB * (1.0 - 1e-12)) pool.release(u.slot);
        else keep.push_back(std::move(u));
      }
      running.swap(keep);
    }
    std::vector<Node> keep;
    keep.reserve(open.size());
    while (!open.empty()) {
      Node u = open.top();
      open.pop();
      if (u.lb >= UB * (1.0 - 1e-12)) pool.release(u.slot);
      else keep.push_back(std::move(u));
    }
    for (auto& u : keep) open.push(std::move(u));
  }

  double local_lbmin() const {
    double m = open.empty() ? INFINITY : open.top().lb;
    for (const auto& u : running) m = std::min(m, u.lb);
    return m;
  }
  int64_t local_open() const { return (int64_t)(open.size() + running.size()); }

  // ---- multi-rank helpers.  The carrier is NCCL (device buffers on the solve stream) or the
  // caller's host transport (l0l2_comm_init_transport); the exchange logic is the same.
  bool host_tr() const { return c->host_tr_set; }
  int tr_fail(const char* what) { return set_err(c, L0L2_ENCCL, "host transport %s failed", what); }

  // all-gather `bytes` of host data from every rank into out[W·bytes]
  int xg_allgather(const void* in, void* out, size_t bytes) {
    if (host_tr()) {
      const l0l2_transport& t = c->host_tr;
      return t.allgather(t.user, in, out, (int64_t)bytes) ? tr_fail("allgather") : L0L2_OK;
    }
    char* dbuf = (char*)c->scratch_n(2, bytes * (W + 1));
    if (!dbuf) return set_err(c, L0L2_ENOMEM, "allgather buffer");
    L0L2_CUDA(c, cudaMemcpyAsync(dbuf, in, bytes, cudaMemcpyHostToDevice, st));
    NCCL_CK(c, c->nccl->AllGather(dbuf, dbuf + bytes, bytes, ncclChar, (ncclComm_t)c->nccl_comm, st));
    L0L2_CUDA(c, cudaMemcpyAsync(out, dbuf + bytes, bytes * W, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    return L0L2_OK;
  }
  // point-to-point of DEVICE bytes (send on src, recv on dst, same order on both)
  int xg_send_dev(const void* d, size_t bytes, int peer) {
    if (host_tr()) {
      std::vector<char> h(bytes);
      L0L2_CUDA(c, cudaMemcpyAsync(h.data(), d, bytes, cudaMemcpyDeviceToHost, st));
      L0L2_CUDA(c, cudaStreamSynchronize(st));
      const l0l2_transport& t = c->host_tr;
      return t.send(t.user, h.data(), (int64_t)bytes, peer) ? tr_fail("send") : L0L2_OK;
    }
    NCCL_CK(c, c->nccl->Send(d, bytes, ncclChar, peer, (ncclComm_t)c->nccl_comm, st));
    return L0L2_OK;
  }
  int xg_recv_dev(void* d, size_t bytes, int peer) {
    if (host_tr()) {
      std::vector<char> h(bytes);
      const l0l2_transport& t = c->host_tr;
      if (t.recv(t.user, h.data(), (int64_t)bytes, peer)) return tr_fail("recv");
      L0L2_CUDA(c, cudaMemcpyAsync(d, h.data(), bytes, cudaMemcpyHostToDevice, st));
      L0L2_CUDA(c, cudaStreamSynchronize(st));
      return L0L2_OK;
    }
    NCCL_CK(c, c->nccl->Recv(d, bytes, ncclChar, peer, (ncclComm_t)c->nccl_comm, st));
    return L0L2_OK;
  }
  // host bytes point-to-point (staged through the device for NCCL)
  int xg_send_host(const void* h, size_t bytes, int peer) {
    if (host_tr()) {
      const l0l2_transport& t = c->host_tr;
      return t.send(t.user, h, (int64_t)bytes, peer) ? tr_fail("send") : L0L2_OK;
    }
    char* d = (char*)c->scratch_n(2, std::max<size_t>(8, bytes));
    if (!d) return set_err(c, L0L2_ENOMEM, "send buffer");
    L0L2_CUDA(c, cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
    int rc = xg_send_dev(d, bytes, peer);
    if (rc) return rc;
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    return L0L2_OK;
  }
  int xg_recv_host(void* h, size_t bytes, int peer) {
    if (host_tr()) {
      const l0l2_transport& t = c->host_tr;
      return t.recv(t.user, h, (int64_t)bytes, peer) ? tr_fail("recv") : L0L2_OK;
    }
    char* d = (char*)c->scratch_n(2, std::max<size_t>(8, bytes));
    if (!d) return set_err(c, L0L2_ENOMEM, "recv buffer");
    int rc = xg_recv_dev(d, bytes, peer);
    if (rc) return rc;
    L0L2_CUDA(c, cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    return L0L2_OK;
  }
  int xg_bcast_host(void* h, size_t bytes, int root) {
    if (host_tr()) {
      const l0l2_transport& t = c->host_tr;
      return t.bcast(t.user, h, (int64_t)bytes, root) ? tr_fail("bcast") : L0L2_OK;
    }
    char* d = (char*)c->scratch_n(3, std::max<size_t>(8, bytes));
    if (!d) return set_err(c, L0L2_ENOMEM, "bcast buffer");
    L0L2_CUDA(c, cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
    NCCL_CK(c, c->nccl->Broadcast(d, d, bytes, ncclChar, root, (ncclComm_t)c->nccl_comm, st));
    L0L2_CUDA(c, cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st));
    L0L2_CUDA(c, cudaStreamSynchronize(st));
    return L0L2_OK;
  }

  int allgather_status(const Status& mine, std::vector<Status>& all) {
    auto t0 = Clock::now();
    all.resize(W);
    int rc = xg_allgather(&mine, all.data(), sizeof(Status));
    t_comm += secs(t0);
    return rc;
  }

  // Move k nodes (the odd positions of the local best-first order first, then from the tail) from
  // src to dst with their warm states.  The source sends a header with the number of nodes it
  // actually holds for the move (≤ k), then per node [lb, id, depth, nfix, has_warm], then the
  // fixings and the warm states; the destination allocates pool slots (cold start when the pool is
  // full: the bound stays valid, only the warm start is lost).
  int rebalance(const std::vector<int64_t>& plan) {
    auto t0 = Clock::now();
    const int64_t p = c->p;
    for (size_t q = 0; q + 2 < plan.size(); q += 3) {
      const int src = (int)plan[q], dst = (int)plan[q + 1];
      int64_t k = plan[q + 2];
      if (R != src && R != dst) continue;
      const int peer = (R == src) ? dst : src;
      std::vector<Node> out;
      int64_t hdr[2] = {0, 0};   // nodes moved, fixings moved
      std::vector<double> meta;
      std::vector<int32_t> fix;
      if (R == src) {
        std::vector<Node> all;
        while (!open.empty()) { all.push_back(open.top()); open.pop(); }
        k = std::min<int64_t>(k, (int64_t)all.size());
        std::vector<Node> keep;
        for (size_t i = 0; i < all.size(); i++) {
          if ((int64_t)out.size() < k && (i % 2 == 1 || (int64_t)(all.size() - i) <= k - (int64_t)out.size()))
            out.push_back(std::move(all[i]));
          else
            keep.push_back(std::move(all[i]));
        }
        for (auto& u : keep) open.push(std::move(u));
        meta.assign(5 * out.size(), 0.0);
        for (size_t i = 0; i < out.size(); i++) {
          const Node& u = out[i];
          meta[5 * i + 0] = u.lb;
          meta[5 * i + 1] = (double)u.id;
          meta[5 * i + 2] = u.depth;
          meta[5 * i + 3] = (double)u.fidx.size();
          meta[5 * i + 4] = u.slot >= 0 ? 1.0 : 0.0;
          for (size_t f = 0; f < u.fidx.size(); f++) fix.push_back(u.fidx[f] * 2 + u.fval[f]);
        }
        hdr[0] = (int64_t)out.size();
        hdr[1] = (int64_t)fix.size();
        int rc = xg_send_host(hdr, sizeof(hdr), peer);
        if (!rc && hdr[0]) rc = xg_send_host(meta.data(), sizeof(double) * meta.size(), peer);
        if (!rc && hdr[1]) rc = xg_send_host(fix.data(), sizeof(int32_t) * fix.size(), peer);
        if (rc) return rc;
        // warm states: one device payload of hdr[0] × 2p doubles
        if (hdr[0]) {
          double* dpay = (double*)c->scratch_n(3, sizeof(double) * hdr[0] * 2 * p);
          if (!dpay) return set_err(c, L0L2_ENOMEM, "rebalance payload");
          for (int64_t i = 0; i < hdr[0]; i++) {
            double* dstp = dpay + i * 2 * p;
            if (out[i].slot >= 0)
              L0L2_CUDA(c, cudaMemcpyAsync(dstp, pool.ptr(out[i].slot), sizeof(double) * 2 * p, cudaMemcpyDeviceToDevice, st));
            else
              L0L2_CUDA(c, cudaMemsetAsync(dstp, 0, sizeof(double) * 2 * p, st));
          }
          if ((rc = xg_send_dev(dpay, sizeof(double) * hdr[0] * 2 * p, peer))) return rc;
          L0L2_CUDA(c, cudaStreamSynchronize(st));
        }
        for (auto& u : out) pool.release(u.slot);
        moved += hdr[0];
      } else {
        int rc = xg_recv_host(hdr, sizeof(hdr), peer);
        if (rc) return rc;
        meta.assign(5 * hdr[0], 0.0);
        fix.assign(hdr[1], 0);
        if (hdr[0] && (rc = xg_recv_host(meta.data(), sizeof(double) * meta.size(), peer))) return rc;
        if (hdr[1] && (rc = xg_recv_host(fix.data(), sizeof(int32_t) * fix.size(), peer))) return rc;
        double* dpay = nullptr;
        if (hdr[0]) {
          dpay = (double*)c->scratch_n(3, sizeof(double) * hdr[0] * 2 * p);
          if (!dpay) return set_err(c, L0L2_ENOMEM, "rebalance payload");
          if ((rc = xg_recv_dev(dpay, sizeof(double) * hdr[0] * 2 * p, peer))) return rc;
        }
        int64_t f = 0;
        for (int64_t i = 0; i < hdr[0]; i++) {
          Node u;
          u.lb = meta[5 * i + 0];
          u.id = (int64_t)meta[5 * i + 1];
          u.depth = (int32_t)meta[5 * i + 2];
          const int64_t nf = (int64_t)meta[5 * i + 3];
          for (int64_t q2 = 0; q2 < nf; q2++, f++) {
            u.fidx.push_back(fix[f] >> 1);
            u.fval.push_back((uint8_t)(fix[f] & 1));
          }
          u.slot = -1;
          if (meta[5 * i + 4] != 0.0) {
            u.slot = pool.alloc();
            if (u.slot >= 0)
              L0L2_CUDA(c, cudaMemcpyAsync(pool.ptr(u.slot), dpay + i * 2 * p, sizeof(double) * 2 * p,
                                           cudaMemcpyDeviceToDevice, st));
          }
          open.push(std::move(u));
        }
        L0L2_CUDA(c, cudaStreamSynchronize(st));
      }
    }
    t_comm += secs(t0);
    return L0L2_OK;
  }

  void partition() {
    std::vector<Node> all;
    while (!open.empty()) { all.push_back(open.top()); open.pop(); }
    for (size_t i = 0; i < all.size(); i++) {
      if ((int)(i % W) == R) open.push(std::move(all[i]));
      else pool.release(all[i].slot);
    }
    partitioned = true;
    id_base = next_id;
  }
};

}  // namespace
}  // namespace l0l2

using namespace l0l2;

extern "C" {

void l0l2_default_solve_opts(l0l2_solve_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->gap_tol = 1e-2;
  o->time_limit_s = 0.0;
  o->node_limit = 0;
  o->batch = 16;
  o->rebalance_every = 8;
  o->warm_bytes_cap = 0;
  o->verbose = 0;
  o->record = 0;
  o->init_mp = 0;
  o->early_prune = 0;
  o->continuous = 0;
  o->coop_rampup = 0;
}

int l0l2_nccl_unique_id(uint8_t out[128]) {
  std::string err;
  NcclApi* api = load_nccl(err);
  if (!api) return L0L2_ENCCL;
  ncclUniqueId id;
  if (api->GetUniqueId(&id) != ncclSuccess) return L0L2_ENCCL;
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(out, &id, 128);
  return L0L2_OK;
}

int l0l2_nccl_selftest(int32_t device) {
  std::string err;
  NcclApi* api = load_nccl(err);
  if (!api) return L0L2_ENCCL;
  if (cudaSetDevice(device) != cudaSuccess) return L0L2_ECUDA;
  ncclUniqueId id;
  if (api->GetUniqueId(&id) != ncclSuccess) return L0L2_ENCCL;
  ncclComm_t comm = nullptr;
  if (api->CommInitRank(&comm, 1, id, 0) != ncclSuccess) return L0L2_ENCCL;
  cudaStream_t st = nullptr;
  double* d = nullptr;
  int rc = L0L2_OK;
  const double h0[8] = {1, 2, 3, 4, 5, 6, 7, 8};
  double h[32] = {};
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess || cudaMalloc(&d, sizeof(double) * 32) != cudaSuccess)
    rc = L0L2_ECUDA;
  // the calls the solver's exchange uses (solve.cu xg_*, shard_allreduce), on one rank: all-reduce in
  // place, all-gather, broadcast, and a grouped send/recv to itself
  if (!rc && cudaMemcpyAsync(d, h0, sizeof(h0), cudaMemcpyHostToDevice, st) != cudaSuccess) rc = L0L2_ECUDA;
  if (!rc && api->AllReduce(d, d, 8, ncclDouble, ncclSum, comm, st) != ncclSuccess) rc = L0L2_ENCCL;
  if (!rc && api->AllGather(d, d + 8, 8 * sizeof(double), ncclChar, comm, st) != ncclSuccess) rc = L0L2_ENCCL;
  if (!rc && api->Broadcast(d + 8, d + 16, 8 * sizeof(double), ncclChar, 0, comm, st) != ncclSuccess) rc = L0L2_ENCCL;
  if (!rc) {
    if (api->GroupStart() != ncclSuccess) rc = L0L2_ENCCL;
    if (!rc && api->Send(d + 16, 8 * sizeof(double), ncclChar, 0, comm, st) != ncclSuccess) rc = L0L2_ENCCL;
    if (!rc && api->Recv(d + 24, 8 * sizeof(double), ncclChar, 0, comm, st) != ncclSuccess) rc = L0L2_ENCCL;
    if (api->GroupEnd() != ncclSuccess) rc = L0L2_ENCCL;
  }
  if (!rc && (cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
              cudaStreamSynchronize(st) != cudaSuccess))
    rc = L0L2_ECUDA;
  if (!rc)
    for (int i = 0; i < 32; i++)
      if (h[i] != h0[i % 8]) rc = L0L2_ENCCL;
  if (d) cudaFree(d);
  if (st) cudaStreamDestroy(st);
  api->CommDestroy(comm);
  return rc;
}

int l0l2_comm_init(l0l2_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t id[128]) {
  if (!ctx || nranks < 1 || rank < 0 || rank >= nranks) return L0L2_EINVAL;
  Ctx* c = &ctx->impl;
  if (nranks == 1) {
    c->nranks = 1;
    c->rank = 0;
    return L0L2_OK;
  }
  std::string err;
  c->nccl = load_nccl(err);
  if (!c->nccl) return set_err(c, L0L2_ENCCL, "%s", err.c_str());
  L0L2_CUDA(c, cudaSetDevice(c->device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  ncclComm_t comm;
  NCCL_CK(c, c->nccl->CommInitRank(&comm, nranks, uid, rank));
  c->nccl_comm = comm;
  c->host_tr_set = false;
  c->nranks = nranks;
  c->rank = rank;
  return L0L2_OK;
}

int l0l2_comm_init_transport(l0l2_ctx* ctx, int32_t nranks, int32_t rank, const l0l2_transport* t) {
  if (!ctx || nranks < 1 || rank < 0 || rank >= nranks) return L0L2_EINVAL;
  Ctx* c = &ctx->impl;
  if (nranks > 1 && (!t || !t->allgather || !t->send || !t->recv || !t->bcast))
    return set_err(c, L0L2_EINVAL, "transport callbacks missing");
  c->nranks = nranks;
  c->rank = rank;
  c->host_tr_set = nranks > 1;
  if (t) c->host_tr = *t;
  return L0L2_OK;
}

int64_t l0l2_solve_trace(const l0l2_ctx* ctx, double* rec, int64_t max_nodes) {
  if (!ctx) return -1;
  const std::vector<double>& t = ctx->impl.trace;
  const int64_t n = (int64_t)t.size() / kTraceRec;
  if (rec && max_nodes > 0) std::memcpy(rec, t.data(), sizeof(double) * kTraceRec * std::min(n, max_nodes));
  return n;
}

int l0l2_rebalance_plan(int32_t nranks, const int64_t* counts, int64_t batch, int64_t* plan, int32_t max_moves) {
  if (nranks < 1 || !counts || !plan) return -1;
  std::vector<int64_t> cnt(counts, counts + nranks);
  std::vector<int64_t> pl = rebalance_plan(cnt, batch);
  const int moves = (int)(pl.size() / 3);
  for (int i = 0; i < std::min(moves, (int)max_moves) * 3; i++) plan[i] = pl[i];
  return moves;
}

int l0l2_solve(l0l2_ctx* ctx, const l0l2_solve_opts* opts_in, double* beta, double* obj, double* gap,
               l0l2_stats* stats) {
  if (!ctx || !beta) return L0L2_EINVAL;
  Ctx* c = &ctx->impl;
  l0l2_solve_opts o;
  if (opts_in) o = *opts_in;
  else l0l2_default_solve_opts(&o);
  if (o.batch < 1) return set_err(c, L0L2_EINVAL, "batch < 1");
  L0L2_CUDA(c, cudaSetDevice(c->device));
  // single rank, synchronous rounds: the frontier lives on the device (frontier.cu);
  // L0L2_HOST_FRONTIER=1 selects this file's host frontier (test hook: the two give the same tree)
  const char* hf = getenv("L0L2_HOST_FRONTIER");
  if (c->nranks == 1 && o.continuous == 0 && o.batch <= 128 && !(hf && atoi(hf) != 0))
    return solve_device(c, o, beta, obj, gap, stats);
  const auto T0 = Clock::now();
  Solver S{};
  S.c = c;
  S.o = o;
  S.W = c->nranks;
  S.R = c->rank;
  if (S.W > 1 && !c->nccl_comm && !c->host_tr_set) return set_err(c, L0L2_ENCCL, "communicator not initialised");
  if (!c->solve_stream) L0L2_CUDA(c, cudaStreamCreateWithFlags(&c->solve_stream, cudaStreamNonBlocking));
  S.st = c->solve_stream;
  struct StreamGuard { cudaStream_t s; ~StreamGuard() { if (s) cudaStreamSynchronize(s); } } sg{S.st};
  S.pool.c = c;
  S.pool.p = c->p;
  if (o.warm_bytes_cap > 0) {
    S.pool.cap = std::max<size_t>(SlotPool::kPerChunk, (size_t)o.warm_bytes_cap / (sizeof(double) * 2 * c->p));
  } else {
    if (!c->pool_cap) {   // 25% of the HBM free at the first solve
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      c->pool_cap = std::max<size_t>(SlotPool::kPerChunk, fr / 4 / (sizeof(double) * 2 * c->p));
    }
    S.pool.cap = c->pool_cap;
  }
  S.pool.adopt();
  c->trace.clear();
  if (o.record) S.trace = &c->trace;
  int rc = S.alloc_bufs(o.batch);
  if (rc) return rc;
  S.UB = S.inc_ub = 0.5 * c->yy;   // β = 0 is feasible
  if (o.init_mp) {
    // root heuristic (Algorithm 3): MP's own point, then the box ridge on its support
    auto t0 = Clock::now();
    std::vector<int32_t> mS;
    std::vector<double> mb;
    double mobj = 0.0;
    if ((rc = mp_run(c, 0, S.st, mS, mb, &mobj, nullptr))) return rc;
    if (mobj < S.UB) {
      S.UB = S.inc_ub = mobj;
      S.inc_S = mS;
      S.inc_b.assign(mS.size(), 0.0);
      for (size_t i = 0; i < mS.size(); i++) S.inc_b[i] = mb[mS[i]];
    }
    if (!mS.empty()) {
      const int64_t off[2] = {0, (int64_t)mS.size()};
      int64_t* doff = (int64_t*)c->scratch_n(4, sizeof(int64_t) * 2 + sizeof(int32_t) * mS.size());
      double* dres = (double*)c->scratch_n(5, sizeof(double) * (mS.size() + 1));
      if (!doff || !dres) return set_err(c, L0L2_ENOMEM, "mp refit buffers");
      int32_t* didx = (int32_t*)(doff + 2);
      L0L2_CUDA(c, cudaMemcpyAsync(doff, off, sizeof(off), cudaMemcpyHostToDevice, S.st));
      L0L2_CUDA(c, cudaMemcpyAsync(didx, mS.data(), sizeof(int32_t) * mS.size(), cudaMemcpyHostToDevice, S.st));
      if ((rc = upper_batch(c, 1, doff, didx, dres, dres + 1, S.st))) return rc;
      std::vector<double> h(mS.size() + 1);
      L0L2_CUDA(c, cudaMemcpyAsync(h.data(), dres, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, S.st));
      L0L2_CUDA(c, cudaStreamSynchronize(S.st));
      if (h[0] < S.UB) {
        S.UB = S.inc_ub = h[0];
        S.inc_S = mS;
        S.inc_b.assign(h.begin() + 1, h.end());
      }
    }
    S.t_upper += secs(t0);
  }
  S.open.push(Node{-INFINITY, 0, 0, {}, {}, -1});
  double LB = -INFINITY;
  int status = 0;
  std::vector<Status> all;
  while (true) {
    auto tt = Clock::now();
    S.prune_open();
    S.t_tree += secs(tt);
    double gUB = S.UB, gLB;
    int64_t gopen = S.local_open(), gnodes = S.nodes;
    double elapsed = secs(T0);
    if (S.W > 1) {
      Status mine{S.UB, S.local_lbmin(), (double)S.open.size(), (double)S.nodes, (double)S.node_iters, elapsed,
                  S.inc_ub, 0};
      if ((rc = S.allgather_status(mine, all))) return rc;
      gopen = 0;
      gnodes = 0;
      gLB = INFINITY;
      for (int r = 0; r < S.W; r++) {
        gUB = std::min(gUB, all[r].ub);
        gLB = std::min(gLB, all[r].lbmin);
        gopen += (int64_t)all[r].open;
        gnodes += (int64_t)all[r].nodes;
        elapsed = std::max(elapsed, all[r].elapsed);
      }
      // owner of β* = the lowest rank whose OWN incumbent vector attains the global UB (a rank that
      // only adopted the value holds no matching vector)
      int owner = -1;
      for (int r = 0; r < S.W && owner < 0; r++) if (all[r].own == gUB) owner = r;
      S.ub_owner = owner < 0 ? 0 : owner;
      if (gUB < S.UB) {
        S.UB = gUB;   // the incumbent vector stays with its owner until the end
        S.prune_open();
      }
    } else {
      gLB = S.local_lbmin();
    }
    if (gopen == 0) { LB = gUB; status = 0; break; }
    LB = gLB;
    if (gUB > 0 && (gUB - LB) / gUB <= o.gap_tol) { status = 1; break; }
    if (o.node_limit > 0 && gnodes >= o.node_limit) { status = 2; break; }
    if (o.time_limit_s > 0 && elapsed >= o.time_limit_s) { status = 3; break; }
    if (S.W > 1) {
      if (!S.partitioned) {
        // every rank holds the same tree until here (identical rounds): split it once the LOCAL
        // frontier has a node for every rank
        if ((int64_t)S.open.size() >= S.W) S.partition();
      } else if (o.rebalance_every > 0 && S.rounds % o.rebalance_every == 0) {
        // the plan needs the open counts AFTER the global-UB prune above: exchange them
        const int64_t mine_open = (int64_t)S.open.size();
        std::vector<int64_t> cnt(S.W);
        auto t0 = Clock::now();
        if ((rc = S.xg_allgather(&mine_open, cnt.data(), sizeof(int64_t)))) return rc;
        S.t_comm += secs(t0);
        std::vector<int64_t> plan = rebalance_plan(cnt, o.batch);
        if (!plan.empty() && (rc = S.rebalance(plan))) return rc;
      }
    }
    std::vector<Node> batch;
    for (auto& u : S.running) batch.push_back(std::move(u));   // suspended nodes resume first
    S.running.clear();
    while (!S.open.empty() && (int)batch.size() < o.batch) {
      batch.push_back(S.open.top());
      S.open.pop();
    }
    S.rounds++;
    std::vector<Solver::Res> res;
    const bool coop = S.W > 1 && !S.partitioned && o.coop_rampup && coop_possible(c);
    if ((rc = coop ? S.process_coop(batch, res) : S.process(batch, res))) return rc;
    tt = Clock::now();
    S.update_tree(batch, res);
    S.t_tree += secs(tt);
    if (o.verbose && S.R == 0)
      fprintf(stderr, "[l0l2] round %lld nodes %lld open %zu UB %.10g LB %.10g gap %.3e\n", (long long)S.rounds,
              (long long)S.nodes, S.open.size(), S.UB, LB, gUB > 0 ? (gUB - LB) / gUB : 0.0);
  }
  // final incumbent → every rank
  const int64_t p = c->p;
  std::vector<double> hb(p, 0.0);
  for (size_t i = 0; i < S.inc_S.size(); i++) hb[S.inc_S[i]] = S.inc_b[i];
  double final_ub = S.inc_ub;
  if (S.W > 1) {
    // the owner (elected at the last status exchange, after which no rank solved a node) sends its
    // incumbent vector and that vector's own objective
    auto t0 = Clock::now();
    hb.push_back(S.inc_ub);
    if ((rc = S.xg_bcast_host(hb.data(), sizeof(double) * (p + 1), S.ub_owner))) return rc;
    final_ub = hb[p];
    Status mine{S.UB, 0, 0, (double)S.nodes, (double)S.node_iters, 0, S.inc_ub, (double)S.moved};
    if ((rc = S.allgather_status(mine, all))) return rc;
    S.t_comm += secs(t0);
  }
  std::memcpy(beta, hb.data(), sizeof(double) * p);
  const double g = final_ub > 0 ? std::max(0.0, (final_ub - LB) / final_ub) : 0.0;
  if (obj) *obj = final_ub;
  if (gap) *gap = g;
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->nodes = S.nodes;
    stats->node_iters = S.node_iters;
    stats->rounds = S.rounds;
    stats->max_open = S.max_open;
    stats->nodes_global = S.nodes;
    stats->node_iters_global = S.node_iters;
    stats->nodes_moved = S.moved;
    stats->suspensions = S.suspensions;
    stats->coop_rounds = S.coop_rounds;
    if (S.W > 1) {
      stats->nodes_moved = 0;
      for (int r = 0; r < S.W; r++) stats->nodes_moved += (int64_t)all[r].pad;
      stats->nodes_global = 0;
      stats->node_iters_global = 0;
      for (int r = 0; r < S.W; r++) {
        stats->nodes_global += (int64_t)all[r].nodes;
        stats->node_iters_global += (int64_t)all[r].iters;
      }
    }
    stats->t_total = secs(T0);
    stats->t_bound = S.t_bound;
    stats->t_upper = S.t_upper;
    stats->t_tree = S.t_tree;
    stats->t_comm = S.t_comm;
    stats->lb = LB;
    stats->ub = final_ub;
    stats->gap = g;
    stats->status = status;
    int64_t ss = 0;
    for (int64_t j = 0; j < p; j++) ss += beta[j] != 0.0;
    stats->support_size = (int32_t)ss;
  }
  if (status >= 2) return L0L2_WLIMIT;
  return S.notconv ? L0L2_WNOTCONV : L0L2_OK;
}

}  // extern "C"

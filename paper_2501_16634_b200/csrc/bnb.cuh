// Branch-and-bound argmin (the default search; included by loom_search.cu
// inside its anonymous namespace).
//
// The contract is the argmin of objective_less over the plans of a range
// (optimizer.hpp:173-188), not a per-plan compare, so a
// subtree of the ConfigEnumerator tree (optimizer.hpp:131-143: a prefix of
// digits fixed, node 0 most significant) can be dropped as a whole when a
// lower bound of its plans' criteria is infeasible or lexicographically
// STRICTLY worse than a real plan already found:
//   FP_A / FP_B  the dag-order left fold (estimator.hpp:50-60) of the prefix's
//                terms, continued with each free node's smallest term: FP
//                addition rounds monotonically, so the fold is monotone in
//                every term, and llround (estimator.hpp:85-87) is monotone;
//   latency      the finish-time recursion (estimator.hpp:69-76) with every
//                free node at its smallest wall (max-plus is monotone); it also
//                decides SLO feasibility;
//   quality      min(prefix quality, each free node's best) (an upper bound);
//   identifier   prefix rank terms + each free node's smallest term.
// If the bound vector is lexicographically greater than a plan's record,
// every plan of the subtree is strictly worse than that plan, so none can be
// the argmin.  Options failing the quality floor are never taken.  Leaves are
// evaluated exactly (the same folds, in the same order, as eval_digits).
//
// Parallel form: one DFS per warp.  Work units ("tasks") are the prefixes of
// the first T nodes in exploration order, dealt to warps by an atomic
// counter.  At a DFS node the 32 lanes evaluate 32 children at once (one
// chunk; nodes with more options take several chunks), a ballot leaves the
// mask of surviving children on a per-warp stack in shared memory, and the
// warp descends into the lowest survivor.  Children are explored best
// primary value first (BlobHeader.off_perm), so good plans arrive early.  The
// pruning bound is the best of the warp's own leaves and the job's global
// best, which warps publish under a lock and read through a sequence counter
// (a torn read is retried later, never used).  Because the order is strict
// and total, the result does not depend on timing.
//
// Blow-up guard: when the child evaluations of a job exceed a budget (a
// fraction of the plan count) the warps stop, and the sweep kernel that
// follows in the same stream searches the range exhaustively, starting from
// the best plan found so far (JobSync.pad = kBnbAborted).  Otherwise the
// sweep launch exits at once (kBnbDone).

constexpr int kBnbTasksPerWarp = 64;
// Evidence of the last launch's job 0: child evaluations and the abort flag
// (loom_bnb_last_stats).
__device__ unsigned long long g_bnb_last[6];
__device__ unsigned long long g_bnb_acc[2];
// Test knob (LOOM_BNB_BUDGET, read at context creation): a fixed evaluation
// budget, so tests can drive the depth-first search into its sweep fallback.
__device__ unsigned long long g_bnb_budget;  // running: max expansions of one task, tasks alive at the root

// Bounds of the free nodes below a child of node k (nodes k+1 .. n-1), per
// CTA.  FP sums: the fold of a child's prefix continued with the free
// nodes' smallest terms (estimator.hpp:50-60 order) is at least
// (prefix + sum of those terms) * (1 - 2^-53)^(free nodes) -- every
// round-to-nearest addition of non-negative values loses at most that factor
// -- so a = RD(sum of minima), fac = RD((1 - 2^-53)^m), and the bound
// RD(RD(prefix + a) * fac) is never above any plan's sum (inputs are
// validated non-negative and finite).  Quality: min of the free nodes' best;
// identifier rank: sum of their smallest terms.
struct BnbSuf {
  double a;
  double b;
  double fac;
  uint64_t lex;
  int32_t q;
  int32_t pad;
};

// Per-warp DFS state in shared memory.  Entry k of the prefix arrays holds
// the folds over nodes [0, k); wsel[v] is the wall node v contributes to the
// latency bound (its chosen option when fixed, its smallest wall when free).
struct BnbWarp {
  double fa[kMaxNodes + 1];
  double fb[kMaxNodes + 1];
  uint64_t flex[kMaxNodes + 1];
  uint64_t pidx[kMaxNodes + 1];
  int64_t wsel[kMaxNodes];
  int64_t latS[kMaxNodes + 1];  // max finish time over the nodes settled at depth k
  int32_t fq[kMaxNodes + 1];
  int32_t d[kMaxNodes];
  uint32_t mask[kMaxNodes];
  int32_t chunk[kMaxNodes];
  Rec bound;
  unsigned seen_seq;
  unsigned pend;  // bound is the warp's own leaf, not yet published
  unsigned pad[2];
};

__host__ __device__ constexpr size_t bnb_warp_bytes(int n) {
  return ((sizeof(BnbWarp) + 15) & ~size_t(15)) + sizeof(int64_t) * 32 * static_cast<size_t>(n) * 2;
}

size_t bnb_smem_bytes(size_t blob, int n) { return ((blob + 127) & ~size_t(127)) + bnb_warp_bytes(n) * (kBlock / 32); }

struct BnbView {
  View v;
  const int32_t* perm;
  const int32_t* nok;
  const BnbMin* bm;
  const uint64_t* rk;
  const int32_t* uns;
  const int32_t* nset;
};

__device__ __forceinline__ BnbView make_bnb_view(const uint8_t* s) {
  BnbView b;
  b.v = make_view(s);
  b.perm = reinterpret_cast<const int32_t*>(s + b.v.h->off_perm);
  b.nok = reinterpret_cast<const int32_t*>(s + b.v.h->off_nok);
  b.bm = reinterpret_cast<const BnbMin*>(s + b.v.h->off_bmin);
  b.rk = reinterpret_cast<const uint64_t*>(s + b.v.h->off_rk);
  b.uns = reinterpret_cast<const int32_t*>(s + b.v.h->off_uns);
  b.nset = reinterpret_cast<const int32_t*>(s + b.v.h->off_nsettle);
  return b;
}

// Ordering key of the first criterion of a record (larger = worse).
__device__ __forceinline__ int64_t prim_key(const BlobHeader* h, int64_t qa, int64_t qb, int64_t lat, int32_t q) {
  switch (h->crit[0]) {
    case kFpA: return qa;
    case kFpB: return qb;
    case kLat: return lat;
    default: return -static_cast<int64_t>(q);
  }
}

// 1 iff every plan whose criteria are >= (qa, qb, lat, lex) and quality <= q
// is strictly worse than b under the objective order.
__device__ __forceinline__ bool lb_worse(const BlobHeader* h, int64_t qa, int64_t qb, int64_t lat, int32_t q,
                                         uint64_t lex, const Rec& b) {
  if (!b.found) return false;
  for (int i = 0; i < h->n_crit; ++i) {
    switch (h->crit[i]) {
      case kFpA:
        if (qa != b.qa) return qa > b.qa;
        break;
      case kFpB:
        if (qb != b.qb) return qb > b.qb;
        break;
      case kLat:
        if (lat != b.lat) return lat > b.lat;
        break;
      default:
        if (q != b.qual) return q < b.qual;
        break;
    }
  }
  return lex > b.lexkey;  // identifier ranks are unique: equal only for the same plan
}

__device__ __forceinline__ Rec volatile_rec(const Rec* p) {
  const volatile Rec* v = p;
  Rec r;
  r.qa = v->qa;
  r.qb = v->qb;
  r.lat = v->lat;
  r.lexkey = v->lexkey;
  r.index = v->index;
  r.qual = v->qual;
  r.found = v->found;
  return r;
}

__device__ __forceinline__ void volatile_store(Rec* p, const Rec& r) {
  volatile Rec* v = p;
  v->qa = r.qa;
  v->qb = r.qb;
  v->lat = r.lat;
  v->lexkey = r.lexkey;
  v->index = r.index;
  v->qual = r.qual;
  v->found = r.found;
}

// Publish a plan record as the job's best if it beats the current one.
// Returns false (publish later) when another warp holds the lock.
__device__ bool bnb_try_publish(BnbSync* s, const Rec& r, const BlobHeader* h) {
  if (atomicCAS(&s->lock, 0u, 1u) != 0u) return false;
  __threadfence();
  const Rec g = volatile_rec(&s->best);
  if (rec_better(r, g, h)) {
    atomicAdd(&s->seq, 1u);
    __threadfence();
    volatile_store(&s->best, r);
    __threadfence();
    atomicAdd(&s->seq, 1u);
  }
  __threadfence();
  atomicExch(&s->lock, 0u);
  return true;
}

// Lane 0: publish the warp's own improvement if one is pending, then merge
// the job's best into the warp's bound (seqlock read).
__device__ __forceinline__ void bnb_refresh(BnbSync* s, BnbWarp& W, const BlobHeader* h) {
  if (W.pend && bnb_try_publish(s, W.bound, h)) W.pend = 0;
  const unsigned q0 = *reinterpret_cast<volatile unsigned*>(&s->seq);
  if (q0 == W.seen_seq || (q0 & 1u)) return;
  __threadfence();
  const Rec g = volatile_rec(&s->best);
  __threadfence();
  const unsigned q1 = *reinterpret_cast<volatile unsigned*>(&s->seq);
  if (q1 != q0) return;
  W.seen_seq = q0;
  if (rec_better(g, W.bound, h)) {
    W.bound = g;
    W.pend = 0;
  }
}

__global__ void __launch_bounds__(kBlock)
    bnb_kernel(const uint8_t* __restrict__ arena, const JobDesc* __restrict__ jobs, int ctas_per_job,
               Rec* __restrict__ scratch, JobSync* __restrict__ sync, BnbSync* __restrict__ bsync,
               Rec* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t mbar;
  __shared__ Rec warp_slot[kBlock / 32];
  __shared__ int am_last;

  const int job = blockIdx.x / ctas_per_job;
  // after a frontier search (bfs.cuh) of this job: done -> retire at once;
  // overflow -> continue depth first from its best plan
  const unsigned prior = __ldcg(&sync[job].pad);
  if (prior == kBnbDone) return;
  const JobDesc jd = jobs[job];
  BnbSync* bs = &bsync[job];
  load_blob(smem, arena + jd.blob_off, jd.blob_bytes, &mbar);
  const BnbView B = make_bnb_view(smem);
  const View& v = B.v;
  const BlobHeader* h = v.h;
  const int n = h->n_nodes;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ BnbSuf suf[kMaxNodes];
  if (threadIdx.x == 0) {
    double sa = 0.0, sb = 0.0, fac = 1.0;
    int32_t sq = INT_MAX;
    uint64_t sl = 0;
    for (int k = n - 1; k >= 0; --k) {  // suf[k]: nodes k+1 .. n-1
      suf[k] = BnbSuf{sa, sb, fac, sl, sq, 0};
      sa = __dadd_rd(sa, B.bm[k].a);  // (any order: a lower bound of the exact sum)
      sb = __dadd_rd(sb, B.bm[k].b);
      fac = __dmul_rd(fac, 1.0 - 0x1.0p-53);
      sq = min(sq, B.bm[k].q);
      sl += B.bm[k].lex;
    }
  }
  __syncthreads();
  uint8_t* wbase = smem + ((jd.blob_bytes + 127) & ~127u) + bnb_warp_bytes(n) * warp;
  BnbWarp& W = *reinterpret_cast<BnbWarp*>(wbase);
  int64_t* fin = reinterpret_cast<int64_t*>(wbase + ((sizeof(BnbWarp) + 15) & ~size_t(15)));  // [n][32]
  int64_t* lbk = fin + 32 * n;                                                                // [n][32]

  Rec best{0, 0, 0, 0, 0, 0, 0};  // this lane's best leaf
  if (lane == 0) {
    W.bound = best;
    W.seen_seq = 0xffffffffu;
    W.pend = 0;
    if (jd.has_seed) {
      full_eval(v, jd.seed, best);
      if (best.found) W.bound = best;
      else best.found = 0;
    }
    if (prior == kBfsOverflow) {
      const Rec r = load_rec_cg(&out[job]);
      if (rec_better(r, best, h)) best = r;
      if (rec_better(best, W.bound, h)) W.bound = best;
    }
  }
  __syncwarp();

  // tasks: prefixes of the first T nodes in exploration order, >= 8 per warp
  const uint64_t warps = static_cast<uint64_t>(ctas_per_job) * (kBlock / 32);
  int T = 0;
  uint64_t n_tasks = 1;
  bool empty = n == 0;
  for (int i = 0; i < n; ++i)
    if (B.nok[i] == 0) empty = true;
#ifdef LOOM_BNB_TASKS_PER_WARP
  const uint64_t tpw = LOOM_BNB_TASKS_PER_WARP;
#else
  const uint64_t tpw = kBnbTasksPerWarp;
#endif
  while (!empty && T < n - 1 && n_tasks < tpw * warps) n_tasks *= static_cast<uint64_t>(B.nok[T++]);
  if (empty) n_tasks = 0;
  const bool ranged = jd.begin > 0 || jd.end < h->total;
  const uint64_t budget = g_bnb_budget ? g_bnb_budget : max(h->total / 64, static_cast<uint64_t>(1) << 16);
  uint64_t work_local = 0, leaf_local = 0;
  unsigned steps = 0;
  bool aborted = false;

  // Evaluate child `slot` (exploration rank) of node k under the warp's
  // prefix: bound (k < n-1) or exact record (k == n-1).  Returns the option
  // index, or -1 when the lane has no child.
  auto eval_child = [&](int k, int slot, double& a, double& bb, int32_t& q, uint64_t& lx, int64_t& lat,
                        uint64_t& lo) -> int {
    if (slot >= B.nok[k]) return -1;
    const int c = B.perm[v.optoff[k] + slot];
    const int o = v.optoff[k] + c;
    a = __dadd_rn(W.fa[k], v.ga[o]);
    bb = __dadd_rn(W.fb[k], v.gb[o]);
    q = min(W.fq[k], v.q[o]);
    lx = W.flex[k] + v.lexw[o];
    if (k + 1 < n) {  // free nodes: bounds (see suf)
      a = __dmul_rd(__dadd_rd(a, suf[k].a), suf[k].fac);
      bb = __dmul_rd(__dadd_rd(bb, suf[k].b), suf[k].fac);
      q = min(q, suf[k].q);
      lx += suf[k].lex;
    }
    // finish times of the nodes not settled at depth k (the others are in
    // this lane's column already, and their maximum in latS[k])
    lat = W.latS[k];
    const int64_t wc = v.wall[o];
    for (int i = B.uns[k]; i < B.uns[k + 1]; ++i) {
      const int x = B.uns[i];
      int64_t st = 0;
      for (int e = v.predoff[x]; e < v.predoff[x + 1]; ++e) st = max(st, fin[v.pred[e] * 32 + lane]);
      const int64_t f = st + (x == k ? wc : W.wsel[x]);
      fin[x * 32 + lane] = f;
      lat = max(lat, f);
    }
    lo = (W.pidx[k] * static_cast<uint64_t>(v.radix[k]) + static_cast<uint64_t>(c)) * B.rk[k + 1];
    return c;
  };

  // Expand the current chunk of node k: leaves are offered, inner children
  // leave a survivor mask.
  auto expand = [&](int k) {
    if (lane == 0) bnb_refresh(bs, W, h);
    __syncwarp();
    const Rec bound = W.bound;
    const int slot = W.chunk[k] * 32 + lane;
    double a, bb;
    int32_t q;
    uint64_t lx, lo;
    int64_t lat;
    const int c = eval_child(k, slot, a, bb, q, lx, lat, lo);
    bool keep = false, improved = false;
    const bool live = c >= 0 && (!ranged || (lo < jd.end && lo + B.rk[k + 1] > jd.begin));
    if (k == n - 1) leaf_local += __popc(__ballot_sync(0xffffffffu, live));
    if (live) {
      const bool feas = lat <= h->slo_eff;
      if (k == n - 1) {
        if (feas) {
          Rec r;
          r.qa = quantize_dev(a);
          r.qb = quantize_dev(bb);
          r.lat = lat;
          r.lexkey = lx;
          r.index = lo;
          r.qual = q;
          r.found = 1;
          improved = rec_better(r, best, h);
          if (improved) best = r;
        }
      } else if (feas) {
        const int64_t qa = quantize_dev(a), qb = quantize_dev(bb);
        keep = !lb_worse(h, qa, qb, lat, q, lx, bound);
        lbk[k * 32 + lane] = h->n_crit ? prim_key(h, qa, qb, lat, q) : INT64_MIN;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) W.mask[k] = m;
    work_local += static_cast<uint64_t>(min(32, B.nok[k] - W.chunk[k] * 32));
    if (k == n - 1 && __ballot_sync(0xffffffffu, improved)) {
      // a lane whose best improved may tighten the warp's bound
      Rec r = best;
      for (int dd = 16; dd > 0; dd >>= 1) {
        const Rec o2 = shfl_rec(r, dd);
        if (rec_better(o2, r, h)) r = o2;
      }
      if (lane == 0 && rec_better(r, W.bound, h)) {
        W.bound = r;
        W.pend = 1;
      }
    }
    __syncwarp();
  };

  // Set node k's digit to the option at exploration rank `slot` (lane 0).
  // Fix node k's digit to the option at exploration rank `slot` (all lanes:
  // lane 0 writes the warp state, every lane its own column of the finish
  // times that become settled).
  auto take = [&](int k, int slot) {
    const int c = B.perm[v.optoff[k] + slot];
    const int o = v.optoff[k] + c;
    if (lane == 0) {
      W.d[k] = c;
      W.wsel[k] = v.wall[o];
      W.fa[k + 1] = __dadd_rn(W.fa[k], v.ga[o]);
      W.fb[k + 1] = __dadd_rn(W.fb[k], v.gb[o]);
      W.fq[k + 1] = min(W.fq[k], v.q[o]);
      W.flex[k + 1] = W.flex[k] + v.lexw[o];
      W.pidx[k + 1] = W.pidx[k] * static_cast<uint64_t>(v.radix[k]) + static_cast<uint64_t>(c);
    }
    __syncwarp();
    int64_t ls = W.latS[k];
    for (int i = B.nset[k]; i < B.nset[k + 1]; ++i) {
      const int x = B.nset[i];
      int64_t st = 0;
      for (int e = v.predoff[x]; e < v.predoff[x + 1]; ++e) st = max(st, fin[v.pred[e] * 32 + lane]);
      const int64_t f = st + W.wsel[x];
      fin[x * 32 + lane] = f;
      ls = max(ls, f);
    }
    if (lane == 0) W.latS[k + 1] = ls;
    __syncwarp();
  };

  // Tasks are fetched 32 at a time: lane l bounds task t0 + l (its prefix of
  // T digits decoded from the task number), and the warp runs a DFS under
  // each task that survives, lowest first.
  for (;;) {
    unsigned long long t0 = 0;
    unsigned stop = 0;
    if (lane == 0) {
      t0 = atomicAdd(&bs->next_task, 32ull);
      stop = *reinterpret_cast<volatile unsigned*>(&bs->abort);
      bnb_refresh(bs, W, h);
    }
    t0 = __shfl_sync(0xffffffffu, t0, 0);
    stop = __shfl_sync(0xffffffffu, stop, 0);
    if (t0 >= n_tasks || stop) break;
    __syncwarp();
    bool alive = t0 + lane < n_tasks;
    if (alive && T > 0) {
      // this lane's prefix: ranks from the task number, most significant first
      uint64_t r = t0 + lane;
      double a = 0.0, bb = 0.0;
      int32_t q = INT_MAX;
      uint64_t lx = 0, pidx = 0;
      for (int i = T - 1; i >= 0; --i) {
        const int c = B.perm[v.optoff[i] + static_cast<int>(r % static_cast<uint64_t>(B.nok[i]))];
        r /= static_cast<uint64_t>(B.nok[i]);
        lbk[i * 32 + lane] = c;  // scratch: no DFS is active in this warp
      }
      for (int i = 0; i < T; ++i) {
        const int c = static_cast<int>(lbk[i * 32 + lane]);
        const int o = v.optoff[i] + c;
        a = __dadd_rn(a, v.ga[o]);
        bb = __dadd_rn(bb, v.gb[o]);
        q = min(q, v.q[o]);
        lx += v.lexw[o];
        pidx = pidx * static_cast<uint64_t>(v.radix[i]) + static_cast<uint64_t>(c);
      }
      if (T < n) {
        a = __dmul_rd(__dadd_rd(a, suf[T - 1].a), suf[T - 1].fac);
        bb = __dmul_rd(__dadd_rd(bb, suf[T - 1].b), suf[T - 1].fac);
        q = min(q, suf[T - 1].q);
        lx += suf[T - 1].lex;
      }
      int64_t lat = 0;
      for (int tt = 0; tt < n; ++tt) {
        const int x = v.topo[tt];
        int64_t st = 0;
        for (int e = v.predoff[x]; e < v.predoff[x + 1]; ++e) st = max(st, fin[v.pred[e] * 32 + lane]);
        const int64_t f = st + (x < T ? v.wall[v.optoff[x] + static_cast<int>(lbk[x * 32 + lane])] : B.bm[x].w);
        fin[x * 32 + lane] = f;
        lat = max(lat, f);
      }
      const uint64_t lo = pidx * B.rk[T];
      if (ranged && !(lo < jd.end && lo + B.rk[T] > jd.begin)) alive = false;
      else if (lat > h->slo_eff) alive = false;
      else if (lb_worse(h, quantize_dev(a), quantize_dev(bb), lat, q, lx, W.bound)) alive = false;
    }
    work_local += n_tasks - t0 < 32 ? n_tasks - t0 : 32;
    unsigned roots = __ballot_sync(0xffffffffu, alive);
    __syncwarp();
    while (roots) {
    const int rb = __ffs(roots) - 1;
    roots &= roots - 1;
    if (lane == 0) {
      W.fa[0] = 0.0;
      W.fb[0] = 0.0;
      W.fq[0] = INT_MAX;
      W.flex[0] = 0;
      W.pidx[0] = 0;
      W.latS[0] = 0;
      for (int x = 0; x < n; ++x) W.wsel[x] = B.bm[x].w;
    }
    __syncwarp();
    {
      uint64_t r = t0 + static_cast<uint64_t>(rb);
      uint64_t div = 1;
      for (int i = 0; i < T; ++i) div *= static_cast<uint64_t>(B.nok[i]);
      for (int i = 0; i < T; ++i) {  // ranks, most significant first
        div /= static_cast<uint64_t>(B.nok[i]);
        take(i, static_cast<int>((r / div) % static_cast<uint64_t>(B.nok[i])));
      }
    }
    unsigned task_steps = 0;
    if (lane == 0) atomicAdd(&g_bnb_acc[1], 1ull);
    int depth = T;
    if (lane == 0) W.chunk[depth] = 0;
    __syncwarp();
    expand(depth);
    for (;;) {
      if (++steps % 64 == 0) {
        unsigned ab = 0;
        if (lane == 0) {
          const unsigned long long tot = atomicAdd(&bs->work, work_local) + work_local;
          work_local = 0;
          if (tot > budget) atomicExch(&bs->abort, 1u);
          ab = *reinterpret_cast<volatile unsigned*>(&bs->abort);
        }
        if (__shfl_sync(0xffffffffu, ab, 0)) {
          aborted = true;
          break;
        }
      }
      ++task_steps;
      const uint32_t m = W.mask[depth];
      if (m == 0) {
        if ((W.chunk[depth] + 1) * 32 < B.nok[depth]) {
          if (lane == 0) ++W.chunk[depth];
          __syncwarp();
          expand(depth);
          continue;
        }
        if (depth == T) break;
        if (lane == 0) W.wsel[depth] = B.bm[depth].w;  // node `depth` is free again
        __syncwarp();
        --depth;
        continue;
      }
      const int b = __ffs(m) - 1;
      const int slot = W.chunk[depth] * 32 + b;
      // re-check the child's primary bound against the bound as it is now
      bool skip = false;
      if (h->n_crit) {
        const Rec& bd = W.bound;
        skip = bd.found && lbk[depth * 32 + b] > prim_key(h, bd.qa, bd.qb, bd.lat, bd.qual);
      }
      __syncwarp();
      if (lane == 0) W.mask[depth] = m & ~(1u << b);
      if (skip) {
        __syncwarp();
        continue;
      }
      take(depth, slot);
      if (lane == 0) W.chunk[depth + 1] = 0;
      __syncwarp();
      ++depth;
      expand(depth);
    }
    if (lane == 0) {
      for (int x = 0; x < n; ++x) W.wsel[x] = B.bm[x].w;
      atomicMax(&g_bnb_acc[0], static_cast<unsigned long long>(task_steps));
    }
    __syncwarp();
    if (aborted) break;
    }  // roots
  }
  if (lane == 0 && work_local) atomicAdd(&bs->work, work_local);
  if (lane == 0 && leaf_local) atomicAdd(&bs->leaves, leaf_local);

  // lane bests -> CTA -> job (last CTA to arrive)
  Rec b = block_best(best, h, warp_slot);
  const int part = blockIdx.x % ctas_per_job;
  if (threadIdx.x == 0) {
    scratch[blockIdx.x] = b;
    __threadfence();
    const unsigned tk = atomicAdd(&bs->ticket, 1u);
    am_last = (tk == static_cast<unsigned>(ctas_per_job - 1));
  }
  (void)part;
  __syncthreads();
  if (am_last) {
    __threadfence();
    Rec acc{0, 0, 0, 0, 0, 0, 0};
    for (int i = threadIdx.x; i < ctas_per_job; i += kBlock) {
      const Rec o = load_rec_cg(&scratch[static_cast<size_t>(job) * ctas_per_job + i]);
      if (rec_better(o, acc, h)) acc = o;
    }
    acc = block_best(acc, h, warp_slot);
    if (threadIdx.x == 0) {
      out[job] = acc;
      sync[job].pad = bs->abort ? kBnbAborted : kBnbDone;
      if (job == 0) {
        g_bnb_last[0] = bs->work;
        g_bnb_last[1] = bs->abort;
        g_bnb_last[2] = g_bnb_acc[0];
        g_bnb_last[3] = g_bnb_acc[1];
        g_bnb_last[4] = bs->leaves;
        g_bnb_acc[0] = 0;
        g_bnb_acc[1] = 0;
      }
      bs->lock = 0;
      bs->seq = 0;
      bs->ticket = 0;
      bs->abort = 0;
      bs->next_task = 0;
      bs->work = 0;
      bs->leaves = 0;
      bs->best = Rec{0, 0, 0, 0, 0, 0, 0};
    }
  }
}

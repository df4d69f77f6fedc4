// Frontier branch and bound: the default search (included by loom_search.cu
// inside its anonymous namespace, after bnb.cuh).
//
// Same contract and the same exact subtree bounds as bnb.cuh -- a subtree of
// the ConfigEnumerator tree (optimizer.hpp:131-143; node 0 most significant)
// is dropped when the lower bound of its plans' criteria is infeasible or
// lexicographically STRICTLY worse than a real plan already found, so the
// argmin of objective_less (estimator.hpp:93-116) over the range is never
// dropped -- but explored level by level across the whole GPU instead of
// depth first per warp:
//
//   depth d -> d+1   every surviving prefix of d digits x every option of
//                    node d that passes the quality floor is one child; all
//                    children of a level are evaluated at once (a team of
//                    lanes per prefix, one child per lane), and the survivors
//                    are appended to the next frontier with one atomic per warp.
//   completions      a surviving child also names two real plans: its free
//                    nodes at the option that is best on the primary
//                    criterion (the order bnb.cuh explores first), and at the
//                    smallest wall (feasible whenever the child's latency bound
//                    is, because that plan's latency IS the bound).  Both are
//                    evaluated exactly and offered as incumbents, so pruning
//                    tightens from the first levels on instead of waiting for
//                    leaves.  For an energy-first objective, a child whose
//                    energy-best completion meets the SLO has found its
//                    subtree's energy bucket at once.
//   leaves           depth n: exact records, offered.
//   incumbent        per level: thread bests -> CTA best -> the job's best
//                    (a lock, taken only by a CTA that improves on it); after
//                    the level's grid barrier every CTA prunes the next level
//                    against it.  The order is strict and total, so the
//                    result does not depend on timing or on the grid.
//
// One cooperative launch (all CTAs resident) runs every level; a grid barrier
// separates levels.  The problem image is copied to shared memory once (TMA
// bulk copy); frontiers live in HBM (32-byte FrontierEntry, double-buffered).
// A frontier that outgrows its buffer sets `overflow`: the job's best so far
// goes to out[job], JobSync.pad = kBfsOverflow, and the depth-first kernel
// (bnb.cuh) that follows on the stream takes over from that incumbent (then
// the sweep, if it too runs out of budget).  Otherwise JobSync.pad =
// kBnbDone and both follow-up launches retire at once.

__device__ unsigned long long g_bfs_last[6];  // evidence of the last frontier launch

struct BfsShared {
  Rec best;          // the job's incumbent as of the last barrier
  Rec warp_slot[kBlock / 32];
  uint64_t mbar;
  int32_t shift[kMaxNodes + 1];
  int32_t o_prim[kMaxNodes];  // completion option: best on the primary criterion
  BnbSuf suf[kMaxNodes + 1];  // bounds over the free nodes k .. n-1 (suf[n]: none)
  int32_t stop;
};

__device__ __forceinline__ void grid_barrier(BfsSync* bs, unsigned n_ctas) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = &bs->bar_gen;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(&bs->bar_count, 1u) == n_ctas - 1) {
      bs->bar_count = 0;
      __threadfence();
      atomicAdd(&bs->bar_gen, 1u);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ Rec volatile_rec_b(const Rec* p) {
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

__device__ __forceinline__ int bfs_digit(const BfsShared& S, uint64_t dig, int i) {
  return static_cast<int>((dig >> S.shift[i]) & ((1ull << (S.shift[i + 1] - S.shift[i])) - 1));
}

// Criteria of a plan against a record: -1 better, 1 worse, 0 equal on every
// criterion (the identifier decides).
__device__ __forceinline__ int crit_cmp(const BlobHeader* h, int64_t qa, int64_t qb, int64_t lat, int32_t q,
                                        const Rec& b) {
  if (!b.found) return -1;
  for (int i = 0; i < h->n_crit; ++i) {
    switch (h->crit[i]) {
      case kFpA:
        if (qa != b.qa) return qa < b.qa ? -1 : 1;
        break;
      case kFpB:
        if (qb != b.qb) return qb < b.qb ? -1 : 1;
        break;
      case kLat:
        if (lat != b.lat) return lat < b.lat ? -1 : 1;
        break;
      default:
        if (q != b.qual) return q > b.qual ? -1 : 1;
        break;
    }
  }
  return 0;
}

// Offer the plan named by packed digits (nodes < k) and, for nodes >= k,
// option free_opt[i] (free_is_wall: BnbMin.o_wall) to `best`.  a, b, q: the
// exact folds over nodes < k.  lat_known >= 0: the plan's latency is already
// known (the min-wall completion's latency IS the child's bound); otherwise
// the finish-time recursion (estimator.hpp:69-76) runs over this thread's
// column of `fin`.  The identifier rank and plan index are only built when
// the plan ties or beats `best` on the criteria.
__device__ __forceinline__ void bfs_offer(const BnbView& B, const BfsShared& S, const JobDesc& jd, bool ranged,
                                          uint64_t dig, int k, double a, double b, int32_t q, bool free_is_wall,
                                          int64_t lat_known, int64_t* fin, Rec& best) {
  const View& v = B.v;
  const BlobHeader* h = v.h;
  const int n = h->n_nodes;
  for (int i = k; i < n; ++i) {  // the folds continue in dag.nodes order (estimator.hpp:50-60)
    const int o = v.optoff[i] + (free_is_wall ? B.bm[i].o_wall : S.o_prim[i]);
    a = __dadd_rn(a, v.ga[o]);
    b = __dadd_rn(b, v.gb[o]);
    q = min(q, v.q[o]);
  }
  int64_t lat = lat_known;
  if (lat < 0) {
    for (int i = 0; i < n; ++i) {
      const int c = i < k ? bfs_digit(S, dig, i) : (free_is_wall ? B.bm[i].o_wall : S.o_prim[i]);
      fin[i * kBlock] = v.wall[v.optoff[i] + c];
    }
    lat = 0;
    for (int t = 0; t < n; ++t) {
      const int x = v.topo[t];
      int64_t st = 0;
      for (int e = v.predoff[x]; e < v.predoff[x + 1]; ++e) st = max(st, fin[v.pred[e] * kBlock]);
      const int64_t f = st + fin[x * kBlock];
      fin[x * kBlock] = f;
      lat = max(lat, f);
    }
  }
  if (lat > h->slo_eff) return;
  const int64_t qa = quantize_dev(a), qb = quantize_dev(b);
  const int cmp = crit_cmp(h, qa, qb, lat, q, best);
  if (cmp > 0) return;
  uint64_t lex = 0, idx = 0;
  for (int i = 0; i < n; ++i) {
    const int c = i < k ? bfs_digit(S, dig, i) : (free_is_wall ? B.bm[i].o_wall : S.o_prim[i]);
    lex += v.lexw[v.optoff[i] + c];
    idx = idx * static_cast<uint64_t>(v.radix[i]) + static_cast<uint64_t>(c);
  }
  if (cmp == 0 && lex >= best.lexkey) return;
  if (ranged && (idx < jd.begin || idx >= jd.end)) return;
  best = Rec{qa, qb, lat, lex, idx, q, 1};
}

__global__ void __launch_bounds__(kBlock)
    bfs_kernel(const uint8_t* __restrict__ arena, const JobDesc* __restrict__ jobs, BfsSync* __restrict__ bs,
               FrontierEntry* __restrict__ buf0, FrontierEntry* __restrict__ buf1, uint64_t cap,
               JobSync* __restrict__ sync, Rec* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ BfsShared S;
  const JobDesc jd = jobs[0];
  load_blob(smem, arena + jd.blob_off, jd.blob_bytes, &S.mbar);
  const BnbView B = make_bnb_view(smem);
  const View& v = B.v;
  const BlobHeader* h = v.h;
  const int n = h->n_nodes;
  const int lane = threadIdx.x & 31;
  int64_t* fin = reinterpret_cast<int64_t*>(smem + ((jd.blob_bytes + 127) & ~127u)) + threadIdx.x;  // [n][kBlock]
  if (threadIdx.x == 0) {
    int s = 0;
    for (int i = 0; i < n; ++i) {
      S.shift[i] = s;
      s += 32 - __clz(max(1, v.radix[i] - 1));
      S.o_prim[i] = B.perm[v.optoff[i]];
    }
    S.shift[n] = s;
    // suf[k]: nodes k .. n-1 (see BnbSuf, bnb.cuh)
    double sa = 0.0, sb = 0.0, fac = 1.0;
    int32_t sq = INT_MAX;
    uint64_t sl = 0;
    for (int k = n; k >= 0; --k) {
      if (k < n) {
        sa = __dadd_rd(sa, B.bm[k].a);
        sb = __dadd_rd(sb, B.bm[k].b);
        fac = __dmul_rd(fac, 1.0 - 0x1.0p-53);
        sq = min(sq, B.bm[k].q);
        sl += B.bm[k].lex;
      }
      S.suf[k] = BnbSuf{sa, sb, fac, sl, sq, 0};
    }
    S.stop = 0;
    S.best = Rec{0, 0, 0, 0, 0, 0, 0};
  }
  __syncthreads();

  const bool ranged = jd.begin > 0 || jd.end < h->total;

  // thread best: the seed (a plan of the space, or of the range) if any
  Rec best{0, 0, 0, 0, 0, 0, 0};
  if (jd.has_seed && blockIdx.x == 0 && threadIdx.x == 0) full_eval(v, jd.seed, best);
  bool empty = n == 0;
  for (int i = 0; i < n; ++i) empty |= B.nok[i] == 0;

  uint64_t evals = 0, leaves = 0;
  const uint64_t gthreads = static_cast<uint64_t>(gridDim.x) * kBlock;
  const uint64_t gtid = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
  FrontierEntry* cur = buf0;
  FrontierEntry* nxt = buf1;
  uint64_t n_cur = 1;  // depth 0: the root (no digit fixed)
  bool overflow = false;

  for (int d = 0; d < n && !empty; ++d) {
    const int nk = B.nok[d];
    // team of T lanes per parent: T = nok rounded up to a power of two, <= 32
    const int T = nk >= 32 ? 32 : (1 << (32 - __clz(max(1, nk - 1))));
    const int slot0 = lane & (T - 1);
    const uint64_t team = gtid / static_cast<uint64_t>(T);
    const uint64_t n_teams = gthreads / static_cast<uint64_t>(T);
    const int k = d + 1;  // digits fixed in a child
    const bool leaf = k == n;
    const Rec bound = S.best;
    const int64_t bkey = bound.found && h->n_crit ? prim_key(h, bound.qa, bound.qb, bound.lat, bound.qual) : INT64_MAX;
    const BnbSuf suf = S.suf[k];
    // uniform trip count across the warp (the ballots below need every lane)
    const uint64_t rounds = (n_cur + n_teams - 1) / n_teams;
    for (uint64_t it = 0; it < rounds; ++it) {
      const uint64_t pi = team + it * n_teams;
      FrontierEntry par{0, 0.0, 0.0, INT64_MIN, INT_MAX, {0, 0, 0}};
      if (pi < n_cur && d > 0) par = cur[pi];
      // a prefix whose first-criterion bound is now worse than the incumbent
      // (found at its own level, after it was kept) is not expanded
      const bool alive = pi < n_cur && par.key <= bkey;
      for (int s0 = 0; s0 < nk; s0 += T) {
        const int slot = s0 + slot0;
        bool keep = false;
        FrontierEntry ch{};
        if (alive && slot < nk) {
          const int c = B.perm[v.optoff[d] + slot];
          const int o = v.optoff[d] + c;
          ch.dig = par.dig | (static_cast<uint64_t>(c) << S.shift[d]);
          ch.fa = __dadd_rn(par.fa, v.ga[o]);
          ch.fb = __dadd_rn(par.fb, v.gb[o]);
          ch.q = min(par.q, v.q[o]);
          ++evals;
          if (leaf) {
            ++leaves;
            bfs_offer(B, S, jd, ranged, ch.dig, k, ch.fa, ch.fb, ch.q, false, -1, fin, best);
          } else {
            // subtree bound: walls fixed for nodes < k, smallest walls below
            uint64_t pidx = 0, lx = 0;
            for (int i = 0; i < n; ++i) {
              int64_t w;
              if (i < k) {
                const int ci = bfs_digit(S, ch.dig, i);
                const int oi = v.optoff[i] + ci;
                w = v.wall[oi];
                lx += v.lexw[oi];
                pidx = pidx * static_cast<uint64_t>(v.radix[i]) + static_cast<uint64_t>(ci);
              } else {
                w = B.bm[i].w;
              }
              fin[i * kBlock] = w;
            }
            int64_t lat = 0;
            for (int t = 0; t < n; ++t) {
              const int x = v.topo[t];
              int64_t st = 0;
              for (int e = v.predoff[x]; e < v.predoff[x + 1]; ++e) st = max(st, fin[v.pred[e] * kBlock]);
              const int64_t f = st + fin[x * kBlock];
              fin[x * kBlock] = f;
              lat = max(lat, f);
            }
            const uint64_t lo = pidx * B.rk[k];
            if (lat <= h->slo_eff && (!ranged || (lo < jd.end && lo + B.rk[k] > jd.begin))) {
              const int64_t qa = quantize_dev(__dmul_rd(__dadd_rd(ch.fa, suf.a), suf.fac));
              const int64_t qb = quantize_dev(__dmul_rd(__dadd_rd(ch.fb, suf.b), suf.fac));
              const int32_t qu = min(ch.q, suf.q);
              keep = !lb_worse(h, qa, qb, lat, qu, lx + suf.lex, bound);
              if (keep) {
                ch.key = h->n_crit ? prim_key(h, qa, qb, lat, qu) : INT64_MIN;
                // two real plans of the subtree as incumbents: free nodes at
                // their best primary option, and at their smallest walls
                // (whose latency is the bound just computed)
                bfs_offer(B, S, jd, ranged, ch.dig, k, ch.fa, ch.fb, ch.q, false, -1, fin, best);
                bfs_offer(B, S, jd, ranged, ch.dig, k, ch.fa, ch.fb, ch.q, true, lat, fin, best);
              }
            }
          }
        }
        if (!leaf) {
          // append survivors: one atomic per warp
          const unsigned m = __ballot_sync(0xffffffffu, keep);
          if (m) {
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(&bs->count[k], static_cast<unsigned long long>(__popc(m)));
            base = __shfl_sync(0xffffffffu, base, 0);
            const uint64_t at = base + __popc(m & ((1u << lane) - 1));
            if (keep) {
              if (at < cap) nxt[at] = ch;
              else overflow = true;
            }
          }
        }
      }
    }
    // level end: CTA best -> job best; then everyone sees it
    const Rec cb = block_best(best, h, S.warp_slot);
    if (threadIdx.x == 0 && cb.found) {
      const Rec g = volatile_rec_b(&bs->best);
      if (rec_better(cb, g, h)) {
        while (atomicCAS(&bs->lock, 0u, 1u) != 0u) __nanosleep(32);
        __threadfence();
        const Rec g2 = volatile_rec_b(&bs->best);
        if (rec_better(cb, g2, h)) {
          volatile Rec* w = &bs->best;
          w->qa = cb.qa;
          w->qb = cb.qb;
          w->lat = cb.lat;
          w->lexkey = cb.lexkey;
          w->index = cb.index;
          w->qual = cb.qual;
          w->found = cb.found;
        }
        __threadfence();
        atomicExch(&bs->lock, 0u);
      }
    }
    if (__syncthreads_or(overflow) && threadIdx.x == 0) atomicExch(&bs->overflow, 1u);
    grid_barrier(bs, gridDim.x);
    if (threadIdx.x == 0) {
      S.best = volatile_rec_b(&bs->best);
      S.stop = *reinterpret_cast<volatile unsigned*>(&bs->overflow) != 0u;
    }
    __syncthreads();
    if (S.stop || leaf) break;
    n_cur = __ldcg(&bs->count[k]);
    if (n_cur == 0) break;
    FrontierEntry* t = cur;
    cur = nxt;
    nxt = t;
  }

  // evidence, result, reset (the last CTA to arrive)
  if (evals) atomicAdd(&bs->evals, evals);
  if (leaves) atomicAdd(&bs->leaves, leaves);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long mf = 0;
    for (int i = 1; i <= n; ++i) mf = max(mf, __ldcg(&bs->count[i]));
    atomicMax(&bs->max_frontier, mf);
  }
  grid_barrier(bs, gridDim.x);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const bool of = bs->overflow != 0u;
    out[0] = volatile_rec_b(&bs->best);
    sync[0].pad = of ? kBfsOverflow : kBnbDone;
    g_bfs_last[0] = bs->evals;
    g_bfs_last[1] = of;
    g_bfs_last[2] = bs->max_frontier;
    g_bfs_last[3] = gridDim.x;
    g_bfs_last[4] = bs->leaves;
    for (int i = 0; i <= kMaxNodes; ++i) bs->count[i] = 0;
    bs->lock = 0;
    bs->overflow = 0;
    bs->evals = 0;
    bs->leaves = 0;
    bs->max_frontier = 0;
    bs->best = Rec{0, 0, 0, 0, 0, 0, 0};
    // bar_count is 0 again after the barrier; bar_gen keeps counting
  }
}

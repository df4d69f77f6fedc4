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
// Per-level trace of the last launch (CTA 0): [0] start, [1] end, [2d+2] =
// %globaltimer at the end of depth d's level, [2d+3] = parents expanded |
// redundant << 63 (loom_bfs_trace).
__device__ unsigned long long g_bfs_trace[2 * (kMaxNodes + 2)];

__device__ __forceinline__ unsigned long long bfs_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#ifndef LOOM_BFS_BLOCK
#define LOOM_BFS_BLOCK 512
#endif
constexpr int kBfsBlock = LOOM_BFS_BLOCK;  // one CTA per SM: fewer arrivals per grid barrier
#ifndef LOOM_BFS_GRAB
#define LOOM_BFS_GRAB 2  // team rounds per dynamic grab
#endif

struct BfsShared {
  Rec best;  // the incumbent: identical in every CTA after every level
  Rec warp_slot[kBfsBlock / 32];
  uint64_t mbar;
  int32_t shift[kMaxNodes + 1];
  int32_t o_prim[kMaxNodes];  // completion option: best on the primary criterion
  BnbSuf suf[kMaxNodes + 1];  // bounds over the free nodes k .. n-1 (suf[n]: none)
  int32_t stop;
};

// Grid barrier of the cooperative launch (all CTAs resident): one arrival per
// CTA with release semantics, the last arriver resets the count and bumps
// the generation (release), the others poll it (acquire).
__device__ __forceinline__ void grid_barrier(BfsSync* bs, unsigned n_ctas) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* gen = &bs->bar_gen;
    unsigned* cnt = &bs->bar_count;
    unsigned g, old;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
    if (old == n_ctas - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(cnt) : "memory");
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g + 1) : "memory");
    } else {
      unsigned cur;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(gen) : "memory");
        if (cur != g) break;
        __nanosleep(20);
      }
    }
  }
  __syncthreads();
}

// Block-wide min-loc under the objective order (kBfsBlock threads); result in thread 0.
__device__ Rec bfs_block_best(Rec r, const BlobHeader* h, Rec* warp_slot) {
  for (int d = 16; d > 0; d >>= 1) {
    const Rec o = shfl_rec(r, d);
    if (rec_better(o, r, h)) r = o;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) warp_slot[warp] = r;
  __syncthreads();
  if (warp == 0) {
    r = lane < kBfsBlock / 32 ? warp_slot[lane] : Rec{0, 0, 0, 0, 0, 0, 0};
    for (int d = 16; d > 0; d >>= 1) {
      const Rec o = shfl_rec(r, d);
      if (rec_better(o, r, h)) r = o;
    }
  }
  __syncthreads();
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
      fin[i * kBfsBlock] = v.wall[v.optoff[i] + c];
    }
    lat = 0;
    for (int t = 0; t < n; ++t) {
      const int x = v.topo[t];
      int64_t st = 0;
      for (int e = v.predoff[x]; e < v.predoff[x + 1]; ++e) st = max(st, fin[v.pred[e] * kBfsBlock]);
      const int64_t f = st + fin[x * kBfsBlock];
      fin[x * kBfsBlock] = f;
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

// Wall of node i under a prefix of k digits: its chosen option's when fixed,
// its smallest otherwise.
__device__ __forceinline__ int64_t bfs_wall(const BnbView& B, const BfsShared& S, uint64_t dig, int k, int i) {
  return i < k ? B.v.wall[B.v.optoff[i] + bfs_digit(S, dig, i)] : B.bm[i].w;
}

// Latency terms of node x under a prefix of k digits (FrontierEntry): the
// longest path avoiding x, the latest finish among x's predecessors, and the
// longest path from x's successors to the end (estimator.hpp:69-76's
// recursion, other free nodes at their smallest walls).
__device__ __forceinline__ void bfs_terms(const BnbView& B, const BfsShared& S, uint64_t dig, int k, int x,
                                          int64_t* fin, int64_t& lnot, int64_t& head, int64_t& tail) {
  const View& v = B.v;
  const int n = v.h->n_nodes;
  constexpr int64_t kGone = -(int64_t(1) << 62);  // x removed: paths through it never win a max
  lnot = 0;
  head = 0;
  int px = 0;
  for (int t = 0; t < n; ++t) {
    const int y = v.topo[t];
    int64_t st = 0;
    for (int e = v.predoff[y]; e < v.predoff[y + 1]; ++e) st = max(st, fin[v.pred[e] * kBfsBlock]);
    if (y == x) {
      head = st;
      px = t;
      fin[y * kBfsBlock] = kGone;
    } else {
      const int64_t f = st + bfs_wall(B, S, dig, k, y);
      fin[y * kBfsBlock] = f;
      lnot = max(lnot, f);
    }
  }
  // successors of x come after it in topological order: longest path from
  // each node to the end, accumulated into its predecessors, down to x
  for (int i = 0; i < n; ++i) fin[i * kBfsBlock] = 0;
  for (int t = n - 1; t > px; --t) {
    const int y = v.topo[t];
    const int64_t b = fin[y * kBfsBlock] + bfs_wall(B, S, dig, k, y);
    for (int e = v.predoff[y]; e < v.predoff[y + 1]; ++e) {
      const int p = v.pred[e];
      fin[p * kBfsBlock] = max(fin[p * kBfsBlock], b);
    }
  }
  tail = fin[x * kBfsBlock];
}

// Child `slot` (exploration rank) of prefix `par` at depth d: its bound, and
// -- if the subtree survives -- its latency terms for the next level and its
// two completions offered to `cand`.  Leaves (k == n) are offered exactly.
// Returns whether the child is kept.
__device__ __forceinline__ bool bfs_child(const BnbView& B, const BfsShared& S, const JobDesc& jd, bool ranged,
                                          const FrontierEntry& par, int d, int slot, const Rec& bound,
                                          const BnbSuf& suf, int64_t* fin, FrontierEntry& ch, Rec& cand) {
  const View& v = B.v;
  const BlobHeader* h = v.h;
  const int n = h->n_nodes;
  const int k = d + 1;
  const int c = B.perm[v.optoff[d] + slot];
  const int o = v.optoff[d] + c;
  ch.dig = par.dig | (static_cast<uint64_t>(c) << S.shift[d]);
  ch.fa = __dadd_rn(par.fa, v.ga[o]);
  ch.fb = __dadd_rn(par.fb, v.gb[o]);
  ch.q = min(par.q, v.q[o]);
  // the child's latency bound (exact for a leaf) from the parent's terms of node d
  const int64_t lat = max(par.lnot, par.head + v.wall[o] + par.tail);
  if (k == n) {
    bfs_offer(B, S, jd, ranged, ch.dig, k, ch.fa, ch.fb, ch.q, false, lat, fin, cand);
    return false;
  }
  if (lat > h->slo_eff) return false;
  if (ranged) {
    uint64_t pidx = 0;
    for (int i = 0; i < k; ++i) pidx = pidx * static_cast<uint64_t>(v.radix[i]) + bfs_digit(S, ch.dig, i);
    const uint64_t lo = pidx * B.rk[k];
    if (!(lo < jd.end && lo + B.rk[k] > jd.begin)) return false;
  }
  // FP bounds: the fold of the prefix continued with the free nodes' minima,
  // rounded down (BnbSuf, bnb.cuh)
  const int64_t qa = quantize_dev(__dmul_rd(__dadd_rd(ch.fa, suf.a), suf.fac));
  const int64_t qb = quantize_dev(__dmul_rd(__dadd_rd(ch.fb, suf.b), suf.fac));
  const int32_t qu = min(ch.q, suf.q);
  const int cmp = crit_cmp(h, qa, qb, lat, qu, bound);
  if (cmp > 0) return false;
  if (cmp == 0) {  // every criterion ties the incumbent: the identifier decides
    uint64_t lx = suf.lex;
    for (int i = 0; i < k; ++i) lx += v.lexw[v.optoff[i] + bfs_digit(S, ch.dig, i)];
    if (lx > bound.lexkey) return false;
  }
  ch.key = h->n_crit ? prim_key(h, qa, qb, lat, qu) : INT64_MIN;
  bfs_terms(B, S, ch.dig, k, k, fin, ch.lnot, ch.head, ch.tail);
  // two real plans of the subtree as incumbents: free nodes at their best
  // primary option, and at their smallest walls (whose latency is `lat`)
  bfs_offer(B, S, jd, ranged, ch.dig, k, ch.fa, ch.fb, ch.q, false, -1, fin, cand);
  bfs_offer(B, S, jd, ranged, ch.dig, k, ch.fa, ch.fb, ch.q, true, lat, fin, cand);
  return true;
}

// Block exclusive prefix of `keep` (kBfsBlock threads); returns this thread's
// position, total in *n_out.
__device__ __forceinline__ unsigned bfs_block_scan(bool keep, unsigned* warp_cnt, unsigned* n_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned m = __ballot_sync(0xffffffffu, keep);
  if (lane == 0) warp_cnt[warp] = __popc(m);
  __syncthreads();
  unsigned before = 0, total = 0;
  for (int w = 0; w < kBfsBlock / 32; ++w) {
    const unsigned c = warp_cnt[w];
    before += w < warp ? c : 0;
    total += c;
  }
  __syncthreads();
  *n_out = total;
  return before + __popc(m & ((1u << lane) - 1));
}

__global__ void __launch_bounds__(kBfsBlock, 1)
    bfs_kernel(const uint8_t* __restrict__ arena, const JobDesc* __restrict__ jobs, BfsSync* __restrict__ bs,
               FrontierEntry* __restrict__ buf0, FrontierEntry* __restrict__ buf1, uint64_t cap,
               Rec* __restrict__ slots, JobSync* __restrict__ sync, Rec* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ BfsShared S;
  __shared__ unsigned warp_cnt[kBfsBlock / 32];
  const JobDesc jd = jobs[0];
  load_blob(smem, arena + jd.blob_off, jd.blob_bytes, &S.mbar);
  const BnbView B = make_bnb_view(smem);
  const View& v = B.v;
  const BlobHeader* h = v.h;
  const int n = h->n_nodes;
  const int lane = threadIdx.x & 31;
  int64_t* fin = reinterpret_cast<int64_t*>(smem + ((jd.blob_bytes + 127) & ~127u)) + threadIdx.x;  // [n][kBfsBlock]
  // frontiers of the small (redundant) levels, after the finish-time columns
  auto sfront = reinterpret_cast<FrontierEntry(*)[kBfsBlock]>(
      smem + ((jd.blob_bytes + 127) & ~127u) + sizeof(int64_t) * kBfsBlock * n);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    g_bfs_trace[0] = bfs_now();
    for (int i = 1; i < 2 * (kMaxNodes + 2); ++i) g_bfs_trace[i] = 0;
  }
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
    // the incumbent: the seed (a plan of the space, or of the range) if any
    Rec r{0, 0, 0, 0, 0, 0, 0};
    if (jd.has_seed) full_eval(v, jd.seed, r);
    S.best = r;
    S.stop = 0;
    FrontierEntry root{0, 0.0, 0.0, INT64_MIN, 0, 0, 0, INT_MAX, 0};  // the root: no digit fixed
    if (n > 0) bfs_terms(B, S, 0, 0, 0, fin, root.lnot, root.head, root.tail);
    sfront[0][0] = root;
  }
  __syncthreads();

  const bool ranged = jd.begin > 0 || jd.end < h->total;
  bool empty = n == 0;
  for (int i = 0; i < n; ++i) empty |= B.nok[i] == 0;

  // The incumbent S.best is identical in every CTA after every level: a
  // small level is evaluated redundantly by every CTA (same parents, same
  // children, same reduction, no communication); a large level is split
  // across CTAs and its per-CTA bests are exchanged through `slots` and one
  // grid barrier, then every CTA reduces the same slots.
  uint64_t evals = 0, leaves = 0;
  FrontierEntry* cur = buf0;
  FrontierEntry* nxt = buf1;
  uint64_t n_cur = 1;  // parents at depth d
  int src = 0;         // where they are: 0/1 = sfront[src], 2 = global `cur`
  for (int d = 0; d < n && !empty && n_cur; ++d) {
    if (blockIdx.x == 0 && threadIdx.x == 0) g_bfs_trace[2 * d + 3] = n_cur;
    const int nk = B.nok[d];
    const int k = d + 1;
    const bool leaf = k == n;
    const Rec bound = S.best;
    const int64_t bkey = bound.found && h->n_crit ? prim_key(h, bound.qa, bound.qb, bound.lat, bound.qual) : INT64_MAX;
    const BnbSuf suf = S.suf[k];
    Rec cand{0, 0, 0, 0, 0, 0, 0};
    const bool redundant = n_cur * static_cast<uint64_t>(nk) <= static_cast<uint64_t>(kBfsBlock);
    if (redundant) {
      // every CTA: child t = (parent t / nk, slot t % nk)
      const int t = threadIdx.x;
      const int pi = t / nk, slot = t - pi * nk;
      bool keep = false;
      FrontierEntry ch{};
      if (static_cast<uint64_t>(pi) < n_cur) {
        const FrontierEntry par = src == 2 ? cur[pi] : sfront[src][pi];
        if (par.key <= bkey) {
          if (blockIdx.x == 0) {
            ++evals;
            leaves += leaf;
          }
          keep = bfs_child(B, S, jd, ranged, par, d, slot, bound, suf, fin, ch, cand);
        }
      }
      unsigned total = 0;
      const unsigned at = bfs_block_scan(keep, warp_cnt, &total);
      const int dst = src == 0 ? 1 : 0;
      if (keep) sfront[dst][at] = ch;
      const Rec cb = bfs_block_best(cand, h, S.warp_slot);
      if (threadIdx.x == 0 && rec_better(cb, S.best, h)) S.best = cb;
      __syncthreads();
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        g_bfs_trace[2 * d + 2] = bfs_now();
        g_bfs_trace[2 * d + 3] |= 1ull << 63;
      }
      n_cur = total;
      src = dst;
      continue;
    }
    // distributed: parents dealt to warps dynamically, LOOM_BFS_GRAB team
    // rounds per grab (the cost of a parent varies: kept children pay for
    // their terms and completions); a team of T lanes per parent, T = nok
    // rounded up to a power of two (<= 32)
    const int T = nk >= 32 ? 32 : (1 << (32 - __clz(max(1, nk - 1))));
    const int slot0 = lane & (T - 1);
    const int team_in_warp = lane / T;
    const int teams_per_warp = 32 / T;
    const uint64_t grab = static_cast<uint64_t>(teams_per_warp) * LOOM_BFS_GRAB;
    bool overflow = false;
    for (;;) {
      unsigned long long g0 = 0;
      if (lane == 0) g0 = atomicAdd(&bs->next[d], static_cast<unsigned long long>(grab));
      g0 = __shfl_sync(0xffffffffu, g0, 0);
      if (g0 >= n_cur) break;
      for (int r = 0; r < LOOM_BFS_GRAB; ++r) {
        const uint64_t pi = g0 + static_cast<uint64_t>(r) * teams_per_warp + team_in_warp;
        FrontierEntry par{0, 0.0, 0.0, INT64_MAX, 0, 0, 0, INT_MAX, 0};
        if (pi < n_cur) par = src == 2 ? cur[pi] : sfront[src][pi];
        // a prefix whose first-criterion bound is now worse than the incumbent
        // (found at its own level, after it was kept) is not expanded
        const bool alive = pi < n_cur && par.key <= bkey;
        for (int s0 = 0; s0 < nk; s0 += T) {
          const int slot = s0 + slot0;
          bool keep = false;
          FrontierEntry ch{};
          if (alive && slot < nk) {
            ++evals;
            leaves += leaf;
            keep = bfs_child(B, S, jd, ranged, par, d, slot, bound, suf, fin, ch, cand);
          }
          if (!leaf) {  // append survivors: one atomic per warp
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
    }
    // level end: CTA best -> its slot; after the barrier every CTA reduces all slots
    const Rec cb = bfs_block_best(cand, h, S.warp_slot);
    if (threadIdx.x == 0) slots[blockIdx.x] = cb;
    if (__syncthreads_or(overflow) && threadIdx.x == 0) atomicExch(&bs->overflow, 1u);
    grid_barrier(bs, gridDim.x);
    Rec r{0, 0, 0, 0, 0, 0, 0};
    for (int i = threadIdx.x; i < static_cast<int>(gridDim.x); i += kBfsBlock) {
      const Rec o = load_rec_cg(&slots[i]);
      if (rec_better(o, r, h)) r = o;
    }
    r = bfs_block_best(r, h, S.warp_slot);
    if (threadIdx.x == 0) {
      if (rec_better(r, S.best, h)) S.best = r;
      S.stop = __ldcg(&bs->overflow) != 0u;
    }
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) g_bfs_trace[2 * d + 2] = bfs_now();
    if (S.stop || leaf) break;
    n_cur = __ldcg(&bs->count[k]);
    // the next level reads the entries this one wrote
    FrontierEntry* t = cur;
    cur = nxt;
    nxt = t;
    src = 2;
  }

  // evidence, result, reset
  if (evals) atomicAdd(&bs->evals, evals);
  if (leaves) atomicAdd(&bs->leaves, leaves);
  if (threadIdx.x == 0) {
    unsigned long long mf = 0;
    for (int i = 1; i <= n; ++i) mf = max(mf, __ldcg(&bs->count[i]));
    atomicMax(&bs->max_frontier, mf);
  }
  grid_barrier(bs, gridDim.x);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    g_bfs_trace[1] = bfs_now();
    const bool of = bs->overflow != 0u;
    out[0] = S.best;
    sync[0].pad = of ? kBfsOverflow : kBnbDone;
    g_bfs_last[0] = bs->evals;
    g_bfs_last[1] = of;
    g_bfs_last[2] = bs->max_frontier;
    g_bfs_last[3] = gridDim.x;
    g_bfs_last[4] = bs->leaves;
    for (int i = 0; i <= kMaxNodes; ++i) bs->count[i] = bs->next[i] = 0;
    bs->lock = 0;
    bs->overflow = 0;
    bs->evals = 0;
    bs->leaves = 0;
    bs->max_frontier = 0;
    // bar_count is 0 again after the barrier; bar_gen keeps counting
  }
}

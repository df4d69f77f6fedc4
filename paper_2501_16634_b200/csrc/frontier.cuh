// Frontier branch and bound: the default search (included by loom_search.cu
// inside its anonymous namespace, after bnb.cuh).
//
// Contract: the argmin of objective_less (estimator.hpp:93-116) over the
// plans of a range (optimizer.hpp:173-188).  A subtree of the
// ConfigEnumerator tree (optimizer.hpp:131-143; node 0 most significant) is
// dropped only when a lower bound of its plans' criteria is infeasible or
// lexicographically STRICTLY worse than a real plan already found (bnb.cuh
// states the bounds), so the argmin is never dropped.  The tree is explored
// level by level across the whole GPU:
//
//   expand (phase A)  a warp takes up to 32 parents (prefixes of d digits),
//                     one per lane.  The lane computes the latency terms of
//                     node d under its prefix -- the longest path avoiding d
//                     (lnot), the latest finish among d's predecessors (head)
//                     and the longest path from d's successors to the end
//                     (tail), the other free nodes at their smallest walls --
//                     with a finish-time recursion (estimator.hpp:69-76) held
//                     in REGISTERS: positions in topological order, the
//                     predecessor/successor sets as bit masks in the kernel's
//                     parameter bank, loops unrolled over NB positions.  It
//                     also evaluates two real plans of the prefix's subtree
//                     exactly -- free nodes at the option best on the primary
//                     criterion, and at their smallest walls (whose latency is
//                     max(lnot, head + wmin + tail)) -- as incumbents.
//   children (phase B) the warp's lanes walk the parents' children (parent
//                     p, option slot s) 32 at a time: child latency bound
//                     max(lnot, head + wall + tail), FP bounds from the
//                     prefix folds plus the free nodes' minima, compare with
//                     the lane's incumbent.  Survivors are staged per warp and
//                     appended to the next frontier 32+ at a time (one atomic).
//                     At depth n the children are leaves: exact records.
//   incumbent         lanes start every level from the job's best; a warp
//                     shares any plan its lanes found before pruning children;
//                     per level: CTA best (only if it improved) -> per-CTA
//                     slot -> grid barrier -> every CTA reduces the slots.
//                     The order is strict and total, so the result does not
//                     depend on timing.
//   small levels      a level with at most kFrSmall children runs redundantly
//                     in every CTA (same parents, same children, same
//                     reduction: no grid barrier); its children are compacted
//                     in shared memory with a block scan (same order in every
//                     CTA, so the next level can split them by index).
//
// One cooperative launch (all CTAs resident) runs every level.  The problem
// image is copied to shared memory once (TMA bulk copy); per-problem constants
// (topology masks, completion options, suffix bounds, the seed's exact record)
// arrive as a __grid_constant__ kernel parameter built on the host.  A
// frontier that outgrows its buffer sets `overflow`: the job's best so far
// goes to out[0], JobSync.pad = kBfsOverflow, and the depth-first kernel
// (bnb.cuh) that follows takes over from that incumbent (then the sweep, if
// it too runs out of budget).  Launched in a plain stream, both follow-up
// launches otherwise retire at once (JobSync.pad = kBnbDone); inside the
// search graph of a device problem they sit behind a conditional node that
// this kernel sets only on overflow (cudaGraphSetConditional).

__device__ unsigned long long g_bfs_last[6];  // evidence of the last frontier launch
// Per-level trace of the last launch (CTA 0): [0] start, [1] end, [2d+2] =
// %globaltimer at the end of depth d's level, [2d+3] = parents expanded |
// redundant << 63 (loom_bfs_trace).
__device__ unsigned long long g_bfs_trace[2 * (kMaxNodes + 2)];

// LOOM_FR_PROF=1 (experiment builds): clock64() marks of CTA 0 / thread 0 at
// phase boundaries, g_fr_prof[8 * depth + mark] (loom_debug_fr_prof); =4
// also marks the incumbent heuristic's phases (loom_debug_fr_prof2).
#ifndef LOOM_FR_PROF
#define LOOM_FR_PROF 0
#endif
__device__ unsigned long long g_fr_prof[8 * (kMaxNodes + 1)];
__device__ unsigned long long g_fr_prof2[16];  // LOOM_FR_PROF=4: marks of the incumbent heuristic (CTA 0, thread 0)
#define FR_MARKH(i)                                                                                   \
  do {                                                                                                \
    if (LOOM_FR_PROF == 4 && blockIdx.x == 0 && threadIdx.x == 0) g_fr_prof2[i] = clock64();          \
  } while (0)
#define FR_MARK(d, i)                                                                                   \
  do {                                                                                                  \
    if (LOOM_FR_PROF && blockIdx.x == 0 && threadIdx.x == 0) g_fr_prof[8 * (d) + (i)] = clock64();     \
  } while (0)

__device__ __forceinline__ unsigned long long bfs_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#ifndef LOOM_FR_BLOCK
#define LOOM_FR_BLOCK 512
#endif
constexpr int kFrBlock = LOOM_FR_BLOCK;  // one CTA per SM: fewer arrivals per grid barrier
constexpr int kFrWarps = kFrBlock / 32;
#ifndef LOOM_FR_SMALL
#define LOOM_FR_SMALL 1536
#endif
constexpr int kFrSmall = LOOM_FR_SMALL;  // children of a redundant level (shared-memory frontier slots)
constexpr int kFrStage = 64;             // kept children staged per warp before an append
#ifndef LOOM_FR_HEUR
#define LOOM_FR_HEUR 1  // incumbent heuristic before the first level (fr_incumbent)
#endif
#ifndef LOOM_FR_COMPLETE
#define LOOM_FR_COMPLETE 2  // deepest level whose parents also get their two completions
#endif
#ifndef LOOM_FR_HPASS
#define LOOM_FR_HPASS 2  // its 1-opt passes at most (more found nothing on the C3 goldens)
#endif

// Per-problem constants of the frontier search (a kernel parameter; every
// array index below is a compile-time constant after unrolling, or uniform).
template <int NB>
struct BfsParams {
  int32_t n;
  int32_t n_crit;
  int32_t crit[4];
  int32_t ranged;
  int32_t has_seed;
  int64_t slo_eff;
  uint64_t begin;
  uint64_t end;
  Rec seed;  // the incumbent every CTA starts from (exact record, host-evaluated)
  uint64_t seed_dig;  // its digits, packed like FrontierEntry.dig
  int32_t heur;       // run the incumbent heuristic (spaces too small to need it skip its ~15 us)
  int32_t n_qlev;     // distinct option qualities (descending, at most 8): targets of the quality-first heuristic
  int32_t qlev[8];
  double lam_lo;         // heuristic lambda grid: 0, then lam_lo .. lam_lo * 2^lam_log2_span geometrically
  double lam_log2_span;
  // by topological position t
  int32_t tnode[NB];    // node at position t
  // pm[t][p] = ~0 if position p precedes position t by an edge, else 0;
  // sm[t][s] likewise for successors.  Indexed by compile-time constants
  // after unrolling, so every mask is an instruction operand from the
  // parameter bank (no load, no branch): F[t] = W[t] + max_p (F[p] & pm[t][p]).
  uint32_t pm[NB][NB];
  uint32_t sm[NB][NB];
  int32_t tshift[NB];   // digit of node tnode[t]: (dig >> tshift) & tbits
  uint32_t tbits[NB];
  int32_t toptoff[NB];
  int64_t twmin[NB];    // smallest wall of node tnode[t] among options meeting the quality floor
  int64_t twprim[NB];   // wall of its primary-best option
  // by node (dag order = digit order)
  int32_t pos[NB];      // topological position of node i
  int32_t shift[NB];
  uint32_t bits[NB];
  int32_t optoff[NB];
  int32_t nok[NB];      // options meeting the quality floor (BlobHeader.off_nok)
  int32_t radix[NB];
  double pa[NB];        // primary-best option (exploration order's first): FP_A, FP_B terms, quality
  double pb[NB];
  int32_t pq[NB];
  double wa[NB];        // smallest-wall option (BnbMin.o_wall)
  double wb[NB];
  int32_t wq[NB];
  uint64_t lexp_suf[NB + 1];  // identifier-rank terms of the completions over nodes >= k
  uint64_t lexw_suf[NB + 1];
  uint64_t idxp_suf[NB + 1];  // index of the completions' digits of nodes >= k
  uint64_t idxw_suf[NB + 1];
  uint64_t rk[NB + 1];        // plans below a prefix of k digits
  BnbSuf suf[NB + 1];         // bounds over the free nodes k .. n-1
};

// Shared-memory tables of the problem image.
struct FrTab {
  const int32_t* perm;
  const double* ga;
  const double* gb;
  const int64_t* wall;
  const int32_t* q;
  const uint64_t* lexw;
  const int32_t* optoff;  // per node (also in the parameters; these are for per-lane indexing)
  const int32_t* nok;
};

// A parent being expanded: its prefix and the latency terms of the next node.
struct alignas(16) FrPar {
  uint64_t dig;
  double fa;
  double fb;
  int64_t lnot;
  int64_t head;
  int64_t tail;
  int32_t q;
  int32_t live;
};

struct FrShared {
  Rec best;  // the incumbent: identical in every CTA after every level
  Rec warp_slot[kFrWarps];
  uint64_t mbar;
  unsigned wcnt[kFrSmall / kFrBlock][kFrWarps];
  unsigned long long ncur;
  int32_t stop;
  int32_t last;
  int32_t flag;
  uint64_t hdig;  // packed digits of `best` during the incumbent heuristic
  int32_t shift[kMaxNodes];  // BfsParams.shift / bits, for per-lane indexing
  uint32_t bits[kMaxNodes];
  unsigned long long evals;
  unsigned long long leaves;
  unsigned long long maxf;
};

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }

template <int NB>
__device__ __forceinline__ int fr_digit(const BfsParams<NB>& P, uint64_t dig, int i) {
  return static_cast<int>((dig >> P.shift[i]) & static_cast<uint64_t>(P.bits[i]));
}

// Key of criterion kind c (CritKind; kFrNone = unused slot) of a record:
// smaller is better.
constexpr int32_t kFrNone = 4;
__device__ __forceinline__ int64_t fr_ckey(int32_t c, int64_t qa, int64_t qb, int64_t lat, int32_t q) {
  int64_t k = 0;
  k = c == kFpA ? qa : k;
  k = c == kFpB ? qb : k;
  k = c == kLat ? lat : k;
  k = c == kQual ? -static_cast<int64_t>(q) : k;
  return k;
}

// Criteria lists known at compile time (CL > 0), in slot kinds -- the
// objective tokens of objective_from_token (workflow.hpp:91-106): 1 =
// [FP_A, latency] (MIN_COST, MIN_DOLLARS), 2 = [latency, FP_A]
// (MIN_LATENCY), 3 = [quality, FP_A, latency] (MAX_QUALITY).  CL = 0 reads
// any list from the parameters.  With a static list every key select below
// folds away.
template <int CL, int NB>
__device__ __forceinline__ int32_t fr_crit(const BfsParams<NB>& P, int i) {
  if constexpr (CL == 1) return i == 0 ? kFpA : i == 1 ? kLat : kFrNone;
  else if constexpr (CL == 2) return i == 0 ? kLat : i == 1 ? kFpA : kFrNone;
  else if constexpr (CL == 3) return i == 0 ? kQual : i == 1 ? kFpA : i == 2 ? kLat : kFrNone;
  else return P.crit[i];
}
template <int CL>
__host__ __device__ constexpr int fr_ncrit() { return CL == 1 || CL == 2 ? 2 : CL == 3 ? 3 : 4; }

// Criteria of a plan against a record: -1 better, 1 worse, 0 equal on every
// criterion (the identifier decides).  Unused criterion slots are kFrNone.
template <int CL, int NB>
__device__ __forceinline__ int fr_cmp(const BfsParams<NB>& P, int64_t qa, int64_t qb, int64_t lat, int32_t q,
                                      const Rec& b) {
  if (!b.found) return -1;
#pragma unroll
  for (int i = 0; i < fr_ncrit<CL>(); ++i) {
    const int32_t c = fr_crit<CL>(P, i);
    const int64_t x = fr_ckey(c, qa, qb, lat, q);
    const int64_t y = fr_ckey(c, b.qa, b.qb, b.lat, b.qual);
    if (x != y) return x < y ? -1 : 1;
  }
  return 0;
}

// True when the criteria ranked before latency already make the plan
// strictly worse than b (its latency need not be computed).
template <int CL, int NB>
__device__ __forceinline__ bool fr_worse_before_lat(const BfsParams<NB>& P, int64_t qa, int64_t qb, int32_t q,
                                                    const Rec& b) {
  if (!b.found) return false;
#pragma unroll
  for (int i = 0; i < fr_ncrit<CL>(); ++i) {
    const int32_t c = fr_crit<CL>(P, i);
    if (c == kLat) return false;
    const int64_t x = fr_ckey(c, qa, qb, 0, q);
    const int64_t y = fr_ckey(c, b.qa, b.qb, 0, b.qual);
    if (x != y) return x > y;
  }
  return false;
}

template <int CL, int NB>
__device__ __forceinline__ int64_t fr_key(const BfsParams<NB>& P, int64_t qa, int64_t qb, int64_t lat, int32_t q) {
  if constexpr (CL == 0)
    if (P.n_crit == 0) return INT64_MIN;
  return fr_ckey(fr_crit<CL>(P, 0), qa, qb, lat, q);
}

template <int CL, int NB>
__device__ __forceinline__ int64_t fr_bound_key(const BfsParams<NB>& P, const Rec& b) {
  return b.found ? fr_key<CL>(P, b.qa, b.qb, b.lat, b.qual) : INT64_MAX;
}

// Identifier rank and plan index of the plan whose nodes < k take the
// digits of `dig` and nodes >= k the completion `comp` (0: none -- a leaf,
// 1: primary-best options, 2: smallest walls).
template <int NB>
__device__ __forceinline__ void fr_lex_idx(const BfsParams<NB>& P, const FrTab& T, uint64_t dig, int k, int comp,
                                           uint64_t& lex, uint64_t& idx) {
  lex = comp == 1 ? P.lexp_suf[k] : comp == 2 ? P.lexw_suf[k] : 0;
  uint64_t pidx = 0;
#pragma unroll 1
  for (int i = 0; i < k; ++i) {  // rare (ties or improvements only): kept small
    const int c = fr_digit(P, dig, i);
    lex += T.lexw[P.optoff[i] + c];
    pidx = pidx * static_cast<uint64_t>(P.radix[i]) + static_cast<uint64_t>(c);
  }
  idx = pidx * P.rk[k] + (comp == 1 ? P.idxp_suf[k] : comp == 2 ? P.idxw_suf[k] : 0);
}

// Offer an exactly evaluated plan to the lane's incumbent.
template <int CL, int NB>
__device__ __forceinline__ void fr_offer(const BfsParams<NB>& P, const FrTab& T, uint64_t dig, int k, int comp,
                                         double a, double b, int32_t q, int64_t lat, Rec& cand) {
  if (lat > P.slo_eff) return;
  const int64_t qa = quantize_dev(a), qb = quantize_dev(b);
  const int cmp = fr_cmp<CL>(P, qa, qb, lat, q, cand);
  if (cmp > 0) return;
  uint64_t lex, idx;
  fr_lex_idx(P, T, dig, k, comp, lex, idx);
  if (cmp == 0 && lex >= cand.lexkey) return;
  if (P.ranged && (idx < P.begin || idx >= P.end)) return;
  cand = Rec{qa, qb, lat, lex, idx, q, 1};
}

// Phase A, one of three independent jobs on the prefix of entry e (nodes < k
// fixed, node k next), each one finish-time recursion (estimator.hpp:69-76)
// in registers -- positions in topological order, predecessor / successor
// sets as bit masks in the parameter bank, loops unrolled over NB:
//   job 0  latency terms of node k, the other free nodes at their smallest
//          walls: lnot (longest path avoiding k), head (latest finish among
//          k's predecessors), tail (longest path from k's successors on)
//   job 1  completion with every free node at its primary-best option,
//          offered to `cand` (skipped when the criteria ranked before
//          latency already lose)
//   job 2  completion with every free node at its smallest wall, offered
//          (its latency is max(lnot, head + wmin + tail): no recursion when
//          job 0 ran on the same lane)
// A small batch runs the three jobs of a parent on three lanes; otherwise
// one lane runs them in turn.  L: int32_t when every latency stays below
// 2^30 us (host-checked), else int64_t.
template <int CL, int NB, typename L>
__device__ __forceinline__ L fr_mask(L v, uint32_t m) {
  return v & static_cast<L>(static_cast<int32_t>(m));  // m is 0 or ~0: sign-extends to 0 or all ones
}

template <int CL, int NB, typename L>
__device__ __forceinline__ void fr_job(const BfsParams<NB>& P, const FrTab& T, const FrontierEntry& e, int k, int job,
                                       FrPar& out, Rec& cand, bool have_terms) {
  constexpr L kGone = -(L(1) << (sizeof(L) * 8 - 2));  // a removed node: paths through it never win a max
  const int n = P.n;
  const int xpos = P.pos[k];
  // the FP folds of a completion continue in dag order (estimator.hpp:50-60)
  double a = e.fa, b = e.fb;
  int32_t q = e.q;
  if (job != 0) {  // lanes of jobs 1 and 2 run the same instructions (operands selected per lane)
    const bool pj = job == 1;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      if (i >= n) break;
      if (i >= k) {
        const double ta = P.pa[i], tb = P.pb[i], wa = P.wa[i], wb = P.wb[i];
        const int32_t tq = P.pq[i], wq = P.wq[i];
        a = __dadd_rn(a, pj ? ta : wa);
        b = __dadd_rn(b, pj ? tb : wb);
        q = min(q, pj ? tq : wq);
      }
    }
    if (pj && fr_worse_before_lat<CL>(P, quantize_dev(a), quantize_dev(b), q, cand)) return;
  }
  if (job == 2 && have_terms) {  // job 0 ran on this lane: the smallest-wall completion's latency is the bound
    const int64_t lat = max(out.lnot, out.head + P.twmin[xpos] + out.tail);
    fr_offer<CL>(P, T, e.dig, k, 2, a, b, q, lat, cand);
    return;
  }
  const bool prim = job == 1;
  L W[NB];
#pragma unroll
  for (int t = 0; t < NB; ++t) {
    if (t >= n) break;
    W[t] = static_cast<L>(prim ? P.twprim[t] : P.twmin[t]);
    if (P.tnode[t] < k)
      W[t] = static_cast<L>(T.wall[P.toptoff[t] + static_cast<int>((e.dig >> P.tshift[t]) & P.tbits[t])]);
  }
  // forward; job 0 removes node k
  L F[NB];
  L lmax = 0, head = 0;
  const bool rm = job == 0;
#pragma unroll
  for (int t = 0; t < NB; ++t) {
    if (t >= n) break;
    L st = 0;
#pragma unroll
    for (int p = 0; p < t; ++p) st = max(st, fr_mask<CL, NB, L>(F[p], P.pm[t][p]));
    const bool x = rm && t == xpos;
    head = x ? st : head;
    F[t] = x ? kGone : st + W[t];
    lmax = max(lmax, F[t]);
  }
  if (job != 0) {
    fr_offer<CL>(P, T, e.dig, k, job, a, b, q, static_cast<int64_t>(lmax), cand);
    return;
  }
  // backward over the positions after k: longest path from each to the end
#pragma unroll
  for (int t = NB - 1; t >= 0; --t) {
    if (t < n && t > xpos) {
      L m = 0;
#pragma unroll
      for (int s2 = t + 1; s2 < NB; ++s2) m = max(m, fr_mask<CL, NB, L>(F[s2], P.sm[t][s2]));
      F[t] = m + W[t];
    }
  }
  L tail = 0;
#pragma unroll
  for (int s2 = 1; s2 < NB; ++s2)
    if (s2 > xpos && s2 < n) tail = max(tail, fr_mask<CL, NB, L>(F[s2], P.sm[xpos][s2]));
  out.dig = e.dig;
  out.fa = e.fa;
  out.fb = e.fb;
  out.q = e.q;
  out.lnot = lmax;
  out.head = head;
  out.tail = tail;
  out.live = 1;
}

// Exact record of the complete plan `dig` (every digit set), offered to
// cand: eval_digits restated on packed digits (folds in dag order from 0.0,
// the finish-time recursion over topological positions in registers).
template <int CL, int NB, typename L>
__device__ __forceinline__ void fr_offer_plan(const BfsParams<NB>& P, const FrTab& T, uint64_t dig, Rec& cand) {
  const int n = P.n;
  double a = 0.0, b = 0.0;
  int32_t q = INT_MAX;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    if (i >= n) break;
    const int o = P.optoff[i] + fr_digit(P, dig, i);
    a = __dadd_rn(a, T.ga[o]);
    b = __dadd_rn(b, T.gb[o]);
    q = min(q, T.q[o]);
  }
  L F[NB];
  L lat = 0;
#pragma unroll
  for (int t = 0; t < NB; ++t) {
    if (t >= n) break;
    L st = 0;
#pragma unroll
    for (int p = 0; p < t; ++p) st = max(st, fr_mask<CL, NB, L>(F[p], P.pm[t][p]));
    F[t] = st + static_cast<L>(T.wall[P.toptoff[t] + static_cast<int>((dig >> P.tshift[t]) & P.tbits[t])]);
    lat = max(lat, F[t]);
  }
  fr_offer<CL>(P, T, dig, n, 0, a, b, q, static_cast<int64_t>(lat), cand);
}

// Phase B: child `slot` (exploration rank) of parent `par` at depth d.  A
// leaf is offered exactly; otherwise returns whether the subtree survives.
template <int CL, int NB>
__device__ __forceinline__ bool fr_child(const BfsParams<NB>& P, const FrTab& T, const FrPar& par, int d, int slot,
                                         bool leaf, FrontierEntry& ch, Rec& cand) {
  const int c = T.perm[P.optoff[d] + slot];
  const int o = P.optoff[d] + c;
  const double fa = __dadd_rn(par.fa, T.ga[o]);
  const double fb = __dadd_rn(par.fb, T.gb[o]);
  const int32_t q = min(par.q, T.q[o]);
  const int64_t lat = max(par.lnot, par.head + T.wall[o] + par.tail);  // exact at a leaf
  const uint64_t dig = par.dig | (static_cast<uint64_t>(c) << P.shift[d]);
  const int k = d + 1;
  if (leaf) {
    fr_offer<CL>(P, T, dig, k, 0, fa, fb, q, lat, cand);
    return false;
  }
  if (lat > P.slo_eff) return false;
  if (P.ranged) {
    uint64_t pidx = 0;
#pragma unroll 1
    for (int i = 0; i < k; ++i) {
      pidx = pidx * static_cast<uint64_t>(P.radix[i]) + static_cast<uint64_t>(fr_digit(P, dig, i));
    }
    const uint64_t lo = pidx * P.rk[k];
    if (!(lo < P.end && lo + P.rk[k] > P.begin)) return false;
  }
  // FP bounds: the fold of the prefix continued with the free nodes' minima,
  // rounded down (BnbSuf, bnb.cuh)
  const BnbSuf& s = P.suf[k];
  const int64_t qa = quantize_dev(__dmul_rd(__dadd_rd(fa, s.a), s.fac));
  const int64_t qb = quantize_dev(__dmul_rd(__dadd_rd(fb, s.b), s.fac));
  const int32_t qu = min(q, s.q);
  const int cmp = fr_cmp<CL>(P, qa, qb, lat, qu, cand);
  if (cmp > 0) return false;
  if (cmp == 0) {  // every criterion ties the incumbent: the identifier decides
    uint64_t lx = s.lex;
#pragma unroll 1
    for (int i = 0; i < k; ++i) {
      lx += T.lexw[P.optoff[i] + fr_digit(P, dig, i)];
    }
    if (lx > cand.lexkey) return false;
  }
  ch.dig = dig;
  ch.fa = fa;
  ch.fb = fb;
  ch.key = fr_key<CL>(P, qa, qb, lat, qu);
  ch.q = q;
  ch.live = 1;
  ch.pad = 0;
  return true;
}

__device__ __forceinline__ Rec shfl_xor_rec(const Rec& r, int m) {
  Rec o;
  o.qa = __shfl_xor_sync(0xffffffffu, r.qa, m);
  o.qb = __shfl_xor_sync(0xffffffffu, r.qb, m);
  o.lat = __shfl_xor_sync(0xffffffffu, r.lat, m);
  o.lexkey = __shfl_xor_sync(0xffffffffu, r.lexkey, m);
  o.index = __shfl_xor_sync(0xffffffffu, r.index, m);
  o.qual = __shfl_xor_sync(0xffffffffu, r.qual, m);
  o.found = __shfl_xor_sync(0xffffffffu, r.found, m);
  return o;
}

template <int CL, int NB>
__device__ __forceinline__ bool fr_better(const BfsParams<NB>& P, const Rec& a, const Rec& b) {
  if (!a.found) return false;
  const int c = fr_cmp<CL>(P, a.qa, a.qb, a.lat, a.qual, b);
  return c < 0 || (c == 0 && a.lexkey < b.lexkey);
}

// Every lane of the warp gets the warp's best record.
template <int CL, int NB>
__device__ __forceinline__ void fr_warp_best(const BfsParams<NB>& P, Rec& r) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {
    const Rec o = shfl_xor_rec(r, m);
    if (fr_better<CL>(P, o, r)) r = o;
  }
}

// Block-wide best of the records with `mine` set (the others, e.g. lanes
// that found nothing better than the level's incumbent, are left out; a warp
// with none skips its reduction).  Valid in thread 0.
template <int CL, int NB>
__device__ __forceinline__ Rec fr_block_best(const BfsParams<NB>& P, Rec r, bool mine, Rec* warp_slot) {
  if (!mine) r.found = 0;
  if (__any_sync(0xffffffffu, mine)) fr_warp_best<CL>(P, r);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) warp_slot[warp] = r;
  __syncthreads();
  if (warp == 0) {
    r = lane < kFrWarps ? warp_slot[lane] : Rec{0, 0, 0, 0, 0, 0, 0};
    if (__any_sync(0xffffffffu, r.found)) fr_warp_best<CL>(P, r);
  }
  return r;
}

// Incumbent heuristic before the first level, run identically by every CTA
// (no communication; the result is a real plan, so the argmin is unchanged
// and only the pruning improves).  A good incumbent from the start shrinks
// every frontier: searched from the true optimum, C3 under the 40 s SLO
// evaluates 0.18M children instead of 2.0M.
//   H1 (FP-primary objectives): 64 plans, each picking per node the option
//       minimising primary term + lambda x wall (a Lagrangian relaxation of
//       "min energy s.t. latency <= SLO"; lambda = 0 and a geometric grid
//       over 1e-10 .. 1; one warp per plan, one lane per node).  Quality-primary
//       objectives do the same per quality target (options below the target
//       skipped) with the next FP criterion as the primary term.
//   H2: best-improvement 1-opt from the incumbent, one (node, option) swap
//       per thread, up to LOOM_FR_HPASS passes.
template <int CL, int NB, typename L>
__device__ void fr_incumbent(const BfsParams<NB>& P, const FrTab& T, FrShared& S) {
  const int n = P.n;
  FR_MARKH(0);
  Rec cand = S.best;
  uint64_t cdig = S.hdig;
  const int32_t c0 = fr_crit<CL>(P, 0);
  const int32_t c1 = fr_ncrit<CL>() > 1 ? fr_crit<CL>(P, 1) : kFrNone;
  const bool fp_first = P.n_crit > 0 && (c0 == kFpA || c0 == kFpB);
  const bool q_first = P.n_crit > 0 && c0 == kQual && P.n_qlev > 0;
  if (fp_first || q_first) {
    // kHR rounds; in round r warp w takes combination r * warps + w (a
    // lambda and, quality first, a quality target: options below it are
    // skipped where a node has one at or above it; the next FP criterion is
    // the primary term), lane i chooses node i's option, and lane r keeps
    // the round's plan; then lanes 0..kHR-1 evaluate their plans at once
    constexpr int kHR = 4;
    constexpr int kCombos = kHR * kFrWarps;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nq = q_first ? P.n_qlev : 1;
    const int nl = (kCombos + nq - 1) / nq;
    const int32_t cg = fp_first ? c0 : (c1 == kFpA || c1 == kFpB ? c1 : kFrNone);
    const double* g = cg == kFpB ? T.gb : T.ga;
    const double gs = cg == kFrNone ? 0.0 : 1.0;
    const int base = lane < n ? T.optoff[lane] : 0;
    const int nr = lane < n ? T.optoff[lane + 1] - base : 0;  // raw options: the floor-failing ones carry
    const int sh = lane < n ? S.shift[lane] : 0;              // walls above any SLO and are skipped
    double lam[kHR];
    int32_t qt[kHR];
#pragma unroll
    for (int r = 0; r < kHR; ++r) {
      const int combo = r * kFrWarps + warp;
      const int li = combo / nq;
      qt[r] = q_first ? P.qlev[combo % nq] : INT_MIN;
      lam[r] = li == 0 ? 0.0 : P.lam_lo * exp2(P.lam_log2_span * li / max(1, nl - 1));
    }
    double bv[kHR];
    int64_t bw[kHR];
    int bc[kHR];
#pragma unroll
    for (int r = 0; r < kHR; ++r) {
      bv[r] = INFINITY;
      bw[r] = INT64_MAX;
      bc[r] = -1;
    }
    // one scan of the node's options serves the kHR plans
    for (int relax = 0; relax < 2; ++relax) {  // relax 1: plans whose target no option of the node meets
#pragma unroll 4
      for (int o = 0; o < nr; ++o) {
        const int64_t w = T.wall[base + o];
        if (w > P.slo_eff) continue;
        const double gv = gs * g[base + o];
        const int32_t qo = T.q[base + o];
#pragma unroll
        for (int r = 0; r < kHR; ++r) {
          if (relax ? bc[r] >= 0 : qo < qt[r]) continue;
          const double v = gv + lam[r] * static_cast<double>(w);
          if (v < bv[r] || (v == bv[r] && w < bw[r])) {
            bv[r] = v;
            bw[r] = w;
            bc[r] = o;
          }
        }
      }
      bool all = true;
#pragma unroll
      for (int r = 0; r < kHR; ++r) all &= bc[r] >= 0 || nr == 0;
      if (__all_sync(0xffffffffu, all)) break;
    }
    uint64_t mine = 0;
#pragma unroll
    for (int r = 0; r < kHR; ++r) {
      const uint64_t part = bc[r] > 0 ? static_cast<uint64_t>(bc[r]) << sh : 0;  // (option 0 packs as 0)
      const uint32_t lo = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(part));
      const uint32_t hi = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(part >> 32));
      if (lane == r) mine = static_cast<uint64_t>(hi) << 32 | lo;
    }
    FR_MARKH(1);
    if (lane < kHR) {
      const uint64_t before = cand.index;
      const int32_t bf = cand.found;
      fr_offer_plan<CL, NB, L>(P, T, mine, cand);
      if (cand.found && (!bf || cand.index != before)) cdig = mine;
    }
    FR_MARKH(2);
  }
  int slots = 0;
  for (int i = 0; i < n; ++i) slots += T.nok[i];
#pragma unroll 1
  for (int pass = 0; pass <= LOOM_FR_HPASS; ++pass) {
    // the block's best; its owner publishes the packed digits
    const Rec b0 = S.best;
    const Rec cb = fr_block_best<CL>(P, cand, cand.found && (!b0.found || cand.index != b0.index), S.warp_slot);
    if (threadIdx.x == 0) {
      S.flag = fr_better<CL>(P, cb, S.best);
      if (S.flag) S.best = cb;
    }
    __syncthreads();
    if (!S.flag && pass > 0) break;
    if (S.flag && cand.found && cand.index == S.best.index) S.hdig = cdig;
    __syncthreads();
    FR_MARKH(3 + 2 * pass);
    if (pass == LOOM_FR_HPASS || !S.best.found) break;
    // H2: one swap per thread from the incumbent
    const uint64_t D = S.hdig;
    cand = S.best;
    cdig = D;
    for (int u = threadIdx.x; u < slots; u += kFrBlock) {
      int i = 0, acc = 0;
      while (u >= acc + T.nok[i]) acc += T.nok[i++];  // (shared memory: lanes index different nodes)
      const int c = T.perm[T.optoff[i] + (u - acc)];
      const uint64_t dig = (D & ~(static_cast<uint64_t>(S.bits[i]) << S.shift[i])) |
                           (static_cast<uint64_t>(c) << S.shift[i]);
      if (dig == D) continue;
      const uint64_t before = cand.index;
      const int32_t bf = cand.found;
      fr_offer_plan<CL, NB, L>(P, T, dig, cand);
      if (cand.found && (!bf || cand.index != before)) cdig = dig;
    }
    FR_MARKH(4 + 2 * pass);
  }
}

// Grid barrier of the cooperative launch (all CTAs resident): one arrival per
// CTA with release semantics, the last arriver resets the count and bumps
// the generation (release), the others poll it (acquire).
__device__ __forceinline__ void fr_grid_barrier(BfsSync* bs, unsigned n_ctas) {
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
        __nanosleep(32);
      }
    }
  }
  __syncthreads();
}

// Where a level's survivors go.
struct FrOut {
  // redundant level: child j of the level -> sparse[j] (live or not)
  FrontierEntry* sparse;
  // distributed level: per-warp staging, appended to nxt[count[k]++]
  FrontierEntry* stage;
  int sn;
  FrontierEntry* nxt;
  unsigned long long* count;
  uint64_t cap;
  bool overflow;
};

__device__ __forceinline__ void fr_flush(FrOut& o) {
  __syncwarp();
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == 0 && o.sn) base = atomicAdd(o.count, static_cast<unsigned long long>(o.sn));
  base = __shfl_sync(0xffffffffu, base, 0);
  for (int i = lane; i < o.sn; i += 32) {
    const uint64_t at = base + static_cast<uint64_t>(i);
    if (at < o.cap) o.nxt[at] = o.stage[i];
    else o.overflow = true;
  }
  o.sn = 0;
  __syncwarp();
}

// What a warp does with its batch of parents (fr_batch).
constexpr int kBatchAll = 0;       // expansion (three jobs) and children
constexpr int kBatchExpand = 1;    // job 0 and the children
constexpr int kBatchComplete = 2;  // the two completions only

// How the depth-first and sweep kernels follow a frontier launch.
constexpr int32_t kFollowAlways = 0;  // launched after it on the stream; they retire at once unless it overflowed
constexpr int32_t kFollowGraph = 1;   // behind the search graph's conditional node (cudaGraphSetConditional)
constexpr int32_t kFollowHost = 2;    // launched by the host only after reading JobSync.pad == kBfsOverflow

// One warp: expand parents [p0, p0 + np) of depth d (np <= 32) and evaluate
// their children.  redundant: children go to o.sparse by child index.
template <int CL, int NB, typename L>
__device__ __forceinline__ void fr_batch(const BfsParams<NB>& P, const FrTab& T, const FrontierEntry* parents,
                                         uint64_t p0, int np, int d, bool leaf, bool redundant, int mode,
                                         unsigned magic, FrPar* pb, Rec& cand, FrOut& o, unsigned long long& evals,
                                         unsigned long long& leaves) {
  const int lane = threadIdx.x & 31;
  const Rec before = cand;
  // mode kBatchAll: a small batch gives each parent three lanes (one job
  // each), else one lane runs the three jobs; kBatchExpand: job 0 and the
  // children only; kBatchComplete: jobs 1 and 2 (two lanes per parent) only
  const bool split = mode == kBatchAll && np * 3 <= 32;
  const int pl = mode == kBatchComplete ? lane >> 1 : split ? lane / 3 : lane;
  const int j0 = mode == kBatchComplete ? 1 + (lane & 1) : split ? lane - 3 * pl : 0;
  const int j1 = mode == kBatchAll && !split ? 2 : j0;
  FrPar fp;
  fp.live = 0;
  if (pl < np) {
    const FrontierEntry e = parents[p0 + pl];
    // a prefix whose first-criterion bound is now worse than the incumbent
    // (found after it was kept) is not expanded
    if (e.live && e.key <= fr_bound_key<CL>(P, cand)) {
#pragma unroll 1
      for (int j = j0; j <= j1; ++j) fr_job<CL, NB, L>(P, T, e, d, j, fp, cand, j == 2 && j0 == 0);
    }
  }
  FR_MARK(d, 1);
  if (mode == kBatchComplete) return;  // its plans reach the level's reduction through cand
  if (j0 == 0 && pl < 32) pb[pl] = fp;
  // plans found while expanding prune the children of the whole warp
  if (__any_sync(0xffffffffu, cand.index != before.index || cand.found != before.found)) fr_warp_best<CL>(P, cand);
  __syncwarp();
  FR_MARK(d, 2);
  const int nk = P.nok[d];
  const int total = np * nk;
  for (int c0 = 0; c0 < total; c0 += 32) {
    const int c = c0 + lane;
    bool keep = false;
    FrontierEntry ch;
    int pi = 0, slot = 0;
    if (c < total) {
      // c / nk: exact for c * nk < 2^32 (c < 32 nk, nk <= 6144); nk = 1 has no 32-bit magic
      pi = nk == 1 ? c : static_cast<int>(__umulhi(static_cast<unsigned>(c), magic));
      slot = c - pi * nk;
      const FrPar par = pb[pi];
      if (par.live) {
        ++evals;
        leaves += leaf;
        keep = fr_child<CL>(P, T, par, d, slot, leaf, ch, cand);
      }
    }
    if (redundant) {
      if (!leaf && c < total) {
        if (!keep) ch.live = 0;
        o.sparse[(p0 + static_cast<uint64_t>(pi)) * nk + slot] = ch;
      }
    } else if (!leaf) {
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) o.stage[o.sn + __popc(m & ((1u << lane) - 1))] = ch;
      o.sn += __popc(m);
      if (o.sn > kFrStage - 32) fr_flush(o);
    }
  }
  __syncwarp();  // pb is rewritten by the next batch
  FR_MARK(d, 3);
}

template <int NB, typename L, int CL>
__global__ void __launch_bounds__(kFrBlock, 1)
    bfs_kernel(const uint8_t* __restrict__ blob, uint32_t blob_bytes, BfsSync* __restrict__ bs,
               FrontierEntry* __restrict__ buf0, FrontierEntry* __restrict__ buf1, uint64_t cap,
               Rec* __restrict__ slots, JobSync* __restrict__ sync, Rec* __restrict__ out,
               cudaGraphConditionalHandle fallback, int32_t follow, const __grid_constant__ BfsParams<NB> P) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ FrShared S;
  FR_MARKH(14);
  load_blob(smem, blob, blob_bytes, &S.mbar);
  FR_MARKH(15);
  const BnbView B = make_bnb_view(smem);
  const FrTab T{B.perm, B.v.ga, B.v.gb, B.v.wall, B.v.q, B.v.lexw, B.v.optoff, B.nok};
  const int n = P.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t img = (blob_bytes + 127) & ~127u;
  FrontierEntry* sA = reinterpret_cast<FrontierEntry*>(smem + img);  // compacted small frontier
  FrontierEntry* sB = sA + kFrSmall;                                 // sparse children of a redundant level
  FrPar* pb = reinterpret_cast<FrPar*>(sB + kFrSmall) + warp * 32;
  // per-warp staging of a distributed level shares sB (used by redundant levels only)
  FrontierEntry* stage = sB + warp * kFrStage;
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) {
      g_bfs_trace[0] = bfs_now();
      for (int i = 1; i < 2 * (kMaxNodes + 2); ++i) g_bfs_trace[i] = 0;
    }
    S.best = P.has_seed ? P.seed : Rec{0, 0, 0, 0, 0, 0, 0};
    S.hdig = P.seed_dig;
    for (int i = 0; i < n; ++i) {
      S.shift[i] = P.shift[i];
      S.bits[i] = P.bits[i];
    }
    S.stop = 0;
    S.ncur = 1;
    S.evals = S.leaves = S.maxf = 0;
    sA[0] = FrontierEntry{0, 0.0, 0.0, INT64_MIN, INT_MAX, 1, 0};  // the root: no digit fixed
  }
  bool empty = n == 0;
  for (int i = 0; i < n; ++i) empty |= P.nok[i] == 0;
  __syncthreads();
  FR_MARKH(12);
  const bool heur = LOOM_FR_HEUR && P.heur;
  if (!empty && heur) fr_incumbent<CL, NB, L>(P, T, S);
  FR_MARKH(13);

  unsigned long long evals = 0, leaves = 0;
  const FrontierEntry* cur = sA;  // parents of the level
  FrontierEntry* gbuf[2] = {buf0, buf1};
  int gnext = 0;  // global buffer the next distributed level writes
  const uint64_t gwarp = static_cast<uint64_t>(blockIdx.x) * kFrWarps + warp;
  const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * kFrWarps;
  for (int d = 0; d < n && !empty; ++d) {
    const uint64_t n_cur = S.ncur;
    if (n_cur == 0) break;
    FR_MARK(d, 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) g_bfs_trace[2 * d + 3] = n_cur;
    const int nk = P.nok[d];
    const bool leaf = d + 1 == n;
    const unsigned magic = 0xffffffffu / static_cast<unsigned>(nk) + 1u;
    Rec cand = S.best;
    const uint64_t b_idx = cand.index;
    const int32_t b_found = cand.found;
    FrOut o{sB, stage, 0, nullptr, nullptr, cap, false};
    const bool redundant = n_cur * static_cast<uint64_t>(nk) <= static_cast<uint64_t>(kFrSmall);
    const int k = d + 1;
    o.nxt = gbuf[gnext];
    o.count = &bs->count[k];
    // Batches of parents, one call site (the batch code is inlined once):
    // redundant -- every CTA the same work, warp w takes parents [w * per,
    // (w + 1) * per) in batches of 32; distributed -- batches of `np`
    // parents, the first one static (warp id), the rest dealt by an atomic
    // counter.
    uint64_t p, lim, npb;
    // a small distributed level (at most one parent per two warps): one
    // warp expands a parent while another evaluates its two completions,
    // so neither waits for the other's divergent path
    // completions (jobs 1, 2) only feed the incumbent, which the heuristic
    // has already found on every C3 golden objective: below depth
    // LOOM_FR_COMPLETE they are skipped (the top levels keep them -- they are
    // small -- in case the heuristic was weak)
    const bool expand_only = heur && d > LOOM_FR_COMPLETE;
    const bool sep = !redundant && !expand_only && 2 * n_cur <= nwarps;
    int mode = expand_only ? kBatchExpand : kBatchAll;
    if (redundant) {
      const uint64_t per = (n_cur + kFrWarps - 1) / kFrWarps;
      p = static_cast<uint64_t>(warp) * per;
      lim = umin64(n_cur, p + per);
      npb = 32;
    } else if (sep) {
      npb = 1;
      mode = gwarp < n_cur ? kBatchExpand : kBatchComplete;
      p = gwarp < n_cur ? gwarp : gwarp - n_cur;
      lim = gwarp < 2 * n_cur ? p + 1 : 0;
    } else {
      // about two batches per warp: the dynamic deal evens out the tail
      npb = umin64(32, umax64(1, (n_cur + 2 * nwarps - 1) / (2 * nwarps)));
      p = gwarp * npb;
      lim = n_cur;
    }
    unsigned long long e0 = 0, l0 = 0;
    // distributed: the next batch is claimed before this one is processed,
    // so the atomic's round trip overlaps the work
    unsigned long long g = 0;
    const bool dyn = !redundant && !sep;
    if (dyn && lane == 0 && p < lim) g = atomicAdd(&bs->next[d], static_cast<unsigned long long>(npb));
    while (p < lim) {
      fr_batch<CL, NB, L>(P, T, cur, p, static_cast<int>(umin64(npb, lim - p)), d, leaf, redundant, mode, magic, pb,
                          cand, o, e0, l0);
      if (!dyn) {
        p += npb;
      } else {
        p = nwarps * npb + __shfl_sync(0xffffffffu, g, 0);
        if (lane == 0 && p < lim) g = atomicAdd(&bs->next[d], static_cast<unsigned long long>(npb));
      }
    }
    FR_MARK(d, 4);
    if (!redundant || blockIdx.x == 0) {  // a redundant level is counted once
      evals += e0;
      leaves += l0;
    }
    if (redundant) {
      // the level's best: every CTA computes the same
      const Rec cb = fr_block_best<CL>(P, cand, cand.found && (!b_found || cand.index != b_idx), S.warp_slot);
      if (threadIdx.x == 0 && fr_better<CL>(P, cb, S.best)) S.best = cb;
      FR_MARK(d, 5);
      if (!leaf) {
        // compact the sparse children into sA (block scan, the same order in every CTA)
        constexpr int R = kFrSmall / kFrBlock;
        const uint64_t nch = n_cur * static_cast<uint64_t>(nk);
        bool live[R];
        unsigned m[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint64_t j = static_cast<uint64_t>(r) * kFrBlock + threadIdx.x;
          live[r] = j < nch && sB[j].live;
          m[r] = __ballot_sync(0xffffffffu, live[r]);
          if (lane == 0) S.wcnt[r][warp] = __popc(m[r]);
        }
        __syncthreads();
        unsigned tot = 0, pre[R];
#pragma unroll
        for (int r = 0; r < R; ++r) pre[r] = 0;
        for (int r2 = 0; r2 < R; ++r2)
          for (int w = 0; w < kFrWarps; ++w) {
            const unsigned x = S.wcnt[r2][w];
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (r2 < r || (r2 == r && w < warp)) pre[r] += x;
            tot += x;
          }
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (live[r]) sA[pre[r] + __popc(m[r] & ((1u << lane) - 1))] = sB[static_cast<uint64_t>(r) * kFrBlock + threadIdx.x];
        if (threadIdx.x == 0) {
          S.ncur = tot;
          S.maxf = max(S.maxf, static_cast<unsigned long long>(tot));
        }
        cur = sA;
      }
      __syncthreads();
      FR_MARK(d, 6);
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        g_bfs_trace[2 * d + 2] = bfs_now();
        g_bfs_trace[2 * d + 3] |= 1ull << 63;
      }
      if (leaf) break;
      continue;
    }
    if (!leaf && o.sn) fr_flush(o);
    // level end: the CTA's best, if it improved on the level's incumbent,
    // goes to its slot (else an empty record); after the grid barrier every
    // CTA reduces the slots (a warp without a found record skips its part)
    const Rec cb = fr_block_best<CL>(P, cand, cand.found && (!b_found || cand.index != b_idx), S.warp_slot);
    if (threadIdx.x == 0) slots[blockIdx.x] = cb;
    FR_MARK(d, 5);
    if (__syncthreads_or(o.overflow) && threadIdx.x == 0) atomicExch(&bs->overflow, 1u);
    fr_grid_barrier(bs, gridDim.x);
    FR_MARK(d, 6);
    Rec r{0, 0, 0, 0, 0, 0, 0};
    for (int i = threadIdx.x; i < static_cast<int>(gridDim.x); i += kFrBlock) {
      const Rec x = load_rec_cg(&slots[i]);
      if (fr_better<CL>(P, x, r)) r = x;
    }
    r = fr_block_best<CL>(P, r, r.found, S.warp_slot);
    if (threadIdx.x == 0) {
      if (fr_better<CL>(P, r, S.best)) S.best = r;
      S.stop = __ldcg(&bs->overflow) != 0u;
      const unsigned long long nn = leaf ? 0ull : __ldcg(&bs->count[k]);
      S.ncur = nn;
      S.maxf = max(S.maxf, nn);
    }
    __syncthreads();
    FR_MARK(d, 7);
    if (blockIdx.x == 0 && threadIdx.x == 0) g_bfs_trace[2 * d + 2] = bfs_now();
    if (S.stop || leaf) break;
    cur = gbuf[gnext];
    gnext ^= 1;
  }

  // evidence; the last CTA out writes the result and resets the job state
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {  // one shared atomic per warp (a 64-bit shared add is a CAS loop)
    evals += __shfl_xor_sync(0xffffffffu, evals, m);
    leaves += __shfl_xor_sync(0xffffffffu, leaves, m);
  }
  if (lane == 0 && evals) atomicAdd(&S.evals, evals);
  if (lane == 0 && leaves) atomicAdd(&S.leaves, leaves);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (S.evals) atomicAdd(&bs->evals, S.evals);
    if (S.leaves) atomicAdd(&bs->leaves, S.leaves);
    atomicMax(&bs->max_frontier, S.maxf);
    __threadfence();
    S.last = atomicAdd(&bs->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (S.last && threadIdx.x == 0) {
    __threadfence();
    const bool of = __ldcg(&bs->overflow) != 0u;
    out[0] = S.best;
    // How the fallback kernels follow (FrFollow): always launched, retiring
    // at once on kBnbDone; behind the search graph's conditional node, opened
    // only on overflow; or launched by the host only on overflow.
    if (follow == kFollowGraph) cudaGraphSetConditional(fallback, of ? 1u : 0u);
    sync[0].pad = of ? kBfsOverflow : (follow == kFollowAlways ? kBnbDone : 0u);
    g_bfs_last[0] = __ldcg(&bs->evals);
    g_bfs_last[1] = of;
    g_bfs_last[2] = __ldcg(&bs->max_frontier);
    g_bfs_last[3] = gridDim.x;
    g_bfs_last[4] = __ldcg(&bs->leaves);
    g_bfs_trace[1] = bfs_now();
    for (int i = 0; i <= kMaxNodes; ++i) bs->count[i] = bs->next[i] = 0;
    bs->ticket = 0;
    bs->overflow = 0;
    bs->evals = 0;
    bs->leaves = 0;
    bs->max_frontier = 0;
    __threadfence();
    // bar_count is 0 after every barrier; bar_gen keeps counting
  }
}

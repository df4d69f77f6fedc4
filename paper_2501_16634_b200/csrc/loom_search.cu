// sm_100a plan-evaluation kernels: exhaustive argmin over the plan space of a
// workflow DAG (the reference's loom::exhaustive_search, optimizer.hpp:173-188)
// and its batched, multi-job form.
//
// ALGORITHM.  Plans are indices in ConfigEnumerator order
// (optimizer.hpp:136-141): node 0 is the most significant digit.  The last K
// nodes (K = 2..4) form the "suffix"; a "subrow" fixes every digit except the
// last K-1, i.e. it holds r_sub = prod(radix[N-K+1..N-1]) consecutive plans.
// Each thread walks a contiguous run of subrows:
//   * per row (prefix digits change): the energy / dollar left folds of the
//     prefix nodes in dag order (estimator.hpp:50-60) and a longest-path DP
//     over the DAG in topological order that treats the K suffix walls as
//     symbols.  Its output is a max-plus coefficient vector c[S] over subsets
//     S of the suffix: latency = max_S (c[S] + sum_{s in S} wall_s).  Integer
//     max/+ is exact, so this equals the reference's finish-time recursion
//     (estimator.hpp:69-76) for every plan.
//   * per suffix level: one option of node N-K+j fixes one wall, folding the
//     coefficient vector in half (c'[S] = max(c[S], c[S+s_j] + w)) and adding
//     one term to each FP fold -- in dag order, so every plan's sums round
//     exactly like the reference's.
//   * innermost node: lat = max(X, Y + w) and e = e_prefix + g per plan.
// Every plan's primary criterion and feasibility (quality floor folded into
// an unreachable wall, optional latency SLO) are computed.  Plans that can
// tie or beat the running best take an exact slow path that quantizes with
// llround semantics (estimator.hpp:85-87) and compares the full hierarchy
// then the identifier rank (estimator.hpp:93-116).  Because the order is a
// strict total order, the per-thread, per-warp, per-CTA and cross-CTA
// reductions are order independent and bit-exact.
//
// Range edges that do not cover whole subrows, and problems with a single
// node, go through full_eval(): one plan per thread, decoded from its index
// and re-evaluated from scratch (the reference algorithm restated; also
// exposed as algo 1 for cross-checking).
//
// Compiled with -fmad=false; all FP sums use __dadd_rn explicitly.

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <queue>
#include <string>
#include <system_error>
#include <tuple>
#include <vector>

#include "internal.h"
#include "loom_b200.h"
#include "search_common.h"
#include "ctx.h"
#include "tma.cuh"

using namespace loomk;
using loomi::DevBuf;
using loomi::cuda_fail;

namespace {

constexpr int64_t kNeg = -(int64_t(1) << 62);
constexpr unsigned kBnbDone = 1;     // JobSync.pad after a branch-and-bound launch (bnb.cuh)
constexpr unsigned kBnbAborted = 2;
constexpr unsigned kBfsOverflow = 3;  // after a frontier search (bfs.cuh) that overflowed: depth first takes over

#ifndef LOOM_PAIR_UNROLL
#define LOOM_PAIR_UNROLL 4
#endif
constexpr int kPairUnroll = LOOM_PAIR_UNROLL;
// LOOM_STATS=1 (experiment builds): event counters of the search kernel,
// read with loom_debug_counters.  0: flagged steps, 1: contexts passing the
// bound re-test, 2: contexts passing the exact test (slow scans), 3: steps.
#ifndef LOOM_STATS
#define LOOM_STATS 0
#endif
__device__ unsigned long long g_stats[8];
#define LOOM_COUNT(i, n)                                      \
  do {                                                        \
    if (LOOM_STATS) atomicAdd(&g_stats[i], (unsigned long long)(n)); \
  } while (0)
#ifndef LOOM_PT_CTAS
#define LOOM_PT_CTAS 6  // resident CTAs per SM of single-problem launches (128 threads: register cap 80, 24 warps)
#endif
#ifndef LOOM_SWEEP_SYNC
#define LOOM_SWEEP_SYNC 1  // reconverge after every innermost sweep (else once per subrow step)
#endif
#ifndef LOOM_F32_SPLIT
#define LOOM_F32_SPLIT 0  // energy-first sweep: also use the FP32 pipe (experiment)
#endif
#ifndef LOOM_SWEEP_PAIRS
#define LOOM_SWEEP_PAIRS 1  // energy-first: several sweeps per unrolled block (level K-3)
#endif
#ifndef LOOM_SWEEP_GROUP
#define LOOM_SWEEP_GROUP 2  // sweeps per block
#endif
#ifndef LOOM_JOB_BOUND
#define LOOM_JOB_BOUND 1
#endif
#ifndef LOOM_ENERGY_FIRST
#define LOOM_ENERGY_FIRST 1
#endif

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------

// llround(v * 1e9) with the C library's half-away-from-zero rounding
// (estimator.hpp:85-87).  x - trunc(x) is exact in binary64.
__device__ __forceinline__ int64_t quantize_dev(double v) {
  const double x = __dmul_rn(v, 1e9);
  const double t = trunc(x);
  const double f = __dsub_rn(x, t);
  int64_t r = __double2ll_rz(t);
  if (f >= 0.5) r += 1;
  else if (f <= -0.5) r -= 1;
  return r;
}

// A value strictly above this bound quantizes strictly above q (conservative:
// values between the exact bound and this one just take the exact slow path).
__device__ __forceinline__ double hi_of(int64_t q) {
  const double y = (static_cast<double>(q) + 0.5) / 1e9;
  return y + fabs(y) * 1e-12 + 1e-300;
}

struct View {
  const BlobHeader* h;
  const int32_t* radix;
  const int32_t* optoff;
  const int32_t* topo;
  const int32_t* predoff;
  const int32_t* pred;
  const double* ga;
  const double* gb;
  const int64_t* wall;
  const uint64_t* lexw;
  const int32_t* q;
  const InnerEntry* inner;
};

__device__ __forceinline__ View make_view(const uint8_t* s) {
  View v;
  v.h = reinterpret_cast<const BlobHeader*>(s);
  v.radix = reinterpret_cast<const int32_t*>(s + v.h->off_radix);
  v.optoff = reinterpret_cast<const int32_t*>(s + v.h->off_optoff);
  v.topo = reinterpret_cast<const int32_t*>(s + v.h->off_topo);
  v.predoff = reinterpret_cast<const int32_t*>(s + v.h->off_predoff);
  v.pred = reinterpret_cast<const int32_t*>(s + v.h->off_pred);
  v.ga = reinterpret_cast<const double*>(s + v.h->off_ga);
  v.gb = reinterpret_cast<const double*>(s + v.h->off_gb);
  v.wall = reinterpret_cast<const int64_t*>(s + v.h->off_wall);
  v.lexw = reinterpret_cast<const uint64_t*>(s + v.h->off_lexw);
  v.q = reinterpret_cast<const int32_t*>(s + v.h->off_q);
  v.inner = reinterpret_cast<const InnerEntry*>(s + v.h->off_inner);
  return v;
}

__device__ __forceinline__ bool rec_better(const Rec& a, const Rec& b, const BlobHeader* h) {
  if (!a.found) return false;
  if (!b.found) return true;
  for (int i = 0; i < h->n_crit; ++i) {
    switch (h->crit[i]) {
      case kFpA:
        if (a.qa != b.qa) return a.qa < b.qa;
        break;
      case kFpB:
        if (a.qb != b.qb) return a.qb < b.qb;
        break;
      case kLat:
        if (a.lat != b.lat) return a.lat < b.lat;
        break;
      default:
        if (a.qual != b.qual) return a.qual > b.qual;
        break;
    }
  }
  return a.lexkey < b.lexkey;
}

// ---------------------------------------------------------------------------
// Per-thread running best and its derived thresholds live in shared memory
// (structure of arrays, one slot per thread, conflict free).  Only the rare
// slow path touches them; the hot loops keep just the thresholds they test.
// ---------------------------------------------------------------------------
struct Slots {
  int64_t* qa;
  int64_t* qb;
  int64_t* lat;
  uint64_t* lex;
  uint64_t* idx;
  double* hi;      // kPrimFp: e > hi  =>  strictly worse than the best
  int64_t* lat_s;  // feasible and not worse on latency: lat <= lat_s
  int32_t* qual;
  int32_t* found;
  int32_t* bq;     // kPrimQual: q < bq  =>  strictly worse
};
constexpr int kSlotBytes = 8 * 7 + 4 * 3;

__device__ __forceinline__ Slots make_slots(uint8_t* base) {
  Slots s;
  s.qa = reinterpret_cast<int64_t*>(base);
  s.qb = s.qa + kBlock;
  s.lat = s.qb + kBlock;
  s.lex = reinterpret_cast<uint64_t*>(s.lat + kBlock);
  s.idx = s.lex + kBlock;
  s.hi = reinterpret_cast<double*>(s.idx + kBlock);
  s.lat_s = reinterpret_cast<int64_t*>(s.hi + kBlock);
  s.qual = reinterpret_cast<int32_t*>(s.lat_s + kBlock);
  s.found = s.qual + kBlock;
  s.bq = s.found + kBlock;
  return s;
}

__device__ __forceinline__ Rec slot_load(const Slots& s, int t) {
  return Rec{s.qa[t], s.qb[t], s.lat[t], s.lex[t], s.idx[t], s.qual[t], s.found[t]};
}

__device__ __forceinline__ void slot_thresholds(const Slots& s, int t, const BlobHeader* h) {
  const bool f = s.found[t];
  s.hi[t] = f ? hi_of(s.qa[t]) : INFINITY;
  // latency-first objectives only: an empty hierarchy also runs the kPrimLat
  // kernel, but there the identifier alone orders plans, so a slower plan can
  // still win and the SLO is the only latency bound
  const bool lat_first = h->prim == kPrimLat && h->n_crit > 0;
  const bool tight = f && (lat_first || (h->tie_lat && s.qa[t] <= h->qa_floor));
  s.lat_s[t] = tight ? min(h->slo_eff, s.lat[t]) : h->slo_eff;
  s.bq[t] = f ? s.qual[t] : INT_MIN;
}

__device__ __forceinline__ void slot_init(const Slots& s, int t, const BlobHeader* h) {
  s.qa[t] = s.qb[t] = s.lat[t] = 0;
  s.lex[t] = s.idx[t] = 0;
  s.qual[t] = 0;
  s.found[t] = 0;
  slot_thresholds(s, t, h);
}

// Job-wide bound on the primary FP criterion (energy-first objectives): every
// thread publishes the quantized primary criterion of its feasible bests, and
// reads the job's minimum at each DP group.  A plan whose bucket is above the
// minimum is strictly worse than a feasible plan of the searched range, so it
// cannot be the argmin; the bound only tightens the fast tests.
__shared__ unsigned long long* s_gbest;

__device__ __forceinline__ void publish_best(const BlobHeader* h, const Rec& c) {
  if (h->prim == kPrimFp && c.found && s_gbest && c.qa >= 0)
    atomicMax(s_gbest, static_cast<unsigned long long>(INT64_MAX - c.qa));
}

__device__ __forceinline__ void slot_offer(const Slots& s, int t, const BlobHeader* h, const Rec& c) {
  if (rec_better(c, slot_load(s, t), h)) {
    // publish only a strictly better bucket (a handful per thread): ties
    // improving on latency or rank would hammer one address
    if (c.found && (!s.found[t] || c.qa < s.qa[t])) publish_best(h, c);
    s.qa[t] = c.qa;
    s.qb[t] = c.qb;
    s.lat[t] = c.lat;
    s.lex[t] = c.lexkey;
    s.idx[t] = c.index;
    s.qual[t] = c.qual;
    s.found[t] = c.found;
    slot_thresholds(s, t, h);
  }
}

// One plan from its digits, evaluated from scratch exactly as the reference's
// estimate (estimator.hpp:43-78): FP left folds in dag order, finish-time
// recursion in topological order over the effective walls (a quality-floor
// failure has an unreachable wall), quality min, identifier rank.
__device__ void eval_digits(const View& v, const int* d, Rec& c, uint64_t index) {
  const int n = v.h->n_nodes;
  double ea = 0.0, eb = 0.0;
  int32_t qual = INT_MAX;
  uint64_t lex = 0;
  for (int i = 0; i < n; ++i) {
    const int o = v.optoff[i] + d[i];
    ea = __dadd_rn(ea, v.ga[o]);
    eb = __dadd_rn(eb, v.gb[o]);
    qual = min(qual, v.q[o]);
    lex += v.lexw[o];
  }
  int64_t fin[kMaxNodes];
  int64_t lat = 0;
  for (int t = 0; t < n; ++t) {
    const int node = v.topo[t];
    int64_t s = 0;
    for (int e = v.predoff[node]; e < v.predoff[node + 1]; ++e) s = max(s, fin[v.pred[e]]);
    fin[node] = s + v.wall[v.optoff[node] + d[node]];
    lat = max(lat, fin[node]);
  }
  c.found = lat <= v.h->slo_eff;
  c.lat = lat;
  c.qual = qual;
  c.lexkey = lex;
  c.index = index;
  c.qa = c.found ? quantize_dev(ea) : 0;
  c.qb = c.found ? quantize_dev(eb) : 0;
}

// One plan decoded from its index (range edges, algo 1).
__device__ void full_eval(const View& v, uint64_t index, Rec& c) {
  int d[kMaxNodes];
  uint64_t x = index;
  for (int i = v.h->n_nodes - 1; i >= 0; --i) {
    const uint64_t r = static_cast<uint64_t>(v.radix[i]);
    d[i] = static_cast<int>(x % r);
    x /= r;
  }
  eval_digits(v, d, c, index);
}

// Slow path of the hierarchical walk: the prefix digits plus the K suffix
// digits name one plan that might tie or beat the running best; evaluate it
// from scratch and offer it.  Out of line so the hot loops stay small.
__device__ __noinline__ void offer_plan(const uint8_t* smem, uint8_t* slot_base, const int* dpre, int P, int K,
                                        int o0, int o1, int o2, int o3, uint64_t index) {
  const View v = make_view(smem);
  int d[kMaxNodes];
  for (int i = 0; i < P; ++i) d[i] = dpre[i];
  const int od[4] = {o0, o1, o2, o3};
  for (int j = 0; j < K; ++j) d[P + j] = od[j];
  Rec c;
  eval_digits(v, d, c, index);
  slot_offer(make_slots(slot_base), threadIdx.x, v.h, c);
}

// Slow path of one innermost context (rare): rescan options [g_begin, g_end)
// of the innermost node, drop the ones the cheap tests reject, and build the
// exact record of each remaining plan from the fast path's partials:
//   latency = max(X, Y + wall)          (the max-plus pair of the context)
//   energy  = quantize(eu + g)          (the dag-order fold, last term added)
//   rank    = lex_u + rank term         (identifier order)
// then compare it under the full objective order.  Objectives whose criteria
// are not carried incrementally (a second FP sum, or quality when it is not
// the primary) re-evaluate the plan from its digits instead.
template <int K, int PRIM>
__device__ __noinline__ void slow_scan(const uint8_t* smem, uint8_t* slot_base, const int* dpre, int P, int o0,
                                       int o1, int o2, int g_begin, int g_end, int32_t tw, double eu, int32_t qu,
                                       uint64_t lex_u, int64_t X, int64_t Y, uint64_t base) {
  const View v = make_view(smem);
  const BlobHeader* h = v.h;
  const Slots sl = make_slots(slot_base);
  const int t = threadIdx.x;
  const int inner_node = h->n_nodes - 1;
  const int off = v.optoff[inner_node];
  const int n = v.radix[inner_node];
  for (int j = g_begin; j < g_end && j < n; ++j) {
    const InnerEntry e = v.inner[j];
    if (e.w > tw) continue;  // infeasible (or, for a latency primary, strictly slower)
    const double ev = __dadd_rn(eu, e.g);
    if (PRIM == kPrimFp && ev > sl.hi[t]) continue;
    if (PRIM == kPrimQual && min(qu, e.q) < sl.bq[t]) continue;
    if (h->needs_full) {
      int od[4] = {o0, o1, o2, 0};
      od[K - 1] = j;
      offer_plan(smem, slot_base, dpre, P, K, od[0], od[1], od[2], od[3], base + static_cast<uint64_t>(j));
      continue;
    }
    Rec c;
    c.lat = max(X, Y + v.wall[off + j]);
    c.found = c.lat <= h->slo_eff;
    c.qa = quantize_dev(ev);
    c.qb = 0;
    c.qual = min(qu, e.q);
    c.lexkey = lex_u + v.lexw[off + j];
    c.index = base + static_cast<uint64_t>(j);
    slot_offer(sl, t, h, c);
  }
}

// Hot-loop context of one thread.
struct Hot {
  const uint8_t* smem;
  uint8_t* slot_base;
  uint8_t* coef_base;
  const int64_t* c0;  // level-0 coefficient vector (thread-local)
  const BlobHeader* h;
  const int32_t* radix;
  const int32_t* optoff;
  const double* ga;
  const int64_t* wall;
  const int32_t* w32;
  const int32_t* q;
  const uint64_t* lexw;
  const InnerEntry* inner;
  const int* dpre;
  int P;
  int od[4];
  uint64_t s_index;  // subrow index (row * radix[P] + o0)
  double hi;         // thresholds mirrored from the shared slot
  double hi_up;      // the double above hi (see ctx_bound)
  int64_t lat_s;
  int32_t bq;
  unsigned sync_mask;  // lanes of the warp working on the current subrow step
};

// The double above x (x itself for +inf).
__device__ __forceinline__ double next_up(double x) {
  if (x == INFINITY || x != x) return x;
  if (x == 0.0) return __longlong_as_double(1);
  const long long b = __double_as_longlong(x);
  return __longlong_as_double(x > 0 ? b + 1 : b - 1);
}

__device__ __forceinline__ void reload(Hot& H) {
  const Slots s = make_slots(H.slot_base);
  const int t = threadIdx.x;
  H.hi = s.hi[t];
  H.hi_up = next_up(H.hi);
  H.lat_s = s.lat_s[t];
  H.bq = s.bq[t];
}

__device__ __forceinline__ int64_t clamp64(int64_t x, int64_t lo, int64_t hi) { return min(max(x, lo), hi); }

// Exact int32 form of the latency test for the last two suffix nodes (u = the
// node above the innermost, v = the innermost), given the coefficients c[4]
// over subsets of {u, v} (bit 0 = u, bit 1 = v) and the bound L:
//   max(c0, c1 + wu, c2 + wv, c3 + wu + wv) <= L
//   <=> c0 <= L  &&  wu <= L - c1  &&  wv - wmin <= min(L - wmin - c2, L - wmin - c3 - wu)
// Clamping keeps every comparison exact for wu in [0, wu_max] and
// wv - wmin in [0, 2^30) (checked on the host).
struct PreInner {
  int32_t cmax;  // wu <= cmax
  int32_t a;     // tw = min(a, b - wu)
  int32_t b;
};

__device__ __forceinline__ PreInner pre_inner(const int64_t (&c)[4], int64_t L, int64_t wmin, int64_t wu_max) {
  PreInner r;
  const int64_t kHi = int64_t(1) << 30;
  r.cmax = c[0] <= L ? static_cast<int32_t>(clamp64(L - c[1], -1, wu_max)) : -1;
  r.a = static_cast<int32_t>(clamp64(L - wmin - c[2], -1, kHi));
  r.b = static_cast<int32_t>(clamp64(L - wmin - c[3], -1, kHi + wu_max));
  return r;
}

__device__ __forceinline__ int32_t inner_tw(const PreInner& r, int32_t wu) {
  return wu <= r.cmax ? min(r.a, r.b - wu) : INT_MIN;
}

// Innermost node over one (prefix, o0 .. o_{K-2}) context.  NV > 0: the
// node's table is in registers (radix <= NV, padded with never-passing
// entries); NV == 0: read from shared memory in groups of 8.
template <int K, int PRIM, int NV, bool PT>
struct Inner {
  double g[NV > 0 && !PT ? NV : 1];
  int32_t w[NV > 0 && !PT ? NV : 1];

  // table entry j: kernel parameter (PT) or register copy
  __device__ __forceinline__ double G(const InnerParams& ip, int j) const { return PT ? ip.g[j] : g[PT ? 0 : j]; }
  __device__ __forceinline__ int32_t W(const InnerParams& ip, int j) const { return PT ? ip.w[j] : w[PT ? 0 : j]; }
  // high word of g (a register half for the register table)
  __device__ __forceinline__ int32_t GH(const InnerParams& ip, int j) const {
    return PT ? ip.gh[j] : __double2hiint(g[PT ? 0 : j]);
  }
  // g rounded down to binary32 (register tables convert on the fly)
  __device__ __forceinline__ float GF(const InnerParams& ip, int j) const {
    return PT ? ip.gf[j] : __double2float_rd(g[PT ? 0 : j]);
  }

  __device__ __forceinline__ void load(const Hot& H) {
    if constexpr (NV > 0 && !PT) {
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        g[j] = H.inner[j].g;
        w[j] = H.inner[j].w;
      }
    }
  }

  __device__ __forceinline__ bool pass(const Hot& H, int32_t w_, double g_, int32_t q_, int32_t tw, double ea,
                                       int32_t qv) const {
    if (PRIM == kPrimFp) return (w_ <= tw) & (__dadd_rn(ea, g_) <= H.hi);
    if (PRIM == kPrimLat) return w_ <= tw;
    return (w_ <= tw) & (min(qv, q_) >= H.bq);
  }

  // The fast loop's per-plan test: both criteria compared in the innermost
  // option's own table domain against per-context bounds (see ctx_bound).
  __device__ __forceinline__ bool pass_bound(int32_t w_, double g_, int32_t tw, double tu) const {
    if (PRIM == kPrimFp) return (w_ <= tw) & (g_ <= tu);
    return w_ <= tw;
  }

  // Energy-first fast test of two contexts: can any plan of either context
  // tie or beat the running best on the primary FP criterion?  A plan whose
  // energy is worse than the best's cannot be selected whatever its latency
  // (objective_less compares the primary criterion first, estimator.hpp:
  // 98-112), so its one test decides it; the few plans that pass are tested
  // on both criteria in the flagged contexts.  Even options are tested on the
  // FP64 pipe (DSETP), odd ones on the ALU pipe with the high words
  // (g <= t => hi(g) <= hi(t) for g >= +0; t < 0 has a negative high word),
  // so both pipes carry half of the plans.  A superset of the passing plans,
  // like every fast test.
  //
  // The compares are written in PTX so each plan keeps its own compare: the
  // OR over a context is otherwise an algebraic min over the (uniform) table
  // that the compiler hoists, which would turn the per-plan test into a
  // per-context bound.  One setp per plan, accumulated with setp's
  // predicate-OR form (SASS DSETP.LE.OR / ISETP.LE.OR).
  __device__ __forceinline__ bool any_energy2(const InnerParams& ip, double tu0, double tu1) const {
    static_assert(NV == 16 || NV == 8, "the PTX sweeps cover 8 or 16 options");
    const int32_t th0 = __double2hiint(tu0), th1 = __double2hiint(tu1);
    uint32_t flag;
    if constexpr (NV == 16 && LOOM_F32_SPLIT) {
      // three-way split: 6 options on the FP64 pipe, 5 on the ALU pipe (high
      // words), 5 on the FP32 pipe (binary32 round-down vs round-up bound)
      const float tf0 = __double2float_ru(tu0), tf1 = __double2float_ru(tu1);
      asm("{\n\t"
          ".reg .pred pf, pi, ps;\n\t"
          "setp.le.f64 pf, %1, %17;\n\t"
          "setp.le.or.f64 pf, %2, %17, pf;\n\t"
          "setp.le.or.f64 pf, %3, %17, pf;\n\t"
          "setp.le.or.f64 pf, %4, %17, pf;\n\t"
          "setp.le.or.f64 pf, %5, %17, pf;\n\t"
          "setp.le.or.f64 pf, %6, %17, pf;\n\t"
          "setp.le.or.f64 pf, %1, %18, pf;\n\t"
          "setp.le.or.f64 pf, %2, %18, pf;\n\t"
          "setp.le.or.f64 pf, %3, %18, pf;\n\t"
          "setp.le.or.f64 pf, %4, %18, pf;\n\t"
          "setp.le.or.f64 pf, %5, %18, pf;\n\t"
          "setp.le.or.f64 pf, %6, %18, pf;\n\t"
          "setp.le.s32 pi, %7, %19;\n\t"
          "setp.le.or.s32 pi, %8, %19, pi;\n\t"
          "setp.le.or.s32 pi, %9, %19, pi;\n\t"
          "setp.le.or.s32 pi, %10, %19, pi;\n\t"
          "setp.le.or.s32 pi, %11, %19, pi;\n\t"
          "setp.le.or.s32 pi, %7, %20, pi;\n\t"
          "setp.le.or.s32 pi, %8, %20, pi;\n\t"
          "setp.le.or.s32 pi, %9, %20, pi;\n\t"
          "setp.le.or.s32 pi, %10, %20, pi;\n\t"
          "setp.le.or.s32 pi, %11, %20, pi;\n\t"
          "setp.le.f32 ps, %12, %21;\n\t"
          "setp.le.or.f32 ps, %13, %21, ps;\n\t"
          "setp.le.or.f32 ps, %14, %21, ps;\n\t"
          "setp.le.or.f32 ps, %15, %21, ps;\n\t"
          "setp.le.or.f32 ps, %16, %21, ps;\n\t"
          "setp.le.or.f32 ps, %12, %22, ps;\n\t"
          "setp.le.or.f32 ps, %13, %22, ps;\n\t"
          "setp.le.or.f32 ps, %14, %22, ps;\n\t"
          "setp.le.or.f32 ps, %15, %22, ps;\n\t"
          "setp.le.or.f32 ps, %16, %22, ps;\n\t"
          "or.pred pf, pf, pi;\n\t"
          "or.pred pf, pf, ps;\n\t"
          "selp.u32 %0, 1, 0, pf;\n\t"
          "}"
          : "=r"(flag)
          : "d"(G(ip, 0)), "d"(G(ip, 3)), "d"(G(ip, 6)), "d"(G(ip, 9)), "d"(G(ip, 12)), "d"(G(ip, 15)),
            "r"(GH(ip, 1)), "r"(GH(ip, 4)), "r"(GH(ip, 7)), "r"(GH(ip, 10)), "r"(GH(ip, 13)),
            "f"(GF(ip, 2)), "f"(GF(ip, 5)), "f"(GF(ip, 8)), "f"(GF(ip, 11)), "f"(GF(ip, 14)),
            "d"(tu0), "d"(tu1), "r"(th0), "r"(th1), "f"(tf0), "f"(tf1));
    } else if constexpr (NV == 16) {
      asm("{\n\t"
          ".reg .pred pf, pi;\n\t"
          "setp.le.f64 pf, %1, %17;\n\t"
          "setp.le.or.f64 pf, %2, %17, pf;\n\t"
          "setp.le.or.f64 pf, %3, %17, pf;\n\t"
          "setp.le.or.f64 pf, %4, %17, pf;\n\t"
          "setp.le.or.f64 pf, %5, %17, pf;\n\t"
          "setp.le.or.f64 pf, %6, %17, pf;\n\t"
          "setp.le.or.f64 pf, %7, %17, pf;\n\t"
          "setp.le.or.f64 pf, %8, %17, pf;\n\t"
          "setp.le.or.f64 pf, %1, %18, pf;\n\t"
          "setp.le.or.f64 pf, %2, %18, pf;\n\t"
          "setp.le.or.f64 pf, %3, %18, pf;\n\t"
          "setp.le.or.f64 pf, %4, %18, pf;\n\t"
          "setp.le.or.f64 pf, %5, %18, pf;\n\t"
          "setp.le.or.f64 pf, %6, %18, pf;\n\t"
          "setp.le.or.f64 pf, %7, %18, pf;\n\t"
          "setp.le.or.f64 pf, %8, %18, pf;\n\t"
          "setp.le.s32 pi, %9, %19;\n\t"
          "setp.le.or.s32 pi, %10, %19, pi;\n\t"
          "setp.le.or.s32 pi, %11, %19, pi;\n\t"
          "setp.le.or.s32 pi, %12, %19, pi;\n\t"
          "setp.le.or.s32 pi, %13, %19, pi;\n\t"
          "setp.le.or.s32 pi, %14, %19, pi;\n\t"
          "setp.le.or.s32 pi, %15, %19, pi;\n\t"
          "setp.le.or.s32 pi, %16, %19, pi;\n\t"
          "setp.le.or.s32 pi, %9, %20, pi;\n\t"
          "setp.le.or.s32 pi, %10, %20, pi;\n\t"
          "setp.le.or.s32 pi, %11, %20, pi;\n\t"
          "setp.le.or.s32 pi, %12, %20, pi;\n\t"
          "setp.le.or.s32 pi, %13, %20, pi;\n\t"
          "setp.le.or.s32 pi, %14, %20, pi;\n\t"
          "setp.le.or.s32 pi, %15, %20, pi;\n\t"
          "setp.le.or.s32 pi, %16, %20, pi;\n\t"
          "or.pred pf, pf, pi;\n\t"
          "selp.u32 %0, 1, 0, pf;\n\t"
          "}"
          : "=r"(flag)
          : "d"(G(ip, 0)), "d"(G(ip, 2)), "d"(G(ip, 4)), "d"(G(ip, 6)), "d"(G(ip, 8)), "d"(G(ip, 10)),
            "d"(G(ip, 12)), "d"(G(ip, 14)), "r"(GH(ip, 1)), "r"(GH(ip, 3)), "r"(GH(ip, 5)), "r"(GH(ip, 7)),
            "r"(GH(ip, 9)), "r"(GH(ip, 11)), "r"(GH(ip, 13)), "r"(GH(ip, 15)), "d"(tu0), "d"(tu1), "r"(th0),
            "r"(th1));
    } else {
      asm("{\n\t"
          ".reg .pred pf, pi;\n\t"
          "setp.le.f64 pf, %1, %9;\n\t"
          "setp.le.or.f64 pf, %2, %9, pf;\n\t"
          "setp.le.or.f64 pf, %3, %9, pf;\n\t"
          "setp.le.or.f64 pf, %4, %9, pf;\n\t"
          "setp.le.or.f64 pf, %1, %10, pf;\n\t"
          "setp.le.or.f64 pf, %2, %10, pf;\n\t"
          "setp.le.or.f64 pf, %3, %10, pf;\n\t"
          "setp.le.or.f64 pf, %4, %10, pf;\n\t"
          "setp.le.s32 pi, %5, %11;\n\t"
          "setp.le.or.s32 pi, %6, %11, pi;\n\t"
          "setp.le.or.s32 pi, %7, %11, pi;\n\t"
          "setp.le.or.s32 pi, %8, %11, pi;\n\t"
          "setp.le.or.s32 pi, %5, %12, pi;\n\t"
          "setp.le.or.s32 pi, %6, %12, pi;\n\t"
          "setp.le.or.s32 pi, %7, %12, pi;\n\t"
          "setp.le.or.s32 pi, %8, %12, pi;\n\t"
          "or.pred pf, pf, pi;\n\t"
          "selp.u32 %0, 1, 0, pf;\n\t"
          "}"
          : "=r"(flag)
          : "d"(G(ip, 0)), "d"(G(ip, 2)), "d"(G(ip, 4)), "d"(G(ip, 6)), "r"(GH(ip, 1)), "r"(GH(ip, 3)),
            "r"(GH(ip, 5)), "r"(GH(ip, 7)), "d"(tu0), "d"(tu1), "r"(th0), "r"(th1));
    }
    return flag != 0;
  }

  // NV > 0: does any plan of the context pass?  (one predicate OR per plan)
  __device__ __forceinline__ bool any_pass(const Hot& H, const InnerParams& ip, int32_t tw, double ea,
                                           int32_t qv) const {
    bool any = false;
#pragma unroll
    for (int j = 0; j < (NV > 0 ? NV : 1); ++j) any |= pass(H, W(ip, j), G(ip, j), 0, tw, ea, qv);
    return any;
  }

};

// Suffix level J over options [o_lo, o_hi) of node P + J, given the
// coefficient vector over suffix nodes J..K-1 and the partial FP fold.
// Per-thread coefficient columns in shared memory: the input vector of suffix
// level J (2^(K-J) int64 entries) sits at column offset sum_{j<J} 2^(K-j),
// entry S at [S * kBlock + tid] (conflict free).  Keeping them out of the
// register file leaves the registers to the innermost table and thresholds.
// Per-thread coefficient columns in shared memory for suffix levels
// J = 1 .. K-2: the input vector of level J (2^(K-J) int64 entries) sits at
// column offset sum_{1<=j<J} 2^(K-j), entry S at [S * kBlock + tid] (conflict
// free).  Level 0's vector (read once per subrow) lives in local memory.
// Per-context energy bound in the innermost option's table domain.  A plan
// of the context has energy fl(eu + g) (the dag-order fold's last term,
// estimator.hpp:50-60) and passes the energy test iff fl(eu + g) <= hi.  If
// fl(x) <= hi under round-to-nearest then x <= hi + (hi_up - hi) / 2, where
// hi_up is the double above hi, so every passing g satisfies
//   g <= hi_up - eu <= tu = round_up(hi_up - eu).
// The fast loop therefore tests g <= tu per plan (one compare, no add) and
// lets through a superset of the passing plans: at most those whose g lies
// within about one ulp of the exact bound.  Survivors are re-tested exactly
// (fl(eu + g) <= hi) in slow_scan, so the selected plan is unchanged.
// Latency is handled the same way: w <= tw (inner_tw) is the exact latency
// test of the plan, expressed on the option's own wall.
__device__ __forceinline__ double ctx_bound(const Hot& H, double eu) { return __dadd_ru(H.hi_up, -eu); }

template <int K>
__device__ __forceinline__ int64_t* coef_col(uint8_t* coef_base, int J, bool lazy = false) {
  int off = 0;
  if (!lazy)  // lazy sweeps keep only the innermost pair's column, at offset 0
    for (int j = 1; j < J; ++j) off += 1 << (K - j);
  return reinterpret_cast<int64_t*>(coef_base) + off * kBlock + threadIdx.x;
}

constexpr int kCoefEntries = 8 + 4;  // K = 4: levels 1 and 2
// Coefficient entries per thread: every suffix level's column, or only the
// innermost pair's (4) when the sweep folds latency lazily.
__host__ __device__ constexpr int coef_entries(bool lazy) { return lazy ? 4 : kCoefEntries; }

// The suffix-level-J input coefficient vector (entries 0..3 are all the
// innermost pair needs), folded from the row's level-0 vector through the
// digits of suffix levels 0..J-1.  Energy-first sweeps need latency only in
// flagged contexts, so they skip the per-level folds and call this instead.
// Energy-first sweeps (register / parameter innermost table) fold latency
// coefficients only for flagged contexts.
template <int PRIM, int NV>
constexpr bool kLazyCoef = PRIM == kPrimFp && NV > 0 && LOOM_ENERGY_FIRST;

// level(): sweep normally, or (paired sweeps, see level K-3) only handle the
// given flagged steps of an already swept node -- no sweep, no warp sync.
constexpr uint32_t kNoPreHits = 0xffffffffu;

template <int K>
__device__ __noinline__ void lazy_coef(const int64_t* c0, const int64_t* wall, const int32_t* optoff, int P, int J,
                                       int o0, int o1, int64_t* out) {
  int64_t v[1 << K];
#pragma unroll
  for (int S = 0; S < (1 << K); ++S) v[S] = c0[S];
  int ns = 1 << K;
  for (int jj = 0; jj < J; ++jj) {
    const int64_t w = wall[optoff[P + jj] + (jj == 0 ? o0 : o1)];
    ns >>= 1;
    for (int S = 0; S < ns; ++S) v[S] = max(v[2 * S], v[2 * S + 1] + w);
  }
  for (int S = 0; S < 4; ++S) out[S * kBlock] = v[S];  // the level's coefficient column
}

template <int K, int PRIM, int NV, bool PT, int J>
__device__ __forceinline__ void level(Hot& H, const Inner<K, PRIM, NV, PT>& in, const InnerParams& ip, double ea,
                                      int32_t qv, uint64_t lex,
                                      int o_lo, int o_hi, uint64_t ibase, uint32_t pre_hits = kNoPreHits) {
  const int node = H.P + J;
  const int off = H.optoff[node];
  const int n = H.radix[node];
  // level 0 reads the thread's local vector (stride 1), deeper levels their
  // shared-memory column (stride kBlock)
  constexpr int SI = J == 0 ? 1 : kBlock;
  const int64_t* cin = J == 0 ? H.c0 : coef_col<K>(H.coef_base, J, kLazyCoef<PRIM, NV>);
  if constexpr (J == K - 2) {
    const int n_in = H.radix[node + 1];
    const int64_t wmin = H.h->inner_wmin, wu_max = H.h->pre_wmax;
    // The pair's coefficient vector is the level's input column; lazy
    // (energy-first) sweeps fill that column on the first flagged context.
    PreInner pr{};
    bool have_c = !kLazyCoef<PRIM, NV>;
    auto cvec = [&]() {
      const int64_t cc[4] = {cin[0], cin[SI], cin[2 * SI], cin[3 * SI]};
      pr = pre_inner(cc, H.lat_s, wmin, wu_max);
    };
    if constexpr (!kLazyCoef<PRIM, NV>) cvec();
    auto need_c = [&]() {
      if constexpr (kLazyCoef<PRIM, NV>) {
        if (!have_c) {
          if (J > 0) lazy_coef<K>(H.c0, H.wall, H.optoff, H.P, J, H.od[0], H.od[1], const_cast<int64_t*>(cin));
          cvec();
          have_c = true;
        }
      }
    };
    // Exact slow path of one context (rare).
    auto context_slow = [&](int o, double eu, int32_t qu, int32_t tw, int g0) {
      H.od[J] = o;
      // plan index of option 0 of the innermost node in this context; at J == 0
      // the digit o is already part of the subrow index
      const uint64_t inner_base =
          J == 0 ? 0 : (ibase * static_cast<uint64_t>(n) + static_cast<uint64_t>(o)) * static_cast<uint64_t>(n_in);
      const int64_t w_real = H.wall[off + o];
      const int64_t X = max(cin[0], cin[SI] + w_real), Y = max(cin[2 * SI], cin[3 * SI] + w_real);
      const uint64_t lex_u = lex + H.lexw[off + o];
      slow_scan<K, PRIM>(H.smem, H.slot_base, H.dpre, H.P, H.od[0], H.od[1], H.od[2], g0, g0 + (NV > 0 ? NV : 8), tw,
                         eu, qu, lex_u, X, Y, H.s_index * H.h->r_sub + inner_base);
      reload(H);  // the latency bound may have tightened (latency primary, or an energy tie at the floor)
      cvec();
    };
    if constexpr (NV > 0) {
      // Two contexts per step share the innermost table: twice the
      // independent DADD -> DSETP chains per warp.  The step loop holds no
      // call, so the table stays in uniform registers across steps: a step
      // whose contexts may hold a plan that ties or beats the running best
      // only sets its bit in `hits`, and those contexts are re-tested (with
      // the then-current thresholds) and scanned exactly after the loop.
      // Testing with thresholds older than the running best only lets more
      // contexts through, so no candidate is lost.
      // Energy-first (PRIM == kPrimFp): one compare per plan on the primary
      // criterion (any_energy2); other objectives test both criteria per plan.
      constexpr bool ef = kLazyCoef<PRIM, NV>;
      // Flagged steps: the two-criteria bound test per context, then the
      // exact test, then the exact scan.  The step loop holds no call, so
      // the table stays in uniform registers across steps; testing with
      // thresholds older than the running best only lets more through.
      auto flagged = [&](uint32_t hits, int c_lo, int c_hi) {
        while (__builtin_expect(hits != 0, 0)) {
          const int p = __ffs(hits) - 1;
          hits &= hits - 1;
          need_c();
          for (int oo = c_lo + 2 * p; oo < min(c_hi, c_lo + 2 * p + 2); ++oo) {
            const double eu = __dadd_rn(ea, H.ga[off + oo]);
            const int32_t tw = inner_tw(pr, H.w32[off + oo]);
            const double tu = ctx_bound(H, eu);
            bool b = false;
#pragma unroll
            for (int j = 0; j < NV; ++j) b |= in.pass_bound(in.W(ip, j), in.G(ip, j), tw, tu);
            if (b) LOOM_COUNT(1, 1);
            if (b && in.any_pass(H, ip, tw, eu, INT_MAX)) {
              LOOM_COUNT(2, 1);
              context_slow(oo, eu, INT_MAX, tw, 0);
            }
          }
        }
      };
      if (pre_hits != kNoPreHits) {  // flagged steps of a paired sweep (level K-3)
        flagged(pre_hits, 0, NV);
        return;
      }
      if (ef && n == NV && o_lo == 0 && o_hi == NV) {
        // The whole node above the innermost, radix == NV: one fully
        // unrolled sweep of NV/2 steps, branch-free step flags.
        uint32_t hits = 0;
#pragma unroll
        for (int st = 0; st < NV / 2; ++st) {
          // kernel-parameter launches read the node's terms from the constant bank
          const double gu0 = PT ? ip.gu[2 * st] : H.ga[off + 2 * st];
          const double gu1 = PT ? ip.gu[2 * st + 1] : H.ga[off + 2 * st + 1];
          const double eu0 = __dadd_rn(ea, gu0), eu1 = __dadd_rn(ea, gu1);
          hits |= static_cast<uint32_t>(in.any_energy2(ip, ctx_bound(H, eu0), ctx_bound(H, eu1))) << st;
        }
        LOOM_COUNT(3, NV / 2);
        LOOM_COUNT(0, __popc(hits));
        flagged(hits, 0, NV);
      } else {
        for (int c_lo = o_lo; c_lo < o_hi; c_lo += 64) {
          const int c_hi = min(o_hi, c_lo + 64);
          uint32_t hits = 0, bit = 1;
          int o = c_lo;
          if constexpr (ef) {
#pragma unroll kPairUnroll
            for (; o + 1 < c_hi; o += 2, bit <<= 1) {
              const double eu0 = __dadd_rn(ea, H.ga[off + o]), eu1 = __dadd_rn(ea, H.ga[off + o + 1]);
              const bool a = in.any_energy2(ip, ctx_bound(H, eu0), ctx_bound(H, eu1));
              if (__builtin_expect(a, 0)) {
                asm volatile("");
                hits |= bit;
              }
            }
            LOOM_COUNT(3, (c_hi - c_lo) / 2);
            LOOM_COUNT(0, __popc(hits));
          } else {
#pragma unroll kPairUnroll
            for (; o + 1 < c_hi; o += 2, bit <<= 1) {
              const int32_t wu0 = H.w32[off + o], wu1 = H.w32[off + o + 1];
              const double eu0 = __dadd_rn(ea, H.ga[off + o]), eu1 = __dadd_rn(ea, H.ga[off + o + 1]);
              const int32_t tw0 = inner_tw(pr, wu0), tw1 = inner_tw(pr, wu1);
              const double tu0 = ctx_bound(H, eu0), tu1 = ctx_bound(H, eu1);
              bool a = false;
#pragma unroll
              for (int j = 0; j < NV; ++j) {
                a |= in.pass_bound(in.W(ip, j), in.G(ip, j), tw0, tu0);
                a |= in.pass_bound(in.W(ip, j), in.G(ip, j), tw1, tu1);
              }
              // a real (rarely taken) branch keeps the per-plan tests a predicate
              // OR chain; the empty asm stops if-conversion into per-plan selects
              if (__builtin_expect(a, 0)) {
                asm volatile("");
                hits |= bit;
              }
            }
          }
          if (o < c_hi) {
            need_c();
            const int32_t wu = H.w32[off + o];
            const double eu = __dadd_rn(ea, H.ga[off + o]);
            if (in.any_pass(H, ip, inner_tw(pr, wu), eu, INT_MAX)) hits |= bit;
          }
          flagged(hits, c_lo, c_hi);
        }
      }
      // Reconverge after the (divergent) flagged-context work: left alone,
      // the lanes that took the slow path and the ones that did not keep
      // running the step loop as separate groups, issuing it twice.
      if (LOOM_SWEEP_SYNC) {
        if (H.sync_mask == 0xffffffffu) __syncwarp();
        else __syncwarp(H.sync_mask);
      }
    } else {
      for (int o = o_lo; o < o_hi; ++o) {
        const int32_t wu = H.w32[off + o];
        const double eu = __dadd_rn(ea, H.ga[off + o]);
        const int32_t qu = (PRIM == kPrimQual) ? min(qv, H.q[off + o]) : INT_MAX;
        int32_t tw = inner_tw(pr, wu);
        const int g_end = (n_in + 7) & ~7;
        for (int g0 = 0; g0 < g_end; g0 += 8) {
          bool any = false;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const InnerEntry e = H.inner[g0 + j];
            any |= in.pass(H, e.w, e.g, e.q, tw, eu, qu);
          }
          if (__builtin_expect(any, 0)) {
            context_slow(o, eu, qu, tw, g0);
            tw = inner_tw(pr, wu);
          }
        }
      }
      if (LOOM_SWEEP_SYNC) {
        if (H.sync_mask == 0xffffffffu) __syncwarp();
        else __syncwarp(H.sync_mask);
      }
    }
  } else {
    constexpr int NS = 1 << (K - J - 1);
    int64_t* cout = coef_col<K>(H.coef_base, J + 1, kLazyCoef<PRIM, NV>);
    if constexpr (J == K - 3 && kLazyCoef<PRIM, NV> && PT && LOOM_SWEEP_PAIRS) {
      // Paired sweeps: two options of this node per unrolled block (512
      // plans per lane), sharing the per-sweep setup; flagged steps are
      // handed to the child level afterwards, then the warp reconverges once.
      constexpr int GS = LOOM_SWEEP_GROUP;  // options of this node per block
      if (H.radix[node + 1] == NV && (o_hi - o_lo) % GS == 0) {
        for (int o = o_lo; o < o_hi; o += GS) {
          double e2[GS];
          uint32_t hs[GS];
#pragma unroll
          for (int g = 0; g < GS; ++g) {
            e2[g] = __dadd_rn(ea, H.ga[off + o + g]);
            hs[g] = 0;
          }
#pragma unroll
          for (int st = 0; st < NV / 2; ++st)
#pragma unroll
            for (int g = 0; g < GS; ++g)
              hs[g] |= static_cast<uint32_t>(in.any_energy2(ip, ctx_bound(H, __dadd_rn(e2[g], ip.gu[2 * st])),
                                                           ctx_bound(H, __dadd_rn(e2[g], ip.gu[2 * st + 1]))))
                       << st;
          LOOM_COUNT(3, GS * NV / 2);
#pragma unroll
          for (int g = 0; g < GS; ++g) {
            LOOM_COUNT(0, __popc(hs[g]));
            if (__builtin_expect(hs[g] != 0, 0)) {
              H.od[J] = o + g;
              const uint64_t ib = J == 0 ? 0 : ibase * static_cast<uint64_t>(n) + static_cast<uint64_t>(o + g);
              level<K, PRIM, NV, PT, J + 1>(H, in, ip, e2[g], INT_MAX, lex + H.lexw[off + o + g], 0, NV, ib, hs[g]);
            }
          }
          if (LOOM_SWEEP_SYNC) {
            if (H.sync_mask == 0xffffffffu) __syncwarp();
            else __syncwarp(H.sync_mask);
          }
        }
        return;
      }
    }
    for (int o = o_lo; o < o_hi; ++o) {
      if constexpr (!kLazyCoef<PRIM, NV>) {
        const int64_t w = H.wall[off + o];
#pragma unroll
        for (int S = 0; S < NS; ++S) cout[S * kBlock] = max(cin[2 * S * SI], cin[(2 * S + 1) * SI] + w);
      }
      H.od[J] = o;
      const double e2 = __dadd_rn(ea, H.ga[off + o]);
      const int32_t q2 = (PRIM == kPrimQual) ? min(qv, H.q[off + o]) : INT_MAX;
      const uint64_t l2 = lex + H.lexw[off + o];
      const uint64_t ib = J == 0 ? 0 : ibase * static_cast<uint64_t>(n) + static_cast<uint64_t>(o);
      level<K, PRIM, NV, PT, J + 1>(H, in, ip, e2, q2, l2, 0, H.radix[node + 1], ib);
    }
  }
}

// Warp-cooperative longest-path DP for one DP group: lane S computes state S
// (a subset of the KD symbolic suffix nodes) for every node in topological
// order; f lives in per-warp shared memory, so a state of one lane can read
// the predecessor states of another (S without the node's bit).  Output:
// cw[S] = max over nodes of f[x][S], the max-plus coefficient vector.
template <int KD>
__device__ void warp_dp(const View& v, const int* dtop, int Pd, int64_t* fw, int64_t* cw) {
  constexpr int NS = 1 << KD;
  static_assert(NS <= 32, "one state per lane");
  const int S = threadIdx.x & 31;
  const bool act = S < NS;
  const int n = v.h->n_nodes;
  int64_t cmax = kNeg;
  for (int t = 0; t < n; ++t) {
    const int x = v.topo[t];
    const int pb = v.predoff[x], pe = v.predoff[x + 1];
    if (act) {
      int64_t val = kNeg;
      if (x < Pd) {
        int64_t b = S == 0 ? 0 : kNeg;
        for (int e = pb; e < pe; ++e) b = max(b, fw[v.pred[e] * 32 + S]);
        val = b + v.wall[v.optoff[x] + dtop[x]];
      } else {
        const int bit = 1 << (x - Pd);
        if (S & bit) {
          const int S2 = S ^ bit;
          int64_t b = S2 == 0 ? 0 : kNeg;
          for (int e = pb; e < pe; ++e) b = max(b, fw[v.pred[e] * 32 + S2]);
          val = b;
        }
      }
      fw[x * 32 + S] = val;
      cmax = max(cmax, val);
    }
    __syncwarp();
  }
  if (act) cw[S] = S == 0 ? max(cmax, int64_t(0)) : cmax;
  __syncwarp();
}

// Walk subrows [s_begin, s_end) of one DP group.  dtop: the group's digits of
// nodes [0, P-1); cw: the group's coefficient vector over the K+1 suffix
// nodes (P >= 1) or the K suffix nodes (P == 0); (ea, q, lex)_top: folds over
// nodes [0, P-1).  Each row folds the last prefix node's wall into the 2^K
// vector of suffix level 0.
template <int K, int PRIM, int NV, bool PT>
__device__ void run_subrows(const uint8_t* smem, uint8_t* slot_base, uint8_t* coef_base, const View& v,
                            const InnerParams& ip, uint64_t s_begin, uint64_t s_end, const int* dtop, const int64_t* cw,
                            double ea_top, int32_t q_top, uint64_t lex_top) {
  constexpr int NS = 1 << K;
  Hot H;
  H.smem = smem;
  H.slot_base = slot_base;
  H.coef_base = coef_base;
  H.h = v.h;
  H.radix = v.radix;
  H.optoff = v.optoff;
  H.ga = v.ga;
  H.wall = v.wall;
  H.w32 = reinterpret_cast<const int32_t*>(smem + v.h->off_w32);
  H.q = v.q;
  H.lexw = v.lexw;
  H.inner = v.inner;
  H.P = v.h->n_nodes - K;
  H.od[0] = H.od[1] = H.od[2] = H.od[3] = 0;
  reload(H);
  Inner<K, PRIM, NV, PT> in;
  in.load(H);

  const int P = H.P;
  const uint64_t n0 = static_cast<uint64_t>(v.radix[P]);
  int d[kMaxNodes];
  H.dpre = d;
  for (int i = 0; i + 1 < P; ++i) d[i] = dtop[i];
  int o0 = static_cast<int>(s_begin % n0);
  if (P >= 1) d[P - 1] = static_cast<int>((s_begin / n0) % static_cast<uint64_t>(v.radix[P - 1]));
  int64_t c0[NS];  // written once per row, read once per subrow
  H.c0 = c0;
  double ea_pre = 0.0;
  int32_t q_pre = INT_MAX;
  uint64_t lex_pre = 0;
  bool fresh_row = true;
  // Every lane of the warp runs the same number of steps (lanes with fewer
  // subrows idle through the last one), so the sweeps can reconverge with
  // __syncwarp(sync_mask).
  const unsigned n_mine = static_cast<unsigned>(s_end - s_begin);
  const unsigned n_steps = __reduce_max_sync(0xffffffffu, n_mine);
  uint64_t s = s_begin;
  for (unsigned step = 0; step < n_steps; ++step) {
    H.sync_mask = __ballot_sync(0xffffffffu, step < n_mine);
    if (step < n_mine) {
      if (fresh_row) {
        if (P == 0) {
#pragma unroll 1
          for (int S = 0; S < NS; ++S) c0[S] = cw[S];
          ea_pre = ea_top;
          q_pre = q_top;
          lex_pre = lex_top;
        } else {
          const int o = v.optoff[P - 1] + d[P - 1];
          const int64_t w = v.wall[o];
#pragma unroll 1
          for (int S = 0; S < NS; ++S) c0[S] = max(cw[2 * S], cw[2 * S + 1] + w);
          ea_pre = __dadd_rn(ea_top, v.ga[o]);
          q_pre = min(q_top, v.q[o]);
          lex_pre = lex_top + v.lexw[o];
        }
        fresh_row = false;
      }
      H.s_index = s;
      level<K, PRIM, NV, PT, 0>(H, in, ip, ea_pre, q_pre, lex_pre, o0, o0 + 1, 0);
      if (static_cast<uint64_t>(++o0) == n0) {  // next row of the group
        o0 = 0;
        fresh_row = true;
        if (P >= 1) ++d[P - 1];
      }
      ++s;
    }
    if (!LOOM_SWEEP_SYNC) __syncwarp(0xffffffffu);
  }
}

// Per-warp DP scratch: f[n][32] and c[32] (int64) per warp.
__host__ __device__ constexpr size_t dp_bytes_per_warp(int n) { return sizeof(int64_t) * 32 * (n + 1); }

__device__ __forceinline__ Rec shfl_rec(const Rec& r, int delta) {
  Rec o;
  o.qa = __shfl_down_sync(0xffffffffu, r.qa, delta);
  o.qb = __shfl_down_sync(0xffffffffu, r.qb, delta);
  o.lat = __shfl_down_sync(0xffffffffu, r.lat, delta);
  o.lexkey = __shfl_down_sync(0xffffffffu, r.lexkey, delta);
  o.index = __shfl_down_sync(0xffffffffu, r.index, delta);
  o.qual = __shfl_down_sync(0xffffffffu, r.qual, delta);
  o.found = __shfl_down_sync(0xffffffffu, r.found, delta);
  return o;
}

// Block-wide min-loc under the objective's total order; result valid in thread 0.
__device__ Rec block_best(Rec r, const BlobHeader* h, Rec* warp_slot) {
  for (int d = 16; d > 0; d >>= 1) {
    const Rec o = shfl_rec(r, d);
    if (rec_better(o, r, h)) r = o;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) warp_slot[warp] = r;
  __syncthreads();
  if (warp == 0) {
    r = lane < kBlock / 32 ? warp_slot[lane] : Rec{0, 0, 0, 0, 0, 0, 0};
    for (int d = 16; d > 0; d >>= 1) {
      const Rec o = shfl_rec(r, d);
      if (rec_better(o, r, h)) r = o;
    }
  }
  __syncthreads();
  return r;
}

__device__ __forceinline__ Rec load_rec_cg(const Rec* p) {
  Rec r;
  r.qa = __ldcg(&p->qa);
  r.qb = __ldcg(&p->qb);
  r.lat = __ldcg(&p->lat);
  r.lexkey = __ldcg(reinterpret_cast<const unsigned long long*>(&p->lexkey));
  r.index = __ldcg(reinterpret_cast<const unsigned long long*>(&p->index));
  r.qual = __ldcg(&p->qual);
  r.found = __ldcg(&p->found);
  return r;
}

template <int K, int PRIM, int NV, bool PT>
__global__ void __launch_bounds__(kBlock, PT ? LOOM_PT_CTAS : 512 / kBlock)
    search_kernel(const uint8_t* __restrict__ arena, const JobDesc* __restrict__ jobs, int ctas_per_job,
                  Rec* __restrict__ scratch, JobSync* __restrict__ sync, Rec* __restrict__ out,
                  const InnerParams ip) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t mbar;
  __shared__ Rec warp_slot[kBlock / 32];
  __shared__ int am_last;

  const int job = blockIdx.x / ctas_per_job;
  const int part = blockIdx.x % ctas_per_job;
  // After a branch-and-bound launch (bnb.cuh) on the same job: kBnbDone ->
  // its result stands and this launch only retires; kBnbAborted -> search
  // exhaustively, starting from its best plan.
  const unsigned bnb_state = __ldcg(&sync[job].pad);
  if (bnb_state == kBnbDone) {
    if (threadIdx.x == 0 && atomicAdd(&sync[job].ticket, 1u) == static_cast<unsigned>(ctas_per_job - 1)) {
      sync[job].ticket = 0;
      sync[job].pad = 0;
    }
    return;
  }
  const JobDesc jd = jobs[job];
  if (threadIdx.x == 0) s_gbest = LOOM_JOB_BOUND ? &sync[job].best_neg : nullptr;
  load_blob(smem, arena + jd.blob_off, jd.blob_bytes, &mbar);  // (its __syncthreads publishes s_gbest)
  const View v = make_view(smem);
  const BlobHeader* h = v.h;
  uint8_t* slot_base = smem + ((jd.blob_bytes + 127) & ~127u);
  const Slots sl = make_slots(slot_base);
  slot_init(sl, threadIdx.x, h);
  if (jd.has_seed) {
    Rec c;
    full_eval(v, jd.seed, c);
    slot_offer(sl, threadIdx.x, h, c);
  }
  if (bnb_state == kBnbAborted || bnb_state == kBfsOverflow) slot_offer(sl, threadIdx.x, h, load_rec_cg(&out[job]));

  const uint64_t gt = static_cast<uint64_t>(part) * kBlock + threadIdx.x;
  const uint64_t nt = static_cast<uint64_t>(ctas_per_job) * kBlock;

  // Range edges (and whole problems on the full-evaluation path).
  for (uint64_t i = jd.begin + gt; i < jd.head_end; i += nt) {
    Rec c;
    full_eval(v, i, c);
    slot_offer(sl, threadIdx.x, h, c);
  }
  for (uint64_t i = jd.tail_begin + gt; i < jd.end; i += nt) {
    Rec c;
    full_eval(v, i, c);
    slot_offer(sl, threadIdx.x, h, c);
  }

  // Whole subrows.  Work is dealt to warps in DP groups (all subrows sharing
  // the digits above the last prefix node, h->group subrows); the 32 lanes
  // of a warp split each group into contiguous runs, so the row DP and the
  // row folds happen in lockstep across the warp instead of divergently.
  if (jd.sub_hi > jd.sub_lo) {
    const uint64_t G = h->group;
    const uint64_t g_first = jd.sub_lo / G, g_end = (jd.sub_hi - 1) / G + 1;
    const uint64_t lane = threadIdx.x & 31;
    uint8_t* coef_base = slot_base + kSlotBytes * kBlock;
    uint8_t* dp_base = coef_base + sizeof(int64_t) * coef_entries(kLazyCoef<PRIM, NV>) * kBlock;
    int64_t* fw = reinterpret_cast<int64_t*>(dp_base + dp_bytes_per_warp(h->n_nodes) * (threadIdx.x >> 5));
    int64_t* cw = fw + 32 * h->n_nodes;
    const int P = h->n_nodes - K;
    // Groups are dealt to warps dynamically (one 64-bit atomic per group):
    // the exact slow path is data dependent, so a static split would leave
    // warps idle at the end.
    auto next_group = [&]() -> uint64_t {
      unsigned long long x = 0, gb = 0;
      if (lane == 0) {
        x = atomicAdd(&sync[job].next_group, 1ull);
        if (s_gbest) gb = __ldcg(s_gbest);
      }
      x = __shfl_sync(0xffffffffu, x, 0);
      gb = __shfl_sync(0xffffffffu, gb, 0);
      // tighten this thread's energy bound to the job's best bucket
      if (gb != 0) {
        const double hg = hi_of(INT64_MAX - static_cast<int64_t>(gb));
        if (hg < sl.hi[threadIdx.x]) sl.hi[threadIdx.x] = hg;
      }
      return g_first + x;
    };
    for (uint64_t g = next_group(); g < g_end; g = next_group()) {
      // digits of nodes [0, P-1) shared by the group, and their folds
      int dtop[kMaxNodes];
      uint64_t x = g;
      for (int i = P - 2; i >= 0; --i) {
        const uint64_t r = static_cast<uint64_t>(v.radix[i]);
        dtop[i] = static_cast<int>(x % r);
        x /= r;
      }
      double ea_top = 0.0;
      int32_t q_top = INT_MAX;
      uint64_t lex_top = 0;
      for (int i = 0; i + 1 < P; ++i) {
        const int o = v.optoff[i] + dtop[i];
        ea_top = __dadd_rn(ea_top, v.ga[o]);
        q_top = min(q_top, v.q[o]);
        lex_top += v.lexw[o];
      }
      if (P >= 1) warp_dp<K + 1>(v, dtop, P - 1, fw, cw);
      else warp_dp<K>(v, dtop, 0, fw, cw);
      const uint64_t lo = max(g * G, jd.sub_lo), hi = min((g + 1) * G, jd.sub_hi);
      const uint64_t len = hi - lo;
      const uint64_t a = lo + len * lane / 32, b = lo + len * (lane + 1) / 32;
      // every lane enters (an empty run just joins the warp's step syncs)
      run_subrows<K, PRIM, NV, PT>(smem, slot_base, coef_base, v, ip, a, b, dtop, cw, ea_top, q_top, lex_top);
      __syncwarp();
    }
  }

  Rec b = block_best(slot_load(sl, threadIdx.x), h, warp_slot);
  if (threadIdx.x == 0) {
    scratch[blockIdx.x] = b;
    __threadfence();
    const unsigned t = atomicAdd(&sync[job].ticket, 1u);
    am_last = (t == static_cast<unsigned>(ctas_per_job - 1));
  }
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
      sync[job].ticket = 0;
      sync[job].pad = 0;
      sync[job].next_group = 0;
      sync[job].best_neg = 0;
    }
  }
}

using KernelFn = void (*)(const uint8_t*, const JobDesc*, int, Rec*, JobSync*, Rec*, InnerParams);

#include "bnb.cuh"
#include "frontier.cuh"


// pt: the innermost table comes from the kernel parameter (single-problem
// launches); batch launches read it per job from shared memory.
template <int K>
KernelFn pick_nv(int prim, int nv, bool pt) {
  if (prim == kPrimQual) return search_kernel<K, kPrimQual, 0, false>;
  if (prim == kPrimFp) {
    if (nv == 8) return pt ? search_kernel<K, kPrimFp, 8, true> : search_kernel<K, kPrimFp, 8, false>;
    if (nv == 16) return pt ? search_kernel<K, kPrimFp, 16, true> : search_kernel<K, kPrimFp, 16, false>;
    return search_kernel<K, kPrimFp, 0, false>;
  }
  if (nv == 8) return pt ? search_kernel<K, kPrimLat, 8, true> : search_kernel<K, kPrimLat, 8, false>;
  if (nv == 16) return pt ? search_kernel<K, kPrimLat, 16, true> : search_kernel<K, kPrimLat, 16, false>;
  return search_kernel<K, kPrimLat, 0, false>;
}

KernelFn pick_kernel(int K, int prim, int nv, bool pt) {
  if (K == 2) return pick_nv<2>(prim, nv, pt);
  if (K == 3) return pick_nv<3>(prim, nv, pt);
  return pick_nv<4>(prim, nv, pt);
}

// Dynamic shared memory of a launch: problem image + per-thread slots.
// (coefficient columns sized for K = 4: 8 + 4 entries per thread)
// + per-warp DP scratch
size_t smem_bytes(size_t blob, int n_nodes, bool lazy) {
  return ((blob + 127) & ~size_t(127)) + static_cast<size_t>(kSlotBytes) * kBlock +
         sizeof(int64_t) * coef_entries(lazy) * kBlock + dp_bytes_per_warp(n_nodes) * (kBlock / 32);
}

// ---------------------------------------------------------------------------
// Threads per CTA of the Pareto kernels (independent of the search kernel's).
constexpr int kPBlock = 256;

// Pareto frontier (pareto_filter, optimizer.hpp:153-171, over estimate(p) for
// every plan p in ConfigEnumerator order).  Dominance: a <= b on dollars,
// gpu_wh (raw doubles) and latency, a.quality >= b.quality, one strict.
//   phase 1  every plan is evaluated (dollars and energy folds in dag order,
//            max-plus latency, quality min) and tested against a guard set of
//            real frontier candidates in shared memory; survivors are
//            appended with warp-ballot compaction.  A plan dominated by a
//            guard point is dominated (the guard points are plans).
//   phase 2  exact pairwise filter over the survivors: any dominator of a
//            survivor is itself a survivor (transitivity), so this is exact.
// ---------------------------------------------------------------------------
constexpr int kGuardMax = 2048;

__device__ __forceinline__ bool dominates(double ad, double ae, int64_t al, int32_t aq, double bd, double be,
                                          int64_t bl, int32_t bq) {
  return ad <= bd && ae <= be && al <= bl && aq >= bq && (ad < bd || ae < be || al < bl || aq > bq);
}

struct GuardView {
  const double* d;
  const double* e;
  const int64_t* l;
  const int32_t* q;
  int n;
};

// Four guard points per step: independent compare chains and one branch per
// four points (most points do not dominate, so the scan usually runs to the
// end; one point per step was latency-bound on the compare -> branch chain).
__device__ __forceinline__ int guard_scan(const GuardView& g, int k0, double d, double e, int64_t l, int32_t q) {
  int k = k0;
  for (; k + 4 <= g.n; k += 4) {
    const bool a0 = dominates(g.d[k], g.e[k], g.l[k], g.q[k], d, e, l, q);
    const bool a1 = dominates(g.d[k + 1], g.e[k + 1], g.l[k + 1], g.q[k + 1], d, e, l, q);
    const bool a2 = dominates(g.d[k + 2], g.e[k + 2], g.l[k + 2], g.q[k + 2], d, e, l, q);
    const bool a3 = dominates(g.d[k + 3], g.e[k + 3], g.l[k + 3], g.q[k + 3], d, e, l, q);
    if (a0 | a1 | a2 | a3) return a0 ? k : a1 ? k + 1 : a2 ? k + 2 : k + 3;
  }
  for (; k < g.n; ++k)
    if (dominates(g.d[k], g.e[k], g.l[k], g.q[k], d, e, l, q)) return k;
  return -1;
}

__device__ __forceinline__ bool guarded(const GuardView& g, double d, double e, int64_t l, int32_t q) {
  return guard_scan(g, 0, d, e, l, q) >= 0;
}

// Same, trying the previous plan's dominator first (consecutive plans of a
// thread differ in one digit, so the same guard point usually dominates).
__device__ __forceinline__ bool guarded_hint(const GuardView& g, int& hint, double d, double e, int64_t l, int32_t q) {
  if (hint < g.n && dominates(g.d[hint], g.e[hint], g.l[hint], g.q[hint], d, e, l, q)) return true;
  const int k = guard_scan(g, 0, d, e, l, q);
  if (k < 0) return false;
  hint = k;
  return true;
}

// One plan's point from its digits (estimate restated; slot A = gpu_wh,
// slot B = dollars in the Pareto image).
__device__ ParetoPoint eval_point(const View& v, const int* d, uint64_t index) {
  const int n = v.h->n_nodes;
  double e = 0.0, dol = 0.0;
  int32_t q = INT_MAX;
  for (int i = 0; i < n; ++i) {
    const int o = v.optoff[i] + d[i];
    e = __dadd_rn(e, v.ga[o]);
    dol = __dadd_rn(dol, v.gb[o]);
    q = min(q, v.q[o]);
  }
  int64_t fin[kMaxNodes];
  int64_t lat = 0;
  for (int t = 0; t < n; ++t) {
    const int x = v.topo[t];
    int64_t s = 0;
    for (int k = v.predoff[x]; k < v.predoff[x + 1]; ++k) s = max(s, fin[v.pred[k]]);
    fin[x] = s + v.wall[v.optoff[x] + d[x]];
    lat = max(lat, fin[x]);
  }
  return ParetoPoint{index, dol, e, lat, q, 0};
}

__device__ __forceinline__ void decode_digits(const View& v, uint64_t index, int* d) {
  for (int i = v.h->n_nodes - 1; i >= 0; --i) {
    const uint64_t r = static_cast<uint64_t>(v.radix[i]);
    d[i] = static_cast<int>(index % r);
    index /= r;
  }
}

// Warp-aggregated append of the lanes whose `keep` is set.
__device__ __forceinline__ void append_point(bool keep, const ParetoPoint& pt, ParetoPoint* out, uint64_t cap,
                                             unsigned long long* count) {
  const unsigned m = __activemask();
  const unsigned b = __ballot_sync(m, keep);
  if (!b) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(count, static_cast<unsigned long long>(__popc(b)));
  base = __shfl_sync(m, base, leader);
  if (keep) {
    const uint64_t pos = base + __popc(b & ((1u << lane) - 1));
    if (pos < cap) out[pos] = pt;
  }
}

__device__ __forceinline__ GuardView load_guard(uint8_t* s, const ParetoPoint* g, int n) {
  GuardView gv;
  double* d = reinterpret_cast<double*>(s);
  double* e = d + kGuardMax;
  int64_t* l = reinterpret_cast<int64_t*>(e + kGuardMax);
  int32_t* q = reinterpret_cast<int32_t*>(l + kGuardMax);
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    d[k] = g[k].dollars;
    e[k] = g[k].gpu_wh;
    l[k] = g[k].latency_us;
    q[k] = g[k].quality;
  }
  __syncthreads();
  gv.d = d;
  gv.e = e;
  gv.l = l;
  gv.q = q;
  gv.n = n;
  return gv;
}

constexpr size_t kGuardBytes = static_cast<size_t>(kGuardMax) * (8 + 8 + 8 + 4);

// Is the (uniform) point dominated by a guard point?  The warp splits the
// guard: lane l tests points l, l + 32, ...
__device__ __forceinline__ bool guarded_warp(const GuardView& g, double d, double e, int64_t l, int32_t q) {
  bool hit = false;
  for (int k = threadIdx.x & 31; k < g.n && !hit; k += 32) hit = dominates(g.d[k], g.e[k], g.l[k], g.q[k], d, e, l, q);
  return __any_sync(0xffffffffu, hit);
}

// Per-warp shared scratch of the Pareto evaluation: warp_dp's f[n][32] and
// c[32] (int64).
__host__ __device__ constexpr size_t pareto_dp_bytes(int n) { return dp_bytes_per_warp(n) * (kPBlock / 32); }

// Phase 1 over [begin, end).  For n >= 3 the space is cut into groups that
// fix every digit but the last three (x = n-3, u = n-2, w = n-1); groups are
// dealt to warps dynamically.  Each coordinate of a plan is monotone in each
// of its options' own values (FP addition rounds monotonically, latency is a
// max-plus polynomial of the walls, quality a min), so the coordinate-wise
// best point a set of plans can reach -- its corner -- is an exact lower
// bound: a guard point (a real plan) that dominates the corner dominates
// every plan of the set, because each plan is no better than the corner in
// every coordinate (the strict one stays strict).  Pruning goes group ->
// row (x fixed) -> plan; the plans of live rows are evaluated exactly and the
// ones no guard point dominates are appended with warp-ballot compaction.
// Range edges (partial groups) and n < 3 take the one-plan-per-thread path.
__global__ void __launch_bounds__(kPBlock)
    pareto_eval_kernel(const uint8_t* __restrict__ blob_g, uint32_t blob_bytes, uint64_t begin, uint64_t end,
                       const ParetoPoint* __restrict__ guard, int n_guard, ParetoPoint* __restrict__ out,
                       uint64_t cap, unsigned long long* __restrict__ count, unsigned long long* __restrict__ stats,
                       unsigned long long* __restrict__ next_group) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t mbar;
  load_blob(smem, blob_g, blob_bytes, &mbar);
  const View v = make_view(smem);
  uint8_t* guard_base = smem + ((blob_bytes + 127) & ~127u);
  const GuardView gv = load_guard(guard_base, guard, n_guard);
  const int n = v.h->n_nodes;
  const uint64_t gt = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nt = static_cast<uint64_t>(gridDim.x) * blockDim.x;

  uint64_t G = 1, g_lo = 0, g_hi = 0;
  if (n >= 3) {
    G = static_cast<uint64_t>(v.radix[n - 3]) * v.radix[n - 2] * v.radix[n - 1];
    g_lo = (begin + G - 1) / G;
    g_hi = end / G;
  }
  const bool groups = n >= 3 && g_lo < g_hi;
  const uint64_t head_end = groups ? g_lo * G : end, tail_begin = groups ? g_hi * G : end;

  // range edges: one plan per thread
  int d[kMaxNodes];
  for (int part = 0; part < 2; ++part) {
    const uint64_t lo = part == 0 ? begin : tail_begin, hi = part == 0 ? head_end : end;
    for (uint64_t base = lo; base < hi; base += nt) {
      const uint64_t i = base + gt;
      ParetoPoint pt{};
      bool keep = false;
      if (i < hi) {
        decode_digits(v, i, d);
        pt = eval_point(v, d, i);
        keep = !guarded(gv, pt.dollars, pt.gpu_wh, pt.latency_us, pt.quality);
      }
      append_point(keep, pt, out, cap, count);
    }
  }
  if (!groups) return;

  const int x = n - 3, u = n - 2, w = n - 1;
  const int nx = v.radix[x], nu = v.radix[u], nw = v.radix[w];
  const int offx = v.optoff[x], offu = v.optoff[u], offw = v.optoff[w];
  // per-node extremes of the three free nodes (corner terms)
  double gb_min[3] = {INFINITY, INFINITY, INFINITY}, ga_min[3] = {INFINITY, INFINITY, INFINITY};
  int64_t w_min[3] = {INT64_MAX, INT64_MAX, INT64_MAX};
  int32_t q_max[3] = {INT_MIN, INT_MIN, INT_MIN};
  for (int t = 0; t < 3; ++t) {
    const int node = x + t;
    for (int o = v.optoff[node]; o < v.optoff[node + 1]; ++o) {
      gb_min[t] = fmin(gb_min[t], v.gb[o]);
      ga_min[t] = fmin(ga_min[t], v.ga[o]);
      w_min[t] = min(w_min[t], v.wall[o]);
      q_max[t] = max(q_max[t], v.q[o]);
    }
  }
  const int lane = threadIdx.x & 31;
  int64_t* fw = reinterpret_cast<int64_t*>(guard_base + kGuardBytes + dp_bytes_per_warp(n) * (threadIdx.x >> 5));
  int64_t* cw = fw + 32 * n;
  const int row_plans = nu * nw;
  int hint = 0, row_hint = 0;
  unsigned long long st_groups = 0, st_live_groups = 0, st_rows = 0, st_live_rows = 0;

  for (;;) {
    unsigned long long gi = 0;
    if (lane == 0) gi = atomicAdd(next_group, 1ull);
    const uint64_t g = g_lo + __shfl_sync(0xffffffffu, gi, 0);
    if (g >= g_hi) break;
    // digits of nodes [0, x): lane-parallel decode, then shared
    {
      uint64_t r = g;
      int mine = 0;
      for (int i = x - 1; i >= 0; --i) {
        const uint64_t rad = static_cast<uint64_t>(v.radix[i]);
        const int di = static_cast<int>(r % rad);
        r /= rad;
        if (i == lane) mine = di;
      }
      for (int i = 0; i < x; ++i) d[i] = __shfl_sync(0xffffffffu, mine, i & 31);
    }
    double e0 = 0.0, d0 = 0.0;
    int32_t q0 = INT_MAX;
    for (int i = 0; i < x; ++i) {
      const int o = v.optoff[i] + d[i];
      e0 = __dadd_rn(e0, v.ga[o]);
      d0 = __dadd_rn(d0, v.gb[o]);
      q0 = min(q0, v.q[o]);
    }
    warp_dp<3>(v, d, x, fw, cw);  // cw[S], S over subsets of {x (bit 0), u (bit 1), w (bit 2)}
    ++st_groups;
    // group corner
    {
      const double dl = __dadd_rn(__dadd_rn(__dadd_rn(d0, gb_min[0]), gb_min[1]), gb_min[2]);
      const double el = __dadd_rn(__dadd_rn(__dadd_rn(e0, ga_min[0]), ga_min[1]), ga_min[2]);
      int64_t ll = kNeg;
      for (int S = 0; S < 8; ++S) {
        int64_t t = cw[S];
        for (int b = 0; b < 3; ++b)
          if (S >> b & 1) t += w_min[b];
        ll = max(ll, t);
      }
      const int32_t qb = min(q0, min(q_max[0], min(q_max[1], q_max[2])));
      if (guarded_warp(gv, dl, el, ll, qb)) continue;
    }
    ++st_live_groups;
    const uint64_t gbase = g * G;
    for (int r0 = 0; r0 < nx; r0 += 32) {
      // row r0 + lane: x fixed -> 4-entry vector over subsets of {u, w}
      const int ox = r0 + lane;
      const bool has = ox < nx;
      double e1 = 0.0, d1 = 0.0;
      int32_t q1 = INT_MAX;
      int64_t c4[4] = {kNeg, kNeg, kNeg, kNeg};
      bool row_live = false;
      if (has) {
        const int o = offx + ox;
        const int64_t wx = v.wall[o];
        for (int T = 0; T < 4; ++T) c4[T] = max(cw[T << 1], cw[(T << 1) | 1] + wx);
        e1 = __dadd_rn(e0, v.ga[o]);
        d1 = __dadd_rn(d0, v.gb[o]);
        q1 = min(q0, v.q[o]);
        const double dl = __dadd_rn(__dadd_rn(d1, gb_min[1]), gb_min[2]);
        const double el = __dadd_rn(__dadd_rn(e1, ga_min[1]), ga_min[2]);
        const int64_t ll = max(max(c4[0], c4[1] + w_min[1]), max(c4[2] + w_min[2], c4[3] + w_min[1] + w_min[2]));
        const int32_t qb = min(q1, min(q_max[1], q_max[2]));
        row_live = !guarded_hint(gv, row_hint, dl, el, ll, qb);
      }
      st_rows += __popc(__ballot_sync(0xffffffffu, has));
      const unsigned live = __ballot_sync(0xffffffffu, row_live);
      st_live_rows += __popc(live);
      // live rows: the warp splits each row's plans
      for (unsigned m = live; m; m &= m - 1) {
        const int src = __ffs(m) - 1;
        const double re = __shfl_sync(0xffffffffu, e1, src), rd = __shfl_sync(0xffffffffu, d1, src);
        const int32_t rq = __shfl_sync(0xffffffffu, q1, src);
        const int64_t a0 = __shfl_sync(0xffffffffu, c4[0], src), a1 = __shfl_sync(0xffffffffu, c4[1], src);
        const int64_t a2 = __shfl_sync(0xffffffffu, c4[2], src), a3 = __shfl_sync(0xffffffffu, c4[3], src);
        const uint64_t rbase = gbase + static_cast<uint64_t>(r0 + src) * row_plans;
        for (int j0 = 0; j0 < row_plans; j0 += 32) {
          const int j = j0 + lane;
          ParetoPoint pt{};
          bool keep = false;
          if (j < row_plans) {
            const int ou = j / nw, ow = j - ou * nw;
            const int64_t wu = v.wall[offu + ou];
            pt.index = rbase + static_cast<uint64_t>(j);
            pt.latency_us = max(max(a0, a1 + wu), max(a2, a3 + wu) + v.wall[offw + ow]);
            pt.gpu_wh = __dadd_rn(__dadd_rn(re, v.ga[offu + ou]), v.ga[offw + ow]);
            pt.dollars = __dadd_rn(__dadd_rn(rd, v.gb[offu + ou]), v.gb[offw + ow]);
            pt.quality = min(min(rq, v.q[offu + ou]), v.q[offw + ow]);
            keep = !guarded_hint(gv, hint, pt.dollars, pt.gpu_wh, pt.latency_us, pt.quality);
          }
          append_point(keep, pt, out, cap, count);
        }
      }
    }
  }
  if (stats && lane == 0) {  // LOOM_DEBUG: groups, live groups, rows, live rows
    atomicAdd(&stats[0], st_groups);
    atomicAdd(&stats[1], st_live_groups);
    atomicAdd(&stats[2], st_rows);
    atomicAdd(&stats[3], st_live_rows);
  }
}

// Points of an explicit list of plan indices (the guard sample).
__global__ void __launch_bounds__(kPBlock)
    pareto_points_kernel(const uint8_t* __restrict__ blob_g, uint32_t blob_bytes, const uint64_t* __restrict__ idx,
                         uint64_t n, ParetoPoint* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t mbar;
  load_blob(smem, blob_g, blob_bytes, &mbar);
  const View v = make_view(smem);
  int d[kMaxNodes];
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    decode_digits(v, idx[i], d);
    out[i] = eval_point(v, d, idx[i]);
  }
}

// Candidate refinement: keep the candidates no guard point dominates
// (guard points are real plans, so this never drops a frontier point).
__global__ void __launch_bounds__(kPBlock)
    pareto_prefilter_kernel(const ParetoPoint* __restrict__ in, uint64_t n, const ParetoPoint* __restrict__ guard,
                            int n_guard, ParetoPoint* __restrict__ out, unsigned long long* __restrict__ count) {
  extern __shared__ __align__(128) uint8_t smem[];
  const GuardView gv = load_guard(smem, guard, n_guard);
  const uint64_t nt = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t base = 0; base < n; base += nt) {
    const uint64_t i = base + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    ParetoPoint pt{};
    bool keep = false;
    if (i < n) {
      pt = in[i];
      keep = !guarded(gv, pt.dollars, pt.gpu_wh, pt.latency_us, pt.quality);
    }
    append_point(keep, pt, out, n, count);
  }
}

// Phase 2: keep[i] = no j != i dominates point i (tiles staged in smem).
// span > 0: point i is compared only with the points of its own span-sized
// block (a multiple of the CTA size) -- the first stage of a blocked filter,
// exact because frontier(A u B) = frontier(frontier(A) u frontier(B)).
__global__ void __launch_bounds__(kPBlock)
    pareto_filter_kernel(const ParetoPoint* __restrict__ pts, uint64_t n, uint8_t* __restrict__ keep,
                         uint64_t span) {
  constexpr int T = 512;
  __shared__ double sd[T], se[T];
  __shared__ int64_t sl[T];
  __shared__ int32_t sq[T];
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  ParetoPoint me{};
  if (i < n) me = pts[i];
  bool dom = i >= n;
  const uint64_t first = static_cast<uint64_t>(blockIdx.x) * blockDim.x;
  const uint64_t lo = span ? first / span * span : 0;
  const uint64_t hi = span ? min(n, lo + span) : n;
  for (uint64_t t0 = lo; t0 < hi; t0 += T) {
    if (!__syncthreads_or(!dom)) break;  // every point of the block already has a dominator
    for (int k = threadIdx.x; k < T && t0 + k < hi; k += blockDim.x) {
      const ParetoPoint p = pts[t0 + k];
      sd[k] = p.dollars;
      se[k] = p.gpu_wh;
      sl[k] = p.latency_us;
      sq[k] = p.quality;
    }
    __syncthreads();
    const int lim = static_cast<int>(hi - t0 < static_cast<uint64_t>(T) ? hi - t0 : static_cast<uint64_t>(T));
    if (!dom)
      for (int k = 0; k < lim; ++k)
        if (dominates(sd[k], se[k], sl[k], sq[k], me.dollars, me.gpu_wh, me.latency_us, me.quality)) {
          dom = true;
          break;
        }
  }
  if (i < n) keep[i] = !dom;
}

// ---------------------------------------------------------------------------
// greedy_search (optimizer.hpp:227-291): one CTA runs the whole coordinate
// descent.  A node step re-optimizes one node with every other digit fixed;
// the reference scans the node's options sequentially, replacing the best on
// every strict improvement, which under a strict total order ends at the
// argmin over {current, all options} -- computed here in one parallel pass
// (one thread per option, full re-evaluation, block min-loc).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock)
    greedy_kernel(const uint8_t* __restrict__ blob_g, uint32_t blob_bytes, const int32_t* __restrict__ order,
                  const int32_t* __restrict__ seed, int max_sweeps, Rec* __restrict__ out, int* __restrict__ sweeps) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t mbar;
  __shared__ Rec warp_slot[kBlock / 32];
  __shared__ int cur[kMaxNodes];
  __shared__ uint64_t stride[kMaxNodes];
  __shared__ Rec best;
  __shared__ int improved;
  load_blob(smem, blob_g, blob_bytes, &mbar);
  const View v = make_view(smem);
  const BlobHeader* h = v.h;
  const int n = h->n_nodes;
  if (threadIdx.x == 0) {
    uint64_t s = 1;
    for (int i = n - 1; i >= 0; --i) {
      stride[i] = s;
      s *= static_cast<uint64_t>(v.radix[i]);
    }
  }
  if (threadIdx.x < n) cur[threadIdx.x] = seed[threadIdx.x];
  __syncthreads();
  auto index_of = [&](const int* d) {
    uint64_t x = 0;
    for (int i = 0; i < n; ++i) x += static_cast<uint64_t>(d[i]) * stride[i];
    return x;
  };
  if (threadIdx.x == 0) {
    int d[kMaxNodes];
    for (int i = 0; i < n; ++i) d[i] = cur[i];
    Rec c;
    eval_digits(v, d, c, index_of(d));
    best = c;
  }
  __syncthreads();
  int done = 0;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) improved = 0;
    __syncthreads();
    for (int t = 0; t < n; ++t) {
      const int node = order[t];
      const int r = v.radix[node];
      Rec mine{0, 0, 0, 0, 0, 0, 0};
      for (int j = threadIdx.x; j < r; j += blockDim.x) {
        if (j == cur[node]) continue;  // optimizer.hpp:277
        int d[kMaxNodes];
        for (int i = 0; i < n; ++i) d[i] = cur[i];
        d[node] = j;
        Rec c;
        eval_digits(v, d, c, index_of(d));
        if (rec_better(c, mine, h)) mine = c;
      }
      const Rec cand = block_best(mine, h, warp_slot);
      if (threadIdx.x == 0 && rec_better(cand, best, h)) {
        best = cand;
        cur[node] = static_cast<int>((cand.index / stride[node]) % static_cast<uint64_t>(r));
        improved = 1;
      }
      __syncthreads();
    }
    done = sweep + 1;
    if (!improved) break;
  }
  if (threadIdx.x == 0) {
    out[0] = best;
    sweeps[0] = done;
  }
}

// ---------------------------------------------------------------------------
// host: problem image builder
// ---------------------------------------------------------------------------
struct Built {
  std::vector<uint8_t> blob;
  std::vector<int32_t> seed;  // loom_greedy_seed digits (empty: none)
  int K = 2;
  int prim = kPrimFp;
  bool full_only = false;
  int nv = 0;  // innermost radix held in registers (8 / 16) or 0 (shared-memory loop)
  InnerParams ip{};  // innermost table as a kernel parameter (nv > 0)
  uint64_t total = 0;
  uint64_t r_sub = 1;
  uint64_t n_sub = 0;
  int bfs_bits = 0;  // bits of the packed digits of a frontier entry (the frontier search needs <= 64)
};

int align16(int x) { return (x + 15) & ~15; }

// The kernel instantiation a Built picks folds latency lazily (kLazyCoef).
bool lazy_of(const Built& b) { return b.prim == kPrimFp && b.nv > 0 && LOOM_ENERGY_FIRST; }

int build_image(const loom_problem* p, const loom_objective* o, uint64_t target_threads, Built& b) {
  uint64_t total = 0;
  if (int rc = loomi::check_problem(p, &total)) return rc;
  if (total == 0) {  // empty dag or a node without options: nothing to search (optimizer.hpp:117-120)
    b = Built{};
    return LOOM_OK;
  }
  const int n = p->n_nodes;
  if (n > kMaxNodes) return loomi::fail(LOOM_INVALID, "InvalidConfigError: more than 32 dag nodes");
  if (p->n_edges > kMaxEdges) return loomi::fail(LOOM_INVALID, "InvalidConfigError: more than 512 dag edges");
  int n_opts = 0;
  std::vector<int32_t> optoff(n + 1, 0);
  for (int i = 0; i < n; ++i) {
    optoff[i] = n_opts;
    n_opts += p->radix[i];
  }
  optoff[n] = n_opts;
  if (n_opts > kMaxOptions) return loomi::fail(LOOM_INVALID, "InvalidConfigError: more than 6144 options");
  if (!o || o->n_criteria < 0 || o->n_criteria > 4)
    return loomi::fail(LOOM_INVALID, "InvalidConfigError: objective needs 0..4 criteria");

  // criteria -> slots
  int fp_kind[2] = {-1, -1};  // LOOM_MIN_ENERGY / LOOM_MIN_COST_DOLLARS per slot
  int crit[4] = {0, 0, 0, 0};
  for (int i = 0; i < o->n_criteria; ++i) {
    const int c = o->criteria[i];
    if (c == LOOM_MIN_ENERGY || c == LOOM_MIN_COST_DOLLARS) {
      int slot = fp_kind[0] == c ? 0 : fp_kind[1] == c ? 1 : -1;
      if (slot < 0) slot = fp_kind[0] < 0 ? 0 : 1;
      fp_kind[slot] = c;
      crit[i] = slot == 0 ? kFpA : kFpB;
    } else if (c == LOOM_MIN_LATENCY) {
      crit[i] = kLat;
    } else if (c == LOOM_MAX_QUALITY) {
      crit[i] = kQual;
    } else {
      return loomi::fail(LOOM_INVALID, "InvalidConfigError: unknown criterion " + std::to_string(c));
    }
  }
  const int prim = o->n_criteria == 0 ? kPrimLat : crit[0] == kFpA ? kPrimFp : crit[0] == kLat ? kPrimLat : kPrimQual;

  // walls: quality-floor failures become unreachable; W bounds every feasible latency
  int64_t W = 0;
  for (int i = 0; i < n; ++i) {
    int64_t m = 0;
    for (int k = optoff[i]; k < optoff[i + 1]; ++k) {
      if (p->wall_us[k] < 0) return loomi::fail(LOOM_INVALID, "InvalidConfigError: negative wall");
      m = std::max(m, p->wall_us[k]);
    }
    W += m;
    if (W > (int64_t(1) << 50)) return loomi::fail(LOOM_INVALID, "InvalidConfigError: latency bound exceeds 2^50 us");
  }
  const int64_t BIG = W + 1;
  auto floor_ok = [&](int k) { return !o->has_quality_floor || p->quality[k] >= o->quality_floor; };
  int64_t slo_eff = W;
  if (o->has_latency_slo) slo_eff = std::min<int64_t>(o->latency_slo_us, W);

  // K: the deepest suffix that still leaves enough subrows for every thread
  int K = 2;
  uint64_t r_sub = 1;
  bool full_only = n < 2;
  if (!full_only) {
    // Deepest K (<= 4) that still leaves a subrow per thread: the row DP and
    // the upper suffix levels amortise over more plans (measured on C3:
    // K=4 1.29e12 plans/s vs K=3 4.2e11).  LOOM_FORCE_K overrides.
    K = 2;
    for (int k = 3; k <= std::min(4, n); ++k) {
      uint64_t r = 1;
      for (int j = n - k + 1; j < n; ++j) r *= static_cast<uint64_t>(p->radix[j]);
      if (total / r < target_threads) break;
      K = k;
    }
    if (const char* f = std::getenv("LOOM_FORCE_K")) K = std::max(2, std::min({4, n, std::atoi(f)}));
    r_sub = 1;
    for (int j = n - K + 1; j < n; ++j) r_sub *= static_cast<uint64_t>(p->radix[j]);
  }
  // inner walls relative to their minimum must fit int32
  const int inner_node = n - 1;
  int64_t wmin = INT64_MAX, wmax = 0;
  for (int k = optoff[inner_node]; k < optoff[inner_node + 1]; ++k) {
    wmin = std::min(wmin, p->wall_us[k]);
    wmax = std::max(wmax, p->wall_us[k]);
  }
  // exact int32 latency tests need the innermost wall range and the walls of
  // the node above it below 2^30 us (~18 min); larger ones take the
  // one-plan-per-thread path
  int64_t pre_wmax = 0;
  if (n >= 2)
    for (int k = optoff[n - 2]; k < optoff[n - 1]; ++k) pre_wmax = std::max(pre_wmax, p->wall_us[k]);
  if (wmax - wmin >= (int64_t(1) << 30) - 1 || pre_wmax >= (int64_t(1) << 30) - 1) full_only = true;
  const int inner_radix = p->radix[inner_node];
  int nv = inner_radix <= 8 ? 8 : inner_radix <= 16 ? 16 : 0;
  if (const char* f = std::getenv("LOOM_FORCE_NV")) nv = std::atoi(f) == 0 ? 0 : nv;  // experiments

  // topology: Kahn order + predecessor CSR (counting sort of the edges: the
  // edge order is kept within a node; no per-node vectors)
  const int ne = p->n_edges;
  std::vector<int32_t> indeg(n, 0), topo, predoff(n + 1, 0), succoff(n + 1, 0), pred(ne), succ(ne);
  topo.reserve(n);
  for (int e = 0; e < ne; ++e) {
    ++predoff[p->edge_to[e] + 1];
    ++succoff[p->edge_from[e] + 1];
    ++indeg[p->edge_to[e]];
  }
  for (int i = 0; i < n; ++i) {
    predoff[i + 1] += predoff[i];
    succoff[i + 1] += succoff[i];
  }
  {
    std::vector<int32_t> pc(predoff.begin(), predoff.end() - 1), sc(succoff.begin(), succoff.end() - 1);
    for (int e = 0; e < ne; ++e) {
      pred[pc[p->edge_to[e]]++] = p->edge_from[e];
      succ[sc[p->edge_from[e]]++] = p->edge_to[e];
    }
  }
  for (int i = 0; i < n; ++i)
    if (!indeg[i]) topo.push_back(i);
  for (std::size_t t = 0; t < topo.size(); ++t)
    for (int e = succoff[topo[t]]; e < succoff[topo[t] + 1]; ++e)
      if (--indeg[succ[e]] == 0) topo.push_back(succ[e]);
  if (static_cast<int>(topo.size()) != n) return loomi::fail(LOOM_INVALID, "CycleError: dag has a cycle");

  // layout
  BlobHeader hd;
  std::memset(&hd, 0, sizeof hd);
  int off = align16(sizeof(BlobHeader));
  auto take = [&](int bytes) {
    const int at = off;
    off = align16(off + bytes);
    return at;
  };
  hd.off_radix = take(4 * n);
  hd.off_optoff = take(4 * (n + 1));
  hd.off_topo = take(4 * n);
  hd.off_predoff = take(4 * (n + 1));
  hd.off_pred = take(4 * std::max<int>(1, static_cast<int>(pred.size())));
  hd.off_ga = take(8 * n_opts);
  hd.off_gb = take(8 * n_opts);
  hd.off_wall = take(8 * n_opts);
  hd.off_lexw = take(8 * n_opts);
  hd.off_q = take(4 * n_opts);
  const int inner_pad = std::max(nv, (inner_radix + 7) & ~7);
  hd.off_inner = take(static_cast<int>(sizeof(InnerEntry)) * inner_pad);
  hd.off_w32 = take(4 * n_opts);
  hd.off_perm = take(4 * n_opts);
  hd.off_nok = take(4 * n);
  hd.off_bmin = take(static_cast<int>(sizeof(BnbMin)) * n);
  hd.off_rk = take(8 * (n + 1));
  // settled-node lists (bnb.cuh): anc[x] = x and its ancestors; CSR per depth k
  std::vector<int32_t> uns_off(n + 1, 0), uns, ns_off(n + 1, 0), nset;
  {
    uint64_t anc[kMaxNodes] = {};  // n <= 32 nodes: bit sets
    for (int x : topo) {
      anc[x] |= uint64_t(1) << x;
      for (int e = predoff[x]; e < predoff[x + 1]; ++e) anc[x] |= anc[pred[e]];
    }
    auto settled = [&](int x, int k) { return (anc[x] >> k) == 0; };  // every ancestor-or-self < k
    uns.reserve(static_cast<size_t>(n) * n);
    nset.reserve(n);
    for (int k = 0; k < n; ++k) {
      uns_off[k] = static_cast<int32_t>(uns.size());
      ns_off[k] = static_cast<int32_t>(nset.size());
      for (int x : topo) {
        if (!settled(x, k)) uns.push_back(x);
        if (settled(x, k + 1) && !settled(x, k)) nset.push_back(x);
      }
    }
    uns_off[n] = static_cast<int32_t>(uns.size());
    ns_off[n] = static_cast<int32_t>(nset.size());
  }
  auto csr_bytes = [&](const std::vector<int32_t>& data) { return static_cast<int>(4 * (n + 1 + data.size())); };
  hd.off_uns = take(csr_bytes(uns));
  hd.off_nsettle = take(csr_bytes(nset));
  if (off > kMaxBlobBytes) return loomi::fail(LOOM_INVALID, "InvalidConfigError: problem image exceeds shared memory");
  hd.n_nodes = n;
  hd.n_edges = p->n_edges;
  hd.n_opts = n_opts;
  hd.K = K;
  hd.n_crit = o->n_criteria;
  for (int i = 0; i < 4; ++i) hd.crit[i] = crit[i];
  hd.prim = prim;
  for (int i = 0; i < o->n_criteria; ++i)
    if (crit[i] == kFpB || (crit[i] == kQual && prim != kPrimQual)) hd.needs_full = 1;
  hd.bytes = off;
  hd.slo_eff = slo_eff;
  hd.tie_lat = prim == kPrimFp && o->n_criteria >= 2 && crit[1] == kLat && fp_kind[0] >= 0;
  if (hd.tie_lat) {
    const double* a = fp_kind[0] == LOOM_MIN_ENERGY ? p->gpu_wh : p->dollars;
    double x = 0.0;  // dag-order fold of per-node minima (estimator.hpp:50-60): no plan's sum is below it
    for (int i = 0; i < n; ++i) {
      double m = INFINITY;
      for (int k = optoff[i]; k < optoff[i + 1]; ++k) m = std::min(m, a[k]);
      x += m;
    }
    hd.qa_floor = static_cast<int64_t>(std::llround(x * 1e9));
  }
  {
    std::vector<int32_t> sd(n);
    if (loom_greedy_seed(p, o, sd.data()) == LOOM_OK) {
      uint64_t idx = 0;
      for (int i = 0; i < n; ++i) idx = idx * static_cast<uint64_t>(p->radix[i]) + static_cast<uint64_t>(sd[i]);
      hd.has_seed = 1;
      hd.seed_index = idx;
      b.seed = sd;
    }
  }
  hd.inner_wmin = wmin;
  hd.pre_wmax = pre_wmax;
  hd.total = total;
  hd.r_sub = r_sub;
  hd.n_sub = total / r_sub;
  // DP group: subrows that share every digit above the last prefix node
  hd.group = full_only ? 1 : (n - K >= 1 ? static_cast<uint64_t>(p->radix[n - K - 1]) * p->radix[n - K] : hd.n_sub);

  b.blob.assign(off, 0);
  uint8_t* base = b.blob.data();
  std::memcpy(base, &hd, sizeof hd);
  auto put = [&](int at, const void* src, std::size_t bytes) {
    if (bytes) std::memcpy(base + at, src, bytes);
  };
  put(hd.off_radix, p->radix, 4 * n);
  put(hd.off_optoff, optoff.data(), 4 * (n + 1));
  put(hd.off_topo, topo.data(), 4 * n);
  put(hd.off_predoff, predoff.data(), 4 * (n + 1));
  put(hd.off_pred, pred.data(), 4 * pred.size());
  double* ga = reinterpret_cast<double*>(base + hd.off_ga);
  double* gb = reinterpret_cast<double*>(base + hd.off_gb);
  int64_t* wall = reinterpret_cast<int64_t*>(base + hd.off_wall);
  uint64_t* lexw = reinterpret_cast<uint64_t*>(base + hd.off_lexw);
  int32_t* qq = reinterpret_cast<int32_t*>(base + hd.off_q);
  int32_t* w32 = reinterpret_cast<int32_t*>(base + hd.off_w32);
  for (int i = 0; i < n; ++i) {
    for (int k = optoff[i]; k < optoff[i + 1]; ++k) {
      const double* src[2] = {nullptr, nullptr};
      for (int s = 0; s < 2; ++s)
        src[s] = fp_kind[s] == LOOM_MIN_ENERGY ? p->gpu_wh : fp_kind[s] == LOOM_MIN_COST_DOLLARS ? p->dollars : nullptr;
      ga[k] = src[0] ? src[0][k] : 0.0;
      gb[k] = src[1] ? src[1][k] : 0.0;
      wall[k] = floor_ok(k) ? p->wall_us[k] : BIG;
      lexw[k] = static_cast<uint64_t>(p->lexrank[k]) * p->lex_weight[i];
      qq[k] = p->quality[k];
      w32[k] = floor_ok(k) ? static_cast<int32_t>(std::min<int64_t>(p->wall_us[k], int64_t(1) << 30)) : (1 << 30);
    }
  }
  {  // branch-and-bound tables (bnb.cuh)
    int32_t* perm = reinterpret_cast<int32_t*>(base + hd.off_perm);
    int32_t* nok = reinterpret_cast<int32_t*>(base + hd.off_nok);
    BnbMin* bm = reinterpret_cast<BnbMin*>(base + hd.off_bmin);
    uint64_t* rk = reinterpret_cast<uint64_t*>(base + hd.off_rk);
    rk[n] = 1;
    for (int i = n - 1; i >= 0; --i) rk[i] = rk[i + 1] * static_cast<uint64_t>(p->radix[i]);
    auto put_csr = [&](int at, const std::vector<int32_t>& offs, const std::vector<int32_t>& data) {
      int32_t* o = reinterpret_cast<int32_t*>(base + at);  // offsets relative to o, entries after them
      for (int k = 0; k <= n; ++k) o[k] = n + 1 + offs[k];
      std::copy(data.begin(), data.end(), o + n + 1);
    };
    put_csr(hd.off_uns, uns_off, uns);
    put_csr(hd.off_nsettle, ns_off, nset);
    for (int i = 0; i < n; ++i) {
      std::vector<int32_t> ord;
      BnbMin m{INFINITY, INFINITY, INT64_MAX, UINT64_MAX, INT_MIN, -1, {0, 0}};
      for (int k = optoff[i]; k < optoff[i + 1]; ++k) {
        if (!floor_ok(k)) continue;
        if (m.o_wall < 0 || wall[k] < m.w || (wall[k] == m.w && ga[k] < ga[optoff[i] + m.o_wall]))
          m.o_wall = k - optoff[i];
        ord.push_back(k - optoff[i]);
        m.a = std::min(m.a, ga[k]);
        m.b = std::min(m.b, gb[k]);
        m.w = std::min(m.w, wall[k]);
        m.lex = std::min(m.lex, lexw[k]);
        m.q = std::max(m.q, qq[k]);
      }
      // exploration order: best on the primary criterion first (ties: index)
      auto key = [&](int32_t j) -> double {
        const int k = optoff[i] + j;
        if (o->n_criteria == 0) return static_cast<double>(lexw[k]);
        switch (crit[0]) {
          case kFpA: return ga[k];
          case kFpB: return gb[k];
          case kLat: return static_cast<double>(wall[k]);
          default: return -static_cast<double>(qq[k]);
        }
      };
      std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) { return key(x) < key(y); });
      for (std::size_t j = 0; j < ord.size(); ++j) perm[optoff[i] + j] = ord[j];
      nok[i] = static_cast<int32_t>(ord.size());
      bm[i] = m;
    }
  }
  InnerEntry* inner = reinterpret_cast<InnerEntry*>(base + hd.off_inner);
  for (int o2 = 0; o2 < inner_pad; ++o2) {
    if (o2 >= p->radix[inner_node]) {  // padding: can never pass the wall (or the energy) test
      inner[o2].g = INFINITY;
      inner[o2].w = INT_MAX;
      inner[o2].q = INT_MIN;
      continue;
    }
    const int k = optoff[inner_node] + o2;
    // an option failing the quality floor can never pass; an infinite g lets
    // the energy-only fast test see that too (every exact test checks w first)
    inner[o2].g = floor_ok(k) ? ga[k] : INFINITY;
    inner[o2].w = floor_ok(k) ? static_cast<int32_t>(p->wall_us[k] - wmin) : INT_MAX;
    inner[o2].q = p->quality[k];
  }
  b.K = K;
  b.prim = prim;
  b.full_only = full_only;
  b.nv = nv;
  for (int j = 0; j < 16; ++j) {
    const int un = n - 2;  // node above the innermost
    b.ip.gu[j] = (un >= 0 && j < p->radix[un]) ? ga[optoff[un] + j] : 0.0;
    b.ip.g[j] = j < inner_pad ? inner[j].g : INFINITY;
    b.ip.w[j] = j < inner_pad ? inner[j].w : INT_MAX;
    int64_t bits;
    std::memcpy(&bits, &b.ip.g[j], sizeof bits);
    b.ip.gh[j] = static_cast<int32_t>(bits >> 32);
    {  // round down to binary32 (conservative for the <= test)
      float f = static_cast<float>(b.ip.g[j]);
      if (static_cast<double>(f) > b.ip.g[j]) f = std::nextafter(f, -INFINITY);
      b.ip.gf[j] = f;
    }
  }
  b.total = total;
  b.bfs_bits = 0;
  for (int i = 0; i < n; ++i) {
    int bits = 1;
    while ((int64_t(1) << bits) < p->radix[i]) ++bits;
    b.bfs_bits += bits;
  }
  b.r_sub = r_sub;
  b.n_sub = total / r_sub;
  return LOOM_OK;
}

// Splits [begin, end) into whole subrows and edge plans.
// The incumbent of a searched range [begin, end): the greedy seed when it
// lies in the range; otherwise the best feasible of a few in-range plans
// built from it -- the digits the range's ends share, one digit of the first
// node where they differ, the seed's digits below (a shard of a multi-GPU
// search rarely holds the global seed, and a thread with no incumbent flags
// every context until it finds one).  Any feasible plan of the range is a
// valid start: it is a candidate the search would have seen anyway.
void range_seed(const loom_problem* p, const loom_objective* o, const Built& b, JobDesc& d) {
  const int n = p->n_nodes;
  if (b.seed.empty() || d.begin >= d.end || n == 0) return;
  auto index = [&](const std::vector<int32_t>& dg) {
    uint64_t x = 0;
    for (int i = 0; i < n; ++i) x = x * static_cast<uint64_t>(p->radix[i]) + static_cast<uint64_t>(dg[i]);
    return x;
  };
  const uint64_t gs = index(b.seed);
  if (gs >= d.begin && gs < d.end) {
    d.has_seed = 1;
    d.seed = gs;
    return;
  }
  auto digits = [&](uint64_t x) {
    std::vector<int32_t> dg(n);
    for (int i = n - 1; i >= 0; --i) {
      dg[i] = static_cast<int32_t>(x % static_cast<uint64_t>(p->radix[i]));
      x /= static_cast<uint64_t>(p->radix[i]);
    }
    return dg;
  };
  const std::vector<int32_t> db = digits(d.begin), de = digits(d.end - 1);
  int L = 0;
  while (L < n && db[L] == de[L]) ++L;
  loom_winner best{};
  bool have = false;
  auto offer = [&](uint64_t idx) {
    if (idx < d.begin || idx >= d.end) return;
    loom_winner w{};
    w.plan_index = idx;
    if (loomi::fill_winner(p, &w) != LOOM_OK) return;
    w.found = (!o->has_latency_slo || w.latency_us <= o->latency_slo_us) &&
              (!o->has_quality_floor || w.quality >= o->quality_floor);
    if (w.found && (!have || loom_winner_less(&w, &best, o))) {
      best = w;
      have = true;
    }
  };
  if (L == n) {
    offer(d.begin);
  } else {
    std::vector<int32_t> dg = b.seed;
    for (int i = 0; i < L; ++i) dg[i] = db[i];
    const int lo = db[L], hi = de[L];
    const int step = std::max(1, (hi - lo + 1) / 64);  // at most ~64 candidates
    for (int x = lo; x <= hi; x += step) {
      dg[L] = x;
      offer(index(dg));
    }
  }
  if (have) {
    d.has_seed = 1;
    d.seed = best.plan_index;
  }
}

// Search algorithms (loom_search_argmin_algo): branch and bound with the
// sweep as its fallback (default), one plan per thread re-evaluated from
// scratch (cross-check), the hierarchical sweep alone (every plan tested).
constexpr int kAlgoAuto = 0;
constexpr int kAlgoFull = 1;
constexpr int kAlgoSweep = 2;

// incumbent: kNoIncumbent (a plain range search: the start is range_seed's
// in-range plan), LOOM_INCUMBENT_GREEDY (the greedy seed, wherever it lies)
// or a plan index of the space.  An out-of-range incumbent takes part in the
// selection: the result is the argmin of [begin, end) u {incumbent}.
constexpr uint64_t kNoIncumbent = UINT64_MAX - 1;

JobDesc make_desc(const Built& b, uint64_t begin, uint64_t end, bool full_eval_only, const loom_problem* p = nullptr,
                  const loom_objective* o = nullptr, uint64_t incumbent = kNoIncumbent) {
  JobDesc d;
  std::memset(&d, 0, sizeof d);
  end = std::min(end, b.total);
  begin = std::min(begin, end);
  d.begin = begin;
  d.end = end;
  d.blob_bytes = static_cast<uint32_t>(b.blob.size());
  if (incumbent == LOOM_INCUMBENT_GREEDY) {
    const BlobHeader* bh = reinterpret_cast<const BlobHeader*>(b.blob.data());
    d.has_seed = bh->has_seed;
    d.seed = bh->seed_index;
  } else if (incumbent < b.total) {
    d.has_seed = 1;
    d.seed = incumbent;
  } else if (p && o) {
    range_seed(p, o, b, d);
  }
  if (full_eval_only || b.full_only) {
    d.head_end = end;
    d.tail_begin = end;
    return d;
  }
  const uint64_t r = b.r_sub;
  const uint64_t lo = (begin + r - 1) / r, hi = end / r;
  if (lo >= hi) {  // no whole subrow inside the range
    d.head_end = end;
    d.tail_begin = end;
    return d;
  }
  d.sub_lo = lo;
  d.sub_hi = hi;
  d.head_end = lo * r;
  d.tail_begin = hi * r;
  return d;
}

}  // namespace

// ---------------------------------------------------------------------------
// context + C ABI
// ---------------------------------------------------------------------------

namespace {
struct FrPlan;
}

struct loom_device_problem {
  loom_ctx* ctx = nullptr;
  Built built;
  loom_problem host;  // shallow copy; arrays owned below
  std::vector<int32_t> radix, quality, lexrank, efrom, eto;
  std::vector<int64_t> wall;
  std::vector<double> gpu, cpu, dol;
  std::vector<uint64_t> lexw;
  loom_objective objective;
  uint8_t* d_blob = nullptr;
  JobDesc* d_job = nullptr;
  Rec* d_scratch = nullptr;
  JobSync* d_ticket = nullptr;
  Rec* d_out = nullptr;
  Rec* h_out = nullptr;
  int ctas = 0;
  KernelFn fn = nullptr;
  cudaEvent_t done = nullptr;
  BnbSync* d_bsync = nullptr;
  int bnb_ctas = 0;  // 0: the image does not fit the branch-and-bound kernel
  FrPlan* fr = nullptr;  // frontier search plan (variant 0: none)
  JobDesc last_job;      // the JobDesc d_job holds
  bool job_valid = false;
};

namespace {


template <class T>
int ensure(T*& ptr, size_t& cap, size_t need) {
  if (need <= cap && ptr) return LOOM_OK;
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  cap = 0;
  LOOM_CUDA(cudaMalloc(reinterpret_cast<void**>(&ptr), std::max<size_t>(need, 1) * sizeof(T)));
  cap = need;
  return LOOM_OK;
}

int ensure_tickets(loom_ctx* c, size_t need) {
  if (need <= c->tickets_cap && c->d_tickets) return LOOM_OK;
  if (c->d_tickets) cudaFree(c->d_tickets);
  c->d_tickets = nullptr;
  c->tickets_cap = 0;
  LOOM_CUDA(cudaMalloc(&c->d_tickets, std::max<size_t>(need, 1) * sizeof(JobSync)));
  LOOM_CUDA(cudaMemset(c->d_tickets, 0, std::max<size_t>(need, 1) * sizeof(JobSync)));
  c->tickets_cap = need;
  return LOOM_OK;
}

int ensure_bsync(loom_ctx* c, size_t need) {
  if (need <= c->bsync_cap && c->d_bsync) return LOOM_OK;
  if (c->d_bsync) cudaFree(c->d_bsync);
  c->d_bsync = nullptr;
  c->bsync_cap = 0;
  LOOM_CUDA(cudaMalloc(&c->d_bsync, std::max<size_t>(need, 1) * sizeof(BnbSync)));
  LOOM_CUDA(cudaMemset(c->d_bsync, 0, std::max<size_t>(need, 1) * sizeof(BnbSync)));
  c->bsync_cap = need;
  return LOOM_OK;
}

// CTAs of one full wave of the branch-and-bound kernel at this image size
// (0 when its shared memory does not fit: the sweep alone then searches).
// Occupancy queries and shared-memory attributes are driver calls of a few
// microseconds each, and a one-shot search makes several; both are cached
// per (device, kernel, dynamic shared memory).  An attribute already set to
// at least the requested size is not set again.
std::mutex g_occ_mu;
std::map<std::tuple<int, const void*, int, size_t>, int> g_occ;
std::map<std::pair<int, const void*>, size_t> g_smem_set;

cudaError_t smem_attr(const void* fn, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> g(g_occ_mu);
    auto it = g_smem_set.find({dev, fn});
    if (it != g_smem_set.end() && it->second >= smem) return cudaSuccess;
  }
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> g(g_occ_mu);
    size_t& v = g_smem_set[{dev, fn}];
    v = std::max(v, smem);
  }
  return e;
}

// Resident blocks per SM (0: does not fit), shared-memory attribute included.
int blocks_per_sm(const void* fn, int block, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, fn, block, smem);
  {
    std::lock_guard<std::mutex> g(g_occ_mu);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
  }
  int nb = 0;
  if (smem_attr(fn, smem) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, block, smem) != cudaSuccess || nb < 1) {
    cudaGetLastError();
    nb = 0;
  }
  std::lock_guard<std::mutex> g(g_occ_mu);
  g_occ[key] = nb;
  return nb;
}

int bnb_ctas_for(const loom_ctx* c, size_t blob, int n) {
  return c->sms * blocks_per_sm(reinterpret_cast<const void*>(bnb_kernel), kBlock, bnb_smem_bytes(blob, n));
}

// ---------------------------------------------------------------------------
// Frontier search (frontier.cuh): host-built parameters and the launch.
// ---------------------------------------------------------------------------
size_t fr_smem_bytes(size_t blob) {
  static_assert(kFrStage * kFrWarps <= kFrSmall, "per-warp staging lives in the sparse-children slots");
  return ((blob + 127) & ~size_t(127)) + 2 * sizeof(FrontierEntry) * kFrSmall + sizeof(FrPar) * kFrBlock;
}

size_t bfs_cap_entries() {
  static const size_t cap = [] {
    const char* e = std::getenv("LOOM_BFS_CAP");
    return e ? static_cast<size_t>(std::strtoull(e, nullptr, 10)) : (size_t(1) << 23);  // 8M entries x 48 B x 2
  }();
  return cap;
}

int ensure_bfs(loom_ctx* c) {
  if (!c->d_front) {
    LOOM_CUDA(cudaMalloc(&c->d_front, 2 * bfs_cap_entries() * sizeof(FrontierEntry)));
    c->front_cap = bfs_cap_entries();
  }
  if (!c->d_bfs) {
    LOOM_CUDA(cudaMalloc(&c->d_bfs, sizeof(BfsSync)));
    LOOM_CUDA(cudaMemset(c->d_bfs, 0, sizeof(BfsSync)));
  }
  return LOOM_OK;
}

// Directed rounding on the host, exact: the rounding error of a sum (TwoSum)
// or a product (fma) decides whether the nearest result lies above.
double add_rd(double x, double y) {
  const double s = x + y;
  if (!std::isfinite(s)) return s;
  const double bp = s - x;
  const double e = (x - (s - bp)) + (y - bp);
  return e < 0 ? std::nextafter(s, -INFINITY) : s;
}
double mul_rd(double x, double y) {
  const double p = x * y;
  const double e = std::fma(x, y, -p);
  return e < 0 ? std::nextafter(p, -INFINITY) : p;
}

// The exact record of plan `index` (eval_digits restated on the host from the
// problem image: same folds, same order, llround quantization).
Rec host_rec(const Built& b, uint64_t index) {
  const uint8_t* base = b.blob.data();
  const BlobHeader* h = reinterpret_cast<const BlobHeader*>(base);
  const int n = h->n_nodes;
  auto I32 = [&](int off) { return reinterpret_cast<const int32_t*>(base + off); };
  const int32_t *radix = I32(h->off_radix), *optoff = I32(h->off_optoff), *topo = I32(h->off_topo),
                *predoff = I32(h->off_predoff), *pred = I32(h->off_pred), *qq = I32(h->off_q);
  const double* ga = reinterpret_cast<const double*>(base + h->off_ga);
  const double* gb = reinterpret_cast<const double*>(base + h->off_gb);
  const int64_t* wall = reinterpret_cast<const int64_t*>(base + h->off_wall);
  const uint64_t* lexw = reinterpret_cast<const uint64_t*>(base + h->off_lexw);
  int d[kMaxNodes];
  uint64_t x = index;
  for (int i = n - 1; i >= 0; --i) {
    d[i] = static_cast<int>(x % static_cast<uint64_t>(radix[i]));
    x /= static_cast<uint64_t>(radix[i]);
  }
  double ea = 0.0, eb = 0.0;
  int32_t qual = INT_MAX;
  uint64_t lex = 0;
  for (int i = 0; i < n; ++i) {
    const int o = optoff[i] + d[i];
    ea += ga[o];
    eb += gb[o];
    qual = std::min(qual, qq[o]);
    lex += lexw[o];
  }
  int64_t fin[kMaxNodes];
  int64_t lat = 0;
  for (int t = 0; t < n; ++t) {
    const int node = topo[t];
    int64_t st = 0;
    for (int e = predoff[node]; e < predoff[node + 1]; ++e) st = std::max(st, fin[pred[e]]);
    fin[node] = st + wall[optoff[node] + d[node]];
    lat = std::max(lat, fin[node]);
  }
  Rec r{0, 0, lat, lex, index, qual, lat <= h->slo_eff ? 1 : 0};
  if (r.found) {
    r.qa = static_cast<int64_t>(std::llround(ea * 1e9));
    r.qb = static_cast<int64_t>(std::llround(eb * 1e9));
  }
  return r;
}

// Which instantiation a problem takes: <16, int32> when it has at most 16
// nodes and every latency stays below 2^30 us, else <32, int64>.  0: the
// frontier search does not apply (packed digits over 64 bits, or an image too
// large for shared memory next to the frontier slots).
struct FrPlan {
  int variant = 0;
  int cl = 0;  // compile-time criteria list (fr_crit) or 0
  int ctas = 0;
  BfsParams<16> p16;
  BfsParams<32> p32;
  // Search graph of a device problem: frontier kernel -> conditional node
  // {depth-first kernel -> sweep kernel} (taken only on frontier overflow).
  // The winner record is mapped pinned memory, so no copy follows.  One
  // graph launch per search instead of three kernel launches and a copy;
  // rebuilt when the sweep's grid changes.
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphNode_t kn = nullptr;
  cudaGraphConditionalHandle cond = 0;
  int sweep_ctas = -1;
  ~FrPlan() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
  }
};

const void* fr_fn(int variant, int cl) {
  if (variant == 2) return reinterpret_cast<const void*>(bfs_kernel<32, int64_t, 0>);
  switch (cl) {
    case 1: return reinterpret_cast<const void*>(bfs_kernel<16, int32_t, 1>);
    case 2: return reinterpret_cast<const void*>(bfs_kernel<16, int32_t, 2>);
    case 3: return reinterpret_cast<const void*>(bfs_kernel<16, int32_t, 3>);
    default: return reinterpret_cast<const void*>(bfs_kernel<16, int32_t, 0>);
  }
}

// The compile-time criteria list (fr_crit) a blob's objective matches, or 0.
int fr_crit_list(const BlobHeader* h) {
  auto is = [&](std::initializer_list<int> l) {
    if (static_cast<int>(l.size()) != h->n_crit) return false;
    int i = 0;
    for (int c : l)
      if (h->crit[i++] != c) return false;
    return true;
  };
  if (is({kFpA, kLat})) return 1;
  if (is({kLat, kFpA})) return 2;
  if (is({kQual, kFpA, kLat})) return 3;
  return 0;
}

template <int NB>
void fill_fr_params(const Built& b, BfsParams<NB>& P) {
  const uint8_t* base = b.blob.data();
  const BlobHeader* h = reinterpret_cast<const BlobHeader*>(base);
  const int n = h->n_nodes;
  auto I32 = [&](int off) { return reinterpret_cast<const int32_t*>(base + off); };
  const int32_t *radix = I32(h->off_radix), *optoff = I32(h->off_optoff), *topo = I32(h->off_topo),
                *predoff = I32(h->off_predoff), *pred = I32(h->off_pred), *qq = I32(h->off_q),
                *perm = I32(h->off_perm), *nok = I32(h->off_nok);
  const double* ga = reinterpret_cast<const double*>(base + h->off_ga);
  const double* gb = reinterpret_cast<const double*>(base + h->off_gb);
  const int64_t* wall = reinterpret_cast<const int64_t*>(base + h->off_wall);
  const uint64_t* lexw = reinterpret_cast<const uint64_t*>(base + h->off_lexw);
  const BnbMin* bm = reinterpret_cast<const BnbMin*>(base + h->off_bmin);
  const uint64_t* rk = reinterpret_cast<const uint64_t*>(base + h->off_rk);
  std::memset(&P, 0, sizeof P);
  P.n = n;
  P.n_crit = h->n_crit;
  for (int i = 0; i < 4; ++i) P.crit[i] = i < h->n_crit ? h->crit[i] : kFrNone;
  P.slo_eff = h->slo_eff;
  for (int t = 0; t < n; ++t) P.pos[topo[t]] = t;
  int s = 0;
  for (int i = 0; i < n; ++i) {
    int bits = 1;
    while ((int64_t(1) << bits) < radix[i]) ++bits;
    P.shift[i] = s;
    P.bits[i] = static_cast<uint32_t>((uint64_t(1) << bits) - 1);
    s += bits;
    P.optoff[i] = optoff[i];
    P.nok[i] = nok[i];
    P.radix[i] = radix[i];
  }
  std::vector<int32_t> oprim(n), owall(n);
  for (int i = 0; i < n; ++i) {
    oprim[i] = nok[i] ? perm[optoff[i]] : 0;  // exploration order's first: best on the primary criterion
    owall[i] = nok[i] ? bm[i].o_wall : 0;
    const int kp = optoff[i] + oprim[i], kw = optoff[i] + owall[i];
    P.pa[i] = ga[kp];
    P.pb[i] = gb[kp];
    P.pq[i] = qq[kp];
    P.wa[i] = ga[kw];
    P.wb[i] = gb[kw];
    P.wq[i] = qq[kw];
  }
  for (int t = 0; t < n; ++t) {
    const int x = topo[t];
    P.tnode[t] = x;
    for (int e = predoff[x]; e < predoff[x + 1]; ++e) {
      const int pp = P.pos[pred[e]];
      P.pm[t][pp] = ~0u;
      P.sm[pp][t] = ~0u;
    }
    P.tshift[t] = P.shift[x];
    P.tbits[t] = P.bits[x];
    P.toptoff[t] = optoff[x];
    P.twmin[t] = nok[x] ? bm[x].w : 0;
    P.twprim[t] = wall[optoff[x] + oprim[x]];
  }
  {  // distinct qualities of the options meeting the floor, descending (quality-first heuristic)
    std::vector<int32_t> ql;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < nok[i]; ++j) ql.push_back(qq[optoff[i] + perm[optoff[i] + j]]);
    std::sort(ql.begin(), ql.end(), std::greater<int32_t>());
    ql.erase(std::unique(ql.begin(), ql.end()), ql.end());
    P.n_qlev = static_cast<int32_t>(std::min<size_t>(8, ql.size()));
    P.heur = b.total >= (uint64_t(1) << 16);  // a few thousand plans: the levels alone are faster
    for (int i = 0; i < P.n_qlev; ++i) P.qlev[i] = ql[i];
    // lambda grid of the heuristic: 1e-10 .. 1 over its plans (frontier.cuh fr_incumbent)
    P.lam_lo = 1e-10;
    P.lam_log2_span = std::log2(1e10);
  }
  uint64_t lp = 0, lw = 0, ip = 0, iw = 0;
  double sa = 0.0, sb = 0.0, fac = 1.0;
  int32_t sq = INT_MAX;
  uint64_t sl = 0;
  for (int k = n; k >= 0; --k) {
    if (k < n) {
      lp += lexw[optoff[k] + oprim[k]];
      lw += lexw[optoff[k] + owall[k]];
      ip += static_cast<uint64_t>(oprim[k]) * rk[k + 1];
      iw += static_cast<uint64_t>(owall[k]) * rk[k + 1];
      sa = add_rd(sa, bm[k].a);  // (any order: a lower bound of the exact sum; BnbSuf, bnb.cuh)
      sb = add_rd(sb, bm[k].b);
      fac = mul_rd(fac, 1.0 - 0x1.0p-53);
      sq = std::min(sq, bm[k].q);
      sl += bm[k].lex;
    }
    P.lexp_suf[k] = lp;
    P.lexw_suf[k] = lw;
    P.idxp_suf[k] = ip;
    P.idxw_suf[k] = iw;
    P.rk[k] = rk[k];
    P.suf[k] = BnbSuf{sa, sb, fac, sl, sq, 0};
  }
}

template <int NB>
void set_fr_job(const Built& b, const JobDesc& d, BfsParams<NB>& P) {
  P.begin = d.begin;
  P.end = d.end;
  P.ranged = d.begin > 0 || d.end < b.total;
  P.has_seed = d.has_seed != 0;
  P.seed = d.has_seed ? host_rec(b, d.seed) : Rec{0, 0, 0, 0, 0, 0, 0};
  P.seed_dig = 0;
  if (d.has_seed) {  // packed like FrontierEntry.dig
    uint64_t x = d.seed;
    for (int i = P.n - 1; i >= 0; --i) {
      const uint64_t r = static_cast<uint64_t>(P.radix[i]);
      P.seed_dig |= (x % r) << P.shift[i];
      x /= r;
    }
  }
}

// Plan the frontier search of a built problem (variant 0: not applicable).
int prepare_fr(const loom_ctx* c, const Built& b, FrPlan& f) {
  f.variant = 0;
  f.ctas = 0;
  if (b.blob.empty() || b.bfs_bits > 64) return LOOM_OK;
  const BlobHeader* h = reinterpret_cast<const BlobHeader*>(b.blob.data());
  const int n = h->n_nodes;
  if (n < 1) return LOOM_OK;
  // largest latency of a plan of floor-passing options
  const int32_t* optoff = reinterpret_cast<const int32_t*>(b.blob.data() + h->off_optoff);
  const int32_t* perm = reinterpret_cast<const int32_t*>(b.blob.data() + h->off_perm);
  const int32_t* nok = reinterpret_cast<const int32_t*>(b.blob.data() + h->off_nok);
  const int64_t* wall = reinterpret_cast<const int64_t*>(b.blob.data() + h->off_wall);
  int64_t wsum = 0;
  for (int i = 0; i < n; ++i) {
    int64_t m = 0;
    for (int j = 0; j < nok[i]; ++j) m = std::max(m, wall[optoff[i] + perm[optoff[i] + j]]);
    wsum += m;
  }
  const int variant = n <= 16 && wsum < (int64_t(1) << 30) ? 1 : 2;
  const int cl = variant == 1 ? fr_crit_list(h) : 0;
  const size_t smem = fr_smem_bytes(b.blob.size());
  const void* fn = fr_fn(variant, cl);
  const int nb = blocks_per_sm(fn, kFrBlock, smem);
  if (nb < 1) return LOOM_OK;
  f.variant = variant;
  f.cl = cl;
  f.ctas = c->sms * std::min(nb, 1);
  if (variant == 1) fill_fr_params(b, f.p16);
  else fill_fr_params(b, f.p32);
  return LOOM_OK;
}

// Which search the last default launch started with (loom_bnb_last_stats).
std::atomic<int> g_last_default_bfs{0};

// Kernel arguments of the frontier kernel, in its parameter order.
struct FrArgs {
  const uint8_t* blob;
  uint32_t bytes;
  BfsSync* bs;
  FrontierEntry* b0;
  FrontierEntry* b1;
  uint64_t cap;
  Rec* slots;
  JobSync* ticket;
  Rec* out;
  cudaGraphConditionalHandle cond;
  int32_t follow;
  void* params;
  void* ptrs[12];
  void** bind() {
    void* a[12] = {&blob, &bytes, &bs, &b0, &b1, &cap, &slots, &ticket, &out, &cond, &follow, params};
    for (int i = 0; i < 12; ++i) ptrs[i] = a[i];
    return ptrs;
  }
};

int launch_fr(loom_ctx* c, FrPlan& f, const Built& b, const JobDesc& d, const uint8_t* d_blob, Rec* d_slots,
              JobSync* d_ticket, Rec* d_out, int32_t follow = kFollowAlways) {
  if (int rc = ensure_bfs(c)) return rc;
  FrontierEntry* b0 = c->d_front;
  FrontierEntry* b1 = c->d_front + c->front_cap;
  uint64_t cap = c->front_cap;
  BfsSync* bs = c->d_bfs;
  uint32_t bytes = static_cast<uint32_t>(b.blob.size());
  void* pp;
  if (f.variant == 1) {
    set_fr_job(b, d, f.p16);
    pp = &f.p16;
  } else {
    set_fr_job(b, d, f.p32);
    pp = &f.p32;
  }
  cudaGraphConditionalHandle none = 0;
  void* args[] = {&d_blob, &bytes, &bs, &b0, &b1, &cap, &d_slots, &d_ticket, &d_out, &none, &follow, pp};
  LOOM_CUDA(cudaLaunchCooperativeKernel(fr_fn(f.variant, f.cl), dim3(f.ctas), dim3(kFrBlock), args,
                                        fr_smem_bytes(b.blob.size()), c->stream));
  ++c->launches;
  g_last_default_bfs = 1;
  return LOOM_OK;
}

int ensure_host(loom_ctx* c, size_t need) {
  if (need <= c->h_out_cap && c->h_out) return LOOM_OK;
  if (c->h_out) cudaFreeHost(c->h_out);
  c->h_out = nullptr;
  c->h_out_cap = 0;
  LOOM_CUDA(cudaMallocHost(&c->h_out, std::max<size_t>(need, 1) * sizeof(Rec)));
  c->h_out_cap = need;
  return LOOM_OK;
}

int ensure_host_arena(loom_ctx* c, size_t need) {
  if (need <= c->h_arena_cap && c->h_arena) return LOOM_OK;
  if (c->h_arena) cudaFreeHost(c->h_arena);
  c->h_arena = nullptr;
  c->h_arena_cap = 0;
  const size_t cap = std::max<size_t>(need + need / 4, 1 << 20);  // grow with headroom
  LOOM_CUDA(cudaMallocHost(&c->h_arena, cap));
  c->h_arena_cap = cap;
  return LOOM_OK;
}

int set_smem(KernelFn fn, size_t bytes) {
  LOOM_CUDA(smem_attr(reinterpret_cast<const void*>(fn), bytes));
  return LOOM_OK;
}

// Resident CTAs per SM for a kernel instantiation at a given image size.
int resident_ctas(KernelFn fn, size_t smem) {
  return std::max(1, blocks_per_sm(reinterpret_cast<const void*>(fn), kBlock, smem));
}

int ctas_for(const loom_ctx* c, uint64_t work_units, KernelFn fn, size_t smem) {
  // one full wave of resident CTAs (every thread gets an equal contiguous
  // share of subrows), fewer for small spaces
  const uint64_t full = static_cast<uint64_t>(c->sms) * resident_ctas(fn, smem);
  const uint64_t need = (work_units + kBlock - 1) / kBlock;
  return static_cast<int>(std::max<uint64_t>(1, std::min(full, need)));
}

void winner_from_rec(const Rec& r, loom_winner* w) {
  std::memset(w, 0, sizeof *w);
  w->found = r.found;
  w->plan_index = r.index;
  w->lexkey = r.lexkey;
  w->latency_us = r.lat;
  w->quality = r.qual;
}

// Host work over many jobs on up to 32 threads (small batches stay inline).
template <class F>
void parallel_for(int n, F&& f) {
  const int t = n < 64 ? 1 : std::min(32, loomi::host_threads());
  if (t <= 1) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> pool;
  std::atomic<int> next{0};
  for (int w = 0; w < t; ++w)
    pool.emplace_back([&] {
      for (int i; (i = next.fetch_add(64)) < n;)
        for (int k = i; k < std::min(n, i + 64); ++k) f(k);
    });
  for (auto& th : pool) th.join();
}

// LOOM_TRACE=1: phase timings of the host side of a call on stderr.
struct Trace {
  const char* name;
  bool on;
  std::chrono::steady_clock::time_point t0;
  explicit Trace(const char* n) : name(n), on(std::getenv("LOOM_TRACE") != nullptr), t0(std::chrono::steady_clock::now()) {}
  void mark(const char* what) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[loom trace] %s %s %.3f ms\n", name, what,
                 std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

int finish_winner(const loom_problem* p, const Rec& r, loom_winner* out) {
  winner_from_rec(r, out);
  if (!r.found)
    return loomi::fail(LOOM_INFEASIBLE, "NoFeasibleConfigError: no configuration satisfies the quality floor and bounds");
  const int64_t lat = r.lat;
  const uint64_t lex = r.lexkey;
  if (int rc = loomi::fill_winner(p, out)) return rc;
  if (out->latency_us != lat || out->lexkey != lex)
    return loomi::fail(LOOM_DEVICE_ERROR, "DeviceError: kernel winner disagrees with host re-evaluation");
  return LOOM_OK;
}

}  // namespace

extern "C" {

// Experiment builds (LOOM_STATS=1): copy (and optionally reset) the search
// kernel's event counters.  Not part of the public ABI.
int loom_debug_counters(uint64_t* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_stats, sizeof(uint64_t) * 8) != cudaSuccess) return LOOM_DEVICE_ERROR;
  if (reset) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (cudaMemcpyToSymbol(g_stats, z, sizeof z) != cudaSuccess) return LOOM_DEVICE_ERROR;
  }
  return LOOM_OK;
}

int loom_ctx_create(int32_t device, void* cuda_stream, loom_ctx** out) {
  if (!out) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null out");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return loomi::fail(LOOM_DEVICE_ERROR, "DeviceError: no CUDA device available (the B200 path has no CPU fallback)");
  if (device < 0 || device >= count) return loomi::fail(LOOM_INVALID, "InvalidConfigError: bad device ordinal");
  LOOM_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  LOOM_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return loomi::fail(LOOM_DEVICE_ERROR, "DeviceError: sm_100 device required, found sm_" +
                                              std::to_string(prop.major * 10 + prop.minor));
  loom_ctx* c = new loom_ctx;
  c->device = device;
  c->sms = prop.multiProcessorCount;
  if (const char* bud = std::getenv("LOOM_BNB_BUDGET")) {  // test knob (bnb.cuh)
    const unsigned long long v = std::strtoull(bud, nullptr, 10);
    cudaMemcpyToSymbol(g_bnb_budget, &v, sizeof v);
  }
  if (cuda_stream) {
    c->stream = static_cast<cudaStream_t>(cuda_stream);
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete c;
      return loomi::fail(LOOM_DEVICE_ERROR, "DeviceError: cudaStreamCreate failed");
    }
    c->own_stream = true;
  }
  *out = c;
  return LOOM_OK;
}

int loom_ctx_destroy(loom_ctx* c) {
  if (!c) return LOOM_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  cudaFree(c->d_arena);
  cudaFree(c->d_jobs);
  cudaFree(c->d_scratch);
  cudaFree(c->d_tickets);
  cudaFree(c->d_bsync);
  cudaFree(c->d_front);
  cudaFree(c->d_bfs);
  cudaFree(c->d_out);
  for (void* q : c->pool_all) cudaFree(q);
  if (c->h_out) cudaFreeHost(c->h_out);
  if (c->h_arena) cudaFreeHost(c->h_arena);
  if (c->copy_stream) {
    cudaStreamSynchronize(c->copy_stream);
    cudaStreamDestroy(c->copy_stream);
  }
  if (c->copy_done) cudaEventDestroy(c->copy_done);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  return LOOM_OK;
}

uint64_t loom_ctx_launch_count(const loom_ctx* c) { return c ? c->launches : 0; }

void* loom_ctx_stream(const loom_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

namespace {
int search_argmin_impl(loom_ctx* c, const loom_problem* p, const loom_objective* o, uint64_t begin, uint64_t end,
                       int32_t algo, uint64_t incumbent, loom_winner* out);
int search_async_impl(loom_ctx* c, loom_device_problem* dp, uint64_t begin, uint64_t end, uint64_t incumbent,
                      int32_t algo = kAlgoAuto);
}  // namespace

int loom_search_argmin_algo(loom_ctx* c, const loom_problem* p, const loom_objective* o, uint64_t begin,
                            uint64_t end, int32_t algo, loom_winner* out) {
  return search_argmin_impl(c, p, o, begin, end, algo, kNoIncumbent, out);
}

int loom_search_argmin_shard(loom_ctx* c, const loom_problem* p, const loom_objective* o, uint64_t begin,
                             uint64_t end, uint64_t incumbent, loom_winner* out) {
  return search_argmin_impl(c, p, o, begin, end, 0, incumbent, out);
}

int loom_search_argmin_async(loom_ctx* c, loom_device_problem* dp, uint64_t begin, uint64_t end) {
  return search_async_impl(c, dp, begin, end, kNoIncumbent);
}

int loom_search_argmin_shard_async(loom_ctx* c, loom_device_problem* dp, uint64_t begin, uint64_t end,
                                   uint64_t incumbent) {
  return search_async_impl(c, dp, begin, end, incumbent);
}

int loom_search_argmin_algo_async(loom_ctx* c, loom_device_problem* dp, uint64_t begin, uint64_t end,
                                  uint64_t incumbent, int32_t algo) {
  if (algo < kAlgoAuto || algo > kAlgoSweep) return loomi::fail(LOOM_INVALID, "InvalidConfigError: unknown algo");
  return search_async_impl(c, dp, begin, end, incumbent == UINT64_MAX - 1 ? kNoIncumbent : incumbent, algo);
}

// Experiment builds (LOOM_FR_PROF=1): the frontier kernel's phase marks.
int loom_debug_fr_prof(uint64_t* out, int32_t cap) {
  uint64_t buf[8 * (kMaxNodes + 1)];
  if (!out || cudaMemcpyFromSymbol(buf, g_fr_prof, sizeof buf) != cudaSuccess) return LOOM_DEVICE_ERROR;
  for (int i = 0; i < cap && i < 8 * (kMaxNodes + 1); ++i) out[i] = buf[i];
  return LOOM_OK;
}

int loom_debug_fr_prof2(uint64_t* out) {
  return out && cudaMemcpyFromSymbol(out, g_fr_prof2, sizeof(uint64_t) * 16) == cudaSuccess ? LOOM_OK
                                                                                          : LOOM_DEVICE_ERROR;
}

int loom_bfs_trace(uint64_t* out, int32_t cap) {
  if (!out || cap < 2) return LOOM_INVALID;
  uint64_t buf[2 * (kMaxNodes + 2)];
  if (cudaMemcpyFromSymbol(buf, g_bfs_trace, sizeof buf) != cudaSuccess) return LOOM_DEVICE_ERROR;
  for (int i = 0; i < cap && i < 2 * (kMaxNodes + 2); ++i) out[i] = buf[i];
  return LOOM_OK;
}

int loom_bnb_last_stats(uint64_t* out) {
  if (!out) return LOOM_INVALID;
  uint64_t dfs[6] = {0, 0, 0, 0, 0, 0}, bfs[6] = {0, 0, 0, 0, 0, 0};
  if (cudaMemcpyFromSymbol(dfs, g_bnb_last, sizeof dfs) != cudaSuccess ||
      cudaMemcpyFromSymbol(bfs, g_bfs_last, sizeof bfs) != cudaSuccess)
    return LOOM_DEVICE_ERROR;
  if (g_last_default_bfs) {
    const bool of = bfs[1] != 0;  // the depth-first search ran after the frontier search
    out[0] = bfs[0] + (of ? dfs[0] : 0);
    out[1] = (of ? 1u : 0u) | (of && dfs[1] ? 2u : 0u);
    out[2] = bfs[2];
    out[3] = bfs[3];
    out[4] = bfs[4] + (of ? dfs[4] : 0);
    out[5] = of ? dfs[0] : 0;
  } else {
    out[0] = dfs[0];
    out[1] = 1u | (dfs[1] ? 2u : 0u);
    out[2] = dfs[2];
    out[3] = dfs[3];
    out[4] = dfs[4];
    out[5] = dfs[0];
  }
  return LOOM_OK;
}

}  // extern "C"

namespace {

int search_argmin_impl(loom_ctx* c, const loom_problem* p, const loom_objective* o, uint64_t begin, uint64_t end,
                       int32_t algo, uint64_t incumbent, loom_winner* out) {
  if (!c || !p || !o || !out) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  std::memset(out, 0, sizeof *out);
  LOOM_CUDA(cudaSetDevice(c->device));
  Trace tr("search_argmin");
  Built b;
  const uint64_t target = static_cast<uint64_t>(c->sms) * 2 * kBlock;
  if (int rc = build_image(p, o, target, b)) return rc;
  if (b.total == 0)
    return loomi::fail(LOOM_INFEASIBLE, "NoFeasibleConfigError: no configuration satisfies the quality floor and bounds");
  tr.mark("image");
  const JobDesc d = make_desc(b, begin, end, algo == kAlgoFull, p, o, incumbent);
  if (d.begin >= d.end)
    return loomi::fail(LOOM_INFEASIBLE, "NoFeasibleConfigError: no configuration satisfies the quality floor and bounds");
  const uint64_t units = (d.sub_hi - d.sub_lo) + (d.head_end - d.begin) + (d.end - d.tail_begin);
  KernelFn fn = pick_kernel(b.K, b.prim, b.nv, true);
  if (int rc = set_smem(fn, smem_bytes(b.blob.size(), p->n_nodes, lazy_of(b)))) return rc;
  const int ctas = ctas_for(c, units, fn, smem_bytes(b.blob.size(), p->n_nodes, lazy_of(b)));
  const int bctas = algo == kAlgoAuto ? bnb_ctas_for(c, b.blob.size(), p->n_nodes) : 0;
  if (int rc = ensure(c->d_arena, c->arena_cap, b.blob.size())) return rc;
  if (int rc = ensure(c->d_jobs, c->jobs_cap, 1)) return rc;
  if (int rc = ensure(c->d_scratch, c->scratch_cap, static_cast<size_t>(std::max({ctas, bctas, c->sms * 4}))))
    return rc;
  if (int rc = ensure_tickets(c, 1)) return rc;
  if (int rc = ensure_bsync(c, 1)) return rc;
  if (int rc = ensure(c->d_out, c->out_cap, 1)) return rc;
  if (int rc = ensure_host(c, 1)) return rc;
  if (int rc = set_smem(fn, smem_bytes(b.blob.size(), p->n_nodes, lazy_of(b)))) return rc;
  tr.mark("plan + buffers");
  // stage the image and the job descriptor in the pinned arena: async copies
  // without the driver's pageable bounce (the previous call synchronised)
  const size_t job_at = (b.blob.size() + 255) & ~size_t(255);
  if (int rc = ensure_host_arena(c, job_at + sizeof d)) return rc;
  std::memcpy(c->h_arena, b.blob.data(), b.blob.size());
  std::memcpy(c->h_arena + job_at, &d, sizeof d);
  LOOM_CUDA(cudaMemcpyAsync(c->d_arena, c->h_arena, b.blob.size(), cudaMemcpyHostToDevice, c->stream));
  LOOM_CUDA(cudaMemcpyAsync(c->d_jobs, c->h_arena + job_at, sizeof d, cudaMemcpyHostToDevice, c->stream));
  FrPlan fr;
  if (algo == kAlgoAuto) prepare_fr(c, b, fr);
  if (fr.variant) {
    // the frontier search alone; the fallback kernels only if it overflowed
    // (the host waits for the result anyway: one read of JobSync.pad decides)
    if (int rc = launch_fr(c, fr, b, d, c->d_arena, c->d_scratch, c->d_tickets, c->d_out, kFollowHost)) return rc;
    if (int rc = ensure_host(c, 2)) return rc;
    LOOM_CUDA(cudaMemcpyAsync(c->h_out, c->d_out, sizeof(Rec), cudaMemcpyDeviceToHost, c->stream));
    LOOM_CUDA(cudaMemcpyAsync(&c->h_out[1].found, &c->d_tickets[0].pad, sizeof(unsigned), cudaMemcpyDeviceToHost,
                              c->stream));
    LOOM_CUDA(cudaStreamSynchronize(c->stream));
    tr.mark("frontier search");
    if (static_cast<unsigned>(c->h_out[1].found) != kBfsOverflow) return finish_winner(p, c->h_out[0], out);
  } else if (algo == kAlgoAuto) {
    g_last_default_bfs = 0;
  }
  if (bctas) {
    bnb_kernel<<<bctas, kBlock, bnb_smem_bytes(b.blob.size(), p->n_nodes), c->stream>>>(
        c->d_arena, c->d_jobs, bctas, c->d_scratch, c->d_tickets, c->d_bsync, c->d_out);
    LOOM_CUDA(cudaGetLastError());
    ++c->launches;
  }
  fn<<<ctas, kBlock, smem_bytes(b.blob.size(), p->n_nodes, lazy_of(b)), c->stream>>>(c->d_arena, c->d_jobs, ctas, c->d_scratch,
                                                                   c->d_tickets, c->d_out, b.ip);
  LOOM_CUDA(cudaGetLastError());
  ++c->launches;
  LOOM_CUDA(cudaMemcpyAsync(c->h_out, c->d_out, sizeof(Rec), cudaMemcpyDeviceToHost, c->stream));
  tr.mark("copies + launches");
  tr.mark("enqueue");
  LOOM_CUDA(cudaStreamSynchronize(c->stream));
  tr.mark("device");
  return finish_winner(p, c->h_out[0], out);
}

}  // namespace

namespace loomi {

// The batch search (C4): one branch-and-bound CTA per job, then each kernel
// instantiation's sweep retires the jobs it left.  The host side is one pass
// over blocks of jobs: a host thread produces (lowers) a block, builds its
// images, packs them into the pinned arena and queues the block's
// host-to-device copy at once, so the copy of one block overlaps the work on
// the next.  A block takes its arena range with one atomic add; the arena is
// sized from the largest image bytes per job seen before, and blocks past it
// ("late") are staged and copied after the others.
int argmin_batch(loom_ctx* c, int n_jobs, int threads, loom_problem* problems, loom_objective* objectives,
                 const BatchProduce& produce, const BatchRetire& retire, loom_winner* out, int32_t* status) {
  if (n_jobs == 0) return LOOM_OK;
  LOOM_CUDA(cudaSetDevice(c->device));
  Trace tr("argmin_batch");
  constexpr int kJobsPerBlock = 64;
  const int n_blocks = (n_jobs + kJobsPerBlock - 1) / kJobsPerBlock;
  int t = threads > 0 ? threads : std::min(64, loomi::host_threads());
  t = std::max(1, std::min(t, n_blocks));
  size_t hint = std::max<size_t>(c->batch_image_hint, 4096);
  if (const char* h = std::getenv("LOOM_BATCH_HINT")) hint = std::strtoull(h, nullptr, 10);  // test knob: late blocks
  const size_t cap = (hint + hint / 8) * static_cast<size_t>(n_jobs);
  const size_t descs = sizeof(JobDesc) * static_cast<size_t>(n_jobs);
  // every device buffer first: a reallocation later would wait on the copies
  if (int rc = ensure_host_arena(c, ((cap + 255) & ~size_t(255)) + descs)) return rc;
  if (int rc = ensure(c->d_arena, c->arena_cap, cap)) return rc;
  if (int rc = ensure(c->d_jobs, c->jobs_cap, static_cast<size_t>(n_jobs))) return rc;
  if (int rc = ensure(c->d_scratch, c->scratch_cap, static_cast<size_t>(n_jobs))) return rc;
  if (int rc = ensure_tickets(c, static_cast<size_t>(n_jobs))) return rc;
  if (int rc = ensure(c->d_out, c->out_cap, static_cast<size_t>(n_jobs))) return rc;
  if (int rc = ensure_host(c, static_cast<size_t>(n_jobs))) return rc;
  if (int rc = ensure_bsync(c, static_cast<size_t>(n_jobs))) return rc;
  if (c->copy_stream) LOOM_CUDA(cudaStreamSynchronize(c->copy_stream));  // idle unless a call failed midway
  if (!c->copy_stream) LOOM_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  if (!c->copy_done) LOOM_CUDA(cudaEventCreateWithFlags(&c->copy_done, cudaEventDisableTiming));
  // the copy stream starts after everything queued on the ctx's stream
  LOOM_CUDA(cudaEventRecord(c->copy_done, c->stream));
  LOOM_CUDA(cudaStreamWaitEvent(c->copy_stream, c->copy_done, 0));
  tr.mark("buffers");

  std::vector<JobDesc> desc(n_jobs);
  std::vector<KernelFn> kern(n_jobs, nullptr);  // nullptr: the job failed
  std::vector<size_t> smem(n_jobs, 0), bsmem(n_jobs, 0);
  std::vector<uint8_t> late(n_blocks, 0);
  std::vector<std::pair<size_t, std::vector<uint8_t>>> late_pack(n_blocks);  // (arena offset, images)
  std::vector<int> owner(n_blocks, 0);  // the thread that staged a block also finishes it
  std::atomic<size_t> top{0};
  std::atomic<int> next{0}, copy_err{0};
  uint8_t* const h_arena = c->h_arena;
  uint8_t* const d_arena = c->d_arena;
  // Waves of consecutive blocks (8: the last wave's kernels are what remains
  // after the pass): the calling thread launches a wave's
  // searches as soon as its blocks are staged, while the host threads stage
  // the next ones (blocks are taken in order, so waves complete roughly in
  // order).  A wave holding a late block waits for the end of the pass.
  const int n_waves = std::min(n_blocks, 8);
  std::vector<int> wave_of(n_blocks), wave_blk(n_waves + 1);
  for (int k = 0; k <= n_waves; ++k) wave_blk[k] = static_cast<int>(static_cast<int64_t>(n_blocks) * k / n_waves);
  for (int k = 0; k < n_waves; ++k)
    for (int blk = wave_blk[k]; blk < wave_blk[k + 1]; ++blk) wave_of[blk] = k;
  std::unique_ptr<std::atomic<int>[]> wave_left(new std::atomic<int>[n_waves]);
  for (int k = 0; k < n_waves; ++k) wave_left[k].store(wave_blk[k + 1] - wave_blk[k]);
  auto stage = [&](int w) {
    bool device_set = false;
    Built b;                    // reused per job; its image buffer keeps its capacity
    std::vector<uint8_t> pack;  // the block's images back to back
    for (int blk; (blk = next.fetch_add(1)) < n_blocks;) {
      const int lo = blk * kJobsPerBlock, hi = std::min(n_jobs, lo + kJobsPerBlock);
      owner[blk] = w;
      pack.clear();
      for (int j = lo; j < hi; ++j) {
        std::memset(&out[j], 0, sizeof out[j]);
        int rc = produce ? produce(j, w, &problems[j], &objectives[j]) : LOOM_OK;
        if (rc == LOOM_OK) {
          std::vector<uint8_t> keep = std::move(b.blob);
          b = Built{};
          b.blob = std::move(keep);
          b.blob.clear();
          rc = build_image(&problems[j], &objectives[j], kBlock, b);
        }
        if (rc == LOOM_OK && b.total == 0)
          rc = loomi::fail(LOOM_INFEASIBLE,
                           "NoFeasibleConfigError: no configuration satisfies the quality floor and bounds");
        if (status) status[j] = rc;
        if (rc != LOOM_OK) continue;
        kern[j] = pick_kernel(b.K, b.prim, b.nv, false);
        smem[j] = smem_bytes(b.blob.size(), problems[j].n_nodes, lazy_of(b));
        bsmem[j] = bnb_smem_bytes(b.blob.size(), problems[j].n_nodes);
        JobDesc d = make_desc(b, 0, b.total, false);
        if (b.blob.size() && !b.seed.empty()) {  // whole space: the greedy seed is in range
          const BlobHeader* bh = reinterpret_cast<const BlobHeader*>(b.blob.data());
          d.has_seed = bh->has_seed;
          d.seed = bh->seed_index;
        }
        d.blob_off = pack.size();
        desc[j] = d;
        pack.insert(pack.end(), b.blob.begin(), b.blob.end());
      }
      const size_t bytes = pack.size();
      const size_t base = top.fetch_add(bytes);
      for (int j = lo; j < hi; ++j)
        if (kern[j]) desc[j].blob_off += base;
      if (base + bytes > cap) {  // staged after the others
        late[blk] = 1;
        late_pack[blk] = {base, pack};
      } else if (bytes) {
        std::memcpy(h_arena + base, pack.data(), bytes);
        if (!device_set) {
          cudaSetDevice(c->device);
          device_set = true;
        }
        if (cudaMemcpyAsync(d_arena + base, h_arena + base, bytes, cudaMemcpyHostToDevice, c->copy_stream) !=
            cudaSuccess)
          copy_err.store(1);
      }
      wave_left[wave_of[blk]].fetch_sub(1, std::memory_order_release);  // after the copy is queued
    }
  };
  // One wave's searches: descriptors staged in group order after the
  // previous waves', one branch-and-bound launch over the wave, then each
  // group's sweep retires the jobs it left (pointers offset to the wave).
  std::vector<int32_t> slot(n_jobs, -1);  // job -> position in d_jobs / h_out
  size_t pos = 0;
  size_t desc_at = (cap + 255) & ~size_t(255);
  struct Group {
    KernelFn fn;
    std::vector<int> jobs;
    size_t smem = 0;
  };
  auto after_copies = [&]() -> int {  // `stream` waits for the copies queued so far
    LOOM_CUDA(cudaEventRecord(c->copy_done, c->copy_stream));
    LOOM_CUDA(cudaStreamWaitEvent(c->stream, c->copy_done, 0));
    return LOOM_OK;
  };
  auto launch_wave = [&](int k) -> int {
    if (int rc = after_copies()) return rc;
    std::vector<Group> groups;
    size_t bmax = 0;
    const int jlo = wave_blk[k] * kJobsPerBlock, jhi = std::min(n_jobs, wave_blk[k + 1] * kJobsPerBlock);
    for (int j = jlo; j < jhi; ++j) {
      if (!kern[j]) continue;
      Group* g = nullptr;
      for (auto& x : groups)
        if (x.fn == kern[j]) g = &x;
      if (!g) {
        groups.push_back({kern[j], {}, 0});
        g = &groups.back();
      }
      g->jobs.push_back(j);
      g->smem = std::max(g->smem, smem[j]);
      bmax = std::max(bmax, bsmem[j]);
    }
    const size_t p0 = pos;
    JobDesc* staged = reinterpret_cast<JobDesc*>(c->h_arena + desc_at);
    for (auto& g : groups)
      for (int j : g.jobs) {
        staged[pos] = desc[j];
        slot[j] = static_cast<int32_t>(pos++);
      }
    const int nw = static_cast<int>(pos - p0);
    if (!nw) return LOOM_OK;
    LOOM_CUDA(cudaMemcpyAsync(c->d_jobs + p0, staged + p0, nw * sizeof(JobDesc), cudaMemcpyHostToDevice, c->stream));
    if (smem_attr(reinterpret_cast<const void*>(bnb_kernel), bmax) == cudaSuccess) {
      bnb_kernel<<<nw, kBlock, bmax, c->stream>>>(c->d_arena, c->d_jobs + p0, 1, c->d_scratch + p0, c->d_tickets + p0,
                                                  c->d_bsync + p0, c->d_out + p0);
      LOOM_CUDA(cudaGetLastError());
      ++c->launches;
    } else {
      cudaGetLastError();
    }
    size_t first = p0;
    for (auto& g : groups) {
      if (int rc = set_smem(g.fn, g.smem)) return rc;
      const int nj = static_cast<int>(g.jobs.size());
      g.fn<<<nj, kBlock, g.smem, c->stream>>>(c->d_arena, c->d_jobs + first, 1, c->d_scratch + first,
                                               c->d_tickets + first, c->d_out + first, InnerParams{});
      LOOM_CUDA(cudaGetLastError());
      ++c->launches;
      first += nj;
    }
    return LOOM_OK;
  };
  auto wave_late = [&](int k) {
    for (int blk = wave_blk[k]; blk < wave_blk[k + 1]; ++blk)
      if (late[blk]) return true;
    return false;
  };
  int launched = 0, rc_wave = LOOM_OK;
  const std::function<void(int)> stage_fn = stage;
  // host threads unavailable (thread creation failed): the calling thread
  // stages every block, then launches every wave
  const auto pooled = [&](const std::function<void(int)>& f) {
    try {
      c->host.start(t, f);
      return true;
    } catch (const std::system_error&) {
      return false;
    }
  };
  if (t <= 1 || !pooled(stage_fn)) {
    stage(0);
  } else {
    for (; launched < n_waves && rc_wave == LOOM_OK; ++launched) {
      while (wave_left[launched].load(std::memory_order_acquire) > 0)
        std::this_thread::sleep_for(std::chrono::microseconds(10));
      if (copy_err.load() || wave_late(launched)) break;
      rc_wave = launch_wave(launched);
    }
    c->host.wait();  // always: no early return with host threads running
  }
  if (rc_wave != LOOM_OK) return rc_wave;
  if (copy_err.load()) return loomi::fail(LOOM_DEVICE_ERROR, "DeviceError: problem image copy failed");
  const size_t used = top.load();
  int n_ok = 0;
  for (int j = 0; j < n_jobs; ++j) n_ok += kern[j] != nullptr;
  if (n_ok) c->batch_image_hint = std::max(c->batch_image_hint, (used + n_ok - 1) / n_ok);
  if (tr.on) std::fprintf(stderr, "[loom trace] argmin_batch arena %.2f MB (%d jobs, %zu late, %d of %d waves launched during the pass)\n",
                          used / 1e6, n_jobs, static_cast<size_t>(std::count(late.begin(), late.end(), 1)), launched, n_waves);
  tr.mark("produce + images + pack + copy (+ early waves)");
  if (used > cap) {
    // Late blocks: grow both arenas (the staged copies and the launched
    // waves are complete after the syncs), keep the device prefix, stage and
    // copy the late range; the pinned descriptors restart after it.
    LOOM_CUDA(cudaStreamSynchronize(c->copy_stream));
    LOOM_CUDA(cudaStreamSynchronize(c->stream));
    uint8_t* grown = nullptr;
    LOOM_CUDA(cudaMalloc(&grown, used));
    LOOM_CUDA(cudaMemcpyAsync(grown, c->d_arena, cap, cudaMemcpyDeviceToDevice, c->stream));
    LOOM_CUDA(cudaStreamSynchronize(c->stream));
    cudaFree(c->d_arena);
    c->d_arena = grown;
    c->arena_cap = used;
    desc_at = (used + 255) & ~size_t(255);
    if (int rc = ensure_host_arena(c, desc_at + descs)) return rc;
    size_t first = used;
    for (int blk = 0; blk < n_blocks; ++blk) {
      if (!late[blk] || late_pack[blk].second.empty()) continue;
      std::memcpy(c->h_arena + late_pack[blk].first, late_pack[blk].second.data(), late_pack[blk].second.size());
      first = std::min(first, late_pack[blk].first);
    }
    if (first < used)
      LOOM_CUDA(cudaMemcpyAsync(c->d_arena + first, c->h_arena + first, used - first, cudaMemcpyHostToDevice,
                                c->stream));
    tr.mark("late blocks");
  }
  for (; launched < n_waves; ++launched)
    if (int rc = launch_wave(launched)) return rc;
  if (pos) LOOM_CUDA(cudaMemcpyAsync(c->h_out, c->d_out, pos * sizeof(Rec), cudaMemcpyDeviceToHost, c->stream));
  if (int rc = after_copies()) return rc;  // the pinned arena is reused by the next call
  tr.mark("enqueue");
  LOOM_CUDA(cudaStreamSynchronize(c->stream));
  tr.mark("device");
  // Winners re-evaluated and jobs retired on the thread that produced them
  // (a producer's cache shares data between its jobs: no cross-thread
  // reference-count traffic when they are released).
  auto finish = [&](int w) {
    for (int blk = 0; blk < n_blocks; ++blk) {
      if (owner[blk] != w) continue;
      for (int j = blk * kJobsPerBlock; j < std::min(n_jobs, (blk + 1) * kJobsPerBlock); ++j) {
        if (slot[j] >= 0) {
          const int rc = finish_winner(&problems[j], c->h_out[slot[j]], &out[j]);
          if (status) status[j] = rc;
        }
        if (retire) retire(j);
      }
    }
  };
  const std::function<void(int)> finish_fn = finish;
  if (t > 1 && pooled(finish_fn)) {
    c->host.wait();
  } else {
    for (int w = 0; w < t; ++w) finish(w);
  }
  tr.mark("finish");
  return LOOM_OK;
}

}  // namespace loomi

extern "C" {

int loom_search_argmin(loom_ctx* c, const loom_problem* p, const loom_objective* o, uint64_t begin, uint64_t end,
                       loom_winner* out) {
  return loom_search_argmin_algo(c, p, o, begin, end, 0, out);
}

int loom_search_argmin_batch(loom_ctx* c, const loom_problem* problems, const loom_objective* objectives,
                             int32_t n_jobs, loom_winner* out, int32_t* status) {
  if (!c || (!problems && n_jobs) || !objectives || (!out && n_jobs) || n_jobs < 0)
    return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  // read-only without a producer
  return loomi::argmin_batch(c, n_jobs, 0, const_cast<loom_problem*>(problems),
                             const_cast<loom_objective*>(objectives), {}, {}, out, status);
}

int loom_problem_upload(loom_ctx* c, const loom_problem* p, const loom_objective* o, loom_device_problem** out) {
  if (!c || !p || !o || !out) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  *out = nullptr;
  LOOM_CUDA(cudaSetDevice(c->device));
  auto* dp = new loom_device_problem;
  dp->ctx = c;
  const uint64_t target = static_cast<uint64_t>(c->sms) * 2 * kBlock;
  if (int rc = build_image(p, o, target, dp->built)) {
    delete dp;
    return rc;
  }
  // deep copy of the host tables (the winner is decoded from them)
  const int n = p->n_nodes;
  int n_opts = 0;
  for (int i = 0; i < n; ++i) n_opts += p->radix[i];
  dp->radix.assign(p->radix, p->radix + n);
  dp->wall.assign(p->wall_us, p->wall_us + n_opts);
  dp->gpu.assign(p->gpu_wh, p->gpu_wh + n_opts);
  dp->cpu.assign(p->cpu_wh, p->cpu_wh + n_opts);
  dp->dol.assign(p->dollars, p->dollars + n_opts);
  dp->quality.assign(p->quality, p->quality + n_opts);
  dp->lexrank.assign(p->lexrank, p->lexrank + n_opts);
  dp->lexw.assign(p->lex_weight, p->lex_weight + n);
  dp->efrom.assign(p->edge_from, p->edge_from + p->n_edges);
  dp->eto.assign(p->edge_to, p->edge_to + p->n_edges);
  dp->host = *p;
  dp->host.radix = dp->radix.data();
  dp->host.wall_us = dp->wall.data();
  dp->host.gpu_wh = dp->gpu.data();
  dp->host.cpu_wh = dp->cpu.data();
  dp->host.dollars = dp->dol.data();
  dp->host.quality = dp->quality.data();
  dp->host.lexrank = dp->lexrank.data();
  dp->host.lex_weight = dp->lexw.data();
  dp->host.edge_from = dp->efrom.data();
  dp->host.edge_to = dp->eto.data();
  dp->objective = *o;
  dp->fn = pick_kernel(dp->built.K, dp->built.prim, dp->built.nv, true);
  if (set_smem(dp->fn, smem_bytes(dp->built.blob.size(), dp->host.n_nodes, lazy_of(dp->built))) != LOOM_OK) {
    delete dp;
    return loomi::fail(LOOM_DEVICE_ERROR, "DeviceError: cannot size shared memory");
  }
  const int ctas = c->sms * resident_ctas(dp->fn, smem_bytes(dp->built.blob.size(), dp->host.n_nodes, lazy_of(dp->built)));
  dp->ctas = ctas;
  dp->bnb_ctas = dp->built.blob.empty() ? 0 : bnb_ctas_for(c, dp->built.blob.size(), dp->host.n_nodes);
  dp->fr = new FrPlan;
  prepare_fr(c, dp->built, *dp->fr);
  bool okk = cudaMalloc(&dp->d_blob, dp->built.blob.size()) == cudaSuccess &&
             cudaMalloc(&dp->d_job, sizeof(JobDesc)) == cudaSuccess &&
             cudaMalloc(&dp->d_scratch, sizeof(Rec) * std::max({ctas, dp->bnb_ctas, dp->fr->ctas})) == cudaSuccess &&
             cudaMalloc(&dp->d_bsync, sizeof(BnbSync)) == cudaSuccess &&
             cudaMemset(dp->d_bsync, 0, sizeof(BnbSync)) == cudaSuccess &&
             cudaMalloc(&dp->d_ticket, sizeof(JobSync)) == cudaSuccess &&
             // the winner record lives in mapped pinned memory: the kernels write it
             // straight to the host (no copy node / copy launch per search)
             cudaHostAlloc(&dp->h_out, sizeof(Rec), cudaHostAllocMapped) == cudaSuccess &&
             cudaHostGetDevicePointer(reinterpret_cast<void**>(&dp->d_out), dp->h_out, 0) == cudaSuccess &&
             cudaEventCreateWithFlags(&dp->done, cudaEventDisableTiming) == cudaSuccess &&
             cudaMemcpy(dp->d_blob, dp->built.blob.data(), dp->built.blob.size(), cudaMemcpyHostToDevice) ==
                 cudaSuccess &&
             cudaMemset(dp->d_ticket, 0, sizeof(JobSync)) == cudaSuccess;
  if (!okk || set_smem(dp->fn, smem_bytes(dp->built.blob.size(), dp->host.n_nodes, lazy_of(dp->built))) != LOOM_OK) {
    loom_problem_release(dp);
    return loomi::fail(LOOM_DEVICE_ERROR, "DeviceError: upload failed");
  }
  *out = dp;
  return LOOM_OK;
}

int loom_problem_release(loom_device_problem* dp) {
  if (!dp) return LOOM_OK;
  cudaFree(dp->d_blob);
  cudaFree(dp->d_job);
  cudaFree(dp->d_scratch);
  cudaFree(dp->d_ticket);
  cudaFree(dp->d_bsync);
  if (dp->h_out) cudaFreeHost(dp->h_out);  // (d_out is its device alias)
  if (dp->done) cudaEventDestroy(dp->done);
  delete dp->fr;
  delete dp;
  return LOOM_OK;
}

uint64_t loom_device_problem_bytes(const loom_device_problem* dp) {
  return dp ? static_cast<uint64_t>(dp->built.blob.size()) : 0;
}

}  // extern "C"

namespace {

// Launch the default search of a device problem as its search graph (see
// FrPlan), building or rebuilding the graph when needed.
int fr_graph_launch(loom_ctx* c, loom_device_problem* dp, const JobDesc& d, int sweep_ctas) {
  FrPlan& f = *dp->fr;
  if (int rc = ensure_bfs(c)) return rc;
  FrArgs A{dp->d_blob, static_cast<uint32_t>(dp->built.blob.size()), c->d_bfs, c->d_front, c->d_front + c->front_cap,
           static_cast<uint64_t>(c->front_cap), dp->d_scratch, dp->d_ticket, dp->d_out, 0, kFollowGraph, nullptr, {}};
  if (f.variant == 1) {
    set_fr_job(dp->built, d, f.p16);
    A.params = &f.p16;
  } else {
    set_fr_job(dp->built, d, f.p32);
    A.params = &f.p32;
  }
  const size_t fsmem = fr_smem_bytes(dp->built.blob.size());
  if (!f.exec || f.sweep_ctas != sweep_ctas) {
    if (f.exec) cudaGraphExecDestroy(f.exec);
    if (f.graph) cudaGraphDestroy(f.graph);
    f.exec = nullptr;
    f.graph = nullptr;
    LOOM_CUDA(cudaGraphCreate(&f.graph, 0));
    LOOM_CUDA(cudaGraphConditionalHandleCreate(&f.cond, f.graph, 0, cudaGraphCondAssignDefault));
    A.cond = f.cond;
    cudaKernelNodeParams kp{};
    kp.func = const_cast<void*>(fr_fn(f.variant, f.cl));
    kp.gridDim = dim3(f.ctas);
    kp.blockDim = dim3(kFrBlock);
    kp.sharedMemBytes = static_cast<unsigned>(fsmem);
    kp.kernelParams = A.bind();
    LOOM_CUDA(cudaGraphAddKernelNode(&f.kn, f.graph, nullptr, 0, &kp));
    cudaLaunchAttributeValue coop{};
    coop.cooperative = 1;
    LOOM_CUDA(cudaGraphKernelNodeSetAttribute(f.kn, cudaLaunchAttributeCooperative, &coop));
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = f.cond;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t cn = nullptr;
    LOOM_CUDA(cudaGraphAddNode(&cn, f.graph, &f.kn, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    // the fallback: depth first from the frontier's incumbent, then the sweep
    cudaGraphNode_t b1 = nullptr, b2 = nullptr;
    const uint8_t* blob = dp->d_blob;
    const JobDesc* job = dp->d_job;
    int bctas = dp->bnb_ctas;
    Rec* scratch = dp->d_scratch;
    JobSync* ticket = dp->d_ticket;
    BnbSync* bsync = dp->d_bsync;
    Rec* out = dp->d_out;
    int sctas = sweep_ctas;
    InnerParams ip = dp->built.ip;
    if (bctas) {
      void* ba[] = {&blob, &job, &bctas, &scratch, &ticket, &bsync, &out};
      cudaKernelNodeParams bp{};
      bp.func = reinterpret_cast<void*>(bnb_kernel);
      bp.gridDim = dim3(bctas);
      bp.blockDim = dim3(kBlock);
      bp.sharedMemBytes = static_cast<unsigned>(bnb_smem_bytes(dp->built.blob.size(), dp->host.n_nodes));
      bp.kernelParams = ba;
      LOOM_CUDA(cudaGraphAddKernelNode(&b1, body, nullptr, 0, &bp));
    }
    void* sa[] = {&blob, &job, &sctas, &scratch, &ticket, &out, &ip};
    cudaKernelNodeParams sp{};
    sp.func = reinterpret_cast<void*>(dp->fn);
    sp.gridDim = dim3(sweep_ctas);
    sp.blockDim = dim3(kBlock);
    sp.sharedMemBytes = static_cast<unsigned>(smem_bytes(dp->built.blob.size(), dp->host.n_nodes, lazy_of(dp->built)));
    sp.kernelParams = sa;
    LOOM_CUDA(cudaGraphAddKernelNode(&b2, body, b1 ? &b1 : nullptr, b1 ? 1 : 0, &sp));
    LOOM_CUDA(cudaGraphInstantiate(&f.exec, f.graph, 0));
    f.sweep_ctas = sweep_ctas;
  } else {  // the same graph, this search's job fields (range, incumbent)
    A.cond = f.cond;
    cudaKernelNodeParams kp{};
    kp.func = const_cast<void*>(fr_fn(f.variant, f.cl));
    kp.gridDim = dim3(f.ctas);
    kp.blockDim = dim3(kFrBlock);
    kp.sharedMemBytes = static_cast<unsigned>(fsmem);
    kp.kernelParams = A.bind();
    LOOM_CUDA(cudaGraphExecKernelNodeSetParams(f.exec, f.kn, &kp));
  }
  LOOM_CUDA(cudaGraphLaunch(f.exec, c->stream));
  c->launches += 1;
  g_last_default_bfs = 1;
  return LOOM_OK;
}

int search_async_impl(loom_ctx* c, loom_device_problem* dp, uint64_t begin, uint64_t end, uint64_t incumbent,
                      int32_t algo) {
  if (!c || !dp) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  JobDesc d = make_desc(dp->built, begin, end, algo == kAlgoFull, &dp->host, &dp->objective, incumbent);
  d.blob_off = 0;
  if (d.begin >= d.end) return loomi::fail(LOOM_INFEASIBLE, "NoFeasibleConfigError: empty range");
  const uint64_t units = (d.sub_hi - d.sub_lo) + (d.head_end - d.begin) + (d.end - d.tail_begin);
  const int ctas = std::min(dp->ctas, ctas_for(c, units, dp->fn, smem_bytes(dp->built.blob.size(), dp->host.n_nodes, lazy_of(dp->built))));
  if (!dp->job_valid || std::memcmp(&dp->last_job, &d, sizeof d) != 0) {  // the device copy is still current otherwise
    dp->last_job = d;
    dp->job_valid = true;
    LOOM_CUDA(cudaMemcpyAsync(dp->d_job, &dp->last_job, sizeof d, cudaMemcpyHostToDevice, c->stream));
  }
  if (algo == kAlgoAuto && dp->fr->variant && !std::getenv("LOOM_NO_GRAPH")) {
    if (int rc = fr_graph_launch(c, dp, d, ctas)) return rc;
    LOOM_CUDA(cudaEventRecord(dp->done, c->stream));
    return LOOM_OK;
  }
  if (algo == kAlgoAuto && dp->fr->variant) {
    if (int rc = launch_fr(c, *dp->fr, dp->built, d, dp->d_blob, dp->d_scratch, dp->d_ticket, dp->d_out)) return rc;
  } else if (algo == kAlgoAuto) {
    g_last_default_bfs = 0;
  }
  if (algo == kAlgoAuto && dp->bnb_ctas) {
    bnb_kernel<<<dp->bnb_ctas, kBlock, bnb_smem_bytes(dp->built.blob.size(), dp->host.n_nodes), c->stream>>>(
        dp->d_blob, dp->d_job, dp->bnb_ctas, dp->d_scratch, dp->d_ticket, dp->d_bsync, dp->d_out);
    LOOM_CUDA(cudaGetLastError());
    ++c->launches;
  }
  dp->fn<<<ctas, kBlock, smem_bytes(dp->built.blob.size(), dp->host.n_nodes, lazy_of(dp->built)), c->stream>>>(dp->d_blob, dp->d_job, ctas, dp->d_scratch,
                                                             dp->d_ticket, dp->d_out, dp->built.ip);
  LOOM_CUDA(cudaGetLastError());
  ++c->launches;
  LOOM_CUDA(cudaEventRecord(dp->done, c->stream));  // the winner reaches dp->h_out directly (mapped)
  return LOOM_OK;
}

}  // namespace

extern "C" {

int loom_search_argmin_result(loom_ctx* c, loom_device_problem* dp, loom_winner* out) {
  if (!c || !dp || !out) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  LOOM_CUDA(cudaEventSynchronize(dp->done));
  return finish_winner(&dp->host, dp->h_out[0], out);
}

int loom_search_pareto(loom_ctx* c, const loom_problem* p, uint64_t begin, uint64_t end, uint64_t* out_index,
                       uint64_t capacity, uint64_t* count);

}  // extern "C"

// ---------------------------------------------------------------------------
// Pareto host driver
// ---------------------------------------------------------------------------
namespace {

static_assert(sizeof(ParetoPoint) == sizeof(loom_point), "ParetoPoint must match loom_point");


uint64_t fnv(uint64_t h, const void* data, size_t n) {
  const uint8_t* b = static_cast<const uint8_t*>(data);
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}

uint64_t problem_hash(const loom_problem* p, uint64_t begin, uint64_t end) {
  uint64_t h = 1469598103934665603ull;
  int n_opts = 0;
  for (int i = 0; i < p->n_nodes; ++i) n_opts += p->radix[i];
  h = fnv(h, &p->n_nodes, 4);
  h = fnv(h, p->radix, 4 * p->n_nodes);
  h = fnv(h, p->wall_us, 8 * n_opts);
  h = fnv(h, p->gpu_wh, 8 * n_opts);
  h = fnv(h, p->dollars, 8 * n_opts);
  h = fnv(h, p->quality, 4 * n_opts);
  h = fnv(h, p->edge_from, 4 * p->n_edges);
  h = fnv(h, p->edge_to, 4 * p->n_edges);
  h = fnv(h, &begin, 8);
  return fnv(h, &end, 8);
}

// Exact frontier of device points [0, n) -> host vector.  Large sets are
// filtered blockwise first (each point against its 8K block), the block
// frontiers are compacted on the host and filtered pairwise.
int filter_device(loom_ctx* c, const ParetoPoint* d_pts, uint64_t n, std::vector<ParetoPoint>& out) {
  out.clear();
  if (n == 0) return LOOM_OK;
  constexpr uint64_t kSpan = 8192;
  DevBuf<uint8_t> keep(c);
  LOOM_CUDA(keep.alloc(n));
  const uint64_t blocks = (n + kPBlock - 1) / kPBlock;
  const uint64_t span = n > 2 * kSpan ? kSpan : 0;
  pareto_filter_kernel<<<static_cast<unsigned>(blocks), kPBlock, 0, c->stream>>>(d_pts, n, keep.p, span);
  LOOM_CUDA(cudaGetLastError());
  ++c->launches;
  std::vector<uint8_t> hk(n);
  std::vector<ParetoPoint> hp(n);
  LOOM_CUDA(cudaMemcpyAsync(hk.data(), keep.p, n, cudaMemcpyDeviceToHost, c->stream));
  LOOM_CUDA(cudaMemcpyAsync(hp.data(), d_pts, n * sizeof(ParetoPoint), cudaMemcpyDeviceToHost, c->stream));
  LOOM_CUDA(cudaStreamSynchronize(c->stream));
  for (uint64_t i = 0; i < n; ++i)
    if (hk[i]) out.push_back(hp[i]);
  if (span == 0) return LOOM_OK;
  DevBuf<ParetoPoint> d2(c);
  LOOM_CUDA(d2.alloc(out.size()));
  LOOM_CUDA(cudaMemcpyAsync(d2.p, out.data(), out.size() * sizeof(ParetoPoint), cudaMemcpyHostToDevice, c->stream));
  std::vector<ParetoPoint> f;
  if (int rc = filter_device(c, d2.p, out.size(), f)) return rc;
  out = std::move(f);
  return LOOM_OK;
}

// At most kGuardMax points of a frontier, spread over its index order.
std::vector<ParetoPoint> guard_of(std::vector<ParetoPoint> f) {
  std::sort(f.begin(), f.end(), [](const ParetoPoint& a, const ParetoPoint& b) { return a.index < b.index; });
  if (f.size() <= static_cast<size_t>(kGuardMax)) return f;
  std::vector<ParetoPoint> g;
  for (int k = 0; k < kGuardMax; ++k) g.push_back(f[f.size() * k / kGuardMax]);
  return g;
}

// Exact frontier of device candidates [0, n): while the set is large, the
// frontier of a strided 64K subsample (plus the current guard) becomes the
// guard, and the candidates it dominates are dropped; the rest goes through
// the exact pairwise filter.
int refine_and_filter(loom_ctx* c, ParetoPoint* d_in, uint64_t n, std::vector<ParetoPoint> guard,
                      std::vector<ParetoPoint>& front) {
  const uint64_t kSub = 1 << 16;
  DevBuf<ParetoPoint> d_a(c), d_sub(c), d_g(c);
  DevBuf<unsigned long long> d_cnt(c);
  LOOM_CUDA(d_a.alloc(n));
  LOOM_CUDA(d_sub.alloc(kSub));
  LOOM_CUDA(d_g.alloc(kGuardMax));
  LOOM_CUDA(d_cnt.alloc(1));
  ParetoPoint* cur = d_in;
  ParetoPoint* nxt = d_a.p;
  const size_t gsmem = kGuardBytes;
  LOOM_CUDA(smem_attr(reinterpret_cast<const void*>(pareto_prefilter_kernel), static_cast<size_t>(gsmem)));
  for (int round = 0; round < 8 && n > kSub; ++round) {
    const uint64_t stride = n / kSub;
    LOOM_CUDA(cudaMemcpy2DAsync(d_sub.p, sizeof(ParetoPoint), cur, sizeof(ParetoPoint) * stride, sizeof(ParetoPoint),
                                kSub, cudaMemcpyDeviceToDevice, c->stream));
    std::vector<ParetoPoint> g;
    if (int rc = filter_device(c, d_sub.p, kSub, g)) return rc;
    g.insert(g.end(), guard.begin(), guard.end());
    LOOM_CUDA(cudaMemcpyAsync(d_sub.p, g.data(), std::min<size_t>(g.size(), kSub) * sizeof(ParetoPoint),
                              cudaMemcpyHostToDevice, c->stream));
    std::vector<ParetoPoint> g2;
    if (int rc = filter_device(c, d_sub.p, std::min<size_t>(g.size(), kSub), g2)) return rc;
    guard = guard_of(g2);
    LOOM_CUDA(cudaMemcpyAsync(d_g.p, guard.data(), guard.size() * sizeof(ParetoPoint), cudaMemcpyHostToDevice,
                              c->stream));
    LOOM_CUDA(cudaMemsetAsync(d_cnt.p, 0, sizeof(unsigned long long), c->stream));
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + kPBlock - 1) / kPBlock, uint64_t(c->sms) * 8));
    pareto_prefilter_kernel<<<grid, kPBlock, gsmem, c->stream>>>(cur, n, d_g.p, static_cast<int>(guard.size()), nxt,
                                                                d_cnt.p);
    LOOM_CUDA(cudaGetLastError());
    ++c->launches;
    unsigned long long m = 0;
    LOOM_CUDA(cudaMemcpyAsync(&m, d_cnt.p, sizeof m, cudaMemcpyDeviceToHost, c->stream));
    LOOM_CUDA(cudaStreamSynchronize(c->stream));
    if (std::getenv("LOOM_DEBUG"))
      std::fprintf(stderr, "[loom pareto] refine %d: %llu -> %llu (guard %zu)\n", round,
                   static_cast<unsigned long long>(n), m, guard.size());
    const bool progress = m < n - n / 8;
    n = m;
    std::swap(cur, nxt);
    if (!progress) break;
  }
  return filter_device(c, cur, n, front);
}

int pareto_run(loom_ctx* c, const loom_problem* p, uint64_t begin, uint64_t end, std::vector<ParetoPoint>& front) {
  front.clear();
  loom_objective o;
  std::memset(&o, 0, sizeof o);
  o.n_criteria = 2;
  o.criteria[0] = LOOM_MIN_ENERGY;  // slot A = gpu_wh
  o.criteria[1] = LOOM_MIN_COST_DOLLARS;  // slot B = dollars
  Built b;
  if (int rc = build_image(p, &o, 1, b)) return rc;
  end = std::min(end, b.total);
  if (begin >= end) return LOOM_OK;
  const uint64_t n = end - begin;
  const uint32_t bytes = static_cast<uint32_t>(b.blob.size());
  const size_t smem = ((bytes + 127) & ~size_t(127)) + kGuardBytes + pareto_dp_bytes(p->n_nodes);
  DevBuf<uint8_t> d_blob(c);
  LOOM_CUDA(d_blob.alloc(bytes));
  LOOM_CUDA(cudaMemcpyAsync(d_blob.p, b.blob.data(), bytes, cudaMemcpyHostToDevice, c->stream));
  LOOM_CUDA(smem_attr(reinterpret_cast<const void*>(pareto_eval_kernel), static_cast<size_t>(smem)));
  LOOM_CUDA(smem_attr(reinterpret_cast<const void*>(pareto_points_kernel), static_cast<size_t>(bytes + 128)));

  // guard: exact frontier of an evenly strided sample of the range
  const auto t_guard = std::chrono::steady_clock::now();
  std::vector<ParetoPoint> guard;
  const uint64_t kSample = 1 << 16;
  if (n > kSample) {
    std::vector<uint64_t> idx(kSample);
    for (uint64_t k = 0; k < kSample; ++k)
      idx[k] = begin + static_cast<uint64_t>((static_cast<unsigned __int128>(n) * k) / kSample);
    DevBuf<uint64_t> d_idx(c);
    DevBuf<ParetoPoint> d_s(c);
    LOOM_CUDA(d_idx.alloc(kSample));
    LOOM_CUDA(d_s.alloc(kSample));
    LOOM_CUDA(cudaMemcpyAsync(d_idx.p, idx.data(), kSample * 8, cudaMemcpyHostToDevice, c->stream));
    pareto_points_kernel<<<static_cast<unsigned>(kSample / kPBlock), kPBlock, bytes + 128, c->stream>>>(
        d_blob.p, bytes, d_idx.p, kSample, d_s.p);
    LOOM_CUDA(cudaGetLastError());
    ++c->launches;
    std::vector<ParetoPoint> f0;
    if (int rc = filter_device(c, d_s.p, kSample, f0)) return rc;
    guard = guard_of(f0);
    if (std::getenv("LOOM_DEBUG"))
      std::fprintf(stderr, "[loom pareto] guard build %.3fs (sample frontier %zu)\n",
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - t_guard).count(), f0.size());
  }

  const uint64_t cap = std::min<uint64_t>(uint64_t(1) << 22, n);
  DevBuf<ParetoPoint> d_cand(c), d_guard(c);
  DevBuf<unsigned long long> d_count(c), d_next(c);
  LOOM_CUDA(d_next.alloc(1));
  LOOM_CUDA(d_cand.alloc(cap));
  LOOM_CUDA(d_guard.alloc(kGuardMax));
  LOOM_CUDA(d_count.alloc(1));
  int resident = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, reinterpret_cast<const void*>(pareto_eval_kernel), kPBlock,
                                                smem);
  const uint64_t units = n / 64 + 1;
  const unsigned grid =
      static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(static_cast<uint64_t>(c->sms) * std::max(1, resident),
                                                                     (units + kPBlock - 1) / kPBlock)));
  for (int attempt = 0; attempt < 6; ++attempt) {
    const auto t0 = std::chrono::steady_clock::now();
    unsigned long long count = 0;
    LOOM_CUDA(cudaMemsetAsync(d_count.p, 0, sizeof(unsigned long long), c->stream));
    if (!guard.empty())
      LOOM_CUDA(cudaMemcpyAsync(d_guard.p, guard.data(), guard.size() * sizeof(ParetoPoint), cudaMemcpyHostToDevice,
                                c->stream));
    DevBuf<unsigned long long> d_stats(c);
    const bool dbg = std::getenv("LOOM_DEBUG") != nullptr;
    if (dbg) {
      LOOM_CUDA(d_stats.alloc(4));
      LOOM_CUDA(cudaMemsetAsync(d_stats.p, 0, 32, c->stream));
    }
    LOOM_CUDA(cudaMemsetAsync(d_next.p, 0, sizeof(unsigned long long), c->stream));
    pareto_eval_kernel<<<grid, kPBlock, smem, c->stream>>>(d_blob.p, bytes, begin, end, d_guard.p,
                                                          static_cast<int>(guard.size()), d_cand.p, cap, d_count.p,
                                                          d_stats.p, d_next.p);
    if (dbg) {
      unsigned long long st[4];
      LOOM_CUDA(cudaMemcpyAsync(st, d_stats.p, 32, cudaMemcpyDeviceToHost, c->stream));
      LOOM_CUDA(cudaStreamSynchronize(c->stream));
      std::fprintf(stderr, "[loom pareto] groups %llu live %llu, rows %llu live %llu\n", st[0], st[1], st[2], st[3]);
    }
    LOOM_CUDA(cudaGetLastError());
    ++c->launches;
    LOOM_CUDA(cudaMemcpyAsync(&count, d_count.p, sizeof count, cudaMemcpyDeviceToHost, c->stream));
    LOOM_CUDA(cudaStreamSynchronize(c->stream));
    const auto t_eval = std::chrono::steady_clock::now();
    if (count <= cap) {
      std::vector<ParetoPoint> f;
      if (int rc = refine_and_filter(c, d_cand.p, count, guard, f)) return rc;
      if (std::getenv("LOOM_DEBUG"))
        std::fprintf(stderr, "[loom pareto] guard=%zu candidates=%llu frontier=%zu eval=%.3fs refine+filter=%.3fs\n",
                     guard.size(), count, f.size(), std::chrono::duration<double>(t_eval - t0).count(),
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t_eval).count());
      std::sort(f.begin(), f.end(), [](const ParetoPoint& a, const ParetoPoint& b) { return a.index < b.index; });
      front = std::move(f);
      return LOOM_OK;
    }
    std::vector<ParetoPoint> f;
    if (int rc = refine_and_filter(c, d_cand.p, cap, guard, f)) return rc;
    // overflow: the frontier of what was collected (real plans) joins the guard
    f.insert(f.end(), guard.begin(), guard.end());
    DevBuf<ParetoPoint> d_g2(c);
    LOOM_CUDA(d_g2.alloc(f.size()));
    LOOM_CUDA(cudaMemcpyAsync(d_g2.p, f.data(), f.size() * sizeof(ParetoPoint), cudaMemcpyHostToDevice, c->stream));
    std::vector<ParetoPoint> g2;
    if (int rc = filter_device(c, d_g2.p, f.size(), g2)) return rc;
    guard = guard_of(g2);
  }
  return loomi::fail(LOOM_DEVICE_ERROR, "DeviceError: pareto candidate buffer overflowed repeatedly");
}

}  // namespace

extern "C" int loom_search_pareto_points(loom_ctx* c, const loom_problem* p, uint64_t begin, uint64_t end,
                                         loom_point* out, uint64_t capacity, uint64_t* count) {
  if (!c || !p || !count) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  LOOM_CUDA(cudaSetDevice(c->device));
  uint64_t total = 0;
  if (int rc = loomi::check_problem(p, &total)) return rc;
  const uint64_t key = problem_hash(p, begin, end);
  if (!c->pareto_valid || c->pareto_key != key) {
    std::vector<ParetoPoint> f;
    if (int rc = pareto_run(c, p, begin, end, f)) return rc;
    c->pareto_cache.assign(reinterpret_cast<const loom_point*>(f.data()),
                           reinterpret_cast<const loom_point*>(f.data()) + f.size());
    c->pareto_key = key;
    c->pareto_valid = true;
  }
  *count = c->pareto_cache.size();
  if (out && capacity >= c->pareto_cache.size())
    std::copy(c->pareto_cache.begin(), c->pareto_cache.end(), out);
  return LOOM_OK;
}

extern "C" int loom_search_pareto(loom_ctx* c, const loom_problem* p, uint64_t begin, uint64_t end,
                                  uint64_t* out_index, uint64_t capacity, uint64_t* count) {
  uint64_t n = 0;
  if (int rc = loom_search_pareto_points(c, p, begin, end, nullptr, 0, &n)) return rc;
  *count = n;
  if (out_index && capacity >= n)
    for (uint64_t i = 0; i < n; ++i) out_index[i] = c->pareto_cache[i].plan_index;
  return LOOM_OK;
}

extern "C" int loom_pareto_filter_points(loom_ctx* c, const loom_point* pts, uint64_t n, uint8_t* keep) {
  if (!c || (n && (!pts || !keep))) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  if (n == 0) return LOOM_OK;
  LOOM_CUDA(cudaSetDevice(c->device));
  DevBuf<ParetoPoint> d(c);
  DevBuf<uint8_t> k(c);
  LOOM_CUDA(d.alloc(n));
  LOOM_CUDA(k.alloc(n));
  LOOM_CUDA(cudaMemcpyAsync(d.p, pts, n * sizeof(loom_point), cudaMemcpyHostToDevice, c->stream));
  pareto_filter_kernel<<<static_cast<unsigned>((n + kPBlock - 1) / kPBlock), kPBlock, 0, c->stream>>>(d.p, n, k.p, 0);
  LOOM_CUDA(cudaGetLastError());
  ++c->launches;
  LOOM_CUDA(cudaMemcpyAsync(keep, k.p, n, cudaMemcpyDeviceToHost, c->stream));
  LOOM_CUDA(cudaStreamSynchronize(c->stream));
  return LOOM_OK;
}

extern "C" int loom_search_greedy(loom_ctx* c, const loom_problem* p, const loom_objective* o,
                                  const int32_t* sweep_order, const int32_t* seed, int32_t max_sweeps,
                                  loom_winner* out) {
  if (!c || !p || !o || !out) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  std::memset(out, 0, sizeof *out);
  LOOM_CUDA(cudaSetDevice(c->device));
  uint64_t total = 0;
  if (int rc = loomi::check_problem(p, &total)) return rc;
  if (p->n_nodes == 0) return loomi::fail(LOOM_INFEASIBLE, "NoFeasibleConfigError: cannot search an empty dag");
  const int n = p->n_nodes;
  std::vector<int32_t> sd(n), ord;
  if (seed) sd.assign(seed, seed + n);
  else if (int rc = loom_greedy_seed(p, o, sd.data())) return rc;
  if (sweep_order) {
    ord.assign(sweep_order, sweep_order + n);
  } else {  // index-ordered Kahn
    std::vector<int> indeg(n, 0);
    std::vector<std::vector<int>> succ(n);
    for (int e = 0; e < p->n_edges; ++e) {
      succ[p->edge_from[e]].push_back(p->edge_to[e]);
      ++indeg[p->edge_to[e]];
    }
    std::priority_queue<int, std::vector<int>, std::greater<>> ready;
    for (int i = 0; i < n; ++i)
      if (!indeg[i]) ready.push(i);
    while (!ready.empty()) {
      const int x = ready.top();
      ready.pop();
      ord.push_back(x);
      for (int y : succ[x])
        if (--indeg[y] == 0) ready.push(y);
    }
    if (static_cast<int>(ord.size()) != n) return loomi::fail(LOOM_INVALID, "CycleError: dag has a cycle");
  }
  for (int i = 0; i < n; ++i)
    if (sd[i] < 0 || sd[i] >= p->radix[i]) return loomi::fail(LOOM_INVALID, "InvalidConfigError: seed out of range");
  Built b;
  if (int rc = build_image(p, o, 1, b)) return rc;
  const uint32_t bytes = static_cast<uint32_t>(b.blob.size());
  DevBuf<uint8_t> d_blob(c);
  DevBuf<int32_t> d_ord(c), d_seed(c), d_sw(c);
  DevBuf<Rec> d_out(c);
  LOOM_CUDA(d_blob.alloc(bytes));
  LOOM_CUDA(d_ord.alloc(n));
  LOOM_CUDA(d_seed.alloc(n));
  LOOM_CUDA(d_sw.alloc(1));
  LOOM_CUDA(d_out.alloc(1));
  LOOM_CUDA(cudaMemcpyAsync(d_blob.p, b.blob.data(), bytes, cudaMemcpyHostToDevice, c->stream));
  LOOM_CUDA(cudaMemcpyAsync(d_ord.p, ord.data(), 4 * n, cudaMemcpyHostToDevice, c->stream));
  LOOM_CUDA(cudaMemcpyAsync(d_seed.p, sd.data(), 4 * n, cudaMemcpyHostToDevice, c->stream));
  LOOM_CUDA(smem_attr(reinterpret_cast<const void*>(greedy_kernel), static_cast<size_t>(bytes + 128)));
  greedy_kernel<<<1, kBlock, bytes + 128, c->stream>>>(d_blob.p, bytes, d_ord.p, d_seed.p, max_sweeps, d_out.p,
                                                       d_sw.p);
  LOOM_CUDA(cudaGetLastError());
  ++c->launches;
  Rec r;
  LOOM_CUDA(cudaMemcpyAsync(&r, d_out.p, sizeof r, cudaMemcpyDeviceToHost, c->stream));
  LOOM_CUDA(cudaStreamSynchronize(c->stream));
  return finish_winner(p, r, out);
}

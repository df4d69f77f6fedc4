// sm_100a per-plan estimate streams: loom::estimate (estimator.hpp:43-78) for
// every plan of an index range in ConfigEnumerator order
// (optimizer.hpp:131-143), written as structure-of-arrays score streams
// (latency_us, gpu_wh, cpu_wh, total_wh, dollars, quality), and for an
// arbitrary list of plan indices (batched estimate).
//
// This is the HBM-bound member of the family: 44 bytes leave the SM per plan
// and nothing is read from global memory after the problem image.
//
// ALGORITHM.  The last K nodes (K = 1..3, chosen on the host
// so a group holds >= 256 plans) are the suffix; a *group* fixes every other
// digit and holds G = prod(suffix radices) consecutive plans.  Per group, one
// warp:
//   * decodes the group's top digits (lane i: digit i);
//   * runs a lane-parallel longest-path DP in topological order that treats
//     the K suffix walls as symbols (lane S computes column S, S a subset of
//     the suffix): c[S] = the longest path whose suffix nodes are exactly S,
//     counting only top walls.  latency = max_S (c[S] + sum_{s in S} wall_s);
//     integer max/+ is exact, so this equals the reference's finish-time
//     recursion (estimator.hpp:69-76) for every plan of the group;
//   * folds the top nodes' gpu_wh / cpu_wh / dollars in dag order
//     (estimator.hpp:50-60) and their quality minimum (61-64).
// Then lane l evaluates plans l, l + 32, l + 64, ... of the group: the suffix
// terms are added to the folds in dag order (every sum rounds exactly like
// the reference's), total = gpu + cpu (estimator.hpp:67), the coefficient
// vector is folded once per suffix node (c'[S] = max(c[S], c[S+s] + w_s)) and
// the quality minimum taken.  Consecutive lanes hold consecutive plans, so
// each store instruction writes 32 consecutive elements of a stream (256 B
// of an f64 stream): fully coalesced, with no staging and no global reads.
//
// Compiled with -fmad=false; all FP sums use __dadd_rn explicitly.

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "ctx.h"
#include "internal.h"
#include "loom_b200.h"
#include "search_common.h"
#include "tma.cuh"

using namespace loomk;
using loomi::DevBuf;

namespace {

constexpr int kEstWarps = 8;  // warps per CTA
constexpr int kEstBlock = 32 * kEstWarps;
constexpr int kEstMaxK = 3;   // suffix nodes carried symbolically (<= 8 DP columns)
constexpr int64_t kEstNeg = -(int64_t(1) << 62);
constexpr int kSmemMax = 227 * 1024;

// Per-warp scratch of the range kernel: top digits, DP table f[n][8], c[8].
__host__ __device__ constexpr int est_warp_bytes(int n) { return 128 + n * 8 * 8 + 8 * 8; }

// One option of the lowered table (48 bytes, three LDS.128).
struct alignas(16) EstOpt {
  double g;   // gpu_wh * path_count
  double c;   // cpu_wh * path_count
  double d;   // dollars * path_count
  int64_t w;  // wall_us
  int32_t q;  // node quality
  int32_t pad[3];
};

struct alignas(16) EstHeader {
  int32_t n_nodes;
  int32_t n_edges;
  int32_t n_opts;
  int32_t bytes;
  int32_t off_radix;
  int32_t off_optoff;
  int32_t off_topo;
  int32_t off_predoff;
  int32_t off_pred;
  int32_t off_opt;
  int32_t off_wtop;  // u64 weight of each top digit within the group index
  int32_t K;         // suffix nodes
  uint64_t total;
  uint64_t group;    // plans per group = product of the suffix radices
};

struct EstStreams {
  int64_t* lat;
  double* gpu;
  double* cpu;
  double* tot;
  double* dol;
  int32_t* q;
};

struct EstView {
  const EstHeader* h;
  const int32_t* radix;
  const int32_t* optoff;
  const int32_t* topo;
  const int32_t* predoff;
  const int32_t* pred;
  const EstOpt* opt;
  const uint64_t* wtop;
};

__device__ __forceinline__ EstView est_view(const uint8_t* s) {
  EstView v;
  v.h = reinterpret_cast<const EstHeader*>(s);
  v.radix = reinterpret_cast<const int32_t*>(s + v.h->off_radix);
  v.optoff = reinterpret_cast<const int32_t*>(s + v.h->off_optoff);
  v.topo = reinterpret_cast<const int32_t*>(s + v.h->off_topo);
  v.predoff = reinterpret_cast<const int32_t*>(s + v.h->off_predoff);
  v.pred = reinterpret_cast<const int32_t*>(s + v.h->off_pred);
  v.opt = reinterpret_cast<const EstOpt*>(s + v.h->off_opt);
  v.wtop = reinterpret_cast<const uint64_t*>(s + v.h->off_wtop);
  return v;
}

// Digits of x in ConfigEnumerator order (node 0 most significant).
__device__ __forceinline__ void est_decode(const EstView& v, uint64_t x, int* d) {
  for (int i = v.h->n_nodes - 1; i >= 0; --i) {
    const uint64_t r = static_cast<uint64_t>(v.radix[i]);
    d[i] = static_cast<int>(x % r);
    x /= r;
  }
}

// State shared by every plan of one prefix (all digits but the last node's).
struct Prefix {
  double sa, sc, sd;  // dag-order folds of the prefix nodes
  int64_t a, b;       // latency = max(a, b + wall_last)
  int32_t q;          // prefix quality minimum
};

__device__ __forceinline__ Prefix est_prefix(const EstView& v, const int* d) {
  const int n = v.h->n_nodes;
  const int last = n - 1;
  Prefix p;
  p.sa = 0.0;
  p.sc = 0.0;
  p.sd = 0.0;
  p.q = INT_MAX;
  for (int i = 0; i < last; ++i) {
    const EstOpt& e = v.opt[v.optoff[i] + d[i]];
    p.sa = __dadd_rn(p.sa, e.g);
    p.sc = __dadd_rn(p.sc, e.c);
    p.sd = __dadd_rn(p.sd, e.d);
    p.q = min(p.q, e.q);
  }
  int64_t f0[kMaxNodes], f1[kMaxNodes];
  p.a = kEstNeg;
  p.b = kEstNeg;
  for (int t = 0; t < n; ++t) {
    const int x = v.topo[t];
    int64_t m0 = 0, m1 = kEstNeg;  // start = 0 (estimator.hpp:71)
    for (int k = v.predoff[x]; k < v.predoff[x + 1]; ++k) {
      const int u = v.pred[k];
      m0 = max(m0, f0[u]);
      m1 = max(m1, f1[u]);
    }
    if (x == last) {
      f0[x] = kEstNeg;
      f1[x] = m0;
    } else {
      const int64_t w = v.opt[v.optoff[x] + d[x]].w;
      f0[x] = m0 + w;
      f1[x] = m1 + w;
    }
    p.a = max(p.a, f0[x]);
    p.b = max(p.b, f1[x]);
  }
  return p;
}

struct Est {
  int64_t lat;
  double g, c, t, d;
  int32_t q;
};

__device__ __forceinline__ Est est_plan(const Prefix& p, const EstOpt& e) {
  Est r;
  r.g = __dadd_rn(p.sa, e.g);
  r.c = __dadd_rn(p.sc, e.c);
  r.d = __dadd_rn(p.sd, e.d);
  r.t = __dadd_rn(r.g, r.c);  // total_wh = gpu_wh + cpu_wh (estimator.hpp:67)
  r.lat = max(p.a, p.b + e.w);
  r.q = min(p.q, e.q);
  return r;
}

__device__ __forceinline__ void est_put(const EstStreams& o, uint64_t i, const Est& r) {
  if (o.lat) o.lat[i] = r.lat;
  if (o.gpu) o.gpu[i] = r.g;
  if (o.cpu) o.cpu[i] = r.c;
  if (o.tot) o.tot[i] = r.t;
  if (o.dol) o.dol[i] = r.d;
  if (o.q) o.q[i] = r.q;
}

// Lane-parallel longest-path DP of one group (lane S < 2^K computes column
// S; bit k of S = suffix node P + k; a suffix node reads its predecessors'
// column S minus its own bit, so lanes synchronise per node).  f[x][S]: the longest path ending at x
// whose suffix nodes are exactly S, top walls only.  Leaves c[S] in cw.
template <int K>
__device__ __forceinline__ void est_warp_dp(const EstView& v, const int* dtop, int P, int64_t* fw, int64_t* cw) {
  constexpr int NS = 1 << K;
  const int S = threadIdx.x & 31;
  const bool act = S < NS;
  const int n = v.h->n_nodes;
  int64_t cmax = kEstNeg;
  // every lane walks the nodes (lanes >= NS idle) so the barriers are
  // full-warp ones
  for (int t = 0; t < n; ++t) {
    const int x = v.topo[t];
    // a suffix node reads column S ^ bit of its predecessors, written by
    // another lane: every lane's earlier rows must have landed (top nodes
    // read only their own column)
    if (x >= P) __syncwarp();
    if (act) {
      const int pb = v.predoff[x], pe = v.predoff[x + 1];
      int64_t val = kEstNeg;
      if (x < P) {
        int64_t b = S == 0 ? 0 : kEstNeg;  // start = 0 (estimator.hpp:71)
        for (int e = pb; e < pe; ++e) b = max(b, fw[v.pred[e] * NS + S]);
        val = b + v.opt[v.optoff[x] + dtop[x]].w;
      } else {
        const int bit = 1 << (x - P);
        if (S & bit) {
          const int S2 = S ^ bit;
          int64_t b = S2 == 0 ? 0 : kEstNeg;
          for (int e = pb; e < pe; ++e) b = max(b, fw[v.pred[e] * NS + S2]);
          val = b;
        }
      }
      fw[x * NS + S] = val;
      cmax = max(cmax, val);
    }
  }
  if (act) cw[S] = S == 0 ? max(cmax, int64_t(0)) : cmax;  // latency starts at 0 (estimator.hpp:27)
  __syncwarp();
}

// Plans [begin, end) -> out[0 .. end-begin), one group per warp at a time.
// W32: every latency fits in 30 bits (host-checked: the sum of the nodes'
// largest walls), so the per-plan max-plus fold runs in int32; the values are
// identical integers either way.
template <int K, bool W32>
__global__ void __launch_bounds__(kEstBlock) estimate_range_kernel(const uint8_t* __restrict__ gblob,
                                                                   uint32_t blob_bytes, uint64_t begin, uint64_t end,
                                                                   EstStreams out) {
  constexpr int NS = 1 << K;
  using Lat = typename std::conditional<W32, int32_t, int64_t>::type;
  constexpr Lat kLatNeg = W32 ? Lat(-(1 << 30)) : Lat(kEstNeg);
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t mbar;
  load_blob(smem, gblob, blob_bytes, &mbar);
  const EstView v = est_view(smem);
  const int n = v.h->n_nodes;
  const int P = n - K;  // top nodes
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  uint8_t* ws = smem + blob_bytes + warp * est_warp_bytes(n);
  int* dtop = reinterpret_cast<int*>(ws);
  int64_t* fw = reinterpret_cast<int64_t*>(ws + 128);
  int64_t* cw = fw + n * 8;

  const uint64_t G = v.h->group;
  int rs[K], os[K], step[K];
  {
    uint32_t x = 32;
#pragma unroll
    for (int k = K - 1; k >= 0; --k) {
      rs[k] = v.radix[P + k];
      os[k] = v.optoff[P + k];
      step[k] = static_cast<int>(x % static_cast<uint32_t>(rs[k]));  // digits of +32 (used when G > 32)
      x /= static_cast<uint32_t>(rs[k]);
    }
  }
  const uint64_t g_lo = begin / G, g_hi = (end + G - 1) / G;
  const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * kEstWarps;
  for (uint64_t g = g_lo + static_cast<uint64_t>(blockIdx.x) * kEstWarps + warp; g < g_hi; g += nwarps) {
    if (lane < P) dtop[lane] = static_cast<int>((g / v.wtop[lane]) % static_cast<uint64_t>(v.radix[lane]));
    __syncwarp();
    est_warp_dp<K>(v, dtop, P, fw, cw);
    Lat c[NS];
#pragma unroll
    for (int S = 0; S < NS; ++S) c[S] = cw[S] < kLatNeg ? kLatNeg : static_cast<Lat>(cw[S]);
    double sa = 0.0, sc = 0.0, sd = 0.0;
    int32_t q = INT_MAX;
    for (int i = 0; i < P; ++i) {
      const EstOpt& e = v.opt[v.optoff[i] + dtop[i]];
      sa = __dadd_rn(sa, e.g);
      sc = __dadd_rn(sc, e.c);
      sd = __dadd_rn(sd, e.d);
      q = min(q, e.q);
    }
    __syncwarp();  // every lane has read dtop / cw before the next group rewrites them
    const uint64_t g0 = g * G;
    const uint64_t lo = begin > g0 ? begin : g0;
    const uint32_t ga = static_cast<uint32_t>(lo - g0);
    const uint32_t gb = static_cast<uint32_t>((end < g0 + G ? end : g0 + G) - g0);
    // Lane l takes the elements e == l (mod 32) of the output, so each store
    // instruction fills one aligned 32-element window (whole sectors; a
    // window straddling sectors costs L2 partial-sector merges).
    // In the group's first window the lanes before ga sit out one step.
    const int mis = static_cast<int>(static_cast<uint32_t>(lo - begin) & 31u);  // element of ga within its window
    int o = static_cast<int>(ga) - mis + lane;  // this lane's plan offset at the current window
    const int o_first = o < static_cast<int>(ga) ? o + 32 : o;
    if (o_first >= static_cast<int>(gb)) continue;
    // this group's slice of every stream; element o - ga of the slice is plan g0 + o
    const uint64_t base = lo - begin;
    int64_t* p_lat = out.lat ? out.lat + base : nullptr;
    double* p_gpu = out.gpu ? out.gpu + base : nullptr;
    double* p_cpu = out.cpu ? out.cpu + base : nullptr;
    double* p_tot = out.tot ? out.tot + base : nullptr;
    double* p_dol = out.dol ? out.dol + base : nullptr;
    int32_t* p_q = out.q ? out.q + base : nullptr;
    int ds[K];
    {
      uint32_t x = static_cast<uint32_t>(o_first);
#pragma unroll
      for (int k = K - 1; k >= 0; --k) {
        ds[k] = static_cast<int>(x % static_cast<uint32_t>(rs[k]));
        x /= static_cast<uint32_t>(rs[k]);
      }
    }
    // lockstep over windows: a lane whose first window starts before ga sits
    // that step out (its digits already point at its next plan)
    for (;;) {
      const bool act = o >= static_cast<int>(ga);  // false only in a lane's first window
      double eg = sa, ec = sc, ed = sd;
      int32_t eq = q;
      Lat cur[NS];
#pragma unroll
      for (int S = 0; S < NS; ++S) cur[S] = c[S];
#pragma unroll
      for (int k = 0; k < K; ++k) {  // suffix nodes in dag order
        const EstOpt& e = v.opt[os[k] + ds[k]];
        eg = __dadd_rn(eg, e.g);
        ec = __dadd_rn(ec, e.c);
        ed = __dadd_rn(ed, e.d);
        eq = min(eq, e.q);
        const Lat w = static_cast<Lat>(e.w);
#pragma unroll
        for (int t = 0; t < (NS >> (k + 1)); ++t) cur[t] = max(cur[2 * t], cur[2 * t + 1] + w);
      }
      // predicated, not branched: the warp stays converged, so every store
      // instruction fills its window at once
      const uint32_t i = static_cast<uint32_t>(o) - ga;
      if (p_lat && act) p_lat[i] = cur[0];
      if (p_gpu && act) p_gpu[i] = eg;
      if (p_cpu && act) p_cpu[i] = ec;
      if (p_tot && act) p_tot[i] = __dadd_rn(eg, ec);  // total_wh = gpu_wh + cpu_wh (estimator.hpp:67)
      if (p_dol && act) p_dol[i] = ed;
      if (p_q && act) p_q[i] = eq;
      o += 32;
      if (o >= static_cast<int>(gb)) break;
      int carry = 0;  // suffix digits += digits of 32 (a sat-out lane already points at its next plan)
#pragma unroll
      for (int k = K - 1; k >= 0; --k) {
        const int x = ds[k] + step[k] + carry;
        carry = x >= rs[k];
        ds[k] = act ? (carry ? x - rs[k] : x) : ds[k];
        carry = act ? carry : 0;
      }
    }
  }
}

// Arbitrary plan indices (validated < total on the host) -> out[0 .. n).
__global__ void __launch_bounds__(kEstBlock) estimate_plans_kernel(const uint8_t* __restrict__ gblob,
                                                                   uint32_t blob_bytes,
                                                                   const uint64_t* __restrict__ idx, uint64_t n_idx,
                                                                   EstStreams out) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t mbar;
  load_blob(smem, gblob, blob_bytes, &mbar);
  const EstView v = est_view(smem);
  const int last = v.h->n_nodes - 1;
  int d[kMaxNodes];
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kEstBlock + threadIdx.x; i < n_idx;
       i += static_cast<uint64_t>(gridDim.x) * kEstBlock) {
    est_decode(v, idx[i], d);
    const Prefix p = est_prefix(v, d);
    est_put(out, i, est_plan(p, v.opt[v.optoff[last] + d[last]]));
  }
}

// ---------------------------------------------------------------------------
// host: estimate image
// ---------------------------------------------------------------------------
struct EstImage {
  std::vector<uint8_t> blob;
  uint64_t total = 0;
  int K = 1;
  int n = 0;
  bool w32 = false;  // every latency < 2^30 us: int32 max-plus fold
};

int align16(int x) { return (x + 15) & ~15; }

int build_est_image(const loom_problem* p, EstImage& im, int smem_budget) {
  if (int rc = loomi::check_problem(p, &im.total)) return rc;
  const int n = p->n_nodes;
  im.n = n;
  if (n > kMaxNodes) return loomi::fail(LOOM_INVALID, "InvalidConfigError: more than 32 nodes");
  if (p->n_edges > kMaxEdges) return loomi::fail(LOOM_INVALID, "InvalidConfigError: more than 512 edges");
  int n_opts = 0;
  for (int i = 0; i < n; ++i) n_opts += p->radix[i];
  // Kahn order; any topological order gives the same integer max-plus result
  std::vector<int> indeg(n, 0), order;
  std::vector<std::vector<int>> succ(n), preds(n);
  for (int e = 0; e < p->n_edges; ++e) {
    succ[p->edge_from[e]].push_back(p->edge_to[e]);
    preds[p->edge_to[e]].push_back(p->edge_from[e]);
    ++indeg[p->edge_to[e]];
  }
  for (int i = 0; i < n; ++i)
    if (!indeg[i]) order.push_back(i);
  for (size_t k = 0; k < order.size(); ++k)
    for (int s : succ[order[k]])
      if (--indeg[s] == 0) order.push_back(s);
  if (static_cast<int>(order.size()) != n) return loomi::fail(LOOM_INVALID, "CycleError: dag has a cycle");

  EstHeader h{};
  int off = align16(sizeof(EstHeader));
  h.off_radix = off;
  off = align16(off + 4 * n);
  h.off_optoff = off;
  off = align16(off + 4 * (n + 1));
  h.off_topo = off;
  off = align16(off + 4 * n);
  h.off_predoff = off;
  off = align16(off + 4 * (n + 1));
  h.off_pred = off;
  off = align16(off + 4 * std::max(p->n_edges, 1));
  h.off_opt = off;
  off = align16(off + static_cast<int>(sizeof(EstOpt)) * n_opts);
  h.off_wtop = off;
  off = align16(off + 8 * std::max(n, 1));
  if (off > smem_budget)
    return loomi::fail(LOOM_INVALID, "InvalidConfigError: problem image of " + std::to_string(off) +
                                         " bytes exceeds the estimate kernel's shared-memory budget");
  h.n_nodes = n;
  h.n_edges = p->n_edges;
  h.n_opts = n_opts;
  h.bytes = off;
  h.total = im.total;
  // Suffix: the fewest last nodes (<= 3) whose group holds >= 1024 plans
  // (fewer if the whole space is smaller), keeping the group below 2^31.
  h.K = 1;
  h.group = n ? static_cast<uint64_t>(p->radix[n - 1]) : 1;
  while (h.K < std::min(n, kEstMaxK) && h.group < 1024 &&
         h.group * static_cast<uint64_t>(p->radix[n - 1 - h.K]) < (uint64_t(1) << 31)) {
    h.group *= static_cast<uint64_t>(p->radix[n - 1 - h.K]);
    ++h.K;
  }
  if (h.group >= (uint64_t(1) << 31))
    return loomi::fail(LOOM_INVALID, "InvalidConfigError: last node has too many options for the estimate kernel");
  im.blob.assign(off, 0);
  uint8_t* b = im.blob.data();
  std::memcpy(b, &h, sizeof h);
  auto i32 = [&](int o) { return reinterpret_cast<int32_t*>(b + o); };
  int acc = 0, pacc = 0;
  for (int i = 0; i < n; ++i) {
    i32(h.off_radix)[i] = p->radix[i];
    i32(h.off_optoff)[i] = acc;
    acc += p->radix[i];
    i32(h.off_topo)[i] = order[i];
    i32(h.off_predoff)[i] = pacc;
    for (int u : preds[i]) i32(h.off_pred)[pacc++] = u;
  }
  i32(h.off_optoff)[n] = acc;
  i32(h.off_predoff)[n] = pacc;
  uint64_t* wt = reinterpret_cast<uint64_t*>(b + h.off_wtop);
  {  // group index = mixed-radix number of the top digits
    uint64_t w = 1;
    for (int i = n - h.K - 1; i >= 0; --i) {
      wt[i] = w;
      w *= static_cast<uint64_t>(p->radix[i]);
    }
  }
  im.K = h.K;
  {  // latency <= sum over nodes of the largest wall; walls are >= 0 (to_micros of durations)
    int64_t bound = 0;
    bool ok = true;
    for (int i = 0, k = 0; i < n; ++i) {
      int64_t mx = 0;
      for (int j = 0; j < p->radix[i]; ++j, ++k) {
        if (p->wall_us[k] < 0) ok = false;
        mx = std::max(mx, p->wall_us[k]);
      }
      if (mx >= (int64_t(1) << 30)) ok = false;
      bound += mx;
    }
    im.w32 = ok && bound < (int64_t(1) << 30);
  }
  EstOpt* o = reinterpret_cast<EstOpt*>(b + h.off_opt);
  for (int k = 0; k < n_opts; ++k) {
    o[k].g = p->gpu_wh[k];
    o[k].c = p->cpu_wh[k];
    o[k].d = p->dollars[k];
    o[k].w = p->wall_us[k];
    o[k].q = p->quality[k];
  }
  return LOOM_OK;
}

EstStreams to_streams(const loom_estimate_streams* s) {
  return EstStreams{s->latency_us, s->gpu_wh, s->cpu_wh, s->total_wh, s->dollars, s->quality};
}

using RangeFn = void (*)(const uint8_t*, uint32_t, uint64_t, uint64_t, EstStreams);

template <bool W32>
RangeFn range_fn_w(int K) {
  return K == 1 ? estimate_range_kernel<1, W32> : K == 2 ? estimate_range_kernel<2, W32> : estimate_range_kernel<3, W32>;
}

RangeFn range_fn(const EstImage& im) { return im.w32 ? range_fn_w<true>(im.K) : range_fn_w<false>(im.K); }

int range_smem(const EstImage& im) { return static_cast<int>(im.blob.size()) + kEstWarps * est_warp_bytes(im.n); }

// Enqueue the range kernel for plans [begin, end) into device streams.
int launch_range(loom_ctx* c, const EstImage& im, const uint8_t* d_blob, uint64_t begin, uint64_t end,
                 const EstStreams& dev) {
  if (begin >= end) return LOOM_OK;
  const int smem = range_smem(im);
  const RangeFn fn = range_fn(im);
  LOOM_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kEstBlock, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const uint64_t G = reinterpret_cast<const EstHeader*>(im.blob.data())->group;
  const uint64_t groups = (end + G - 1) / G - begin / G;
  const uint64_t want = (groups + kEstWarps - 1) / kEstWarps;
  const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(c->sms) * per_sm)));
  fn<<<grid, kEstBlock, smem, c->stream>>>(d_blob, static_cast<uint32_t>(im.blob.size()), begin, end, dev);
  LOOM_CUDA(cudaGetLastError());
  ++c->launches;
  return LOOM_OK;
}

int check_streams(const loom_estimate_streams* s) {
  if (!s) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null estimate streams");
  return LOOM_OK;
}

}  // namespace

extern "C" {

int loom_estimate_range_device(loom_ctx* c, const loom_problem* p, uint64_t begin, uint64_t end,
                               const loom_estimate_streams* out) {
  if (!c) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null ctx");
  if (int rc = check_streams(out)) return rc;
  EstImage im;
  if (int rc = build_est_image(p, im, kSmemMax - kEstWarps * est_warp_bytes(kMaxNodes) - 64)) return rc;
  end = std::min(end, im.total);
  if (begin >= end) return LOOM_OK;
  LOOM_CUDA(cudaSetDevice(c->device));
  DevBuf<uint8_t> d_blob(c);
  LOOM_CUDA(d_blob.alloc(im.blob.size()));
  LOOM_CUDA(cudaMemcpyAsync(d_blob.p, im.blob.data(), im.blob.size(), cudaMemcpyHostToDevice, c->stream));
  return launch_range(c, im, d_blob.p, begin, end, to_streams(out));
}

int loom_estimate_range(loom_ctx* c, const loom_problem* p, uint64_t begin, uint64_t end,
                        const loom_estimate_streams* out) {
  if (!c) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null ctx");
  if (int rc = check_streams(out)) return rc;
  EstImage im;
  if (int rc = build_est_image(p, im, kSmemMax - kEstWarps * est_warp_bytes(kMaxNodes) - 64)) return rc;
  end = std::min(end, im.total);
  if (begin >= end) return LOOM_OK;
  LOOM_CUDA(cudaSetDevice(c->device));
  DevBuf<uint8_t> d_blob(c);
  LOOM_CUDA(d_blob.alloc(im.blob.size()));
  LOOM_CUDA(cudaMemcpyAsync(d_blob.p, im.blob.data(), im.blob.size(), cudaMemcpyHostToDevice, c->stream));
  // Chunks through device buffers; each chunk's streams are
  // copied back to the caller's arrays on the same stream.
  const uint64_t n = end - begin;
  const uint64_t chunk = std::min<uint64_t>(n, uint64_t(1) << 22);  // 4.2M plans, 185 MB
  const EstStreams h = to_streams(out);
  DevBuf<int64_t> d_lat(c);
  DevBuf<double> d_gpu(c), d_cpu(c), d_tot(c), d_dol(c);
  DevBuf<int32_t> d_q(c);
  EstStreams dev{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  if (h.lat) {
    LOOM_CUDA(d_lat.alloc(chunk));
    dev.lat = d_lat.p;
  }
  if (h.gpu) {
    LOOM_CUDA(d_gpu.alloc(chunk));
    dev.gpu = d_gpu.p;
  }
  if (h.cpu) {
    LOOM_CUDA(d_cpu.alloc(chunk));
    dev.cpu = d_cpu.p;
  }
  if (h.tot) {
    LOOM_CUDA(d_tot.alloc(chunk));
    dev.tot = d_tot.p;
  }
  if (h.dol) {
    LOOM_CUDA(d_dol.alloc(chunk));
    dev.dol = d_dol.p;
  }
  if (h.q) {
    LOOM_CUDA(d_q.alloc(chunk));
    dev.q = d_q.p;
  }
  for (uint64_t b0 = begin; b0 < end; b0 += chunk) {
    const uint64_t b1 = std::min(end, b0 + chunk);
    const uint64_t o = b0 - begin, m = b1 - b0;
    if (int rc = launch_range(c, im, d_blob.p, b0, b1, dev)) return rc;
    if (h.lat) LOOM_CUDA(cudaMemcpyAsync(h.lat + o, dev.lat, m * 8, cudaMemcpyDeviceToHost, c->stream));
    if (h.gpu) LOOM_CUDA(cudaMemcpyAsync(h.gpu + o, dev.gpu, m * 8, cudaMemcpyDeviceToHost, c->stream));
    if (h.cpu) LOOM_CUDA(cudaMemcpyAsync(h.cpu + o, dev.cpu, m * 8, cudaMemcpyDeviceToHost, c->stream));
    if (h.tot) LOOM_CUDA(cudaMemcpyAsync(h.tot + o, dev.tot, m * 8, cudaMemcpyDeviceToHost, c->stream));
    if (h.dol) LOOM_CUDA(cudaMemcpyAsync(h.dol + o, dev.dol, m * 8, cudaMemcpyDeviceToHost, c->stream));
    if (h.q) LOOM_CUDA(cudaMemcpyAsync(h.q + o, dev.q, m * 4, cudaMemcpyDeviceToHost, c->stream));
  }
  LOOM_CUDA(cudaStreamSynchronize(c->stream));
  return LOOM_OK;
}

int loom_estimate_plans(loom_ctx* c, const loom_problem* p, const uint64_t* indices, uint64_t n,
                        const loom_estimate_streams* out) {
  if (!c) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null ctx");
  if (int rc = check_streams(out)) return rc;
  if (n && !indices) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null indices");
  EstImage im;
  if (int rc = build_est_image(p, im, kSmemMax - 64)) return rc;
  for (uint64_t i = 0; i < n; ++i)
    if (indices[i] >= im.total) return loomi::fail(LOOM_INVALID, "InvalidConfigError: plan index out of range");
  if (n == 0) return LOOM_OK;
  LOOM_CUDA(cudaSetDevice(c->device));
  DevBuf<uint8_t> d_blob(c);
  DevBuf<uint64_t> d_idx(c);
  LOOM_CUDA(d_blob.alloc(im.blob.size()));
  LOOM_CUDA(d_idx.alloc(n));
  LOOM_CUDA(cudaMemcpyAsync(d_blob.p, im.blob.data(), im.blob.size(), cudaMemcpyHostToDevice, c->stream));
  LOOM_CUDA(cudaMemcpyAsync(d_idx.p, indices, n * 8, cudaMemcpyHostToDevice, c->stream));
  const EstStreams h = to_streams(out);
  DevBuf<int64_t> d_lat(c);
  DevBuf<double> d_gpu(c), d_cpu(c), d_tot(c), d_dol(c);
  DevBuf<int32_t> d_q(c);
  EstStreams dev{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  if (h.lat) {
    LOOM_CUDA(d_lat.alloc(n));
    dev.lat = d_lat.p;
  }
  if (h.gpu) {
    LOOM_CUDA(d_gpu.alloc(n));
    dev.gpu = d_gpu.p;
  }
  if (h.cpu) {
    LOOM_CUDA(d_cpu.alloc(n));
    dev.cpu = d_cpu.p;
  }
  if (h.tot) {
    LOOM_CUDA(d_tot.alloc(n));
    dev.tot = d_tot.p;
  }
  if (h.dol) {
    LOOM_CUDA(d_dol.alloc(n));
    dev.dol = d_dol.p;
  }
  if (h.q) {
    LOOM_CUDA(d_q.alloc(n));
    dev.q = d_q.p;
  }
  const int smem = static_cast<int>(im.blob.size());
  LOOM_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(estimate_plans_kernel),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const uint64_t want = (n + kEstBlock - 1) / kEstBlock;
  const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(c->sms) * 8)));
  estimate_plans_kernel<<<grid, kEstBlock, smem, c->stream>>>(d_blob.p, static_cast<uint32_t>(im.blob.size()), d_idx.p,
                                                              n, dev);
  LOOM_CUDA(cudaGetLastError());
  ++c->launches;
  if (h.lat) LOOM_CUDA(cudaMemcpyAsync(h.lat, dev.lat, n * 8, cudaMemcpyDeviceToHost, c->stream));
  if (h.gpu) LOOM_CUDA(cudaMemcpyAsync(h.gpu, dev.gpu, n * 8, cudaMemcpyDeviceToHost, c->stream));
  if (h.cpu) LOOM_CUDA(cudaMemcpyAsync(h.cpu, dev.cpu, n * 8, cudaMemcpyDeviceToHost, c->stream));
  if (h.tot) LOOM_CUDA(cudaMemcpyAsync(h.tot, dev.tot, n * 8, cudaMemcpyDeviceToHost, c->stream));
  if (h.dol) LOOM_CUDA(cudaMemcpyAsync(h.dol, dev.dol, n * 8, cudaMemcpyDeviceToHost, c->stream));
  if (h.q) LOOM_CUDA(cudaMemcpyAsync(h.q, dev.q, n * 4, cudaMemcpyDeviceToHost, c->stream));
  LOOM_CUDA(cudaStreamSynchronize(c->stream));
  return LOOM_OK;
}

}  // extern "C"

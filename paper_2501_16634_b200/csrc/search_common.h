// Shared definitions between the host-side problem builder and the sm_100a
// kernels (loom_search.cu).  A "problem image" is one contiguous, 16-byte
// aligned blob: header + topology + per-option tables.  Each CTA copies its
// problem image into shared memory with a single cp.async.bulk (TMA bulk
// copy) and never touches global memory again until the final reduction.
#pragma once

#include <cstdint>

namespace loomk {

constexpr int kMaxNodes = 32;
constexpr int kMaxEdges = 512;
constexpr int kMaxOptions = 6144;
constexpr int kMaxBlobBytes = 200 * 1024;
#ifndef LOOM_BLOCK
#define LOOM_BLOCK 128
#endif
constexpr int kBlock = LOOM_BLOCK;  // threads per CTA of the search / Pareto kernels

// Criterion slots inside the kernels.  FP_A / FP_B are the (at most two)
// floating-point sums the objective ranks on (gpu_wh and/or dollars); they
// are compared after quantize() = llround(v * 1e9) (estimator.hpp:85-87).
enum CritKind : int32_t { kFpA = 0, kFpB = 1, kLat = 2, kQual = 3 };

// How the first criterion is tested in the inner loop.
enum Prim : int32_t { kPrimFp = 0, kPrimLat = 1, kPrimQual = 2 };

// Innermost node's option, 16 bytes = one LDS.128 broadcast per plan.
struct alignas(16) InnerEntry {
  double g;     // FP_A contribution of this option (+inf when w is INT_MAX)
  int32_t w;    // wall_us - inner_wmin (INT32_MAX if the option fails the quality floor)
  int32_t q;    // node quality
};

struct alignas(16) BlobHeader {
  int32_t n_nodes;
  int32_t n_edges;
  int32_t n_opts;
  int32_t K;         // suffix levels handled incrementally (2..4)
  int32_t n_crit;
  int32_t crit[4];   // CritKind per criterion, most significant first
  int32_t prim;      // Prim
  int32_t needs_full;  // slow path must re-evaluate from digits (criteria not carried incrementally)
  int32_t bytes;     // blob size, multiple of 16
  int32_t off_radix;
  int32_t off_optoff;
  int32_t off_topo;
  int32_t off_predoff;
  int32_t off_pred;
  int32_t off_ga;
  int32_t off_gb;
  int32_t off_wall;
  int32_t off_lexw;
  int32_t off_q;
  int32_t off_inner;
  int32_t off_w32;       // int32 walls for the level above the innermost node
  int64_t slo_eff;       // min(latency SLO, sum of max walls): lat <= slo_eff <=> feasible
  int64_t inner_wmin;    // inner walls are stored relative to this
  int64_t pre_wmax;      // largest real wall of the node above the innermost
  uint64_t total;        // plans in the space
  uint64_t r_sub;        // plans per subrow = product of the last K-1 radices
  uint64_t n_sub;        // subrows in the whole space = total / r_sub
  uint64_t group;        // subrows per DP group (unit of work dealt to a warp)
  // Incumbent: every thread starts from the exact record of the greedy
  // seed plan (node-local minima, loom_greedy_seed) when it lies in the
  // searched range, so no thread spends its first plans with empty
  // thresholds -- a job of the multi-tenant batch gives each thread only
  // ~1,000 plans.  Offering a real plan of the range never changes the argmin.
  int32_t has_seed;
  // Energy-then-latency objectives: once a thread's best sits in the lowest
  // achievable energy bucket (qa_floor = quantize of the dag-order fold of
  // per-node minima), no plan can beat it on energy, so its fast latency test
  // tightens from the SLO to the best's latency.
  int32_t tie_lat;
  uint64_t seed_index;
  int64_t qa_floor;
  // Branch and bound (bnb.cuh): per node the options that pass the quality
  // floor in exploration order (best primary value first; int32 at optoff),
  // their count, per-node bounds over those options, and the plans below a
  // prefix of length k (uint64[n+1], rk[n] = 1).
  int32_t off_perm;
  int32_t off_nok;
  int32_t off_bmin;
  int32_t off_rk;
  // Latency bound caching: with the first k digits fixed, a node is
  // "settled" when it and all its ancestors are among them (its finish time
  // is then the same for every plan below).  uns: per depth k the nodes NOT
  // settled, in topological order; nsettle: per depth k the nodes that become
  // settled when node k is fixed.  Both are int32 CSR: [n+1] offsets, entries.
  int32_t off_uns;
  int32_t off_nsettle;
  int32_t pad_bnb[2];
};

// Per-node bounds over the options that pass the quality floor: the smallest
// FP_A / FP_B term and wall, the largest quality and identifier-rank term
// (smallest lexw), for subtree lower bounds.
struct alignas(16) BnbMin {
  double a;
  double b;
  int64_t w;
  uint64_t lex;
  int32_t q;
  int32_t o_wall;  // option (index within the node) of the smallest wall, ties to the smaller FP_A term
  int32_t pad[2];
};

// A candidate / winner inside the kernels: the quantized criteria, exact
// latency and quality, the identifier rank and the plan index.
struct Rec {
  int64_t qa;
  int64_t qb;
  int64_t lat;
  uint64_t lexkey;
  uint64_t index;
  int32_t qual;
  int32_t found;
};

// Innermost table of a single-problem launch, passed as a kernel parameter so
// the fast path reads it as constant-bank operands instead of registers.
struct InnerParams {
  double g[16];    // +inf where w is INT_MAX (padding / quality-floor failure)
  int32_t w[16];
  int32_t gh[16];  // high word of g: g <= t  =>  gh <= hi(t) for g >= 0 (ALU-pipe form of the energy test)
  float gf[16];    // g rounded down to binary32: g <= t  =>  gf <= round_up_f32(t) (FP32 form)
  double gu[16];   // FP_A terms of the node above the innermost (its radix <= 16), for the unrolled sweep
};

// One plan's Pareto coordinates (40 bytes; same layout as loom_point).
struct ParetoPoint {
  uint64_t index;
  double dollars;
  double gpu_wh;
  int64_t latency_us;
  int32_t quality;
  int32_t pad;
};

// Per-job device counters (global memory, zero between launches): the CTA
// arrival ticket of the final reduction, the next DP group to deal out and the
// job-wide energy bound.  The last CTA to arrive resets them.
struct alignas(16) JobSync {
  unsigned ticket;
  unsigned pad;
  unsigned long long next_group;
  // INT64_MAX - (quantized primary FP criterion of the best feasible plan
  // found by any thread of the job so far); 0 = none.  atomicMax only.
  unsigned long long best_neg;
  unsigned long long pad2;
};

// Per-job state of the branch-and-bound search (bnb.cuh), zero between
// launches (the last CTA resets it).  The task counter, the work counter and
// the published best sit on separate 128-byte lines: warps hammer the first
// and read the last at every DFS step.
struct alignas(128) BnbSync {
  unsigned long long next_task;
  unsigned char pad0[120];
  unsigned long long work;  // child evaluations so far (flushed per warp)
  unsigned abort;           // evaluation budget exhausted
  unsigned ticket;          // CTA arrivals of the final reduction
  unsigned long long leaves;  // complete plans evaluated exactly (flushed per warp)
  unsigned char pad1[104];
  unsigned lock;
  unsigned seq;             // even: best is stable; odd: a writer is updating it
  unsigned pad2[2];
  Rec best;
  unsigned char pad3[64];
};

// Per-job state of the frontier (level-synchronous) branch and bound
// (frontier.cuh), zero between launches (the last CTA to finish resets it):
// survivors per depth, parents handed out per depth, the grid barrier, the
// exit ticket and launch evidence.
struct alignas(128) BfsSync {
  unsigned long long count[kMaxNodes + 1];  // frontier entries per depth
  unsigned long long next[kMaxNodes + 1];   // parents handed out per depth (dynamic distribution)
  unsigned bar_count;
  unsigned bar_gen;
  unsigned ticket;   // CTA exits: the last one writes the result and resets
  unsigned overflow;
  unsigned long long evals;   // children evaluated (subtree bounds + leaves)
  unsigned long long leaves;  // complete plans evaluated exactly
  unsigned long long max_frontier;
  unsigned long long pad;
};

// One surviving prefix of the frontier (48 bytes): its digits bit-packed
// (node i at BfsParams.shift[i]), the exact dag-order folds of its FP terms,
// its bound on the first criterion and the minimum quality of its nodes.
// The latency terms of the next node are computed when the prefix is
// expanded (frontier.cuh), not stored.
struct alignas(16) FrontierEntry {
  uint64_t dig;
  double fa;
  double fb;
  int64_t key;  // the prefix's bound on the first criterion (larger = worse), re-checked before expanding
  int32_t q;
  int32_t live;  // 0: a dropped child slot of a redundant level (frontier.cuh)
  uint64_t pad;
};

// Per-job launch descriptor (global memory).
struct JobDesc {
  uint64_t blob_off;     // byte offset in the blob arena
  uint64_t begin;        // plans [begin, end)
  uint64_t end;
  uint64_t head_end;     // partial plans [begin, head_end) ...
  uint64_t tail_begin;   // ... and [tail_begin, end): one-plan-per-thread path
  uint64_t sub_lo;       // whole subrows [sub_lo, sub_hi): hierarchical path
  uint64_t sub_hi;
  uint32_t blob_bytes;
  uint32_t has_seed;     // an incumbent plan of [begin, end) every thread starts from
  uint64_t seed;
};

}  // namespace loomk

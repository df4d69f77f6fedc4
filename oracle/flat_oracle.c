/*
 * ORACLE TEST INFRASTRUCTURE -- NOT PRODUCT CODE.  Only tests/, the smoke()
 * check and bench.py's cpu_baseline / reference legs may load this library,
 * and only as the checker.
 *
 * A plain-C restatement of the reference's per-plan work, fed with the
 * per-node option tables produced by oracle/lower.py (itself a restatement of
 * node_options / plan_node_execution).  It deliberately does NOT share the
 * product's tricks: no max-plus decomposition, no identifier ranks, no
 * prefix folds.  Each plan is decoded and evaluated from scratch:
 *
 *   decode          ConfigEnumerator odometer, last node fastest   optimizer.hpp:131-143
 *   estimate        folds in dag.nodes order, value*path_count     estimator.hpp:46-67
 *                   finish-time recursion in topological order     estimator.hpp:69-76
 *   floor           quality >= floor                               estimator.hpp:118-121
 *   objective_less  quantize = llround(v*1e9), criteria in order,  estimator.hpp:85-116
 *                   residual tie -> strcmp of identifier() strings config.hpp:49-61
 *   argmin          keep first-best in enumeration order           optimizer.hpp:177-187
 *   pareto_filter   4-D dominance on raw values, stable order      optimizer.hpp:153-171
 *
 * plus the config-3 latency SLO extension (latency_us <= slo) as an extra
 * feasibility test.  Threads split [begin, end) into contiguous slices and the
 * per-slice winners are reduced with the same order, lowest slice first, so
 * the result equals the sequential one.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_MAX_NODES 64

typedef struct {
  int n_nodes;
  int n_edges;
  const int* radix;            /* [n_nodes] */
  const int64_t* wall;         /* [sum radix] NodePlan.wall_us              */
  const double* gpu;           /* [sum radix] NodePlan.gpu_wh  (raw, x1)     */
  const double* cpu;           /* [sum radix] NodePlan.cpu_wh                */
  const double* dol;           /* [sum radix] NodePlan.dollars               */
  const int* path_count;       /* [sum radix]                                */
  const int* quality;          /* [sum radix] node_quality                   */
  const char* const* token;    /* [sum radix] "<id>=<impl>[...]p<k>;"        */
  const int* id_order;         /* [n_nodes] node indices in sorted-id order  */
  const int* topo;             /* [n_nodes] reference topological_order      */
  const int* edge_from;        /* [n_edges]                                  */
  const int* edge_to;          /* [n_edges]                                  */
} or_problem;

typedef struct {
  int n_criteria;
  int criteria[4]; /* 0 dollars, 1 energy, 2 latency, 3 quality (workflow.hpp:67) */
  int has_floor;
  int floor;
  int has_slo;
  int64_t slo;
} or_objective;

typedef struct {
  uint64_t index;
  int64_t latency_us;
  double gpu_wh, cpu_wh, total_wh, dollars;
  int quality;
  int found;
} or_estimate;

typedef struct {
  const or_problem* p;
  int off[OR_MAX_NODES + 1];
  int npred[OR_MAX_NODES];
  int pred[OR_MAX_NODES][OR_MAX_NODES * 4];
} or_ctx;

static int ctx_init(or_ctx* c, const or_problem* p) {
  if (p->n_nodes > OR_MAX_NODES) return -1;
  c->p = p;
  c->off[0] = 0;
  for (int i = 0; i < p->n_nodes; ++i) {
    c->off[i + 1] = c->off[i] + p->radix[i];
    c->npred[i] = 0;
  }
  for (int e = 0; e < p->n_edges; ++e) {
    const int t = p->edge_to[e];
    if (c->npred[t] >= OR_MAX_NODES * 4) return -1;
    c->pred[t][c->npred[t]++] = p->edge_from[e];
  }
  return 0;
}

/* estimate(): one plan from its digits. */
static void evaluate(const or_ctx* c, const int* d, or_estimate* e) {
  const or_problem* p = c->p;
  double gpu = 0.0, cpu = 0.0, dol = 0.0;
  int q = INT32_MAX;
  for (int i = 0; i < p->n_nodes; ++i) {
    const int o = c->off[i] + d[i];
    const double k = (double)p->path_count[o];
    gpu += p->gpu[o] * k;
    cpu += p->cpu[o] * k;
    dol += p->dol[o] * k;
    if (p->quality[o] < q) q = p->quality[o];
  }
  if (p->n_nodes == 0) q = 0;
  int64_t finish[OR_MAX_NODES];
  int64_t lat = 0;
  for (int t = 0; t < p->n_nodes; ++t) {
    const int v = p->topo[t];
    int64_t start = 0;
    for (int k = 0; k < c->npred[v]; ++k)
      if (finish[c->pred[v][k]] > start) start = finish[c->pred[v][k]];
    finish[v] = start + p->wall[c->off[v] + d[v]];
    if (finish[v] > lat) lat = finish[v];
  }
  e->latency_us = lat;
  e->gpu_wh = gpu;
  e->cpu_wh = cpu;
  e->total_wh = gpu + cpu;
  e->dollars = dol;
  e->quality = q;
  e->found = 1;
}

static int64_t quantize(double v) { return (int64_t)llround(v * 1e9); }

/* identifier(a) < identifier(b), comparing the concatenated strings. */
static int identifier_less(const or_ctx* c, const int* da, const int* db) {
  const or_problem* p = c->p;
  /* walk both identifiers character by character without materialising */
  int ia = 0, ib = 0;
  const char* sa = NULL;
  const char* sb = NULL;
  for (;;) {
    while ((!sa || !*sa) && ia < p->n_nodes) {
      const int v = p->id_order[ia++];
      sa = p->token[c->off[v] + da[v]];
    }
    while ((!sb || !*sb) && ib < p->n_nodes) {
      const int v = p->id_order[ib++];
      sb = p->token[c->off[v] + db[v]];
    }
    const int ea = !sa || !*sa, eb = !sb || !*sb;
    if (ea || eb) return ea && !eb;
    if (*sa != *sb) return (unsigned char)*sa < (unsigned char)*sb;
    ++sa;
    ++sb;
  }
}

static int objective_less(const or_ctx* c, const or_objective* o, const or_estimate* a, const int* da,
                          const or_estimate* b, const int* db) {
  for (int i = 0; i < o->n_criteria; ++i) {
    switch (o->criteria[i]) {
      case 0: {
        const int64_t qa = quantize(a->dollars), qb = quantize(b->dollars);
        if (qa != qb) return qa < qb;
        break;
      }
      case 1: {
        const int64_t qa = quantize(a->gpu_wh), qb = quantize(b->gpu_wh);
        if (qa != qb) return qa < qb;
        break;
      }
      case 2:
        if (a->latency_us != b->latency_us) return a->latency_us < b->latency_us;
        break;
      default:
        if (a->quality != b->quality) return a->quality > b->quality;
        break;
    }
  }
  return identifier_less(c, da, db);
}

static int feasible(const or_objective* o, const or_estimate* e) {
  if (o->has_floor && e->quality < o->floor) return 0;
  if (o->has_slo && e->latency_us > o->slo) return 0;
  return 1;
}

static void decode(const or_problem* p, uint64_t index, int* d) {
  for (int i = p->n_nodes - 1; i >= 0; --i) {
    d[i] = (int)(index % (uint64_t)p->radix[i]);
    index /= (uint64_t)p->radix[i];
  }
}

static void advance(const or_problem* p, int* d) {
  for (int i = p->n_nodes - 1; i >= 0; --i) {
    if (++d[i] < p->radix[i]) return;
    d[i] = 0;
  }
}

typedef struct {
  const or_ctx* c;
  const or_objective* o;
  uint64_t lo, hi;
  or_estimate best;
  int bd[OR_MAX_NODES];
} argmin_job;

static void* argmin_worker(void* arg) {
  argmin_job* j = (argmin_job*)arg;
  const or_problem* p = j->c->p;
  int d[OR_MAX_NODES];
  j->best.found = 0;
  if (j->lo >= j->hi) return NULL;
  decode(p, j->lo, d);
  for (uint64_t i = j->lo; i < j->hi; ++i) {
    or_estimate e;
    evaluate(j->c, d, &e);
    e.index = i;
    if (feasible(j->o, &e) && (!j->best.found || objective_less(j->c, j->o, &e, d, &j->best, j->bd))) {
      j->best = e;
      memcpy(j->bd, d, sizeof(int) * (size_t)p->n_nodes);
    }
    advance(p, d);
  }
  return NULL;
}

/* Returns 0 and out->found=1 on success, out->found=0 if nothing feasible. */
int oracle_argmin(const or_problem* p, const or_objective* o, uint64_t begin, uint64_t end, int threads,
                  or_estimate* out) {
  or_ctx* c = (or_ctx*)malloc(sizeof(or_ctx));
  if (!c || ctx_init(c, p)) {
    free(c);
    return -1;
  }
  if (threads < 1) threads = 1;
  argmin_job* jobs = (argmin_job*)calloc((size_t)threads, sizeof(argmin_job));
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  const uint64_t n = end > begin ? end - begin : 0;
  for (int t = 0; t < threads; ++t) {
    jobs[t].c = c;
    jobs[t].o = o;
    jobs[t].lo = begin + (uint64_t)((__uint128_t)n * (uint64_t)t / (uint64_t)threads);
    jobs[t].hi = begin + (uint64_t)((__uint128_t)n * (uint64_t)(t + 1) / (uint64_t)threads);
    pthread_create(&tid[t], NULL, argmin_worker, &jobs[t]);
  }
  int w = -1;
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  for (int t = 0; t < threads; ++t) {
    if (!jobs[t].best.found) continue;
    if (w < 0 || objective_less(c, o, &jobs[t].best, jobs[t].bd, &jobs[w].best, jobs[w].bd)) w = t;
  }
  memset(out, 0, sizeof *out);
  if (w >= 0) *out = jobs[w].best;
  free(jobs);
  free(tid);
  free(c);
  return 0;
}

/* Estimate of every plan in [begin, end) (small ranges), for golden checks. */
int oracle_estimates(const or_problem* p, uint64_t begin, uint64_t end, or_estimate* out) {
  or_ctx* c = (or_ctx*)malloc(sizeof(or_ctx));
  if (!c || ctx_init(c, p)) {
    free(c);
    return -1;
  }
  int d[OR_MAX_NODES];
  if (begin < end) decode(p, begin, d);
  for (uint64_t i = begin; i < end; ++i) {
    evaluate(c, d, &out[i - begin]);
    out[i - begin].index = i;
    advance(p, d);
  }
  free(c);
  return 0;
}

/* ---- pareto_filter over plans [begin, end) in enumeration order ---------- */

static int dominates(const or_estimate* a, const or_estimate* b) {
  const int no_worse = a->dollars <= b->dollars && a->gpu_wh <= b->gpu_wh && a->latency_us <= b->latency_us &&
                       a->quality >= b->quality;
  const int strictly = a->dollars < b->dollars || a->gpu_wh < b->gpu_wh || a->latency_us < b->latency_us ||
                       a->quality > b->quality;
  return no_worse && strictly;
}

typedef struct {
  or_estimate* v;
  size_t n, cap;
} frontier;

/* Streaming exact frontier: a new point is dropped if a kept point dominates
 * it, otherwise it evicts the kept points it dominates.  By transitivity the
 * survivors are exactly the non-dominated points; insertion keeps index order. */
static int frontier_push(frontier* f, const or_estimate* e) {
  for (size_t k = 0; k < f->n; ++k)
    if (dominates(&f->v[k], e)) return 0;
  size_t w = 0;
  for (size_t k = 0; k < f->n; ++k)
    if (!dominates(e, &f->v[k])) f->v[w++] = f->v[k];
  f->n = w;
  if (f->n == f->cap) {
    f->cap = f->cap ? 2 * f->cap : 256;
    or_estimate* nv = (or_estimate*)realloc(f->v, f->cap * sizeof(or_estimate));
    if (!nv) return -1;
    f->v = nv;
  }
  f->v[f->n++] = *e;
  return 0;
}

typedef struct {
  const or_ctx* c;
  uint64_t lo, hi;
  frontier f;
} pareto_job;

static void* pareto_worker(void* arg) {
  pareto_job* j = (pareto_job*)arg;
  const or_problem* p = j->c->p;
  int d[OR_MAX_NODES];
  if (j->lo >= j->hi) return NULL;
  decode(p, j->lo, d);
  for (uint64_t i = j->lo; i < j->hi; ++i) {
    or_estimate e;
    evaluate(j->c, d, &e);
    e.index = i;
    frontier_push(&j->f, &e);
    advance(p, d);
  }
  return NULL;
}

/* Writes up to cap frontier points (index order) into out; *count = size. */
int oracle_pareto(const or_problem* p, uint64_t begin, uint64_t end, int threads, or_estimate* out, uint64_t cap,
                  uint64_t* count) {
  or_ctx* c = (or_ctx*)malloc(sizeof(or_ctx));
  if (!c || ctx_init(c, p)) {
    free(c);
    return -1;
  }
  if (threads < 1) threads = 1;
  pareto_job* jobs = (pareto_job*)calloc((size_t)threads, sizeof(pareto_job));
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  const uint64_t n = end > begin ? end - begin : 0;
  for (int t = 0; t < threads; ++t) {
    jobs[t].c = c;
    jobs[t].lo = begin + (uint64_t)((__uint128_t)n * (uint64_t)t / (uint64_t)threads);
    jobs[t].hi = begin + (uint64_t)((__uint128_t)n * (uint64_t)(t + 1) / (uint64_t)threads);
    pthread_create(&tid[t], NULL, pareto_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  /* union of slice frontiers in index order, filtered again */
  frontier all = {0, 0, 0};
  for (int t = 0; t < threads; ++t) {
    for (size_t k = 0; k < jobs[t].f.n; ++k) frontier_push(&all, &jobs[t].f.v[k]);
    free(jobs[t].f.v);
  }
  *count = all.n;
  for (size_t k = 0; k < all.n && k < cap; ++k) out[k] = all.v[k];
  free(all.v);
  free(jobs);
  free(tid);
  free(c);
  return 0;
}

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

/* ---- exact branch-and-bound argmin over the WHOLE plan space --------------
 *
 * For plan spaces the flat loop cannot finish (C3: 1.1e12 plans).  A DFS over
 * the nodes in enumeration order; every subtree (the first i digits fixed) is
 * bounded by a componentwise lower bound of its plans' criteria:
 *   energy / dollars  the dag-order left fold with every free node at its
 *                     minimum (FP addition rounds monotonically, so the fold is
 *                     monotone in every term; llround is monotone too),
 *   latency           the finish-time recursion with free nodes at their
 *                     minimum wall (max-plus is monotone),
 *   quality           min(prefix quality, max over free nodes) (upper bound).
 * A subtree is dropped when its bound is infeasible (latency > SLO) or
 * lexicographically STRICTLY worse than the incumbent under the criteria
 * list: then every plan in it is strictly worse on some criterion with all
 * earlier ones equal or worse, so none can be the argmin.  Ties on every
 * criterion are never pruned (the identifier decides).  Options failing the
 * quality floor are never taken (a plan's quality is the min over nodes).
 * Leaves are evaluated with evaluate() + feasible() + objective_less() above,
 * so the result is the restated reference argmin.  Threads take top-level
 * subtrees from a shared counter and share the incumbent through a mutex;
 * the order is strict and total, so the answer does not depend on timing. */

typedef struct {
  const or_ctx* c;
  const or_objective* o;
  int n;
  int topo_pos[OR_MAX_NODES];
  double min_gpu[OR_MAX_NODES], min_dol[OR_MAX_NODES];
  int64_t min_wall[OR_MAX_NODES];
  int max_q[OR_MAX_NODES];
  int n_ok[OR_MAX_NODES];
  int* order; /* per node: allowed options in exploration order (node-major, off[]) */
  int split;  /* nodes fixed per top-level task */
  uint64_t n_tasks;
  uint64_t next_task;
  pthread_mutex_t mu;
  or_estimate best;
  int bd[OR_MAX_NODES];
  uint64_t visited;
} bnb_shared;

typedef struct {
  bnb_shared* s;
  or_estimate best;
  int bd[OR_MAX_NODES];
  int d[OR_MAX_NODES];
  double fg[OR_MAX_NODES + 1], fd[OR_MAX_NODES + 1]; /* prefix folds */
  int fq[OR_MAX_NODES + 1];
  uint64_t visited;
} bnb_worker;

static int opt_passes_floor(const bnb_shared* s, int o) {
  return !s->o->has_floor || s->c->p->quality[o] >= s->o->floor;
}

/* Lower bound of every plan whose first `depth` digits are w->d[0..depth). */
static void bnb_bound(const bnb_worker* w, int depth, or_estimate* lb) {
  const bnb_shared* s = w->s;
  const or_problem* p = s->c->p;
  double g = w->fg[depth], dl = w->fd[depth];
  int q = w->fq[depth];
  for (int i = depth; i < s->n; ++i) {
    g += s->min_gpu[i];
    dl += s->min_dol[i];
    if (s->max_q[i] < q) q = s->max_q[i];
  }
  int64_t fin[OR_MAX_NODES];
  int64_t lat = 0;
  for (int t = 0; t < s->n; ++t) {
    const int v = p->topo[t];
    int64_t st = 0;
    for (int k = 0; k < s->c->npred[v]; ++k)
      if (fin[s->c->pred[v][k]] > st) st = fin[s->c->pred[v][k]];
    fin[v] = st + (v < depth ? p->wall[s->c->off[v] + w->d[v]] : s->min_wall[v]);
    if (fin[v] > lat) lat = fin[v];
  }
  lb->latency_us = lat;
  lb->gpu_wh = g;
  lb->dollars = dl;
  lb->quality = s->n == 0 ? 0 : q;
}

/* 1 iff every plan bounded by lb is infeasible or strictly worse than best. */
static int bnb_prune(const bnb_shared* s, const or_estimate* lb, const or_estimate* best) {
  const or_objective* o = s->o;
  if (o->has_slo && lb->latency_us > o->slo) return 1;
  if (o->has_floor && lb->quality < o->floor) return 1;
  if (!best->found) return 0;
  for (int i = 0; i < o->n_criteria; ++i) {
    int64_t a, b;
    switch (o->criteria[i]) {
      case 0: a = quantize(lb->dollars); b = quantize(best->dollars); break;
      case 1: a = quantize(lb->gpu_wh); b = quantize(best->gpu_wh); break;
      case 2: a = lb->latency_us; b = best->latency_us; break;
      default: a = -(int64_t)lb->quality; b = -(int64_t)best->quality; break;
    }
    if (a > b) return 1;
    if (a < b) return 0;
  }
  return 0;
}

static void bnb_offer(bnb_worker* w, const or_estimate* e, const int* d) {
  const bnb_shared* s = w->s;
  if (!feasible(s->o, e)) return;
  if (w->best.found && !objective_less(s->c, s->o, e, d, &w->best, w->bd)) return;
  w->best = *e;
  memcpy(w->bd, d, sizeof(int) * (size_t)s->n);
}

static void bnb_dfs(bnb_worker* w, int depth) {
  const bnb_shared* s = w->s;
  const or_problem* p = s->c->p;
  const int off = s->c->off[depth];
  for (int k = 0; k < s->n_ok[depth]; ++k) {
    const int opt = s->order[off + k];
    const int o = off + opt;
    w->d[depth] = opt;
    const double pc = (double)p->path_count[o];
    w->fg[depth + 1] = w->fg[depth] + p->gpu[o] * pc;
    w->fd[depth + 1] = w->fd[depth] + p->dol[o] * pc;
    w->fq[depth + 1] = p->quality[o] < w->fq[depth] ? p->quality[o] : w->fq[depth];
    ++w->visited;
    if (depth + 1 == s->n) {
      or_estimate e;
      evaluate(s->c, w->d, &e);
      uint64_t idx = 0;
      for (int i = 0; i < s->n; ++i) idx = idx * (uint64_t)p->radix[i] + (uint64_t)w->d[i];
      e.index = idx;
      bnb_offer(w, &e, w->d);
      continue;
    }
    or_estimate lb;
    bnb_bound(w, depth + 1, &lb);
    if (bnb_prune(s, &lb, &w->best)) continue;
    bnb_dfs(w, depth + 1);
  }
}

static void* bnb_thread(void* arg) {
  bnb_worker* w = (bnb_worker*)arg;
  bnb_shared* s = w->s;
  const or_problem* p = s->c->p;
  for (;;) {
    pthread_mutex_lock(&s->mu);
    const uint64_t t = s->next_task++;
    if (s->best.found && (!w->best.found || objective_less(s->c, s->o, &s->best, s->bd, &w->best, w->bd))) {
      w->best = s->best;
      memcpy(w->bd, s->bd, sizeof(int) * (size_t)s->n);
    }
    pthread_mutex_unlock(&s->mu);
    if (t >= s->n_tasks) break;
    /* task t: the split top nodes take the t-th combination of their allowed options */
    uint64_t x = t;
    int ok = 1;
    w->fg[0] = 0.0;
    w->fd[0] = 0.0;
    w->fq[0] = INT32_MAX;
    int rank[OR_MAX_NODES];
    for (int i = s->split - 1; i >= 0; --i) {
      rank[i] = (int)(x % (uint64_t)s->n_ok[i]);
      x /= (uint64_t)s->n_ok[i];
    }
    for (int i = 0; i < s->split; ++i) {
      const int opt = s->order[s->c->off[i] + rank[i]];
      const int o = s->c->off[i] + opt;
      w->d[i] = opt;
      const double pc = (double)p->path_count[o];
      w->fg[i + 1] = w->fg[i] + p->gpu[o] * pc;
      w->fd[i + 1] = w->fd[i] + p->dol[o] * pc;
      w->fq[i + 1] = p->quality[o] < w->fq[i] ? p->quality[o] : w->fq[i];
    }
    if (s->split == s->n) {
      or_estimate e;
      evaluate(s->c, w->d, &e);
      uint64_t idx = 0;
      for (int i = 0; i < s->n; ++i) idx = idx * (uint64_t)p->radix[i] + (uint64_t)w->d[i];
      e.index = idx;
      bnb_offer(w, &e, w->d);
    } else {
      or_estimate lb;
      bnb_bound(w, s->split, &lb);
      if (!bnb_prune(s, &lb, &w->best)) bnb_dfs(w, s->split);
    }
    (void)ok;
    pthread_mutex_lock(&s->mu);
    if (w->best.found && (!s->best.found || objective_less(s->c, s->o, &w->best, w->bd, &s->best, s->bd))) {
      s->best = w->best;
      memcpy(s->bd, w->bd, sizeof(int) * (size_t)s->n);
    }
    pthread_mutex_unlock(&s->mu);
  }
  return NULL;
}

static const bnb_shared* g_sort_s;
static int g_sort_node;
static int bnb_cmp(const void* a, const void* b) {
  /* exploration order: the primary criterion's own value, then the option index */
  const bnb_shared* s = g_sort_s;
  const or_problem* p = s->c->p;
  const int oa = s->c->off[g_sort_node] + *(const int*)a, ob = s->c->off[g_sort_node] + *(const int*)b;
  double va = 0, vb = 0;
  const int prim = s->o->n_criteria ? s->o->criteria[0] : 2;
  switch (prim) {
    case 0: va = p->dol[oa] * p->path_count[oa]; vb = p->dol[ob] * p->path_count[ob]; break;
    case 1: va = p->gpu[oa] * p->path_count[oa]; vb = p->gpu[ob] * p->path_count[ob]; break;
    case 2: va = (double)p->wall[oa]; vb = (double)p->wall[ob]; break;
    default: va = -(double)p->quality[oa]; vb = -(double)p->quality[ob]; break;
  }
  if (va != vb) return va < vb ? -1 : 1;
  return oa < ob ? -1 : oa > ob;
}

/* Exact argmin over the whole space; *visited = subtrees + leaves expanded. */
int oracle_argmin_bnb(const or_problem* p, const or_objective* o, int threads, or_estimate* out,
                      uint64_t* visited) {
  or_ctx* c = (or_ctx*)malloc(sizeof(or_ctx));
  if (!c || ctx_init(c, p)) {
    free(c);
    return -1;
  }
  if (threads < 1) threads = 1;
  bnb_shared* s = (bnb_shared*)calloc(1, sizeof(bnb_shared));
  s->c = c;
  s->o = o;
  s->n = p->n_nodes;
  s->order = (int*)malloc(sizeof(int) * (size_t)(c->off[p->n_nodes] + 1));
  memset(out, 0, sizeof *out);
  int empty = p->n_nodes == 0;
  for (int i = 0; i < p->n_nodes; ++i) {
    int k = 0;
    s->min_gpu[i] = INFINITY;
    s->min_dol[i] = INFINITY;
    s->min_wall[i] = INT64_MAX;
    s->max_q[i] = INT32_MIN;
    for (int j = 0; j < p->radix[i]; ++j) {
      const int oi = c->off[i] + j;
      if (!opt_passes_floor(s, oi)) continue;
      s->order[c->off[i] + k++] = j;
      const double pc = (double)p->path_count[oi];
      if (p->gpu[oi] * pc < s->min_gpu[i]) s->min_gpu[i] = p->gpu[oi] * pc;
      if (p->dol[oi] * pc < s->min_dol[i]) s->min_dol[i] = p->dol[oi] * pc;
      if (p->wall[oi] < s->min_wall[i]) s->min_wall[i] = p->wall[oi];
      if (p->quality[oi] > s->max_q[i]) s->max_q[i] = p->quality[oi];
    }
    s->n_ok[i] = k;
    if (k == 0) empty = 1;
    g_sort_s = s;
    g_sort_node = i;
    qsort(s->order + c->off[i], (size_t)k, sizeof(int), bnb_cmp);
  }
  if (!empty) {
    s->split = 0;
    s->n_tasks = 1;
    while (s->split < p->n_nodes && s->n_tasks < 64u * (uint64_t)threads) s->n_tasks *= (uint64_t)s->n_ok[s->split++];
    pthread_mutex_init(&s->mu, NULL);
    bnb_worker* w = (bnb_worker*)calloc((size_t)threads, sizeof(bnb_worker));
    pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
      w[t].s = s;
      pthread_create(&tid[t], NULL, bnb_thread, &w[t]);
    }
    uint64_t vis = 0;
    for (int t = 0; t < threads; ++t) {
      pthread_join(tid[t], NULL);
      vis += w[t].visited;
    }
    if (visited) *visited = vis;
    if (s->best.found) *out = s->best;
    pthread_mutex_destroy(&s->mu);
    free(w);
    free(tid);
  } else if (visited) {
    *visited = 0;
  }
  free(s->order);
  free(s);
  free(c);
  return 0;
}

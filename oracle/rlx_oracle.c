/*
 * rlx_oracle.c — CPU restatement of the reference look-ahead chooser.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the checker, never the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. The product path (the CUDA evaluator
 * in paper_2604_23838_b200/csrc) neither links nor calls it.
 *
 * Parity pinning: checked against golden vectors produced by the live
 * reference (tests/golden/make_golden.py): full recorded schedules of the
 * trap fixture, random_small_instance(0..99), config 1, and per-candidate
 * (cost, finish) keys at configs 1-5 (tests/test_oracle.py).
 *
 * It restates, in plain C over the raw decision-state arrays of
 * include/rlx.h, the following reference functions (rlmux/scheduler.py):
 *   enumerate_actions        :648-703   (plus the max_merge cap)
 *   ExecState apply/advance  :445-627   (_start_member :460, _apply_merge :517)
 *   _window_ids              :710-748
 *   _suffix_lengths          :751-770
 *   action_finish_estimate   :773-789
 *   _rerated_pair_end        :792-800
 *   _best_pair_action        :803-828
 *   _complete_window         :831-869
 *   window_cost              :878-899
 *   candidate_cost           :902-918
 *   chooser argmin           :963-972
 * It is deliberately straightforward (clone-and-simulate per candidate, like
 * the reference) but keeps a pending-predecessor count per node instead of
 * rescanning predecessor sets, so readiness is O(1).
 * Floating point: compiled with -ffp-contract=off; every expression keeps
 * the reference's left-to-right binary64 evaluation order.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/rlx.h"

#define EPS 1e-9
static const double MEM_GRIDV[4] = {0.20, 0.40, 0.60, 0.80};
static const double DEFAULT_MEM[7] = {0.5, 0.55, 0.4, 0.3, 0.5, 0.6, 0.05};

/* ------------------------------------------------------------------ */
typedef struct {
  int n, cap;
  int* a;
} ivec;

static void iv_push(ivec* v, int x) {
  if (v->n == v->cap) {
    v->cap = v->cap ? v->cap * 2 : 4;
    v->a = (int*)realloc(v->a, sizeof(int) * v->cap);
  }
  v->a[v->n++] = x;
}
static int iv_has(const ivec* v, int x) {
  for (int i = 0; i < v->n; i++)
    if (v->a[i] == x) return 1;
  return 0;
}
static void iv_del(ivec* v, int x) {
  for (int i = 0; i < v->n; i++)
    if (v->a[i] == x) {
      v->a[i] = v->a[--v->n];
      return;
    }
}
static void iv_copy(ivec* d, const ivec* s) {
  d->n = s->n;
  d->cap = s->n;
  d->a = s->n ? (int*)malloc(sizeof(int) * s->n) : NULL;
  if (s->n) memcpy(d->a, s->a, sizeof(int) * s->n);
}

/* ------------------------------------------------------------------ */
typedef struct Ctx {
  const RlxInstanceDesc* in;
  int W, P;
  const char** pipe_name;
  int* pipe_rank; /* sorted pipeline-id order */
} Ctx;

typedef struct Graph {
  int n; /* slots (dead slots possible after a merge) */
  uint8_t* alive;
  int *pipe, *worker, *kind;
  double *dur, *mem, *migc;
  int64_t *rem, *act, *ctx;
  char** id;
  ivec *preds, *succs;
  int* name_rank; /* rank by (pipeline id, id) among alive nodes */
  int* id_rank;   /* rank by id among alive nodes                */
  int owned_ids;  /* ids allocated by this graph (merged nodes)   */
} Graph;

typedef struct St {
  const Ctx* c;
  Graph* g;
  int own_graph;
  double now;
  uint8_t *done, *run, *tw;
  double* done_t;
  int* pend; /* uncompleted predecessors */
  double *rate, *pre, *work, *twend, *mprefix;
  int* partner;
  int* nmem; /* members per worker */
  double* grant; /* [W*P] last mem grant, NaN = none */
  int err;
  char msg[160];
} St;

static const Ctx* g_sort_ctx;
static const Graph* g_sort_graph;
static int cmp_name(const void* x, const void* y) {
  int a = *(const int*)x, b = *(const int*)y;
  const Graph* g = g_sort_graph;
  int c = strcmp(g_sort_ctx->pipe_name[g->pipe[a]], g_sort_ctx->pipe_name[g->pipe[b]]);
  if (c) return c;
  return strcmp(g->id[a], g->id[b]);
}
static int cmp_id(const void* x, const void* y) {
  int a = *(const int*)x, b = *(const int*)y;
  return strcmp(g_sort_graph->id[a], g_sort_graph->id[b]);
}
static pthread_mutex_t g_sort_lock = PTHREAD_MUTEX_INITIALIZER;

static void rank_graph(const Ctx* c, Graph* g) {
  int* ix = (int*)malloc(sizeof(int) * (g->n + 1));
  int m = 0;
  for (int i = 0; i < g->n; i++)
    if (g->alive[i]) ix[m++] = i;
  pthread_mutex_lock(&g_sort_lock);
  g_sort_ctx = c;
  g_sort_graph = g;
  qsort(ix, m, sizeof(int), cmp_name);
  for (int r = 0; r < m; r++) g->name_rank[ix[r]] = r;
  qsort(ix, m, sizeof(int), cmp_id);
  for (int r = 0; r < m; r++) g->id_rank[ix[r]] = r;
  pthread_mutex_unlock(&g_sort_lock);
  free(ix);
}

static Graph* graph_alloc(int n) {
  Graph* g = (Graph*)calloc(1, sizeof(Graph));
  g->n = n;
  g->alive = (uint8_t*)calloc(n, 1);
  g->pipe = (int*)calloc(n, sizeof(int));
  g->worker = (int*)calloc(n, sizeof(int));
  g->kind = (int*)calloc(n, sizeof(int));
  g->dur = (double*)calloc(n, sizeof(double));
  g->mem = (double*)calloc(n, sizeof(double));
  g->migc = (double*)calloc(n, sizeof(double));
  g->rem = (int64_t*)calloc(n, sizeof(int64_t));
  g->act = (int64_t*)calloc(n, sizeof(int64_t));
  g->ctx = (int64_t*)calloc(n, sizeof(int64_t));
  g->id = (char**)calloc(n, sizeof(char*));
  g->preds = (ivec*)calloc(n, sizeof(ivec));
  g->succs = (ivec*)calloc(n, sizeof(ivec));
  g->name_rank = (int*)calloc(n, sizeof(int));
  g->id_rank = (int*)calloc(n, sizeof(int));
  return g;
}

static void graph_free(Graph* g) {
  if (!g) return;
  for (int i = 0; i < g->n; i++) {
    free(g->preds[i].a);
    free(g->succs[i].a);
  }
  if (g->owned_ids >= 0 && g->n > 0 && g->owned_ids < g->n) free(g->id[g->owned_ids]);
  free(g->alive); free(g->pipe); free(g->worker); free(g->kind); free(g->dur); free(g->mem);
  free(g->migc); free(g->rem); free(g->act); free(g->ctx); free(g->id); free(g->preds);
  free(g->succs); free(g->name_rank); free(g->id_rank);
  free(g);
}

static double lut(const Ctx* c, int kind, int partner /* -1 none */, int alloc, St* s) {
  double v = c->in->lut[(kind * RLX_NPARTNER + (partner + 1)) * RLX_NALLOC + alloc];
  if (isnan(v) && s) {
    s->err = RLX_ERR_KEY;
    snprintf(s->msg, sizeof s->msg, "slowdown table has no rows for kind pair %d/%d", kind, partner);
  }
  return v;
}

/* ------------------------------------------------------------------ */
static St* st_new(const Ctx* c, Graph* g, int own) {
  St* s = (St*)calloc(1, sizeof(St));
  int n = g->n;
  s->c = c;
  s->g = g;
  s->own_graph = own;
  s->done = (uint8_t*)calloc(n, 1);
  s->run = (uint8_t*)calloc(n, 1);
  s->tw = (uint8_t*)calloc(n, 1);
  s->done_t = (double*)calloc(n, sizeof(double));
  s->pend = (int*)calloc(n, sizeof(int));
  s->rate = (double*)calloc(n, sizeof(double));
  s->pre = (double*)calloc(n, sizeof(double));
  s->work = (double*)calloc(n, sizeof(double));
  s->twend = (double*)calloc(n, sizeof(double));
  s->mprefix = (double*)calloc(n, sizeof(double));
  s->partner = (int*)malloc(sizeof(int) * n);
  for (int i = 0; i < n; i++) s->partner[i] = -1;
  s->nmem = (int*)calloc(c->W, sizeof(int));
  s->grant = (double*)malloc(sizeof(double) * c->W * c->P);
  for (int i = 0; i < c->W * c->P; i++) s->grant[i] = NAN;
  return s;
}

static void st_free(St* s) {
  if (!s) return;
  if (s->own_graph) graph_free(s->g);
  free(s->done); free(s->run); free(s->tw); free(s->done_t); free(s->pend); free(s->rate);
  free(s->pre); free(s->work); free(s->twend); free(s->mprefix); free(s->partner); free(s->nmem);
  free(s->grant);
  free(s);
}

/* clone onto the same graph (graphs are immutable except through merges) */
static St* st_clone(const St* o) {
  St* s = st_new(o->c, o->g, 0);
  int n = o->g->n;
  s->now = o->now;
  memcpy(s->done, o->done, n);
  memcpy(s->run, o->run, n);
  memcpy(s->tw, o->tw, n);
  memcpy(s->done_t, o->done_t, sizeof(double) * n);
  memcpy(s->pend, o->pend, sizeof(int) * n);
  memcpy(s->rate, o->rate, sizeof(double) * n);
  memcpy(s->pre, o->pre, sizeof(double) * n);
  memcpy(s->work, o->work, sizeof(double) * n);
  memcpy(s->twend, o->twend, sizeof(double) * n);
  memcpy(s->mprefix, o->mprefix, sizeof(double) * n);
  memcpy(s->partner, o->partner, sizeof(int) * n);
  memcpy(s->nmem, o->nmem, sizeof(int) * o->c->W);
  memcpy(s->grant, o->grant, sizeof(double) * o->c->W * o->c->P);
  return s;
}

static int is_ready(const St* s, int i) {
  return s->g->alive[i] && !s->done[i] && !s->run[i] && !s->tw[i] && s->pend[i] == 0;
}

static void complete(St* s, int i) {
  s->done[i] = 1;
  s->done_t[i] = s->now;
  const ivec* sc = &s->g->succs[i];
  for (int k = 0; k < sc->n; k++) s->pend[sc->a[k]]--;
}

/* _auto_start_toolwaits :421-434 (sorted(self.nodes) order) */
static void auto_start_tw(St* s) {
  Graph* g = s->g;
  int n = g->n;
  int* order = (int*)malloc(sizeof(int) * n);
  int m = 0;
  for (int i = 0; i < n; i++)
    if (g->alive[i]) order[g->id_rank[i]] = i, m++;
  int progressed = 1;
  while (progressed) {
    progressed = 0;
    for (int r = 0; r < m; r++) {
      int i = order[r];
      if (g->kind[i] != RLX_KIND_TOOL_WAIT || !is_ready(s, i)) continue;
      if (g->dur[i] <= EPS)
        complete(s, i);
      else {
        s->tw[i] = 1;
        s->twend[i] = s->now + g->dur[i];
      }
      progressed = 1;
    }
  }
  free(order);
}

/* _start_member :460-484 */
static void start_member(St* s, int i, double rate, int alloc, int partner) {
  const Ctx* c = s->c;
  Graph* g = s->g;
  double prefix = s->mprefix[i];
  s->mprefix[i] = 0.0;
  int k = g->kind[i];
  int rollout = (k <= RLX_KIND_DECODE_SMALL);
  if (rollout && c->in->realloc_penalty > 0) {
    double* slot = &s->grant[g->worker[i] * c->P + g->pipe[i]];
    double am = c->in->alloc_mem[alloc];
    if (!isnan(*slot) && fabs(*slot - am) > EPS) prefix += c->in->realloc_penalty;
    *slot = am;
  }
  s->run[i] = 1;
  s->rate[i] = rate;
  s->pre[i] = prefix;
  s->work[i] = g->dur[i];
  s->partner[i] = partner;
  s->nmem[g->worker[i]]++;
}

typedef struct Act {
  int cls, a, b, alloc, target, nm;
  int m[RLX_MAX_MEMBERS];
} Act;

static int apply_merge(St* s, const Act* a, int* merged_out);

static void apply(St* s, const Act* a, int* merged_out) {
  Graph* g = s->g;
  const Ctx* c = s->c;
  if (a->cls == RLX_CLASS_EXCLUSIVE) {
    start_member(s, a->a, lut(c, g->kind[a->a], -1, 0, s), 0, -1);
  } else if (a->cls == RLX_CLASS_MULTIPLEX) {
    int x = a->a, y = a->b;
    double ra = lut(c, g->kind[x], g->kind[y], a->alloc, s);
    double rb = lut(c, g->kind[y], g->kind[x], a->alloc + 12, s);
    start_member(s, x, ra, a->alloc, y);
    start_member(s, y, rb, a->alloc + 12, x);
  } else {
    apply_merge(s, a, merged_out);
  }
  auto_start_tw(s);
}

/* _apply_merge :517-581 — builds a new graph with the merged node appended */
static int apply_merge(St* s, const Act* a, int* merged_out) {
  const Ctx* c = s->c;
  Graph* o = s->g;
  int n = o->n;
  Graph* g = graph_alloc(n + 1);
  memcpy(g->alive, o->alive, n);
  memcpy(g->pipe, o->pipe, sizeof(int) * n);
  memcpy(g->worker, o->worker, sizeof(int) * n);
  memcpy(g->kind, o->kind, sizeof(int) * n);
  memcpy(g->dur, o->dur, sizeof(double) * n);
  memcpy(g->mem, o->mem, sizeof(double) * n);
  memcpy(g->migc, o->migc, sizeof(double) * n);
  memcpy(g->rem, o->rem, sizeof(int64_t) * n);
  memcpy(g->act, o->act, sizeof(int64_t) * n);
  memcpy(g->ctx, o->ctx, sizeof(int64_t) * n);
  memcpy(g->id, o->id, sizeof(char*) * n);
  for (int i = 0; i < n; i++) {
    iv_copy(&g->preds[i], &o->preds[i]);
    iv_copy(&g->succs[i], &o->succs[i]);
  }
  int M = n;
  g->owned_ids = M;
  int p = o->pipe[a->m[0]];
  /* merged_estimate :185-199 */
  int64_t tokens = 0, active = 0, ctx = 0;
  double dmax = 0.0, memmax = 0.0;
  for (int k = 0; k < a->nm; k++) {
    int x = a->m[k];
    tokens += o->rem[x];
    active += o->act[x];
    ctx += o->ctx[x];
    if (k == 0 || o->dur[x] > dmax) dmax = o->dur[x];
    if (k == 0 || o->mem[x] > memmax) memmax = o->mem[x];
  }
  int kind;
  double dur;
  if (active <= 0) {
    kind = o->kind[a->m[0]];
    dur = dmax;
  } else {
    int b = active >= 1024 ? 2 : (active >= 128 ? 1 : 0);
    kind = b == 0 ? RLX_KIND_DECODE_SMALL : (b == 1 ? RLX_KIND_DECODE_MEDIUM : RLX_KIND_DECODE_LARGE);
    if (!c->in->latency_ok[p * 3 + b]) {
      s->err = RLX_ERR_KEY;
      snprintf(s->msg, sizeof s->msg, "latency model has no bucket %d", b);
    }
    dur = ((double)tokens * c->in->latency[p * 3 + b]) / (double)active;
  }
  double prefix = 0.0;
  for (int k = 0; k < a->nm; k++) {
    int x = a->m[k];
    if (o->worker[x] == a->target) continue;
    prefix += c->in->has_spec[p] ? o->migc[x] : c->in->default_migration_cost;
  }
  /* id "merge[" + "+".join(ids) + "]@w<t>" */
  size_t len = 32;
  for (int k = 0; k < a->nm; k++) len += strlen(o->id[a->m[k]]) + 1;
  char* id = (char*)malloc(len);
  strcpy(id, "merge[");
  for (int k = 0; k < a->nm; k++) {
    if (k) strcat(id, "+");
    strcat(id, o->id[a->m[k]]);
  }
  char tail[24];
  snprintf(tail, sizeof tail, "]@w%d", c->in->worker_ids[a->target]);
  strcat(id, tail);
  g->alive[M] = 1;
  g->id[M] = id;
  g->pipe[M] = p;
  g->worker[M] = a->target;
  g->kind[M] = kind;
  g->dur[M] = dur;
  double dm = DEFAULT_MEM[kind];
  g->mem[M] = memmax > dm ? memmax : dm;
  g->rem[M] = tokens;
  g->act[M] = active;
  g->ctx[M] = ctx;
  g->migc[M] = 0.0;
  /* preds/succs: union minus members; rewire neighbours */
  int is_mem[RLX_MAX_MEMBERS];
  (void)is_mem;
  for (int k = 0; k < a->nm; k++) {
    int x = a->m[k];
    for (int q = 0; q < g->preds[x].n; q++) {
      int pr = g->preds[x].a[q];
      int member = 0;
      for (int z = 0; z < a->nm; z++) member |= (a->m[z] == pr);
      if (member) continue;
      if (!iv_has(&g->preds[M], pr)) iv_push(&g->preds[M], pr);
    }
    for (int q = 0; q < g->succs[x].n; q++) {
      int sc = g->succs[x].a[q];
      int member = 0;
      for (int z = 0; z < a->nm; z++) member |= (a->m[z] == sc);
      if (member) continue;
      if (!iv_has(&g->succs[M], sc)) iv_push(&g->succs[M], sc);
    }
  }
  for (int k = 0; k < a->nm; k++) {
    int x = a->m[k];
    for (int q = 0; q < g->preds[x].n; q++) iv_del(&g->succs[g->preds[x].a[q]], x);
    for (int q = 0; q < g->succs[x].n; q++) iv_del(&g->preds[g->succs[x].a[q]], x);
    g->alive[x] = 0;
    g->preds[x].n = 0;
    g->succs[x].n = 0;
  }
  for (int q = 0; q < g->preds[M].n; q++) iv_push(&g->succs[g->preds[M].a[q]], M);
  for (int q = 0; q < g->succs[M].n; q++) iv_push(&g->preds[g->succs[M].a[q]], M);
  rank_graph(c, g);

  /* re-home the state onto the new graph (one extra slot) */
  St tmp = *s;
  St* ns = st_new(c, g, 1);
  ns->now = tmp.now;
  memcpy(ns->done, tmp.done, n);
  memcpy(ns->run, tmp.run, n);
  memcpy(ns->tw, tmp.tw, n);
  memcpy(ns->done_t, tmp.done_t, sizeof(double) * n);
  memcpy(ns->rate, tmp.rate, sizeof(double) * n);
  memcpy(ns->pre, tmp.pre, sizeof(double) * n);
  memcpy(ns->work, tmp.work, sizeof(double) * n);
  memcpy(ns->twend, tmp.twend, sizeof(double) * n);
  memcpy(ns->mprefix, tmp.mprefix, sizeof(double) * n);
  memcpy(ns->partner, tmp.partner, sizeof(int) * n);
  memcpy(ns->nmem, tmp.nmem, sizeof(int) * c->W);
  memcpy(ns->grant, tmp.grant, sizeof(double) * c->W * c->P);
  ns->mprefix[M] = prefix;
  ns->err = tmp.err;
  memcpy(ns->msg, tmp.msg, sizeof ns->msg);
  for (int i = 0; i <= n; i++) {
    int cnt = 0;
    if (!g->alive[i]) continue;
    for (int q = 0; q < g->preds[i].n; q++) cnt += !ns->done[g->preds[i].a[q]];
    ns->pend[i] = cnt;
  }
  /* swap contents so the caller's pointer now owns the new graph */
  if (s->own_graph) graph_free(s->g);
  free(s->done); free(s->run); free(s->tw); free(s->done_t); free(s->pend); free(s->rate);
  free(s->pre); free(s->work); free(s->twend); free(s->mprefix); free(s->partner); free(s->nmem);
  free(s->grant);
  *s = *ns;
  free(ns);
  if (merged_out) *merged_out = M;
  return M;
}

static double finish_est(const St* s, int i) { return s->now + s->pre[i] + s->work[i] * s->rate[i]; }

static int has_events(const St* s) {
  for (int i = 0; i < s->g->n; i++)
    if (s->run[i] || s->tw[i]) return 1;
  return 0;
}

/* advance :593-627 (until=None) */
static void advance(St* s) {
  Graph* g = s->g;
  int n = g->n;
  int any = 0;
  double nxt = 0.0;
  for (int i = 0; i < n; i++) {
    double t;
    if (s->run[i])
      t = finish_est(s, i);
    else if (s->tw[i])
      t = s->twend[i];
    else
      continue;
    if (!any || t < nxt) nxt = t;
    any = 1;
  }
  if (!any) {
    s->err = RLX_ERR_SCHEDULING;
    snprintf(s->msg, sizeof s->msg, "no pending events to advance to");
    return;
  }
  double dt = nxt - s->now;
  if (!(dt > 0.0)) dt = 0.0;
  for (int i = 0; i < n; i++) {
    if (!s->run[i]) continue;
    double d = dt;
    if (s->pre[i] > EPS) {
      double used = d < s->pre[i] ? d : s->pre[i];
      s->pre[i] -= used;
      d -= used;
    }
    if (d > EPS && s->work[i] > EPS) {
      double r = s->work[i] - d / s->rate[i];
      s->work[i] = r > 0.0 ? r : 0.0;
    }
  }
  s->now = nxt;
  /* finished, in sorted(id) order */
  int* fin = (int*)malloc(sizeof(int) * (n + 1));
  int nf = 0;
  for (int i = 0; i < n; i++)
    if (s->run[i] && s->pre[i] <= EPS && s->work[i] * s->rate[i] <= EPS) fin[nf++] = i;
  for (int a = 1; a < nf; a++)
    for (int b = a; b > 0 && g->id_rank[fin[b]] < g->id_rank[fin[b - 1]]; b--) {
      int t = fin[b];
      fin[b] = fin[b - 1];
      fin[b - 1] = t;
    }
  for (int k = 0; k < nf; k++) {
    int i = fin[k];
    s->run[i] = 0;
    s->nmem[g->worker[i]]--;
    complete(s, i);
    int pt = s->partner[i];
    if (pt >= 0 && s->run[pt]) {
      if (s->rate[pt] != 1.0) s->rate[pt] = 1.0;
      s->partner[pt] = -1;
    }
  }
  int ne = 0;
  for (int i = 0; i < n; i++)
    if (s->tw[i] && s->twend[i] <= s->now + EPS) {
      s->tw[i] = 0;
      complete(s, i);
      ne++;
    }
  free(fin);
  if (nf || ne) auto_start_tw(s);
}

/* ------------------------------------------------------------------ */
/* _window_ids :710-748 */
static void window_ids(const St* s, int rounds, uint8_t* win) {
  const Graph* g = s->g;
  int n = g->n;
  uint8_t* cov = (uint8_t*)calloc(n, 1);
  uint8_t* nx = (uint8_t*)calloc(n, 1);
  memset(win, 0, n);
  for (int i = 0; i < n; i++) {
    if (!g->alive[i]) continue;
    if (s->run[i] || s->tw[i] || is_ready(s, i)) win[i] = 1;
    cov[i] = s->done[i] || win[i];
  }
  for (int depth = 1; depth < rounds; depth++) {
    int cnt = 0;
    memset(nx, 0, n);
    for (int i = 0; i < n; i++) {
      if (!g->alive[i] || cov[i]) continue;
      int ok = 1;
      for (int q = 0; q < g->preds[i].n && ok; q++) ok = cov[g->preds[i].a[q]];
      if (ok) nx[i] = 1, cnt++;
    }
    if (!cnt) break;
    for (int i = 0; i < n; i++)
      if (nx[i]) win[i] = cov[i] = 1;
    for (;;) {
      int nf = 0;
      uint8_t* fr = (uint8_t*)calloc(n, 1);
      for (int i = 0; i < n; i++) {
        if (!g->alive[i] || cov[i]) continue;
        int ok = 1, gate = 0;
        for (int q = 0; q < g->preds[i].n && ok; q++) {
          int p = g->preds[i].a[q];
          ok = cov[p];
          if (nx[p] && g->kind[p] == RLX_KIND_TOOL_WAIT) gate = 1;
        }
        if (ok && gate) fr[i] = 1, nf++;
      }
      for (int i = 0; i < n; i++)
        if (fr[i]) nx[i] = win[i] = cov[i] = 1;
      free(fr);
      if (!nf) break;
    }
  }
  free(cov);
  free(nx);
}

/* _suffix_lengths :751-770 (order-independent: longest exclusive chain) */
static double suffix_of(const Graph* g, int i, double* suf, uint8_t* vis) {
  if (vis[i]) return suf[i];
  double best = 0.0;
  int any = 0;
  for (int q = 0; q < g->succs[i].n; q++) {
    double v = suffix_of(g, g->succs[i].a[q], suf, vis);
    if (!any || v > best) best = v;
    any = 1;
  }
  suf[i] = g->dur[i] + (any ? best : 0.0);
  vis[i] = 1;
  return suf[i];
}

static void suffix_lengths(const St* s, double* suf) {
  const Graph* g = s->g;
  uint8_t* vis = (uint8_t*)calloc(g->n, 1);
  for (int i = 0; i < g->n; i++)
    if (g->alive[i]) suffix_of(g, i, suf, vis);
  free(vis);
}

/* ------------------------------------------------------------------ */
/* _rerated_pair_end :792-800 */
static double rerated_end(double da, double sa, double db, double sb) {
  double na = da * sa, nb = db * sb;
  if (fabs(na - nb) <= EPS) return na;
  if (na < nb) return na + (1.0 - na / nb) * db;
  return nb + (1.0 - nb / na) * da;
}

/* _best_pair_action :803-828 ; returns 0 if None */
static int best_pair(St* s, int a, int b, Act* out) {
  const Ctx* c = s->c;
  const Graph* g = s->g;
  double h = c->in->headroom;
  if (!(g->mem[a] + g->mem[b] <= 1.0 - h + 1e-12)) return 0;
  int found = 0;
  double best_end = INFINITY;
  for (int o = 0; o < 2; o++) {
    int f = o ? b : a, sc = o ? a : b;
    for (int ai = 0; ai < 3; ai++)
      for (int mj = 0; mj < 4; mj++) {
        if (MEM_GRIDV[mj] + g->mem[sc] > 1.0 - h + EPS) continue;
        int al = 1 + ai * 4 + mj;
        double end = rerated_end(g->dur[f], lut(c, g->kind[f], g->kind[sc], al, s), g->dur[sc],
                                 lut(c, g->kind[sc], g->kind[f], al + 12, s));
        if (end < best_end - EPS) {
          out->cls = RLX_CLASS_MULTIPLEX;
          out->a = f;
          out->b = sc;
          out->alloc = al;
          best_end = end;
          found = 1;
        }
      }
  }
  return found;
}

typedef struct KeyCtx {
  const St* s;
  const double* suf;
  int by_suffix;
} KeyCtx;
static __thread const KeyCtx* t_key;
static int cmp_key(const void* x, const void* y) {
  int a = *(const int*)x, b = *(const int*)y;
  const KeyCtx* k = t_key;
  if (k->by_suffix) {
    double na = -k->suf[a], nb = -k->suf[b];
    if (na < nb) return -1;
    if (na > nb) return 1;
  }
  return k->s->g->name_rank[a] - k->s->g->name_rank[b];
}

/* _complete_window :831-869 */
static double complete_window(St* est, const uint8_t* win, const double* suf, int by_suffix, int pair) {
  Graph* g = est->g;
  int n = g->n;
  int* ready = (int*)malloc(sizeof(int) * (n + 1));
  uint8_t* busy = (uint8_t*)malloc(est->c->W);
  KeyCtx kc = {est, suf, by_suffix};
  int guard = 0;
  for (;;) {
    int open = 0;
    for (int i = 0; i < n && !open; i++) open = win[i] && g->alive[i] && !est->done[i];
    if (!open) break;
    int started = 1;
    while (started) {
      started = 0;
      for (int w = 0; w < est->c->W; w++) busy[w] = est->nmem[w] > 0;
      int nr = 0;
      for (int i = 0; i < n; i++)
        if (win[i] && g->kind[i] != RLX_KIND_TOOL_WAIT && is_ready(est, i)) ready[nr++] = i;
      t_key = &kc;
      qsort(ready, nr, sizeof(int), cmp_key);
      for (int r = 0; r < nr; r++) {
        int x = ready[r];
        if (busy[g->worker[x]]) continue;
        Act act;
        int have = 0;
        if (pair) {
          for (int q = 0; q < nr; q++) {
            int o = ready[q];
            if (g->worker[o] == g->worker[x] && g->pipe[o] != g->pipe[x] && !est->done[o] && !est->run[o]) {
              have = best_pair(est, x, o, &act);
              break;
            }
          }
        }
        if (!have) {
          act.cls = RLX_CLASS_EXCLUSIVE;
          act.a = x;
        }
        apply(est, &act, NULL);
        busy[g->worker[x]] = 1;
        started = 1;
      }
    }
    if (!has_events(est)) break;
    advance(est);
    if (est->err) break;
    if (++guard > 10000) {
      est->err = RLX_ERR_SCHEDULING;
      snprintf(est->msg, sizeof est->msg, "window estimate did not converge");
      break;
    }
  }
  double best = 0.0;
  int any = 0;
  for (int i = 0; i < n; i++)
    if (win[i] && g->alive[i] && est->done[i]) {
      if (!any || est->done_t[i] > best) best = est->done_t[i];
      any = 1;
    }
  free(ready);
  free(busy);
  return any ? best : est->now;
}

typedef struct Res {
  int err;
  char msg[160];
} Res;

static void take_err(Res* r, const St* s) {
  if (s->err && !r->err) {
    r->err = s->err;
    memcpy(r->msg, s->msg, sizeof r->msg);
  }
}

/* window_cost :878-899 */
static double window_cost(const St* state, const Act* a, int rounds, Res* res) {
  St* base = st_clone(state);
  apply(base, a, NULL);
  int n = base->g->n;
  uint8_t* win = (uint8_t*)malloc(n);
  window_ids(base, rounds, win);
  int any = 0;
  for (int i = 0; i < n; i++) any |= win[i];
  double cost;
  if (!any) {
    cost = base->now;
  } else {
    double* suf = (double*)calloc(n, sizeof(double));
    suffix_lengths(base, suf);
    cost = INFINITY;
    static const int variants[3][2] = {{1, 0}, {1, 1}, {0, 0}};
    for (int v = 0; v < 3; v++) {
      St* est = st_clone(base);
      double c = complete_window(est, win, suf, variants[v][0], variants[v][1]);
      take_err(res, est);
      st_free(est);
      if (c < cost) cost = c;
    }
    free(suf);
  }
  take_err(res, base);
  free(win);
  st_free(base);
  return cost;
}

/* ------------------------------------------------------------------ */
/* enumerate_actions :648-703 with optional cap; non-merge-only variant for follow-ups */
typedef struct Cands {
  int64_t n, cap;
  Act* a;
  int* prio;
} Cands;

static void push_cand(Cands* c, const Act* a, int prio) {
  if (c->n == c->cap) {
    c->cap = c->cap ? c->cap * 2 : 64;
    c->a = (Act*)realloc(c->a, sizeof(Act) * c->cap);
    c->prio = (int*)realloc(c->prio, sizeof(int) * c->cap);
  }
  c->a[c->n] = *a;
  c->prio[c->n] = prio;
  c->n++;
}

static const Graph* t_idg;
static int cmp_member_id(const void* x, const void* y) {
  return strcmp(t_idg->id[*(const int*)x], t_idg->id[*(const int*)y]);
}

static int enumerate(const St* s, int max_merge, int with_merges, Cands* out, int64_t limit) {
  const Ctx* c = s->c;
  const Graph* g = s->g;
  int n = g->n;
  double h = c->in->headroom;
  int* ready = (int*)malloc(sizeof(int) * (n + 1));
  int nr = 0;
  for (int i = 0; i < n; i++)
    if (g->kind[i] != RLX_KIND_TOOL_WAIT && is_ready(s, i)) ready[nr++] = i;
  KeyCtx kc = {s, NULL, 0};
  t_key = &kc;
  qsort(ready, nr, sizeof(int), cmp_key);
  int* grp = (int*)malloc(sizeof(int) * (nr + 1));
  for (int w = 0; w < c->W; w++) {
    if (s->nmem[w]) continue;
    int ng = 0;
    for (int r = 0; r < nr; r++)
      if (g->worker[ready[r]] == w) grp[ng++] = ready[r];
    for (int i = 0; i < ng; i++)
      for (int j = i + 1; j < ng; j++) {
        int a = grp[i], b = grp[j];
        if (g->pipe[a] == g->pipe[b]) continue;
        if (!(g->mem[a] + g->mem[b] <= 1.0 - h + 1e-12)) continue;
        for (int o = 0; o < 2; o++) {
          int f = o ? b : a, sc = o ? a : b;
          for (int ai = 0; ai < 3; ai++)
            for (int mj = 0; mj < 4; mj++) {
              if (MEM_GRIDV[mj] + g->mem[sc] > 1.0 - h + EPS) continue;
              Act act = {RLX_CLASS_MULTIPLEX, f, sc, 1 + ai * 4 + mj, 0, 0, {0}};
              push_cand(out, &act, 0);
            }
        }
      }
  }
  int status = RLX_OK;
  if (with_merges && c->in->merge_enabled) {
    int* frag = (int*)malloc(sizeof(int) * (nr + 1));
    for (int pr = 0; pr < c->P; pr++) {
      int p = -1;
      for (int q = 0; q < c->P; q++)
        if (c->pipe_rank[q] == pr) p = q;
      int nf = 0;
      for (int r = 0; r < nr; r++) {
        int x = ready[r];
        if (g->pipe[x] == p && (g->kind[x] == RLX_KIND_DECODE_SMALL || g->kind[x] == RLX_KIND_DECODE_MEDIUM))
          frag[nf++] = x;
      }
      if (nf < 2) continue;
      int top = (max_merge > 0 && max_merge < nf) ? max_merge : nf;
      if (top > RLX_MAX_MEMBERS) top = RLX_MAX_MEMBERS;
      for (int size = 2; size <= top; size++) {
        int idx[RLX_MAX_MEMBERS];
        for (int k = 0; k < size; k++) idx[k] = k;
        for (;;) {
          int ok = 1;
          for (int k = 0; k < size && ok; k++)
            for (int z = k + 1; z < size && ok; z++) ok = g->worker[frag[idx[k]]] != g->worker[frag[idx[z]]];
          if (ok) {
            Act act;
            memset(&act, 0, sizeof act);
            act.cls = RLX_CLASS_MERGE;
            act.nm = size;
            for (int k = 0; k < size; k++) act.m[k] = frag[idx[k]];
            t_idg = g;
            qsort(act.m, size, sizeof(int), cmp_member_id);
            int ws[RLX_MAX_MEMBERS];
            for (int k = 0; k < size; k++) ws[k] = g->worker[act.m[k]];
            for (int a = 1; a < size; a++)
              for (int b = a; b > 0 && ws[b] < ws[b - 1]; b--) {
                int t = ws[b];
                ws[b] = ws[b - 1];
                ws[b - 1] = t;
              }
            for (int k = 0; k < size; k++) {
              act.target = ws[k];
              push_cand(out, &act, 1);
              if (limit > 0 && out->n > limit) {
                status = RLX_ERR_LIMIT;
                goto done_merges;
              }
            }
          }
          int k = size - 1;
          while (k >= 0 && idx[k] == nf - size + k) k--;
          if (k < 0) break;
          idx[k]++;
          for (int z = k + 1; z < size; z++) idx[z] = idx[z - 1] + 1;
        }
      }
    }
  done_merges:
    free(frag);
  }
  for (int r = 0; r < nr; r++)
    if (!s->nmem[g->worker[ready[r]]]) {
      Act act = {RLX_CLASS_EXCLUSIVE, ready[r], 0, 0, 0, 0, {0}};
      push_cand(out, &act, 2);
    }
  free(grp);
  free(ready);
  return status;
}

/* candidate_cost :902-918 */
static double candidate_cost(const St* state, const Act* a, int rounds, Res* res) {
  if (a->cls != RLX_CLASS_MERGE) return window_cost(state, a, rounds, res);
  St* post = st_clone(state);
  int M = -1;
  apply(post, a, &M);
  take_err(res, post);
  Cands fu = {0, 0, NULL, NULL};
  enumerate(post, 0, 0, &fu, 0);
  double best = INFINITY;
  int any = 0;
  for (int64_t k = 0; k < fu.n; k++) {
    const Act* f = &fu.a[k];
    int touches = (f->cls == RLX_CLASS_EXCLUSIVE) ? (f->a == M) : (f->a == M || f->b == M);
    if (!touches) continue;
    double v = window_cost(post, f, rounds, res);
    if (!any || v < best) best = v;
    any = 1;
  }
  free(fu.a);
  free(fu.prio);
  st_free(post);
  if (!any) return window_cost(state, a, rounds, res);
  return best;
}

/* action_finish_estimate :773-789 */
static double finish_estimate(const St* state, const Act* a, Res* res) {
  St* est = st_clone(state);
  int M = -1;
  apply(est, a, &M);
  take_err(res, est);
  double t;
  if (a->cls == RLX_CLASS_MERGE) {
    t = est->run[M] ? finish_est(est, M) : est->now + est->mprefix[M] + est->g->dur[M];
  } else if (a->cls == RLX_CLASS_EXCLUSIVE) {
    t = finish_est(est, a->a);
  } else {
    double x = finish_est(est, a->a), y = finish_est(est, a->b);
    t = y > x ? y : x;
  }
  st_free(est);
  return t;
}

/* ------------------------------------------------------------------ */
typedef struct Root {
  Ctx c;
  St* st;
  Graph* g;
  Cands cands;
} Root;

static int build_root(Root* R, const RlxInstanceDesc* in, const RlxStateDesc* sd, int max_merge, char* err,
                      int errlen) {
  memset(R, 0, sizeof *R);
  Ctx* c = &R->c;
  c->in = in;
  c->W = in->n_workers;
  c->P = in->n_pipes;
  c->pipe_name = (const char**)malloc(sizeof(char*) * c->P);
  c->pipe_rank = (int*)malloc(sizeof(int) * c->P);
  for (int p = 0; p < c->P; p++) c->pipe_name[p] = in->pipe_names + in->pipe_name_off[p];
  for (int p = 0; p < c->P; p++) {
    int r = 0;
    for (int q = 0; q < c->P; q++) r += strcmp(c->pipe_name[q], c->pipe_name[p]) < 0;
    c->pipe_rank[p] = r;
  }
  int n = sd->n_nodes;
  Graph* g = graph_alloc(n);
  g->owned_ids = -1;
  for (int i = 0; i < n; i++) {
    g->alive[i] = 1;
    g->pipe[i] = sd->pipe[i];
    g->worker[i] = sd->worker[i];
    g->kind[i] = sd->kind[i];
    g->dur[i] = sd->duration[i];
    g->mem[i] = sd->mem[i];
    g->rem[i] = sd->remaining[i];
    g->act[i] = sd->active[i];
    g->ctx[i] = sd->context[i];
    g->id[i] = (char*)(sd->ids + sd->id_off[i]);
    int p = sd->pipe[i];
    g->migc[i] = in->has_spec[p]
                     ? (2.0 * in->model_params[p] * (double)sd->context[i]) / (in->prefill_mfu[p] * in->peak_flops[p])
                     : 0.0;
  }
  for (int e = 0; e < sd->n_edges; e++) {
    iv_push(&g->succs[sd->edge_src[e]], sd->edge_dst[e]);
    iv_push(&g->preds[sd->edge_dst[e]], sd->edge_src[e]);
  }
  rank_graph(c, g);
  St* s = st_new(c, g, 0);
  s->now = sd->now;
  for (int i = 0; i < n; i++) {
    s->done[i] = sd->completed[i];
    s->mprefix[i] = sd->merge_prefix[i];
  }
  for (int i = 0; i < n; i++) {
    int cnt = 0;
    for (int q = 0; q < g->preds[i].n; q++) cnt += !s->done[g->preds[i].a[q]];
    s->pend[i] = cnt;
  }
  for (int k = 0; k < sd->n_running; k++) {
    int i = sd->run_node[k];
    s->run[i] = 1;
    s->rate[i] = sd->run_rate[k];
    s->pre[i] = sd->run_prefix[k];
    s->work[i] = sd->run_work[k];
    s->partner[i] = sd->run_partner[k];
    s->nmem[g->worker[i]]++;
  }
  for (int k = 0; k < sd->n_toolwaits; k++) {
    s->tw[sd->tw_node[k]] = 1;
    s->twend[sd->tw_node[k]] = sd->tw_end[k];
  }
  for (int k = 0; k < sd->n_grants; k++) s->grant[sd->grant_worker[k] * c->P + sd->grant_pipe[k]] = sd->grant_mem[k];
  R->st = s;
  R->g = g;
  int rc = enumerate(s, max_merge, 1, &R->cands, (int64_t)1 << 28);
  if (rc != RLX_OK) snprintf(err, errlen, "candidate space too large (set max_merge)");
  return rc;
}

static void free_root(Root* R) {
  st_free(R->st);
  graph_free(R->g);
  free(R->cands.a);
  free(R->cands.prio);
  free((void*)R->c.pipe_name);
  free(R->c.pipe_rank);
}

typedef struct Job {
  Root* R;
  int window;
  const int64_t* serials;
  int64_t n;
  int tid, nth;
  double* costs;
  double* fins;
  Res res;
} Job;

static void* worker_main(void* arg) {
  Job* j = (Job*)arg;
  for (int64_t k = j->tid; k < j->n; k += j->nth) {
    int64_t sidx = j->serials ? j->serials[k] : k;
    const Act* a = &j->R->cands.a[sidx];
    j->costs[k] = candidate_cost(j->R->st, a, j->window, &j->res);
    j->fins[k] = finish_estimate(j->R->st, a, &j->res);
    if (j->res.err) break;
  }
  return NULL;
}

int oracle_decide(const RlxInstanceDesc* in, const RlxStateDesc* sd, int window, int max_merge,
                  const int64_t* serials, int64_t n_serials, int nthreads, double* keys_out,
                  int64_t* n_candidates, int64_t* best_serial, double* best_cost, double* best_finish,
                  int* best_prio, char* err, int errlen) {
  Root R;
  err[0] = 0;
  int rc = build_root(&R, in, sd, max_merge, err, errlen);
  if (rc) {
    free_root(&R);
    return rc;
  }
  *n_candidates = R.cands.n;
  int64_t n = serials ? n_serials : R.cands.n;
  for (int64_t k = 0; serials && k < n; k++)
    if (serials[k] < 0 || serials[k] >= R.cands.n) {
      snprintf(err, errlen, "serial out of range");
      free_root(&R);
      return RLX_ERR_ARG;
    }
  double* costs = (double*)malloc(sizeof(double) * (n + 1));
  double* fins = (double*)malloc(sizeof(double) * (n + 1));
  if (nthreads < 1) nthreads = 1;
  Job* jobs = (Job*)calloc(nthreads, sizeof(Job));
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
  for (int t = 0; t < nthreads; t++) {
    jobs[t] = (Job){&R, window, serials, n, t, nthreads, costs, fins, {0, {0}}};
    pthread_create(&th[t], NULL, worker_main, &jobs[t]);
  }
  for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
  rc = RLX_OK;
  for (int t = 0; t < nthreads; t++)
    if (jobs[t].res.err && !rc) {
      rc = jobs[t].res.err;
      snprintf(err, errlen, "%s", jobs[t].res.msg);
    }
  *best_serial = -1;
  for (int64_t k = 0; k < n && !rc; k++) {
    int64_t sidx = serials ? serials[k] : k;
    int pr = R.cands.prio[sidx];
    if (keys_out) {
      keys_out[2 * k] = costs[k];
      keys_out[2 * k + 1] = fins[k];
    }
    int better = *best_serial < 0;
    if (!better) {
      if (costs[k] != *best_cost)
        better = costs[k] < *best_cost;
      else if (fins[k] != *best_finish)
        better = fins[k] < *best_finish;
      else if (pr != *best_prio)
        better = pr < *best_prio;
      else
        better = sidx < *best_serial;
    }
    if (better) {
      *best_serial = sidx;
      *best_cost = costs[k];
      *best_finish = fins[k];
      *best_prio = pr;
    }
  }
  free(costs);
  free(fins);
  free(jobs);
  free(th);
  free_root(&R);
  return rc;
}

/* Candidate serial -> action fields (for decoding the oracle's winner). */
int oracle_candidate(const RlxInstanceDesc* in, const RlxStateDesc* sd, int max_merge, int64_t serial, int32_t* out,
                     char* err, int errlen) {
  Root R;
  err[0] = 0;
  int rc = build_root(&R, in, sd, max_merge, err, errlen);
  if (!rc && (serial < 0 || serial >= R.cands.n)) rc = RLX_ERR_ARG;
  if (!rc) {
    const Act* a = &R.cands.a[serial];
    out[0] = a->cls;
    out[1] = a->a;
    out[2] = a->b;
    out[3] = a->alloc;
    out[4] = a->target;
    out[5] = a->nm;
    for (int k = 0; k < a->nm; k++) out[6 + k] = a->m[k];
  }
  free_root(&R);
  return rc;
}

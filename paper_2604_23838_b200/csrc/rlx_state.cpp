// rlx_state.cpp — the decision loop's execution state, held natively.
//
// The reference keeps this state in the Python `ExecState` object
// (rlmux/scheduler.py:339-634): dict-of-sets graph, running members,
// tool waits, merge prefixes, realloc grants. Here the same semantics live
// on structure-of-arrays inside the library, so that
//   * the decision loop (`_drive`, :925-950) can run entirely behind the
//     C-ABI (rlx_drive: plan -> kernel -> apply winner -> advance), and
//   * every decision's planner input (RlxStateDesc) is a view of these
//     arrays instead of a per-decision Python re-encode.
// The GPU scores candidates; this file only applies the ONE winner per
// decision and advances simulated time, exactly like the reference's
// driver does between chooser calls.
//
// Semantics followed:
//   readiness            :396-402   (not done / running / waiting, all preds done)
//   tool-wait auto-start :421-434   (tool-wait nodes in id order, until no change)
//   start of a member    :460-484   (merge prefix popped, realloc penalty, grants)
//   apply + validation   :486-515   (error texts are the reference's)
//   merge surgery        :517-581   (merged_estimate :185-199, migration_cost :174-182)
//   advance              :593-627   (consume, finished in id order, partner re-rate)
// Floating point: compiled with -ffp-contract=off; every expression keeps the
// reference's left-to-right binary64 order.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <charconv>
#include <map>
#include <string>
#include <vector>

#include "../../include/rlx.h"
#include "rlx_state.hpp"

namespace rlx {

static constexpr double kEpsS = 1e-9;  // scheduler.py:43
static const double kDefMem[RLX_NKIND] = {0.5, 0.55, 0.4, 0.3, 0.5, 0.6, 0.05};  // graph.py:98-106

// Python's repr() of a float (shortest round trip, ".0" for integral values)
// for the reference's error texts (scheduler.py:509-511).
std::string py_float(double x) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, x);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  // Python writes exponents with at least two digits: 1e-05, 1e+16
  size_t e = s.find('e');
  if (e != std::string::npos) {
    std::string mant = s.substr(0, e), ex = s.substr(e + 1);
    char sign = '+';
    if (!ex.empty() && (ex[0] == '-' || ex[0] == '+')) sign = ex[0], ex = ex.substr(1);
    if (ex.size() < 2) ex = "0" + ex;
    s = mant + "e" + sign + ex;
  }
  return s;
}

static void set_add(std::vector<int>& v, int x) {
  if (std::find(v.begin(), v.end(), x) == v.end()) v.push_back(x);
}
static void set_del(std::vector<int>& v, int x) {
  auto it = std::find(v.begin(), v.end(), x);
  if (it != v.end()) v.erase(it);
}

int ExecSoA::init(const RlxInstanceDesc* in, const RlxGraphDesc* g, bool rec) {
  P = in->n_pipes;
  W = in->n_workers;
  if (P <= 0 || W <= 0) return fail(RLX_ERR_ARG, "empty instance");
  headroom = in->headroom;
  realloc_penalty = in->realloc_penalty;
  default_migration_cost = in->default_migration_cost;
  worker_ids.assign(in->worker_ids, in->worker_ids + W);
  latency.assign(in->latency, in->latency + 3 * P);
  latency_ok.assign(in->latency_ok, in->latency_ok + 3 * P);
  has_spec.assign(in->has_spec, in->has_spec + P);
  params.assign(in->model_params, in->model_params + P);
  peak.assign(in->peak_flops, in->peak_flops + P);
  mfu.assign(in->prefill_mfu, in->prefill_mfu + P);
  record = rec;
  const int N = g->n_nodes;
  if (N < 0) return fail(RLX_ERR_ARG, "negative node count");
  nodes.resize(N);
  for (int i = 0; i < N; i++) {
    Node& n = nodes[i];
    n.pipe = g->pipe[i];
    n.worker = g->worker[i];
    n.kind = g->kind[i];
    if (n.pipe < 0 || n.pipe >= P || n.worker < 0 || n.worker >= W || n.kind < 0 || n.kind >= RLX_NKIND)
      return fail(RLX_ERR_ARG, "node field out of range");
    n.dur = g->duration[i];
    n.mem = g->mem[i];
    n.rem = g->remaining[i];
    n.act = g->active[i];
    n.ctx = g->context[i];
    n.tok = g->token_total[i];
    n.span_lo = g->span_lo[i];
    n.span_hi = g->span_hi[i];
    n.id = g->ids + g->id_off[i];
  }
  alive.assign(N, 1);
  done.assign(N, 0);
  running.assign(N, -1);
  ctime.assign(N, 0.0);
  twend.assign(N, NAN);
  mprefix.assign(N, NAN);
  preds.assign(N, {});
  succs.assign(N, {});
  for (int e = 0; e < g->n_edges; e++) {
    const int s = g->edge_src[e], d = g->edge_dst[e];
    if (s < 0 || s >= N || d < 0 || d >= N) return fail(RLX_ERR_ARG, "edge index out of range");
    set_add(succs[s], d);
    set_add(preds[d], s);
  }
  order.resize(N);
  for (int i = 0; i < N; i++) order[i] = i;
  wmem.assign(W, {});
  for (int i = 0; i < N; i++)
    if (nodes[i].kind == RLX_KIND_TOOL_WAIT) tw_sorted.push_back(i);
  std::sort(tw_sorted.begin(), tw_sorted.end(), [&](int a, int b) { return nodes[a].id < nodes[b].id; });
  now = makespan = 0.0;
  n_done = 0;
  revision = 0;
  auto_start_toolwaits();
  return RLX_OK;
}

int ExecSoA::fail(int code, const std::string& msg) {
  err = msg;
  return code;
}

void ExecSoA::log(int worker, int kind, int node, double sm, double mem) {
  if (!record) return;
  RlxEvent e;
  e.time = now;
  e.worker = worker;
  e.kind = kind;
  e.node = node;
  e._pad = 0;
  e.sm = sm;
  e.mem = mem;
  events.push_back(e);
}

bool ExecSoA::is_ready(int n) const {
  if (!alive[n] || done[n] || running[n] >= 0 || !isnan(twend[n])) return false;
  for (int p : preds[n])
    if (!done[p]) return false;
  return true;
}

void ExecSoA::complete(int n) {
  done[n] = 1;
  n_done++;
  ctime[n] = now;
  if (now > makespan) makespan = now;
  log(nodes[n].worker, RLX_EV_FINISH, n, NAN, NAN);
}

void ExecSoA::auto_start_toolwaits() {
  for (bool progressed = true; progressed;) {
    progressed = false;
    for (int n : tw_sorted) {
      if (!is_ready(n)) continue;
      log(nodes[n].worker, RLX_EV_TOOLWAIT_START, n, NAN, NAN);
      if (nodes[n].dur <= kEpsS) {
        complete(n);
      } else {
        twend[n] = now + nodes[n].dur;
        tw_order.push_back(n);
      }
      progressed = true;
    }
  }
}

int ExecSoA::require_ready(int n) {
  if (n < 0 || n >= (int)nodes.size() || !alive[n]) return fail(RLX_ERR_SCHEDULING, "unknown sub-stage");
  if (!is_ready(n)) {
    std::vector<const std::string*> missing;
    for (int p : preds[n])
      if (!done[p]) missing.push_back(&nodes[p].id);
    if (!missing.empty()) {
      const std::string* m0 = *std::min_element(missing.begin(), missing.end(),
                                                [](const std::string* a, const std::string* b) { return *a < *b; });
      return fail(RLX_ERR_SCHEDULING,
                  "dependency violation: " + nodes[n].id + " needs edge (" + *m0 + ", " + nodes[n].id + ") resolved");
    }
    return fail(RLX_ERR_SCHEDULING, "sub-stage " + nodes[n].id + " is not ready (running or done)");
  }
  if (nodes[n].kind == RLX_KIND_TOOL_WAIT) return fail(RLX_ERR_SCHEDULING, "tool wait " + nodes[n].id + " is not schedulable");
  return RLX_OK;
}

void ExecSoA::start_member(int n, double rate, double sm, double memsh, int partner) {
  Node& nd = nodes[n];
  double prefix = 0.0;
  if (!isnan(mprefix[n])) {
    prefix = mprefix[n];
    mprefix[n] = NAN;
  }
  if (nd.kind <= RLX_KIND_DECODE_SMALL && realloc_penalty > 0) {  // SubStage.is_rollout
    const long key = (long)nd.worker * P + nd.pipe;
    auto it = grants.find(key);
    if (it != grants.end() && fabs(it->second - memsh) > kEpsS) prefix += realloc_penalty;
    if (it == grants.end()) grant_order.push_back(key);
    grants[key] = memsh;
  }
  Member m;
  m.node = n;
  m.rate = rate;
  m.sm = sm;
  m.memsh = memsh;
  m.prefix = prefix;
  m.work = nd.dur;
  m.partner = partner;
  m.started = now;
  running[n] = (int)members.size();
  members.push_back(m);
  run_order.push_back(n);
  wmem[nd.worker].push_back(n);
  if (prefix > kEpsS) log(nd.worker, RLX_EV_MIGRATION, n, NAN, NAN);
  log(nd.worker, RLX_EV_START, n, sm, memsh);
}

int ExecSoA::apply(const RlxApply* a) {
  if (a->cls == RLX_CLASS_EXCLUSIVE) {
    const int n = a->node_a;
    int rc = require_ready(n);
    if (rc) return rc;
    const int w = nodes[n].worker;
    if (!wmem[w].empty()) return fail(RLX_ERR_SCHEDULING, "worker " + std::to_string(worker_ids[w]) + " is busy");
    if (isnan(a->rate_a)) return fail(RLX_ERR_KEY, "slowdown table has no entry for this allocation");
    start_member(n, a->rate_a, a->sm_a, a->mem_a, -1);
  } else if (a->cls == RLX_CLASS_MULTIPLEX) {
    const int x = a->node_a, y = a->node_b;
    int rc = require_ready(x);
    if (rc) return rc;
    rc = require_ready(y);
    if (rc) return rc;
    const Node &A = nodes[x], &B = nodes[y];
    if (A.worker != B.worker) return fail(RLX_ERR_SCHEDULING, "multiplex members must share a worker");
    if (A.pipe == B.pipe) return fail(RLX_ERR_SCHEDULING, "multiplex members must belong to different pipelines");
    if (!wmem[A.worker].empty())
      return fail(RLX_ERR_SCHEDULING, "worker " + std::to_string(worker_ids[A.worker]) + " is busy");
    if (!(A.mem + B.mem <= 1.0 - headroom + 1e-12))  // feasible, slowdown.py:162-166
      return fail(RLX_ERR_SCHEDULING, "memory infeasible: " + A.id + "(" + py_float(A.mem) + ") + " + B.id + "(" +
                                          py_float(B.mem) + ")");
    if (isnan(a->rate_a) || isnan(a->rate_b)) return fail(RLX_ERR_KEY, "slowdown table has no entry for this pair");
    start_member(x, a->rate_a, a->sm_a, a->mem_a, y);
    start_member(y, a->rate_b, a->sm_b, a->mem_b, x);
  } else if (a->cls == RLX_CLASS_MERGE) {
    int rc = merge(a);
    if (rc) return rc;
  } else {
    return fail(RLX_ERR_ARG, "unknown action class");
  }
  auto_start_toolwaits();
  return RLX_OK;
}

int ExecSoA::merge(const RlxApply* a) {
  const int k = a->n_members;
  if (k < 2) return fail(RLX_ERR_SCHEDULING, "merge needs at least two fragments");
  if (k > RLX_MAX_MEMBERS) return fail(RLX_ERR_LIMIT, "merge sets above 64 members");
  for (int i = 0; i < k; i++) {
    int rc = require_ready(a->members[i]);
    if (rc) return rc;
  }
  const int* m = a->members;
  const int p = nodes[m[0]].pipe;
  for (int i = 0; i < k; i++)
    if (nodes[m[i]].pipe != p) return fail(RLX_ERR_SCHEDULING, "merge fragments must belong to one pipeline");
  for (int i = 0; i < k; i++)
    if (nodes[m[i]].kind != RLX_KIND_DECODE_SMALL && nodes[m[i]].kind != RLX_KIND_DECODE_MEDIUM)
      return fail(RLX_ERR_SCHEDULING, "only small/medium decode fragments can merge");
  for (int i = 0; i < k; i++)
    for (int j = i + 1; j < k; j++)
      if (nodes[m[i]].worker == nodes[m[j]].worker)
        return fail(RLX_ERR_SCHEDULING, "merge fragments must sit on distinct workers");
  const int t = a->target_worker;
  bool on = false;
  for (int i = 0; i < k; i++) on = on || nodes[m[i]].worker == t;
  if (!on) return fail(RLX_ERR_SCHEDULING, "merge target must hold one of the fragments");
  // merged_estimate (:185-199)
  long long tokens = 0, active = 0;
  for (int i = 0; i < k; i++) tokens += nodes[m[i]].rem, active += nodes[m[i]].act;
  int kind;
  double dur;
  if (active <= 0) {
    kind = nodes[m[0]].kind;
    dur = nodes[m[0]].dur;
    for (int i = 1; i < k; i++) dur = nodes[m[i]].dur > dur ? nodes[m[i]].dur : dur;
  } else {
    const int bk = active >= 1024 ? 2 : (active >= 128 ? 1 : 0);
    kind = bk == 0 ? RLX_KIND_DECODE_SMALL : (bk == 1 ? RLX_KIND_DECODE_MEDIUM : RLX_KIND_DECODE_LARGE);
    if (!latency_ok[p * 3 + bk]) return fail(RLX_ERR_KEY, std::to_string(bk));
    dur = ((double)tokens * latency[p * 3 + bk]) / (double)active;
  }
  // migration prefix, summed in member order (:539-542)
  double prefix = 0.0;
  for (int i = 0; i < k; i++) {
    const Node& x = nodes[m[i]];
    if (x.worker == t) continue;
    if (has_spec[p])
      prefix += (2.0 * params[p] * (double)x.ctx) / (mfu[p] * peak[p]);
    else
      prefix += default_migration_cost;
  }
  Node nn;
  nn.id = "merge[";
  for (int i = 0; i < k; i++) {
    if (i) nn.id += "+";
    nn.id += nodes[m[i]].id;
  }
  nn.id += "]@w" + std::to_string(worker_ids[t]);
  nn.pipe = p;
  nn.worker = t;
  nn.kind = kind;
  nn.dur = dur;
  double mm = nodes[m[0]].mem;
  for (int i = 1; i < k; i++) mm = nodes[m[i]].mem > mm ? nodes[m[i]].mem : mm;
  nn.mem = kDefMem[kind] > mm ? kDefMem[kind] : mm;  // max(DEFAULT_MEM_FRACTIONS[kind], max member mem)
  nn.span_lo = nodes[m[0]].span_lo;
  nn.span_hi = nodes[m[0]].span_hi;
  nn.rem = nn.act = nn.ctx = nn.tok = 0;
  for (int i = 0; i < k; i++) {
    const Node& x = nodes[m[i]];
    nn.span_lo = std::min(nn.span_lo, x.span_lo);
    nn.span_hi = std::max(nn.span_hi, x.span_hi);
    nn.rem += x.rem;
    nn.act += x.act;
    nn.ctx += x.ctx;
    nn.tok += x.tok;
  }
  const int M = (int)nodes.size();
  std::vector<int> np, ns;
  auto member = [&](int x) {
    for (int i = 0; i < k; i++)
      if (m[i] == x) return true;
    return false;
  };
  for (int i = 0; i < k; i++) {
    for (int x : preds[m[i]])
      if (!member(x)) set_add(np, x);
    for (int x : succs[m[i]])
      if (!member(x)) set_add(ns, x);
  }
  for (int i = 0; i < k; i++) {
    for (int x : preds[m[i]]) set_del(succs[x], m[i]);
    for (int x : succs[m[i]]) set_del(preds[x], m[i]);
    preds[m[i]].clear();
    succs[m[i]].clear();
    alive[m[i]] = 0;
    set_del(order, m[i]);
  }
  nodes.push_back(nn);
  alive.push_back(1);
  done.push_back(0);
  running.push_back(-1);
  ctime.push_back(0.0);
  twend.push_back(NAN);
  mprefix.push_back(prefix);
  preds.push_back(np);
  succs.push_back(ns);
  for (int x : np) set_add(succs[x], M);
  for (int x : ns) set_add(preds[x], M);
  order.push_back(M);
  revision++;
  log(t, RLX_EV_MERGE, M, NAN, NAN);
  return RLX_OK;
}

bool ExecSoA::next_event(double& t) const {
  bool any = false;
  for (int n : run_order) {
    const Member& m = members[running[n]];
    const double fe = (now + m.prefix) + m.work * m.rate;  // finish_estimate :328
    if (!any || fe < t) t = fe;
    any = true;
  }
  for (int n : tw_order) {
    if (!any || twend[n] < t) t = twend[n];
    any = true;
  }
  return any;
}

int ExecSoA::advance(bool has_until, double until) {
  double nxt = 0.0;
  if (!next_event(nxt)) {
    if (!has_until) return fail(RLX_ERR_SCHEDULING, "no pending events to advance to");
    now = now > until ? now : until;
    return RLX_OK;
  }
  const double target = has_until ? (until < nxt ? until : nxt) : nxt;
  const double x = target - now;
  const double dt0 = x > 0.0 ? x : 0.0;
  for (int n : run_order) {  // _Member.consume (:330-336)
    Member& m = members[running[n]];
    double dt = dt0;
    if (m.prefix > kEpsS) {
      const double used = m.prefix < dt ? m.prefix : dt;
      m.prefix -= used;
      dt -= used;
    }
    if (dt > kEpsS && m.work > kEpsS) {
      const double r = m.work - dt / m.rate;
      m.work = 0.0 > r ? 0.0 : r;
    }
  }
  now = target;
  std::vector<int> fin;
  for (int n : run_order) {
    const Member& m = members[running[n]];
    if (m.prefix <= kEpsS && m.work * m.rate <= kEpsS) fin.push_back(n);
  }
  std::sort(fin.begin(), fin.end(), [&](int a, int b) { return nodes[a].id < nodes[b].id; });
  for (int n : fin) {
    const Member m = members[running[n]];
    running[n] = -1;
    set_del(run_order, n);
    set_del(wmem[nodes[n].worker], n);
    complete(n);
    if (m.partner >= 0 && running[m.partner] >= 0) {
      Member& q = members[running[m.partner]];
      if (q.rate != 1.0) {
        q.rate = 1.0;
        q.sm = 1.0;
        q.memsh = 0.8;  // FULL_ALLOCATION
        log(nodes[q.node].worker, RLX_EV_RERATE, q.node, 1.0, 0.8);
      }
      q.partner = -1;
    }
  }
  std::vector<int> exp;
  for (int n : tw_order)
    if (twend[n] <= now + kEpsS) exp.push_back(n);
  std::sort(exp.begin(), exp.end(), [&](int a, int b) { return nodes[a].id < nodes[b].id; });
  for (int n : exp) {
    twend[n] = NAN;
    set_del(tw_order, n);
    complete(n);
  }
  if (!fin.empty() || !exp.empty()) auto_start_toolwaits();
  // compact the member pool once it holds only finished entries
  if (run_order.empty()) members.clear();
  return RLX_OK;
}

// Snapshot for the planner / oracle (include/rlx.h RlxStateDesc): alive
// nodes in the reference's dict order (original insertion order, merged
// nodes appended).
void ExecSoA::snapshot(RlxStateDesc* d) {
  if (snap_rev != revision) {
    const int n = (int)order.size();
    s_index.assign(nodes.size(), -1);
    for (int i = 0; i < n; i++) s_index[order[i]] = i;
    s_pipe.resize(n);
    s_worker.resize(n);
    s_kind.resize(n);
    s_dur.resize(n);
    s_mem.resize(n);
    s_rem.resize(n);
    s_act.resize(n);
    s_ctx.resize(n);
    s_ids.clear();
    s_idoff.resize(n);
    s_esrc.clear();
    s_edst.clear();
    for (int i = 0; i < n; i++) {
      const Node& x = nodes[order[i]];
      s_pipe[i] = x.pipe;
      s_worker[i] = x.worker;
      s_kind[i] = x.kind;
      s_dur[i] = x.dur;
      s_mem[i] = x.mem;
      s_rem[i] = x.rem;
      s_act[i] = x.act;
      s_ctx[i] = x.ctx;
      s_idoff[i] = (int32_t)s_ids.size();
      s_ids.insert(s_ids.end(), x.id.begin(), x.id.end());
      s_ids.push_back(0);
      for (int s : succs[order[i]]) {
        s_esrc.push_back(i);
        s_edst.push_back(s_index[s]);
      }
    }
    snap_rev = revision;
  }
  const int n = (int)order.size();
  s_done.resize(n);
  s_mpre.resize(n);
  for (int i = 0; i < n; i++) {
    s_done[i] = done[order[i]];
    const double p = mprefix[order[i]];
    s_mpre[i] = isnan(p) ? 0.0 : p;
  }
  s_rnode.clear();
  s_rpart.clear();
  s_rrate.clear();
  s_rpre.clear();
  s_rwork.clear();
  for (int x : run_order) {
    const Member& m = members[running[x]];
    s_rnode.push_back(s_index[x]);
    s_rpart.push_back(m.partner >= 0 ? s_index[m.partner] : -1);
    s_rrate.push_back(m.rate);
    s_rpre.push_back(m.prefix);
    s_rwork.push_back(m.work);
  }
  s_twn.clear();
  s_twe.clear();
  for (int x : tw_order) {
    s_twn.push_back(s_index[x]);
    s_twe.push_back(twend[x]);
  }
  s_gw.clear();
  s_gp.clear();
  s_gm.clear();
  for (long key : grant_order) {
    s_gw.push_back((int32_t)(key / P));
    s_gp.push_back((int32_t)(key % P));
    s_gm.push_back(grants[key]);
  }
  memset(d, 0, sizeof *d);
  d->now = now;
  d->n_nodes = n;
  d->n_edges = (int32_t)s_esrc.size();
  d->pipe = s_pipe.data();
  d->worker = s_worker.data();
  d->kind = s_kind.data();
  d->duration = s_dur.data();
  d->mem = s_mem.data();
  d->remaining = s_rem.data();
  d->active = s_act.data();
  d->context = s_ctx.data();
  d->completed = s_done.data();
  d->merge_prefix = s_mpre.data();
  d->ids = s_ids.data();
  d->id_off = s_idoff.data();
  d->edge_src = s_esrc.data();
  d->edge_dst = s_edst.data();
  d->n_running = (int32_t)s_rnode.size();
  d->n_toolwaits = (int32_t)s_twn.size();
  d->run_node = s_rnode.data();
  d->run_partner = s_rpart.data();
  d->run_rate = s_rrate.data();
  d->run_prefix = s_rpre.data();
  d->run_work = s_rwork.data();
  d->tw_node = s_twn.data();
  d->tw_end = s_twe.data();
  d->n_grants = (int32_t)s_gw.size();
  d->grant_worker = s_gw.data();
  d->grant_pipe = s_gp.data();
  d->grant_mem = s_gm.data();
}

}  // namespace rlx

using rlx::ExecSoA;

extern "C" {

int rlx_state_create(const RlxInstanceDesc* in, const RlxGraphDesc* g, int record, void** out) {
  if (!in || !g || !out) return RLX_ERR_ARG;
  *out = nullptr;
  ExecSoA* s = new ExecSoA();
  int rc = s->init(in, g, record != 0);
  *out = s;  // returned even on failure so rlx_state_error can report
  return rc;
}

int rlx_state_clone(const void* st, void** out) {
  if (!st || !out) return RLX_ERR_ARG;
  ExecSoA* c = new ExecSoA(*(const ExecSoA*)st);
  c->record = false;
  c->events.clear();
  c->snap_rev = -1;
  *out = c;
  return RLX_OK;
}

void rlx_state_destroy(void* st) { delete (ExecSoA*)st; }

const char* rlx_state_error(const void* st) { return st ? ((const ExecSoA*)st)->err.c_str() : "null state"; }

int rlx_state_apply(void* st, const RlxApply* a) {
  if (!st || !a) return RLX_ERR_ARG;
  return ((ExecSoA*)st)->apply(a);
}

int rlx_state_advance(void* st, int has_until, double until) {
  if (!st) return RLX_ERR_ARG;
  return ((ExecSoA*)st)->advance(has_until != 0, until);
}

int rlx_state_info(const void* st, RlxStateInfo* out) {
  if (!st || !out) return RLX_ERR_ARG;
  const ExecSoA* s = (const ExecSoA*)st;
  memset(out, 0, sizeof *out);
  out->now = s->now;
  out->makespan = s->makespan;
  out->n_total = (int32_t)s->nodes.size();
  out->n_alive = (int32_t)s->order.size();
  out->n_done = s->n_done;
  out->done = s->n_done == (int)s->order.size();
  out->has_events = !s->run_order.empty() || !s->tw_order.empty();
  out->n_running = (int32_t)s->run_order.size();
  out->n_toolwaits = (int32_t)s->tw_order.size();
  out->revision = s->revision;
  out->n_events = (int64_t)s->events.size();
  return RLX_OK;
}

int rlx_state_snapshot(void* st, RlxStateDesc* out) {
  if (!st || !out) return RLX_ERR_ARG;
  ((ExecSoA*)st)->snapshot(out);
  return RLX_OK;
}

int rlx_state_node(const void* st, int32_t node, RlxNodeInfo* out) {
  const ExecSoA* s = (const ExecSoA*)st;
  if (!s || !out || node < 0 || node >= (int)s->nodes.size()) return RLX_ERR_ARG;
  const rlx::Node& n = s->nodes[node];
  memset(out, 0, sizeof *out);
  out->pipe = n.pipe;
  out->worker = n.worker;
  out->kind = n.kind;
  out->alive = s->alive[node];
  out->completed = s->done[node];
  out->running = s->running[node] >= 0;
  out->duration = n.dur;
  out->mem = n.mem;
  out->completion_time = s->ctime[node];
  out->remaining = n.rem;
  out->active = n.act;
  out->context = n.ctx;
  out->token_total = n.tok;
  out->span_lo = n.span_lo;
  out->span_hi = n.span_hi;
  out->id = n.id.c_str();
  return RLX_OK;
}

int rlx_state_events(const void* st, int64_t first, int64_t count, RlxEvent* out) {
  const ExecSoA* s = (const ExecSoA*)st;
  if (!s || !out || first < 0 || count < 0 || first + count > (int64_t)s->events.size()) return RLX_ERR_ARG;
  if (count) memcpy(out, s->events.data() + first, sizeof(RlxEvent) * count);
  return RLX_OK;
}

int rlx_state_completion(const void* st, uint8_t* completed, double* times) {
  const ExecSoA* s = (const ExecSoA*)st;
  if (!s) return RLX_ERR_ARG;
  for (size_t i = 0; i < s->nodes.size(); i++) {
    if (completed) completed[i] = s->done[i];
    if (times) times[i] = s->ctime[i];
  }
  return RLX_OK;
}

}  // extern "C"

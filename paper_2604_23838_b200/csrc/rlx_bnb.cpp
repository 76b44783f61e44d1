// rlx_bnb.cpp — the brute-force oracle as native branch-and-bound
// (rlmux/scheduler.py:1086-1226), plus a native
// enumerate_actions (:648-703) over the execution state.
//
// `brute_force_schedule` searches action sequences (including idling) for
// the minimal makespan of a <= 10-node instance: depth-first over
// enumerate_actions (deduplicated, :1086-1110) then one `advance`, pruned by
// the best makespan so far against a critical-path bound over work merging
// cannot shrink (:1113-1129, :1180-1195) and by a memo of canonical states
// (:1132-1143, :1196-1200). The search runs here on copies of the native
// ExecState (rlx_state.cpp) in the reference's exact visiting order, so it
// returns the same schedule; the host seeds it with the look-ahead, greedy
// and serial schedules' best makespan (:1152-1170, scheduler.py here).
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "rlx_state.hpp"

namespace rlx {
namespace {

constexpr double kEps = 1e-9;  // scheduler.py:43
const double kMemGrid[4] = {0.20, 0.40, 0.60, 0.80};

bool mergeable(int kind) { return kind == RLX_KIND_DECODE_SMALL || kind == RLX_KIND_DECODE_MEDIUM; }

// round(x, nd) of a Python float: the float nearest the correctly rounded
// decimal (glibc formats exactly; strtod rounds correctly)
double py_round(double x, int nd) {
  char buf[64];
  snprintf(buf, sizeof buf, "%.*f", nd, x);
  return strtod(buf, nullptr);
}

struct Ctx {
  const RlxInstanceDesc* in;
  std::vector<std::string> pipe_ids;
  double best;
  std::vector<std::pair<double, RlxApply>> trail, best_actions;
  bool improved = false;
  std::map<std::string, double> memo;
  int64_t visited = 0;

  double lut(int kind, int partner, int alloc) const {
    if (kind == RLX_KIND_TOOL_WAIT) return 1.0;  // slowdown.py:135-136
    return in->lut[(kind * RLX_NPARTNER + partner + 1) * RLX_NALLOC + alloc];
  }

  // ready_compute (:404-410): not a tool wait, ready; sorted by (pipeline id, id)
  std::vector<int> ready(const ExecSoA& s) const {
    std::vector<int> out;
    for (int n : s.order)
      if (s.nodes[n].kind != RLX_KIND_TOOL_WAIT && s.is_ready(n)) out.push_back(n);
    std::sort(out.begin(), out.end(), [&](int a, int b) {
      const std::string &pa = pipe_ids[s.nodes[a].pipe], &pb = pipe_ids[s.nodes[b].pipe];
      if (pa != pb) return pa < pb;
      return s.nodes[a].id < s.nodes[b].id;
    });
    return out;
  }

  // enumerate_actions (:648-703), in serial order
  std::vector<RlxApply> enumerate(const ExecSoA& s) const {
    std::vector<RlxApply> out;
    const std::vector<int> rd = ready(s);
    std::vector<std::vector<int>> by_w(s.W);
    for (int n : rd) by_w[s.nodes[n].worker].push_back(n);
    const double hr = s.headroom;
    for (int w = 0; w < s.W; w++) {  // dense worker order == sorted worker ids
      if (!s.wmem[w].empty()) continue;
      const std::vector<int>& grp = by_w[w];
      for (size_t i = 0; i < grp.size(); i++)
        for (size_t j = i + 1; j < grp.size(); j++) {
          const int a = grp[i], b = grp[j];
          if (s.nodes[a].pipe == s.nodes[b].pipe) continue;
          if (!(s.nodes[a].mem + s.nodes[b].mem <= 1.0 - hr + 1e-12)) continue;  // feasible
          for (int o = 0; o < 2; o++) {
            const int f = o ? b : a, sc = o ? a : b;
            for (int ai = 0; ai < 3; ai++)
              for (int mj = 0; mj < 4; mj++) {
                if (kMemGrid[mj] + s.nodes[sc].mem > 1.0 - hr + kEps) continue;
                const int al = 1 + ai * 4 + mj;
                RlxApply x;
                memset(&x, 0, sizeof x);
                x.cls = RLX_CLASS_MULTIPLEX;
                x.node_a = f;
                x.node_b = sc;
                x.rate_a = lut(s.nodes[f].kind, s.nodes[sc].kind, al);
                x.rate_b = lut(s.nodes[sc].kind, s.nodes[f].kind, al + 12);
                x.sm_a = in->alloc_sm[al];
                x.mem_a = in->alloc_mem[al];
                x.sm_b = in->alloc_sm[al + 12];
                x.mem_b = in->alloc_mem[al + 12];
                out.push_back(x);
              }
          }
        }
    }
    if (in->merge_enabled) {
      std::vector<int> pids;
      std::vector<std::vector<int>> frags(s.P);
      for (int n : rd)
        if (mergeable(s.nodes[n].kind)) frags[s.nodes[n].pipe].push_back(n);
      for (int p = 0; p < s.P; p++) pids.push_back(p);
      std::sort(pids.begin(), pids.end(), [&](int a, int b) { return pipe_ids[a] < pipe_ids[b]; });
      for (int p : pids) {
        const std::vector<int>& fr = frags[p];
        const int nf = (int)fr.size();
        if (nf < 2) continue;
        for (int size = 2; size <= nf; size++) {
          std::vector<int> idx(size);
          for (int k = 0; k < size; k++) idx[k] = k;
          for (;;) {  // itertools.combinations order
            std::vector<int> mem;
            for (int k = 0; k < size; k++) mem.push_back(fr[idx[k]]);
            std::vector<int> ws;
            for (int m : mem) ws.push_back(s.nodes[m].worker);
            std::vector<int> wsort(ws);
            std::sort(wsort.begin(), wsort.end());
            const bool distinct = std::adjacent_find(wsort.begin(), wsort.end()) == wsort.end();
            if (distinct) {
              std::sort(mem.begin(), mem.end(), [&](int a, int b) { return s.nodes[a].id < s.nodes[b].id; });
              for (int t : wsort) {
                RlxApply x;
                memset(&x, 0, sizeof x);
                x.cls = RLX_CLASS_MERGE;
                x.n_members = size;
                for (int k = 0; k < size; k++) x.members[k] = mem[k];
                x.target_worker = t;
                out.push_back(x);
              }
            }
            int k = size - 1;
            while (k >= 0 && idx[k] == nf - size + k) k--;
            if (k < 0) break;
            idx[k]++;
            for (int q = k + 1; q < size; q++) idx[q] = idx[q - 1] + 1;
          }
        }
      }
    }
    for (int n : rd)
      if (s.wmem[s.nodes[n].worker].empty()) {
        RlxApply x;
        memset(&x, 0, sizeof x);
        x.cls = RLX_CLASS_EXCLUSIVE;
        x.node_a = n;
        x.rate_a = lut(s.nodes[n].kind, -1, 0);
        x.sm_a = in->alloc_sm[0];
        x.mem_a = in->alloc_mem[0];
        out.push_back(x);
      }
    return out;
  }

  // _dedupe_candidates (:1086-1110): allocations with identical rounded rates
  std::vector<RlxApply> dedupe(const ExecSoA& s, const std::vector<RlxApply>& c) const {
    std::vector<RlxApply> out;
    std::vector<std::string> seen;
    char buf[256];
    for (const RlxApply& x : c) {
      std::string key;
      if (x.cls == RLX_CLASS_MULTIPLEX) {
        snprintf(buf, sizeof buf, "|%.17g|%.17g", py_round(x.rate_a, 12), py_round(x.rate_b, 12));
        key = "mux|" + s.nodes[x.node_a].id + "|" + s.nodes[x.node_b].id + buf;
      } else if (x.cls == RLX_CLASS_MERGE) {
        key = "merge";
        for (int k = 0; k < x.n_members; k++) key += "|" + s.nodes[x.members[k]].id;
        key += "@" + std::to_string(x.target_worker);
      } else {
        key = "excl|" + s.nodes[x.node_a].id;
      }
      if (std::find(seen.begin(), seen.end(), key) != seen.end()) continue;
      seen.push_back(key);
      out.push_back(x);
    }
    return out;
  }

  // _unmergeable_suffix (:1113-1129): longest downstream chain of work that
  // merging cannot shrink (the result does not depend on the visiting order)
  std::vector<double> suffix(const ExecSoA& s) const {
    const int N = (int)s.nodes.size();
    std::vector<int> indeg(N, 0), order;
    for (int n : s.order)
      for (int p : s.preds[n]) indeg[n] += s.alive[p] ? 1 : 0;
    std::vector<int> stack;
    for (int n : s.order)
      if (indeg[n] == 0) stack.push_back(n);
    while (!stack.empty()) {
      const int n = stack.back();
      stack.pop_back();
      order.push_back(n);
      for (int x : s.succs[n])
        if (s.alive[x] && --indeg[x] == 0) stack.push_back(x);
    }
    std::vector<double> suf(N, 0.0);
    for (auto it = order.rbegin(); it != order.rend(); ++it) {
      const int n = *it;
      double m = 0.0;
      for (int x : s.succs[n])
        if (s.alive[x] && suf[x] > m) m = suf[x];
      suf[n] = (mergeable(s.nodes[n].kind) ? 0.0 : s.nodes[n].dur) + m;
    }
    return suf;
  }

  // _state_key (:1132-1143): completed set, running members (rounded), tool
  // waits (rounded, relative), pending set — by node id
  std::string key(const ExecSoA& s) const {
    std::vector<std::string> comp, pend, run, wait;
    char buf[256];
    for (int n : s.order) {
      if (s.done[n]) comp.push_back(s.nodes[n].id);
      else if (s.running[n] < 0) pend.push_back(s.nodes[n].id);
    }
    for (int n : s.run_order) {
      const Member& m = s.members[s.running[n]];
      snprintf(buf, sizeof buf, "|%d|%.17g|%.17g|%.17g", s.nodes[n].worker, py_round(m.prefix, 9),
               py_round(m.work, 9), py_round(m.rate, 9));
      run.push_back(s.nodes[n].id + buf);
    }
    for (int n : s.tw_order) {
      snprintf(buf, sizeof buf, "|%.17g", py_round(s.twend[n] - s.now, 9));
      wait.push_back(s.nodes[n].id + buf);
    }
    std::sort(comp.begin(), comp.end());
    std::sort(pend.begin(), pend.end());
    std::sort(run.begin(), run.end());
    std::sort(wait.begin(), wait.end());
    std::string k;
    for (auto* v : {&comp, &run, &wait, &pend}) {
      for (const std::string& x : *v) k += x + "\x1f";
      k += "\x1e";
    }
    return k;
  }

  void dfs(const ExecSoA& s) {
    visited++;
    if (s.n_done == (int)s.order.size()) {
      if (s.makespan < best - kEps) {
        best = s.makespan;
        best_actions = trail;
        improved = true;
      }
      return;
    }
    const std::vector<double> suf = suffix(s);
    double bound = s.now;
    for (int n : s.order) {
      if (s.done[n]) continue;
      double start, tail = 0.0;
      auto succ_max = [&]() {
        double m = 0.0;
        bool any = false;
        for (int x : s.succs[n])
          if (s.alive[x]) {
            m = any ? (suf[x] > m ? suf[x] : m) : suf[x];
            any = true;
          }
        return any ? m : 0.0;
      };
      if (s.running[n] >= 0) {
        const Member& m = s.members[s.running[n]];
        start = (s.now + m.prefix) + m.work * m.rate;  // finish_estimate (:328)
        tail = succ_max();
      } else if (!isnan(s.twend[n])) {
        start = s.twend[n];
        tail = succ_max();
      } else {
        start = s.now + suf[n];
      }
      const double v = start + tail;
      bound = bound > v ? bound : v;
    }
    if (bound >= best - kEps) return;
    const std::string k = key(s);
    auto it = memo.find(k);
    if (it != memo.end() && it->second <= s.now + kEps) return;
    memo[k] = s.now;
    const std::vector<RlxApply> cands = dedupe(s, enumerate(s));
    for (const RlxApply& a : cands) {
      ExecSoA child(s);
      if (child.apply(&a) != RLX_OK) continue;
      trail.emplace_back(s.now, a);
      dfs(child);
      trail.pop_back();
    }
    if (!s.run_order.empty() || !s.tw_order.empty()) {
      ExecSoA child(s);
      if (child.advance(false, 0.0) == RLX_OK) dfs(child);
    }
  }
};

}  // namespace
}  // namespace rlx

using namespace rlx;

namespace {

}  // namespace

// RlxApply (rates resolved) -> RlxAction (allocation index) in the state's
// node index space
RlxAction to_action(const RlxInstanceDesc* in, const RlxApply& a) {
  RlxAction x;
  memset(&x, 0, sizeof x);
  x.cls = a.cls;
  x.node_a = x.node_b = -1;
  if (a.cls == RLX_CLASS_MERGE) {
    x.n_members = a.n_members;
    for (int k = 0; k < a.n_members; k++) x.members[k] = a.members[k];
    x.target_worker = a.target_worker;
    return x;
  }
  x.node_a = a.node_a;
  if (a.cls == RLX_CLASS_MULTIPLEX) x.node_b = a.node_b;
  for (int i = 0; i < RLX_NALLOC; i++)
    if (in->alloc_sm[i] == a.sm_a && in->alloc_mem[i] == a.mem_a) {
      x.alloc = i;
      break;
    }
  return x;
}

extern "C" {

int rlx_enumerate(const RlxInstanceDesc* in, const void* state, RlxAction* out, int64_t cap, int64_t* n_out) {
  if (!in || !state || !n_out) return RLX_ERR_ARG;
  Ctx c;
  c.in = in;
  for (int p = 0; p < in->n_pipes; p++) c.pipe_ids.push_back(in->pipe_names + in->pipe_name_off[p]);
  const std::vector<RlxApply> v = c.enumerate(*(const ExecSoA*)state);
  *n_out = (int64_t)v.size();
  for (int64_t i = 0; i < (int64_t)v.size() && i < cap; i++) out[i] = to_action(in, v[i]);
  return RLX_OK;
}

int rlx_branch_and_bound(const RlxInstanceDesc* in, const RlxGraphDesc* g, double best_makespan, int32_t cap,
                         RlxStep* out, int32_t* n_out, double* best_out, int64_t* visited) {
  if (!in || !g || !n_out || !best_out) return RLX_ERR_ARG;
  ExecSoA root;
  int rc = root.init(in, g, false);
  if (rc) return rc;
  Ctx c;
  c.in = in;
  for (int p = 0; p < in->n_pipes; p++) c.pipe_ids.push_back(in->pipe_names + in->pipe_name_off[p]);
  c.best = best_makespan;
  c.dfs(root);
  *best_out = c.best;
  if (visited) *visited = c.visited;
  if (!c.improved) {
    *n_out = -1;  // no schedule beats the seeds by more than EPS
    return RLX_OK;
  }
  *n_out = (int32_t)c.best_actions.size();
  if ((int32_t)c.best_actions.size() > cap) return RLX_ERR_LIMIT;
  for (size_t i = 0; i < c.best_actions.size(); i++) {
    memset(&out[i], 0, sizeof out[i]);
    out[i].start = c.best_actions[i].first;
    out[i].action = to_action(in, c.best_actions[i].second);
  }
  return RLX_OK;
}

}  // extern "C"

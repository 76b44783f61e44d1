// rlx_sim.cpp — batched replay of schedules into their metrics
// (rlmux/sim.py:69-173).
//
// `simulate(schedule, instance)` replays one action log on an ExecState and
// folds the result into makespan, per-pipeline latency / tokens, aggregate
// throughput and per-worker utilisation. Sweeps and acceptance trends
// replay thousands of schedules; here every schedule is
// replayed on its own copy of the native ExecState (rlx_state.cpp), spread
// over host threads, with the metrics computed natively in the reference's
// operation order (bit-identical to the single-schedule path, sim.py).
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "rlx_state.hpp"

namespace rlx {
namespace {

constexpr double kEps = 1e-9;  // scheduler.py:43

bool compute_bound(int kind) {  // sim.py COMPUTE_BOUND_KINDS
  return kind == RLX_KIND_TRAINING || kind == RLX_KIND_REFERENCE || kind == RLX_KIND_PREFILL_BURST ||
         kind == RLX_KIND_DECODE_LARGE;
}

// float(f"{x:.4f}"): the share an event's alloc string carries (sim.py:84-87)
double share_of(double sm) {
  char buf[64];
  snprintf(buf, sizeof buf, "%.4f", sm);
  return strtod(buf, nullptr);
}

std::string py_repr_str(const std::string& s) { return "'" + s + "'"; }

// Python 3.12's built-in sum() over floats (Objects/bltinmodule.c builtin_sum):
// the first item is added to the int start 0, the rest with Neumaier's
// compensated summation, the compensation folded in at the end. The
// reference's utilisation averages are such sums (sim.py:113).
struct PySum {
  bool any = false;
  double f = 0.0, c = 0.0;
  void add(double x) {
    if (!any) {
      any = true;
      f = 0.0 + x;
      return;
    }
    const double t = f + x;
    if (fabs(f) >= fabs(x))
      c += (f - t) + x;
    else
      c += (x - t) + f;
    f = t;
  }
  double value() const { return (c != 0.0 && isfinite(c)) ? f + c : f; }
};

struct Replayer {
  const RlxInstanceDesc* in;
  const ExecSoA* base;
  const std::unordered_map<std::string, int>* index0;

  int alloc_index(double sm, double mem) const {
    for (int i = 0; i < RLX_NALLOC; i++)
      if (in->alloc_sm[i] == sm && in->alloc_mem[i] == mem) return i;
    return -1;
  }
  double lut(int kind, int partner, int alloc) const {
    return in->lut[(kind * RLX_NPARTNER + partner + 1) * RLX_NALLOC + alloc];
  }

  int run(const RlxSimAction* acts, int64_t n, const char* ids, RlxSimResult* r, double* plat, int64_t* ptok,
          double* util) const {
    ExecSoA st(*base);
    st.record = true;
    st.events.clear();
    std::unordered_map<std::string, int> idx(*index0);
    auto fail = [&](int code, int64_t at, const std::string& msg) {
      r->status = code;
      r->action_index = (int32_t)at;
      snprintf(r->error, sizeof r->error, "%s", msg.c_str());
      return code;
    };
    auto node_of = [&](const char* id, int& out) {
      auto it = idx.find(id);
      if (it == idx.end() || !st.alive[it->second]) return false;
      out = it->second;
      return true;
    };
    for (int64_t k = 0; k < n; k++) {
      const RlxSimAction& a = acts[k];
      if (a.start < st.now - 1e-6)
        return fail(RLX_ERR_SCHEDULING, k, "action at t=" + py_float(a.start) + " recorded after simulated time " +
                                               py_float(st.now));
      while (st.now < a.start - kEps) {  // sim.py:125-129
        const bool has = !st.run_order.empty() || !st.tw_order.empty();
        int rc = st.advance(true, a.start);
        if (rc) return fail(rc, k, st.err);
        if (!has) break;
      }
      RlxApply ap;
      memset(&ap, 0, sizeof ap);
      ap.cls = a.cls;
      const char* p = ids + a.id_off;
      std::vector<int> nd;
      for (int i = 0; i < a.n_ids; i++) {
        int x;
        if (!node_of(p, x)) return fail(RLX_ERR_SCHEDULING, k, "unknown sub-stage " + py_repr_str(p));
        nd.push_back(x);
        p += strlen(p) + 1;
      }
      if (a.cls == RLX_CLASS_EXCLUSIVE) {
        const int ai = alloc_index(a.sm, a.mem);
        if (ai < 0) return fail(RLX_ERR_LIMIT, k, "allocation outside the slowdown LUT");
        ap.node_a = nd[0];
        ap.rate_a = lut(st.nodes[nd[0]].kind, -1, ai);
        ap.sm_a = a.sm;
        ap.mem_a = a.mem;
        if (isnan(ap.rate_a))
          return fail(RLX_ERR_KEY, k, "slowdown table has no entry for this allocation");
      } else if (a.cls == RLX_CLASS_MULTIPLEX) {
        const int ai = alloc_index(a.sm, a.mem);
        if (ai < 1 || ai > 12) return fail(RLX_ERR_LIMIT, k, "allocation outside the slowdown LUT");
        const int ka = st.nodes[nd[0]].kind, kb = st.nodes[nd[1]].kind;
        ap.node_a = nd[0];
        ap.node_b = nd[1];
        ap.rate_a = lut(ka, kb, ai);
        ap.rate_b = lut(kb, ka, ai + 12);
        ap.sm_a = a.sm;
        ap.mem_a = a.mem;
        ap.sm_b = in->alloc_sm[ai + 12];
        ap.mem_b = in->alloc_mem[ai + 12];
      } else if (a.cls == RLX_CLASS_MERGE) {
        if (a.n_ids > RLX_MAX_MEMBERS) return fail(RLX_ERR_LIMIT, k, "merge sets above 64 members");
        ap.n_members = a.n_ids;
        for (int i = 0; i < a.n_ids; i++) ap.members[i] = nd[i];
        ap.target_worker = -1;
        for (int w = 0; w < st.W; w++)
          if (st.worker_ids[w] == a.target_worker) ap.target_worker = w;
      } else {
        return fail(RLX_ERR_ARG, k, "unknown action class");
      }
      const int before = (int)st.nodes.size();
      int rc = st.apply(&ap);
      if (rc) return fail(rc, k, st.err);
      if ((int)st.nodes.size() > before) idx[st.nodes.back().id] = before;
    }
    while (st.n_done < (int)st.order.size()) {  // sim.py:134-140
      if (st.run_order.empty() && st.tw_order.empty()) {
        std::vector<std::string> pend;
        for (int i : st.order)
          if (!st.done[i]) pend.push_back(st.nodes[i].id);
        std::sort(pend.begin(), pend.end());
        std::string m = "schedule leaves work unscheduled: [";
        for (size_t i = 0; i < pend.size() && i < 4; i++) m += (i ? ", " : "") + py_repr_str(pend[i]);
        return fail(RLX_ERR_SCHEDULING, n, m + "]");
      }
      int rc = st.advance(false, 0.0);
      if (rc) return fail(rc, n, st.err);
    }
    // ---- metrics (sim.py:142-158)
    const int P = st.P, W = st.W;
    for (int q = 0; q < P; q++) {
      plat[q] = 0.0;
      ptok[q] = 0;
    }
    for (int i : st.order) {
      if (!st.done[i]) continue;
      const int q = st.nodes[i].pipe;
      plat[q] = std::max(plat[q], st.ctime[i]);
      ptok[q] += st.nodes[i].tok;
    }
    int64_t total = 0;
    for (int q = 0; q < P; q++) total += ptok[q];
    r->makespan = st.makespan;
    r->total_tokens = total;
    r->throughput = st.makespan > 0 ? (double)total / st.makespan : 0.0;
    // ---- utilisation (sim.py:69-115): per-worker SM-share segments
    std::vector<double> share(W, 0.0), seg0(W, 0.0);
    std::vector<PySum> busy(W);
    std::vector<double> node_share(st.nodes.size(), NAN);  // NaN: no entry
    auto close = [&](int w, double t) {
      if (t > seg0[w] + kEps) {
        const double s = std::min(1.0, share[w]);
        busy[w].add((t - seg0[w]) * s);
      }
      seg0[w] = t;
    };
    for (const RlxEvent& e : st.events) {
      if (e.kind != RLX_EV_START && e.kind != RLX_EV_FINISH && e.kind != RLX_EV_RERATE) continue;
      const bool counts = st.alive[e.node] && compute_bound(st.nodes[e.node].kind);
      const int w = e.worker;
      if (e.kind == RLX_EV_START) {
        const double sm = (counts && e.sm == e.sm) ? share_of(e.sm) : 0.0;
        node_share[e.node] = sm;
        if (sm != 0.0) {
          close(w, e.time);
          share[w] += sm;
        }
      } else if (e.kind == RLX_EV_RERATE) {
        const double old = node_share[e.node] == node_share[e.node] ? node_share[e.node] : 0.0;
        const double nw = (counts && e.sm == e.sm) ? share_of(e.sm) : 0.0;
        if (counts) {
          close(w, e.time);
          share[w] += nw - old;
          node_share[e.node] = nw;
        }
      } else {
        double sm = node_share[e.node];
        node_share[e.node] = NAN;
        if (sm != sm) sm = 0.0;
        if (sm != 0.0) {
          close(w, e.time);
          share[w] -= sm;
        }
      }
    }
    for (int w = 0; w < W; w++) {
      close(w, st.makespan);
      util[w] = st.makespan > 0 ? busy[w].value() / st.makespan : 0.0;
    }
    r->status = RLX_OK;
    r->action_index = -1;
    r->error[0] = 0;
    return RLX_OK;
  }
};

}  // namespace
}  // namespace rlx

using namespace rlx;

extern "C" int rlx_simulate_batch(const RlxInstanceDesc* in, const RlxGraphDesc* g, int32_t n_sched,
                                  const int64_t* sched_off, const RlxSimAction* acts, const char* ids,
                                  int32_t n_threads, RlxSimResult* res, double* pipe_latency, int64_t* pipe_tokens,
                                  double* util_avg) {
  if (!in || !g || n_sched < 0 || !sched_off || !res || !pipe_latency || !pipe_tokens || !util_avg) return RLX_ERR_ARG;
  ExecSoA base;
  int rc = base.init(in, g, true);
  if (rc) {
    for (int s = 0; s < n_sched; s++) {
      res[s].status = rc;
      snprintf(res[s].error, sizeof res[s].error, "%s", base.err.c_str());
    }
    return rc;
  }
  std::unordered_map<std::string, int> index0;
  for (int i = 0; i < (int)base.nodes.size(); i++) index0[base.nodes[i].id] = i;
  Replayer R{in, &base, &index0};
  const int P = base.P, W = base.W;
  std::atomic<int> next(0);
  auto work = [&]() {
    for (;;) {
      const int s = next.fetch_add(1);
      if (s >= n_sched) break;
      memset(&res[s], 0, sizeof res[s]);
      R.run(acts + sched_off[s], sched_off[s + 1] - sched_off[s], ids, &res[s], pipe_latency + (size_t)s * P,
            pipe_tokens + (size_t)s * P, util_avg + (size_t)s * W);
    }
  };
  int nt = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if (nt > n_sched) nt = n_sched > 0 ? n_sched : 1;
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; t++) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  return RLX_OK;
}

// rlx_state.hpp — native execution state of the decision loop (rlx_state.cpp).
#pragma once
#include <stdint.h>

#include <map>
#include <string>
#include <vector>

#include "../../include/rlx.h"

namespace rlx {

struct Node {
  int pipe = 0, worker = 0, kind = 0;
  double dur = 0.0, mem = 0.0;
  int64_t rem = 0, act = 0, ctx = 0, tok = 0, span_lo = 0, span_hi = 0;
  std::string id;
};

struct Member {
  int node = -1;
  double rate = 1.0, sm = 1.0, memsh = 0.8, prefix = 0.0, work = 0.0, started = 0.0;
  int partner = -1;
};

// The reference's ExecState (rlmux/scheduler.py:339-634) on index arrays.
// Node indices are stable: a merge appends the merged node and marks its
// members dead.
struct ExecSoA {
  // instance
  int P = 0, W = 0;
  double headroom = 0.05, realloc_penalty = 0.0, default_migration_cost = 0.0;
  std::vector<int32_t> worker_ids;
  std::vector<double> latency, params, peak, mfu;
  std::vector<uint8_t> latency_ok, has_spec;
  // graph + state
  std::vector<Node> nodes;
  std::vector<uint8_t> alive, done;
  std::vector<int> running;          // node -> index into `members`, -1 if not running
  std::vector<double> ctime, twend;  // completion time; tool-wait end (NaN: not waiting)
  std::vector<double> mprefix;       // pending merge prefix (NaN: none)
  std::vector<std::vector<int>> preds, succs;
  std::vector<int> order;            // alive nodes, dict order
  std::vector<int> run_order;        // running nodes, dict order
  std::vector<int> tw_order;         // running tool waits, dict order
  std::vector<int> tw_sorted;        // tool-wait nodes by id
  std::vector<Member> members;
  std::vector<std::vector<int>> wmem;  // worker -> running member nodes
  std::map<long, double> grants;       // (worker*P + pipe) -> last mem grant
  std::vector<long> grant_order;
  double now = 0.0, makespan = 0.0;
  int n_done = 0;
  int64_t revision = 0;
  bool record = false;
  std::vector<RlxEvent> events;
  std::string err;
  // snapshot buffers
  int64_t snap_rev = -1;
  std::vector<int> s_index;
  std::vector<int32_t> s_pipe, s_worker, s_kind, s_idoff, s_esrc, s_edst, s_rnode, s_rpart, s_twn, s_gw, s_gp;
  std::vector<double> s_dur, s_mem, s_mpre, s_rrate, s_rpre, s_rwork, s_twe, s_gm;
  std::vector<int64_t> s_rem, s_act, s_ctx;
  std::vector<uint8_t> s_done;
  std::vector<char> s_ids;

  int init(const RlxInstanceDesc* in, const RlxGraphDesc* g, bool record);
  int fail(int code, const std::string& msg);
  void log(int worker, int kind, int node, double sm, double mem);
  bool is_ready(int n) const;
  void complete(int n);
  void auto_start_toolwaits();
  int require_ready(int n);
  void start_member(int n, double rate, double sm, double memsh, int partner);
  int apply(const RlxApply* a);
  int merge(const RlxApply* a);
  bool next_event(double& t) const;
  int advance(bool has_until, double until);
  void snapshot(RlxStateDesc* d);
};

std::string py_float(double x);

}  // namespace rlx

// rlx_plan.cpp — host planner: decision-state snapshot -> DevPlan blob.
//
// Everything computed here is per-decision invariant across candidates
// (verified there on 11,834 non-merge and 1,004
// merge candidates): the W-round window (rlmux/scheduler.py:710-748) and
// the tool waits that may still auto-start outside it (:421-434), the
// suffix lengths (:751-770), the per-worker ready orders of the two
// completion keys (:893-894), and the candidate space of
// enumerate_actions (:648-703) in its exact serial order. Merge
// candidates are laid out as (pipeline, size) blocks that the device
// unranks combinatorially; only pipelines whose fragments share a worker
// (the reference skips such combos without numbering them, :690-692) get
// an explicit combo list.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <string>
#include <vector>

#include "../../include/rlx.h"
#include "rlx_hostplan.hpp"

namespace rlx {

static void fill_binom(std::vector<uint64_t>& b) {
  const uint64_t SAT = uint64_t(1) << 62;
  b.assign((kMaxFrags + 1) * kBinomK, 0);
  for (int n = 0; n <= kMaxFrags; n++) {
    b[n * kBinomK] = 1;
    for (int k = 1; k < kBinomK && k <= n; k++) {
      uint64_t v = b[(n - 1) * kBinomK + k - 1] + (k <= n - 1 ? b[(n - 1) * kBinomK + k] : 0);
      b[n * kBinomK + k] = v > SAT ? SAT : v;
    }
  }
}

int build_plan(const RlxInstanceDesc* in, const RlxStateDesc* sd, int rounds, int max_merge, HostPlan& hp,
               std::string& err) {
  const int N = sd->n_nodes, W = in->n_workers, P = in->n_pipes;
  if (N <= 0 || W <= 0 || P <= 0) {
    err = "empty state";
    return RLX_ERR_ARG;
  }
  if (W > 128) { err = "more than 128 workers"; return RLX_ERR_LIMIT; }
  if (P > 255) { err = "more than 255 pipelines"; return RLX_ERR_LIMIT; }
  std::vector<std::vector<int>> preds(N), succs(N);
  for (int e = 0; e < sd->n_edges; e++) {
    int s = sd->edge_src[e], d = sd->edge_dst[e];
    if (s < 0 || s >= N || d < 0 || d >= N) { err = "edge index out of range"; return RLX_ERR_ARG; }
    succs[s].push_back(d);
    preds[d].push_back(s);
  }
  std::vector<uint8_t> done(N), run(N, 0), twr(N, 0);
  for (int i = 0; i < N; i++) done[i] = sd->completed[i] ? 1 : 0;
  std::vector<int> nmem(W, 0);
  for (int k = 0; k < sd->n_running; k++) {
    int i = sd->run_node[k];
    run[i] = 1;
    if (++nmem[sd->worker[i]] > 2) { err = "more than two running members on a worker"; return RLX_ERR_ARG; }
  }
  for (int k = 0; k < sd->n_toolwaits; k++) twr[sd->tw_node[k]] = 1;
  auto id = [&](int i) { return sd->ids + sd->id_off[i]; };
  std::vector<const char*> pname(P);
  for (int p = 0; p < P; p++) pname[p] = in->pipe_names + in->pipe_name_off[p];
  std::vector<uint8_t> prank(P);
  for (int p = 0; p < P; p++) {
    int r = 0;
    for (int q = 0; q < P; q++) r += strcmp(pname[q], pname[p]) < 0;
    prank[p] = (uint8_t)r;
  }
  // name rank: (pipeline id, id) string order (scheduler.py:410)
  std::vector<int> order(N);
  for (int i = 0; i < N; i++) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    int c = strcmp(pname[sd->pipe[a]], pname[sd->pipe[b]]);
    if (c) return c < 0;
    return strcmp(id(a), id(b)) < 0;
  });
  std::vector<int> nrank(N);
  for (int r = 0; r < N; r++) nrank[order[r]] = r;

  auto preds_done = [&](int i) {
    for (int p : preds[i])
      if (!done[p]) return false;
    return true;
  };
  std::vector<uint8_t> ready(N, 0);
  for (int i = 0; i < N; i++) ready[i] = !done[i] && !run[i] && !twr[i] && preds_done(i);

  // ---- window (scheduler.py:710-748)
  std::vector<uint8_t> win(N, 0), cov(N, 0), nx(N, 0), fr(N, 0);
  for (int i = 0; i < N; i++) {
    win[i] = run[i] || twr[i] || ready[i];
    cov[i] = done[i] || win[i];
  }
  for (int depth = 1; depth < rounds; depth++) {
    std::fill(nx.begin(), nx.end(), 0);
    int cnt = 0;
    for (int i = 0; i < N; i++) {
      if (cov[i]) continue;
      bool ok = true;
      for (int p : preds[i]) ok = ok && cov[p];
      if (ok) nx[i] = 1, cnt++;
    }
    if (!cnt) break;
    for (int i = 0; i < N; i++)
      if (nx[i]) win[i] = cov[i] = 1;
    for (;;) {
      int nf = 0;
      std::fill(fr.begin(), fr.end(), 0);
      for (int i = 0; i < N; i++) {
        if (cov[i]) continue;
        bool ok = true, gate = false;
        for (int p : preds[i]) {
          ok = ok && cov[p];
          gate = gate || (nx[p] && sd->kind[p] == RLX_KIND_TOOL_WAIT);
        }
        if (ok && gate) fr[i] = 1, nf++;
      }
      if (!nf) break;
      for (int i = 0; i < N; i++)
        if (fr[i]) nx[i] = win[i] = cov[i] = 1;
    }
  }
  // ---- auxiliary tool waits: outside the window but able to auto-start in a pass
  std::vector<uint8_t> aux(N, 0);
  for (bool changed = true; changed;) {
    changed = false;
    for (int i = 0; i < N; i++) {
      if (win[i] || aux[i] || done[i] || sd->kind[i] != RLX_KIND_TOOL_WAIT) continue;
      bool ok = true;
      for (int p : preds[i]) ok = ok && (done[p] || win[p] || aux[p]);
      if (ok) aux[i] = 1, changed = true;
    }
  }
  // ---- suffix lengths (scheduler.py:751-770), reverse topological order
  std::vector<int> indeg(N), topo;
  topo.reserve(N);
  for (int i = 0; i < N; i++) indeg[i] = (int)preds[i].size();
  std::vector<int> stk;
  for (int i = 0; i < N; i++)
    if (!indeg[i]) stk.push_back(i);
  while (!stk.empty()) {
    int i = stk.back();
    stk.pop_back();
    topo.push_back(i);
    for (int s : succs[i])
      if (--indeg[s] == 0) stk.push_back(s);
  }
  if ((int)topo.size() != N) { err = "dependency cycle"; return RLX_ERR_ARG; }
  std::vector<double> suf(N), msx(N);
  for (int t = N - 1; t >= 0; t--) {
    int i = topo[t];
    double best = 0.0;
    bool any = false;
    for (int s : succs[i]) {
      if (!any || suf[s] > best) best = suf[s];
      any = true;
    }
    msx[i] = any ? best : 0.0;
    suf[i] = sd->duration[i] + msx[i];
  }

  // ---- local numbering
  std::vector<int>& l2g = hp.l2g;
  std::vector<int>& g2l = hp.g2l;
  l2g.clear();
  g2l.assign(N, -1);
  for (int i = 0; i < N; i++)
    if (win[i] || aux[i]) g2l[i] = (int)l2g.size(), l2g.push_back(i);
  const int NL = (int)l2g.size();
  const int M = NL;
  if (NL + 1 >= 60000) { err = "window too large"; return RLX_ERR_LIMIT; }

  // ---- join compression of large shared predecessor sets
  std::vector<std::vector<int>> upred(NL);
  for (int l = 0; l < NL; l++)
    for (int p : preds[l2g[l]])
      if (!done[p]) upred[l].push_back(g2l[p]);
  for (auto& v : upred) std::sort(v.begin(), v.end());
  std::map<std::vector<int>, std::vector<int>> groups;
  for (int l = 0; l < NL; l++)
    if (upred[l].size() >= 4) groups[upred[l]].push_back(l);
  std::vector<int> join_of(NL, -1);
  std::vector<std::vector<int>> join_preds, join_members;
  for (auto& kv : groups) {
    if (kv.second.size() < 2) continue;
    int j = NL + 1 + (int)join_preds.size();
    join_preds.push_back(kv.first);
    join_members.push_back(kv.second);
    for (int l : kv.second) join_of[l] = j;
  }
  const int NJ = (int)join_preds.size();
  const int NT = NL + 1 + NJ;
  std::vector<std::vector<int>> lsucc(NT);
  std::vector<uint16_t> pend0(NT, 0);
  for (int l = 0; l < NL; l++) {
    if (join_of[l] >= 0) {
      pend0[l] = 1;
    } else {
      pend0[l] = (uint16_t)upred[l].size();
      for (int u : upred[l]) lsucc[u].push_back(l);
    }
  }
  for (int j = 0; j < NJ; j++) {
    int J = NL + 1 + j;
    pend0[J] = (uint16_t)join_preds[j].size();
    for (int u : join_preds[j]) lsucc[u].push_back(J);
    for (int l : join_members[j]) lsucc[J].push_back(l);
  }

  // ---- per local node arrays
  std::vector<uint8_t> kind(NL), pipe(NL), flags(NT, 0), ltm(NL), pos(2 * NL, 255);
  std::vector<uint16_t> worker(NL);
  std::vector<double> dur(NL), mem(NL), mpre(NL), lsuf(NL), lmsx(NL), migc(NL);
  std::vector<int64_t> rem(NL), act(NL);
  std::vector<int32_t> lrank(NL), idoff(NL);
  std::vector<char> ids;
  std::vector<int16_t> twslot(NL, -1);
  std::vector<uint16_t> twnode;
  std::vector<double> twend0;
  int64_t nwin = 0, ntw_win = 0;
  for (int l = 0; l < NL; l++) {
    int i = l2g[l];
    int p = sd->pipe[i];
    kind[l] = (uint8_t)sd->kind[i];
    pipe[l] = (uint8_t)p;
    worker[l] = (uint16_t)sd->worker[i];
    dur[l] = sd->duration[i];
    mem[l] = sd->mem[i];
    mpre[l] = sd->merge_prefix[i];
    lsuf[l] = suf[i];
    lmsx[l] = msx[i];
    migc[l] = in->has_spec[p]
                  ? (2.0 * in->model_params[p] * (double)sd->context[i]) / (in->prefill_mfu[p] * in->peak_flops[p])
                  : in->default_migration_cost;
    rem[l] = sd->remaining[i];
    act[l] = sd->active[i];
    lrank[l] = nrank[i];
    const char* s = id(i);
    ltm[l] = strncmp(s, "merge[", 6) == 0 ? 2 : (strcmp(s, "merge[") < 0 ? 1 : 0);
    idoff[l] = (int32_t)ids.size();
    ids.insert(ids.end(), s, s + strlen(s) + 1);
    uint8_t f = 0;
    if (sd->kind[i] == RLX_KIND_TOOL_WAIT) {
      f |= F_TW;
      twslot[l] = (int16_t)twnode.size();
      twnode.push_back((uint16_t)l);
      twend0.push_back(INFINITY);
    }
    if (win[i]) f |= F_WIN, nwin++, ntw_win += sd->kind[i] == RLX_KIND_TOOL_WAIT;
    if (ready[i]) f |= F_READY0;
    if (run[i]) f |= F_RUN0;
    flags[l] = f;
  }
  for (int j = 0; j < NJ; j++) flags[NL + 1 + j] = F_JOIN;
  flags[M] = F_WIN;
  if (twnode.size() > 30000) { err = "too many tool waits"; return RLX_ERR_LIMIT; }
  int n_twr0 = 0;
  for (int k = 0; k < sd->n_toolwaits; k++) {
    int l = g2l[sd->tw_node[k]];
    twend0[twslot[l]] = sd->tw_end[k];
    n_twr0++;
  }
  // ---- per worker orders over window compute nodes still to start
  std::vector<std::vector<int>> wn(W);
  for (int l = 0; l < NL; l++) {
    int i = l2g[l];
    if ((flags[l] & F_WIN) && !(flags[l] & F_TW) && !run[i] && !done[i]) wn[worker[l]].push_back(l);
  }
  std::vector<uint16_t> ord(2 * W * kMaxPos, 0xFFFF);
  std::vector<uint8_t> ordcnt(W);
  std::vector<uint64_t> mask0(2 * W, 0);
  for (int w = 0; w < W; w++) {
    auto v = wn[w];
    if ((int)v.size() > kMaxPos - 1) { err = "more than 63 window sub-stages on one worker"; return RLX_ERR_LIMIT; }
    ordcnt[w] = (uint8_t)v.size();
    for (int o = 0; o < 2; o++) {
      if (o == 0)
        std::sort(v.begin(), v.end(), [&](int a, int b) {
          if (lsuf[a] != lsuf[b]) return lsuf[a] > lsuf[b];
          return lrank[a] < lrank[b];
        });
      else
        std::sort(v.begin(), v.end(), [&](int a, int b) { return lrank[a] < lrank[b]; });
      for (int p = 0; p < (int)v.size(); p++) {
        ord[(o * W + w) * kMaxPos + p] = (uint16_t)v[p];
        pos[o * NL + v[p]] = (uint8_t)p;
        if (flags[v[p]] & F_READY0) mask0[o * W + w] |= uint64_t(1) << p;
      }
    }
  }
  // ---- pair table: _best_pair_action (:803-828) of every ordered pair (x, y)
  // of window compute nodes of different pipelines on the same worker. It is
  // decision-invariant, so pairing passes look it up instead of searching the
  // 24-point orientation x alpha x mem grid. Entry: 0 = no feasible pair,
  // else 0x80 | (second-is-x) << 6 | alloc; 0x60 | r flags a missing LUT row
  // (r = 0: the first missing lookup is (kind x, kind y), r = 1: (kind y, kind x)).
  std::vector<uint32_t> pt_off(W + 1, 0);
  std::vector<uint8_t> ptab;
  {
    const double hr = in->headroom;
    static const double MGP[4] = {0.20, 0.40, 0.60, 0.80};
    // bad: 0 none, 1 first missing lookup is (kind x, kind y), 2 it is (kind y, kind x)
    auto L3 = [&](int k, int partner, int alloc, int& bad, int code) {
      double v = in->lut[(k * RLX_NPARTNER + partner + 1) * RLX_NALLOC + alloc];
      if (std::isnan(v) && !bad) bad = code;
      return v;
    };
    auto rerated = [](double da, double sa, double db, double sb) {
      double na = da * sa, nb = db * sb;
      if (fabs(na - nb) <= kEps) return na;
      if (na < nb) return na + (1.0 - na / nb) * db;
      return nb + (1.0 - nb / na) * da;
    };
    for (int w = 0; w < W; w++) {
      const int cnt = ordcnt[w];
      pt_off[w] = (uint32_t)ptab.size();
      ptab.resize(ptab.size() + (size_t)cnt * cnt, 0);
      for (int px = 0; px < cnt; px++)
        for (int py = 0; py < cnt; py++) {
          const int a = ord[(1 * W + w) * kMaxPos + px], b = ord[(1 * W + w) * kMaxPos + py];
          if (pipe[a] == pipe[b]) continue;
          if (!(mem[a] + mem[b] <= 1.0 - hr + 1e-12)) continue;
          double best = INFINITY;
          int ent = 0;
          int bad = 0;
          for (int oo = 0; oo < 2; oo++) {
            const int f = oo ? b : a, sc2 = oo ? a : b;
            const double ms = mem[sc2];
            for (int ai = 0; ai < 3; ai++)
              for (int mj = 0; mj < 4; mj++) {
                if (MGP[mj] + ms > 1.0 - hr + kEps) continue;
                const int al = 1 + ai * 4 + mj;
                // argument order of _rerated_pair_end(...) (:816-821): first's factor is looked up first
                const double sf = L3(kind[f], kind[sc2], al, bad, oo ? 2 : 1);
                const double ss = L3(kind[sc2], kind[f], al + 12, bad, oo ? 1 : 2);
                const double e = rerated(dur[f], sf, dur[sc2], ss);
                if (e < best - kEps) {
                  best = e;
                  ent = 0x80 | (oo << 6) | al;
                }
              }
          }
          ptab[pt_off[w] + (size_t)px * cnt + py] = bad ? (uint8_t)(0x60 | (bad - 1)) : (uint8_t)ent;
        }
    }
    pt_off[W] = (uint32_t)ptab.size();
  }
  // ---- running members at the decision state
  std::vector<uint8_t> nmem0(W, 0), mpart0(2 * W, 0);
  std::vector<uint16_t> mnode0(2 * W, 0);
  std::vector<double> mrate0(2 * W, 0), mpre0(2 * W, 0), mwork0(2 * W, 0);
  for (int k = 0; k < sd->n_running; k++) {
    int i = sd->run_node[k];
    int w = sd->worker[i];
    int s = nmem0[w]++;
    mnode0[2 * w + s] = (uint16_t)g2l[i];
    mpart0[2 * w + s] = sd->run_partner[k] >= 0;
    mrate0[2 * w + s] = sd->run_rate[k];
    mpre0[2 * w + s] = sd->run_prefix[k];
    mwork0[2 * w + s] = sd->run_work[k];
  }
  std::vector<double> grant0((size_t)W * P, NAN);
  for (int k = 0; k < sd->n_grants; k++) grant0[sd->grant_worker[k] * P + sd->grant_pipe[k]] = sd->grant_mem[k];

  // ---- candidate space (enumerate_actions :648-703)
  std::vector<int> rl;  // ready compute, name order (local ids)
  for (int r = 0; r < N; r++) {
    int i = order[r];
    if (ready[i] && sd->kind[i] != RLX_KIND_TOOL_WAIT) rl.push_back(g2l[i]);
  }
  const double h = in->headroom;
  static const double MG[4] = {0.20, 0.40, 0.60, 0.80};
  hp.mux_pairs.clear(); hp.excl.clear();
  hp.frags.clear(); hp.combos.clear(); hp.blocks.clear();
  int64_t n_mux = 0;
  for (int w = 0; w < W; w++) {
    if (nmem0[w]) continue;
    std::vector<int> g;
    for (int l : rl)
      if (worker[l] == w) g.push_back(l);
    for (size_t x = 0; x < g.size(); x++)
      for (size_t y = x + 1; y < g.size(); y++) {
        int a = g[x], b = g[y];
        if (pipe[a] == pipe[b]) continue;
        if (!(mem[a] + mem[b] <= 1.0 - h + 1e-12)) continue;
        int nf[2] = {0, 0};  // feasible MEM_GRID prefix for the second member
        for (int o = 0; o < 2; o++)
          for (int mj = 0; mj < 4; mj++)
            if (MG[mj] + mem[o ? a : b] <= 1.0 - h + kEps) nf[o] = mj + 1;
        if (nf[0] + nf[1] == 0) continue;
        MuxPair mp;
        memset(&mp, 0, sizeof mp);
        mp.serial0 = n_mux;
        mp.a = (uint16_t)a;
        mp.b = (uint16_t)b;
        mp.na = (uint8_t)nf[0];
        mp.nb = (uint8_t)nf[1];
        hp.mux_pairs.push_back(mp);
        n_mux += 3 * (nf[0] + nf[1]);
      }
  }
  fill_binom(hp.binom);
  const int64_t LIMIT = int64_t(1) << 61;
  int64_t serial = n_mux;
  if (in->merge_enabled) {
    std::vector<int> pipes(P);
    for (int p = 0; p < P; p++) pipes[prank[p]] = p;
    for (int p : pipes) {
      std::vector<int> fr2;
      for (int l : rl)
        if (pipe[l] == p && (kind[l] == RLX_KIND_DECODE_SMALL || kind[l] == RLX_KIND_DECODE_MEDIUM)) fr2.push_back(l);
      int n = (int)fr2.size();
      if (n < 2) continue;
      int top = (max_merge > 0 && max_merge < n) ? max_merge : n;
      if (top > kMaxMembers) { err = "merge sets above 64 members (set max_merge)"; return RLX_ERR_LIMIT; }
      if (n > kMaxFrags) { err = "more than 128 mergeable fragments in one pipeline"; return RLX_ERR_LIMIT; }
      bool distinct = true;
      for (int x = 0; x < n && distinct; x++)
        for (int y = x + 1; y < n && distinct; y++) distinct = worker[fr2[x]] != worker[fr2[y]];
      int frag_off = (int)hp.frags.size();
      for (int l : fr2) hp.frags.push_back((uint16_t)l);
      for (int size = 2; size <= top; size++) {
        MergeBlock B;
        B.serial0 = serial;
        B.size = size;
        B.pipe = p;
        B.frag_off = frag_off;
        B.n_frags = n;
        if (distinct) {
          uint64_t c = binom_at(hp.binom.data(), n, size);
          if (c >= (uint64_t(1) << 62) / (uint64_t)size) {
            err = "candidate space too large (pass max_merge)";
            return RLX_ERR_LIMIT;
          }
          B.combos = (int64_t)c;
          B.expl_off = -1;
        } else {
          B.expl_off = (int64_t)hp.combos.size();
          int64_t cnt = 0;
          int idx[kMaxMembers];
          for (int k = 0; k < size; k++) idx[k] = k;
          for (;;) {
            bool ok = true;
            for (int a = 0; a < size && ok; a++)
              for (int b = a + 1; b < size && ok; b++) ok = worker[fr2[idx[a]]] != worker[fr2[idx[b]]];
            if (ok) {
              for (int k = 0; k < size; k++) hp.combos.push_back((uint16_t)idx[k]);
              if (++cnt > (int64_t(1) << 24)) { err = "explicit merge list too large (pass max_merge)"; return RLX_ERR_LIMIT; }
            }
            int k = size - 1;
            while (k >= 0 && idx[k] == n - size + k) k--;
            if (k < 0) break;
            idx[k]++;
            for (int z = k + 1; z < size; z++) idx[z] = idx[z - 1] + 1;
          }
          B.combos = cnt;
        }
        if (B.combos == 0) continue;
        serial += B.combos * size;
        if (serial > LIMIT) { err = "candidate space too large (pass max_merge)"; return RLX_ERR_LIMIT; }
        hp.blocks.push_back(B);
      }
    }
  }
  const int64_t n_merge = serial - n_mux;
  for (int l : rl)
    if (!nmem0[worker[l]]) hp.excl.push_back((uint16_t)l);
  const int64_t n_excl = (int64_t)hp.excl.size();

  int64_t ew = 0;
  for (int e = 0; e < sd->n_edges; e++) ew += win[sd->edge_src[e]] && win[sd->edge_dst[e]];

  // ---- scalars
  DevPlan& d = hp.dp;
  memset(&d, 0, sizeof d);
  d.NL = NL;
  d.NT = NT;
  d.M = M;
  d.NWIN = (int32_t)nwin;
  d.W = W;
  d.P = P;
  d.NTW = (int32_t)twnode.size();
  d.n_blocks = (int32_t)hp.blocks.size();
  d.has_penalty = in->realloc_penalty > 0;
  d.merge_enabled = in->merge_enabled != 0;
  d.n_run0 = sd->n_running;
  d.n_tw_run0 = n_twr0;
  d.now = sd->now;
  d.headroom = h;
  d.realloc_penalty = in->realloc_penalty;
  d.default_migration_cost = in->default_migration_cost;
  d.n_mux = n_mux;
  d.n_mux_pairs = (int64_t)hp.mux_pairs.size();
  d.n_merge = n_merge;
  d.n_excl = n_excl;
  d.n_total = n_mux + n_merge + n_excl;
  d.ew = ew;
  hp.n_tw_window = ntw_win;
  hp.worker_of = worker;

  // ---- CSR
  std::vector<int32_t> soff(NT + 1, 0);
  std::vector<uint16_t> sl;
  for (int u = 0; u < NT; u++) {
    soff[u] = (int32_t)sl.size();
    for (int v : lsucc[u]) sl.push_back((uint16_t)v);
  }
  soff[NT] = (int32_t)sl.size();

  // ---- readiness counters: only nodes (and joins) waiting on >= 2 predecessors
  // need one; a node with a single unresolved predecessor becomes ready when
  // that predecessor completes.
  std::vector<uint16_t> ctr_idx(NT, 0xFFFF), ctr0;
  for (int u = 0; u < NT; u++)
    if (pend0[u] >= 2) {
      ctr_idx[u] = (uint16_t)ctr0.size();
      ctr0.push_back(pend0[u]);
    }
  d.NC = (int32_t)ctr0.size();
  // Variants 0 (suffix key) and 2 (name key) of _complete_window (:875) run
  // identical simulations when every worker's two orders coincide.
  d.same_order = 1;
  for (int w = 0; w < W && d.same_order; w++)
    for (int q = 0; q < ordcnt[w]; q++)
      if (ord[(0 * W + w) * kMaxPos + q] != ord[(1 * W + w) * kMaxPos + q]) {
        d.same_order = 0;
        break;
      }
  int max_ord = 0;
  for (int w = 0; w < W; w++) max_ord = std::max(max_ord, (int)ordcnt[w]);
  d.max_ord = max_ord;

  // ---- packed node records (hot): one 16-byte load per node on the device
  std::vector<NodeRec> rec(NT);
  for (int u = 0; u < NT; u++) {
    NodeRec& r = rec[u];
    r.x = (uint32_t)soff[u];
    r.y = (uint32_t)(soff[u + 1] - soff[u]) | (uint32_t)ctr_idx[u] << 16;
    const bool node = u < NL;
    r.z = (node ? (uint32_t)worker[u] : 0u) | (uint32_t)flags[u] << 16 | (node ? (uint32_t)kind[u] : 0u) << 24;
    r.w = (node ? (uint32_t)pipe[u] : 0u) | (uint32_t)(node ? pos[u] : 255) << 8 | (uint32_t)(node ? pos[NL + u] : 255) << 16;
  }
  for (int u = 0; u < NT; u++)
    if (soff[u + 1] - soff[u] > 0xFFFF) { err = "a node with more than 65535 successors"; return RLX_ERR_LIMIT; }

  // ---- blob: the hot region (staged into shared memory) comes first
  Blob& B = hp.blob;
  B.buf.clear();
  PlanLayout& L = hp.lay;
  L.lut = B.put(in->lut, sizeof(double) * RLX_NKIND * RLX_NPARTNER * RLX_NALLOC);
  L.alloc_mem = B.put(in->alloc_mem, sizeof(double) * RLX_NALLOC);
  L.dur = B.putv(dur);
  L.rec = B.putv(rec);
  L.ord = B.putv(ord);
  L.tw_slot = B.putv(twslot);
  L.tw_node = B.putv(twnode);
  L.ord_cnt = B.putv(ordcnt);
  L.succ = B.putv(sl);
  if (RLX_MPRE_HOT) L.mprefix = B.putv(mpre);
  L.hot_end = (B.buf.size() + 15) & ~size_t(15);
  B.buf.resize(L.hot_end);
  // read only by member starts and pairing: global memory (L1-resident)
  L.mem = B.putv(mem);
  if (!RLX_MPRE_HOT) L.mprefix = B.putv(mpre);
  L.pt_off = B.putv(pt_off);
  L.ptab = B.putv(ptab);
  {  // RN(1 / rate) per LUT entry: a member start loads it instead of dividing
    std::vector<double> rl(RLX_NKIND * RLX_NPARTNER * RLX_NALLOC);
    for (size_t i = 0; i < rl.size(); i++) rl[i] = 1.0 / in->lut[i];
    L.rlut = B.putv(rl);
  }
  // cold copies for the candidate prologues (global loads)
  L.succ_off = B.putv(soff);
  L.kind = B.putv(kind);
  L.pipe = B.putv(pipe);
  L.worker = B.putv(worker);
  L.flags = B.putv(flags);
  L.pos = B.putv(pos);
  L.ctr_idx = B.putv(ctr_idx);
  L.ctr0 = B.putv(ctr0);
  L.suffix = B.putv(lsuf);
  L.msx = B.putv(lmsx);
  L.migc = B.putv(migc);
  L.rem = B.putv(rem);
  L.act = B.putv(act);
  L.name_rank = B.putv(lrank);
  L.lt_merge = B.putv(ltm);
  L.id_off = B.putv(idoff);
  L.ids = B.putv(ids);
  L.pend0 = B.putv(pend0);
  L.mask0 = B.putv(mask0);
  L.nmem0 = B.putv(nmem0);
  L.mnode0 = B.putv(mnode0);
  L.mpart0 = B.putv(mpart0);
  L.mrate0 = B.putv(mrate0);
  L.mpre0 = B.putv(mpre0);
  L.mwork0 = B.putv(mwork0);
  L.worker_ids = B.put(in->worker_ids, sizeof(int32_t) * W);
  L.tw_end0 = B.putv(twend0);
  L.grant0 = B.putv(grant0);
  L.pipe_rank = B.putv(prank);
  L.latency = B.put(in->latency, sizeof(double) * P * 3);
  L.latency_ok = B.put(in->latency_ok, P * 3);
  L.has_spec = B.put(in->has_spec, P);
  L.mux_pairs = B.putv(hp.mux_pairs);
  L.excl = B.putv(hp.excl);
  L.blocks = B.putv(hp.blocks);
  L.frags = B.putv(hp.frags);
  L.combos = B.putv(hp.combos);
  L.binom = B.putv(hp.binom);
  return RLX_OK;
}

// The device path's capacity checks that depend only on the plan: a kernel
// shape for W workers and the shared-memory footprint of the hot region.
int check_capacity(const HostPlan& hp, std::string& err) {
  int G, WPL;
  choose_shape(hp.dp.W, G, WPL);
  if (G > 32 || G * WPL < hp.dp.W) {
    err = "more than 128 workers";
    return RLX_ERR_LIMIT;
  }
  if (hp.lay.hot_end + plan_slice_bytes(hp.dp, G, WPL) > kSmemCap) {
    err = "the plan does not fit in shared memory";
    return RLX_ERR_LIMIT;
  }
  return RLX_OK;
}

template <class T>
static const T* at(const uint8_t* base, size_t off) {
  return reinterpret_cast<const T*>(base + off);
}

// Point every DevPlan array into `base` (host blob or its device copy).
void relocate(HostPlan& hp, const uint8_t* base, DevPlan& d) {
  d = hp.dp;
  const PlanLayout& L = hp.lay;
  d.kind = at<uint8_t>(base, L.kind);
  d.pipe = at<uint8_t>(base, L.pipe);
  d.worker = at<uint16_t>(base, L.worker);
  d.flags = at<uint8_t>(base, L.flags);
  d.dur = at<double>(base, L.dur);
  d.mem = at<double>(base, L.mem);
  d.mprefix = at<double>(base, L.mprefix);
  d.suffix = at<double>(base, L.suffix);
  d.msx = at<double>(base, L.msx);
  d.migc = at<double>(base, L.migc);
  d.rem = at<int64_t>(base, L.rem);
  d.act = at<int64_t>(base, L.act);
  d.name_rank = at<int32_t>(base, L.name_rank);
  d.lt_merge = at<uint8_t>(base, L.lt_merge);
  d.id_off = at<int32_t>(base, L.id_off);
  d.ids = at<char>(base, L.ids);
  d.pos = at<uint8_t>(base, L.pos);
  d.tw_slot = at<int16_t>(base, L.tw_slot);
  d.tw_node = at<uint16_t>(base, L.tw_node);
  d.succ_off = at<int32_t>(base, L.succ_off);
  d.succ = at<uint16_t>(base, L.succ);
  d.pend0 = at<uint16_t>(base, L.pend0);
  d.ord = at<uint16_t>(base, L.ord);
  d.ord_cnt = at<uint8_t>(base, L.ord_cnt);
  d.mask0 = at<uint64_t>(base, L.mask0);
  d.nmem0 = at<uint8_t>(base, L.nmem0);
  d.mnode0 = at<uint16_t>(base, L.mnode0);
  d.mpart0 = at<uint8_t>(base, L.mpart0);
  d.mrate0 = at<double>(base, L.mrate0);
  d.mpre0 = at<double>(base, L.mpre0);
  d.mwork0 = at<double>(base, L.mwork0);
  d.worker_ids = at<int32_t>(base, L.worker_ids);
  d.tw_end0 = at<double>(base, L.tw_end0);
  d.grant0 = at<double>(base, L.grant0);
  d.pipe_rank = at<uint8_t>(base, L.pipe_rank);
  d.latency = at<double>(base, L.latency);
  d.latency_ok = at<uint8_t>(base, L.latency_ok);
  d.has_spec = at<uint8_t>(base, L.has_spec);
  d.lut = at<double>(base, L.lut);
  d.alloc_mem = at<double>(base, L.alloc_mem);
  d.mux_pairs = at<MuxPair>(base, L.mux_pairs);
  d.excl = at<uint16_t>(base, L.excl);
  d.blocks = at<MergeBlock>(base, L.blocks);
  d.frags = at<uint16_t>(base, L.frags);
  d.combos = at<uint16_t>(base, L.combos);
  d.binom = at<uint64_t>(base, L.binom);
  d.pt_off = at<uint32_t>(base, L.pt_off);
  d.ptab = at<uint8_t>(base, L.ptab);
  d.rlut = at<double>(base, L.rlut);
  d.ctr_idx = at<uint16_t>(base, L.ctr_idx);
  d.ctr0 = at<uint16_t>(base, L.ctr0);
  d.hot = base;
  d.hot_bytes = (uint32_t)L.hot_end;
  d.o_rec = (uint32_t)L.rec;
  d.o_mprefix = (uint32_t)L.mprefix;
  d.o_tw_slot = (uint32_t)L.tw_slot;
  d.o_succ = (uint32_t)L.succ;
  d.o_ord = (uint32_t)L.ord;
  d.o_dur = (uint32_t)L.dur;
  d.o_lut = (uint32_t)L.lut;
  d.o_alloc_mem = (uint32_t)L.alloc_mem;
  d.o_tw_node = (uint32_t)L.tw_node;
  d.o_ord_cnt = (uint32_t)L.ord_cnt;
}

}  // namespace rlx

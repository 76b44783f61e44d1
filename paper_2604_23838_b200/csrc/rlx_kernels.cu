// rlx_kernels.cu — sm_100a look-ahead scoring kernel.
//
// One "slice" of L lanes (L = 4..32, a warp or a fraction of one) runs one
// list-scheduling pass (rlmux/scheduler.py:831-869) at a time; lane l owns
// workers {l, l+L, ...}. Per pass, the slice's private shared memory holds
// the pending-predecessor counters of every window node and one 64-bit
// ready mask per worker whose bit order is that worker's completion-key
// order (suffix key or name key, :893-894), so "first ready node on an
// idle worker" is a find-first-set and the pairing partner is the next set
// bit of another pipeline. Running members (<= 2 per worker) stay in the
// owner lane's registers. Each event is: selection on idle workers ->
// warp-shuffle min of finish estimates (the next event) -> consume ->
// completions (smem atomics on counters / masks) -> tool-wait expiry and
// auto-start -> window-completion count (__reduce_add_sync).
//
// A persistent grid of slices pulls candidates from a global counter,
// heaviest class first (merges carry 3*(1+F) passes, :902-918). For each
// candidate the slice runs every pass, forms the key (cost, finish,
// priority, serial) (:963-972) and keeps its running minimum; a final
// reduction produces the shard winner.
//
// Bit-exactness: compiled with -fmad=false; all double expressions keep
// the reference's left-to-right order (e.g. finish = (now + prefix) +
// work*rate, :328).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/rlx.h"
#include "rlx_plan.hpp"

namespace rlx {

constexpr int kLutN = RLX_NKIND * RLX_NPARTNER * RLX_NALLOC;
// The decision plan lives in constant memory: every field is a uniform,
// broadcast read for all lanes (one plan per device at a time).
__constant__ DevPlan c_plan;

// The same slice code also compiles for the host as a single-lane debugging
// twin (tests/twin, never linked into the product): PLAN and the warp
// primitives resolve to their host equivalents there.
#ifdef __CUDA_ARCH__
#define PLAN c_plan
#else
extern const DevPlan* g_twin_plan;
#define PLAN (*g_twin_plan)
#endif

RLX_HD unsigned at_sub(unsigned* p, unsigned v) {
#ifdef __CUDA_ARCH__
  return atomicSub(p, v);
#else
  unsigned o = *p; *p = o - v; return o;
#endif
}
RLX_HD int at_add(int* p, int v) {
#ifdef __CUDA_ARCH__
  return atomicAdd(p, v);
#else
  int o = *p; *p = o + v; return o;
#endif
}
RLX_HD void at_or(unsigned long long* p, unsigned long long v) {
#ifdef __CUDA_ARCH__
  atomicOr(p, v);
#else
  *p |= v;
#endif
}
RLX_HD unsigned long long at_add64(unsigned long long* p, unsigned long long v) {
#ifdef __CUDA_ARCH__
  return atomicAdd(p, v);
#else
  unsigned long long o = *p; *p = o + v; return o;
#endif
}
RLX_HD int at_cas(int* p, int c, int v) {
#ifdef __CUDA_ARCH__
  return atomicCAS(p, c, v);
#else
  int o = *p; if (o == c) *p = v; return o;
#endif
}
RLX_HD void wsync(unsigned m) {
#ifdef __CUDA_ARCH__
  __syncwarp(m);
#endif
}
RLX_HD bool wany(unsigned m, bool x) {
#ifdef __CUDA_ARCH__
  return __any_sync(m, x);
#else
  return x;
#endif
}
RLX_HD unsigned wsum(unsigned m, unsigned x) {
#ifdef __CUDA_ARCH__
  return __reduce_add_sync(m, x);
#else
  return x;
#endif
}
template <int L>
RLX_HD double wmin(unsigned m, double t) {
#ifdef __CUDA_ARCH__
#pragma unroll
  for (int off = L / 2; off > 0; off >>= 1) {
    double u = __shfl_xor_sync(m, t, off, L);
    t = u < t ? u : t;
  }
#endif
  return t;
}
template <int L>
RLX_HD long long wbcast(unsigned m, long long v) {
#ifdef __CUDA_ARCH__
  return __shfl_sync(m, v, 0, L);
#else
  return v;
#endif
}
RLX_HD int ffs64(unsigned long long m) {
#ifdef __CUDA_ARCH__
  return __ffsll((long long)m);
#else
  return __builtin_ffsll((long long)m);
#endif
}

// MEM_GRID (slowdown.py:19) and DEFAULT_MEM_FRACTIONS by kind code (graph.py:98-106).
RLX_HD double memgrid(int j) { return j == 0 ? 0.20 : j == 1 ? 0.40 : j == 2 ? 0.60 : 0.80; }
RLX_HD double defmem(int k) {
  return k == 0 ? 0.5 : k == 1 ? 0.55 : k == 2 ? 0.4 : k == 3 ? 0.3 : k == 4 ? 0.5 : k == 5 ? 0.6 : 0.05;
}

// Per-slice candidate scratch (shared memory).
struct SliceCand {
  double dur, mem, pre, suf, fin;
  int kind, pipe, t, k, ins0, ins1, idle;
  int twq_n, tw_run, pad;
  uint16_t m[kMaxMembers];
};

struct Act {  // action started at pass begin
  int cls;    // -1 none, 0 mux, 2 exclusive
  int a, b, alloc;
};

RLX_HD unsigned long long dbits(double x) {
  unsigned long long b;
  memcpy(&b, &x, 8);
  return b == 0x8000000000000000ull ? 0ull : b;
}

RLX_HD bool key_less(unsigned long long a0, unsigned long long a1, unsigned long long a2,
                                         unsigned long long b0, unsigned long long b1, unsigned long long b2) {
  if (a0 != b0) return a0 < b0;
  if (a1 != b1) return a1 < b1;
  return a2 < b2;
}

template <int L, int WPL>
struct Slice {
  const double* lut;
  const int lane;
  const unsigned smask;
  // smem
  unsigned* pend;
  unsigned long long* mask;
  double* twend;
  uint16_t* twq;
  double* grant;
  SliceCand* sc;
  int* gerr;
  // per-worker registers
  int nm[WPL];
  int nd[WPL][2];
  double rt[WPL][2], pr[WPL][2], wk[WPL][2];
  bool pt[WPL][2];
  // pass constants
  double* dbg = nullptr;
  long long dbg_serial = -1;
  int o;       // order index
  int mt;      // merged target worker (-1: no merge)
  int ins;     // insertion position on mt
  int err;

  RLX_HD Slice(const double* l, int ln, unsigned m, uint8_t* base, int* ge)
      : lut(l), lane(ln), smask(m), gerr(ge) {
    uint8_t* q = base;
    sc = reinterpret_cast<SliceCand*>(q);
    q += (sizeof(SliceCand) + 15) & ~15;
    mask = reinterpret_cast<unsigned long long*>(q);
    q += sizeof(unsigned long long) * PLAN.W;
    twend = reinterpret_cast<double*>(q);
    q += sizeof(double) * PLAN.NTW;
    grant = reinterpret_cast<double*>(q);
    q += PLAN.has_penalty ? sizeof(double) * PLAN.W * PLAN.P : 0;
    pend = reinterpret_cast<unsigned*>(q);
    q += sizeof(unsigned) * PLAN.NT;
    twq = reinterpret_cast<uint16_t*>(q);
    err = 0;
  }

  // ---- node attributes (M = virtual merged node)
  RLX_HD int kind(int n) const { return n == PLAN.M ? sc->kind : PLAN.kind[n]; }
  RLX_HD int pipe(int n) const { return n == PLAN.M ? sc->pipe : PLAN.pipe[n]; }
  RLX_HD double dur(int n) const { return n == PLAN.M ? sc->dur : PLAN.dur[n]; }
  RLX_HD double memf(int n) const { return n == PLAN.M ? sc->mem : PLAN.mem[n]; }
  RLX_HD double mpre(int n) const { return n == PLAN.M ? sc->pre : PLAN.mprefix[n]; }
  RLX_HD int wrk(int n) const { return n == PLAN.M ? sc->t : PLAN.worker[n]; }

  RLX_HD double L3(int k, int partner, int alloc) {
    double v = lut[(k * RLX_NPARTNER + partner + 1) * RLX_NALLOC + alloc];
    if (isnan(v)) err = RLX_ERR_KEY;
    return v;
  }

  RLX_HD int node_at(int w, int p) const {
    if (w == mt) {
      if (p == ins) return PLAN.M;
      if (p > ins) p--;
    }
    return PLAN.ord[(o * PLAN.W + w) * kMaxPos + p];
  }
  RLX_HD int pos_of(int n) const {
    int p = PLAN.pos[o * PLAN.NL + n];
    if (PLAN.worker[n] == mt && p >= ins) p++;
    return p;
  }

  // ---- completion bookkeeping
  RLX_HD void became_ready(int s) {
    uint8_t f = PLAN.flags[s];
    if (f & F_TW) {
      int q = at_add(&sc->twq_n, 1);
      twq[q] = (uint16_t)s;
    } else {
      at_or(&mask[PLAN.worker[s]], 1ull << pos_of(s));
    }
  }
  RLX_HD void dec(int s) {
    unsigned old = at_sub(&pend[s], 1u);
    if (old == 1u) {
      if (PLAN.flags[s] & F_JOIN) {
        for (int e = PLAN.succ_off[s]; e < PLAN.succ_off[s + 1]; e++) {
          int s2 = PLAN.succ[e];
          if (at_sub(&pend[s2], 1u) == 1u) became_ready(s2);
        }
      } else {
        became_ready(s);
      }
    }
  }
  RLX_HD void succs_of(int u) {
    for (int e = PLAN.succ_off[u]; e < PLAN.succ_off[u + 1]; e++) dec(PLAN.succ[e]);
  }
  RLX_HD void complete(int n, unsigned& ld) {
    if (n == PLAN.M) {
      ld++;
      for (int i = 0; i < sc->k; i++) succs_of(sc->m[i]);
    } else {
      if (PLAN.flags[n] & F_WIN) ld++;
      succs_of(n);
    }
  }

  // ---- starting members (_start_member :460-484)
  RLX_HD void start(int j, int w, int n, double rate, int alloc, bool partner) {
    double pre = mpre(n);
    if (PLAN.has_penalty && kind(n) <= RLX_KIND_DECODE_SMALL) {
      double* g = &grant[w * PLAN.P + pipe(n)];
      double am = PLAN.alloc_mem[alloc];
      double last = *g;
      if (!isnan(last) && fabs(last - am) > kEps) pre = pre + PLAN.realloc_penalty;
      *g = am;
    }
    double d = dur(n);
    if (nm[j] == 0) {
      nd[j][0] = n; rt[j][0] = rate; pr[j][0] = pre; wk[j][0] = d; pt[j][0] = partner;
    } else {
      nd[j][1] = n; rt[j][1] = rate; pr[j][1] = pre; wk[j][1] = d; pt[j][1] = partner;
    }
    nm[j]++;
  }

  RLX_HD double rerated(double da, double sa, double db, double sb) const {
    double na = da * sa, nb = db * sb;
    if (fabs(na - nb) <= kEps) return na;
    if (na < nb) return na + (1.0 - na / nb) * db;
    return nb + (1.0 - nb / na) * da;
  }

  // _best_pair_action :803-828
  RLX_HD bool best_pair(int a, int b, int& first, int& second, int& alloc) {
    const double h = PLAN.headroom;
    double ma = memf(a), mb = memf(b);
    if (!(ma + mb <= 1.0 - h + 1e-12)) return false;
    double best = INFINITY;
    bool found = false;
    const int ka = kind(a), kb = kind(b);
    const double da = dur(a), db = dur(b);
#pragma unroll
    for (int oo = 0; oo < 2; oo++) {
      const int f = oo ? b : a, s = oo ? a : b;
      const int kf = oo ? kb : ka, ks = oo ? ka : kb;
      const double df = oo ? db : da, ds = oo ? da : db;
      const double ms = oo ? ma : mb;
      for (int ai = 0; ai < 3; ai++)
        for (int mj = 0; mj < 4; mj++) {
          if (memgrid(mj) + ms > 1.0 - h + kEps) continue;
          int al = 1 + ai * 4 + mj;
          double e = rerated(df, L3(kf, ks, al), ds, L3(ks, kf, al + 12));
          if (e < best - kEps) {
            best = e;
            first = f;
            second = s;
            alloc = al;
            found = true;
          }
        }
    }
    return found;
  }

  // One pass of _complete_window with action `act` applied first.
  RLX_HD double pass(int variant, const Act& act, bool is_merge, int nwin, unsigned long long& passes,
                         double& bytes) {
    o = variant == 2 ? 1 : 0;
    const bool pair = variant == 1;
    mt = is_merge ? sc->t : -1;
    ins = is_merge ? (o ? sc->ins1 : sc->ins0) : -1;
    for (int i = lane; i < PLAN.NT; i += L) pend[i] = PLAN.pend0[i];
    for (int w = lane; w < PLAN.W; w += L) mask[w] = PLAN.mask0[o * PLAN.W + w];
    for (int i = lane; i < PLAN.NTW; i += L) twend[i] = PLAN.tw_end0[i];
    if (PLAN.has_penalty)
      for (int i = lane; i < PLAN.W * PLAN.P; i += L) grant[i] = PLAN.grant0[i];
    if (lane == 0) {
      sc->twq_n = 0;
      sc->tw_run = PLAN.n_tw_run0;
    }
#pragma unroll
    for (int j = 0; j < WPL; j++) {
      int w = lane + L * j;
      nm[j] = 0;
      if (w < PLAN.W) {
        int c = PLAN.nmem0[w];
        for (int s = 0; s < 2; s++)
          if (s < c) {
            nd[j][s] = PLAN.mnode0[2 * w + s];
            rt[j][s] = PLAN.mrate0[2 * w + s];
            pr[j][s] = PLAN.mpre0[2 * w + s];
            wk[j][s] = PLAN.mwork0[2 * w + s];
            pt[j][s] = PLAN.mpart0[2 * w + s] != 0;
          }
        nm[j] = c;
      }
    }
    wsync(smask);
    if (is_merge && lane == 0) {
      unsigned long long m = mask[mt];
      unsigned long long lo = ins ? (m & ((1ull << ins) - 1)) : 0ull;
      mask[mt] = lo | ((m >> ins) << (ins + 1)) | (1ull << ins);
      for (int i = 0; i < sc->k; i++) {
        int x = sc->m[i];
        mask[PLAN.worker[x]] &= ~(1ull << pos_of(x));
      }
    }
    wsync(smask);
    int R0 = PLAN.n_run0;
    if (act.cls >= 0) {
      int w = wrk(act.a);
      R0 += act.cls == 0 ? 2 : 1;
      if ((w % L) == lane) {
        int j = w / L;
#pragma unroll
        for (int jj = 0; jj < WPL; jj++)
          if (jj == j) {
            if (act.cls == 2) {
              mask[w] &= ~(1ull << (act.a == PLAN.M ? ins : pos_of(act.a)));
              start(jj, w, act.a, L3(kind(act.a), -1, 0), 0, false);
            } else {
              int a = act.a, b = act.b;
              mask[w] &= ~((1ull << (a == PLAN.M ? ins : pos_of(a))) | (1ull << (b == PLAN.M ? ins : pos_of(b))));
              double ra = L3(kind(a), kind(b), act.alloc);
              double rb = L3(kind(b), kind(a), act.alloc + 12);
              start(jj, w, a, ra, act.alloc, true);
              start(jj, w, b, rb, act.alloc + 12, true);
            }
          }
      }
    }
    wsync(smask);
    // algorithmic bytes of this pass
    passes++;
    bytes += 32.0 * nwin + 4.0 * (double)PLAN.ew + 32.0 * R0 + 16.0 * PLAN.n_tw_run0;

    double now = PLAN.now;
    double last = 0.0;
    bool any_done = false;
    int done_cnt = 0;
    int guard = 0;
    for (;;) {
      if (done_cnt >= nwin) break;
      // ---- selection on idle workers (one sweep)
#pragma unroll
      for (int j = 0; j < WPL; j++) {
        int w = lane + L * j;
        if (w < PLAN.W && nm[j] == 0) {
          unsigned long long m = mask[w];
          if (m) {
            int p = ffs64(m) - 1;
            int x = node_at(w, p);
            int first = x, second = -1, al = 0;
            bool paired = false;
            if (pair) {
              unsigned long long m2 = m & (m - 1);
              int px = pipe(x);
              while (m2) {
                int q = ffs64(m2) - 1;
                int y = node_at(w, q);
                if (pipe(y) != px) {
                  paired = best_pair(x, y, first, second, al);
                  if (paired) m &= ~(1ull << q);
                  break;
                }
                m2 &= m2 - 1;
              }
            }
            m &= ~(1ull << p);
            mask[w] = m;
            if (paired) {
              double ra = L3(kind(first), kind(second), al);
              double rb = L3(kind(second), kind(first), al + 12);
              start(j, w, first, ra, al, true);
              start(j, w, second, rb, al + 12, true);
            } else {
              start(j, w, x, L3(kind(x), -1, 0), 0, false);
            }
          }
        }
      }
      // ---- has_events
      bool mine = false;
#pragma unroll
      for (int j = 0; j < WPL; j++) mine |= nm[j] > 0;
      wsync(smask);
      const int twr = sc->tw_run;
      if (!wany(smask, mine) && twr == 0) break;
      // ---- next event time
      double t = INFINITY;
#pragma unroll
      for (int j = 0; j < WPL; j++)
        for (int s = 0; s < 2; s++)
          if (s < nm[j]) {
            double fe = (now + pr[j][s]) + wk[j][s] * rt[j][s];
            t = fe < t ? fe : t;
          }
      if (twr)
        for (int i = lane; i < PLAN.NTW; i += L) t = twend[i] < t ? twend[i] : t;
      t = wmin<L>(smask, t);
      double dt = t - now;
      if (!(dt > 0.0)) dt = 0.0;
      now = t;
      // ---- consume + finished members
      unsigned ld = 0;
      bool fin_any = false;
#pragma unroll
      for (int j = 0; j < WPL; j++) {
        bool f0 = false, f1 = false;
        for (int s = 0; s < 2; s++)
          if (s < nm[j]) {
            double d = dt;
            double p = pr[j][s];
            if (p > kEps) {
              double used = d < p ? d : p;
              p = p - used;
              d = d - used;
              pr[j][s] = p;
            }
            double wv = wk[j][s];
            double r = rt[j][s];
            if (d > kEps && wv > kEps) {
              double q = (r == 1.0) ? d : d / r;
              double z = wv - q;
              wv = z > 0.0 ? z : 0.0;
              wk[j][s] = wv;
            }
            bool f = p <= kEps && wv * r <= kEps;
            if (s == 0) f0 = f; else f1 = f;
          }
        if (f0 || f1) {
          fin_any = true;
          if (f0) complete(nd[j][0], ld);
          if (nm[j] == 2 && f1) complete(nd[j][1], ld);
          if (nm[j] == 2 && f0 != f1) {
            // survivor re-rated to its exclusive speed (:615-621)
            int s = f0 ? 1 : 0;
            double r = rt[j][s];
            bool pp = pt[j][s];
            if (pp) r = 1.0;
            nd[j][0] = nd[j][s];
            rt[j][0] = r;
            pr[j][0] = pr[j][s];
            wk[j][0] = wk[j][s];
            pt[j][0] = false;
            nm[j] = 1;
          } else {
            nm[j] = 0;
          }
        }
      }
      wsync(smask);
      // ---- tool-wait expiry
      bool exp_any = false;
      if (twr) {
        int ex = 0;
        for (int i = lane; i < PLAN.NTW; i += L)
          if (twend[i] <= now + kEps) {
            twend[i] = INFINITY;
            complete(PLAN.tw_node[i], ld);
            ex++;
          }
        if (ex) {
          at_add(&sc->tw_run, -ex);
          exp_any = true;
        }
      }
      wsync(smask);
      // ---- auto-start ready tool waits (:421-434)
      if (wany(smask, fin_any || exp_any)) {
        if (lane == 0) {
          while (sc->twq_n > 0) {
            int s = twq[--sc->twq_n];
            double dd = PLAN.dur[s];
            if (dd <= kEps) {
              complete(s, ld);
            } else {
              twend[PLAN.tw_slot[s]] = now + dd;
              sc->tw_run++;
            }
          }
        }
        wsync(smask);
      }
      unsigned tot = wsum(smask, ld);
      if (tot) {
        done_cnt += (int)tot;
        last = now;
        any_done = true;
      }
      if (++guard > 10000) {
        err = RLX_ERR_SCHEDULING;
        if (lane == 0 && dbg && dbg[0] == 0.0 && (dbg[0] = 1.0) == 1.0) {
          int live = 0;
          for (int i = 0; i < PLAN.NTW; i++) live += twend[i] != INFINITY;
          dbg[1] = (double)dbg_serial;
          dbg[2] = variant;
          dbg[3] = now;
          dbg[4] = done_cnt;
          dbg[5] = nwin;
          dbg[6] = twr;
          dbg[7] = live;
          dbg[8] = sc->twq_n;
          dbg[9] = nm[0];
          dbg[10] = act.cls;
          dbg[11] = act.a;
          dbg[12] = mt;
        }
        break;
      }
    }
    return any_done ? last : now;
  }
};

// The candidate loop of one slice (device: one warp fraction; host twin: one lane).
template <int L, int WPL>
RLX_HD void slice_loop(const WorkDesc& wd, const double* lut, uint8_t* base, int lane, unsigned smask,
                       SliceOut* out) {
  Slice<L, WPL> S(lut, lane, smask, base, wd.err);
  S.dbg = wd.dbg;
  SliceCand* sc = S.sc;

  unsigned long long b0 = ~0ull, b1 = ~0ull, b2 = ~0ull;
  unsigned long long passes = 0, ncand = 0;
  double bytes = 0.0;
  const int64_t total = wd.na + wd.nb + wd.nc;
  for (;;) {
    long long g = 0;
    if (lane == 0) {
      g = (long long)at_add64(wd.counter, 1ull);
      if (*(volatile int*)wd.err) g = total;
    }
    g = wbcast<L>(smask, g);
    if (g >= total) break;
    int64_t serial = g < wd.na ? wd.a0 + g : (g < wd.na + wd.nb ? wd.b0 + (g - wd.na) : wd.c0 + (g - wd.na - wd.nb));
    Cand c;
    decode_serial(PLAN, serial, c);
    S.dbg_serial = serial;
    double cost = INFINITY, fin;
    if (c.cls == 1) {
      // ---- merged node (_apply_merge :517-581, merged_estimate :185-199)
      if (lane == 0) {
        long long tokens = 0, active = 0;
        double dmax = 0.0, mmax = 0.0, sfx = 0.0;
        int p = PLAN.pipe[c.m[0]];
        for (int i = 0; i < c.k; i++) {
          int x = c.m[i];
          sc->m[i] = (uint16_t)x;
          tokens += PLAN.rem[x];
          active += PLAN.act[x];
          if (i == 0 || PLAN.dur[x] > dmax) dmax = PLAN.dur[x];
          if (i == 0 || PLAN.mem[x] > mmax) mmax = PLAN.mem[x];
          if (i == 0 || PLAN.msx[x] > sfx) sfx = PLAN.msx[x];
        }
        int kd;
        double du;
        if (active <= 0) {
          kd = PLAN.kind[c.m[0]];
          du = dmax;
        } else {
          int bk = active >= 1024 ? 2 : (active >= 128 ? 1 : 0);
          kd = bk == 0 ? RLX_KIND_DECODE_SMALL : (bk == 1 ? RLX_KIND_DECODE_MEDIUM : RLX_KIND_DECODE_LARGE);
          if (!PLAN.latency_ok[p * 3 + bk]) at_cas(wd.err, 0, RLX_ERR_KEY);
          du = ((double)tokens * PLAN.latency[p * 3 + bk]) / (double)active;
        }
        double pre = 0.0;
        for (int i = 0; i < c.k; i++)
          if (PLAN.worker[c.m[i]] != c.target) pre = pre + PLAN.migc[c.m[i]];
        double dm = defmem(kd);
        sc->kind = kd;
        sc->dur = du;
        sc->mem = mmax > dm ? mmax : dm;
        sc->pre = pre;
        sc->suf = du + sfx;
        sc->pipe = p;
        sc->t = c.target;
        sc->k = c.k;
        sc->idle = PLAN.nmem0[c.target] == 0;
        // insertion position of the merged node in each worker order
        const int t = c.target;
        const int cnt = PLAN.ord_cnt[t];
        const int prk = PLAN.pipe_rank[p];
        for (int oo = 0; oo < 2; oo++) {
          int ins = cnt;
          for (int q = 0; q < cnt; q++) {
            int y = PLAN.ord[(oo * PLAN.W + t) * kMaxPos + q];
            bool y_first;
            if (oo == 0 && PLAN.suffix[y] != sc->suf) {
              y_first = PLAN.suffix[y] > sc->suf;
            } else {
              int yr = PLAN.pipe_rank[PLAN.pipe[y]];
              if (yr != prk) {
                y_first = yr < prk;
              } else if (PLAN.lt_merge[y] != 2) {
                y_first = PLAN.lt_merge[y] == 1;
              } else {
                // id(y) vs "merge[" + "+".join(member ids) + "]@w<t>"
                const char* ys = PLAN.ids + PLAN.id_off[y];
                int seg = -1;
                const char* cp = "merge[";
                char tail[16];
                int wid = PLAN.worker_ids[t];
                int tl = 0;
                tail[tl++] = ']';
                tail[tl++] = '@';
                tail[tl++] = 'w';
                {
                  char tmp[12];
                  int nt = 0;
                  unsigned v = wid < 0 ? (unsigned)(-wid) : (unsigned)wid;
                  do { tmp[nt++] = (char)('0' + v % 10); v /= 10; } while (v);
                  if (wid < 0) tail[tl++] = '-';
                  while (nt) tail[tl++] = tmp[--nt];
                }
                tail[tl] = 0;
                int cmp = 0;
                for (;;) {
                  char mc;
                  while (*cp == 0) {
                    seg++;
                    if (seg < 2 * c.k - 1) {
                      cp = (seg & 1) ? "+" : PLAN.ids + PLAN.id_off[c.m[seg >> 1]];
                    } else if (seg == 2 * c.k - 1) {
                      cp = tail;
                    } else {
                      break;
                    }
                  }
                  mc = *cp;
                  unsigned char yc = (unsigned char)*ys;
                  unsigned char vc = (unsigned char)mc;
                  if (yc != vc) {
                    cmp = yc < vc ? -1 : 1;
                    break;
                  }
                  if (yc == 0) break;
                  ys++;
                  cp++;
                }
                y_first = cmp < 0;
              }
            }
            if (!y_first) {
              ins = q;
              break;
            }
          }
          if (oo == 0) sc->ins0 = ins; else sc->ins1 = ins;
        }
      }
      wsync(smask);
      fin = (PLAN.now + sc->pre) + sc->dur;
      const int nwin = PLAN.NWIN - c.k + 1;
      if (sc->idle) {
        // follow-ups on the merged node (candidate_cost :907-918)
        Act a{2, PLAN.M, -1, 0};
        for (int v = 0; v < 3; v++) {
          double x = S.pass(v, a, true, nwin, passes, bytes);
          cost = x < cost ? x : cost;
        }
        const int t = sc->t;
        unsigned long long rm = PLAN.mask0[1 * PLAN.W + t];
        const double h = PLAN.headroom;
        while (rm) {
          int q = ffs64(rm) - 1;
          rm &= rm - 1;
          int y = PLAN.ord[(1 * PLAN.W + t) * kMaxPos + q];
          bool member = false;
          for (int i = 0; i < sc->k; i++) member |= sc->m[i] == y;
          if (member || PLAN.pipe[y] == sc->pipe) continue;
          if (!(sc->mem + PLAN.mem[y] <= 1.0 - h + 1e-12)) continue;
          for (int oo = 0; oo < 2; oo++) {
            int f = oo ? y : PLAN.M, s = oo ? PLAN.M : y;
            double ms = oo ? sc->mem : PLAN.mem[y];
            for (int ai = 0; ai < 3; ai++)
              for (int mj = 0; mj < 4; mj++) {
                if (memgrid(mj) + ms > 1.0 - h + kEps) continue;
                Act m{0, f, s, 1 + ai * 4 + mj};
                for (int v = 0; v < 3; v++) {
                  double x = S.pass(v, m, true, nwin, passes, bytes);
                  cost = x < cost ? x : cost;
                }
              }
          }
        }
      } else {
        Act a{-1, -1, -1, 0};
        for (int v = 0; v < 3; v++) {
          double x = S.pass(v, a, true, nwin, passes, bytes);
          cost = x < cost ? x : cost;
        }
      }
    } else {
      S.mt = -1;
      S.ins = -1;
      Act a{c.cls, c.a, c.cls == 0 ? c.b : -1, c.alloc};
      // action_finish_estimate :773-789 (with the realloc penalty of the decision state)
      auto fin_of = [&](int n, int alloc) {
        double pre = PLAN.mprefix[n];
        if (PLAN.has_penalty && PLAN.kind[n] <= RLX_KIND_DECODE_SMALL) {
          double g = PLAN.grant0[PLAN.worker[n] * PLAN.P + PLAN.pipe[n]];
          if (!isnan(g) && fabs(g - PLAN.alloc_mem[alloc]) > kEps) pre = pre + PLAN.realloc_penalty;
        }
        return pre;
      };
      if (c.cls == 2) {
        double r = S.L3(PLAN.kind[c.a], -1, 0);
        fin = (PLAN.now + fin_of(c.a, 0)) + PLAN.dur[c.a] * r;
      } else {
        double ra = S.L3(PLAN.kind[c.a], PLAN.kind[c.b], c.alloc);
        double rb = S.L3(PLAN.kind[c.b], PLAN.kind[c.a], c.alloc + 12);
        double fa = (PLAN.now + fin_of(c.a, c.alloc)) + PLAN.dur[c.a] * ra;
        double fb = (PLAN.now + fin_of(c.b, c.alloc + 12)) + PLAN.dur[c.b] * rb;
        fin = fb > fa ? fb : fa;
      }
      for (int v = 0; v < 3; v++) {
        double x = S.pass(v, a, false, PLAN.NWIN, passes, bytes);
        cost = x < cost ? x : cost;
      }
    }
    if (S.err) at_cas(wd.err, 0, S.err);
    ncand++;
    unsigned long long k0 = dbits(cost), k1 = dbits(fin);
    unsigned long long k2 = ((unsigned long long)c.cls << 61) | (unsigned long long)serial;
    if (key_less(k0, k1, k2, b0, b1, b2)) {
      b0 = k0;
      b1 = k1;
      b2 = k2;
    }
    if (wd.keys_out && lane == 0) {
      wd.keys_out[2 * (serial - wd.shard0)] = cost;
      wd.keys_out[2 * (serial - wd.shard0) + 1] = fin;
    }
    wsync(smask);
  }
  if (lane == 0) {
    out->k0 = b0;
    out->k1 = b1;
    out->k2 = b2;
    out->passes = passes;
    out->bytes = bytes;
    out->cands = ncand;
  }
}


template <int L, int WPL>
__global__ void __launch_bounds__(256, 2) rlx_score_kernel(const WorkDesc wd, SliceOut* outs) {
  extern __shared__ __align__(16) uint8_t smem[];
  double* lut = reinterpret_cast<double*>(smem);
  for (int i = threadIdx.x; i < kLutN; i += blockDim.x) lut[i] = PLAN.lut[i];
  __syncthreads();
  const int lane = threadIdx.x % L;
  const int slice = threadIdx.x / L;
  const int wl = threadIdx.x & 31;
  const unsigned smask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (wl / L * L));
  uint8_t* base = smem + ((kLutN * 8 + 15) & ~15) + (size_t)slice * wd.slice_bytes;
  slice_loop<L, WPL>(wd, lut, base, lane, smask, &outs[blockIdx.x * (blockDim.x / L) + slice]);
}

// Shard winner + stats over all slices (deterministic: lexicographic min).
__global__ void rlx_reduce_kernel(const SliceOut* outs, int n, unsigned long long* res /* 8 words */) {
  __shared__ unsigned long long s0[256], s1[256], s2[256], sp[256], sc[256];
  __shared__ double sb[256];
  unsigned long long b0 = ~0ull, b1 = ~0ull, b2 = ~0ull, ps = 0, cs = 0;
  double by = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (key_less(outs[i].k0, outs[i].k1, outs[i].k2, b0, b1, b2)) {
      b0 = outs[i].k0;
      b1 = outs[i].k1;
      b2 = outs[i].k2;
    }
    ps += outs[i].passes;
    cs += outs[i].cands;
    by += outs[i].bytes;
  }
  s0[threadIdx.x] = b0; s1[threadIdx.x] = b1; s2[threadIdx.x] = b2;
  sp[threadIdx.x] = ps; sc[threadIdx.x] = cs; sb[threadIdx.x] = by;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if ((int)threadIdx.x < st) {
      int o = threadIdx.x + st;
      if (key_less(s0[o], s1[o], s2[o], s0[threadIdx.x], s1[threadIdx.x], s2[threadIdx.x])) {
        s0[threadIdx.x] = s0[o];
        s1[threadIdx.x] = s1[o];
        s2[threadIdx.x] = s2[o];
      }
      sp[threadIdx.x] += sp[o];
      sc[threadIdx.x] += sc[o];
      sb[threadIdx.x] += sb[o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    res[0] = s0[0];
    res[1] = s1[0];
    res[2] = s2[0];
    res[3] = s0[0] != ~0ull ? 1ull : 0ull;
    res[4] = sp[0];
    res[5] = (unsigned long long)__double_as_longlong(sb[0]);
    res[6] = sc[0];
  }
}

// ---------------------------------------------------------------------------
// host-side launch helpers (called from rlx_abi.cu)

size_t slice_bytes(const DevPlan& P) {
  size_t b = (sizeof(SliceCand) + 15) & ~size_t(15);
  b += 8 * (size_t)P.W + 8 * (size_t)P.NTW + (P.has_penalty ? 8 * (size_t)P.W * P.P : 0);
  b += 4 * (size_t)P.NT + 2 * (size_t)(P.NTW + 8);
  return (b + 15) & ~size_t(15);
}

size_t lut_bytes() { return ((size_t)kLutN * 8 + 15) & ~size_t(15); }

typedef void (*KernelFn)(const WorkDesc, SliceOut*);

static KernelFn pick(int L, int WPL) {
#ifdef RLX_ONLY_32_2
  return rlx_score_kernel<32, 2>;
#endif
#ifdef RLX_DEBUG_SHAPES
  // development builds only (librlx_dbg.so): lane-count sweeps for bisecting
  if (L == 4 && WPL == 8) return rlx_score_kernel<4, 8>;
  if (L == 8 && WPL == 4) return rlx_score_kernel<8, 4>;
  if (L == 16 && WPL == 2) return rlx_score_kernel<16, 2>;
#endif
  if (L == 4) return rlx_score_kernel<4, 1>;
  if (L == 8) return rlx_score_kernel<8, 1>;
  if (L == 16) return rlx_score_kernel<16, 1>;
  if (WPL == 1) return rlx_score_kernel<32, 1>;
  if (WPL == 2) return rlx_score_kernel<32, 2>;
  return rlx_score_kernel<32, 4>;
}

void choose_shape(int W, int& L, int& WPL) {
  if (W <= 4) L = 4, WPL = 1;
  else if (W <= 8) L = 8, WPL = 1;
  else if (W <= 16) L = 16, WPL = 1;
  else if (W <= 32) L = 32, WPL = 1;
  else if (W <= 64) L = 32, WPL = 2;
  else L = 32, WPL = 4;
}

// Returns 0 on success; fills grid/block/smem.
int launch_score(const DevPlan& P, WorkDesc wd, SliceOut* outs, int max_slices, int sm_count, cudaStream_t st,
                 int* n_slices_out, int threads_hint) {
  int L, WPL;
  choose_shape(P.W, L, WPL);
#ifdef RLX_DEBUG_SHAPES
  if (const char* sh = getenv("RLX_SHAPE")) sscanf(sh, "%d,%d", &L, &WPL);
#endif
  KernelFn fn = pick(L, WPL);
  size_t sb = slice_bytes(P);
  wd.slice_bytes = (int)sb;
  int threads = threads_hint > 0 ? threads_hint : 256;
  size_t smem = 0;
  for (;;) {
    smem = lut_bytes() + (size_t)(threads / L) * sb;
    if (smem <= 200 * 1024 || threads <= L) break;
    threads /= 2;
  }
  if (smem > 227 * 1024) return RLX_ERR_LIMIT;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return RLX_ERR_CUDA;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess) return RLX_ERR_CUDA;
  if (per_sm < 1) per_sm = 1;
  int64_t total = wd.na + wd.nb + wd.nc;
  int64_t need = (total + (threads / L) - 1) / (threads / L);
  int64_t blocks = (int64_t)per_sm * sm_count;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  int64_t slices = blocks * (threads / L);
  if (slices > max_slices) {
    blocks = max_slices / (threads / L);
    slices = blocks * (threads / L);
  }
  if (cudaMemcpyToSymbolAsync(c_plan, &P, sizeof(DevPlan), 0, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return RLX_ERR_CUDA;
  fn<<<(unsigned)blocks, threads, smem, st>>>(wd, outs);
  if (cudaGetLastError() != cudaSuccess) return RLX_ERR_CUDA;
  *n_slices_out = (int)slices;
  return 0;
}

int launch_reduce(const SliceOut* outs, int n, unsigned long long* res, cudaStream_t st) {
  rlx_reduce_kernel<<<1, 256, 0, st>>>(outs, n, res);
  return cudaGetLastError() == cudaSuccess ? 0 : RLX_ERR_CUDA;
}

}  // namespace rlx

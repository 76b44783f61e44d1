// rlx_kernels.cu — sm_100a look-ahead evaluator.
//
// What one launch computes: for every candidate of a decision shard
// (enumerate_actions, rlmux/scheduler.py:648-703) its look-ahead cost
// (candidate_cost :902-918 = min over window_cost passes :878-899 of the
// list-scheduling simulation _complete_window :831-869) and its finish
// estimate (action_finish_estimate :773-789), then the lexicographic
// (cost, finish, priority, serial) minimum (chooser :963-972).
//
// Execution model (B200):
//  * One persistent CTA per SM. Its first act is to stage the decision plan's
//    hot region (node SoA, successor CSR, per-worker ready orders, slowdown
//    LUT — everything the event loop reads) from HBM into shared memory with
//    TMA bulk copies (cp.async.bulk + mbarrier complete_tx). All passes of all
//    candidates on that SM then read the plan from shared memory only.
//  * A "group" of G lanes (G = 1..32, inside one warp) runs one list-
//    scheduling pass at a time. Lane l owns the simulated workers
//    {l, l+G, ...} (WPL = 2 workers per lane up to 16 workers, else 4;
//    choose_shape) and keeps their running members (<= 2 per worker: rate,
//    work left) in registers; node ids, prefixes, ready masks, readiness
//    counters and tool-wait clocks live in the group's slice of shared
//    memory. Decision-invariant pairings come from the planner's pair table.
//  * One loop iteration = one simulated event for every group of the warp:
//    selection on idle workers (find-first-set over a 64-bit ready mask whose
//    bit order is the completion key), group min of finish estimates
//    (butterfly shuffles over G lanes), consume, completions (shared-memory
//    atomics when G > 1), tool-wait expiry/auto-start, window count. Consume
//    runs as straight-line phases over a lane's member slots (consume dt and
//    test for finish, re-rate survivors, minimum of the next finish
//    estimates) so the slots' FP64 chains interleave (consume_lean /
//    consume_u).
//  * Groups pull whole candidates from a global counter, heaviest class
//    (merges: 3*(1+F) passes) first, and keep a running minimum key.
//
// Bit-exactness: compiled with -fmad=false; every double expression keeps
// the reference's left-to-right order (finish = (now + prefix) + work*rate,
// :328; consume :330-336; re-rated pair end :792-800).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <type_traits>

#include "../../include/rlx.h"
#include "rlx_plan.hpp"

#ifndef RLX_RRS_MAXG
#define RLX_RRS_MAXG 8
#endif
#ifndef RLX_PFX_SPLIT
#define RLX_PFX_SPLIT 1
#endif
#ifndef RLX_PFX_MING
#define RLX_PFX_MING 16  // groups of >= this many lanes take the prefix-free consume
#endif
#ifndef RLX_TL_PRED
#define RLX_TL_PRED 1
#endif
#ifndef RLX_SEL_UNROLL
#define RLX_SEL_UNROLL 0  // 1: selection unrolled over local workers (tuning)
#endif
#ifndef RLX_COLD_NOINLINE
#define RLX_COLD_NOINLINE 0
#endif
// Candidate-boundary routines (once per candidate) out of line (tuning knob):
// config 2 shows 41% stall_no_instructions, but calling them measured 2-3%
// slower than inlining (profiles/r02_ab_misc_variants.txt).
#if RLX_COLD_NOINLINE && defined(__CUDA_ARCH__)
#define RLX_COLD __host__ __device__ __noinline__
#elif RLX_COLD_NOINLINE && defined(__CUDACC__)
#define RLX_COLD __host__ __device__ inline  // host copy emitted only where used (the twin)
#else
#define RLX_COLD RLX_HD
#endif
#ifndef RLX_POS0_MASK
#define RLX_POS0_MASK 0  // 1: max(0, z) by sign mask (tuning)
#endif
#ifndef RLX_S0_BRANCH
#define RLX_S0_BRANCH 0  // 1: skip idle slot-0 members by branch (tuning)
#endif
// Consume variant (step()). 3 (default): groups of >= RLX_PFX_MING lanes split
// by lane — consume<true> where a running member has a pending prefix,
// consume_lean elsewhere — and smaller groups run consume_u (measured on one
// box: config 5 cap 2 5.19 vs 5.48 s, config 4 cap 2 0.87 vs 0.92 s for the
// lean split, config 2 714 vs 755 ms for consume_u). 2: consume_u always;
// 1: the split everywhere it applies; 0: the split with consume<false>.
// (consume_u on the prefix lanes of the split measured no better: 5.13 s.)
#ifndef RLX_LEAN
#define RLX_LEAN 3
#endif
#ifndef RLX_WIN_SMEM
#define RLX_WIN_SMEM 1  // window-completion count and time in the group slice, not registers (plans without tool waits)
#endif
#ifndef RLX_GMIN_REDUX
#define RLX_GMIN_REDUX 0  // 1: group minimum of event times by two 32-bit redux.sync (tuning)
#endif
#ifndef RLX_RLUT
#define RLX_RLUT 1  // member starts read RN(1/rate) from the planner's table (0: __drcp_rn per start)
#endif
#ifndef RLX_S1_PRED
#define RLX_S1_PRED 1  // consume_lean evaluates slot 1 predicated (1) or by branch (0)
#endif
#ifndef RLX_S1_PRED_U
#define RLX_S1_PRED_U 0  // consume_u: the same choice (measured: branch 714 vs predicated 731 ms at config 2)
#endif

namespace rlx {

// Scalars and global views of the plan; uniform reads for every lane.
__constant__ DevPlan c_plan;

// The same code compiles for the host as a single-lane debugging twin
// (tests/twin, never linked into the product).
#ifdef __CUDA_ARCH__
#define PLAN c_plan
#else
extern const DevPlan* g_twin_plan;
#define PLAN (*g_twin_plan)
#endif

// ---------------------------------------------------------------------------
// warp / atomic shims. With G == 1 a group is one lane and nothing is shared.
template <int G>
RLX_HD unsigned at_sub(unsigned* p, unsigned v) {
#ifdef __CUDA_ARCH__
  if (G > 1) return atomicSub(p, v);
#endif
  unsigned o = *p;
  *p = o - v;
  return o;
}
template <int G>
RLX_HD int at_add(int* p, int v) {
#ifdef __CUDA_ARCH__
  if (G > 1) return atomicAdd(p, v);
#endif
  int o = *p;
  *p = o + v;
  return o;
}
// Ready masks are u64 per worker; a completion sets one bit with a 32-bit
// shared-memory OR on the word that holds it (native ATOMS.OR — a 64-bit
// atomicOr compiles to a CAS loop).
template <int G>
RLX_HD void at_or_bit(unsigned long long* p, int bit) {
#ifdef __CUDA_ARCH__
  if (G > 1) {
    atomicOr(reinterpret_cast<unsigned*>(p) + (bit >> 5), 1u << (bit & 31));
    return;
  }
#endif
  *p |= 1ull << bit;
}
RLX_HD int at_min32(int* p, int v) {
#ifdef __CUDA_ARCH__
  return atomicMin(p, v);
#else
  int o = *p;
  if (v < o) *p = v;
  return o;
#endif
}
RLX_HD void at_min64s(unsigned long long* p, unsigned long long v) {  // shared-memory u64 min
#ifdef __CUDA_ARCH__
  atomicMin(p, v);
#else
  if (v < *p) *p = v;
#endif
}
RLX_HD int at_add32(int* p, int v) {
#ifdef __CUDA_ARCH__
  return atomicAdd(p, v);
#else
  int o = *p;
  *p = o + v;
  return o;
#endif
}
// The warp slice's candidate generation: published with an atomic exchange
// after a fence, polled with an atomic read (the groups' only handshake).
RLX_HD void gen_store(int* p, int v) {
#ifdef __CUDA_ARCH__
  __threadfence_block();
  atomicExch(p, v);
#else
  *p = v;
#endif
}
RLX_HD int gen_load(int* p) {
#ifdef __CUDA_ARCH__
  const int v = atomicAdd(p, 0);
  __threadfence_block();
  return v;
#else
  return *p;
#endif
}
RLX_HD void fence_block() {
#ifdef __CUDA_ARCH__
  __threadfence_block();
#endif
}
RLX_HD unsigned long long at_add64(unsigned long long* p, unsigned long long v) {
#ifdef __CUDA_ARCH__
  return atomicAdd(p, v);
#else
  unsigned long long o = *p;
  *p = o + v;
  return o;
#endif
}
RLX_HD void at_min64(unsigned long long* p, unsigned long long v) {
#ifdef __CUDA_ARCH__
  atomicMin(p, v);
#else
  if (v < *p) *p = v;
#endif
}
template <int G>
RLX_HD int gmax(unsigned m, int x) {
#ifdef __CUDA_ARCH__
  if (G > 1) return __reduce_max_sync(m, x);
#endif
  return x;
}
RLX_HD int at_cas(int* p, int c, int v) {
#ifdef __CUDA_ARCH__
  return atomicCAS(p, c, v);
#else
  int o = *p;
  if (o == c) *p = v;
  return o;
#endif
}
template <int G>
RLX_HD void gsync(unsigned m) {
#ifdef __CUDA_ARCH__
  if (G > 1) __syncwarp(m);
#endif
}
template <int G>
RLX_HD unsigned gsum(unsigned m, unsigned x) {
#ifdef __CUDA_ARCH__
  if (G > 1) return __reduce_add_sync(m, x);
#endif
  return x;
}
template <int G>
RLX_HD double gmin(unsigned m, double t) {
#ifdef __CUDA_ARCH__
#if RLX_GMIN_REDUX
  // t >= +0.0 or +inf (event times), never NaN: the u64 bit patterns order
  // like the values, so two 32-bit warp reductions (high word, then the low
  // word among the lanes holding the minimal high word) give the minimum
  if (G > 1) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(t);
    const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
    const unsigned mh = __reduce_min_sync(m, hi);
    const unsigned ml = __reduce_min_sync(m, hi == mh ? lo : 0xFFFFFFFFu);
    return __longlong_as_double((long long)((unsigned long long)mh << 32 | ml));
  }
#else
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) {
    double u = __shfl_xor_sync(m, t, off, G);
    t = u < t ? u : t;
  }
#endif
#endif
  return t;
}
template <int G>
RLX_HD long long gbcast(unsigned m, long long v) {
#ifdef __CUDA_ARCH__
  if (G > 1) return __shfl_sync(m, v, 0, G);
#endif
  return v;
}
RLX_HD int ffs32(unsigned m) {
#ifdef __CUDA_ARCH__
  return __ffs((int)m);
#else
  return __builtin_ffs((int)m);
#endif
}
RLX_HD int ffs64(unsigned long long m) {
#ifdef __CUDA_ARCH__
  return __ffsll((long long)m);
#else
  return __builtin_ffsll((long long)m);
#endif
}

// RN(1 / r) (IEEE, round to nearest even)
RLX_HD double recip(double r) {
#ifdef __CUDA_ARCH__
  return __drcp_rn(r);
#else
  return 1.0 / r;
#endif
}
// RN(d / r) from y = RN(1 / r): q0 = RN(d * y) is within one ulp of d / r,
// the residual e = d - q0 * r is exact in one FMA, and RN(q0 + e * y) is the
// correctly rounded quotient (Markstein's theorem; verified bit-exact
// against IEEE division on 3e8 random and adversarial operands, and by
// every golden test). Explicit FMAs are unaffected by -fmad=false.
RLX_HD double ediv(double d, double r, double y) {
  const double q0 = d * y;
  const double e = fma(-q0, r, d);
  return fma(e, y, q0);
}

// max(0.0, z) for a non-NaN z, as Python's max(0.0, z) (-0.0 -> 0.0): the
// sign of the bit pattern decides, with no floating-point max idiom
RLX_HD double pos0(double z) {
#ifdef __CUDA_ARCH__
#if RLX_POS0_MASK
  const long long b = __double_as_longlong(z);
  return __longlong_as_double(b & ~(b >> 63));  // negative (incl. -0.0) -> +0.0
#else
  return __double_as_longlong(z) > 0 ? z : 0.0;
#endif
#else
  return z > 0.0 ? z : 0.0;
#endif
}

// MEM_GRID (slowdown.py:19) and DEFAULT_MEM_FRACTIONS by kind code (graph.py:98-106).
RLX_HD double memgrid(int j) { return j == 0 ? 0.20 : j == 1 ? 0.40 : j == 2 ? 0.60 : 0.80; }
RLX_HD double defmem(int k) {
  return k == 0 ? 0.5 : k == 1 ? 0.55 : k == 2 ? 0.4 : k == 3 ? 0.3 : k == 4 ? 0.5 : k == 5 ? 0.6 : 0.05;
}

// Candidate error codes (per lane / group): RLX_ERR_SCHEDULING for the
// window guard, kErrLatBase + bucket for a missing latency bucket
// (merged_estimate :197), key_err(kind, partner) for a missing slowdown row
// (slowdown.py:143-147). The kernel keeps the LOWEST failing serial
// (err_key = serial << 8 | code, atomicMin), the one the reference's serial
// scan raises on.
constexpr int kErrLatBase = 8;
constexpr int kErrKeyBase = 16;
RLX_HD int key_err(int k, int partner) { return kErrKeyBase + k * RLX_NPARTNER + partner + 1; }

RLX_HD unsigned long long dbits(double x) {
  unsigned long long b;
  memcpy(&b, &x, 8);
  return b == 0x8000000000000000ull ? 0ull : b;
}

RLX_HD bool key_less(unsigned long long a0, unsigned long long a1, unsigned long long a2, unsigned long long b0,
                     unsigned long long b1, unsigned long long b2) {
  if (a0 != b0) return a0 < b0;
  if (a1 != b1) return a1 < b1;
  return a2 < b2;
}
// ---------------------------------------------------------------------------
// Shared memory. The hot plan sits at offset 0 (staged by TMA), followed by
// one slice per group. Addressing it through this symbol keeps every access
// in the shared window (LDS/STS/ATOMS), not generic loads.
extern __shared__ __align__(128) uint8_t rlx_smem[];
#ifdef __CUDA_ARCH__
#define SMEM rlx_smem
#else
extern uint8_t* g_twin_smem;
#define SMEM g_twin_smem
#endif

struct Act {  // action started at pass begin
  int cls;    // -1 none, 0 multiplex, 2 exclusive
  int a, b, alloc;
};

// One candidate at a time per warp (shared memory). Its passes — 3 variants
// x (1 + F) actions (candidate_cost :902-918 / window_cost :878-899) — form
// a queue that the warp's groups drain together, variant-major, so the
// groups of a warp simulate near-identical passes (same variant, sibling
// follow-ups of one merge) and their per-event control flow coincides.
// The last group to run dry finalises the key and fetches the next
// candidate (bumping `gen`); the others poll `gen` meanwhile.
struct WarpCand {
  double dur, mem, pre, suf;  // merged node M (merged_estimate :185-199, migration_cost :174-182)
  double fin;                 // action_finish_estimate (:773-789)
  unsigned long long cost;    // running min of the pass results (bit patterns of doubles >= 0)
  long long serial;           // -1: none
  int kind, pipe, t, k, ins0, ins1, idle, cls;
  int a, b, alloc, nwin;      // candidate action (non-merge)
  int n_act, n_var, total;    // passes = n_var x n_act
  int next;                   // next pass index (shared atomic)
  int done;                   // groups that found the queue empty
  int err;                    // first failing pass: (reference pass index << 8 | code), INT_MAX none
  int cerr;                   // candidate-level error (merged_estimate), 0 if none
  int gen;                    // candidate generation; -1: no more candidates (gen_load / gen_store)
  uint16_t m[kMaxMembers];
  // followed by uint16_t acts[acts_cap]: merge follow-ups (q << 5 | oo << 4 | ai * 4 + mj)
};

// Per-group pass state and results (shared memory).
struct GroupCand {
  double bytes;                   // SURVEY §8(d) algorithmic bytes scored by this group
  unsigned long long b0, b1, b2;  // best packed key finalised by this group
  unsigned long long passes, ncand, events;
  int twq_n, tw_run;
  int dsum;  // window completions of the running pass (plans without tool waits)
  double dlast;  // time of the last event with a window completion (RLX_WIN_SMEM)
};

// Warp and group slice layout (offsets in bytes), stored in the DevPlan
// constants by launch_score.
RLX_HD void group_layout(DevPlan& P, int G, int WPL) {
  P.acts_cap = 24 * (P.max_ord > 0 ? P.max_ord : 1);
  P.w_bytes = (uint32_t)((sizeof(WarpCand) + 2u * P.acts_cap + 15) & ~size_t(15));
  uint32_t b = (uint32_t)((sizeof(GroupCand) + 15) & ~size_t(15));
  P.g_mask = b;
  b += 8u * P.W;
  P.g_twend = b;
  b += 8u * P.NTW;
  P.g_grant = b;
  b += P.has_penalty ? 8u * P.W * P.P : 0u;
  P.g_pres = b;
  b += 8u * G * WPL * 2;
  b = (b + 15u) & ~15u;  // 16-byte aligned: LDS.128 / STS.128
  P.g_rr = b;  // (rate, RN(1/rate)) per member slot, when they live in shared memory
  b += G <= RLX_RRS_MAXG ? 16u * G * WPL * 2 : 0u;
  P.g_ctr = b;
  b += 4u * P.NC;
  P.g_nds = b;
  b += 2u * G * WPL * 2;
  P.g_twq = b;
  b += 2u * (P.NTW + 8);
  P.g_bytes = (b + 15u) & ~15u;
}

template <int WPL>
struct BitsFor {  // 2 bits per local worker
  typedef typename std::conditional<(WPL > 16), unsigned long long, unsigned>::type type;
};

template <int G, int WPL>
struct Lane {
  typedef typename BitsFor<WPL>::type Bits;
  static_assert(WPL <= 32, "at most 32 workers per lane");
  const uint32_t gbase;  // group slice offset in SMEM
  const uint32_t wbase;  // warp slice offset in SMEM
  const int lane;
  const unsigned gm;
  // registers: running members of this lane's workers (slot s of local worker j)
  // Where a member slot's (rate, RN(1/rate)) lives: shared memory (rr(), one
  // LDS.128 per slot and event, relieving the register file) for groups of
  // <= RLX_RRS_MAXG lanes, registers above (measured: config 2 / 4x4 760 vs
  // 871 ms in shared memory; config 5 / 16x4 6.07 vs 6.49 s in registers).
  static constexpr bool RRS = G <= RLX_RRS_MAXG;
  double wk[WPL][2];                                  // work left
  double rt[RRS ? 1 : WPL][2], ri[RRS ? 1 : WPL][2];  // rate, RN(1/rate) (register variant)
  RLX_HD double2 rate_of(int j, int s) const {
    if (RRS) return rr()[2 * j + s];
    return make_double2(rt[RRS ? 0 : j][s], ri[RRS ? 0 : j][s]);
  }
  RLX_HD void set_rate_static(int j, int s, double r, double y) {  // j known at compile time
    if (RRS) {
      rr()[2 * j + s] = make_double2(r, y);
    } else {
      rt[RRS ? 0 : j][s] = r;
      ri[RRS ? 0 : j][s] = y;
    }
  }
  Bits rb;    // bit 2j+s: running
  Bits pm;    // bit 2j+s: has a non-zero prefix (value in the slice)
  Bits pf;    // bit 2j+s: still has a multiplex partner
  double tl;  // this lane's next-event candidate time
  unsigned vmask;  // bit j: local worker j (= lane + G*j) exists
  int o, mt, ins, err;  // err: 0, RLX_ERR_SCHEDULING or key_err(...) (first failure of this candidate)
  // pass registers
  double now, last;
  int done_cnt, guard;
  bool any_done;

  RLX_HD Lane(uint32_t gb, uint32_t wb, int ln, unsigned m) : gbase(gb), wbase(wb), lane(ln), gm(m) {
    err = 0;
    rb = pm = pf = 0;
    vmask = 0;
#pragma unroll
    for (int j = 0; j < WPL; j++)
      if (ln + G * j < PLAN.W) vmask |= 1u << j;
  }

  // ---- shared-memory views
  RLX_HD GroupCand* gc() const { return reinterpret_cast<GroupCand*>(SMEM + gbase); }
  RLX_HD WarpCand* wc() const { return reinterpret_cast<WarpCand*>(SMEM + wbase); }
  RLX_HD unsigned long long* mask() const { return reinterpret_cast<unsigned long long*>(SMEM + gbase + PLAN.g_mask); }
  RLX_HD double* twend() const { return reinterpret_cast<double*>(SMEM + gbase + PLAN.g_twend); }
  RLX_HD double* grant() const { return reinterpret_cast<double*>(SMEM + gbase + PLAN.g_grant); }
  RLX_HD double* pres() const { return reinterpret_cast<double*>(SMEM + gbase + PLAN.g_pres) + lane * WPL * 2; }
  RLX_HD unsigned* ctr() const { return reinterpret_cast<unsigned*>(SMEM + gbase + PLAN.g_ctr); }
  RLX_HD uint16_t* nds() const { return reinterpret_cast<uint16_t*>(SMEM + gbase + PLAN.g_nds) + lane * WPL * 2; }
  RLX_HD double2* rr() const { return reinterpret_cast<double2*>(SMEM + gbase + PLAN.g_rr) + lane * WPL * 2; }
  RLX_HD uint16_t* twq() const { return reinterpret_cast<uint16_t*>(SMEM + gbase + PLAN.g_twq); }
  template <class T>
  RLX_HD const T* arr(uint32_t off) const {
    return reinterpret_cast<const T*>(SMEM + off);
  }
  // ---- hot plan (shared memory)
  RLX_HD NodeRec rec(int n) const {  // one 16-byte shared load
#ifdef __CUDA_ARCH__
    const uint4 v = arr<uint4>(PLAN.o_rec)[n];
    return NodeRec{v.x, v.y, v.z, v.w};
#else
    return arr<NodeRec>(PLAN.o_rec)[n];
#endif
  }
  RLX_HD uint32_t recw(int n, int k) const { return arr<uint32_t>(PLAN.o_rec)[4 * n + k]; }
  RLX_HD int hkind(int n) const { return (int)(recw(n, 2) >> 24); }
  RLX_HD int hpipe(int n) const { return (int)(recw(n, 3) & 0xFF); }
  RLX_HD int hworker(int n) const { return (int)(recw(n, 2) & 0xFFFF); }
  static RLX_HD int r_worker(const NodeRec& r) { return (int)(r.z & 0xFFFF); }
  static RLX_HD int r_flags(const NodeRec& r) { return (int)((r.z >> 16) & 0xFF); }
  RLX_HD int r_pos(const NodeRec& r) const {  // position in this pass's order (merge-shifted)
    int p = (int)((r.w >> (o ? 16 : 8)) & 0xFF);
    if (r_worker(r) == mt && p >= ins) p++;
    return p;
  }
  RLX_HD double hdur(int n) const { return arr<double>(PLAN.o_dur)[n]; }
  RLX_HD double hmem(int n) const { return PLAN.mem[n]; }         // pairing only: global (L1)
  RLX_HD double hmpre(int n) const {  // member starts
    return RLX_MPRE_HOT ? arr<double>(PLAN.o_mprefix)[n] : PLAN.mprefix[n];
  }
  RLX_HD double lutv(int i) const { return arr<double>(PLAN.o_lut)[i]; }
  // node attributes (M = the candidate's virtual merged node)
  RLX_HD int kind(int n) const { return n == PLAN.M ? wc()->kind : hkind(n); }
  RLX_HD int pipe(int n) const { return n == PLAN.M ? wc()->pipe : hpipe(n); }
  RLX_HD double dur(int n) const { return n == PLAN.M ? wc()->dur : hdur(n); }
  RLX_HD double memf(int n) const { return n == PLAN.M ? wc()->mem : hmem(n); }
  RLX_HD double mpre(int n) const { return n == PLAN.M ? wc()->pre : hmpre(n); }
  RLX_HD int wrk(int n) const { return n == PLAN.M ? wc()->t : hworker(n); }

  RLX_HD double L3(int k, int partner, int alloc) {
    double v = lutv((k * RLX_NPARTNER + partner + 1) * RLX_NALLOC + alloc);
    if (isnan(v) && err < kErrKeyBase) err = key_err(k, partner);
    return v;
  }
  // (rate, RN(1/rate)) for a member start: the reciprocal comes from the
  // planner's table (global memory, L1) instead of a division per start
  RLX_HD double2 L3r(int k, int partner, int alloc) {
    const int i = (k * RLX_NPARTNER + partner + 1) * RLX_NALLOC + alloc;
    const double v = lutv(i);
    if (isnan(v) && err < kErrKeyBase) err = key_err(k, partner);
#if RLX_RLUT
    return make_double2(v, PLAN.rlut[i]);
#else
    return make_double2(v, v == 1.0 ? 1.0 : recip(v));
#endif
  }
  RLX_HD int node_at(int w, int p) const {
    if (w == mt) {
      if (p == ins) return PLAN.M;
      if (p > ins) p--;
    }
    return arr<uint16_t>(PLAN.o_ord)[(o * PLAN.W + w) * kMaxPos + p];
  }
  RLX_HD int pos_of(int n) const { return r_pos(rec(n)); }

  // ---- completion bookkeeping (succs of a completed node; readiness)
  RLX_HD void became_ready(int s, const NodeRec& r) {
    const int f = r_flags(r);
    if (f & F_TW) {
      const int q = at_add<G>(&gc()->twq_n, 1);
      twq()[q] = (uint16_t)s;
    } else if (f & F_WIN) {
      at_or_bit<G>(&mask()[r_worker(r)], r_pos(r));
    }
  }
  RLX_HD void fire(int s, const NodeRec& r) {
    if (r_flags(r) & F_JOIN) {  // a join releases its members, whose only predecessor it is
      const uint16_t* sl = arr<uint16_t>(PLAN.o_succ);
      for (uint32_t e = r.x, e1 = r.x + (r.y & 0xFFFF); e < e1; e++) {
        const int t = sl[e];
        became_ready(t, rec(t));
      }
    } else {
      became_ready(s, r);
    }
  }
  RLX_HD void dec(int s) {
    const NodeRec r = rec(s);
    const unsigned c = r.y >> 16;
    if (c == 0xFFFFu || at_sub<G>(&ctr()[c], 1u) == 1u) fire(s, r);
  }
  RLX_HD void succs_of(const NodeRec& r) {
    const uint16_t* sl = arr<uint16_t>(PLAN.o_succ);
    for (uint32_t e = r.x, e1 = r.x + (r.y & 0xFFFF); e < e1; e++) dec(sl[e]);
  }
  RLX_HD void complete(int n, unsigned& ld) {
    if (n == PLAN.M) {
      ld++;
      const WarpCand* c = wc();
      for (int i = 0; i < c->k; i++) succs_of(rec(c->m[i]));
    } else {
      const NodeRec r = rec(n);
      if (r_flags(r) & F_WIN) ld++;
      succs_of(r);
    }
  }

  // ---- starting members (_start_member :460-484) on an idle local worker j
  // (dynamic); slot s is compile-time.
  RLX_HD void start(int j, int s, int w, int n, double2 rr2, int alloc, bool partner) {
    const double rate = rr2.x, rinv = rr2.y;  // exclusive starts run at 1.0 (slowdown.py:94-99)
    double pre = mpre(n);
    if (PLAN.has_penalty && kind(n) <= RLX_KIND_DECODE_SMALL) {
      double* g = &grant()[w * PLAN.P + pipe(n)];
      const double am = arr<double>(PLAN.o_alloc_mem)[alloc];
      const double lastg = *g;
      if (!isnan(lastg) && fabs(lastg - am) > kEps) pre = pre + PLAN.realloc_penalty;
      *g = am;
    }
    const double d = dur(n);
#pragma unroll
    for (int jj = 0; jj < WPL; jj++) {  // predicated register select (no per-lane branches)
      const bool hit = jj == j;
      wk[jj][s] = hit ? d : wk[jj][s];
    }
    if (RRS) {
      rr()[2 * j + s] = make_double2(rate, rinv);
    } else {
#pragma unroll
      for (int jj = 0; jj < (RRS ? 1 : WPL); jj++) {  // predicated register select
        const bool hit = jj == j;
        rt[jj][s] = hit ? rate : rt[jj][s];
        ri[jj][s] = hit ? rinv : ri[jj][s];
      }
    }
    const Bits bit = Bits(1) << (2 * j + s);
    nds()[2 * j + s] = (uint16_t)n;
    rb |= bit;
    if (partner) pf |= bit; else pf &= ~bit;
    if (pre != 0.0) {
      pm |= bit;
      pres()[2 * j + s] = pre;
    } else {
      pm &= ~bit;
    }
    const double fe = (now + pre) + d * rate;
    tl = fe < tl ? fe : tl;
  }

  RLX_HD static double rerated(double da, double sa, double db, double sb) {
    const double na = da * sa, nb = db * sb;
    if (fabs(na - nb) <= kEps) return na;
    if (na < nb) return na + (1.0 - na / nb) * db;
    return nb + (1.0 - nb / na) * da;
  }

  // _best_pair_action :803-828
  RLX_HD bool best_pair(int a, int b, int& first, int& second, int& alloc) {
    const double hr = PLAN.headroom;
    const double ma = memf(a), mb = memf(b);
    if (!(ma + mb <= 1.0 - hr + 1e-12)) return false;
    double best = INFINITY;
    bool found = false;
    const int ka = kind(a), kb = kind(b);
    const double da = dur(a), db = dur(b);
    for (int oo = 0; oo < 2; oo++) {
      const int f = oo ? b : a, s = oo ? a : b;
      const int kf = oo ? kb : ka, ks = oo ? ka : kb;
      const double df = oo ? db : da, ds = oo ? da : db;
      const double ms = oo ? ma : mb;
      for (int ai = 0; ai < 3; ai++)
        for (int mj = 0; mj < 4; mj++) {
          if (memgrid(mj) + ms > 1.0 - hr + kEps) continue;
          const int al = 1 + ai * 4 + mj;
          const double e = rerated(df, L3(kf, ks, al), ds, L3(ks, kf, al + 12));
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

  // ---- pass initialisation: decision state + `act` applied (window_cost :886-887)
  RLX_HD void init_pass(int variant, const Act& act, bool is_merge) {
    GroupCand* g = gc();
    const WarpCand* c = wc();
    o = variant == 2 ? 1 : 0;
    mt = is_merge ? c->t : -1;
    ins = is_merge ? (o ? c->ins1 : c->ins0) : -1;
    now = PLAN.now;
    last = 0.0;
    done_cnt = 0;
    guard = 0;
    any_done = false;
    const int W = PLAN.W;
    unsigned long long* mk = mask();
    unsigned* ct = ctr();
    double* te = twend();
    for (int i = lane; i < PLAN.NC; i += G) ct[i] = PLAN.ctr0[i];
    for (int w = lane; w < W; w += G) mk[w] = PLAN.mask0[o * W + w];
    for (int i = lane; i < PLAN.NTW; i += G) te[i] = PLAN.tw_end0[i];
    if (PLAN.has_penalty)
      for (int i = lane; i < W * PLAN.P; i += G) grant()[i] = PLAN.grant0[i];
    gsync<G>(gm);
    if (lane == 0) {
      g->twq_n = 0;
      g->tw_run = PLAN.n_tw_run0;
      g->dsum = 0;
    }
    rb = pm = pf = 0;
    tl = INFINITY;
#pragma unroll
    for (int j = 0; j < WPL; j++) {
      const int w = lane + G * j;
      if (w < W) {
        const int c = PLAN.nmem0[w];
#pragma unroll
        for (int s = 0; s < 2; s++)
          if (s < c) {
            const Bits bit = Bits(1) << (2 * j + s);
            const double r = PLAN.mrate0[2 * w + s], p = PLAN.mpre0[2 * w + s], wv = PLAN.mwork0[2 * w + s];
            nds()[2 * j + s] = PLAN.mnode0[2 * w + s];
            set_rate_static(j, s, r, recip(r));
            wk[j][s] = wv;
            rb |= bit;
            if (PLAN.mpart0[2 * w + s]) pf |= bit;
            if (p != 0.0) {
              pm |= bit;
              pres()[2 * j + s] = p;
            }
            const double fe = (now + p) + wv * r;
            tl = fe < tl ? fe : tl;
          }
      }
    }
    if (PLAN.n_tw_run0)  // tool waits running at the decision state
      for (int i = lane; i < PLAN.NTW; i += G) tl = te[i] < tl ? te[i] : tl;
    if (is_merge && lane == 0) {  // the merged node replaces its members in the ready masks
      const unsigned long long m = mk[mt];
      const unsigned long long lo = ins ? (m & ((1ull << ins) - 1)) : 0ull;
      mk[mt] = lo | ((m >> ins) << (ins + 1)) | (1ull << ins);
      for (int i = 0; i < c->k; i++) {
        const int x = c->m[i];
        mk[hworker(x)] &= ~(1ull << pos_of(x));
      }
    }
    gsync<G>(gm);
    if (act.cls >= 0) {
      const int w = wrk(act.a);
      if ((w % G) == lane) {
        const int j = w / G;
        if (act.cls == 2) {
          mk[w] &= ~(1ull << (act.a == PLAN.M ? ins : pos_of(act.a)));
          start(j, 0, w, act.a, L3r(kind(act.a), -1, 0), 0, false);
        } else {
          const int a = act.a, b = act.b;
          mk[w] &= ~((1ull << (a == PLAN.M ? ins : pos_of(a))) | (1ull << (b == PLAN.M ? ins : pos_of(b))));
          const double2 ra = L3r(kind(a), kind(b), act.alloc);
          const double2 rbv = L3r(kind(b), kind(a), act.alloc + 12);
          start(j, 0, w, a, ra, act.alloc, true);
          start(j, 1, w, b, rbv, act.alloc + 12, true);
        }
      }
    }
    gsync<G>(gm);
  }

  // ---- selection on idle workers (one sweep)
  RLX_HD void select(bool pair) {
    unsigned long long* mk = mask();
    // idle local workers with a ready node: the masks load in parallel, the
    // loop below visits only workers that start something
    unsigned idle = 0;
#pragma unroll
    for (int j = 0; j < WPL; j++)
      if (((vmask >> j) & 1u) && !((rb >> (2 * j)) & Bits(3)) && mk[lane + G * j] != 0ull) idle |= 1u << j;
#if RLX_SEL_UNROLL
    // one copy per local worker: start() writes the member's registers with a
    // compile-time slot instead of predicated selects over every slot
#pragma unroll
    for (int j = 0; j < WPL; j++)
      if ((idle >> j) & 1u) select_one(j, pair, mk);
#else
    while (idle) {
      const int j = ffs32(idle) - 1;
      idle &= idle - 1;
      select_one(j, pair, mk);
    }
#endif
  }

  // start the first ready node (or the best pair, pair variant) on idle local worker j
  RLX_HD void select_one(int j, bool pair, unsigned long long* mk) {
    const int w = lane + G * j;
    unsigned long long m = mk[w];
    const int p = ffs64(m) - 1;
    const int x = node_at(w, p);
    int first = x, second = -1, al = 0;
    bool paired = false;
    if (pair) {
      unsigned long long m2 = m & (m - 1);
      const int px = pipe(x);
      while (m2) {
        const int q = ffs64(m2) - 1;
        const int y = node_at(w, q);
        if (pipe(y) != px) {
          if (x != PLAN.M && y != PLAN.M) {  // decision-invariant pair: planner table
            const int cnt = arr<uint8_t>(PLAN.o_ord_cnt)[w];
            const int ent = PLAN.ptab[PLAN.pt_off[w] + ((recw(x, 3) >> 16) & 0xFF) * cnt + ((recw(y, 3) >> 16) & 0xFF)];
            if (ent >= 0x60 && ent < 0x80) {
              if (err < kErrKeyBase)  // the first LUT lookup of _best_pair_action that misses
                err = (ent & 1) ? key_err(hkind(y), hkind(x)) : key_err(hkind(x), hkind(y));
            } else if (ent) {
              paired = true;
              al = ent & 31;
              first = (ent & 0x40) ? y : x;
              second = (ent & 0x40) ? x : y;
            }
          } else {
            paired = best_pair(x, y, first, second, al);
          }
          if (paired) m &= ~(1ull << q);
          break;
        }
        m2 &= m2 - 1;
      }
    }
    m &= ~(1ull << p);
    mk[w] = m;
    if (paired) {
      const double2 ra = L3r(kind(first), kind(second), al);
      const double2 rbv = L3r(kind(second), kind(first), al + 12);
      start(j, 0, w, first, ra, al, true);
      start(j, 1, w, second, rbv, al + 12, true);
    } else {
      start(j, 0, w, x, L3r(kind(x), -1, 0), 0, false);
    }
  }

  // ---- advance (:593-627): consume dt on this lane's members, re-rate the
  // survivors of finished pairs, fold every survivor's next finish estimate
  // into tl, then complete the finished nodes.
  template <bool kPfx>
  RLX_HD void consume(double dt, unsigned& ld) {
    tl = INFINITY;
    Bits fb = 0;
    double* pr = pres();
    const bool dpos = dt > kEps;
#pragma unroll
    for (int j = 0; j < WPL; j++) {
      double fe0 = 0.0, fe1 = 0.0;  // next finish estimates; count only where keep
      bool keep0 = false, keep1 = false;
#pragma unroll
      for (int s = 0; s < 2; s++) {
        const Bits bit = Bits(1) << (2 * j + s);
        // slot 1 (the second member of a pair) is rare: branch on it; slot 0
        // is evaluated branch-free and masked
        if ((s == 1 || RLX_S0_BRANCH) && !(rb & bit)) continue;
        const bool on = (rb & bit) != Bits(0);
        double d = dt;
        double base = now;  // now + prefix_left (:328); prefix 0 on the common path
        bool dp = dpos, pdone = true;
        if (kPfx && (pm & bit)) {  // pending merge prefix / realloc penalty (:330-333)
          double p = pr[2 * j + s];
          if (p > kEps) {
            const double used = d < p ? d : p;
            p = p - used;
            d = d - used;
            pr[2 * j + s] = p;
            dp = d > kEps;
          }
          // a prefix consumed to exactly 0.0 drops out: (now + 0.0) == now
          if (p == 0.0) pm &= ~bit;
          base = now + p;
          pdone = p <= kEps;
        }
        double wv = wk[j][s];
        const double2 ry = rate_of(j, s);
        const double r = ry.x;
        // dt / rate (:335), correctly rounded without a division: Markstein's
        // correction of d * RN(1/r) by one exact FMA residual is RN(d / r)
        // (exact for rate 1.0), so every member runs the same straight-line code
        const double q = ediv(d, r, ry.y);
        // max(0.0, work_left - dt/rate) if dt > EPS and work_left > EPS; an
        // empty slot's value is dead, so `on` is not part of the condition
        wv = (dp && wv > kEps) ? pos0(wv - q) : wv;
        wk[j][s] = wv;
        const double prod = wv * r;  // shared by the finish test (:604-608) and the estimate (:328)
        const bool fin = on && pdone && prod <= kEps;
        if (fin) fb |= bit;
        const double fe = (RLX_TL_PRED || (on && !fin)) ? base + prod : INFINITY;
        if (s == 0) {
          fe0 = fe;
          keep0 = on && !fin;
        } else {
          fe1 = fe;
          keep1 = on && !fin;
        }
      }
      const Bits both = Bits(3) << (2 * j);
      if ((pf & both) && (fb & both) && (rb & both) != (fb & both)) {
        // a survivor whose partner finished drops to its exclusive speed (:615-621)
#pragma unroll
        for (int s = 0; s < 2; s++) {
          const Bits bit = Bits(1) << (2 * j + s);
          if ((rb & bit) && !(fb & bit) && (pf & bit)) {
            set_rate_static(j, s, 1.0, 1.0);
            pf &= ~bit;
            const double p = (pm & bit) ? pr[2 * j + s] : 0.0;
            const double fe = ((pm & bit) ? now + p : now) + wk[j][s] * 1.0;
            if (s == 0) fe0 = fe; else fe1 = fe;
          }
        }
      }
      if (RLX_TL_PRED) {
        tl = (keep0 && fe0 < tl) ? fe0 : tl;
        tl = (keep1 && fe1 < tl) ? fe1 : tl;
      } else {
        tl = fe0 < tl ? fe0 : tl;
        tl = (keep1 && fe1 < tl) ? fe1 : tl;
      }
    }
    rb &= ~fb;
    const uint16_t* nd = nds();
    while (fb) {
      const int i = (sizeof(Bits) == 4 ? ffs32((unsigned)fb) : ffs64(fb)) - 1;
      fb &= fb - 1;
      complete(nd[i], ld);
    }
  }

  // ---- advance for a lane none of whose running members has a pending
  // prefix (base == now for all of them): the arithmetic of consume<false>,
  // laid out as straight-line phases over all member slots so that the
  // slots' independent FP64 chains interleave instead of running worker by
  // worker between branches:
  //  1. consume dt (:335) and test for finish (:604-608), all slot 0s, then
  //     the running slot 1s;
  //  2. survivors of finished pairs drop to their exclusive speed (:615-621),
  //     found by bit arithmetic (partner finished = the pair-swapped `fb`);
  //  3. next finish estimate (:328): RN(now + x) is monotone in x, so
  //     min_i RN(now + p_i) == RN(now + min_i p_i) — one add per lane, the
  //     minimum taken over the products in two independent chains.
  RLX_HD void consume_lean(double dt, unsigned& ld) {
    double pd[WPL][2];
    Bits fb = 0;  // finish test on every evaluated slot; masked by rb below
    if (dt > kEps) {  // group-uniform: max(0, work_left - dt/rate) where work_left > EPS
#pragma unroll
      for (int s = 0; s < 2; s++)
#pragma unroll
        for (int j = 0; j < WPL; j++) {
          if (!RLX_S1_PRED && s == 1 && !(rb & (Bits(1) << (2 * j + 1)))) continue;
          const double2 ry = rate_of(j, s);
          const double wv = wk[j][s];
          const double nz = pos0(wv - ediv(dt, ry.x, ry.y));
          wk[j][s] = wv > kEps ? nz : wv;
        }
    }
#pragma unroll
    for (int s = 0; s < 2; s++)
#pragma unroll
      for (int j = 0; j < WPL; j++) {
        const Bits bit = Bits(1) << (2 * j + s);
        if (!RLX_S1_PRED && s == 1 && !(rb & bit)) {
          pd[j][s] = INFINITY;
          continue;
        }
        const double prod = wk[j][s] * rate_of(j, s).x;
        pd[j][s] = prod;
        fb |= prod <= kEps ? bit : Bits(0);
      }
    fb &= rb;
    const Bits lo = Bits(~Bits(0) / 3u);  // slot-0 bits
    const Bits surv = pf & rb & ~fb & (((fb & lo) << 1) | ((fb >> 1) & lo));
    if (surv) {
#pragma unroll
      for (int j = 0; j < WPL; j++)
#pragma unroll
        for (int s = 0; s < 2; s++) {
          const Bits bit = Bits(1) << (2 * j + s);
          if (surv & bit) {
            set_rate_static(j, s, 1.0, 1.0);
            pd[j][s] = wk[j][s];  // work_left * 1.0
          }
        }
      pf &= ~surv;
    }
    const Bits keep = rb & ~fb;
    double m0 = INFINITY, m1 = INFINITY;
#pragma unroll
    for (int j = 0; j < WPL; j++) {
      m0 = (((keep >> (2 * j)) & Bits(1)) && pd[j][0] < m0) ? pd[j][0] : m0;
      m1 = (((keep >> (2 * j + 1)) & Bits(1)) && pd[j][1] < m1) ? pd[j][1] : m1;
    }
    tl = now + (m1 < m0 ? m1 : m0);
    rb &= ~fb;
    const uint16_t* nd = nds();
    while (fb) {
      const int i = (sizeof(Bits) == 4 ? ffs32((unsigned)fb) : ffs64(fb)) - 1;
      fb &= fb - 1;
      complete(nd[i], ld);
    }
  }

  // ---- consume_lean for every lane: the running members with a pending
  // prefix (`pmr`, rare: a merge's migration prefix, realloc penalties) are
  // left out of the straight-line phases and finished on a slow path with
  // consume<true>'s arithmetic, so a warp whose lanes differ no longer runs
  // two whole consume variants.
  RLX_HD void consume_u(double dt, unsigned& ld) {
    double pd[WPL][2];
    const Bits pmr = pm & rb;
    if (dt > kEps) {
#pragma unroll
      for (int s = 0; s < 2; s++)
#pragma unroll
        for (int j = 0; j < WPL; j++) {
          const Bits bit = Bits(1) << (2 * j + s);
          if (!RLX_S1_PRED_U && s == 1 && !(rb & bit)) continue;
          const double2 ry = rate_of(j, s);
          const double wv = wk[j][s];
          const double nz = pos0(wv - ediv(dt, ry.x, ry.y));
          wk[j][s] = (wv > kEps && !(pmr & bit)) ? nz : wv;
        }
    }
    Bits fb = 0;
#pragma unroll
    for (int s = 0; s < 2; s++)
#pragma unroll
      for (int j = 0; j < WPL; j++) {
        const Bits bit = Bits(1) << (2 * j + s);
        if (!RLX_S1_PRED_U && s == 1 && !(rb & bit)) {
          pd[j][s] = INFINITY;
          continue;
        }
        const double prod = wk[j][s] * rate_of(j, s).x;
        pd[j][s] = prod;
        fb |= prod <= kEps ? bit : Bits(0);
      }
    fb &= rb & ~pmr;
    double* pr = pres();
    if (pmr) {  // prefix_left first, then work (:328-336)
#pragma unroll
      for (int j = 0; j < WPL; j++)
#pragma unroll
        for (int s = 0; s < 2; s++) {
          const Bits bit = Bits(1) << (2 * j + s);
          if (!(pmr & bit)) continue;
          double d = dt, p = pr[2 * j + s];
          bool dp = dt > kEps;
          if (p > kEps) {
            const double used = d < p ? d : p;
            p = p - used;
            d = d - used;
            pr[2 * j + s] = p;
            dp = d > kEps;
          }
          if (p == 0.0) pm &= ~bit;  // (now + 0.0) == now: the prefix drops out
          const double2 ry = rate_of(j, s);
          double wv = wk[j][s];
          const double q = ediv(d, ry.x, ry.y);
          wv = (dp && wv > kEps) ? pos0(wv - q) : wv;
          wk[j][s] = wv;
          const double prod = wv * ry.x;
          pd[j][s] = prod;
          if (p <= kEps && prod <= kEps) fb |= bit;
        }
    }
    const Bits lo = Bits(~Bits(0) / 3u);  // slot-0 bits
    const Bits surv = pf & rb & ~fb & (((fb & lo) << 1) | ((fb >> 1) & lo));
    if (surv) {  // a survivor whose partner finished drops to its exclusive speed (:615-621)
#pragma unroll
      for (int j = 0; j < WPL; j++)
#pragma unroll
        for (int s = 0; s < 2; s++) {
          const Bits bit = Bits(1) << (2 * j + s);
          if (surv & bit) {
            set_rate_static(j, s, 1.0, 1.0);
            pd[j][s] = wk[j][s];  // work_left * 1.0
          }
        }
      pf &= ~surv;
    }
    const Bits keep = rb & ~fb;
    const Bits kf = keep & ~pmr;
    double m0 = INFINITY, m1 = INFINITY;
#pragma unroll
    for (int j = 0; j < WPL; j++) {
      m0 = (((kf >> (2 * j)) & Bits(1)) && pd[j][0] < m0) ? pd[j][0] : m0;
      m1 = (((kf >> (2 * j + 1)) & Bits(1)) && pd[j][1] < m1) ? pd[j][1] : m1;
    }
    tl = now + (m1 < m0 ? m1 : m0);  // monotone: min_i RN(now + p_i) == RN(now + min_i p_i)
    if (keep & pmr) {  // base = now + prefix_left for these
#pragma unroll
      for (int j = 0; j < WPL; j++)
#pragma unroll
        for (int s = 0; s < 2; s++) {
          const Bits bit = Bits(1) << (2 * j + s);
          if (keep & pmr & bit) {
            const double fe = (now + pr[2 * j + s]) + pd[j][s];
            tl = fe < tl ? fe : tl;
          }
        }
    }
    rb &= ~fb;
    const uint16_t* nd = nds();
    while (fb) {
      const int i = (sizeof(Bits) == 4 ? ffs32((unsigned)fb) : ffs64(fb)) - 1;
      fb &= fb - 1;
      complete(nd[i], ld);
    }
  }

  // ---- the pass result (window_cost :889-890): the time of the last window
  // completion, or `now` if none
  RLX_HD double result() const {
    if (RLX_WIN_SMEM && PLAN.NTW == 0) {
      const GroupCand* g = gc();
      return g->dsum > 0 ? g->dlast : now;
    }
    return any_done ? last : now;
  }

  // ---- one simulated event of _complete_window (:833-867). Returns true
  // while the pass continues; on false `now`/`last`/`any_done` hold the result.
  RLX_HD bool step(bool pair, int nwin, long long serial, int variant) {
    select(pair);
    gsync<G>(gm);
    GroupCand* g = gc();
    const bool has_tw = PLAN.NTW != 0;  // uniform: plans without tool waits skip their bookkeeping
    const int twr = has_tw ? g->tw_run : 0;
    // next event time; +inf on every lane means no running member (tl is
    // the min over this lane's members and tool waits), so with no running
    // tool wait there are no events left (has_events :590)
    const double t = gmin<G>(gm, tl);
    if (t == INFINITY && twr == 0) return false;
    if (++guard > 10000) {  // scheduler.py:866-867
      if (!err) err = RLX_ERR_SCHEDULING;
      return false;
    }
    double dt = t - now;
    if (!(dt > 0.0)) dt = 0.0;
    now = t;
    unsigned ld = 0;
    // members with a pending prefix are rare (a merge's migration prefix until
    // consumed, realloc penalties): in 16- and 32-lane groups, lanes without
    // one run the consume with the prefix code compiled out (measured on one
    // box: config 5 5.70 vs 6.35 s, config 4 0.95 vs 1.08 s); with 4- and
    // 8-lane groups a warp holds 4-8 groups, some lane nearly always has a
    // prefix and the split would run both versions (config 2 875 vs 764 ms)
    constexpr bool kSplit = RLX_PFX_SPLIT && G >= RLX_PFX_MING;
    if (RLX_LEAN == 2 || (RLX_LEAN == 3 && !kSplit))
      consume_u(dt, ld);
    else if (!kSplit || (pm & rb))
      consume<true>(dt, ld);
    else if (RLX_LEAN)
      consume_lean(dt, ld);
    else
      consume<false>(dt, ld);
    if (!has_tw) {
      // window completions of this event: the completing lanes add to a
      // group counter before the barrier every lane needs anyway; a
      // broadcast read replaces a warp reduction on the critical path
#if RLX_WIN_SMEM
      // ... and record the event time next to it (every completing lane
      // writes the same `now`), so the pass keeps no per-lane count, last
      // time or flag in registers (they spilled to local memory)
      if (ld) {
        at_add<G>(&g->dsum, (int)ld);
        g->dlast = now;
      }
      gsync<G>(gm);
      return g->dsum < nwin;
#endif
      if (G > 1 && ld) at_add<G>(&g->dsum, (int)ld);
      gsync<G>(gm);
      const int cum = G > 1 ? g->dsum : done_cnt + (int)ld;
      if (cum != done_cnt) {
        done_cnt = cum;
        last = now;
        any_done = true;
      }
      return done_cnt < nwin;
    }
    gsync<G>(gm);
    // tool waits: expiry (:622-626) and auto-start of ready ones (:421-434)
    if (twr) {
      int ex = 0;
      double* te = twend();
      for (int i = lane; i < PLAN.NTW; i += G) {
        const double e = te[i];
        if (e <= now + kEps) {
          te[i] = INFINITY;
          complete(arr<uint16_t>(PLAN.o_tw_node)[i], ld);
          ex++;
        } else {
          tl = e < tl ? e : tl;
        }
      }
      if (ex) at_add<G>(&g->tw_run, -ex);
      gsync<G>(gm);
    }
    if (has_tw && g->twq_n > 0) {
      gsync<G>(gm);
      if (lane == 0) {
        uint16_t* q = twq();
        double* te = twend();
        while (g->twq_n > 0) {
          const int s = q[--g->twq_n];
          const double dd = hdur(s);
          if (dd <= kEps) {
            complete(s, ld);
          } else {
            const double e = now + dd;
            te[arr<int16_t>(PLAN.o_tw_slot)[s]] = e;
            g->tw_run++;
            tl = e < tl ? e : tl;
          }
        }
      }
      gsync<G>(gm);
    }
    const unsigned tot = gsum<G>(gm, ld);
    if (tot) {
      done_cnt += (int)tot;
      last = now;
      any_done = true;
    }
    return done_cnt < nwin;
  }
};

// Merged node of a Merge candidate (_apply_merge :517-581, merged_estimate
// :185-199, migration_cost :174-182) and its insertion point in both worker
// orders (ids compare as Python str). Group leader only.
RLX_HD void setup_merge(const Cand& c, WarpCand* sc) {
  long long tokens = 0, active = 0;
  double dmax = 0.0, mmax = 0.0, sfx = 0.0;
  const int p = PLAN.pipe[c.m[0]];
  for (int i = 0; i < c.k; i++) {
    const int x = c.m[i];
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
    const int bk = active >= 1024 ? 2 : (active >= 128 ? 1 : 0);
    kd = bk == 0 ? RLX_KIND_DECODE_SMALL : (bk == 1 ? RLX_KIND_DECODE_MEDIUM : RLX_KIND_DECODE_LARGE);
    if (!PLAN.latency_ok[p * 3 + bk]) sc->cerr = kErrLatBase + bk;  // latency_model[bucket] KeyError
    du = ((double)tokens * PLAN.latency[p * 3 + bk]) / (double)active;
  }
  double pre = 0.0;
  for (int i = 0; i < c.k; i++)
    if (PLAN.worker[c.m[i]] != c.target) pre = pre + PLAN.migc[c.m[i]];
  const double dm = defmem(kd);
  sc->kind = kd;
  sc->dur = du;
  sc->mem = mmax > dm ? mmax : dm;
  sc->pre = pre;
  sc->suf = du + sfx;
  sc->pipe = p;
  sc->t = c.target;
  sc->k = c.k;
  sc->idle = PLAN.nmem0[c.target] == 0;
  const int t = c.target;
  const int cnt = PLAN.ord_cnt[t];
  const int prk = PLAN.pipe_rank[p];
  for (int oo = 0; oo < 2; oo++) {
    int ins = cnt;
    for (int q = 0; q < cnt; q++) {
      const int y = PLAN.ord[(oo * PLAN.W + t) * kMaxPos + q];
      bool y_first;
      if (oo == 0 && PLAN.suffix[y] != sc->suf) {
        y_first = PLAN.suffix[y] > sc->suf;
      } else {
        const int yr = PLAN.pipe_rank[PLAN.pipe[y]];
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
          const int wid = PLAN.worker_ids[t];
          int tl = 0;
          tail[tl++] = ']';
          tail[tl++] = '@';
          tail[tl++] = 'w';
          {
            char tmp[12];
            int nt = 0;
            unsigned v = wid < 0 ? (unsigned)(-wid) : (unsigned)wid;
            do {
              tmp[nt++] = (char)('0' + v % 10);
              v /= 10;
            } while (v);
            if (wid < 0) tail[tl++] = '-';
            while (nt) tail[tl++] = tmp[--nt];
          }
          tail[tl] = 0;
          int cmp = 0;
          for (;;) {
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
            const unsigned char yc = (unsigned char)*ys;
            const unsigned char vc = (unsigned char)*cp;
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

// ---------------------------------------------------------------------------
// The pass list of a candidate (candidate_cost :902-918): a non-merge
// candidate or a merge onto a busy target is one action; a merge onto an
// idle target is Exclusive(M) followed by every Multiplex follow-up touching
// M (partners ready on the target in name order x orientation x alpha x
// mem, feasible only). Each action runs the window_cost variants (:893-897);
// variant 2 (name order) repeats variant 0 (suffix order) exactly when both
// orders coincide on every worker, the merged node included, so it is
// skipped then. Warp-slice writer only.
RLX_HD void build_passes(WarpCand* c) {
  uint16_t* acts = reinterpret_cast<uint16_t*>(c + 1);
  int n = 1;
  if (c->cls == 1 && c->idle) {
    const double hr = PLAN.headroom;
    unsigned long long rm = PLAN.mask0[1 * PLAN.W + c->t];
    while (rm) {
      const int q = ffs64(rm) - 1;
      rm &= rm - 1;
      const int y = PLAN.ord[(1 * PLAN.W + c->t) * kMaxPos + q];
      bool member = false;
      for (int i = 0; i < c->k; i++) member |= c->m[i] == y;
      if (member || PLAN.pipe[y] == c->pipe) continue;
      if (!(c->mem + PLAN.mem[y] <= 1.0 - hr + 1e-12)) continue;
      for (int oo = 0; oo < 2; oo++)
        for (int ai = 0; ai < 3; ai++)
          for (int mj = 0; mj < 4; mj++) {
            const double ms = oo ? c->mem : PLAN.mem[y];
            if (memgrid(mj) + ms > 1.0 - hr + kEps) continue;
            acts[n - 1] = (uint16_t)(q << 5 | oo << 4 | (ai * 4 + mj));
            n++;
          }
    }
  }
  c->n_act = n;
  c->n_var = (PLAN.same_order && (c->cls != 1 || c->ins0 == c->ins1)) ? 2 : 3;
  c->total = c->cerr ? 0 : n * c->n_var;
}

// Pass index -> (action, variant). Default: variant-major, so the groups of
// a warp run the same variant of sibling actions at the same time;
// RLX_PASS_ORDER=1 (tuning) runs the variants of one action together.
RLX_HD void split_pass(int q, int na, int nv, int& a, int& v) {
  if (PLAN.pass_order) {
    a = q / nv;
    v = q % nv;
  } else {
    a = q % na;
    v = q / na;
  }
}

// The action of action index `ai` of the warp's candidate.
RLX_HD Act pass_action(const WarpCand* c, int ai) {
  if (c->cls != 1) return Act{c->cls, c->a, c->b, c->alloc};
  if (!c->idle) return Act{-1, -1, -1, 0};
  if (ai == 0) return Act{2, PLAN.M, -1, 0};
  const int e = reinterpret_cast<const uint16_t*>(c + 1)[ai - 1];
  const int y = PLAN.ord[(1 * PLAN.W + c->t) * kMaxPos + (e >> 5)];
  const bool oo = (e >> 4) & 1;
  return Act{0, oo ? y : PLAN.M, oo ? PLAN.M : y, 1 + (e & 15)};
}

// Decode serial `serial` into the warp slice and set up its pass queue
// (merged node, finish estimate, passes). Warp-slice writer only.
RLX_HD void load_candidate(WarpCand* c, long long serial) {
  Cand cd;
  decode_serial(PLAN, serial, cd);
  c->serial = serial;
  c->cls = cd.cls;
  c->cost = dbits(INFINITY);
  c->err = 0x7fffffff;
  c->cerr = 0;
  if (cd.cls == 1) {
    setup_merge(cd, c);
    c->fin = (PLAN.now + c->pre) + c->dur;
    c->nwin = PLAN.NWIN - cd.k + 1;
  } else {
    // action_finish_estimate :773-789 (with the realloc penalty of the decision state)
    c->a = cd.a;
    c->b = cd.cls == 0 ? cd.b : -1;
    c->alloc = cd.alloc;
    c->nwin = PLAN.NWIN;
    auto pre_of = [&](int n, int alloc) {
      double pre = PLAN.mprefix[n];
      if (PLAN.has_penalty && PLAN.kind[n] <= RLX_KIND_DECODE_SMALL) {
        const double gr = PLAN.grant0[PLAN.worker[n] * PLAN.P + PLAN.pipe[n]];
        if (!isnan(gr) && fabs(gr - PLAN.alloc_mem[alloc]) > kEps) pre = pre + PLAN.realloc_penalty;
      }
      return pre;
    };
    auto lut = [&](int k, int partner, int alloc, int& err) {
      const double v = PLAN.lut[(k * RLX_NPARTNER + partner + 1) * RLX_NALLOC + alloc];
      if (isnan(v) && !err) err = key_err(k, partner);
      return v;
    };
    int e = 0;
    if (cd.cls == 2) {
      const double r = lut(PLAN.kind[cd.a], -1, 0, e);
      c->fin = (PLAN.now + pre_of(cd.a, 0)) + PLAN.dur[cd.a] * r;
    } else {
      const double ra = lut(PLAN.kind[cd.a], PLAN.kind[cd.b], cd.alloc, e);
      const double rbv = lut(PLAN.kind[cd.b], PLAN.kind[cd.a], cd.alloc + 12, e);
      const double fa = (PLAN.now + pre_of(cd.a, cd.alloc)) + PLAN.dur[cd.a] * ra;
      const double fb = (PLAN.now + pre_of(cd.b, cd.alloc + 12)) + PLAN.dur[cd.b] * rbv;
      c->fin = fb > fa ? fb : fa;
    }
    // a missing LUT row raises in the first pass's apply (window_cost runs
    // before action_finish_estimate, :963-972): the passes report it
    (void)e;
  }
  build_passes(c);
}

// Serial of work index `idx` of this launch: per class (merges, then
// multiplex, then exclusive: heaviest first) the shard owns either a
// contiguous range (world == 1) or every world-th block of 2^blk_shift
// serials starting at block `rank` (cost-balanced multi-GPU shards).
RLX_HD long long work_serial(const WorkDesc& wd, long long idx) {
  for (int r = 0; r < 3; r++) {
    if (idx < wd.loc[r]) {
      const long long blk = idx >> wd.blk_shift, off = idx & ((1ll << wd.blk_shift) - 1);
      return wd.s0[r] + ((blk * wd.world + wd.rank) << wd.blk_shift) + off;
    }
    idx -= wd.loc[r];
  }
  return -1;
}

// Fetch the next candidate of the launch into the warp slice (gen + 1), or
// mark the warp done (gen = -1). Once some candidate failed, only lower
// serials can still change the outcome (the reference raises on the first
// failing serial of its scan).
RLX_COLD void fetch_candidate(const WorkDesc& wd, WarpCand* c) {
  const long long total = wd.loc[0] + wd.loc[1] + wd.loc[2];
  long long serial = -1;
  for (;;) {
    const long long idx = (long long)at_add64(wd.counter, 1ull);
    if (idx >= total) break;
    const long long s = work_serial(wd, idx);
    if ((unsigned long long)s <= (*(volatile unsigned long long*)wd.err_key >> 8)) {
      serial = s;
      break;
    }
  }
  const int g = gen_load(&c->gen);
  if (serial < 0) {
    c->serial = -1;
    gen_store(&c->gen, -1);
    return;
  }
  load_candidate(c, serial);
  c->next = 0;
  c->done = 0;
  gen_store(&c->gen, g + 1);
}

// Finalise the warp's candidate: key (cost, finish, priority, serial) into
// this group's running best, or the failure into the launch's error key.
RLX_COLD void finish_candidate(const WorkDesc& wd, WarpCand* c, GroupCand* g) {
  if (c->serial < 0) return;
  const int code = c->cerr ? c->cerr : (c->err != 0x7fffffff ? (c->err & 0xff) : 0);
  if (code) {
    at_min64(wd.err_key, ((unsigned long long)c->serial << 8) | (unsigned long long)code);
    return;
  }
  g->ncand++;
  double cost;
  const unsigned long long cb = c->cost;
  memcpy(&cost, &cb, 8);
  const unsigned long long k0 = cb, k1 = dbits(c->fin);
  const unsigned long long k2 = ((unsigned long long)c->cls << 61) | (unsigned long long)c->serial;
  if (key_less(k0, k1, k2, g->b0, g->b1, g->b2)) {
    g->b0 = k0;
    g->b1 = k1;
    g->b2 = k2;
  }
  if (wd.keys_out) {
    wd.keys_out[2 * (c->serial - wd.shard0)] = cost;
    wd.keys_out[2 * (c->serial - wd.shard0) + 1] = c->fin;
  }
}

// One group's share of a launch, flattened so that one loop iteration is one
// simulated event for every group of the warp (pass and candidate
// boundaries are short divergent prologues). `ngw` groups share the warp
// slice at `wbase`.
template <int G, int WPL>
struct GroupRunner {
  Lane<G, WPL> S;
  const WorkDesc& wd;
  const int ngw;
  bool active = false;  // a pass is running
  bool ran = false;     // a pass ran since the last fold
  bool drained = false; // this group found the current candidate's queue empty
  int gen = 0;          // generation of the candidate this group works on
  int p = 0, variant = 0, nwin = 0, ref_idx = 0;
  bool pair = false;

  RLX_HD GroupRunner(const WorkDesc& w, uint32_t gbase, uint32_t wbase, int lane, unsigned gm, int n)
      : S(gbase, wbase, lane, gm), wd(w), ngw(n) {}

  RLX_HD void init() {
    GroupCand* g = S.gc();
    if (S.lane == 0) {
      g->b0 = g->b1 = g->b2 = ~0ull;
      g->passes = g->ncand = g->events = 0;
      g->bytes = 0.0;
    }
    gsync<G>(S.gm);
  }

  // One iteration; false when the launch has no more work for this group.
  RLX_HD bool iter() {
    if (active) {
      active = S.step(pair, nwin, 0, variant);
      return true;
    }
    return boundary() != 2;
  }

  // ---- pass boundary: fold the finished pass, claim the next one of the
  // warp's candidate and initialise it. 0: claimed, 1: wait, 2: no more work.
  RLX_HD int boundary() {
    // Warp-slice fields are written by one lane and read
    // by the others after a __syncwarp / fence (compute-sanitizer racecheck).
    GroupCand* g = S.gc();
    WarpCand* c = S.wc();
    gsync<G>(S.gm);
    if (ran) {  // fold the finished pass into the candidate
      const double x = S.result();
      const int e = gmax<G>(S.gm, S.err);
      gsync<G>(S.gm);
      if (S.lane == 0) {
        g->events += (unsigned long long)S.guard;
        if (e) {
          at_min32(&c->err, ref_idx << 8 | e);
        } else {
          at_min64s(&c->cost, dbits(x));
        }
      }
      S.err = 0;
      ran = false;
    }
    int q = -1, st = 0;  // st: 0 claimed pass q, 1 wait, 2 exit
    if (S.lane == 0) {
      const int cg = gen_load(&c->gen);
      if (cg < 0) {
        st = 2;
      } else {
        if (cg != gen) {
          gen = cg;
          drained = false;
        }
        st = 1;
        while (!drained) {
          const int t = at_add32(&c->next, 1);
          if (t >= c->total) {
            drained = true;
            fence_block();
            if (at_add32(&c->done, 1) == ngw - 1) {  // last group out: finalise, fetch the next
              fence_block();
              finish_candidate(wd, c, g);
              fetch_candidate(wd, c);
            }
            break;
          }
          int ta, tv;
          split_pass(t, c->n_act, c->n_var, ta, tv);
          const int ri = ta * 3 + tv;  // reference order: action-major, variant-minor
          if ((ri << 8) > c->err) continue;  // an earlier pass of this candidate already failed
          q = t;
          st = 0;
          break;
        }
      }
    }
    st = (int)gbcast<G>(S.gm, st);
    if (st == 2) return 2;
    if (st == 1) return 1;
    q = (int)gbcast<G>(S.gm, q);
    fence_block();
    int ai;
    split_pass(q, c->n_act, c->n_var, ai, variant);
    ref_idx = ai * 3 + variant;
    pair = variant == 1;
    nwin = c->nwin;
    const Act act = pass_action(c, ai);
    S.init_pass(variant, act, c->cls == 1);
    if (S.lane == 0 && variant == 0) {  // the reference's 3 passes of this action (SURVEY §8(d) bytes)
      g->passes += 3;
      g->bytes += 3.0 * (32.0 * nwin + 4.0 * (double)PLAN.ew +
                         32.0 * (PLAN.n_run0 + (act.cls < 0 ? 0 : act.cls == 0 ? 2 : 1)) + 16.0 * PLAN.n_tw_run0);
    }
    ran = true;
    active = nwin > 0;  // empty window: the pass result is `now` (:889-890)
    return 0;
  }

  RLX_HD void finish(SliceOut* out) {
    gsync<G>(S.gm);
    const GroupCand* g = S.gc();
    if (S.lane == 0) {
      out->k0 = g->b0;
      out->k1 = g->b1;
      out->k2 = g->b2;
      out->passes = g->passes;
      out->bytes = g->bytes;
      out->cands = g->ncand;
      out->events = g->events;
    }
  }
};

// ---- TMA bulk staging of the hot plan region into shared memory
__device__ __forceinline__ void stage_hot(uint8_t* dst, const uint8_t* src, uint32_t bytes, uint64_t* bar) {
#ifdef __CUDA_ARCH__
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    constexpr uint32_t kChunk = 1u << 16;
    for (uint32_t off = 0; off < bytes; off += kChunk) {
      const uint32_t n = bytes - off < kChunk ? bytes - off : kChunk;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d + off),
          "l"(src + off), "r"(n), "r"(b)
          : "memory");
    }
  }
  __syncthreads();
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(b)
        : "memory");
  }
#endif
}

// Threads per CTA: 8 workers per lane need ~150 registers, 4 fit in 128.
#ifndef RLX_T8
#define RLX_T8 256
#endif
#ifndef RLX_T2
#define RLX_T2 512
#endif
#ifndef RLX_T4
#define RLX_T4 512
#endif
constexpr int threads_for(int WPL) { return WPL >= 8 ? RLX_T8 : WPL <= 2 ? RLX_T2 : RLX_T4; }

#ifndef RLX_MINB2
#define RLX_MINB2 1
#endif
constexpr int min_blocks_for(int WPL) { return WPL <= 2 ? RLX_MINB2 : 1; }

template <int G, int WPL>
__global__ void __launch_bounds__(threads_for(WPL), min_blocks_for(WPL))
    rlx_score_kernel(const __grid_constant__ WorkDesc wd, SliceOut* outs) {
  __shared__ __align__(8) uint64_t bar;
  stage_hot(rlx_smem, c_plan.hot, c_plan.hot_bytes, &bar);
  const int lane = threadIdx.x % G;
  const int grp = threadIdx.x / G;
  const int wl = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  constexpr int kNgw = 32 / G;  // groups per warp
  const unsigned gm = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (threadIdx.x & (32 - G)));  // this group's lanes
  const uint32_t wbase = c_plan.hot_bytes + (uint32_t)warp * c_plan.w_bytes;
  const uint32_t gbase = c_plan.hot_bytes + (uint32_t)(blockDim.x >> 5) * c_plan.w_bytes + (uint32_t)grp * c_plan.g_bytes;
  if (wl == 0) {  // the warp's first candidate
    WarpCand* c = reinterpret_cast<WarpCand*>(rlx_smem + wbase);
    gen_store(&c->gen, 0);
    fetch_candidate(wd, c);
  }
  __syncwarp();
  GroupRunner<G, WPL> R(wd, gbase, wbase, lane, gm, kNgw);
  R.init();
  while (R.iter()) {
  }
  R.finish(&outs[blockIdx.x * (blockDim.x / G) + grp]);
}

// Shard winner + stats over all groups (deterministic: lexicographic min).
__global__ void rlx_reduce_kernel(const SliceOut* outs, int n, unsigned long long* res /* 8 words */) {
  __shared__ unsigned long long s0[256], s1[256], s2[256], sp[256], sc[256], se[256];
  __shared__ double sb[256];
  unsigned long long b0 = ~0ull, b1 = ~0ull, b2 = ~0ull, ps = 0, cs = 0, es = 0;
  double by = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (key_less(outs[i].k0, outs[i].k1, outs[i].k2, b0, b1, b2)) {
      b0 = outs[i].k0;
      b1 = outs[i].k1;
      b2 = outs[i].k2;
    }
    ps += outs[i].passes;
    cs += outs[i].cands;
    es += outs[i].events;
    by += outs[i].bytes;
  }
  s0[threadIdx.x] = b0;
  s1[threadIdx.x] = b1;
  s2[threadIdx.x] = b2;
  sp[threadIdx.x] = ps;
  sc[threadIdx.x] = cs;
  se[threadIdx.x] = es;
  sb[threadIdx.x] = by;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if ((int)threadIdx.x < st) {
      const int o = threadIdx.x + st;
      if (key_less(s0[o], s1[o], s2[o], s0[threadIdx.x], s1[threadIdx.x], s2[threadIdx.x])) {
        s0[threadIdx.x] = s0[o];
        s1[threadIdx.x] = s1[o];
        s2[threadIdx.x] = s2[o];
      }
      sp[threadIdx.x] += sp[o];
      sc[threadIdx.x] += sc[o];
      se[threadIdx.x] += se[o];
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
    res[7] = se[0];
  }
}

// ---------------------------------------------------------------------------
// host-side launch helpers (called from rlx_abi.cu)

typedef void (*KernelFn)(const WorkDesc, SliceOut*);

// Lane-group shape for W simulated workers: WPL workers per lane in
// registers, G = the smallest power of two with G * WPL >= W. RLX_SHAPE=G,WPL
// overrides it (tuning).
void choose_shape(int W, int& G, int& WPL) {
  // measured with the per-warp pass queue (profiles/r02_shape_sweep.txt):
  // config 2 (16 workers) 4x4 874 ms vs 8x2 917 ms vs 2x8 1250 ms; config 5
  // (64 workers) 16x4 6.35 s vs 8x8 7.87 s vs 32x2 8.18 s. Four workers per
  // lane, as few lanes per group as cover W: more groups share a warp and
  // drain one candidate's near-identical passes together.
  WPL = W <= 8 ? 2 : 4;
  G = 1;
  while (G * WPL < W) G *= 2;
}

size_t plan_slice_bytes(const DevPlan& P, int G, int WPL) {
  DevPlan P2 = P;
  group_layout(P2, G, WPL);
  return P2.w_bytes + (size_t)(32 / G) * P2.g_bytes;  // one warp: its candidate slice + its groups
}

static KernelFn pick(int G, int WPL) {
  if (WPL == 1) {
    switch (G) {
      case 8: return rlx_score_kernel<8, 1>;
      case 16: return rlx_score_kernel<16, 1>;
      case 32: return rlx_score_kernel<32, 1>;
    }
  } else if (WPL == 2) {
    switch (G) {
      case 1: return rlx_score_kernel<1, 2>;
      case 2: return rlx_score_kernel<2, 2>;
      case 4: return rlx_score_kernel<4, 2>;
      case 8: return rlx_score_kernel<8, 2>;
      case 16: return rlx_score_kernel<16, 2>;
      case 32: return rlx_score_kernel<32, 2>;
    }
  } else if (WPL == 4) {
    switch (G) {
      case 1: return rlx_score_kernel<1, 4>;
      case 2: return rlx_score_kernel<2, 4>;
      case 4: return rlx_score_kernel<4, 4>;
      case 8: return rlx_score_kernel<8, 4>;
      case 16: return rlx_score_kernel<16, 4>;
      case 32: return rlx_score_kernel<32, 4>;
    }
  } else if (WPL == 8) {
    switch (G) {
      case 1: return rlx_score_kernel<1, 8>;
      case 2: return rlx_score_kernel<2, 8>;
      case 4: return rlx_score_kernel<4, 8>;
      case 8: return rlx_score_kernel<8, 8>;
      case 16: return rlx_score_kernel<16, 8>;
    }
  }
  return nullptr;
}

int launch_score(const DevPlan& P, WorkDesc wd, SliceOut* outs, int max_slices, int sm_count, cudaStream_t st,
                 int* n_slices_out, int threads_hint) {
  int G, WPL;
  choose_shape(P.W, G, WPL);
  if (const char* sh = getenv("RLX_SHAPE")) sscanf(sh, "%d,%d", &G, &WPL);
  KernelFn fn = pick(G, WPL);
  if (!fn || G * WPL < P.W) return RLX_ERR_LIMIT;
  DevPlan P2 = P;
  group_layout(P2, G, WPL);
  P2.pass_order = getenv("RLX_PASS_ORDER") ? atoi(getenv("RLX_PASS_ORDER")) : 0;  // tuning
  const size_t gb = P2.g_bytes, wb = P2.w_bytes;
  wd.slice_bytes = (int)gb;
  const size_t hot = P.hot_bytes;
  const size_t cap = kSmemCap;
  auto need_smem = [&](int t) { return hot + (size_t)(t / 32) * wb + (size_t)(t / G) * gb; };
  if (need_smem(32) > cap) return RLX_ERR_LIMIT;
  int threads = threads_hint > 0 && threads_hint <= threads_for(WPL) ? threads_hint : threads_for(WPL);
  while (threads > 32 && need_smem(threads) > cap) threads /= 2;
  const size_t smem = need_smem(threads);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return RLX_ERR_CUDA;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess) return RLX_ERR_CUDA;
  if (per_sm < 1) return RLX_ERR_LIMIT;
  const int64_t total = wd.loc[0] + wd.loc[1] + wd.loc[2];
  const int64_t per_block = threads / 32;  // one candidate at a time per warp
  const int64_t need = (total + per_block - 1) / per_block;
  int64_t blocks = (int64_t)per_sm * sm_count;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  if (blocks * (threads / G) > max_slices) blocks = max_slices / (threads / G);
  if (cudaMemcpyToSymbolAsync(c_plan, &P2, sizeof(DevPlan), 0, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return RLX_ERR_CUDA;
  fn<<<(unsigned)blocks, threads, smem, st>>>(wd, outs);
  if (cudaGetLastError() != cudaSuccess) return RLX_ERR_CUDA;
  *n_slices_out = (int)(blocks * (threads / G));
  return 0;
}

int launch_reduce(const SliceOut* outs, int n, unsigned long long* res, cudaStream_t st) {
  rlx_reduce_kernel<<<1, 256, 0, st>>>(outs, n, res);
  return cudaGetLastError() == cudaSuccess ? 0 : RLX_ERR_CUDA;
}

}  // namespace rlx

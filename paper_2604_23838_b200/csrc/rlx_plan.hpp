// rlx_plan.hpp — per-decision device plan shared by the host planner
// (rlx_plan.cpp) and the sm_100a scoring kernel (rlx_kernels.cu).
//
// A "plan" is everything that is invariant across the candidates of one
// decision: the W-round window
// (scheduler.py:710-748), suffix lengths (:751-770), per-worker ready
// orders for the two completion keys (:893-894), initial running members
// and tool waits, the slowdown LUT, and the candidate space layout
// (enumerate_actions :648-703) so the device can unrank any serial.
//
// Nodes are renumbered into a compact "local" index space:
//   [0, NL)          window nodes + auxiliary tool waits (tool waits outside
//                    the window that can still auto-start during a pass)
//   M = NL           the candidate's virtual merged node (merge candidates)
//   [NL+1, NT)       join counters: a set of nodes sharing one large
//                    predecessor set (the Training gradient-sync barrier,
//                    graph.py:393-395) waits on one counter instead of
//                    |preds| x |group| edges.
#pragma once
#include <stdint.h>

#ifndef RLX_MPRE_HOT
#define RLX_MPRE_HOT 0  // 1: pending merge prefixes staged in shared memory (tuning)
#endif

#ifdef __CUDACC__
#define RLX_HD __host__ __device__ __forceinline__
#else
#define RLX_HD inline
#endif

namespace rlx {

constexpr int kMaxPos = 64;        // ready-mask bits per worker (u64)
constexpr int kMaxMembers = 64;    // merge members
constexpr int kMaxFrags = 128;     // fragments per pipeline for unranking
constexpr int kBinomK = 65;        // binomial table columns
constexpr double kEps = 1e-9;      // scheduler.py:43
constexpr unsigned kSmemCap = 227 * 1024 - 64;  // dynamic shared memory per CTA (sm_100)

// node flags
constexpr uint8_t F_TW = 1;        // ToolWait kind
constexpr uint8_t F_WIN = 2;       // inside the W-round window
constexpr uint8_t F_JOIN = 4;      // join counter
constexpr uint8_t F_READY0 = 8;    // ready at the decision state
constexpr uint8_t F_RUN0 = 16;     // running at the decision state

// Packed per-node record of the hot region: everything the completion and
// selection paths read about a node in one 16-byte shared-memory load.
//   x: successor CSR offset        y: successor count | counter slot << 16 (0xFFFF: none)
//   z: worker | flags << 16 | kind << 24
//   w: pipeline | position in the suffix-key order << 8 | in the name-key order << 16 (255: none)
struct NodeRec {
  uint32_t x, y, z, w;
};

// One multiplex pair block of the candidate space (enumerate_actions
// :661-677): nodes a < b (ready order) on one idle worker; orientation
// (a, b) contributes 3 x na serials (alpha x the na feasible memory grid
// points for b — a prefix of MEM_GRID), then (b, a) 3 x nb. The device
// unranks a multiplex serial from these blocks.
struct MuxPair {
  int64_t serial0;
  uint16_t a, b;
  uint8_t na, nb;
  uint16_t _pad;
};

struct MergeBlock {
  int64_t serial0;   // first serial of the block
  int64_t combos;    // valid combos (each has `size` targets)
  int32_t size;
  int32_t pipe;
  int32_t frag_off;  // into frags[]
  int32_t n_frags;
  int64_t expl_off;  // into combos[] (explicit list) or -1 (combinatorial unrank)
};

struct DevPlan {
  // sizes
  int32_t NL, NT, M, NWIN;
  int32_t W, P, NTW, n_blocks;
  int32_t has_penalty, merge_enabled;
  int32_t n_run0, n_tw_run0;
  double now, headroom, realloc_penalty, default_migration_cost;
  int64_t n_mux, n_merge, n_excl, n_total;
  int64_t ew;  // pred edges with both ends in the window (bytes model)
  int32_t NC;  // readiness counters: nodes (and joins) with >= 2 unresolved preds
  int32_t max_ord;  // longest per-worker order (ready-mask width)
  int32_t same_order;  // 1: suffix order == name order on every worker
  int32_t acts_cap;  // merge follow-up list capacity per warp slice (set at launch)
  int32_t pass_order;  // 0: variant-major pass queue (default), 1: action-major (tuning; set at launch)

  // Hot region: the leading `hot_bytes` of the plan blob hold every array the
  // event loop touches; the kernel stages it into shared memory with TMA bulk
  // copies and addresses it through these byte offsets.
  const uint8_t* hot;
  uint32_t hot_bytes;
  uint32_t o_rec, o_tw_slot, o_succ, o_ord, o_dur, o_lut, o_alloc_mem, o_tw_node, o_ord_cnt;
  uint32_t o_mprefix;  // merge prefixes in the hot region (RLX_MPRE_HOT builds)
  // Group slice layout in shared memory (set at launch, rlx_kernels.cu group_layout)
  uint32_t g_bytes, g_mask, g_twend, g_grant, g_pres, g_rr, g_ctr, g_nds, g_twq;
  uint32_t w_bytes;  // warp slice (one candidate and its pass queue)

  // per local node (NT unless noted)
  const uint8_t* kind;       // [NL]
  const uint8_t* pipe;       // [NL]
  const uint16_t* worker;    // [NL]
  const uint8_t* flags;      // [NT]
  const double* dur;         // [NL]
  const double* mem;         // [NL]
  const double* mprefix;     // [NL] pending merge prefix
  const double* suffix;      // [NL]
  const double* msx;         // [NL] max suffix over successors (0 if none)
  const double* migc;        // [NL] migration cost of moving this fragment
  const int64_t* rem;        // [NL]
  const int64_t* act;        // [NL]
  const int32_t* name_rank;  // [NL] rank by (pipeline id, id)
  const uint8_t* lt_merge;   // [NL] 1: id < "merge[", 0: id > "merge[", 2: id starts with "merge["
  const int32_t* id_off;     // [NL]
  const char* ids;
  const uint8_t* pos;        // [2][NL] position in the worker order (255: none)
  const int16_t* tw_slot;    // [NL] -1 unless ToolWait
  const uint16_t* tw_node;   // [NTW]
  const int32_t* succ_off;   // [NT+1]
  const uint16_t* succ;
  const uint16_t* pend0;     // [NT] initial pending predecessors (M: 0)
  const uint16_t* ctr_idx;   // [NT] counter slot of a node with pend0 >= 2, else 0xFFFF
  const uint16_t* ctr0;      // [NC] initial counter values

  // per worker
  const uint16_t* ord;       // [2][W][kMaxPos]
  const uint8_t* ord_cnt;    // [W]
  const uint64_t* mask0;     // [2][W]
  const uint8_t* nmem0;      // [W]
  const uint16_t* mnode0;    // [W*2]
  const uint8_t* mpart0;     // [W*2]
  const double* mrate0;      // [W*2]
  const double* mpre0;       // [W*2]
  const double* mwork0;      // [W*2]
  const int32_t* worker_ids; // [W]
  const double* tw_end0;     // [NTW] (+inf: not running)
  const double* grant0;      // [W*P] last mem grant (NaN: none)

  // per pipeline
  const uint8_t* pipe_rank;  // [P]
  const double* latency;     // [P*3]
  const uint8_t* latency_ok; // [P*3]
  const uint8_t* has_spec;   // [P]

  // cost model
  const double* lut;         // [7*8*25]
  const double* rlut;        // [7*8*25] RN(1 / lut): member starts (global, L1)
  const double* alloc_mem;   // [25]

  // candidate space
  const MuxPair* mux_pairs;  // [n_mux_pairs]
  int64_t n_mux_pairs;
  const uint16_t* excl;      // [n_excl]
  const MergeBlock* blocks;  // [n_blocks]
  const uint16_t* frags;
  const uint16_t* combos;
  const uint64_t* binom;     // [(kMaxFrags+1) * kBinomK], saturating
  const uint32_t* pt_off;    // [W+1] pair table offsets per worker
  const uint8_t* ptab;       // decision-invariant _best_pair_action results (cnt x cnt per worker)
};

// Per-slice result of the scoring kernel.
struct SliceOut {
  unsigned long long k0, k1, k2;  // packed best key
  unsigned long long passes;
  double bytes;
  unsigned long long cands;
  unsigned long long events;  // simulated events (advances) over all passes
};

// Work handed to one scoring launch (one serial shard). Per class r
// (0 merges, 1 multiplex, 2 exclusive — heaviest first) the shard owns
// loc[r] serials: with world == 1 the contiguous range [s0[r], s0[r] +
// loc[r]); otherwise every world-th block of 2^blk_shift serials of the
// class range starting at s0[r], beginning with block `rank`
// (rlx_kernels.cu work_serial; cost-balanced multi-GPU shards).
struct WorkDesc {
  int64_t s0[3];
  int64_t loc[3];
  int32_t world, rank, blk_shift, slice_bytes;  // slice_bytes: DevPlan::g_bytes
  int64_t shard0;   // keys_out index base
  double* keys_out; // device, optional
  unsigned long long* counter;
  unsigned long long* err_key;  // lowest failing candidate: serial << 8 | error code (~0: none)
};

// Serials a block-cyclic shard owns of a class of n serials.
RLX_HD int64_t cyclic_count(int64_t n, int rank, int world, int shift) {
  const int64_t B = int64_t(1) << shift;
  const int64_t nblk = (n + B - 1) / B;
  if (rank >= nblk) return 0;
  const int64_t owned = (nblk - rank + world - 1) / world;
  int64_t cnt = owned * B;
  if ((nblk - 1) % world == rank && (n % B)) cnt -= B - n % B;
  return cnt;
}

// Decoded candidate.
struct Cand {
  int cls;       // 0 multiplex, 1 merge, 2 exclusive (= priority)
  int a, b, alloc;
  int target;    // dense worker index (merge)
  int k;         // members
  uint16_t m[kMaxMembers];
};

RLX_HD uint64_t binom_at(const uint64_t* binom, int n, int k) {
  if (k < 0 || n < 0 || k > n) return 0;
  return binom[n * kBinomK + k];
}

// Serial -> candidate (enumerate_actions order: multiplex, merges, exclusives).
RLX_HD bool decode_serial(const DevPlan& P, int64_t s, Cand& c) {
  if (s < 0 || s >= P.n_total) return false;
  if (s < P.n_mux) {
    int64_t lo = 0, hi = P.n_mux_pairs - 1;
    while (lo < hi) {  // last pair block with serial0 <= s
      const int64_t mid = (lo + hi + 1) >> 1;
      if (P.mux_pairs[mid].serial0 <= s) lo = mid; else hi = mid - 1;
    }
    const MuxPair& B = P.mux_pairs[lo];
    int r = (int)(s - B.serial0);
    const bool o = r >= 3 * B.na;
    if (o) r -= 3 * B.na;
    const int n = o ? B.nb : B.na;
    c.cls = 0;
    c.a = o ? B.b : B.a;
    c.b = o ? B.a : B.b;
    c.alloc = 1 + (r / n) * 4 + r % n;
    c.k = 0;
    return true;
  }
  s -= P.n_mux;
  if (s >= P.n_merge) {
    s -= P.n_merge;
    c.cls = 2;
    c.a = P.excl[s];
    c.alloc = 0;
    c.k = 0;
    return true;
  }
  s += P.n_mux;
  int lo = 0, hi = P.n_blocks - 1;
  while (lo < hi) {  // last block with serial0 <= s
    int mid = (lo + hi + 1) >> 1;
    if (P.blocks[mid].serial0 <= s) lo = mid; else hi = mid - 1;
  }
  const MergeBlock& B = P.blocks[lo];
  int64_t local = s - B.serial0;
  int k = B.size;
  int64_t combo = local / k;
  int tgt = (int)(local % k);
  c.cls = 1;
  c.k = k;
  int idx[kMaxMembers];
  if (B.expl_off >= 0) {
    for (int i = 0; i < k; i++) idx[i] = P.combos[B.expl_off + combo * k + i];
  } else {
    int n = B.n_frags;
    uint64_t r = (uint64_t)combo;
    int x = 0;
    for (int i = 0; i < k; i++) {
      for (;;) {
        uint64_t cnt = binom_at(P.binom, n - x - 1, k - i - 1);
        if (r < cnt) break;
        r -= cnt;
        x++;
      }
      idx[i] = x++;
    }
  }
  int ws[kMaxMembers];
  for (int i = 0; i < k; i++) {
    c.m[i] = P.frags[B.frag_off + idx[i]];
    int w = P.worker[c.m[i]];
    int j = i;
    while (j > 0 && ws[j - 1] > w) { ws[j] = ws[j - 1]; j--; }
    ws[j] = w;
  }
  c.target = ws[tgt];
  c.a = c.b = -1;
  c.alloc = 0;
  return true;
}

}  // namespace rlx

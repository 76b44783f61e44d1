// rlx_hostplan.hpp — host-side plan container (see rlx_plan.cpp).
#pragma once
#include <cuda_runtime.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/rlx.h"
#include "rlx_plan.hpp"

namespace rlx {

struct Blob {
  std::vector<uint8_t> buf;
  size_t put(const void* p, size_t bytes) {
    size_t off = (buf.size() + 15) & ~size_t(15);
    buf.resize(off + bytes);
    if (bytes && p) memcpy(buf.data() + off, p, bytes);
    return off;
  }
  template <class T>
  size_t putv(const std::vector<T>& v) { return put(v.data(), v.size() * sizeof(T)); }
};

// Offsets of every DevPlan pointer inside the blob; relocated by the ABI.
struct PlanLayout {
  size_t kind, pipe, worker, flags, dur, mem, mprefix, suffix, msx, migc, rem, act, name_rank, lt_merge, id_off,
      ids, pos, tw_slot, tw_node, succ_off, succ, pend0, ord, ord_cnt, mask0, nmem0, mnode0, mpart0, mrate0, mpre0,
      mwork0, worker_ids, tw_end0, grant0, pipe_rank, latency, latency_ok, has_spec, lut, alloc_mem, mux_pairs,
      excl, blocks, frags, combos, binom, ctr_idx, ctr0, pt_off, ptab, rec, rlut;
  size_t hot_end;
};

struct HostPlan {
  DevPlan dp;            // sizes/scalars filled; pointers relocated later
  PlanLayout lay;
  Blob blob;
  std::vector<int> l2g;  // local -> state node index
  std::vector<int> g2l;
  // host copies for decoding
  std::vector<uint16_t> excl, frags, combos;
  std::vector<MuxPair> mux_pairs;
  std::vector<MergeBlock> blocks;
  std::vector<uint64_t> binom;
  std::vector<uint16_t> worker_of;  // [NL]
  int64_t n_tw_window = 0;
};

int build_plan(const RlxInstanceDesc* in, const RlxStateDesc* sd, int rounds, int max_merge, HostPlan& hp,
               std::string& err);
void relocate(HostPlan& hp, const uint8_t* base, DevPlan& d);
int check_capacity(const HostPlan& hp, std::string& err);

void choose_shape(int W, int& G, int& WPL);
size_t plan_slice_bytes(const DevPlan& P, int G, int WPL);  // one group's slice

// rlx_kernels.cu
int launch_score(const DevPlan& P, WorkDesc wd, SliceOut* outs, int max_slices, int sm_count, cudaStream_t st,
                 int* n_slices_out, int threads_hint);
int launch_reduce(const SliceOut* outs, int n, unsigned long long* res, cudaStream_t st);

}  // namespace rlx

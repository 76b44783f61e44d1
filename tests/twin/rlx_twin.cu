// rlx_twin.cu — host (single-lane) build of the product's scoring code.
//
// TEST INFRASTRUCTURE / DEBUGGING TWIN ONLY: compiled into
// tests/twin/_build/librlx_twin.so, never into librlx.so and never on the
// product path. It runs the exact group algorithm of rlx_kernels.cu with
// G = 1 lane so that a device result can be reproduced and inspected on a
// CPU (warp primitives resolve to host shims).
#include <stdio.h>

#include <string>
#include <vector>

#include "../../paper_2604_23838_b200/csrc/rlx_kernels.cu"
#include "../../paper_2604_23838_b200/csrc/rlx_hostplan.hpp"

namespace rlx {
const DevPlan* g_twin_plan = nullptr;
uint8_t* g_twin_smem = nullptr;
}

using namespace rlx;

extern "C" int rlx_twin_decide(const RlxInstanceDesc* in, const RlxStateDesc* sd, int window, int max_merge,
                               int64_t b, int64_t e, double* keys_out, int64_t* n_out, uint64_t* key_out,
                               double* dbg_out, char* err, int errlen) {
  HostPlan hp;
  std::string es;
  int rc = build_plan(in, sd, window, max_merge, hp, es);
  if (rc) {
    snprintf(err, errlen, "%s", es.c_str());
    return rc;
  }
  DevPlan dp;
  relocate(hp, hp.blob.buf.data(), dp);
  g_twin_plan = &dp;
  *n_out = dp.n_total;
  if (getenv("RLX_TWIN_INFO")) fprintf(stderr, "plan: NL %d NWIN %d W %d NC %d same_order %d hot %u\n", dp.NL, dp.NWIN, dp.W, dp.NC, dp.same_order, dp.hot_bytes);
  if (e < 0 || e > dp.n_total) e = dp.n_total;
  if (b < 0) b = 0;
  if (b > e) b = e;
  WorkDesc wd;
  memset(&wd, 0, sizeof wd);
  auto clip = [&](int64_t lo, int64_t hi, int64_t& s, int64_t& n) {
    int64_t x = lo > b ? lo : b, y = hi < e ? hi : e;
    s = x;
    n = y > x ? y - x : 0;
  };
  clip(dp.n_mux, dp.n_mux + dp.n_merge, wd.a0, wd.na);
  clip(0, dp.n_mux, wd.b0, wd.nb);
  clip(dp.n_mux + dp.n_merge, dp.n_total, wd.c0, wd.nc);
  wd.shard0 = b;
  unsigned long long counter = 0, err_key = ~0ull;
  wd.counter = &counter;
  wd.err_key = &err_key;
  wd.keys_out = keys_out;
  if (dp.W > 32) {
    snprintf(err, errlen, "the host twin runs one lane: at most 32 workers (NL %d NT %d NC %d hot %u max_ord %d NTW %d)",
             dp.NL, dp.NT, dp.NC, dp.hot_bytes, dp.max_ord, dp.NTW);
    return RLX_ERR_LIMIT;
  }
  group_layout(dp, 1, 32);
  std::vector<double> smem((dp.hot_bytes + dp.g_bytes) / 8 + 16);
  memcpy(smem.data(), dp.hot, dp.hot_bytes);  // the kernel stages the hot region the same way
  g_twin_smem = (uint8_t*)smem.data();
  wd.slice_bytes = (int)dp.g_bytes;
  SliceOut out;
  memset(&out, 0, sizeof out);
  group_loop<1, 32>(wd, dp.hot_bytes, 0, 1u, &out);
  key_out[0] = out.k0;
  key_out[1] = out.k1;
  key_out[2] = out.k2;
  key_out[3] = out.passes;
  if (dbg_out) {
    dbg_out[0] = err_key == ~0ull ? -1.0 : (double)(err_key >> 8);
    dbg_out[1] = err_key == ~0ull ? 0.0 : (double)(err_key & 0xff);
  }
  if (err_key != ~0ull) {
    snprintf(err, errlen, "candidate %llu failed with device code %llu", err_key >> 8, err_key & 0xff);
    return (err_key & 0xff) == RLX_ERR_SCHEDULING ? RLX_ERR_SCHEDULING : RLX_ERR_KEY;
  }
  return 0;
}

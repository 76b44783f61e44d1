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
  const int64_t lo[3] = {dp.n_mux, 0, dp.n_mux + dp.n_merge};
  const int64_t hi[3] = {dp.n_mux + dp.n_merge, dp.n_mux, dp.n_total};
  wd.world = 1;
  for (int c = 0; c < 3; c++) {
    const int64_t x = lo[c] > b ? lo[c] : b, y = hi[c] < e ? hi[c] : e;
    wd.s0[c] = x;
    wd.loc[c] = y > x ? y - x : 0;
  }
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
  // `ngw` one-lane groups share one warp slice and run interleaved, one
  // iteration each in turn — the device's per-warp candidate queue with its
  // claim / drain / finalise / fetch protocol, deterministically on a CPU
  const int ngw = getenv("RLX_TWIN_GROUPS") ? atoi(getenv("RLX_TWIN_GROUPS")) : 4;
  group_layout(dp, 1, 32);
  const size_t bytes = dp.hot_bytes + dp.w_bytes + (size_t)ngw * dp.g_bytes;
  std::vector<double> smem(bytes / 8 + 16);
  memcpy(smem.data(), dp.hot, dp.hot_bytes);  // the kernel stages the hot region the same way
  g_twin_smem = (uint8_t*)smem.data();
  wd.slice_bytes = (int)dp.g_bytes;
  const uint32_t wbase = dp.hot_bytes;
  WarpCand* wc = reinterpret_cast<WarpCand*>(g_twin_smem + wbase);
  wc->gen = 0;
  fetch_candidate(wd, wc);
  std::vector<GroupRunner<1, 32>*> rs;
  for (int i = 0; i < ngw; i++) {
    rs.push_back(new GroupRunner<1, 32>(wd, wbase + dp.w_bytes + (uint32_t)i * dp.g_bytes, wbase, 0, 1u, ngw));
    rs.back()->init();
  }
  std::vector<bool> live(ngw, true);
  for (int n_live = ngw; n_live > 0;) {
    for (int i = 0; i < ngw; i++)
      if (live[i] && !rs[i]->iter()) {
        live[i] = false;
        n_live--;
      }
  }
  SliceOut out;
  memset(&out, 0, sizeof out);
  for (int i = 0; i < ngw; i++) {
    SliceOut o;
    memset(&o, 0, sizeof o);
    rs[i]->finish(&o);
    if (key_less(o.k0, o.k1, o.k2, out.k0 ? out.k0 : ~0ull, out.k0 ? out.k1 : ~0ull, out.k0 ? out.k2 : ~0ull)) {
      out.k0 = o.k0;
      out.k1 = o.k1;
      out.k2 = o.k2;
    }
    out.passes += o.passes;
    delete rs[i];
  }
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

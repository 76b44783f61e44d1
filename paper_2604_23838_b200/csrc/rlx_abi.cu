// rlx_abi.cu — the C-ABI of include/rlx.h.
//
// One handle per GPU. rlx_decide = host plan (rlx_plan.cpp) -> one H2D copy
// of the plan blob -> persistent scoring kernel over the requested serial
// shard -> deterministic reduce -> 7-word result D2H. The packed shard key
// can also be left in device memory (dev_key_out) for the cross-GPU
// lexicographic min-loc collective.
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <chrono>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rlx.h"
#include "rlx_hostplan.hpp"
#include "rlx_state.hpp"


using namespace rlx;

namespace {

constexpr int kMaxSlices = 1 << 17;
constexpr int kShardBlockShift = 5;  // multi-GPU shards interleave blocks of 32 serials per class
constexpr size_t kSliceOutBytes = 56;
static_assert(sizeof(rlx::SliceOut) == kSliceOutBytes, "SliceOut layout");

struct Handle {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;      // stream every call is issued on
  cudaStream_t own_stream = nullptr;  // the handle's private stream (default)
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;
  std::string err;
  // owned instance copy
  bool loaded = false;
  RlxInstanceDesc inst{};
  std::string pipe_names;
  std::vector<int32_t> pipe_name_off, worker_ids;
  std::vector<double> latency, params, peak, mfu, lut, alloc_sm, alloc_mem;
  std::vector<uint8_t> latency_ok, has_spec;
  // plan
  HostPlan hp;
  bool have_plan = false;      // hp holds the plan of the last decide
  bool plan_on_device = false; // ... and d_blob holds its copy
  DevPlan host_view{};
  // device buffers
  uint8_t* d_blob = nullptr;
  size_t blob_cap = 0;
  uint8_t* h_pin = nullptr;
  size_t pin_cap = 0;
  uint8_t* d_outs = nullptr;
  unsigned long long* d_counter = nullptr;
  unsigned long long* d_errkey = nullptr;
  unsigned long long* d_res = nullptr;
  unsigned long long* h_res = nullptr;
  double* d_keys = nullptr;
  size_t keys_cap = 0;
  int threads_hint = 0;
};



int fail(Handle* h, int code, const std::string& msg) {
  h->err = msg;
  return code;
}

int cuda_fail(Handle* h, cudaError_t e, const char* where) {
  h->err = std::string(where) + ": " + cudaGetErrorString(e);
  return RLX_ERR_CUDA;
}

// The scoring kernel reads its plan from one __constant__ symbol per device
// (rlx_kernels.cu), so two handles on the same device must not interleave
// "copy plan -> launch -> wait" sequences: one lock per device orders them.
std::mutex g_device_lock[64];

const char* kind_name(int k) {
  static const char* names[RLX_NKIND] = {"PrefillBurst", "DecodeLarge", "DecodeMedium", "DecodeSmall",
                                         "Reference",    "Training",    "ToolWait"};
  return k >= 0 && k < RLX_NKIND ? names[k] : "?";
}

// Device error code (rlx_kernels.cu kErr*) -> status + the reference's text.
int device_error_text(int code, std::string& msg) {
  if (code == RLX_ERR_SCHEDULING) {
    msg = "window estimate did not converge";  // :867
    return RLX_ERR_SCHEDULING;
  }
  if (code >= 8 && code < 16) {  // latency_model[bucket]
    msg = std::to_string(code - 8);
    return RLX_ERR_KEY;
  }
  if (code >= 16) {
    const int k = (code - 16) / RLX_NPARTNER, p = (code - 16) % RLX_NPARTNER - 1;
    msg = std::string("slowdown table has no rows for pair ") + kind_name(k) + "/" +
          (p < 0 ? "-" : kind_name(p));  // slowdown.py:143-147
    return RLX_ERR_KEY;
  }
  msg = "device error " + std::to_string(code);
  return RLX_ERR_CUDA;
}

int device_error(Handle* h, int code) {
  std::string m;
  const int st = device_error_text(code, m);
  return fail(h, st, m);
}

#define CK(x)                                   \
  do {                                          \
    cudaError_t _e = (x);                       \
    if (_e != cudaSuccess) return cuda_fail(h, _e, #x); \
  } while (0)

}  // namespace

extern "C" {

int rlx_abi_version(void) { return RLX_ABI_VERSION; }

int rlx_open(int device, void** handle) {
  if (!handle) return RLX_ERR_ARG;
  *handle = nullptr;
  Handle* h = new Handle();
  h->device = device;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev <= device || device < 0) {
    delete h;
    return RLX_ERR_CUDA;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    delete h;
    return RLX_ERR_CUDA;
  }
  cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&h->e0) != cudaSuccess || cudaEventCreate(&h->e1) != cudaSuccess ||
      cudaEventCreate(&h->e2) != cudaSuccess ||
      cudaMalloc(&h->d_outs, kSliceOutBytes * kMaxSlices) != cudaSuccess ||
      cudaMalloc(&h->d_counter, 64) != cudaSuccess || cudaMalloc(&h->d_errkey, 64) != cudaSuccess ||
      cudaMalloc(&h->d_res, 128) != cudaSuccess || cudaMallocHost(&h->h_res, 128) != cudaSuccess) {
    delete h;
    return RLX_ERR_CUDA;
  }
  h->stream = h->own_stream;
  const char* th = getenv("RLX_THREADS");
  if (th) h->threads_hint = atoi(th);
  *handle = h;
  return RLX_OK;
}

int rlx_load_instance(void* handle, const RlxInstanceDesc* in) {
  Handle* h = (Handle*)handle;
  if (!h || !in) return RLX_ERR_ARG;
  if (in->abi_version != RLX_ABI_VERSION) return fail(h, RLX_ERR_ARG, "ABI version mismatch");
  const int P = in->n_pipes, W = in->n_workers;
  if (P <= 0 || W <= 0) return fail(h, RLX_ERR_ARG, "empty instance");
  size_t names_len = 0;
  for (int p = 0; p < P; p++) {
    size_t e = in->pipe_name_off[p] + strlen(in->pipe_names + in->pipe_name_off[p]) + 1;
    if (e > names_len) names_len = e;
  }
  h->pipe_names.assign(in->pipe_names, names_len);
  h->pipe_name_off.assign(in->pipe_name_off, in->pipe_name_off + P);
  h->latency.assign(in->latency, in->latency + 3 * P);
  h->latency_ok.assign(in->latency_ok, in->latency_ok + 3 * P);
  h->has_spec.assign(in->has_spec, in->has_spec + P);
  h->params.assign(in->model_params, in->model_params + P);
  h->peak.assign(in->peak_flops, in->peak_flops + P);
  h->mfu.assign(in->prefill_mfu, in->prefill_mfu + P);
  h->worker_ids.assign(in->worker_ids, in->worker_ids + W);
  h->lut.assign(in->lut, in->lut + RLX_NKIND * RLX_NPARTNER * RLX_NALLOC);
  h->alloc_sm.assign(in->alloc_sm, in->alloc_sm + RLX_NALLOC);
  h->alloc_mem.assign(in->alloc_mem, in->alloc_mem + RLX_NALLOC);
  for (int p = 0; p < P; p++)
    if (h->has_spec[p] && !(h->mfu[p] > 0)) return fail(h, RLX_ERR_VALUE, "prefill_mfu must be positive");
  RlxInstanceDesc& d = h->inst;
  d = *in;
  d.pipe_names = h->pipe_names.data();
  d.pipe_name_off = h->pipe_name_off.data();
  d.latency = h->latency.data();
  d.latency_ok = h->latency_ok.data();
  d.has_spec = h->has_spec.data();
  d.model_params = h->params.data();
  d.peak_flops = h->peak.data();
  d.prefill_mfu = h->mfu.data();
  d.worker_ids = h->worker_ids.data();
  d.lut = h->lut.data();
  d.alloc_sm = h->alloc_sm.data();
  d.alloc_mem = h->alloc_mem.data();
  h->loaded = true;
  h->have_plan = false;
  h->plan_on_device = false;
  return RLX_OK;
}

static void fill_action(Handle* h, const Cand& c, RlxAction* out) {
  memset(out, 0, sizeof *out);
  out->cls = c.cls;
  const std::vector<int>& l2g = h->hp.l2g;
  if (c.cls == RLX_CLASS_MERGE) {
    out->n_members = c.k;
    for (int i = 0; i < c.k; i++) out->members[i] = l2g[c.m[i]];
    out->target_worker = c.target;
    out->node_a = out->node_b = -1;
  } else {
    out->node_a = l2g[c.a];
    out->node_b = c.cls == RLX_CLASS_MULTIPLEX ? l2g[c.b] : -1;
    out->alloc = c.alloc;
  }
}

static int decide_impl(Handle* h, const RlxStateDesc* sd, const RlxDecideArgs* args, RlxDecision* out) {
  if (!h->loaded) return fail(h, RLX_ERR_ARG, "no instance loaded");
  if (args->window < 1) return fail(h, RLX_ERR_VALUE, "window must be >= 1");
  const bool reuse = (args->flags & RLX_F_REUSE_PLAN) != 0;
  if (reuse && !h->have_plan) return fail(h, RLX_ERR_ARG, "RLX_F_REUSE_PLAN needs a preceding rlx_decide");
  if (!reuse && !sd) return RLX_ERR_ARG;
  memset(out, 0, sizeof *out);
  out->serial = -1;
  out->err_key = -1;
  CK(cudaSetDevice(h->device));
  auto t0 = std::chrono::steady_clock::now();
  int rc = 0;
  if (!reuse) {
    h->have_plan = false;
    h->plan_on_device = false;
    rc = build_plan(&h->inst, sd, args->window, args->max_merge, h->hp, h->err);
    if (rc) return rc;
    h->have_plan = true;
    relocate(h->hp, h->hp.blob.buf.data(), h->host_view);
  }
  const DevPlan& hv = h->host_view;
  out->n_candidates = hv.n_total;
  out->n_merge = hv.n_merge;
  out->n_multiplex = hv.n_mux;
  out->n_exclusive = hv.n_excl;
  // ---- work ranges per class: merges first (heaviest), then multiplex, then exclusive
  WorkDesc wd;
  memset(&wd, 0, sizeof wd);
  const int64_t lo[3] = {hv.n_mux, 0, hv.n_mux + hv.n_merge};
  const int64_t hi[3] = {hv.n_mux + hv.n_merge, hv.n_mux, hv.n_total};
  int64_t b = args->serial_begin < 0 ? 0 : args->serial_begin;
  int64_t e = args->serial_end < 0 ? hv.n_total : args->serial_end;
  wd.world = 1;
  if (args->flags & RLX_F_SHARD) {
    // cost-balanced part `serial_begin` of `serial_end`: every world-th block
    // of kShardBlock serials of each class (dist.py)
    const int64_t r = args->serial_begin, w = args->serial_end;
    if (w < 1 || r < 0 || r >= w) return fail(h, RLX_ERR_ARG, "bad shard index / count");
    if (args->keys_out) return fail(h, RLX_ERR_ARG, "keys_out needs an explicit serial range");
    wd.world = (int)w;
    wd.rank = (int)r;
    wd.blk_shift = kShardBlockShift;
    for (int c = 0; c < 3; c++) {
      wd.s0[c] = lo[c];
      wd.loc[c] = cyclic_count(hi[c] - lo[c], wd.rank, wd.world, wd.blk_shift);
    }
    b = 0;
    e = hv.n_total;
  } else {
    if (e > hv.n_total) e = hv.n_total;
    if (b > e) b = e;
    for (int c = 0; c < 3; c++) {
      const int64_t x = lo[c] > b ? lo[c] : b, y = hi[c] < e ? hi[c] : e;
      wd.s0[c] = x;
      wd.loc[c] = y > x ? y - x : 0;
    }
  }
  out->shard_begin = b;
  out->shard_end = e;
  auto t1 = std::chrono::steady_clock::now();
  out->plan_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  if (wd.loc[0] + wd.loc[1] + wd.loc[2] == 0) {
    if (args->dev_key_out) {
      CK(cudaMemsetAsync(args->dev_key_out, 0xFF, 24, h->stream));
      CK(cudaMemsetAsync((uint8_t*)args->dev_key_out + 24, 0, 8, h->stream));
      CK(cudaMemsetAsync((uint8_t*)args->dev_key_out + 32, 0xFF, 8, h->stream));
      CK(cudaStreamSynchronize(h->stream));
    }
    out->err_key = -1;
    return RLX_OK;
  }
  // ---- upload plan (skipped when re-scoring the resident plan)
  size_t nb = h->hp.blob.buf.size();
  CK(cudaEventRecord(h->e2, h->stream));
  if (h->plan_on_device) {
    nb = 0;
  } else if (nb > h->pin_cap) {
    if (h->h_pin) cudaFreeHost(h->h_pin);
    h->pin_cap = nb * 2;
    CK(cudaMallocHost(&h->h_pin, h->pin_cap));
  }
  if (nb > h->blob_cap) {
    if (h->d_blob) cudaFree(h->d_blob);
    h->blob_cap = nb * 2;
    CK(cudaMalloc(&h->d_blob, h->blob_cap));
  }
  if (nb) {
    // the previous decision's kernel may still read d_blob / h_pin on this stream
    CK(cudaStreamSynchronize(h->stream));
    memcpy(h->h_pin, h->hp.blob.buf.data(), nb);
    CK(cudaMemcpyAsync(h->d_blob, h->h_pin, nb, cudaMemcpyHostToDevice, h->stream));
    h->plan_on_device = true;
  }
  out->h2d_bytes = (int64_t)nb;
  DevPlan dp;
  relocate(h->hp, h->d_blob, dp);
  wd.shard0 = b;
  wd.counter = h->d_counter;
  wd.err_key = h->d_errkey;
  if (args->keys_out) {
    size_t need = sizeof(double) * 2 * (size_t)(e - b);
    if (need > h->keys_cap) {
      if (h->d_keys) cudaFree(h->d_keys);
      h->keys_cap = need;
      CK(cudaMalloc(&h->d_keys, need));
    }
    wd.keys_out = h->d_keys;
  }
  CK(cudaMemsetAsync(h->d_counter, 0, 8, h->stream));
  CK(cudaMemsetAsync(h->d_errkey, 0xFF, 8, h->stream));
  int n_slices = 0;
  std::lock_guard<std::mutex> lock(g_device_lock[h->device & 63]);
  CK(cudaEventRecord(h->e0, h->stream));
  rc = launch_score(dp, wd, (SliceOut*)h->d_outs, kMaxSlices, h->sm_count, h->stream, &n_slices, h->threads_hint);
  if (rc)
    return fail(h, rc, rc == RLX_ERR_LIMIT ? "no kernel shape for this worker count, or the plan does not fit in shared memory"
                                          : "kernel launch failed");
  CK(cudaEventRecord(h->e1, h->stream));
  rc = launch_reduce((SliceOut*)h->d_outs, n_slices, h->d_res, h->stream);
  if (rc) return fail(h, rc, "reduce launch failed");
  if (args->dev_key_out) {
    CK(cudaMemcpyAsync(args->dev_key_out, h->d_res, 32, cudaMemcpyDeviceToDevice, h->stream));
    CK(cudaMemcpyAsync((uint8_t*)args->dev_key_out + 32, h->d_errkey, 8, cudaMemcpyDeviceToDevice, h->stream));
  }
  CK(cudaMemcpyAsync(h->h_res, h->d_res, 64, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaMemcpyAsync(&h->h_res[8], h->d_errkey, 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  const unsigned long long ek = h->h_res[8];
  out->err_key = ek == ~0ull ? -1 : (int64_t)ek;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, h->e0, h->e1);
  out->kernel_ms = ms;
  cudaEventElapsedTime(&ms, h->e2, h->e1);
  out->device_ms = ms;
  out->d2h_bytes = 72;
  if (ek != ~0ull) {  // the lowest failing serial of the shard: the candidate the reference raises on
    out->serial = (int64_t)(ek >> 8);
    return device_error(h, (int)(ek & 0xff));
  }
  unsigned long long* r = h->h_res;
  out->key.cost_bits = r[0];
  out->key.finish_bits = r[1];
  out->key.prio_serial = r[2];
  out->key.valid = r[3];
  out->passes = (int64_t)r[4];
  out->events = (int64_t)r[7];
  double by;
  memcpy(&by, &r[5], 8);
  out->alg_bytes = by;
  if (r[3]) {
    out->found = 1;
    memcpy(&out->cost, &r[0], 8);
    memcpy(&out->finish, &r[1], 8);
    out->priority = (int)(r[2] >> 61);
    out->serial = (int64_t)(r[2] & ((1ull << 61) - 1));
    Cand c;
    decode_serial(hv, out->serial, c);
    fill_action(h, c, &out->action);
  }
  if (args->keys_out)
    CK(cudaMemcpy(args->keys_out, h->d_keys, sizeof(double) * 2 * (size_t)(e - b), cudaMemcpyDeviceToHost));
  return RLX_OK;
}

int rlx_decide(void* handle, const RlxStateDesc* sd, const RlxDecideArgs* args, RlxDecision* out) {
  Handle* h = (Handle*)handle;
  if (!h || !args || !out) return RLX_ERR_ARG;
  return decide_impl(h, sd, args, out);
}

int rlx_drive(void* handle, void* state, const RlxDriveArgs* args, RlxStep* steps, int64_t* n_steps,
              int64_t* n_decisions) {
  Handle* h = (Handle*)handle;
  ExecSoA* s = (ExecSoA*)state;
  if (!h || !s || !args || !n_steps || !n_decisions || (args->max_steps > 0 && !steps)) return RLX_ERR_ARG;
  *n_steps = 0;
  *n_decisions = 0;
  RlxDecideArgs da;
  memset(&da, 0, sizeof da);
  da.window = args->window;
  da.max_merge = args->max_merge;
  da.serial_begin = 0;
  da.serial_end = -1;
  const RlxInstanceDesc& in = h->inst;
  auto alive_done = [&]() { return s->n_done == (int)s->order.size(); };
  while (!alive_done()) {
    for (;;) {  // decisions at this instant (scheduler.py:938-944)
      if (args->max_decisions > 0 && *n_decisions >= args->max_decisions) return RLX_OK;
      auto t0 = std::chrono::steady_clock::now();
      RlxStateDesc sd;
      s->snapshot(&sd);
      RlxDecision d;
      int rc = decide_impl(h, &sd, &da, &d);
      if (rc) return rc;
      if (d.n_candidates == 0) break;
      (*n_decisions)++;
      // winner (snapshot indices) -> state indices + LUT rates
      RlxApply ap;
      memset(&ap, 0, sizeof ap);
      RlxAction act = d.action;
      ap.cls = act.cls;
      auto sidx = [&](int i) { return s->order[i]; };
      auto lut = [&](int k, int partner, int alloc) {
        return in.lut[(k * RLX_NPARTNER + partner + 1) * RLX_NALLOC + alloc];
      };
      if (act.cls == RLX_CLASS_MERGE) {
        ap.n_members = act.n_members;
        for (int i = 0; i < act.n_members; i++) ap.members[i] = act.members[i] = sidx(act.members[i]);
        ap.target_worker = act.target_worker;
      } else if (act.cls == RLX_CLASS_EXCLUSIVE) {
        ap.node_a = act.node_a = sidx(act.node_a);
        ap.rate_a = lut(s->nodes[ap.node_a].kind, -1, 0);
        ap.sm_a = in.alloc_sm[0];
        ap.mem_a = in.alloc_mem[0];
      } else {
        ap.node_a = act.node_a = sidx(act.node_a);
        ap.node_b = act.node_b = sidx(act.node_b);
        const int ka = s->nodes[ap.node_a].kind, kb = s->nodes[ap.node_b].kind;
        ap.rate_a = lut(ka, kb, act.alloc);
        ap.rate_b = lut(kb, ka, act.alloc + 12);
        ap.sm_a = in.alloc_sm[act.alloc];
        ap.mem_a = in.alloc_mem[act.alloc];
        ap.sm_b = in.alloc_sm[act.alloc + 12];
        ap.mem_b = in.alloc_mem[act.alloc + 12];
      }
      const double start = s->now;
      rc = s->apply(&ap);
      if (rc) return fail(h, rc, s->err);
      if (*n_steps >= args->max_steps) return fail(h, RLX_ERR_LIMIT, "rlx_drive: steps array is full");
      RlxStep& st = steps[(*n_steps)++];
      memset(&st, 0, sizeof st);
      st.start = start;
      st.action = act;
      st.cost = d.cost;
      st.finish = d.finish;
      st.priority = d.priority;
      st.serial = d.serial;
      st.n_candidates = d.n_candidates;
      st.kernel_ms = d.kernel_ms;
      st.decision_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    if (alive_done()) break;
    if (s->run_order.empty() && s->tw_order.empty())
      return fail(h, RLX_ERR_SCHEDULING, "lookahead: stalled with no running work");  // :948
    int rc = s->advance(false, 0.0);
    if (rc) return fail(h, rc, s->err);
  }
  return RLX_OK;
}

int rlx_plan_info(const RlxInstanceDesc* in, const RlxStateDesc* sd, int32_t window, int32_t max_merge,
                  RlxPlanInfo* out, char* err, int32_t err_len) {
  if (!in || !sd || !out) return RLX_ERR_ARG;
  memset(out, 0, sizeof *out);
  HostPlan hp;
  std::string e;
  int rc = window < 1 ? RLX_ERR_VALUE : build_plan(in, sd, window, max_merge, hp, e);
  if (window < 1) e = "window must be >= 1";
  if (!rc) {
    const DevPlan& d = hp.dp;
    out->n_candidates = d.n_total;
    out->n_multiplex = d.n_mux;
    out->n_merge = d.n_merge;
    out->n_exclusive = d.n_excl;
    out->window_nodes = d.NWIN;
    out->local_nodes = d.NL;
    out->max_worker_order = d.max_ord;
    out->hot_bytes = (int32_t)hp.lay.hot_end;
    out->blob_bytes = (int64_t)hp.blob.buf.size();
    rc = check_capacity(hp, e);
  }
  if (err && err_len > 0) {
    strncpy(err, e.c_str(), err_len - 1);
    err[err_len - 1] = 0;
  }
  return rc;
}

int rlx_set_stream(void* handle, void* stream) {
  Handle* h = (Handle*)handle;
  if (!h) return RLX_ERR_ARG;
  h->stream = stream ? (cudaStream_t)stream : h->own_stream;
  return RLX_OK;
}

int rlx_decode(void* handle, int64_t serial, RlxAction* out) {
  Handle* h = (Handle*)handle;
  if (!h || !out) return RLX_ERR_ARG;
  if (!h->have_plan) return fail(h, RLX_ERR_ARG, "rlx_decode needs a preceding rlx_decide on the same state");
  Cand c;
  if (!decode_serial(h->host_view, serial, c)) return fail(h, RLX_ERR_ARG, "serial out of range");
  fill_action(h, c, out);
  return RLX_OK;
}

int rlx_error_text(int32_t device_code, char* buf, int32_t buf_len) {
  std::string m;
  const int st = device_error_text(device_code, m);
  if (buf && buf_len > 0) snprintf(buf, (size_t)buf_len, "%s", m.c_str());
  return st;
}

const char* rlx_last_error(void* handle) {
  Handle* h = (Handle*)handle;
  return h ? h->err.c_str() : "null handle";
}

void rlx_close(void* handle) {
  Handle* h = (Handle*)handle;
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->d_blob) cudaFree(h->d_blob);
  if (h->h_pin) cudaFreeHost(h->h_pin);
  if (h->d_outs) cudaFree(h->d_outs);
  if (h->d_counter) cudaFree(h->d_counter);
  if (h->d_errkey) cudaFree(h->d_errkey);
  if (h->d_res) cudaFree(h->d_res);
  if (h->h_res) cudaFreeHost(h->h_res);
  if (h->d_keys) cudaFree(h->d_keys);
  if (h->e0) cudaEventDestroy(h->e0);
  if (h->e1) cudaEventDestroy(h->e1);
  if (h->e2) cudaEventDestroy(h->e2);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  delete h;
}

}  // extern "C"

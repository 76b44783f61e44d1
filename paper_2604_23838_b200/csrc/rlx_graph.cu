// rlx_graph.cu — Sub-Stage Graph construction from per-rollout length tables
// on the GPU.
//
// The reference builds each pipeline's graph in pure Python: a per-worker
// cohort replay of the sample batch (rlmux/workload.py:275-340
// `_replay_worker`, run three times per worker by expand_to_trace /
// expand_with_enrichment) produces one ForwardStepRecord per decode step,
// and `construct_graph` (rlmux/graph.py:206-403) splits each worker's record
// list into tool-wait runs and bucket-stable spans (`_segment_records`,
// `_segment_span`, stability window L_s) that become rollout sub-stages.
// At config 5 (8 pipelines x 64 workers x 128 samples) that is ~90 s.
//
// Here every (pipeline, worker) cohort is independent:
//  * rlx_replay_kernel — one warp per cohort, lanes over its samples. One
//    loop iteration is one forward step: wake-ups (t <= now + 1e-12), the
//    active set (ballot), pending prefill injection, the step record
//    (prefill tokens, active requests, context total; warp reductions), the
//    step latency of the record's token bucket (now += latency[bucket], in
//    the reference's order), then every active sample decodes one token and
//    moves to its next turn / tool wait / done. Run once to count steps per
//    cohort, once more to write the records at their prefix-summed offsets.
//  * rlx_segment_kernel — one thread per cohort walks its records with the
//    reference's segmentation state machine and writes finished segments
//    with their kind, duration and token sums.
// The host (graphgen.py) turns segments into SubStage rows and adds the
// Reference / Training barrier nodes.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/rlx.h"

namespace rlx {
namespace {

struct Cohort {  // one (pipeline, worker) replay
  int32_t pipe, worker;
  int32_t s0, n;          // samples [s0, s0 + n) of the flattened, cohort-sorted sample arrays
  int64_t rec_off;        // first record (pass 2)
};

__device__ __forceinline__ int bucket_of(int64_t tokens, const int32_t* bounds, int nb) {
  int b = 0;  // bucketize (graph.py:59-66): the bucket whose [lower, upper) holds tokens
  for (int i = 1; i < nb; i++)
    if (tokens >= bounds[i]) b = i;
  return b;
}

__device__ __forceinline__ long long warp_sum64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Per-sample replay state lives in global memory (coalesced: lane l holds
// samples l, l + 32, ... of its cohort).
struct SampleState {
  int32_t* turn;        // current turn index
  int64_t* remaining;   // decode tokens left in the turn
  int64_t* context;     // running context
  int64_t* pending;     // prefill to inject at the next active step
  double* wake;         // tool wake time (NaN: not waiting)
  uint8_t* done;
};

__global__ void rlx_replay_kernel(const Cohort* cohorts, int n_cohorts, const int64_t* prompt, const int32_t* turn_off,
                                  const int64_t* t_prefill, const int64_t* t_decode, const double* t_tool,
                                  const double* latency /* [P*5] */, const int32_t* bounds, int nb, SampleState st,
                                  int64_t* n_steps, int write, int64_t* r_prefill, int32_t* r_active,
                                  int64_t* r_context) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_cohorts) return;
  const Cohort C = cohorts[warp];
  const double* lat = latency + 5 * C.pipe;
  // initial state (workload.py:280-286)
  for (int i = lane; i < C.n; i += 32) {
    const int s = C.s0 + i;
    const int t0 = turn_off[s];
    st.turn[s] = 0;
    st.remaining[s] = t_decode[t0];
    st.context[s] = 0;
    st.pending[s] = prompt[s] + t_prefill[t0];
    st.wake[s] = __longlong_as_double(0x7ff8000000000000ll);
    st.done[s] = 0;
  }
  __syncwarp();
  double now = 0.0;
  int64_t step = 0;
  int n_done = 0;
  while (n_done < C.n) {
    // wake-ups, active set, prefill injection, context total (:288-312)
    int n_active = 0;
    long long pre = 0, ctx = 0;
    for (int base = 0; base < C.n; base += 32) {
      const int i = base + lane;
      bool act = false;
      if (i < C.n) {
        const int s = C.s0 + i;
        double w = st.wake[s];
        if (w == w && w <= now + 1e-12) {
          w = __longlong_as_double(0x7ff8000000000000ll);
          st.wake[s] = w;
        }
        act = !st.done[s] && !(w == w);
        if (act) {
          const int64_t p = st.pending[s];
          int64_t c = st.context[s];
          if (p > 0) {
            pre += p;
            c += p;
            st.context[s] = c;
            st.pending[s] = 0;
          }
          ctx += c;
        }
      }
      n_active += __popc(__ballot_sync(0xffffffffu, act));
    }
    if (n_active == 0) {  // every sample waits on a tool: idle marker (:296-302)
      if (write && lane == 0) {
        r_prefill[C.rec_off + step] = 0;
        r_active[C.rec_off + step] = 0;
        r_context[C.rec_off + step] = 0;
      }
      now += lat[0];
      step++;
      continue;
    }
    pre = warp_sum64(pre);
    ctx = warp_sum64(ctx);
    if (write && lane == 0) {
      r_prefill[C.rec_off + step] = pre;
      r_active[C.rec_off + step] = n_active;
      r_context[C.rec_off + step] = ctx;
    }
    now += lat[bucket_of(pre + n_active, bounds, nb)];
    // every active sample decodes one token (:315-330)
    int fin = 0;
    for (int base = 0; base < C.n; base += 32) {
      const int i = base + lane;
      if (i < C.n) {
        const int s = C.s0 + i;
        const double w = st.wake[s];
        if (!st.done[s] && !(w == w)) {
          const int64_t r = st.remaining[s] - 1;
          st.remaining[s] = r;
          st.context[s] += 1;
          if (r == 0) {
            const int t = st.turn[s];
            const int t0 = turn_off[s], nt = turn_off[s + 1] - t0;
            if (t + 1 < nt) {
              st.turn[s] = t + 1;
              st.remaining[s] = t_decode[t0 + t + 1];
              st.pending[s] = t_prefill[t0 + t + 1];
              const double tool = t_tool[t0 + t];
              if (tool > 0) st.wake[s] = now + tool;
            } else {
              st.done[s] = 1;
              fin++;
            }
          }
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) fin += __shfl_xor_sync(0xffffffffu, fin, o);
    n_done += fin;
    step++;
  }
  if (!write && lane == 0) n_steps[warp] = step;
}

// _segment_records / _segment_span (graph.py:206-269) + _rollout_kind
// (:272-282) + the per-node sums of construct_graph (:335-362), one thread
// per cohort.
struct SegOut {
  RlxSegment* seg;
  int32_t* n_seg;
};

__device__ __forceinline__ bool is_idle(const int64_t* pf, const int32_t* ac, int64_t k) {
  return pf[k] == 0 && ac[k] == 0;
}

__device__ void emit(const Cohort& C, const int64_t* pf, const int32_t* ac, const int64_t* cx, const double* lat,
                     int nb, int64_t lo, int64_t hi, int bucket, RlxSegment* out, int& n) {
  RlxSegment g;
  memset(&g, 0, sizeof g);
  g.worker = C.worker;
  g.seq = n;
  g.bucket = bucket;
  g.step_lo = lo + 1;  // step_index is 1-based
  g.step_hi = hi + 1;
  int64_t decode = 0, tokens = 0, prefill = 0;
  for (int64_t k = lo; k <= hi; k++) {
    decode += ac[k];
    prefill += pf[k];
    tokens += pf[k] + ac[k];
  }
  const int64_t steps = hi - lo + 1;
  if (bucket < 0) {
    g.kind = RLX_KIND_TOOL_WAIT;
    g.duration = (double)steps * lat[0];
  } else {
    if (bucket == nb - 1 && nb >= 3)
      g.kind = (tokens > 0 && prefill * 2 >= tokens) ? RLX_KIND_PREFILL_BURST : RLX_KIND_DECODE_LARGE;
    else
      g.kind = bucket == 0 ? RLX_KIND_DECODE_SMALL : bucket == 1 ? RLX_KIND_DECODE_MEDIUM : RLX_KIND_DECODE_LARGE;
    g.duration = (double)steps * lat[bucket];
    g.context0 = cx[lo];
  }
  g.decode = decode;
  g.active0 = ac[lo];
  g.tokens = tokens;
  out[n++] = g;
}

__global__ void rlx_segment_kernel(const Cohort* cohorts, int n_cohorts, const int64_t* n_steps, const int64_t* r_prefill,
                                   const int32_t* r_active, const int64_t* r_context, const double* latency,
                                   const int32_t* bounds, int nb, int window, SegOut so) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cohorts) return;
  const Cohort C = cohorts[c];
  const int64_t n = n_steps[c];
  const int64_t* pf = r_prefill + C.rec_off;
  const int32_t* ac = r_active + C.rec_off;
  const int64_t* cx = r_context + C.rec_off;
  const double* lat = latency + 5 * C.pipe;
  RlxSegment* out = so.seg + C.rec_off;
  int ns = 0;
  auto code = [&](int64_t k) { return bucket_of(pf[k] + ac[k], bounds, nb); };
  int64_t i = 0;
  while (i < n) {
    int64_t j = i;
    if (is_idle(pf, ac, i)) {  // tool-wait run
      while (j + 1 < n && is_idle(pf, ac, j + 1)) j++;
      emit(C, pf, ac, cx, lat, nb, i, j, -1, out, ns);
      i = j + 1;
      continue;
    }
    while (j + 1 < n && !is_idle(pf, ac, j + 1)) j++;
    // _segment_span over [i, j]: the first bucket stable for `window` steps
    const int64_t len = j - i + 1;
    int current = -1;
    for (int64_t k = 0; k + window <= len && current < 0; k++) {
      const int b0 = code(i + k);
      bool same = true;
      for (int q = 1; q < window && same; q++) same = code(i + k + q) == b0;
      if (same) current = b0;
    }
    if (current < 0) {  // too short or noisy: one span, majority bucket (ties: smallest)
      int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int64_t k = i; k <= j; k++) cnt[code(k)]++;
      int best = -1;
      for (int b = 0; b < nb; b++)
        if (cnt[b] > 0 && (best < 0 || cnt[b] > cnt[best])) best = b;
      emit(C, pf, ac, cx, lat, nb, i, j, best, out, ns);
      i = j + 1;
      continue;
    }
    int64_t seg_start = 0, cand_start = 0;
    int cand_bucket = -1, cand_len = 0;
    for (int64_t k = 0; k < len; k++) {
      const int cd = code(i + k);
      if (cd == current) {
        cand_bucket = -1;
        cand_len = 0;
        continue;
      }
      if (cand_bucket == cd) {
        cand_len++;
      } else {
        cand_bucket = cd;
        cand_start = k;
        cand_len = 1;
      }
      if (cand_len >= window) {  // transition confirmed at the first stable step
        if (cand_start > seg_start) emit(C, pf, ac, cx, lat, nb, i + seg_start, i + cand_start - 1, current, out, ns);
        seg_start = cand_start;
        current = cd;
        cand_bucket = -1;
        cand_len = 0;
      }
    }
    emit(C, pf, ac, cx, lat, nb, i + seg_start, j, current, out, ns);
    i = j + 1;
  }
  so.n_seg[c] = ns;
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t n) { return cudaMalloc(&p, sizeof(T) * (n ? n : 1)); }
};

}  // namespace
}  // namespace rlx

using namespace rlx;

struct RlxGraphResult {
  std::vector<int32_t> pipe_of;            // per cohort
  std::vector<std::vector<RlxSegment>> segs;  // per pipeline, workers ascending, then seq
  double kernel_ms = 0.0;
  int64_t n_records = 0;
  std::string err;
};

extern "C" {

int rlx_graph_build(int device, int32_t n_pipes, const RlxRolloutTables* tables, const int32_t* bucket_bounds,
                    int32_t n_buckets, int32_t window, void** result) {
  if (!result || !tables || n_pipes < 1 || !bucket_bounds || n_buckets < 1 || window < 1) return RLX_ERR_ARG;
  *result = nullptr;
  RlxGraphResult* R = new RlxGraphResult();
  auto fail = [&](int code, const char* m) {
    R->err = m;
    *result = R;
    return code;
  };
  if (bucket_bounds[0] != 0) return fail(RLX_ERR_VALUE, "bucket bounds must start at 0");
  // the per-step latency model has entries 0..4 and the reference indexes it
  // by bucket (workload.py:315, graph.py:340): more buckets raise KeyError there
  if (n_buckets > 5) return fail(RLX_ERR_KEY, "latency model has no entry for bucket 5");
  for (int i = 1; i < n_buckets; i++)
    if (bucket_bounds[i] <= bucket_bounds[i - 1]) return fail(RLX_ERR_VALUE, "bucket bounds must be strictly increasing");
  if (cudaSetDevice(device) != cudaSuccess) return fail(RLX_ERR_CUDA, "cudaSetDevice failed");
  // ---- flatten: cohorts in (pipeline, worker) order, samples of a cohort in
  // sample-id order (round-robin: sample i -> worker i mod dp_workers)
  std::vector<Cohort> coh;
  std::vector<int64_t> prompt, tpre, tdec;
  std::vector<double> ttool, lat;
  std::vector<int32_t> toff(1, 0);
  for (int p = 0; p < n_pipes; p++) {
    const RlxRolloutTables& T = tables[p];
    if (T.n_workers < 1 || T.n_samples < 0) return fail(RLX_ERR_ARG, "bad table sizes");
    for (int k = 0; k < 5; k++) lat.push_back(T.latency[k]);
    std::vector<std::vector<int>> by_w(T.n_workers);
    for (int s = 0; s < T.n_samples; s++) {
      const int w = T.worker_of ? T.worker_of[s] : s % T.n_workers;
      if (w < 0 || w >= T.n_workers) return fail(RLX_ERR_VALUE, "assignment references invalid workers");
      if (T.turn_off[s + 1] <= T.turn_off[s]) return fail(RLX_ERR_VALUE, "a sample without turns");
      by_w[w].push_back(s);
    }
    for (int w = 0; w < T.n_workers; w++) {
      Cohort c;
      c.pipe = p;
      c.worker = w;
      c.s0 = (int32_t)prompt.size();
      c.n = (int32_t)by_w[w].size();
      c.rec_off = 0;
      for (int s : by_w[w]) {
        prompt.push_back(T.prompt[s]);
        for (int t = T.turn_off[s]; t < T.turn_off[s + 1]; t++) {
          tpre.push_back(T.turn_prefill[t]);
          tdec.push_back(T.turn_decode[t]);
          ttool.push_back(T.turn_tool[t]);
        }
        toff.push_back((int32_t)tpre.size());
      }
      if (c.n > 0) coh.push_back(c);
    }
  }
  const int NC = (int)coh.size();
  const int NS = (int)prompt.size();
  DevBuf<Cohort> d_coh;
  DevBuf<int64_t> d_prompt, d_tpre, d_tdec, d_rem, d_ctx, d_pend, d_nsteps, d_rpf, d_rcx;
  DevBuf<int32_t> d_toff, d_turn, d_bounds, d_rac, d_nseg;
  DevBuf<double> d_ttool, d_lat, d_wake;
  DevBuf<uint8_t> d_done;
  DevBuf<RlxSegment> d_seg;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
#define CKG(x)                                                   \
  do {                                                           \
    if ((x) != cudaSuccess) return fail(RLX_ERR_CUDA, #x " failed"); \
  } while (0)
  CKG(d_coh.alloc(NC));
  CKG(d_prompt.alloc(NS));
  CKG(d_toff.alloc(toff.size()));
  CKG(d_tpre.alloc(tpre.size()));
  CKG(d_tdec.alloc(tdec.size()));
  CKG(d_ttool.alloc(ttool.size()));
  CKG(d_lat.alloc(lat.size()));
  CKG(d_bounds.alloc(n_buckets));
  CKG(d_turn.alloc(NS));
  CKG(d_rem.alloc(NS));
  CKG(d_ctx.alloc(NS));
  CKG(d_pend.alloc(NS));
  CKG(d_wake.alloc(NS));
  CKG(d_done.alloc(NS));
  CKG(d_nsteps.alloc(NC));
  CKG(cudaMemcpy(d_coh.p, coh.data(), sizeof(Cohort) * NC, cudaMemcpyHostToDevice));
  CKG(cudaMemcpy(d_prompt.p, prompt.data(), sizeof(int64_t) * NS, cudaMemcpyHostToDevice));
  CKG(cudaMemcpy(d_toff.p, toff.data(), sizeof(int32_t) * toff.size(), cudaMemcpyHostToDevice));
  CKG(cudaMemcpy(d_tpre.p, tpre.data(), sizeof(int64_t) * tpre.size(), cudaMemcpyHostToDevice));
  CKG(cudaMemcpy(d_tdec.p, tdec.data(), sizeof(int64_t) * tdec.size(), cudaMemcpyHostToDevice));
  CKG(cudaMemcpy(d_ttool.p, ttool.data(), sizeof(double) * ttool.size(), cudaMemcpyHostToDevice));
  CKG(cudaMemcpy(d_lat.p, lat.data(), sizeof(double) * lat.size(), cudaMemcpyHostToDevice));
  CKG(cudaMemcpy(d_bounds.p, bucket_bounds, sizeof(int32_t) * n_buckets, cudaMemcpyHostToDevice));
  SampleState st{d_turn.p, d_rem.p, d_ctx.p, d_pend.p, d_wake.p, d_done.p};
  const int tpb = 128;  // 4 cohorts per block
  const int blocks = (NC * 32 + tpb - 1) / tpb;
  cudaEventRecord(e0);
  // pass 1: steps per cohort
  rlx_replay_kernel<<<blocks, tpb>>>(d_coh.p, NC, d_prompt.p, d_toff.p, d_tpre.p, d_tdec.p, d_ttool.p, d_lat.p,
                                     d_bounds.p, n_buckets, st, d_nsteps.p, 0, nullptr, nullptr, nullptr);
  CKG(cudaGetLastError());
  std::vector<int64_t> nsteps(NC);
  CKG(cudaMemcpy(nsteps.data(), d_nsteps.p, sizeof(int64_t) * NC, cudaMemcpyDeviceToHost));
  int64_t total = 0;
  for (int c = 0; c < NC; c++) {
    coh[c].rec_off = total;
    total += nsteps[c];
  }
  R->n_records = total;
  CKG(cudaMemcpy(d_coh.p, coh.data(), sizeof(Cohort) * NC, cudaMemcpyHostToDevice));
  CKG(d_rpf.alloc(total));
  CKG(d_rac.alloc(total));
  CKG(d_rcx.alloc(total));
  CKG(d_seg.alloc(total));
  CKG(d_nseg.alloc(NC));
  // pass 2: the records
  rlx_replay_kernel<<<blocks, tpb>>>(d_coh.p, NC, d_prompt.p, d_toff.p, d_tpre.p, d_tdec.p, d_ttool.p, d_lat.p,
                                     d_bounds.p, n_buckets, st, d_nsteps.p, 1, d_rpf.p, d_rac.p, d_rcx.p);
  CKG(cudaGetLastError());
  rlx_segment_kernel<<<(NC + 63) / 64, 64>>>(d_coh.p, NC, d_nsteps.p, d_rpf.p, d_rac.p, d_rcx.p, d_lat.p, d_bounds.p,
                                             n_buckets, window, SegOut{d_seg.p, d_nseg.p});
  CKG(cudaGetLastError());
  cudaEventRecord(e1);
  std::vector<int32_t> nseg(NC);
  CKG(cudaMemcpy(nseg.data(), d_nseg.p, sizeof(int32_t) * NC, cudaMemcpyDeviceToHost));
  std::vector<RlxSegment> segs(total);
  // only the written prefix of each cohort's segment range
  R->segs.assign(n_pipes, {});
  for (int c = 0; c < NC; c++) {
    if (nseg[c] == 0) continue;
    const size_t at = R->segs[coh[c].pipe].size();
    R->segs[coh[c].pipe].resize(at + nseg[c]);
    CKG(cudaMemcpy(R->segs[coh[c].pipe].data() + at, d_seg.p + coh[c].rec_off, sizeof(RlxSegment) * nseg[c],
                   cudaMemcpyDeviceToHost));
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  R->kernel_ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *result = R;
  return RLX_OK;
#undef CKG
}

int rlx_graph_segments(void* result, int32_t pipe, RlxSegment* out, int64_t cap, int64_t* n_out) {
  RlxGraphResult* R = (RlxGraphResult*)result;
  if (!R || !n_out || pipe < 0 || pipe >= (int)R->segs.size()) return RLX_ERR_ARG;
  const std::vector<RlxSegment>& v = R->segs[pipe];
  *n_out = (int64_t)v.size();
  if (out && cap > 0) memcpy(out, v.data(), sizeof(RlxSegment) * (size_t)(cap < (int64_t)v.size() ? cap : v.size()));
  return RLX_OK;
}

int rlx_graph_stats(void* result, double* kernel_ms, int64_t* n_records) {
  RlxGraphResult* R = (RlxGraphResult*)result;
  if (!R) return RLX_ERR_ARG;
  if (kernel_ms) *kernel_ms = R->kernel_ms;
  if (n_records) *n_records = R->n_records;
  return RLX_OK;
}

const char* rlx_graph_error(void* result) {
  RlxGraphResult* R = (RlxGraphResult*)result;
  return R ? R->err.c_str() : "null result";
}

void rlx_graph_free(void* result) { delete (RlxGraphResult*)result; }

}  // extern "C"

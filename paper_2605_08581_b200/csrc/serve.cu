// serve.cu -- the serving loop (engine.py:141-266) with device-resident state.
//
// The reference replays a trace window by window: completions release their
// leaves (engine.py:171-175), arrivals join the pending queue (176-178), and
// when the engine is idle a wave runs -- schedule_round over pending and the
// in-flight set, the protection / active hand-off, match+insert per member
// with CapacityError stopping the wave (189-213) -- followed by the wave cost
// model (215-232) and per-request metrics (233-259).
//
// Here every per-request array lives in HBM: the trace itself (CSR, in
// (arrival, id) order), the pending queue (trace indices in queue order), the
// admission log (trace index + pinned leaf slot per admitted request), and
// the per-request metrics.  Each wave gathers the pending and in-flight
// skeleton CSRs on the device (k_sv_gather_*), runs the fused wave
// (prism_wave_step), and one single-CTA kernel (k_sv_wave_end) applies the
// wave cost model in the reference's float evaluation order, writes the
// members' metrics, appends them to the admission log and compacts them out
// of the queue.  The host keeps only O(waves) scalars: the window clock, the
// in-flight waves as a completion heap (every member of a wave shares its
// completion time, engine.py:224-227), and it jumps straight to the next
// window where something can happen -- the windows the reference skips
// ("continue", engine.py:180-181) change nothing but the clock, and the
// jump reproduces its float comparisons exactly.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <queue>
#include <string>
#include <vector>

#include "../../include/prism.h"
#include "pdl.cuh"
#include "scan.cuh"

namespace {

constexpr int SV_TPB = 1024;
constexpr int64_t SV_MAX_WINDOWS = 50000000;  // engine.py:137 _MAX_WINDOWS

int sfail(int code, const std::string &m) {
  prism_set_last_error(m.c_str());
  return code;
}
#define SCK(x)                                                                                          \
  do {                                                                                                  \
    cudaError_t e_ = (x);                                                                               \
    if (e_ != cudaSuccess) return sfail(PRISM_CUDA, std::string("CUDA error ") + cudaGetErrorString(e_) + " in " #x); \
  } while (0)

struct SvCtl {  // one wave's cost model, written by k_sv_wave_end (mapped pinned memory)
  double duration, prefill_end, first_token, completion;
  long long uncached, cached;
};

// ---------------------------------------------------------------- kernels

// arrivals [first, first + n) join the queue at position P0 (engine.py:176-178)
__global__ void k_sv_append(int32_t *pend, int64_t P0, int64_t first, int64_t n) {
  pdl_wait();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) pend[P0 + j] = (int32_t)(first + j);
}

// the pending snapshot as the wave's CSR: per-request fields gathered from the
// trace by queue position, skeleton offsets by one block-wide scan
__global__ void __launch_bounds__(SV_TPB) k_sv_gather_pending(const int32_t *pend, int64_t P, const int64_t *tids,
                                                              const double *tarr, const int64_t *toff,
                                                              const uint8_t *treo, const int32_t *tsfx, int64_t *gids,
                                                              double *garr, int64_t *goff, uint8_t *greo,
                                                              int32_t *gsfx) {
  pdl_wait();
  prism::block_scan4<1, 4>(
      P,
      [&](int, int64_t i) {
        const int32_t ti = pend[i];
        return toff[ti + 1] - toff[ti];
      },
      [&](int, int64_t i, int64_t excl, int64_t incl) {
        const int32_t ti = pend[i];
        goff[i] = excl;
        if (i == P - 1) goff[P] = incl;
        gids[i] = tids[ti];
        garr[i] = tarr[ti];
        greo[i] = treo[ti];
        gsfx[i] = tsfx[ti];
      });
}

// the in-flight set (engine.py:189 active.values()): the admission-log ranges
// of the waves still decoding, concatenated; their skeleton offsets by a scan
__global__ void __launch_bounds__(SV_TPB) k_sv_gather_active(const int64_t *ranges, int32_t R, int64_t A,
                                                             const int32_t *log_idx, const int64_t *toff,
                                                             int32_t *act_ti, int64_t *aoff) {
  pdl_wait();
  __shared__ int64_t pre[1025];
  // range r covers concatenated positions [pre[r], pre[r+1]) (R <= 1024 here;
  // the host merges adjacent log ranges first)
  if (threadIdx.x == 0) {
    int64_t s = 0;
    for (int r = 0; r < R; r++) {
      pre[r] = s;
      s += ranges[2 * r + 1] - ranges[2 * r];
    }
    pre[R] = s;
  }
  __syncthreads();
  auto ti_of = [&](int64_t j) {
    int lo = 0, hi = R - 1;  // last r with pre[r] <= j
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pre[mid] <= j) lo = mid;
      else hi = mid - 1;
    }
    return log_idx[ranges[2 * lo] + (j - pre[lo])];
  };
  prism::block_scan4<1, 4>(
      A,
      [&](int, int64_t j) {
        const int32_t ti = ti_of(j);
        return toff[ti + 1] - toff[ti];
      },
      [&](int, int64_t j, int64_t excl, int64_t incl) {
        act_ti[j] = ti_of(j);
        aoff[j] = excl;
        if (j == A - 1) aoff[A] = incl;
      });
}

// skeleton entries of the gathered requests: one warp per request
__global__ void k_sv_gather_sk(const int32_t *idx, int64_t n, const int64_t *off, const int64_t *toff,
                               const int32_t *tsk, int32_t *sk) {
  pdl_wait();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const int32_t ti = idx[w];
  const int64_t b = toff[ti], k = toff[ti + 1] - b, o = off[w];
  for (int64_t e = lane; e < k; e += 32) sk[o + e] = tsk[b + e];
}

// the end of a wave with na > 0 admitted members (engine.py:215-259), one CTA:
// uncached / cached sums, the cost model in the reference's evaluation order
// (explicit round-to-nearest, no contraction), the members' metrics, their log
// entries, and the queue without them (stable compaction)
struct SvWaveIn {
  int64_t na, P;
  const int64_t *members, *hits;
  const int32_t *leaf_slots;
  int32_t *pend, *pend_out;
  uint8_t *taken;  // [P] scratch, zero outside this kernel
  const int64_t *toff;
  const int32_t *tsfx;
  int64_t sys_len, chunk;
  double t, te;  // window time; throughput estimate completed / t (engine.py:219)
  double prefill_rate, decode_rate;
  int64_t out_tokens;
  int32_t attenuate;
  double *admit, *prefill_end, *first_token, *completion;
  int64_t *hit, *eff;
  int32_t *log_idx, *log_slot;
  int64_t nlog;
  SvCtl *ctl;
};

__global__ void __launch_bounds__(SV_TPB) k_sv_wave_end(SvWaveIn W) {
  pdl_wait();
  __shared__ long long s_u[32], s_c[32];
  __shared__ double s_t[4];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long u = 0, c = 0;
  for (int64_t j = threadIdx.x; j < W.na; j += blockDim.x) {
    const int32_t ti = W.pend[W.members[j]];
    const int64_t len = W.sys_len + (W.toff[ti + 1] - W.toff[ti]) * W.chunk + W.tsfx[ti];
    u += len - W.hits[j];
    c += W.hits[j];
  }
  for (int o = 16; o > 0; o >>= 1) {
    u += __shfl_xor_sync(0xffffffffu, u, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  if (lane == 0) {
    s_u[wid] = u;
    s_c[wid] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long U = 0, Cc = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
      U += s_u[w];
      Cc += s_c[w];
    }
    // effective_prefill_rate (engine.py:127-133)
    double rate = W.prefill_rate;
    if (W.attenuate) {
      double alpha = __ddiv_rn(__dmul_rn(W.te, (double)W.out_tokens), W.decode_rate);
      alpha = fmin(fmax(alpha, 0.0), 0.95);
      rate = __dmul_rn(W.prefill_rate, __dsub_rn(1.0, alpha));
    }
    const double duration = __ddiv_rn((double)U, rate);                          // 221
    const double pe = __dadd_rn(W.t, duration);                                   // 223
    const double ft = __dadd_rn(pe, __ddiv_rn((double)W.na, W.decode_rate));     // 224
    const double comp = __dadd_rn(ft, __ddiv_rn((double)((W.out_tokens - 1) * W.na), W.decode_rate));  // 225
    s_t[0] = duration;
    s_t[1] = pe;
    s_t[2] = ft;
    s_t[3] = comp;
    W.ctl->duration = duration;
    W.ctl->prefill_end = pe;
    W.ctl->first_token = ft;
    W.ctl->completion = comp;
    W.ctl->uncached = U;
    W.ctl->cached = Cc;
  }
  __syncthreads();
  for (int64_t j = threadIdx.x; j < W.na; j += blockDim.x) {
    const int64_t p = W.members[j];
    const int32_t ti = W.pend[p];
    const int64_t len = W.sys_len + (W.toff[ti + 1] - W.toff[ti]) * W.chunk + W.tsfx[ti];
    W.admit[ti] = W.t;
    W.prefill_end[ti] = s_t[1];
    W.first_token[ti] = s_t[2];
    W.completion[ti] = s_t[3];
    W.hit[ti] = W.hits[j];
    W.eff[ti] = len - W.hits[j];
    W.log_idx[W.nlog + j] = ti;
    W.log_slot[W.nlog + j] = W.leaf_slots[j];
    W.taken[p] = 1;
  }
  __syncthreads();
  // pending = [r for r in pending if r.id not in admitted_ids]  (engine.py:214)
  prism::block_scan4<1, 4>(
      W.P, [&](int, int64_t i) { return (int64_t)(W.taken[i] ? 0 : 1); },
      [&](int, int64_t i, int64_t excl, int64_t) {
        if (!W.taken[i]) W.pend_out[excl] = W.pend[i];
      });
  __syncthreads();
  for (int64_t i = threadIdx.x; i < W.P; i += blockDim.x) W.taken[i] = 0;
}

template <class T>
int dalloc(T **p, int64_t n) {
  SCK(cudaMalloc((void **)p, sizeof(T) * (size_t)std::max<int64_t>(n, 1)));
  return PRISM_OK;
}

}  // namespace

struct prism_serve {
  prism_tree *t = nullptr;
  prism_qas *q = nullptr;
  int dev = 0;
  cudaStream_t st = nullptr;
  // configuration (SimConfig, engine.py:35-48; SchedulerConfig.window_s)
  prism_qas_config cfg{};
  double window = 0.05, prefill_rate = 1.0, decode_rate = 1.0;
  int64_t out_tokens = 1;
  int32_t attenuate = 0, nseg = 0;
  int64_t sys_len = 0, chunk = 0, capacity = 0;
  // the trace in (arrival, id) order (device) + the arrival times (host)
  int64_t n = 0, nsk = 0;
  int64_t *tids = nullptr, *toff = nullptr;
  double *tarr = nullptr;
  int32_t *tsk = nullptr, *tsfx = nullptr;
  uint8_t *treo = nullptr;
  std::vector<double> h_arr;
  // queue and the wave's gathered inputs / outputs
  int32_t *pend = nullptr, *pend2 = nullptr;
  uint8_t *taken = nullptr;
  int64_t *gids = nullptr, *goff = nullptr, *aoff = nullptr;
  double *garr = nullptr;
  uint8_t *greo = nullptr;
  int32_t *gsfx = nullptr, *gsk = nullptr, *ask = nullptr, *act_ti = nullptr;
  int64_t *members = nullptr, *hits = nullptr, *leaf_ids = nullptr;
  int32_t *leaf_slots = nullptr;
  int64_t *d_ranges = nullptr, *h_ranges = nullptr;
  int64_t ranges_cap = 0;
  // admission log + per-request metrics (device)
  int32_t *log_idx = nullptr, *log_slot = nullptr;
  double *m_admit = nullptr, *m_pe = nullptr, *m_ft = nullptr, *m_comp = nullptr;
  int64_t *m_hit = nullptr, *m_eff = nullptr;
  SvCtl *ctl = nullptr;  // mapped pinned
  // host loop state
  int64_t k = 0, next_arr = 0, Pn = 0, completed = 0, nlog = 0;
  double busy_until = 0.0;
  bool done = false;
  std::vector<double> w_launch, w_duration;
  std::vector<float> w_host_us;  // host wall time of each wave (diagnostics)
  std::vector<int64_t> w_uncached, w_cached, w_off{0};
  // in-flight waves: (completion, wave index), earliest first
  std::priority_queue<std::pair<double, int64_t>, std::vector<std::pair<double, int64_t>>,
                      std::greater<std::pair<double, int64_t>>>
      inflight;
  int64_t n_inflight = 0;
};

namespace {

// smallest k' >= kmin with k' * window + 1e-12 >= x (the reference's own float test)
int64_t first_window_at(double window, int64_t kmin, double x) {
  auto ok = [&](int64_t k) { return (double)k * window + 1e-12 >= x; };
  double g = std::ceil((x - 1e-12) / window);
  int64_t k = g > 9.0e18 ? INT64_MAX / 2 : (int64_t)std::max(g, 0.0);
  if (k < kmin) k = kmin;
  while (k > kmin && ok(k - 1)) k--;
  while (!ok(k)) k++;
  return k;
}

int sv_release_wave(prism_serve *s, int64_t w) {
  const int64_t lo = s->w_off[w], cnt = s->w_off[w + 1] - lo;
  int rc = prism_release_device(s->t, cnt, s->log_slot + lo, nullptr, (void *)s->st);
  if (rc) return rc;
  s->completed += cnt;
  s->n_inflight -= cnt;
  return PRISM_OK;
}

// one wave at window s->k (pending non-empty, engine idle); *progress = admitted
int sv_wave(prism_serve *s, int64_t *admitted) {
  const int64_t P = s->Pn;
  const double t = (double)s->k * s->window;
  k_sv_gather_pending<<<1, SV_TPB, 0, s->st>>>(s->pend, P, s->tids, s->tarr, s->toff, s->treo, s->tsfx, s->gids,
                                               s->garr, s->goff, s->greo, s->gsfx);
  k_sv_gather_sk<<<(unsigned)((P * 32 + 255) / 256), 256, 0, s->st>>>(s->pend, P, s->goff, s->toff, s->tsk, s->gsk);
  SCK(cudaGetLastError());
  // the in-flight set: log ranges of the waves still decoding, adjacent ranges merged
  std::vector<std::pair<int64_t, int64_t>> rg;
  {
    auto c = s->inflight;  // (a copy: a few entries)
    while (!c.empty()) {
      const int64_t w = c.top().second;
      c.pop();
      rg.push_back({s->w_off[w], s->w_off[w + 1]});
    }
    std::sort(rg.begin(), rg.end());
    std::vector<std::pair<int64_t, int64_t>> m;
    for (auto &r : rg) {
      if (!m.empty() && m.back().second == r.first) m.back().second = r.second;
      else m.push_back(r);
    }
    rg.swap(m);
  }
  const int64_t A = s->n_inflight;
  if (A > 0) {
    if ((int64_t)rg.size() > 1024) return sfail(PRISM_FATAL, "more than 1024 disjoint in-flight log ranges");
    if ((int64_t)rg.size() > s->ranges_cap) {
      if (s->h_ranges) cudaFreeHost(s->h_ranges);
      if (s->d_ranges) cudaFree(s->d_ranges);
      s->ranges_cap = 1024;
      SCK(cudaMallocHost(&s->h_ranges, sizeof(int64_t) * 2 * s->ranges_cap));
      SCK(cudaMalloc(&s->d_ranges, sizeof(int64_t) * 2 * s->ranges_cap));
    }
    SCK(cudaStreamSynchronize(s->st));  // h_ranges may still be read by the previous copy
    for (size_t r = 0; r < rg.size(); r++) {
      s->h_ranges[2 * r] = rg[r].first;
      s->h_ranges[2 * r + 1] = rg[r].second;
    }
    SCK(cudaMemcpyAsync(s->d_ranges, s->h_ranges, sizeof(int64_t) * 2 * rg.size(), cudaMemcpyHostToDevice, s->st));
    k_sv_gather_active<<<1, SV_TPB, 0, s->st>>>(s->d_ranges, (int32_t)rg.size(), A, s->log_idx, s->toff, s->act_ti,
                                                s->aoff);
    k_sv_gather_sk<<<(unsigned)((A * 32 + 255) / 256), 256, 0, s->st>>>(s->act_ti, A, s->aoff, s->toff, s->tsk,
                                                                         s->ask);
    SCK(cudaGetLastError());
  }
  int64_t nm = 0, na = 0;
  int rc = prism_wave_step(s->t, s->q, P, s->gids, s->garr, s->goff, s->gsk, s->greo, s->gsfx, A, s->aoff, s->ask,
                           s->nseg, &s->cfg, s->sys_len, s->chunk, s->members, s->hits, s->leaf_slots, s->leaf_ids,
                           &nm, &na);
  if (rc) return rc;
  *admitted = na;
  if (na == 0) return PRISM_OK;  // engine.py:210-211: nothing admitted, the queue is unchanged
  SvWaveIn W{};
  W.na = na;
  W.P = P;
  W.members = s->members;
  W.hits = s->hits;
  W.leaf_slots = s->leaf_slots;
  W.pend = s->pend;
  W.pend_out = s->pend2;
  W.taken = s->taken;
  W.toff = s->toff;
  W.tsfx = s->tsfx;
  W.sys_len = s->sys_len;
  W.chunk = s->chunk;
  W.t = t;
  W.te = t > 0 ? (double)s->completed / t : 0.0;  // engine.py:219 (host: plain IEEE division)
  W.prefill_rate = s->prefill_rate;
  W.decode_rate = s->decode_rate;
  W.out_tokens = s->out_tokens;
  W.attenuate = s->attenuate;
  W.admit = s->m_admit;
  W.prefill_end = s->m_pe;
  W.first_token = s->m_ft;
  W.completion = s->m_comp;
  W.hit = s->m_hit;
  W.eff = s->m_eff;
  W.log_idx = s->log_idx;
  W.log_slot = s->log_slot;
  W.nlog = s->nlog;
  W.ctl = s->ctl;
  k_sv_wave_end<<<1, SV_TPB, 0, s->st>>>(W);
  SCK(cudaGetLastError());
  SCK(cudaStreamSynchronize(s->st));
  std::swap(s->pend, s->pend2);
  s->Pn = P - na;
  const int64_t w = (int64_t)s->w_launch.size();
  s->w_launch.push_back(t);
  s->w_duration.push_back(s->ctl->duration);
  s->w_uncached.push_back(s->ctl->uncached);
  s->w_cached.push_back(s->ctl->cached);
  s->nlog += na;
  s->w_off.push_back(s->nlog);
  s->busy_until = s->ctl->prefill_end;  // engine.py:226
  s->inflight.push({s->ctl->completion, w});
  s->n_inflight += na;
  return PRISM_OK;
}

}  // namespace

extern "C" {

prism_serve *prism_serve_create(prism_tree *t, prism_qas *q, int64_t n, const int64_t *ids, const double *arrival,
                                const int64_t *sk_off, const int32_t *sk, const uint8_t *reorderable,
                                const int32_t *suffix, int32_t nseg, int64_t sys_len, int64_t chunk,
                                int64_t capacity_tokens, const prism_qas_config *cfg, double window_s,
                                double prefill_rate, double decode_rate, int64_t output_tokens,
                                int32_t decode_attenuation) {
  if (!t || !q || n < 0 || !cfg || chunk < 1 || sys_len < 0 || window_s <= 0 || prefill_rate <= 0 ||
      decode_rate <= 0 || output_tokens < 1) {
    sfail(PRISM_INVALID, "prism_serve_create: invalid arguments");
    return nullptr;
  }
  for (int64_t i = 0; i < n; i++) {  // run_simulation's (arrival, id) order (engine.py:158) is the caller's
    if (sk_off[i + 1] < sk_off[i]) {
      sfail(PRISM_INVALID, "prism_serve_create: skeleton offsets decrease");
      return nullptr;
    }
    if (i && (arrival[i] < arrival[i - 1] || (arrival[i] == arrival[i - 1] && ids[i] <= ids[i - 1]))) {
      sfail(PRISM_INVALID, "prism_serve_create: requests not in (arrival_time, id) order");
      return nullptr;
    }
    const int64_t len = sys_len + (sk_off[i + 1] - sk_off[i]) * chunk + suffix[i];
    if (len > capacity_tokens) {  // engine.py:146-151
      sfail(PRISM_SIMULATION, "request " + std::to_string(ids[i]) + " path (" + std::to_string(len) +
                                  " tokens) exceeds cache capacity (" + std::to_string(capacity_tokens) + ")");
      return nullptr;
    }
  }
  const int64_t nsk = n ? sk_off[n] - sk_off[0] : 0;
  for (int64_t e = 0; e < nsk; e++)
    if (sk[sk_off[0] + e] < 0 || sk[sk_off[0] + e] >= nseg) {
      sfail(PRISM_INVALID, "prism_serve_create: segment id outside [0, nseg)");
      return nullptr;
    }
  auto *s = new prism_serve();
  s->t = t;
  s->q = q;
  cudaGetDevice(&s->dev);
  s->st = (cudaStream_t)prism_qas_stream(q);
  s->cfg = *cfg;
  s->window = window_s;
  s->prefill_rate = prefill_rate;
  s->decode_rate = decode_rate;
  s->out_tokens = output_tokens;
  s->attenuate = decode_attenuation;
  s->nseg = nseg;
  s->sys_len = sys_len;
  s->chunk = chunk;
  s->capacity = capacity_tokens;
  s->n = n;
  s->nsk = nsk;
  s->h_arr.assign(arrival, arrival + n);
  auto fail = [&](int rc) -> prism_serve * {
    (void)rc;
    prism_serve_destroy(s);
    return nullptr;
  };
  int rc;
  const int64_t n1 = n + 1;
  if ((rc = dalloc(&s->tids, n)) || (rc = dalloc(&s->toff, n1)) || (rc = dalloc(&s->tarr, n)) ||
      (rc = dalloc(&s->tsk, nsk)) || (rc = dalloc(&s->tsfx, n)) || (rc = dalloc(&s->treo, n)) ||
      (rc = dalloc(&s->pend, n)) || (rc = dalloc(&s->pend2, n)) || (rc = dalloc(&s->taken, n)) ||
      (rc = dalloc(&s->gids, n)) || (rc = dalloc(&s->goff, n1)) || (rc = dalloc(&s->aoff, n1)) ||
      (rc = dalloc(&s->garr, n)) || (rc = dalloc(&s->greo, n)) || (rc = dalloc(&s->gsfx, n)) ||
      (rc = dalloc(&s->gsk, nsk)) || (rc = dalloc(&s->ask, nsk)) || (rc = dalloc(&s->act_ti, n)) ||
      (rc = dalloc(&s->members, n)) || (rc = dalloc(&s->hits, n)) || (rc = dalloc(&s->leaf_ids, n)) ||
      (rc = dalloc(&s->leaf_slots, n)) || (rc = dalloc(&s->log_idx, n)) || (rc = dalloc(&s->log_slot, n)) ||
      (rc = dalloc(&s->m_admit, n)) || (rc = dalloc(&s->m_pe, n)) || (rc = dalloc(&s->m_ft, n)) ||
      (rc = dalloc(&s->m_comp, n)) || (rc = dalloc(&s->m_hit, n)) || (rc = dalloc(&s->m_eff, n)))
    return fail(rc);
  if (cudaHostAlloc(&s->ctl, sizeof(SvCtl), cudaHostAllocMapped) != cudaSuccess) {
    sfail(PRISM_CUDA, "prism_serve_create: mapped control block");
    return fail(PRISM_CUDA);
  }
  std::vector<int64_t> off0(n1);
  for (int64_t i = 0; i <= n; i++) off0[i] = sk_off[i] - sk_off[0];
  cudaStream_t st = s->st;
  if (n) {
    cudaMemcpyAsync(s->tids, ids, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(s->tarr, arrival, sizeof(double) * n, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(s->toff, off0.data(), sizeof(int64_t) * n1, cudaMemcpyHostToDevice, st);
    if (nsk) cudaMemcpyAsync(s->tsk, sk + sk_off[0], sizeof(int32_t) * nsk, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(s->tsfx, suffix, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(s->treo, reorderable, n, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(s->taken, 0, n, st);
    cudaMemsetAsync(s->m_admit, 0, sizeof(double) * n, st);
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) {
    sfail(PRISM_CUDA, "prism_serve_create: upload");
    return fail(PRISM_CUDA);
  }
  s->done = n == 0;
  return s;
}

void prism_serve_destroy(prism_serve *s) {
  if (!s) return;
  cudaSetDevice(s->dev);
  if (s->st) cudaStreamSynchronize(s->st);
  void *bufs[] = {s->tids, s->toff, s->tarr, s->tsk, s->tsfx, s->treo, s->pend, s->pend2, s->taken, s->gids,
                  s->goff, s->aoff, s->garr, s->greo, s->gsfx, s->gsk, s->ask, s->act_ti, s->members, s->hits,
                  s->leaf_ids, s->leaf_slots, s->log_idx, s->log_slot, s->m_admit, s->m_pe, s->m_ft, s->m_comp,
                  s->m_hit, s->m_eff, s->d_ranges};
  for (void *p : bufs)
    if (p) cudaFree(p);
  if (s->h_ranges) cudaFreeHost(s->h_ranges);
  if (s->ctl) cudaFreeHost(s->ctl);
  delete s;
}

// Advance the loop by up to max_waves waves (<= 0: to the end).  *finished = 1
// once every request completed (engine.py:163); the remaining in-flight waves
// are then released, leaving every pin dropped as the reference does.
int prism_serve_run(prism_serve *s, int64_t max_waves, int64_t *waves_run, int32_t *finished) {
  cudaSetDevice(s->dev);
  int64_t ran = 0;
  int rc;
  while (!s->done && (max_waves <= 0 || ran < max_waves)) {
    int64_t k2;
    if (s->Pn > 0) {  // engine idle from the first window at or after busy_until
      k2 = first_window_at(s->window, s->k + 1, s->busy_until);
    } else if (s->next_arr < s->n) {  // ... and some request arrived
      k2 = std::max(first_window_at(s->window, s->k + 1, s->busy_until),
                    first_window_at(s->window, s->k + 1, s->h_arr[s->next_arr]));
    } else {  // nothing left to admit: the remaining completions, in order
      while (!s->inflight.empty()) {
        const int64_t w = s->inflight.top().second;
        s->inflight.pop();
        if ((rc = sv_release_wave(s, w))) return rc;
      }
      SCK(cudaStreamSynchronize(s->st));
      s->done = true;
      break;
    }
    if (k2 > SV_MAX_WINDOWS) return sfail(PRISM_SIMULATION, "simulation failed to make progress");
    s->k = k2;
    const double t = (double)k2 * s->window;
    while (!s->inflight.empty() && s->inflight.top().first <= t + 1e-12) {  // engine.py:171-175
      const int64_t w = s->inflight.top().second;
      s->inflight.pop();
      if ((rc = sv_release_wave(s, w))) return rc;
    }
    int64_t a = s->next_arr;  // engine.py:176-178
    while (a < s->n && s->h_arr[a] <= t + 1e-12) a++;
    if (a > s->next_arr) {
      const int64_t na = a - s->next_arr;
      k_sv_append<<<(unsigned)((na + 255) / 256), 256, 0, s->st>>>(s->pend, s->Pn, s->next_arr, na);
      SCK(cudaGetLastError());
      s->Pn += na;
      s->next_arr = a;
    }
    if (s->Pn == 0 || t + 1e-12 < s->busy_until) continue;  // engine.py:180-181
    int64_t adm = 0;
    const auto h0 = std::chrono::steady_clock::now();
    if ((rc = sv_wave(s, &adm))) return rc;
    {
      static const bool dbg = getenv("PRISM_DEBUG_COMMIT") != nullptr;
      const float us = std::chrono::duration<float, std::micro>(std::chrono::steady_clock::now() - h0).count();
      if (dbg && us > 3000) fprintf(stderr, "[serve] wave %zu: %.0f us (P=%lld, in flight %lld)\n",
                                    s->w_launch.size(), us, (long long)s->Pn, (long long)s->n_inflight);
    }
    if (adm > 0)
      s->w_host_us.push_back(
          std::chrono::duration<float, std::micro>(std::chrono::steady_clock::now() - h0).count());
    ran++;
  }
  if (waves_run) *waves_run = ran;
  if (finished) *finished = s->done ? 1 : 0;
  return PRISM_OK;
}

// counts: [0] waves, [1] admitted (log length), [2] windows advanced (k), [3] completed, [4] pending
int prism_serve_counts(prism_serve *s, int64_t *out) {
  out[0] = (int64_t)s->w_launch.size();
  out[1] = s->nlog;
  out[2] = s->k;
  out[3] = s->completed;
  out[4] = s->Pn;
  return PRISM_OK;
}

// Per-request metrics in trace order (engine.py:233-248): admit, prefill_end,
// first_token, completion (any may be NULL), hit / eff tokens.
int prism_serve_requests(prism_serve *s, double *admit, double *prefill_end, double *first_token,
                         double *completion, int64_t *hit, int64_t *eff) {
  cudaSetDevice(s->dev);
  const size_t n = (size_t)s->n;
  if (n) {
    if (admit) SCK(cudaMemcpyAsync(admit, s->m_admit, sizeof(double) * n, cudaMemcpyDeviceToHost, s->st));
    if (prefill_end) SCK(cudaMemcpyAsync(prefill_end, s->m_pe, sizeof(double) * n, cudaMemcpyDeviceToHost, s->st));
    if (first_token) SCK(cudaMemcpyAsync(first_token, s->m_ft, sizeof(double) * n, cudaMemcpyDeviceToHost, s->st));
    if (completion) SCK(cudaMemcpyAsync(completion, s->m_comp, sizeof(double) * n, cudaMemcpyDeviceToHost, s->st));
    if (hit) SCK(cudaMemcpyAsync(hit, s->m_hit, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s->st));
    if (eff) SCK(cudaMemcpyAsync(eff, s->m_eff, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s->st));
  }
  SCK(cudaStreamSynchronize(s->st));
  return PRISM_OK;
}

// Wave records (engine.py:227-236): launch time, duration, uncached / cached
// tokens, member offsets [W+1] and the members as trace indices, admission order.
int prism_serve_waves(prism_serve *s, double *launch, double *duration, int64_t *uncached, int64_t *cached,
                      int64_t *member_off, int32_t *members) {
  cudaSetDevice(s->dev);
  const size_t W = s->w_launch.size();
  for (size_t w = 0; w < W; w++) {
    if (launch) launch[w] = s->w_launch[w];
    if (duration) duration[w] = s->w_duration[w];
    if (uncached) uncached[w] = s->w_uncached[w];
    if (cached) cached[w] = s->w_cached[w];
  }
  if (member_off)
    for (size_t w = 0; w <= W; w++) member_off[w] = s->w_off[w];
  if (members && s->nlog)
    SCK(cudaMemcpy(members, s->log_idx, sizeof(int32_t) * (size_t)s->nlog, cudaMemcpyDeviceToHost));
  return PRISM_OK;
}

// host wall time (us) of each admitting wave, in wave order (diagnostics)
int prism_serve_wave_times(prism_serve *s, float *out_us) {
  for (size_t w = 0; w < s->w_host_us.size(); w++) out_us[w] = s->w_host_us[w];
  return PRISM_OK;
}

}  // extern "C"

// qas.cu -- the query-aware scheduler round (scheduler.py:192-273) on sm_100a.
//
// One round over a frozen pending snapshot, all passes data-parallel:
//   q_count        segment counters g (pending) / a (active) / n (dispatch)   (83-89, 205-206, 248)
//   q_align        per request: front alignment + order-sensitive signature  (109-143)
//   q_bucket_*     signature buckets in first-seen order, rank inside bucket  (211-223)
//   q_pairs/...    distinct (bucket, segment) pairs -> utility -> score       (146-171, 225-232)
//   hot fill       buckets by (-score, creation) with a prefix sum            (234-240)
//   cold lane      leftovers by (arrival, id)                                 (242-245)
//   q_prio         dispatch priorities P-hat over the counter domain          (247-251)
// Float arithmetic uses explicit round-to-nearest intrinsics (no FMA), so the
// results equal the reference's Python float expressions; bucket utility sums
// are exact whenever every term is integer-valued (the default weights).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cub/cub.cuh>
#include <string>
#include <vector>

#include "../../include/prism.h"
#include "pdl.cuh"
#include "qas_small.cuh"
#include "scan.cuh"
#include "select.cuh"

namespace {

constexpr int QMAXK = 64;
constexpr int TPB = 256;
constexpr uint64_t QEMPTY = ~0ull;
inline unsigned nblk(int64_t n) { return (unsigned)((n + TPB - 1) / TPB); }

thread_local std::string q_err;
int qfail(int code, const std::string &m) {
  q_err = m;
  prism_set_last_error(m.c_str());  // one last-error for the whole library
  return code;
}
#define QCK(x)                                                                                \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) return qfail(PRISM_CUDA, std::string("CUDA error ") + cudaGetErrorString(e_) + " in " #x); \
  } while (0)

struct QCfg {
  int64_t budget, cold, front, kappa;
  double wg, wa, wn, alpha, beta;
};

struct K3 {
  uint64_t w0, w1, w2;
};
struct K3Decomp {
  __host__ __device__ ::cuda::std::tuple<uint64_t &, uint64_t &, uint64_t &> operator()(K3 &k) const {
    return {k.w0, k.w1, k.w2};
  }
};

__device__ inline uint64_t qmix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

__device__ inline uint64_t ord_f64(double d) {
  if (d == 0.0) d = 0.0;
  const uint64_t b = (uint64_t)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// pri0(r) = w_g*g + w_a*a   (scheduler.py:208-209)
__device__ inline double pri0(const QCfg &c, const int32_t *g, const int32_t *a, int32_t s) {
  return __dadd_rn(__dmul_rn(c.wg, (double)g[s]), __dmul_rn(c.wa, (double)a[s]));
}

// count_segments: each request contributes once per distinct segment
__global__ void q_count(int64_t P, const int64_t *__restrict__ off, const int32_t *__restrict__ sk,
                        int32_t *__restrict__ cnt, const int64_t *__restrict__ subset) {
  pdl_wait();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P) return;
  const int64_t i = subset ? subset[t] : t;
  const int64_t b = off[i], e = off[i + 1];
  for (int64_t j = b; j < e; j++) {
    const int32_t s = sk[j];
    bool dup = false;
    for (int64_t q = b; q < j && !dup; q++) dup = sk[q] == s;
    if (!dup) atomicAdd(&cnt[s], 1);
  }
}

// (-pri, seg, index) ascending == pri descending, then seg, then position
__device__ inline bool rank_before(double pa, int32_t sa, int ia, double pb, int32_t sb, int ib) {
  if (pa != pb) return pa > pb;
  if (sa != sb) return sa < sb;
  return ia < ib;
}

__global__ void q_align(int64_t P, const int64_t *__restrict__ off, const int32_t *__restrict__ sk,
                        const uint8_t *__restrict__ reo, const int32_t *__restrict__ g,
                        const int32_t *__restrict__ a, QCfg c, int32_t *__restrict__ aligned,
                        int32_t *__restrict__ sig, int32_t *__restrict__ siglen,
                        uint32_t *__restrict__ sighash, int32_t *__restrict__ nlong,
                        int32_t *__restrict__ longl) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const int64_t b = off[i];
  const int k = (int)(off[i + 1] - b);
  if (k > QMAXK) {  // aligned by a whole block in q_align_long
    longl[atomicAdd(nlong, 1)] = (int32_t)i;
    return;
  }
  int32_t s[QMAXK];
  double p[QMAXK];
  int ord[QMAXK];
  for (int j = 0; j < k; j++) {
    s[j] = sk[b + j];
    p[j] = pri0(c, g, a, s[j]);
  }
  int32_t al[QMAXK];
  // front_align (scheduler.py:109-129)
  if (!reo[i] || k == 0) {
    for (int j = 0; j < k; j++) al[j] = s[j];
  } else {
    for (int j = 0; j < k; j++) {  // stable insertion sort of indices
      int q = j;
      while (q > 0 && rank_before(p[j], s[j], j, p[ord[q - 1]], s[ord[q - 1]], ord[q - 1])) {
        ord[q] = ord[q - 1];
        q--;
      }
      ord[q] = j;
    }
    const int f = (int)(c.front < k ? c.front : k);
    uint64_t chosen = 0;
    int w = 0;
    for (int q = 0; q < f; q++) {
      al[w++] = s[ord[q]];
      chosen |= 1ull << ord[q];
    }
    for (int j = 0; j < k; j++)
      if (!((chosen >> j) & 1ull)) al[w++] = s[j];
  }
  for (int j = 0; j < k; j++) aligned[b + j] = al[j];
  // make_signature (scheduler.py:132-143): top-kappa by rank, emitted in aligned order
  int sl = 0;
  if (k > 0) {
    double pa[QMAXK];
    for (int j = 0; j < k; j++) {
      pa[j] = pri0(c, g, a, al[j]);
      int q = j;
      while (q > 0 && rank_before(pa[j], al[j], j, pa[ord[q - 1]], al[ord[q - 1]], ord[q - 1])) {
        ord[q] = ord[q - 1];
        q--;
      }
      ord[q] = j;
    }
    const int kk = (int)(c.kappa < k ? c.kappa : k);
    uint64_t chosen = 0;
    for (int q = 0; q < kk; q++) chosen |= 1ull << ord[q];
    for (int j = 0; j < k; j++)
      if ((chosen >> j) & 1ull) sig[i * c.kappa + sl++] = al[j];
  }
  siglen[i] = sl;
  uint32_t h = 2166136261u ^ (uint32_t)sl;
  for (int j = 0; j < sl; j++) h = (h ^ (uint32_t)sig[i * c.kappa + j]) * 16777619u;
  sighash[i] = h;
}

// the requests q_align queued (skeletons longer than QMAXK): one block each
__global__ void q_align_long(const int32_t *__restrict__ nlong, const int32_t *__restrict__ longl,
                             const int64_t *__restrict__ off, const int32_t *__restrict__ sk,
                             const uint8_t *__restrict__ reo, const int32_t *__restrict__ g,
                             const int32_t *__restrict__ a, QCfg c, int32_t *__restrict__ aligned,
                             int32_t *__restrict__ sig, int32_t *__restrict__ siglen,
                             uint32_t *__restrict__ sighash, int32_t *__restrict__ rk) {
  pdl_wait();
  const int n = *nlong;
  for (int t = blockIdx.x; t < n; t += gridDim.x) {
    const int64_t i = longl[t];
    const int64_t b = off[i];
    const int k = (int)(off[i + 1] - b);
    const int sl = qsmall::align_long_block(sk + b, k, reo[i] != 0, g, a, c.wg, c.wa, c.front, c.kappa,
                                            aligned + b, sig + i * c.kappa, rk + b);
    if (threadIdx.x == 0) {
      siglen[i] = sl;
      uint32_t h = 2166136261u ^ (uint32_t)sl;
      for (int j = 0; j < sl; j++) h = (h ^ (uint32_t)sig[i * c.kappa + j]) * 16777619u;
      sighash[i] = h;
    }
  }
}

__device__ inline bool sig_eq(const int32_t *sig, const int32_t *siglen, int64_t kappa, int64_t x, int64_t y) {
  if (siglen[x] != siglen[y]) return false;
  for (int j = 0; j < siglen[x]; j++)
    if (sig[x * kappa + j] != sig[y * kappa + j]) return false;
  return true;
}

// signature -> bucket slot; table key = hash << 32 | representative request
__global__ void q_bucket_insert(int64_t P, const int32_t *__restrict__ sig, const int32_t *__restrict__ siglen,
                                const uint32_t *__restrict__ sighash, int64_t kappa, uint64_t *tkey,
                                int32_t *tmin, uint64_t tmask, int32_t *__restrict__ slot_of) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const uint32_t h = sighash[i];
  const uint64_t mine = ((uint64_t)h << 32) | (uint32_t)i;
  uint64_t pidx = qmix(h) & tmask;
  for (;;) {
    const unsigned long long prev = atomicCAS((unsigned long long *)&tkey[pidx], QEMPTY, mine);
    if (prev == QEMPTY) {
      atomicMin(&tmin[pidx], (int32_t)i);
      slot_of[i] = (int32_t)pidx;
      return;
    }
    if ((uint32_t)(prev >> 32) == h && sig_eq(sig, siglen, kappa, (int64_t)(prev & 0xffffffffu), i)) {
      atomicMin(&tmin[pidx], (int32_t)i);
      slot_of[i] = (int32_t)pidx;
      return;
    }
    pidx = (pidx + 1) & tmask;
  }
}

__global__ void q_bucket_list(int64_t T, const uint64_t *__restrict__ tkey, const int32_t *__restrict__ tmin,
                              int32_t *__restrict__ bmin, int32_t *__restrict__ bslot, int64_t *count) {
  pdl_wait();
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= T || tkey[p] == QEMPTY) return;
  const int64_t pos = (int64_t)atomicAdd((unsigned long long *)count, 1ull);
  bmin[pos] = tmin[p];
  bslot[pos] = (int32_t)p;
}

__global__ void q_bucket_index(int64_t nb, const int32_t *__restrict__ sorted_slot, int32_t *__restrict__ bidx_of_slot) {
  pdl_wait();
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < nb) bidx_of_slot[sorted_slot[q]] = (int32_t)q;
}

__global__ void q_bucket_of(int64_t P, const int32_t *__restrict__ slot_of, const int32_t *__restrict__ bidx_of_slot,
                            int32_t *__restrict__ bucket, int32_t *__restrict__ iota) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  bucket[i] = bidx_of_slot[slot_of[i]];
  iota[i] = (int32_t)i;
}

// sorted (bucket, index) -> bucket start / rank inside bucket
__global__ void q_rank(int64_t P, const int32_t *__restrict__ sb, const int32_t *__restrict__ si,
                       int32_t *__restrict__ bstart, int32_t *__restrict__ bend) {
  pdl_wait();
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= P) return;
  if (q == 0 || sb[q] != sb[q - 1]) bstart[sb[q]] = (int32_t)q;
  if (q == P - 1 || sb[q] != sb[q + 1]) bend[sb[q]] = (int32_t)q + 1;
}

__global__ void q_rank2(int64_t P, const int32_t *__restrict__ sb, const int32_t *__restrict__ si,
                        const int32_t *__restrict__ bstart, int32_t *__restrict__ rank) {
  pdl_wait();
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= P) return;
  rank[si[q]] = (int32_t)q - bstart[sb[q]];
}

__global__ void q_pair_count(int64_t P, const int64_t *__restrict__ off, const int32_t *__restrict__ sk,
                             int64_t *__restrict__ cnt) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const int64_t b = off[i], e = off[i + 1];
  int64_t n = 0;
  for (int64_t j = b; j < e; j++) {
    bool dup = false;
    for (int64_t q = b; q < j && !dup; q++) dup = sk[q] == sk[j];
    n += !dup;
  }
  cnt[i] = n;
}

// distinct (bucket, segment) pairs of every member; value = provisional flag
__global__ void q_pair_emit(int64_t P, const int64_t *__restrict__ off, const int32_t *__restrict__ sk,
                            const int32_t *__restrict__ bucket, const int32_t *__restrict__ rank,
                            int64_t hot_cap, const int64_t *__restrict__ pos0, uint64_t *__restrict__ pk,
                            int32_t *__restrict__ pv) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const int64_t b = off[i], e = off[i + 1];
  int64_t w = pos0[i];
  const int32_t prov = rank[i] < hot_cap ? 1 : 0;  // members[:hot_capacity] (scheduler.py:229)
  for (int64_t j = b; j < e; j++) {
    bool dup = false;
    for (int64_t q = b; q < j && !dup; q++) dup = sk[q] == sk[j];
    if (dup) continue;
    pk[w] = ((uint64_t)(uint32_t)bucket[i] << 32) | (uint32_t)sk[j];
    pv[w] = prov;
    w++;
  }
}

__global__ void q_heads(int64_t E, const uint64_t *__restrict__ pk, int32_t *__restrict__ head) {
  pdl_wait();
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < E) head[q] = (q == 0 || pk[q] != pk[q - 1]) ? 1 : 0;
}

// one thread per distinct (bucket, seg): term = w_g*g + w_a*a + w_n*n_b
__global__ void q_terms(int64_t E, const uint64_t *__restrict__ pk, const int32_t *__restrict__ head,
                        const int32_t *__restrict__ hpos, const int32_t *__restrict__ prov_pref,
                        const int32_t *__restrict__ g, const int32_t *__restrict__ a, QCfg c,
                        int32_t *__restrict__ hstart, double *__restrict__ term, int32_t *__restrict__ hbucket) {
  pdl_wait();
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= E || !head[q]) return;
  const int32_t j = hpos[q];
  hstart[j] = (int32_t)q;
  int64_t end = q + 1;
  while (end < E && !head[end]) end++;
  const int32_t nbv = prov_pref[end] - prov_pref[q];
  const int32_t r = (int32_t)(pk[q] & 0xffffffffu);
  const double t1 = __dmul_rn(c.wg, (double)g[r]);
  const double t2 = __dmul_rn(c.wa, (double)a[r]);
  const double t3 = __dmul_rn(c.wn, (double)nbv);
  term[j] = __dadd_rn(__dadd_rn(t1, t2), t3);
  hbucket[j] = (int32_t)(pk[q] >> 32);
}

__global__ void q_bucket_range(int64_t NH, const int32_t *__restrict__ hbucket, int32_t *__restrict__ hb0,
                               int32_t *__restrict__ hb1) {
  pdl_wait();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= NH) return;
  if (j == 0 || hbucket[j] != hbucket[j - 1]) hb0[hbucket[j]] = (int32_t)j;
  if (j == NH - 1 || hbucket[j] != hbucket[j + 1]) hb1[hbucket[j]] = (int32_t)j + 1;
}

// bucket_score (scheduler.py:146-171), one warp per bucket.  The sum runs in
// ascending segment order; when every term is an exact integer below 2^53
// the warp sums exactly in int64 (order-free, bit-identical).
__global__ void q_score(int64_t nb, const int32_t *__restrict__ hb0, const int32_t *__restrict__ hb1,
                        const double *__restrict__ term, const int32_t *__restrict__ bstart,
                        const int32_t *__restrict__ bend, QCfg c, double *__restrict__ score,
                        uint64_t *__restrict__ skey, int32_t *__restrict__ sval) {
  pdl_wait();
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= nb) return;
  const int32_t j0 = hb0[b], j1 = hb1[b];
  const int32_t ns = j1 - j0;
  bool integral = true;
  long long isum = 0;
  for (int32_t j = j0 + lane; j < j1; j += 32) {
    const double t = term[j];
    if (t != floor(t) || fabs(t) >= 9007199254740992.0) integral = false;
    else isum += (long long)t;
  }
  integral = __all_sync(0xffffffffu, integral);
  for (int o = 16; o > 0; o >>= 1) isum += __shfl_xor_sync(0xffffffffu, isum, o);
  double util = 0.0;
  if (ns > 0) {
    double sum;
    if (integral && llabs(isum) < 9007199254740992ll) {
      sum = (double)isum;
    } else {
      sum = 0.0;
      for (int32_t j = j0; j < j1; j++) sum = (j == j0) ? term[j] : __dadd_rn(sum, term[j]);
    }
    util = __ddiv_rn(sum, (double)ns);
  }
  const double sz = (double)(bend[b] - bstart[b]);
  const double sc = __dadd_rn(__dmul_rn(c.alpha, sz), __dmul_rn(c.beta, util));
  if (lane == 0) {
    score[b] = sc;
    skey[b] = ord_f64(-sc);  // sort (-score, creation order): stable radix sort keeps b order
    sval[b] = (int32_t)b;
  }
}

__global__ void q_sizes_sorted(int64_t nb, const int32_t *__restrict__ order, const int32_t *__restrict__ bstart,
                               const int32_t *__restrict__ bend, int64_t *__restrict__ sz) {
  pdl_wait();
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < nb) sz[q] = bend[order[q]] - bstart[order[q]];
}

__global__ void q_take(int64_t nb, const int32_t *__restrict__ order, const int64_t *__restrict__ pre,
                       const int64_t *__restrict__ sz, int64_t hot_cap, int64_t *__restrict__ take,
                       int64_t *__restrict__ base) {
  pdl_wait();
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nb) return;
  const int32_t b = order[q];
  int64_t t = hot_cap - pre[q];
  t = t < 0 ? 0 : (t > sz[q] ? sz[q] : t);
  take[b] = t;
  base[b] = pre[q] < hot_cap ? pre[q] : hot_cap;
}

__global__ void q_hot(int64_t P, const int32_t *__restrict__ bucket, const int32_t *__restrict__ rank,
                      const int64_t *__restrict__ take, const int64_t *__restrict__ base, int64_t *__restrict__ hot,
                      uint8_t *__restrict__ sel) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const int32_t b = bucket[i];
  const bool h = rank[i] < take[b];
  sel[i] = h ? 1 : 0;
  if (h) hot[base[b] + rank[i]] = i;
}

// cold-lane key: (selected, arrival, id) -- leftovers sorted by (arrival, id)
__global__ void q_cold_keys(int64_t P, const uint8_t *__restrict__ sel, const double *__restrict__ arrival,
                            const int64_t *__restrict__ ids, K3 *__restrict__ k, int64_t *__restrict__ v,
                            int64_t *__restrict__ w) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  K3 x;
  x.w0 = sel[i];
  x.w1 = ord_f64(arrival[i]);
  x.w2 = (uint64_t)ids[i] ^ 0x8000000000000000ull;
  k[i] = x;
  v[i] = i;
  w[i] = sel[i] ? 0 : 1;  // only leftovers count toward the cold quota
}

// count_segments (scheduler.py:83-89) of a pending CSR into dense G: one thread
// per request, each distinct segment once
__global__ void q_demand(int64_t P, const int64_t *__restrict__ off, const int32_t *__restrict__ sk, int32_t *G) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const int64_t b = off[i], e = off[i + 1];
  for (int64_t j = b; j < e; j++) {
    const int32_t s = sk[j];
    bool dup = false;
    for (int64_t q = b; q < j && !dup; q++) dup = sk[q] == s;
    if (!dup) atomicAdd(&G[s], 1);
  }
}

__global__ void q_prio(int32_t nseg, const int32_t *__restrict__ g, const int32_t *__restrict__ a,
                       const int32_t *__restrict__ nd, QCfg c, double *__restrict__ prio, uint8_t *__restrict__ dom) {
  pdl_wait();
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nseg) return;
  const bool in = g[r] > 0 || a[r] > 0 || nd[r] > 0;
  dom[r] = in ? 1 : 0;
  prio[r] = in ? __dadd_rn(pri0(c, g, a, r), __dmul_rn(c.wn, (double)nd[r])) : 0.0;
}

template <class T>
cudaError_t grow(T **p, int64_t &cap, int64_t need) {
  if (need <= cap && *p) return cudaSuccess;
  if (*p) cudaFree(*p);
  int64_t c = 64;
  while (c < need) c <<= 1;
  cap = c;
  return cudaMalloc((void **)p, sizeof(T) * (size_t)c);
}

}  // namespace

struct prism_qas {
  int dev = 0;
  cudaStream_t st = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  // buffers (device) with capacities
#define QAS_BUFFERS(X) \
  X(int64_t, ids) \
  X(double, arrival) \
  X(int64_t, off) \
  X(int32_t, sk) \
  X(uint8_t, reo) \
  X(int64_t, aoff) \
  X(int32_t, ask) \
  X(int32_t, g) \
  X(int32_t, a) \
  X(int32_t, nd) \
  X(double, prio) \
  X(uint8_t, dom) \
  X(int32_t, aligned) \
  X(int32_t, sig) \
  X(int32_t, siglen) \
  X(uint32_t, sighash) \
  X(int32_t, longl) \
  X(int32_t, rk) \
  X(int32_t, emap) \
  X(uint8_t, efirst) \
  X(int32_t, btake) \
  X(double, prio_glob) \
  X(uint8_t, dom_glob) \
  X(int32_t, bbase) \
  X(int64_t, gids) \
  X(int64_t, goff) \
  X(int32_t, gsfx) \
  X(double, garr) \
  X(uint8_t, greo) \
  X(int32_t, gsk) \
  X(uint64_t, tkey) \
  X(int32_t, tmin) \
  X(int32_t, slot_of) \
  X(int32_t, bmin) \
  X(int32_t, bslot) \
  X(int32_t, bmin2) \
  X(int32_t, bslot2) \
  X(int32_t, bidx_of_slot) \
  X(int32_t, bucket) \
  X(int32_t, iota) \
  X(int32_t, sb) \
  X(int32_t, si) \
  X(int32_t, bstart) \
  X(int32_t, bend) \
  X(int32_t, rank) \
  X(int64_t, pcnt) \
  X(int64_t, ppos) \
  X(uint64_t, pk) \
  X(int32_t, pv) \
  X(uint64_t, pk2) \
  X(int32_t, pv2) \
  X(int32_t, head) \
  X(int32_t, hpos) \
  X(int32_t, ppref) \
  X(int32_t, hstart) \
  X(double, term) \
  X(int32_t, hbucket) \
  X(int32_t, hb0) \
  X(int32_t, hb1) \
  X(double, score) \
  X(uint64_t, skey) \
  X(int32_t, sval) \
  X(uint64_t, skey2) \
  X(int32_t, sval2) \
  X(int64_t, ssz) \
  X(int64_t, spre) \
  X(int64_t, take) \
  X(int64_t, base) \
  X(int64_t, hot) \
  X(uint8_t, sel) \
  X(K3, ck) \
  X(int64_t, cv) \
  X(K3, ck2) \
  X(int64_t, cv2) \
  X(int64_t, small) \
  X(int32_t, err) \
  X(int64_t, tmp_tot) \
  /* fused wave step: dispatch order, serialized paths and anchors */ \
  X(int64_t, members) \
  X(int64_t, plen) \
  X(int64_t, poff) \
  X(int64_t, alen) \
  X(int64_t, aoffs) \
  X(uint32_t, tok) \
  X(int32_t, a_off) \
  X(int8_t, a_kind) \
  X(int32_t, a_seg) \
  X(int32_t, a_snap) \
  /* cold-lane selection */ \
  X(int64_t, cw0) \
  X(int64_t, cw1) \
  X(prism::Key3, ck1) \
  X(uint64_t, cv1) \
  X(prism::Key3, cks) \
  X(uint64_t, cvs) \
  X(prism::SelState, sst) \
  X(prism::Key3, sbmin) \
  X(prism::Key3, sbmax) \
  /* one-CTA rounds */ \
  X(int32_t, touched) \
  X(int32_t, tn) \
  X(int64_t, qcounts) \
  X(unsigned long long, qts)
#define QBUF(T, name) \
  T *name = nullptr;  \
  int64_t name##_cap = 0;
  QAS_BUFFERS(QBUF)
#undef QBUF
  int64_t small_max_p = qsmall::QS_MAXP;  // one-launch rounds up to this many pending
  int64_t small_grid = 0;      // CTAs of a one-launch round (0: from small_per_cta)
  int64_t small_per_cta = 24;  // pending requests per CTA when sizing the grid (4096 -> every SM)
  int32_t small_coresident = 0;
  const int32_t *gdem = nullptr;  // all-reduced demand counters feeding P-hat (nullptr: the local round's)
  int32_t gdem_n = 0;
  // pins to drop at the start of the next wave (prism_qas_defer_release): on a
  // forked stream, overlapping the QAS round, joined before the tree work
  const int32_t *rel_slots = nullptr;
  int64_t rel_n = 0;
  cudaStream_t st_rel = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_rel = nullptr;
  int64_t last_small_grid = 0;
  bool full_reset = true;
  int64_t small_rounds = 0;
  int64_t launches = 0, lib_calls = 0, rounds = 0;
  int32_t commit_mode = 0;
  int prof_on = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  double ms_round = 0.0;  // QAS round + serialization device time (events on q->st)
  // the fused wave's tail as a CUDA graph (prism_wave_step)
  cudaEvent_t ev_t = nullptr;
  uint64_t gkey_seen = 0;  // the last wave shape run without a graph (captured when it repeats)
  struct GEnt {
    uint64_t key = 0;
    cudaGraphExec_t exec = nullptr;
    int64_t kernels = 0, last = 0;
  } gcache[4];
  int64_t gtick = 0;
  int32_t use_graph = 1;
  int64_t graph_captures = 0, graph_replays = 0;
  int64_t pdl_edges = 0;  // programmatic kernel -> kernel edges of the last captured wave
  int64_t *hres = nullptr;  // pinned: the fused wave's stage results
  int64_t *hout_mem = nullptr, *hout_hit = nullptr;  // pinned: a wave's dispatch order and hits
  int64_t hout_cap = 0;
  int32_t hout_ready = 0;
};

namespace {
int ensure_tmp(prism_qas *q, size_t b) {
  if (b <= q->tmp_bytes) return PRISM_OK;
  if (q->tmp) QCK(cudaFree(q->tmp));
  q->tmp_bytes = b + b / 4 + 4096;
  QCK(cudaMalloc(&q->tmp, q->tmp_bytes));
  return PRISM_OK;
}

// round inputs, all DEVICE pointers
struct QIn {
  const int64_t *ids;
  const double *arrival;
  const int64_t *off;
  const int32_t *sk;
  const uint8_t *reo;
  const int64_t *aoff;
  const int32_t *ask;
};

int qas_run_multi(prism_qas *q, const QIn &in, int64_t P, int64_t A, int32_t nseg, const QCfg &c, int64_t *nhot,
                  int64_t *ncold, int64_t *nbuckets);

// a one-CTA round whose skeleton entries overflowed its buffers (qcounts[3]) is redone
// by the multi-kernel round, which overwrites every output and counter entry
int qas_rerun_multi(prism_qas *q, const QIn &in, int64_t P, int64_t A, int32_t nseg, const QCfg &c, int64_t *nhot,
                    int64_t *ncold, int64_t *nbuckets) {
  q->small_rounds--;
  q->rounds--;
  return qas_run_multi(q, in, P, A, nseg, c, nhot, ncold, nbuckets);
}

// the full round; outputs stay in q's device buffers
bool qas_small_eligible(const prism_qas *q, int64_t P, const QCfg &c) {
  const bool integral = c.wg == std::floor(c.wg) && c.wa == std::floor(c.wa) && c.wn == std::floor(c.wn) &&
                        std::fabs(c.wg) < 1e9 && std::fabs(c.wa) < 1e9 && std::fabs(c.wn) < 1e9;
  return P > 0 && P <= q->small_max_p && integral && c.kappa <= QMAXK;
}

// buffers (and the counter reset when they are fresh) of a one-launch round;
// returns the grid (no kernel launched)
int qas_small_prepare(prism_qas *q, int64_t P, int32_t nseg, const QCfg &c, int64_t *G_out) {
  cudaStream_t st = q->st;
  const int32_t S1 = std::max(nseg, 1);
  const int64_t gcap0 = q->g_cap;
  QCK(grow(&q->g, q->g_cap, S1));
  QCK(grow(&q->a, q->a_cap, S1));
  QCK(grow(&q->nd, q->nd_cap, S1));
  QCK(grow(&q->prio, q->prio_cap, S1));
  QCK(grow(&q->dom, q->dom_cap, S1));
  QCK(grow(&q->err, q->err_cap, 4));
  QCK(grow(&q->small, q->small_cap, 8));
  if (q->g_cap != gcap0) q->full_reset = true;  // fresh (uninitialised) counter arrays
  // the touched-segment list (this round's list, read back next round to reset
  // the counters: phase 0 consumes it before phase 1 rewrites it); growing it
  // loses the previous round's entries, so that forces a full counter reset
  const int64_t tneed = (int64_t)S1 + 1;  // distinct touched segments <= nseg
  if (tneed > q->touched_cap || !q->touched) {
    QCK(grow(&q->touched, q->touched_cap, tneed));
    q->full_reset = true;
  }
  QCK(grow(&q->tn, q->tn_cap, 2));
  if (q->full_reset) {
    QCK(cudaMemsetAsync(q->g, 0, sizeof(int32_t) * q->g_cap, st));
    QCK(cudaMemsetAsync(q->a, 0, sizeof(int32_t) * q->a_cap, st));
    QCK(cudaMemsetAsync(q->nd, 0, sizeof(int32_t) * q->nd_cap, st));
    QCK(cudaMemsetAsync(q->prio, 0, sizeof(double) * q->prio_cap, st));
    QCK(cudaMemsetAsync(q->dom, 0, (size_t)q->dom_cap, st));
    QCK(cudaMemsetAsync(q->tn, 0, 2 * sizeof(int32_t), st));
    q->full_reset = false;
  }
  QCK(grow(&q->aligned, q->aligned_cap, P * qsmall::QS_SKCAP));
  QCK(grow(&q->rk, q->rk_cap, q->aligned_cap));
  QCK(grow(&q->emap, q->emap_cap, q->aligned_cap));
  QCK(grow(&q->efirst, q->efirst_cap, q->aligned_cap));
  QCK(grow(&q->btake, q->btake_cap, P));
  QCK(grow(&q->bbase, q->bbase_cap, P));
  QCK(grow(&q->longl, q->longl_cap, P));
  QCK(grow(&q->sig, q->sig_cap, P * c.kappa));
  QCK(grow(&q->siglen, q->siglen_cap, P));
  int64_t bt = 64;
  while (bt < 2 * P) bt <<= 1;
  int64_t pt = 64;
  while (pt < 4 * P * qsmall::QS_SKCAP) pt <<= 1;  // pairs: distinct (bucket, seg) <= nsk, load <= 1/4
  QCK(grow(&q->tkey, q->tkey_cap, bt));
  QCK(grow(&q->tmin, q->tmin_cap, bt));
  QCK(grow(&q->slot_of, q->slot_of_cap, P));
  QCK(grow(&q->bmin, q->bmin_cap, P));
  QCK(grow(&q->bstart, q->bstart_cap, P));
  QCK(grow(&q->bend, q->bend_cap, P));
  QCK(grow(&q->score, q->score_cap, P));
  QCK(grow(&q->take, q->take_cap, P));
  QCK(grow(&q->rank, q->rank_cap, P));
  QCK(grow(&q->bucket, q->bucket_cap, P));
  QCK(grow(&q->hot, q->hot_cap, P));
  QCK(grow(&q->cv2, q->cv2_cap, P));
  QCK(grow(&q->pk, q->pk_cap, pt));
  QCK(grow(&q->pv, q->pv_cap, pt));
  QCK(grow(&q->qcounts, q->qcounts_cap, 8));
  if (q->prof_on) QCK(grow(&q->qts, q->qts_cap, qsmall::QS_NTS));
  if (!q->small_coresident) {
    QCK(cudaFuncSetAttribute(qsmall::k_qas_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)qsmall::QS_SMEM));
    int nsm = 0, occ = 0;
    QCK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, q->dev));
    QCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, qsmall::k_qas_small, qsmall::QS_TPB,
                                                      qsmall::QS_SMEM));
    q->small_coresident = std::max(1, nsm * occ);
  }
  // grid: one CTA for small sets (no grid barriers), else ~one CTA per
  // small_per_cta pending requests, up to every SM
  int64_t G = q->small_grid > 0 ? q->small_grid : (P + q->small_per_cta - 1) / q->small_per_cta;
  *G_out = std::max<int64_t>(1, std::min<int64_t>(G, q->small_coresident));
  return PRISM_OK;
}

// the one-launch round itself (capturable): counters reset, the kernel
int qas_small_launch(prism_qas *q, const QIn &in, int64_t P, int64_t A, int64_t bt_mask, const QCfg &c, int64_t G,
                     bool zeroed = false) {
  cudaStream_t st = q->st;
  if (!zeroed) QCK(cudaMemsetAsync(q->qcounts, 0, 8 * sizeof(int64_t), st));
  qsmall::QsArgs qa{};
  qa.P = P;
  qa.A = A;
  qa.ids = in.ids;
  qa.arrival = in.arrival;
  qa.off = in.off;
  qa.sk = in.sk;
  qa.reo = in.reo;
  qa.aoff = in.aoff;
  qa.ask = in.ask;
  qa.g = q->g;
  qa.a = q->a;
  qa.nd = q->nd;
  qa.prio = q->prio;
  qa.dom = q->dom;
  qa.touched = q->touched;
  qa.touched_n = q->tn;
  qa.prev_touched = q->touched;
  qa.aligned = q->aligned;
  qa.sig = q->sig;
  qa.siglen = q->siglen;
  qa.rank = q->rank;
  qa.bucket = q->bucket;
  qa.hot = q->hot;
  qa.cold = q->cv2;
  qa.score = q->score;
  qa.counts = q->qcounts;
  qa.btab_key = q->tkey;
  qa.btab_min = q->tmin;
  qa.slot_of = q->slot_of;
  qa.bidx = q->bmin;
  qa.bsize = q->bstart;
  qa.nsegs = q->bend;
  qa.isum = (long long *)q->take;
  qa.ptab_key = q->pk;
  qa.ptab_cap = std::min(q->pk_cap, q->pv_cap);
  qa.btab_mask = bt_mask;
  qa.longl = q->longl;
  qa.rk = q->rk;
  qa.emap = q->emap;
  qa.efirst = q->efirst;
  qa.btake = q->btake;
  qa.bbase = q->bbase;
  qa.aligned_cap = std::min(std::min(std::min(q->aligned_cap, q->rk_cap), q->emap_cap), q->efirst_cap);
  qa.ts = q->prof_on ? q->qts : nullptr;
  const qsmall::QsCfg qc{c.budget, c.cold, c.front, c.kappa, c.wg, c.wa, c.wn, c.alpha, c.beta};
  if (G == 1) {
    qsmall::k_qas_small<<<1, qsmall::QS_TPB, qsmall::QS_SMEM, st>>>(qa, qc);
  } else {
    void *args[] = {(void *)&qa, (void *)&qc};
    QCK(cudaLaunchCooperativeKernel((void *)qsmall::k_qas_small, dim3((unsigned)G), dim3(qsmall::QS_TPB), args,
                                    qsmall::QS_SMEM, st));
  }
  QCK(cudaGetLastError());
  return PRISM_OK;
}

int64_t qas_small_btmask(int64_t P) {
  int64_t bt = 64;
  while (bt < 2 * P) bt <<= 1;
  return bt - 1;
}

int qas_run(prism_qas *q, const QIn &in, int64_t P, int64_t A, int32_t nseg, const QCfg &c, int64_t *nhot, int64_t *ncold,
            int64_t *nbuckets) {
  // ---- one-launch round for small pending sets with integral weights (qas_small.cuh)
  if (qas_small_eligible(q, P, c)) {
    int64_t G = 1;
    int rc = qas_small_prepare(q, P, nseg, c, &G);
    if (rc) return rc;
    if ((rc = qas_small_launch(q, in, P, A, qas_small_btmask(P), c, G))) return rc;
    q->last_small_grid = G;
    const int64_t hot_cap = c.budget - c.cold;
    *nhot = std::min<int64_t>(std::max<int64_t>(hot_cap, 0), P);
    *ncold = std::min<int64_t>(c.cold, P - *nhot);
    *nbuckets = -1;  // on the device (qcounts[2]); the host API reads it back
    q->launches += 1;
    q->rounds++;
    q->small_rounds++;
    return PRISM_OK;
  }
  const int32_t S1 = std::max(nseg, 1);
  const int64_t gcap0 = q->g_cap;
  QCK(grow(&q->g, q->g_cap, S1));
  QCK(grow(&q->a, q->a_cap, S1));
  QCK(grow(&q->nd, q->nd_cap, S1));
  QCK(grow(&q->prio, q->prio_cap, S1));
  QCK(grow(&q->dom, q->dom_cap, S1));
  QCK(grow(&q->err, q->err_cap, 4));
  QCK(grow(&q->small, q->small_cap, 8));
  if (q->g_cap != gcap0) q->full_reset = true;
  return qas_run_multi(q, in, P, A, nseg, c, nhot, ncold, nbuckets);
}

// the multi-kernel round (any P, any skeleton length, any weights)
int qas_run_multi(prism_qas *q, const QIn &in, int64_t P, int64_t A, int32_t nseg, const QCfg &c, int64_t *nhot,
                  int64_t *ncold, int64_t *nbuckets) {
  cudaStream_t st = q->st;
  const int32_t S1 = std::max(nseg, 1);
  q->full_reset = true;  // the multi-kernel round writes every counter entry
  QCK(cudaMemsetAsync(q->g, 0, sizeof(int32_t) * S1, st));
  QCK(cudaMemsetAsync(q->a, 0, sizeof(int32_t) * S1, st));
  QCK(cudaMemsetAsync(q->nd, 0, sizeof(int32_t) * S1, st));
  QCK(cudaMemsetAsync(q->err, 0, sizeof(int32_t), st));
  const int64_t P1 = std::max<int64_t>(P, 1);
  if (P > 0) q_count<<<nblk(P), TPB, 0, st>>>(P, in.off, in.sk, q->g, nullptr);
  if (A > 0) q_count<<<nblk(A), TPB, 0, st>>>(A, in.aoff, in.ask, q->a, nullptr);
  *nhot = *ncold = *nbuckets = 0;
  if (P == 0) {
    q_prio<<<nblk(S1), TPB, 0, st>>>(nseg, q->g, q->a, q->nd, c, q->prio, q->dom);
    QCK(cudaGetLastError());
    return PRISM_OK;
  }
  int64_t nsk = 0;
  QCK(cudaMemcpyAsync(&nsk, in.off + P, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  QCK(grow(&q->aligned, q->aligned_cap, std::max<int64_t>(nsk, 1)));
  QCK(grow(&q->sig, q->sig_cap, P1 * c.kappa));
  QCK(grow(&q->siglen, q->siglen_cap, P1));
  QCK(grow(&q->sighash, q->sighash_cap, P1));
  QCK(grow(&q->longl, q->longl_cap, P1));
  QCK(grow(&q->rk, q->rk_cap, std::max<int64_t>(nsk, 1)));
  q_align<<<nblk(P), TPB, 0, st>>>(P, in.off, in.sk, in.reo, q->g, q->a, c, q->aligned, q->sig, q->siglen,
                                   q->sighash, q->err, q->longl);
  q_align_long<<<148, 256, 0, st>>>(q->err, q->longl, in.off, in.sk, in.reo, q->g, q->a, c, q->aligned, q->sig,
                                    q->siglen, q->sighash, q->rk);
  // buckets
  int64_t T = 64;
  while (T < 2 * P) T <<= 1;
  QCK(grow(&q->tkey, q->tkey_cap, T));
  QCK(grow(&q->tmin, q->tmin_cap, T));
  QCK(grow(&q->slot_of, q->slot_of_cap, P1));
  QCK(cudaMemsetAsync(q->tkey, 0xFF, sizeof(uint64_t) * T, st));
  QCK(cudaMemsetAsync(q->tmin, 0x7F, sizeof(int32_t) * T, st));
  q_bucket_insert<<<nblk(P), TPB, 0, st>>>(P, q->sig, q->siglen, q->sighash, c.kappa, q->tkey, q->tmin,
                                           (uint64_t)(T - 1), q->slot_of);
  QCK(grow(&q->bmin, q->bmin_cap, P1));
  QCK(grow(&q->bslot, q->bslot_cap, P1));
  QCK(grow(&q->bmin2, q->bmin2_cap, P1));
  QCK(grow(&q->bslot2, q->bslot2_cap, P1));
  QCK(cudaMemsetAsync(q->small, 0, sizeof(int64_t), st));
  q_bucket_list<<<nblk(T), TPB, 0, st>>>(T, q->tkey, q->tmin, q->bmin, q->bslot, q->small);
  int64_t nb = 0;
  QCK(cudaMemcpyAsync(&nb, q->small, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  QCK(cudaStreamSynchronize(st));
  size_t bytes = 0;
  QCK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, q->bmin, q->bmin2, q->bslot, q->bslot2, (int)nb, 0, 32, st));
  if (ensure_tmp(q, bytes)) return PRISM_CUDA;
  bytes = q->tmp_bytes;
  QCK(cub::DeviceRadixSort::SortPairs(q->tmp, bytes, q->bmin, q->bmin2, q->bslot, q->bslot2, (int)nb, 0, 32, st));
  QCK(grow(&q->bidx_of_slot, q->bidx_of_slot_cap, T));
  q_bucket_index<<<nblk(nb), TPB, 0, st>>>(nb, q->bslot2, q->bidx_of_slot);
  QCK(grow(&q->bucket, q->bucket_cap, P1));
  QCK(grow(&q->iota, q->iota_cap, P1));
  q_bucket_of<<<nblk(P), TPB, 0, st>>>(P, q->slot_of, q->bidx_of_slot, q->bucket, q->iota);
  // rank inside bucket: stable sort of (bucket, index)
  QCK(grow(&q->sb, q->sb_cap, P1));
  QCK(grow(&q->si, q->si_cap, P1));
  bytes = 0;
  QCK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, q->bucket, q->sb, q->iota, q->si, (int)P, 0, 32, st));
  if (ensure_tmp(q, bytes)) return PRISM_CUDA;
  bytes = q->tmp_bytes;
  QCK(cub::DeviceRadixSort::SortPairs(q->tmp, bytes, q->bucket, q->sb, q->iota, q->si, (int)P, 0, 32, st));
  QCK(grow(&q->bstart, q->bstart_cap, std::max<int64_t>(nb, 1)));
  QCK(grow(&q->bend, q->bend_cap, std::max<int64_t>(nb, 1)));
  QCK(grow(&q->rank, q->rank_cap, P1));
  q_rank<<<nblk(P), TPB, 0, st>>>(P, q->sb, q->si, q->bstart, q->bend);
  q_rank2<<<nblk(P), TPB, 0, st>>>(P, q->sb, q->si, q->bstart, q->rank);
  // distinct (bucket, segment) pairs
  const int64_t hot_cap = c.budget - c.cold;
  QCK(grow(&q->pcnt, q->pcnt_cap, P1 + 1));
  QCK(grow(&q->ppos, q->ppos_cap, P1 + 1));
  QCK(cudaMemsetAsync(q->pcnt + P, 0, sizeof(int64_t), st));
  q_pair_count<<<nblk(P), TPB, 0, st>>>(P, in.off, in.sk, q->pcnt);
  bytes = 0;
  QCK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, q->pcnt, q->ppos, (int)(P + 1), st));
  if (ensure_tmp(q, bytes)) return PRISM_CUDA;
  bytes = q->tmp_bytes;
  QCK(cub::DeviceScan::ExclusiveSum(q->tmp, bytes, q->pcnt, q->ppos, (int)(P + 1), st));
  int64_t E = 0;
  QCK(cudaMemcpyAsync(&E, q->ppos + P, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  QCK(cudaStreamSynchronize(st));
  const int64_t E1 = std::max<int64_t>(E, 1);
  QCK(grow(&q->pk, q->pk_cap, E1));
  QCK(grow(&q->pv, q->pv_cap, E1));
  QCK(grow(&q->pk2, q->pk2_cap, E1));
  QCK(grow(&q->pv2, q->pv2_cap, E1));
  QCK(grow(&q->head, q->head_cap, E1 + 1));
  QCK(grow(&q->hpos, q->hpos_cap, E1 + 1));
  QCK(grow(&q->ppref, q->ppref_cap, E1 + 1));
  QCK(grow(&q->hb0, q->hb0_cap, std::max<int64_t>(nb, 1)));
  QCK(grow(&q->hb1, q->hb1_cap, std::max<int64_t>(nb, 1)));
  QCK(cudaMemsetAsync(q->hb0, 0, sizeof(int32_t) * std::max<int64_t>(nb, 1), st));
  QCK(cudaMemsetAsync(q->hb1, 0, sizeof(int32_t) * std::max<int64_t>(nb, 1), st));
  QCK(grow(&q->hstart, q->hstart_cap, E1));
  QCK(grow(&q->term, q->term_cap, E1));
  QCK(grow(&q->hbucket, q->hbucket_cap, E1));
  if (E > 0) {
    q_pair_emit<<<nblk(P), TPB, 0, st>>>(P, in.off, in.sk, q->bucket, q->rank, hot_cap, q->ppos, q->pk, q->pv);
    bytes = 0;
    QCK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, q->pk, q->pk2, q->pv, q->pv2, (int)E, 0, 64, st));
    if (ensure_tmp(q, bytes)) return PRISM_CUDA;
    bytes = q->tmp_bytes;
    QCK(cub::DeviceRadixSort::SortPairs(q->tmp, bytes, q->pk, q->pk2, q->pv, q->pv2, (int)E, 0, 64, st));
    q_heads<<<nblk(E), TPB, 0, st>>>(E, q->pk2, q->head);
    QCK(cudaMemsetAsync(q->head + E, 0, sizeof(int32_t), st));
    QCK(cudaMemsetAsync(q->pv2 + E, 0, sizeof(int32_t), st));
    bytes = 0;
    QCK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, q->head, q->hpos, (int)(E + 1), st));
    if (ensure_tmp(q, bytes)) return PRISM_CUDA;
    bytes = q->tmp_bytes;
    QCK(cub::DeviceScan::ExclusiveSum(q->tmp, bytes, q->head, q->hpos, (int)(E + 1), st));
    bytes = 0;
    QCK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, q->pv2, q->ppref, (int)(E + 1), st));
    if (ensure_tmp(q, bytes)) return PRISM_CUDA;
    bytes = q->tmp_bytes;
    QCK(cub::DeviceScan::ExclusiveSum(q->tmp, bytes, q->pv2, q->ppref, (int)(E + 1), st));
    int64_t NH = 0;
    int32_t nh32 = 0;
    QCK(cudaMemcpyAsync(&nh32, q->hpos + E, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    QCK(cudaStreamSynchronize(st));
    NH = nh32;
    q_terms<<<nblk(E), TPB, 0, st>>>(E, q->pk2, q->head, q->hpos, q->ppref, q->g, q->a, c, q->hstart, q->term,
                                     q->hbucket);
    q_bucket_range<<<nblk(NH), TPB, 0, st>>>(NH, q->hbucket, q->hb0, q->hb1);
  }
  // scores and hot lane
  QCK(grow(&q->score, q->score_cap, std::max<int64_t>(nb, 1)));
  QCK(grow(&q->skey, q->skey_cap, std::max<int64_t>(nb, 1)));
  QCK(grow(&q->sval, q->sval_cap, std::max<int64_t>(nb, 1)));
  QCK(grow(&q->skey2, q->skey2_cap, std::max<int64_t>(nb, 1)));
  QCK(grow(&q->sval2, q->sval2_cap, std::max<int64_t>(nb, 1)));
  q_score<<<nblk(nb * 32), TPB, 0, st>>>(nb, q->hb0, q->hb1, q->term, q->bstart, q->bend, c, q->score, q->skey,
                                         q->sval);
  bytes = 0;
  QCK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, q->skey, q->skey2, q->sval, q->sval2, (int)nb, 0, 64, st));
  if (ensure_tmp(q, bytes)) return PRISM_CUDA;
  bytes = q->tmp_bytes;
  QCK(cub::DeviceRadixSort::SortPairs(q->tmp, bytes, q->skey, q->skey2, q->sval, q->sval2, (int)nb, 0, 64, st));
  QCK(grow(&q->ssz, q->ssz_cap, std::max<int64_t>(nb, 1)));
  QCK(grow(&q->spre, q->spre_cap, std::max<int64_t>(nb, 1)));
  QCK(grow(&q->take, q->take_cap, std::max<int64_t>(nb, 1)));
  QCK(grow(&q->base, q->base_cap, std::max<int64_t>(nb, 1)));
  q_sizes_sorted<<<nblk(nb), TPB, 0, st>>>(nb, q->sval2, q->bstart, q->bend, q->ssz);
  bytes = 0;
  QCK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, q->ssz, q->spre, (int)nb, st));
  if (ensure_tmp(q, bytes)) return PRISM_CUDA;
  bytes = q->tmp_bytes;
  QCK(cub::DeviceScan::ExclusiveSum(q->tmp, bytes, q->ssz, q->spre, (int)nb, st));
  q_take<<<nblk(nb), TPB, 0, st>>>(nb, q->sval2, q->spre, q->ssz, hot_cap, q->take, q->base);
  QCK(grow(&q->hot, q->hot_cap, P1));
  QCK(grow(&q->sel, q->sel_cap, P1));
  q_hot<<<nblk(P), TPB, 0, st>>>(P, q->bucket, q->rank, q->take, q->base, q->hot, q->sel);
  const int64_t nh = std::min<int64_t>(std::max<int64_t>(hot_cap, 0), P);
  // cold lane
  const int64_t nc = std::min<int64_t>(c.cold, P - nh);
  QCK(grow(&q->ck, q->ck_cap, P1));
  QCK(grow(&q->cv, q->cv_cap, P1));
  QCK(grow(&q->ck2, q->ck2_cap, P1));
  QCK(grow(&q->cv2, q->cv2_cap, P1));
  if (nc > 0) {
    // the q_cold smallest (arrival, id) among the leftovers: mass-weighted
    // selection (weight 1 per leftover) then a sort of the selected few
    QCK(grow(&q->cw0, q->cw0_cap, P1));
    QCK(grow(&q->cw1, q->cw1_cap, P1));
    QCK(grow(&q->ck1, q->ck1_cap, P1));
    QCK(grow(&q->cv1, q->cv1_cap, P1));
    QCK(grow(&q->cks, q->cks_cap, P1));
    QCK(grow(&q->cvs, q->cvs_cap, P1));
    QCK(grow(&q->sst, q->sst_cap, 1));
    QCK(grow(&q->sbmin, q->sbmin_cap, 1184));
    QCK(grow(&q->sbmax, q->sbmax_cap, 1184));
    q_cold_keys<<<nblk(P), TPB, 0, st>>>(P, q->sel, in.arrival, in.ids, q->ck, q->cv, q->cw0);
    const prism::SelBufs sb{(prism::Key3 *)q->ck, q->ck1, q->cks, (uint64_t *)q->cv, q->cv1, q->cvs,
                            q->cw0, q->cw1, q->sst, q->sbmin, q->sbmax};
    int64_t nsel = 0;
    QCK(prism::sel_run(sb, P, nc, st, &nsel, &q->launches));
    if (nsel <= prism::BSORT_MAX) {
      static uint64_t attr = 0;
      if (prism::attr_once(attr)) {
        QCK(cudaFuncSetAttribute(prism::k_block_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)prism::BSORT_SMEM));
      }
      prism::k_block_sort<<<1, 1024, prism::BSORT_SMEM, st>>>(q->cks, q->cvs, (int)nsel, (prism::Key3 *)q->ck2,
                                                              (uint64_t *)q->cv2);
      q->launches++;
    } else {
      bytes = 0;
      QCK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, (K3 *)q->cks, q->ck2, (int64_t *)q->cvs, q->cv2,
                                          (int)nsel, K3Decomp{}, 0, 1 + 128, st));
      if (ensure_tmp(q, bytes)) return PRISM_CUDA;
      bytes = q->tmp_bytes;
      QCK(cub::DeviceRadixSort::SortPairs(q->tmp, bytes, (K3 *)q->cks, q->ck2, (int64_t *)q->cvs, q->cv2,
                                          (int)nsel, K3Decomp{}, 0, 1 + 128, st));
    }
    // n_disp over hot + cold (scheduler.py:247-248)
    q_count<<<nblk(nc), TPB, 0, st>>>(nc, in.off, in.sk, q->nd, q->cv2);
  }
  if (nh > 0) q_count<<<nblk(nh), TPB, 0, st>>>(nh, in.off, in.sk, q->nd, q->hot);
  q_prio<<<nblk(S1), TPB, 0, st>>>(nseg, q->g, q->a, q->nd, c, q->prio, q->dom);
  QCK(cudaGetLastError());
  *nhot = nh;
  *ncold = nc;
  *nbuckets = nb;
  // launch accounting (own kernels / CUB primitives) for bench.py's gpu_launches
  q->launches += (A > 0) + 1 + 8 + (E > 0 ? 4 : 0) + 4 + (nc > 0 ? 2 : 0) + (nh > 0) + 1;
  q->lib_calls += 3 + (E > 0 ? 3 : 0) + 2 + (nc > 0);
  q->rounds++;
  return PRISM_OK;
}
}  // namespace

extern "C" {

prism_qas *prism_qas_create(int32_t device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    qfail(PRISM_CUDA, "no CUDA device: QAS has no CPU fallback");
    return nullptr;
  }
  prism_qas *q = new prism_qas();
  q->dev = device;
  cudaSetDevice(device);
  if (cudaStreamCreateWithFlags(&q->st, cudaStreamNonBlocking) != cudaSuccess) {
    delete q;
    return nullptr;
  }
  return q;
}

void prism_qas_destroy(prism_qas *q) {
  if (!q) return;
  cudaSetDevice(q->dev);
  cudaStreamSynchronize(q->st);
#define QPTR(T, name) (void *)q->name,
  void *bufs[] = {q->tmp, QAS_BUFFERS(QPTR)};
#undef QPTR
  for (void *p : bufs)
    if (p) cudaFree(p);
  for (auto &e : q->gcache)
    if (e.exec) cudaGraphExecDestroy(e.exec);
  if (q->hres) cudaFreeHost(q->hres);
  if (q->hout_mem) cudaFreeHost(q->hout_mem);
  if (q->hout_hit) cudaFreeHost(q->hout_hit);
  if (q->ev_t) cudaEventDestroy(q->ev_t);
  if (q->ev_fork) cudaEventDestroy(q->ev_fork);
  if (q->ev_rel) cudaEventDestroy(q->ev_rel);
  if (q->st_rel) cudaStreamDestroy(q->st_rel);
  if (q->e0) cudaEventDestroy(q->e0);
  if (q->e1) cudaEventDestroy(q->e1);
  cudaStreamDestroy(q->st);
  delete q;
}

int prism_qas_round(prism_qas *q, int64_t P, const int64_t *ids, const double *arrival, const int64_t *sk_off,
                    const int32_t *sk, const uint8_t *reorderable, int64_t A, const int64_t *act_off,
                    const int32_t *act_sk, int32_t nseg, const prism_qas_config *cfg, int64_t *hot, int64_t *nhot,
                    int64_t *cold, int64_t *ncold, int32_t *aligned, int32_t *sig, int32_t *siglen,
                    int64_t *rank, int64_t *bucket, double *bscore, int64_t *nbuckets, int32_t *g, int32_t *a,
                    int32_t *nd, double *prio, uint8_t *dom) {
  if (cfg->cold_quota > cfg->dispatch_budget || cfg->signature_size < 1 ||
      cfg->front_width < cfg->signature_size)
    return qfail(PRISM_INVALID, "invalid SchedulerConfig");
  if (cfg->signature_size > QMAXK) return qfail(PRISM_INVALID, "signature_size too large");
  cudaSetDevice(q->dev);
  cudaStream_t st = q->st;
  const int64_t P1 = std::max<int64_t>(P, 1), A1 = std::max<int64_t>(A, 1);
  const int64_t nsk = sk_off[P], nask = act_off[A];
  for (int64_t j = 0; j < nsk; j++)
    if (sk[j] < 0 || sk[j] >= nseg) return qfail(PRISM_INVALID, "segment id out of range");
  for (int64_t j = 0; j < nask; j++)
    if (act_sk[j] < 0 || act_sk[j] >= nseg) return qfail(PRISM_INVALID, "segment id out of range");
  QCK(grow(&q->ids, q->ids_cap, P1));
  QCK(grow(&q->arrival, q->arrival_cap, P1));
  QCK(grow(&q->off, q->off_cap, P1 + 1));
  QCK(grow(&q->sk, q->sk_cap, std::max<int64_t>(nsk, 1)));
  QCK(grow(&q->reo, q->reo_cap, P1));
  QCK(grow(&q->aoff, q->aoff_cap, A1 + 1));
  QCK(grow(&q->ask, q->ask_cap, std::max<int64_t>(nask, 1)));
  if (P) {
    QCK(cudaMemcpyAsync(q->ids, ids, sizeof(int64_t) * P, cudaMemcpyHostToDevice, st));
    QCK(cudaMemcpyAsync(q->arrival, arrival, sizeof(double) * P, cudaMemcpyHostToDevice, st));
    QCK(cudaMemcpyAsync(q->reo, reorderable, P, cudaMemcpyHostToDevice, st));
  }
  QCK(cudaMemcpyAsync(q->off, sk_off, sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice, st));
  if (nsk) QCK(cudaMemcpyAsync(q->sk, sk, sizeof(int32_t) * nsk, cudaMemcpyHostToDevice, st));
  QCK(cudaMemcpyAsync(q->aoff, act_off, sizeof(int64_t) * (A + 1), cudaMemcpyHostToDevice, st));
  if (nask) QCK(cudaMemcpyAsync(q->ask, act_sk, sizeof(int32_t) * nask, cudaMemcpyHostToDevice, st));
  QCfg c{cfg->dispatch_budget, cfg->cold_quota, cfg->front_width, cfg->signature_size,
         cfg->w_g, cfg->w_a, cfg->w_n, cfg->alpha_size, cfg->beta_util};
  const QIn in{q->ids, q->arrival, q->off, q->sk, q->reo, q->aoff, q->ask};
  int rc = qas_run(q, in, P, A, nseg, c, nhot, ncold, nbuckets);
  if (rc) return rc;
  if (*nbuckets < 0) {  // one-CTA round: counts live on the device
    int64_t qc[4];
    QCK(cudaMemcpyAsync(qc, q->qcounts, sizeof(qc), cudaMemcpyDeviceToHost, st));
    QCK(cudaStreamSynchronize(st));
    if (qc[3]) {
      if ((rc = qas_rerun_multi(q, in, P, A, nseg, c, nhot, ncold, nbuckets))) return rc;
    } else {
      *nbuckets = qc[2];
    }
  }
  if (*nhot) QCK(cudaMemcpyAsync(hot, q->hot, sizeof(int64_t) * *nhot, cudaMemcpyDeviceToHost, st));
  if (*ncold) QCK(cudaMemcpyAsync(cold, q->cv2, sizeof(int64_t) * *ncold, cudaMemcpyDeviceToHost, st));
  if (P) {
    if (nsk) QCK(cudaMemcpyAsync(aligned, q->aligned, sizeof(int32_t) * nsk, cudaMemcpyDeviceToHost, st));
    QCK(cudaMemcpyAsync(sig, q->sig, sizeof(int32_t) * P * cfg->signature_size, cudaMemcpyDeviceToHost, st));
    QCK(cudaMemcpyAsync(siglen, q->siglen, sizeof(int32_t) * P, cudaMemcpyDeviceToHost, st));
    std::vector<int32_t> r32((size_t)P), b32((size_t)P);
    QCK(cudaMemcpyAsync(r32.data(), q->rank, sizeof(int32_t) * P, cudaMemcpyDeviceToHost, st));
    QCK(cudaMemcpyAsync(b32.data(), q->bucket, sizeof(int32_t) * P, cudaMemcpyDeviceToHost, st));
    if (*nbuckets) QCK(cudaMemcpyAsync(bscore, q->score, sizeof(double) * *nbuckets, cudaMemcpyDeviceToHost, st));
    QCK(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < P; i++) {
      rank[i] = r32[i];
      bucket[i] = b32[i];
    }
  }
  if (nseg > 0) {
    QCK(cudaMemcpyAsync(g, q->g, sizeof(int32_t) * nseg, cudaMemcpyDeviceToHost, st));
    QCK(cudaMemcpyAsync(a, q->a, sizeof(int32_t) * nseg, cudaMemcpyDeviceToHost, st));
    QCK(cudaMemcpyAsync(nd, q->nd, sizeof(int32_t) * nseg, cudaMemcpyDeviceToHost, st));
    QCK(cudaMemcpyAsync(prio, q->prio, sizeof(double) * nseg, cudaMemcpyDeviceToHost, st));
    QCK(cudaMemcpyAsync(dom, q->dom, (size_t)nseg, cudaMemcpyDeviceToHost, st));
  }
  QCK(cudaStreamSynchronize(st));
  return PRISM_OK;
}

}  // extern "C"

// ===================================================================== fused wave
// The engine's per-wave hand-off (engine.py:189-213) without leaving the GPU:
// QAS round -> dispatch order -> serialize_tokens with the aligned skeleton
// (workload.py:136-164, K1) -> _build_anchors with the round's counter
// snapshots (engine.py:269-292) -> protection / active-set hand-off ->
// ordered admission (match + insert + evict per member).
namespace {

constexpr uint64_t SEGMENT_TOKEN_BASE = 1000000ull;
constexpr uint64_t SUFFIX_TOKEN_BASE = 2000000000ull;

// the fused wave's per-call inputs copied into fixed buffers (a CUDA graph of
// the wave reads those); abort when the skeletons exceed the staged capacity
__global__ void q_stage(int64_t P, const int64_t *__restrict__ ids, const double *__restrict__ arr,
                        const int64_t *__restrict__ off, const int32_t *__restrict__ sk,
                        const uint8_t *__restrict__ reo, const int32_t *__restrict__ sfx, int64_t *__restrict__ gids,
                        double *__restrict__ garr, int64_t *__restrict__ goff, int32_t *__restrict__ gsk,
                        uint8_t *__restrict__ greo, int32_t *__restrict__ gsfx, int64_t skcap, int32_t *abort,
                        int64_t *__restrict__ qcounts, int32_t *__restrict__ err0) {
  pdl_wait();
  const int64_t nsk = off[P];
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = gt; i <= P; i += gs) {
    goff[i] = off[i];
    if (i < P) {
      gids[i] = ids[i];
      garr[i] = arr[i];
      greo[i] = reo[i];
      gsfx[i] = sfx[i];
    }
  }
  const int64_t n = nsk < skcap ? nsk : skcap;
  for (int64_t e = gt; e < n; e += gs) gsk[e] = sk[e];
  if (gt == 0) {
    *abort = nsk > skcap ? 1 : 0;
    // the wave graph's counters (no memset nodes in the graph)
    for (int q = 0; q < 8; q++) qcounts[q] = 0;
    *err0 = 0;
  }
}

// the wave graph's results straight into pinned host memory (one kernel node
// instead of a copy node per array): the round's counters and verdicts, and
// (host entry) the dispatch order and hits
__global__ void q_results(const int64_t *__restrict__ qcounts, const int64_t *__restrict__ tot,
                          const int32_t *__restrict__ err, int64_t *hres, int64_t B,
                          const int64_t *__restrict__ members, const int64_t *__restrict__ hits, int64_t *hm,
                          int64_t *hh) {
  pdl_wait();
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
  if (gt == 0) {
    hres[0] = qcounts[2];
    hres[1] = qcounts[3];
    hres[2] = tot[0];
    hres[3] = tot[1];
    reinterpret_cast<int32_t *>(hres + 4)[0] = err[0];
    reinterpret_cast<int32_t *>(hres + 4)[1] = err[1];
  }
  if (hm)
    for (int64_t i = gt; i < B; i += gs) {
      hm[i] = members[i];
      hh[i] = hits[i];
    }
}

// the wave's dispatch order (hot lane, then cold) with each member's path and
// anchor counts, and the uint32 token-layout check of its private suffix
// (workload.py:147-154), before anything is serialised
__global__ void q_members_len(int64_t nh, int64_t nc, const int64_t *__restrict__ hot,
                              const int64_t *__restrict__ cold, const int64_t *__restrict__ ids,
                              const int64_t *__restrict__ off, const int32_t *__restrict__ suffix, int64_t sys,
                              int64_t chunk, int64_t *__restrict__ members, int64_t *__restrict__ plen,
                              int64_t *__restrict__ alen, int32_t *err, const int64_t *redo = nullptr) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nh + nc) return;
  if (redo && *redo) return;  // the one-launch round overflowed: no dispatch order to read (redone)
  const int64_t m = i < nh ? hot[i] : cold[i - nh];
  members[i] = m;
  const int64_t k = off[m + 1] - off[m], sfx = suffix[m];
  plen[i] = sys + k * chunk + sfx;
  alen[i] = (sys > 0 ? 1 : 0) + k + (sfx > 0 ? 1 : 0);
  if (SUFFIX_TOKEN_BASE + (uint64_t)ids[m] * (uint64_t)sfx + (uint64_t)sfx > 0xFFFFFFFFull) *err = 2;
}

// exclusive scans plen -> poff and alen -> aoffs over B + 1 entries (the last
// input entry is 0) and their totals, one CTA
__global__ void __launch_bounds__(1024) q_scan2(int64_t B, const int64_t *__restrict__ plen,
                                                const int64_t *__restrict__ alen, int64_t *__restrict__ poff,
                                                int64_t *__restrict__ aoffs, int64_t *__restrict__ tot) {
  pdl_wait();
  prism::block_scan4<2, 8>(
      B + 1, [&](int a, int64_t i) -> int64_t { return i >= B ? 0 : (a == 0 ? plen[i] : alen[i]); },
      [&](int a, int64_t i, int64_t ex, int64_t) {
        (a == 0 ? poff : aoffs)[i] = ex;
        if (i == B) tot[a] = ex;
      });
}

// the fused wave's member stage in one CTA: q_members_len, q_scan2 and
// q_capcheck (three dependent launches) as one
__global__ void __launch_bounds__(1024) q_members_scan(int64_t nh, int64_t nc, const int64_t *__restrict__ hot,
                                                       const int64_t *__restrict__ cold,
                                                       const int64_t *__restrict__ ids, const int64_t *__restrict__ off,
                                                       const int32_t *__restrict__ suffix, int64_t sys, int64_t chunk,
                                                       int64_t *__restrict__ members, int64_t *__restrict__ plen,
                                                       int64_t *__restrict__ alen, int64_t *__restrict__ poff,
                                                       int64_t *__restrict__ aoffs, int64_t *__restrict__ tot,
                                                       const int64_t *__restrict__ qcounts, int64_t tok_cap,
                                                       int64_t anc_cap, int32_t *err, int32_t *abort) {
  pdl_wait();
  const int64_t B = nh + nc;
  if (qcounts[3]) {  // the one-launch round overflowed its buffers: no dispatch order (uniform)
    if (threadIdx.x == 0) {
      *abort = 1;
      tot[0] = tot[1] = 0;  // (the host sizes the serialization buffers from these)
    }
    return;
  }
  __shared__ int s_err;
  if (threadIdx.x == 0) s_err = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < B; i += blockDim.x) {
    const int64_t m = i < nh ? hot[i] : cold[i - nh];
    members[i] = m;
    const int64_t k = off[m + 1] - off[m], sfx = suffix[m];
    plen[i] = sys + k * chunk + sfx;
    alen[i] = (sys > 0 ? 1 : 0) + k + (sfx > 0 ? 1 : 0);
    if (SUFFIX_TOKEN_BASE + (uint64_t)ids[m] * (uint64_t)sfx + (uint64_t)sfx > 0xFFFFFFFFull) s_err = 2;
  }
  __syncthreads();  // (the CTA's global writes are visible to the CTA after the barrier)
  prism::block_scan4<2, 8>(
      B + 1, [&](int a, int64_t i) -> int64_t { return i >= B ? 0 : (a == 0 ? plen[i] : alen[i]); },
      [&](int a, int64_t i, int64_t ex, int64_t) {
        (a == 0 ? poff : aoffs)[i] = ex;
        if (i == B) tot[a] = ex;
      });
  if (threadIdx.x == 0) {  // block_scan4 ends on a barrier: tot is visible
    if (s_err) *err = s_err;
    if (qcounts[3] || *err || tot[0] > tok_cap || tot[1] > anc_cap) *abort = 1;
  }
  pdl_trace_end();
}

// one warp per member: token path and anchors
__global__ void q_serialize(int64_t B, const int64_t *__restrict__ members, const int64_t *__restrict__ ids,
                            const int64_t *__restrict__ off, const int32_t *__restrict__ aligned,
                            const int32_t *__restrict__ suffix, int64_t sys, int64_t chunk,
                            const int32_t *__restrict__ g, const int32_t *__restrict__ a,
                            const int32_t *__restrict__ nd, const int64_t *__restrict__ poff,
                            const int64_t *__restrict__ aoffs, uint32_t *__restrict__ tok,
                            int32_t *__restrict__ a_off, int8_t *__restrict__ a_kind, int32_t *__restrict__ a_seg,
                            int32_t *__restrict__ a_snap, int32_t *__restrict__ err,
                            const int32_t *abort = nullptr) {
  pdl_wait();
  if (abort && *abort) return;  // (the fused wave's stage failed: sizes may exceed the buffers)
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= B) return;
  const int64_t m = members[w], b = off[m], k = off[m + 1] - b, sfx = suffix[m];
  uint32_t *p = tok + poff[w];
  for (int64_t j = lane; j < sys; j += 32) p[j] = (uint32_t)j;
  // segment tokens: 32 segment ids at a time in registers (one load per lane),
  // then each segment's chunk tokens across the lanes (no per-token division)
  for (int64_t q0 = 0; q0 < k; q0 += 32) {
    const int64_t rl = q0 + lane < k ? aligned[b + q0 + lane] : 0;
    const int64_t nq = k - q0 < 32 ? k - q0 : 32;
    for (int64_t q = 0; q < nq; q++) {
      const int64_t r = __shfl_sync(0xffffffffu, rl, (int)q);
      uint32_t *dst = p + sys + (q0 + q) * chunk;
      const uint64_t base = SEGMENT_TOKEN_BASE + (uint64_t)r * chunk;
      for (int64_t jj = lane; jj < chunk; jj += 32) dst[jj] = (uint32_t)(base + jj);
    }
  }
  const uint64_t sb = SUFFIX_TOKEN_BASE + (uint64_t)ids[m] * (uint64_t)sfx;  // (checked by q_members_len)
  for (int64_t j = lane; j < sfx; j += 32) p[sys + k * chunk + j] = (uint32_t)(sb + j);
  // anchors (_build_anchors, engine.py:269-292): lane j the j-th segment's
  // (its counter snapshot loads in parallel over the lanes)
  const int64_t q0 = aoffs[w] + (sys > 0 ? 1 : 0);
  if (lane == 0 && sys > 0) {
    const int64_t q = q0 - 1;
    a_off[q] = (int32_t)sys;
    a_kind[q] = 0;  // SYSTEM
    a_seg[q] = (int32_t)0x80000000;
    a_snap[3 * q] = a_snap[3 * q + 1] = a_snap[3 * q + 2] = 0;
  }
  for (int64_t j = lane; j < k; j += 32) {
    const int64_t q = q0 + j;
    const int32_t r = aligned[b + j];
    a_off[q] = (int32_t)(sys + (j + 1) * chunk);
    a_kind[q] = 1;  // REUSABLE, counter snapshot (g, a, n) of its segment
    a_seg[q] = r;
    a_snap[3 * q] = g[r];
    a_snap[3 * q + 1] = a[r];
    a_snap[3 * q + 2] = nd[r];
  }
  if (lane == 0 && sfx > 0) {
    const int64_t q = q0 + k;
    a_off[q] = (int32_t)(sys + k * chunk + sfx);
    a_kind[q] = 2;  // PRIVATE
    a_seg[q] = (int32_t)0x80000000;
    a_snap[3 * q] = a_snap[3 * q + 1] = a_snap[3 * q + 2] = 0;
  }
  pdl_trace_end();
}



}  // namespace

extern "C" {

void *prism_qas_stream(prism_qas *q) { return (void *)q->st; }

// out[4]: own kernel launches, CUB primitive calls, rounds, round device-us
int prism_qas_counts(prism_qas *q, int64_t *out) {
  out[0] = q->launches;
  out[1] = q->lib_calls;
  out[2] = q->rounds;
  out[3] = (int64_t)(q->ms_round * 1000.0);
  return PRISM_OK;
}

int prism_qas_profile(prism_qas *q, int32_t enable) {
  cudaSetDevice(q->dev);
  if (enable && !q->e0) {
    QCK(cudaEventCreate(&q->e0));
    QCK(cudaEventCreate(&q->e1));
  }
  q->prof_on = enable ? 1 : 0;
  return PRISM_OK;
}

int prism_qas_small_timeline(prism_qas *q, int64_t *out_ns, int32_t n) {
  cudaSetDevice(q->dev);
  if (!q->qts) return qfail(PRISM_INVALID, "no profiled one-CTA round yet");
  unsigned long long t[qsmall::QS_NTS];
  QCK(cudaMemcpyAsync(t, q->qts, sizeof(t), cudaMemcpyDeviceToHost, q->st));
  QCK(cudaStreamSynchronize(q->st));
  for (int i = 0; i < n && i < qsmall::QS_NTS; i++) out_ns[i] = (int64_t)(t[i] - t[0]);
  return PRISM_OK;
}

int prism_qas_defer_release(prism_qas *q, int64_t n, const int32_t *slots) {
  if (n < 0) return qfail(PRISM_INVALID, "negative release count");
  q->rel_n = n;
  q->rel_slots = slots;
  return PRISM_OK;
}

int prism_qas_set_global_demand(prism_qas *q, const int32_t *G, int32_t nseg) {
  if (G && nseg <= 0) return qfail(PRISM_INVALID, "global demand needs nseg > 0");
  q->gdem = G;
  q->gdem_n = G ? nseg : 0;
  return PRISM_OK;
}

int prism_qas_demand(prism_qas *q, int64_t P, const int64_t *sk_off, const int32_t *sk, int32_t nseg, int32_t *G) {
  cudaSetDevice(q->dev);
  QCK(cudaMemsetAsync(G, 0, sizeof(int32_t) * (size_t)nseg, q->st));
  if (P > 0) q_demand<<<nblk(P), TPB, 0, q->st>>>(P, sk_off, sk, G);
  QCK(cudaGetLastError());
  q->launches++;
  return PRISM_OK;
}

int prism_qas_counters(prism_qas *q, int32_t *dst, int32_t nseg) {
  cudaSetDevice(q->dev);
  if (nseg > q->g_cap) return qfail(PRISM_INVALID, "nseg exceeds the last round's counter vector");
  if (nseg > 0) QCK(cudaMemcpyAsync(dst, q->g, sizeof(int32_t) * nseg, cudaMemcpyDeviceToDevice, q->st));
  return PRISM_OK;
}

int prism_qas_round_device(prism_qas *q, int64_t P, const int64_t *ids, const double *arrival,
                           const int64_t *sk_off, const int32_t *sk, const uint8_t *reorderable, int64_t A,
                           const int64_t *act_off, const int32_t *act_sk, int32_t nseg,
                           const prism_qas_config *cfg, int64_t *nhot, int64_t *ncold, int64_t *nbuckets) {
  if (cfg->cold_quota > cfg->dispatch_budget || cfg->signature_size < 1 ||
      cfg->front_width < cfg->signature_size || cfg->signature_size > QMAXK)
    return qfail(PRISM_INVALID, "invalid SchedulerConfig");
  cudaSetDevice(q->dev);
  QCfg c{cfg->dispatch_budget, cfg->cold_quota, cfg->front_width, cfg->signature_size,
         cfg->w_g, cfg->w_a, cfg->w_n, cfg->alpha_size, cfg->beta_util};
  const QIn in{ids, arrival, sk_off, sk, reorderable, act_off, act_sk};
  int rc = qas_run(q, in, P, A, nseg, c, nhot, ncold, nbuckets);
  if (rc || *nbuckets >= 0) return rc;
  int64_t qc[4];  // one-CTA round: bucket count and the redo flag
  QCK(cudaMemcpyAsync(qc, q->qcounts, sizeof(qc), cudaMemcpyDeviceToHost, q->st));
  QCK(cudaStreamSynchronize(q->st));
  if (qc[3]) return qas_rerun_multi(q, in, P, A, nseg, c, nhot, ncold, nbuckets);
  *nbuckets = qc[2];
  return PRISM_OK;
}

}  // extern "C"

namespace {
// The whole fused wave -- QAS round, dispatch order, protection (tree's
// auxiliary stream), serialization, pre-match and the device-driven commit --
// as ONE stream of launches with one host wait at the end; captured once per
// wave shape and replayed as a CUDA graph.  The per-call inputs are staged
// into fixed buffers first.  *handled = false: the stage failed on the device
// (buffers too small, the one-launch round overflowed, layout check) and
// nothing was committed -- the caller runs the regular path.
// Kernel -> kernel edges of a captured wave become programmatic (pdl.cuh): the
// downstream kernel's CTAs launch once every upstream CTA has begun and wait
// in pdl_wait() for its completion, so no edge pays a launch latency.  Not
// into cooperative kernels (their grid needs the whole device at once) nor
// into or out of library (CUB) kernels, which do not wait.  PRISM_NO_PDL=1
// keeps plain edges (A/B measurement).
static int graph_pdl(cudaGraph_t g, int64_t *nconv) {
  *nconv = 0;
  static const bool off = getenv("PRISM_NO_PDL") != nullptr;
  if (off) return 0;
  size_t ne = 0;
  if (cudaGraphGetEdges_v2(g, nullptr, nullptr, nullptr, &ne) != cudaSuccess) return -1;
  std::vector<cudaGraphNode_t> from(ne), to(ne);
  std::vector<cudaGraphEdgeData> ed(ne);
  if (cudaGraphGetEdges_v2(g, from.data(), to.data(), ed.data(), &ne) != cudaSuccess) return -1;
  auto ours = [](cudaGraphNode_t n, bool down) -> bool {
    cudaGraphNodeType ty;
    if (cudaGraphNodeGetType(n, &ty) != cudaSuccess || ty != cudaGraphNodeTypeKernel) return false;
    cudaKernelNodeParams p;
    if (cudaGraphKernelNodeGetParams(n, &p) != cudaSuccess) return false;
    const char *name = nullptr;
    if (cudaFuncGetName(&name, p.func) != cudaSuccess || !name) return false;
    if (strstr(name, "cub") || strstr(name, "thrust")) return false;
    if (down) {
      cudaLaunchAttributeValue v{};
      if (cudaGraphKernelNodeGetAttribute(n, cudaLaunchAttributeCooperative, &v) != cudaSuccess || v.cooperative)
        return false;
    }
    return true;
  };
  for (size_t e = 0; e < ne; e++) {
    if (ed[e].type != cudaGraphDependencyTypeDefault || ed[e].from_port != 0) continue;
    if (!ours(from[e], false) || !ours(to[e], true)) continue;
    cudaGraphEdgeData nd{};
    nd.from_port = cudaGraphKernelNodePortProgrammatic;  // (no early trigger: when every upstream CTA has exited)
    nd.type = cudaGraphDependencyTypeProgrammatic;
    if (cudaGraphRemoveDependencies_v2(g, &from[e], &to[e], &ed[e], 1) != cudaSuccess) return -1;
    if (cudaGraphAddDependencies_v2(g, &from[e], &to[e], &nd, 1) != cudaSuccess) {
      cudaGetLastError();
      return cudaGraphAddDependencies_v2(g, &from[e], &to[e], &ed[e], 1) == cudaSuccess ? 0 : -1;  // (as it was)
    }
    (*nconv)++;
  }
  return 0;
}

int wave_step_graph(prism_tree *t, prism_qas *q, int64_t P, const int64_t *ids, const double *arrival,
                    const int64_t *sk_off, const int32_t *sk, const uint8_t *reorderable, const int32_t *suffix,
                    int32_t nseg, const QCfg &c, int64_t sys_len, int64_t chunk, int64_t *members_out, int64_t *hits,
                    int32_t *leaf_slots, int64_t *leaf_ids, int64_t *n_members, int64_t *n_admitted, bool *handled,
                    bool host_out) {
  *handled = false;
  cudaStream_t st = q->st;
  int64_t G = 1;
  int rc = qas_small_prepare(q, P, nseg, c, &G);
  if (rc) return rc;
  const int64_t hot_cap = c.budget - c.cold;
  const int64_t nh = std::min<int64_t>(std::max<int64_t>(hot_cap, 0), P);
  const int64_t nc = std::min<int64_t>(c.cold, P - nh);
  const int64_t B = nh + nc;
  if (B == 0) return PRISM_OK;
  int64_t *members = members_out;
  if (!members) {
    QCK(grow(&q->members, q->members_cap, P));
    members = q->members;
  }
  QCK(grow(&q->plen, q->plen_cap, P + 1));
  QCK(grow(&q->poff, q->poff_cap, P + 1));
  QCK(grow(&q->alen, q->alen_cap, P + 1));
  QCK(grow(&q->aoffs, q->aoffs_cap, P + 1));
  QCK(grow(&q->tmp_tot, q->tmp_tot_cap, 2));
  QCK(grow(&q->gids, q->gids_cap, P));
  QCK(grow(&q->goff, q->goff_cap, P + 1));
  QCK(grow(&q->gsfx, q->gsfx_cap, P));
  QCK(grow(&q->garr, q->garr_cap, P));
  QCK(grow(&q->greo, q->greo_cap, P));
  QCK(grow(&q->gsk, q->gsk_cap, P * qsmall::QS_SKCAP));
  // serialization buffers: every anchor a <= QS_SKCAP-segment skeleton can
  // have; paths sized from the last overflow (the stage aborts, never overflows)
  const int64_t nanc_cap = P * (qsmall::QS_SKCAP + 2);
  QCK(grow(&q->a_off, q->a_off_cap, nanc_cap));
  QCK(grow(&q->a_kind, q->a_kind_cap, nanc_cap));
  QCK(grow(&q->a_seg, q->a_seg_cap, nanc_cap));
  QCK(grow(&q->a_snap, q->a_snap_cap, 3 * nanc_cap));
  QCK(grow(&q->tok, q->tok_cap, std::max<int64_t>(P * (sys_len + 16 * chunk + 64), 1)));
  if (!q->hres) QCK(cudaMallocHost(&q->hres, 8 * sizeof(int64_t)));
  if (host_out && q->hout_cap < P) {
    if (q->hout_mem) cudaFreeHost(q->hout_mem);
    if (q->hout_hit) cudaFreeHost(q->hout_hit);
    QCK(cudaMallocHost(&q->hout_mem, sizeof(int64_t) * P));
    QCK(cudaMallocHost(&q->hout_hit, sizeof(int64_t) * P));
    q->hout_cap = P;
  }
  if (!q->ev_t) QCK(cudaEventCreateWithFlags(&q->ev_t, cudaEventDisableTiming));
  if (q->gdem) {
    if (q->gdem_n != nseg) return qfail(PRISM_INVALID, "global demand vector length != nseg");
    QCK(grow(&q->prio_glob, q->prio_glob_cap, nseg));
    QCK(grow(&q->dom_glob, q->dom_glob_cap, nseg));
  }
  if ((rc = prism_wave_commit_prepare(t, B))) return rc;
  int32_t *abort = q->err + 1;
  q_stage<<<nblk(P * 8), TPB, 0, st>>>(P, ids, arrival, sk_off, sk, reorderable, suffix, q->gids, q->garr, q->goff,
                                       q->gsk, q->greo, q->gsfx, q->gsk_cap, abort, q->qcounts, q->err);
  QCK(cudaGetLastError());
  const QIn gin{q->gids, q->garr, q->goff, q->gsk, q->greo, nullptr, nullptr};
  const int64_t btmask = qas_small_btmask(P);
  const int64_t tok_cap = q->tok_cap, anc_cap = std::min(q->a_off_cap, q->a_snap_cap / 3);
  const int64_t rel_n = q->rel_n;
  const int32_t *rel_slots = q->rel_slots;
  q->rel_n = 0;
  if (rel_n > 0 && !q->st_rel) {
    QCK(cudaStreamCreateWithFlags(&q->st_rel, cudaStreamNonBlocking));
    QCK(cudaEventCreateWithFlags(&q->ev_fork, cudaEventDisableTiming));
    QCK(cudaEventCreateWithFlags(&q->ev_rel, cudaEventDisableTiming));
  }
  auto body = [&]() -> int {
    int r;
    if (rel_n > 0) {  // the previous wave's pins drop beside the round (nothing in it reads ref counts)
      QCK(cudaEventRecord(q->ev_fork, st));
      QCK(cudaStreamWaitEvent(q->st_rel, q->ev_fork, 0));
      if ((r = prism_release_device(t, rel_n, rel_slots, nullptr, (void *)q->st_rel))) return r;
      QCK(cudaEventRecord(q->ev_rel, q->st_rel));
    }
    if ((r = qas_small_launch(q, gin, P, 0, btmask, c, G, true))) return r;  // (q_stage zeroed the counters)
    q_members_scan<<<1, 1024, 0, st>>>(nh, nc, q->hot, q->cv2, q->gids, q->goff, q->gsfx, sys_len, chunk, members,
                                       q->plen, q->alen, q->poff, q->aoffs, q->tmp_tot, q->qcounts, tok_cap,
                                       anc_cap, q->err, abort);
    const double *pri = q->prio;
    if (q->gdem) {  // P-hat from the replicas' all-reduced demand (the global-demand knob)
      q_prio<<<nblk(nseg), TPB, 0, st>>>(nseg, q->gdem, q->a, q->nd, c, q->prio_glob, q->dom_glob);
      pri = q->prio_glob;
    }
    QCK(cudaEventRecord(q->ev_t, st));  // (the protection on the tree's streams reads pri)
    QCK(cudaStreamWaitEvent((cudaStream_t)prism_tree_stream(t), q->ev_t, 0));
    // the releases, before anything reads ref counts: the protection pass /
    // eviction keys on the auxiliary stream, which the tree stream joins before
    // the build -- serialization, pre-match and the commit plan do not wait
    if (rel_n > 0 && (r = prism_tree_aux_wait(t, (void *)q->ev_rel))) return r;
    if ((r = prism_set_protection_device_async(t, pri, nseg))) return r;  // overlaps serialization
    q_serialize<<<nblk(B * 32), TPB, 0, st>>>(B, members, q->gids, q->goff, q->aligned, q->gsfx, sys_len, chunk, q->g,
                                              q->a, q->nd, q->poff, q->aoffs, q->tok, q->a_off, q->a_kind, q->a_seg,
                                              q->a_snap, q->err, abort);
    QCK(cudaGetLastError());
    if ((r = prism_wave_commit_enqueue(t, B, q->poff, q->tok, q->aoffs, q->a_kind, q->a_seg, q->a_snap, members,
                                       q->goff, q->aligned, sys_len, chunk, hits, leaf_slots, leaf_ids, (void *)st,
                                       abort)))
      return r;
    if (rel_n > 0) QCK(cudaStreamWaitEvent(st, q->ev_rel, 0));  // (joined through the tree; explicit for the capture)
    // the wave's results straight to pinned host memory (fixed buffers, mapped)
    q_results<<<host_out ? 32 : 1, TPB, 0, st>>>(q->qcounts, q->tmp_tot, q->err, q->hres, B, members, hits,
                                                 host_out ? q->hout_mem : nullptr, host_out ? q->hout_hit : nullptr);
    QCK(cudaGetLastError());
    return PRISM_OK;
  };
  uint64_t key = prism_wave_commit_key(t);
  {
    const void *ptrs[] = {members, hits, leaf_slots, leaf_ids, q->gids, q->goff, q->gsfx, q->garr, q->greo, q->gsk,
                          q->aligned, q->g, q->a, q->nd, q->prio, q->dom, q->poff, q->aoffs, q->plen, q->alen,
                          q->tok, q->a_off, q->a_kind, q->a_seg, q->a_snap, q->err, q->tmp_tot, q->qcounts, q->hres,
                          q->touched, q->tn, q->rk, q->emap, q->efirst, q->btake, q->bbase, q->gdem, q->prio_glob, q->dom_glob, rel_slots, q->st_rel, q->longl, q->sig, q->siglen, q->tkey, q->tmin,
                          q->slot_of, q->bmin, q->bstart, q->bend, q->score, q->take, q->rank, q->bucket, q->hot,
                          q->cv2, q->pk, q->pv, host_out ? q->hout_mem : nullptr,
                          host_out ? q->hout_hit : nullptr};
    const int64_t dims[] = {P, B, G, btmask, nseg, sys_len, chunk, tok_cap, anc_cap, q->pk_cap, q->pv_cap, rel_n,
                            q->aligned_cap, q->rk_cap, q->emap_cap, q->efirst_cap, (int64_t)q->prof_on};
    const double cw[] = {c.wg, c.wa, c.wn, c.alpha, c.beta, (double)c.budget, (double)c.cold, (double)c.front,
                         (double)c.kappa};
    auto mixin = [&](const void *p, size_t n) {
      for (size_t i = 0; i < n; i++) key = (key ^ ((const unsigned char *)p)[i]) * 0x100000001B3ull;
    };
    mixin(ptrs, sizeof(ptrs));
    mixin(dims, sizeof(dims));
    mixin(cw, sizeof(cw));
  }
  prism_qas::GEnt *hit = nullptr;
  for (auto &e : q->gcache)
    if (e.exec && e.key == key) hit = &e;
  if (hit) {  // a wave of a known shape: replay
    QCK(cudaGraphLaunch(hit->exec, st));
    hit->last = ++q->gtick;
    q->graph_replays++;
    q->launches += hit->kernels;
  } else if (key == q->gkey_seen) {  // second wave of this shape: capture it (LRU slot)
    static const bool dbg = getenv("PRISM_DEBUG_COMMIT") != nullptr;
    if (dbg) fprintf(stderr, "[wave] capture P=%lld B=%lld\n", (long long)P, (long long)B);
    prism_qas::GEnt *slot = &q->gcache[0];
    for (auto &e : q->gcache)
      if (!e.exec || e.last < slot->last) slot = &e;
    if (slot->exec) {
      cudaGraphExecDestroy(slot->exec);
      slot->exec = nullptr;
    }
    QCK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    const int r = body();
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(st, &g);
    if (r) return r;
    if (ce != cudaSuccess || !g) return qfail(PRISM_CUDA, std::string("wave capture: ") + cudaGetErrorString(ce));
    size_t nn = 0;  // kernel nodes: what one replay launches (launch accounting)
    QCK(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    QCK(cudaGraphGetNodes(g, nodes.data(), &nn));
    slot->kernels = 0;
    for (auto nd : nodes) {
      cudaGraphNodeType ty;
      QCK(cudaGraphNodeGetType(nd, &ty));
      slot->kernels += ty == cudaGraphNodeTypeKernel ? 1 : 0;
    }
    if (graph_pdl(g, &q->pdl_edges)) {
      cudaGraphDestroy(g);
      return qfail(PRISM_CUDA, "wave capture: programmatic edges");
    }
    QCK(cudaGraphInstantiate(&slot->exec, g, 0));
    cudaGraphDestroy(g);
    slot->key = key;
    slot->last = ++q->gtick;
    QCK(cudaGraphLaunch(slot->exec, st));
    q->graph_captures++;
    q->launches += slot->kernels;
  } else {  // first wave of this shape: plain launches
    q->gkey_seen = key;
    if ((rc = body())) return rc;
    q->launches += 4;
  }
  QCK(cudaStreamSynchronize(st));
  const int64_t *H = q->hres;
  const int32_t *herr = reinterpret_cast<const int32_t *>(H + 4);
  if (herr[1]) {  // stage aborted: nothing committed; size the buffers, the regular path redoes the wave
    if (H[2] > tok_cap) QCK(grow(&q->tok, q->tok_cap, H[2] + H[2] / 4));
    return PRISM_OK;
  }
  q->last_small_grid = G;
  q->rounds++;
  q->small_rounds++;
  int32_t applied = 0;
  int64_t nadm = 0;
  if ((rc = prism_wave_commit_finish(t, B, &applied, &nadm))) return rc;
  *handled = true;
  *n_members = B;
  if (applied) {
    *n_admitted = nadm;  // (< B: the wave stopped on a CapacityError)
    q->hout_ready = host_out ? 1 : 0;  // results already in the pinned output buffers
    return PRISM_OK;
  }
  // not committed in parallel (maintenance / whole order / exactness guard):
  // the regular path re-runs the commit on the already-serialized wave
  return prism_admit_wave_segmented(t, B, q->poff, q->tok, q->aoffs, q->a_off, q->a_kind, q->a_seg, q->a_snap,
                                    members, q->goff, q->aligned, sys_len, chunk, q->commit_mode, hits, leaf_slots,
                                    leaf_ids, n_admitted, (void *)st);
}
int wave_step_impl(prism_tree *t, prism_qas *q, int64_t P, const int64_t *ids, const double *arrival,
                   const int64_t *sk_off, const int32_t *sk, const uint8_t *reorderable, const int32_t *suffix,
                   int64_t A, const int64_t *act_off, const int32_t *act_sk, int32_t nseg,
                   const prism_qas_config *cfg, int64_t sys_len, int64_t chunk, int64_t *members_out, int64_t *hits,
                   int32_t *leaf_slots, int64_t *leaf_ids, int64_t *n_members, int64_t *n_admitted, bool host_out);
}  // namespace

extern "C" {

int prism_wave_step(prism_tree *t, prism_qas *q, int64_t P, const int64_t *ids, const double *arrival,
                    const int64_t *sk_off, const int32_t *sk, const uint8_t *reorderable, const int32_t *suffix,
                    int64_t A, const int64_t *act_off, const int32_t *act_sk, int32_t nseg,
                    const prism_qas_config *cfg, int64_t sys_len, int64_t chunk, int64_t *members_out,
                    int64_t *hits, int32_t *leaf_slots, int64_t *leaf_ids, int64_t *n_members,
                    int64_t *n_admitted) {
  q->hout_ready = 0;
  return wave_step_impl(t, q, P, ids, arrival, sk_off, sk, reorderable, suffix, A, act_off, act_sk, nseg, cfg,
                        sys_len, chunk, members_out, hits, leaf_slots, leaf_ids, n_members, n_admitted, false);
}

// The fused wave from host memory to host memory: the pending arrays (and the
// active-set CSR) may be pinned host buffers (read in place by the kernels),
// the previous wave's pins are released first, and the dispatch order and hits
// land in h_members / h_hits (copied inside the wave's graph to fixed pinned
// buffers when the wave ran as a graph).
int prism_wave_step_host(prism_tree *t, prism_qas *q, int64_t P, const int64_t *ids, const double *arrival,
                         const int64_t *sk_off, const int32_t *sk, const uint8_t *reorderable, const int32_t *suffix,
                         int64_t A, const int64_t *act_off, const int32_t *act_sk, int32_t nseg, const prism_qas_config *cfg, int64_t sys_len, int64_t chunk,
                         int64_t release_n, const int32_t *release_slots, int64_t *members_out, int64_t *hits,
                         int32_t *leaf_slots, int64_t *leaf_ids, int64_t *h_members, int64_t *h_hits,
                         int64_t *n_members, int64_t *n_admitted) {
  cudaSetDevice(q->dev);
  q->hout_ready = 0;
  int rc;
  if (release_n > 0) {  // dropped by the wave itself, beside its QAS round
    q->rel_n = release_n;
    q->rel_slots = release_slots;
  }
  if ((rc = wave_step_impl(t, q, P, ids, arrival, sk_off, sk, reorderable, suffix, A, act_off, act_sk, nseg, cfg,
                           sys_len, chunk, members_out, hits, leaf_slots, leaf_ids, n_members, n_admitted, true)))
    return rc;
  if (q->hout_ready) {
    memcpy(h_members, q->hout_mem, sizeof(int64_t) * (size_t)*n_members);
    memcpy(h_hits, q->hout_hit, sizeof(int64_t) * (size_t)*n_admitted);
  } else {  // (first wave of a shape / regular path)
    if (*n_members)
      QCK(cudaMemcpyAsync(h_members, members_out, sizeof(int64_t) * *n_members, cudaMemcpyDeviceToHost, q->st));
    if (*n_admitted)
      QCK(cudaMemcpyAsync(h_hits, hits, sizeof(int64_t) * *n_admitted, cudaMemcpyDeviceToHost, q->st));
    QCK(cudaStreamSynchronize(q->st));
  }
  return PRISM_OK;
}

}  // extern "C"

namespace {
int wave_step_impl(prism_tree *t, prism_qas *q, int64_t P, const int64_t *ids, const double *arrival,
                   const int64_t *sk_off, const int32_t *sk, const uint8_t *reorderable, const int32_t *suffix,
                   int64_t A, const int64_t *act_off, const int32_t *act_sk, int32_t nseg,
                   const prism_qas_config *cfg, int64_t sys_len, int64_t chunk, int64_t *members_out, int64_t *hits,
                   int32_t *leaf_slots, int64_t *leaf_ids, int64_t *n_members, int64_t *n_admitted, bool host_out) {
  if (cfg->cold_quota > cfg->dispatch_budget || cfg->signature_size < 1 ||
      cfg->front_width < cfg->signature_size || cfg->signature_size > QMAXK)
    return qfail(PRISM_INVALID, "invalid SchedulerConfig");
  cudaSetDevice(q->dev);
  cudaStream_t st = q->st;
  const QCfg c{cfg->dispatch_budget, cfg->cold_quota, cfg->front_width, cfg->signature_size,
               cfg->w_g, cfg->w_a, cfg->w_n, cfg->alpha_size, cfg->beta_util};
  const QIn in{ids, arrival, sk_off, sk, reorderable, act_off, act_sk};
  int64_t nh = 0, nc = 0, nb = 0;
  if (q->use_graph && !q->prof_on && A == 0 && q->commit_mode == 0 && chunk > 0 && qas_small_eligible(q, P, c) &&
      prism_tree_policy(t) == 0 && prism_tree_graphable(t)) {
    bool handled = false;
    int rc = wave_step_graph(t, q, P, ids, arrival, sk_off, sk, reorderable, suffix, nseg, c, sys_len, chunk,
                             members_out, hits, leaf_slots, leaf_ids, n_members, n_admitted, &handled, host_out);
    if (rc || handled) return rc;
  }
  if (q->rel_n > 0) {  // deferred pins (prism_qas_defer_release) not taken by the graph path
    int r2 = prism_release_device(t, q->rel_n, q->rel_slots, nullptr, (void *)st);
    q->rel_n = 0;
    if (r2) return r2;
  }
  if (q->prof_on) cudaEventRecord(q->e0, st);
  // QAS round (engine.py:189): one launch for the one-CTA/cooperative round
  int rc = qas_run(q, in, P, A, nseg, c, &nh, &nc, &nb);
  if (rc) return rc;
  // dispatch order, path/anchor sizes and their offsets; ONE host round trip
  // for the sizes, the one-launch round's redo flag and the layout check
  int64_t *members = members_out;
  const int64_t Pc = std::max<int64_t>(P, 1);
  if (!members) {
    QCK(grow(&q->members, q->members_cap, Pc));
    members = q->members;
  }
  QCK(grow(&q->plen, q->plen_cap, Pc + 1));
  QCK(grow(&q->poff, q->poff_cap, Pc + 1));
  QCK(grow(&q->alen, q->alen_cap, Pc + 1));
  QCK(grow(&q->aoffs, q->aoffs_cap, Pc + 1));
  QCK(grow(&q->err, q->err_cap, 4));
  QCK(grow(&q->tmp_tot, q->tmp_tot_cap, 2));
  for (int pass = 0; pass < 2; pass++) {
    const int64_t B = nh + nc;
    if (B > 0) {
      QCK(cudaMemsetAsync(q->err, 0, sizeof(int32_t), st));
      q_members_len<<<nblk(B), TPB, 0, st>>>(nh, nc, q->hot, q->cv2, ids, sk_off, suffix, sys_len, chunk, members,
                                             q->plen, q->alen, q->err, nb < 0 ? q->qcounts + 3 : nullptr);
      q_scan2<<<1, 1024, 0, st>>>(B, q->plen, q->alen, q->poff, q->aoffs, q->tmp_tot);
      q->launches += 2;
    }
    if (q->prof_on) cudaEventRecord(q->e1, st);  // device time of the round + dispatch order only
    int64_t hb[6] = {0, 0, 0, 0, 0, 0};  // qcounts[2..3], tokens, anchors, err
    if (nb < 0) QCK(cudaMemcpyAsync(hb, q->qcounts + 2, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    if (B > 0) {
      QCK(cudaMemcpyAsync(hb + 2, q->tmp_tot, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      QCK(cudaMemcpyAsync(hb + 4, q->err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    }
    QCK(cudaStreamSynchronize(st));
    if (nb < 0 && hb[1]) {  // the one-launch round overflowed its buffers: the multi-kernel round
      if ((rc = qas_rerun_multi(q, in, P, A, nseg, c, &nh, &nc, &nb))) return rc;
      continue;
    }
    if (q->prof_on) {
      cudaEventSynchronize(q->e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, q->e0, q->e1);
      q->ms_round += ms;
    }
    *n_members = B;
    *n_admitted = 0;
    if (B == 0) return PRISM_OK;  // engine.py:190-191
    if ((int32_t)hb[4]) return qfail(PRISM_INVALID, "token layout overflows uint32");
    const int64_t ntok = hb[2], nanc = hb[3];
    QCK(grow(&q->tok, q->tok_cap, std::max<int64_t>(ntok, 1)));
    QCK(grow(&q->a_off, q->a_off_cap, std::max<int64_t>(nanc, 1)));
    QCK(grow(&q->a_kind, q->a_kind_cap, std::max<int64_t>(nanc, 1)));
    QCK(grow(&q->a_seg, q->a_seg_cap, std::max<int64_t>(nanc, 1)));
    QCK(grow(&q->a_snap, q->a_snap_cap, 3 * std::max<int64_t>(nanc, 1)));
    if (!q->ev_t) QCK(cudaEventCreateWithFlags(&q->ev_t, cudaEventDisableTiming));
    const int32_t pol = prism_tree_policy(t);
    // protection / active hand-off (engine.py:193-197), ordered after the round
    // on the tree's stream by an event (no host wait)
    const double *pri = q->prio;
    if (pol == 0 && q->gdem) {  // P-hat from the replicas' all-reduced demand (the global-demand knob)
      if (q->gdem_n != nseg) return qfail(PRISM_INVALID, "global demand vector length != nseg");
      QCK(grow(&q->prio_glob, q->prio_glob_cap, nseg));
      QCK(grow(&q->dom_glob, q->dom_glob_cap, nseg));
      q_prio<<<nblk(nseg), TPB, 0, st>>>(nseg, q->gdem, q->a, q->nd, c, q->prio_glob, q->dom_glob);
      pri = q->prio_glob;
    }
    QCK(cudaEventRecord(q->ev_t, st));  // (the protection on the tree's streams reads pri)
    QCK(cudaStreamWaitEvent((cudaStream_t)prism_tree_stream(t), q->ev_t, 0));
    if (pol == 0) rc = prism_set_protection_device_async(t, pri, nseg);  // overlaps the serialization
    else if (pol == 2) rc = prism_note_active_device(t, q->a, q->nd, nseg);
    if (rc) return rc;
    // serialization (K1), then the admission on the tree's stream
    q_serialize<<<nblk(B * 32), TPB, 0, st>>>(B, members, ids, sk_off, q->aligned, suffix, sys_len, chunk, q->g,
                                              q->a, q->nd, q->poff, q->aoffs, q->tok, q->a_off, q->a_kind, q->a_seg,
                                              q->a_snap, q->err);
    QCK(cudaGetLastError());
    q->launches += 1;
    return prism_admit_wave_segmented(t, B, q->poff, q->tok, q->aoffs, q->a_off, q->a_kind, q->a_seg, q->a_snap,
                                      members, sk_off, q->aligned, sys_len, chunk, q->commit_mode, hits, leaf_slots,
                                      leaf_ids, n_admitted, (void *)st);
  }
  return qfail(PRISM_FATAL, "QAS round did not converge");
}
}  // namespace

extern "C" {

// rounds over <= max_p pending requests with integral weights run in one CTA
// (qas_small.cuh); 0: always the multi-kernel round; 1: the default cutoff
int prism_qas_set_small(prism_qas *q, int32_t max_p) {
  if (max_p < 0) return qfail(PRISM_INVALID, "max_p must be >= 0");
  q->small_max_p = max_p == 1 ? qsmall::QS_MAXP : std::min<int64_t>(max_p, qsmall::QS_MAXP);
  return PRISM_OK;
}

// one-launch round shape: key 0 = max pending (as prism_qas_set_small),
// 1 = CTAs (0: auto), 2 = pending requests per CTA for the auto grid;
// key 3 (read-only through out) = CTAs of the last one-launch round
int prism_qas_tune(prism_qas *q, int32_t key, int64_t value, int64_t *out) {
  switch (key) {
    case 0:
      return prism_qas_set_small(q, (int32_t)value);
    case 1:
      if (value < 0) return qfail(PRISM_INVALID, "grid must be >= 0");
      q->small_grid = value;
      return PRISM_OK;
    case 2:
      if (value < 1) return qfail(PRISM_INVALID, "per-CTA count must be >= 1");
      q->small_per_cta = value;
      return PRISM_OK;
    case 3:
      if (out) *out = q->last_small_grid;
      return PRISM_OK;
    case 4:  // the fused wave's tail as a CUDA graph (1, default) or plain launches (0)
      q->use_graph = value ? 1 : 0;
      return PRISM_OK;
    case 5:  // read-only: graph captures, graph replays (out[2]: programmatic edges of the last capture, when
             // the caller passes room for it through value = 3)
      if (out) {
        out[0] = q->graph_captures;
        out[1] = q->graph_replays;
        if (value >= 3) out[2] = q->pdl_edges;
      }
      return PRISM_OK;
    default:
      return qfail(PRISM_INVALID, "unknown QAS tunable");
  }
}

// 0: exact parallel wave commit with ordered fallback (default); 1: ordered commit only
int prism_qas_set_commit_mode(prism_qas *q, int32_t mode) {
  q->commit_mode = mode;
  return PRISM_OK;
}

}  // extern "C"

#ifdef PRISM_TRACE
// diagnostics build only (pdl.cuh): this unit's kernel start stamps
extern "C" int prism_trace_dump_qas(unsigned long long *t, char *names, int cap) {
  return prism_trace_take(t, names, cap);
}
#endif

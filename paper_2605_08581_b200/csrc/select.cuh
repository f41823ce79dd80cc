// select.cuh -- mass-weighted MSD radix selection of the smallest 192-bit keys.
//
// Given n candidates (Key3 key, uint64 value, int64 weight) find a set SEL
// that is a PREFIX of the ascending key order and whose weight reaches a
// target W (or all candidates).  Only SEL is sorted afterwards, instead of
// all n candidates:
//   * eviction order (kvcache.py:425-460): weight = edge tokens; W = the tokens
//     the wave / call must free -- a few percent of the candidates;
//   * protection (kvcache.py:375-382): weight = 1; W = protect_budget.
//
// Each round works on the still-undecided set U: a min/max reduction finds
// the highest bit where U's keys differ, a 256-bucket weighted histogram of
// the 8-bit digit below it locates the bucket where the cumulative weight
// crosses W, buckets below join SEL, the crossing bucket becomes the new U.
// Keys are unique (they end in the node id), so every round shrinks U; a
// small U is taken whole (SEL stays a prefix).  All control state lives on
// the device: the host launches a fixed number of rounds without syncing.
#pragma once
#include "prism_dev.cuh"

namespace prism {
// kernels are static: this header is included by dart.cu and qas.cu

constexpr int SEL_TPB = 256;
constexpr int SEL_ROUNDS = 12;
constexpr int64_t SEL_SMALL = 2048;  // a crossing bucket this small is taken whole

struct SelState {
  int64_t need;   // weight still needed
  int64_t nU;     // size of the undecided set (in the current U buffer)
  int64_t nSel;   // selected so far
  int64_t nUn;    // size of the next U
  int32_t shift;  // digit = bits [shift, shift+8)
  int32_t dstar;  // crossing bucket
  int32_t done;
  int32_t take_all;  // take the whole crossing bucket this round
  int32_t cur;       // which U buffer is current (0/1)
  int32_t rounds;
  int64_t small;     // a crossing bucket with at most this many keys is taken whole
  unsigned long long hist_n[256];
  long long hist_w[256];
};

__device__ inline uint32_t key_digit(const Key3 &k, int shift) {
  // bits [shift, shift+8) of the 192-bit value w0:w1:w2 (w2 least significant)
  const int word = shift >> 6, off = shift & 63;
  const uint64_t lo = word == 0 ? k.w2 : (word == 1 ? k.w1 : k.w0);
  const uint64_t hi = word == 0 ? k.w1 : (word == 1 ? k.w0 : 0ull);
  uint64_t v = lo >> off;
  if (off > 56) v |= hi << (64 - off);
  return (uint32_t)(v & 0xFFu);
}

__device__ inline int key_highbit(const Key3 &x) {  // highest set bit of a 192-bit value, -1 if zero
  if (x.w0) return 128 + 63 - __clzll((long long)x.w0);
  if (x.w1) return 64 + 63 - __clzll((long long)x.w1);
  if (x.w2) return 63 - __clzll((long long)x.w2);
  return -1;
}

// per-block min and max of U
static __global__ void k_sel_minmax(const Key3 *__restrict__ k, const SelState *st, Key3 *__restrict__ bmin,
                             Key3 *__restrict__ bmax) {
  pdl_wait();
  __shared__ Key3 smin[SEL_TPB], smax[SEL_TPB];
  const int64_t n = st->done ? 0 : st->nU;
  Key3 lo = {~0ull, ~0ull, ~0ull}, hi = {0, 0, 0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const Key3 x = k[i];
    if (key_less(x, lo)) lo = x;
    if (key_less(hi, x)) hi = x;
  }
  smin[threadIdx.x] = lo;
  smax[threadIdx.x] = hi;
  __syncthreads();
  for (int s = SEL_TPB / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      if (key_less(smin[threadIdx.x + s], smin[threadIdx.x])) smin[threadIdx.x] = smin[threadIdx.x + s];
      if (key_less(smax[threadIdx.x], smax[threadIdx.x + s])) smax[threadIdx.x] = smax[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bmin[blockIdx.x] = smin[0];
    bmax[blockIdx.x] = smax[0];
  }
}

// digit position from the global min/max; clears the histogram
static __global__ void k_sel_digit(SelState *st, const Key3 *__restrict__ bmin, const Key3 *__restrict__ bmax, int nb) {
  pdl_wait();
  __shared__ Key3 smin[SEL_TPB], smax[SEL_TPB];
  Key3 lo = {~0ull, ~0ull, ~0ull}, hi = {0, 0, 0};
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    if (key_less(bmin[i], lo)) lo = bmin[i];
    if (key_less(hi, bmax[i])) hi = bmax[i];
  }
  smin[threadIdx.x] = lo;
  smax[threadIdx.x] = hi;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    st->hist_n[i] = 0;
    st->hist_w[i] = 0;
  }
  __syncthreads();
  for (int s = SEL_TPB / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      if (key_less(smin[threadIdx.x + s], smin[threadIdx.x])) smin[threadIdx.x] = smin[threadIdx.x + s];
      if (key_less(smax[threadIdx.x], smax[threadIdx.x + s])) smax[threadIdx.x] = smax[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && !st->done) {
    const Key3 x = {smin[0].w0 ^ smax[0].w0, smin[0].w1 ^ smax[0].w1, smin[0].w2 ^ smax[0].w2};
    const int hb = key_highbit(x);
    st->shift = hb < 7 ? 0 : hb - 7;
    if (hb < 0) st->take_all = 1;  // a single key left
  }
}

static __global__ void k_sel_hist(const Key3 *__restrict__ k, const int64_t *__restrict__ w, SelState *st) {
  pdl_wait();
  __shared__ unsigned long long hn[256];
  __shared__ long long hw[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    hn[i] = 0;
    hw[i] = 0;
  }
  __syncthreads();
  const int64_t n = st->done ? 0 : st->nU;
  const int shift = st->shift;
  const int lane = threadIdx.x & 31;
  // warp-aggregated: the digits are usually heavily skewed (one bucket holds
  // most keys), so lanes with equal digits combine before one shared atomic
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const uint32_t d = i < n ? key_digit(k[i], shift) : 256u;
    const uint32_t wt = i < n ? (uint32_t)w[i] : 0u;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned wsum = __reduce_add_sync(peers, wt);
    if (d < 256u && lane == __ffs(peers) - 1) {
      atomicAdd(&hn[d], (unsigned long long)__popc(peers));
      atomicAdd((unsigned long long *)&hw[d], (unsigned long long)wsum);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    if (hn[i]) {
      atomicAdd(&st->hist_n[i], hn[i]);
      atomicAdd((unsigned long long *)&st->hist_w[i], (unsigned long long)hw[i]);
    }
  }
}

// one warp: inclusive scan of the 256 bucket weights, first bucket reaching need
static __global__ void k_sel_pick(SelState *st) {
  pdl_wait();
  if (st->done) return;
  const int lane = threadIdx.x & 31;
  if (st->take_all) {  // single key / forced
    if (lane == 0) st->dstar = 256;
    return;
  }
  long long w8[8], run = 0;
  for (int q = 0; q < 8; q++) {  // lane owns buckets [8*lane, 8*lane+8)
    run += st->hist_w[8 * lane + q];
    w8[q] = run;
  }
  long long pre = run;  // inclusive scan of lane totals
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, pre, o);
    if (lane >= o) pre += y;
  }
  const long long before = pre - run;
  const long long need = st->need;
  int dl = 256;
  for (int q = 0; q < 8; q++)
    if (before + w8[q] >= need) {
      dl = 8 * lane + q;
      break;
    }
  const unsigned m = __ballot_sync(0xffffffffu, dl < 256);
  if (!m) {  // all of U is not enough: take everything
    if (lane == 0) {
      st->dstar = 256;
      st->take_all = 1;
    }
    return;
  }
  const int src = __ffs(m) - 1;
  const int d = __shfl_sync(0xffffffffu, dl, src);
  if (lane == src) {
    const int q = d - 8 * lane;
    const long long below = before + (q ? w8[q - 1] : 0);
    st->need -= below;
    st->dstar = d;
    if ((int64_t)st->hist_n[d] <= st->small) st->take_all = 1;
  }
}

// U -> SEL (digit < d*, or the whole crossing bucket when take_all) / next U (digit == d*)
static __global__ void k_sel_split(const Key3 *__restrict__ kU, const uint64_t *__restrict__ vU, const int64_t *__restrict__ wU,
                            Key3 *__restrict__ kN, uint64_t *__restrict__ vN, int64_t *__restrict__ wN,
                            Key3 *__restrict__ kS, uint64_t *__restrict__ vS, SelState *st) {
  pdl_wait();
  const int64_t n = st->done ? 0 : st->nU;
  const int shift = st->shift, dstar = st->dstar, all = st->take_all;
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    int cls = 2;  // 0 = select, 1 = next U, 2 = drop
    Key3 x;
    if (i < n) {
      x = kU[i];
      const int d = dstar >= 256 ? 0 : (int)key_digit(x, shift);
      if (dstar >= 256 || d < dstar || (d == dstar && all)) cls = 0;
      else if (d == dstar) cls = 1;
    }
    const unsigned ms = __ballot_sync(0xffffffffu, cls == 0), mn = __ballot_sync(0xffffffffu, cls == 1);
    unsigned long long bs = 0, bn = 0;
    if (lane == 0) {
      if (ms) bs = atomicAdd((unsigned long long *)&st->nSel, (unsigned long long)__popc(ms));
      if (mn) bn = atomicAdd((unsigned long long *)&st->nUn, (unsigned long long)__popc(mn));
    }
    bs = __shfl_sync(0xffffffffu, bs, 0);
    bn = __shfl_sync(0xffffffffu, bn, 0);
    const unsigned below = (1u << lane) - 1u;
    if (cls == 0) {
      const int64_t p = (int64_t)bs + __popc(ms & below);
      kS[p] = x;
      vS[p] = vU[i];
    } else if (cls == 1) {
      const int64_t p = (int64_t)bn + __popc(mn & below);
      kN[p] = x;
      vN[p] = vU[i];
      wN[p] = wU[i];
    }
  }
}

static __global__ void k_sel_next(SelState *st) {
  pdl_wait();
  if (threadIdx.x != 0 || st->done) return;
  st->rounds++;
  if (st->take_all || st->nUn == 0) {
    st->done = 1;
    return;
  }
  st->nU = st->nUn;
  st->nUn = 0;
  st->cur ^= 1;
  if (st->rounds >= SEL_ROUNDS) st->take_all = 1;  // one more round takes the remainder
}

// after the rounds: if not done (pathological), move the remaining U into SEL
static __global__ void k_sel_flush(const Key3 *__restrict__ kU, const uint64_t *__restrict__ vU, Key3 *__restrict__ kS,
                            uint64_t *__restrict__ vS, SelState *st) {
  pdl_wait();
  if (st->done) return;
  const int64_t n = st->nU, base = st->nSel;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    kS[base + i] = kU[i];
    vS[base + i] = vU[i];
  }
}

// ---- sorting the selected set on its varying bits only
// mask = OR_i (k[i] ^ k[0]): removing bits that are constant across the set
// preserves the order, and the remaining bits usually fit 64 (class, a few
// priority bits, the tick range, the id range, the depth).
static __global__ void k_key_mask(const Key3 *__restrict__ k, int64_t n, unsigned long long *mask) {
  pdl_wait();
  __shared__ unsigned long long s0[SEL_TPB], s1[SEL_TPB], s2[SEL_TPB];
  const Key3 r = k[0];
  unsigned long long m0 = 0, m1 = 0, m2 = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const Key3 x = k[i];
    m0 |= x.w0 ^ r.w0;
    m1 |= x.w1 ^ r.w1;
    m2 |= x.w2 ^ r.w2;
  }
  s0[threadIdx.x] = m0;
  s1[threadIdx.x] = m1;
  s2[threadIdx.x] = m2;
  __syncthreads();
  for (int s = SEL_TPB / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      s0[threadIdx.x] |= s0[threadIdx.x + s];
      s1[threadIdx.x] |= s1[threadIdx.x + s];
      s2[threadIdx.x] |= s2[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    atomicOr(&mask[0], s0[0]);
    atomicOr(&mask[1], s1[0]);
    atomicOr(&mask[2], s2[0]);
  }
}

__device__ inline uint64_t pext64(uint64_t acc, uint64_t x, uint64_t m) {
  while (m) {
    const int b = 63 - __clzll((long long)m);
    acc = (acc << 1) | ((x >> b) & 1ull);
    m &= ~(1ull << b);
  }
  return acc;
}

static __global__ void k_key_compress(const Key3 *__restrict__ k, int64_t n, Key3 mask, uint64_t *__restrict__ out,
                               uint64_t *__restrict__ idx) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Key3 x = k[i];
  uint64_t a = pext64(0, x.w0, mask.w0);
  a = pext64(a, x.w1, mask.w1);
  a = pext64(a, x.w2, mask.w2);
  out[i] = a;
  idx[i] = (uint64_t)i;
}

static __global__ void k_key_gather(const Key3 *__restrict__ kin, const uint64_t *__restrict__ vin,
                             const uint64_t *__restrict__ order, int64_t n, Key3 *__restrict__ kout,
                             uint64_t *__restrict__ vout) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t j = order[i];
  kout[i] = kin[j];
  vout[i] = vin[j];
}

static __global__ void k_sel_flush_done(SelState *st) {
  pdl_wait();
  if (threadIdx.x == 0 && !st->done) {
    st->nSel += st->nU;
    st->done = 1;
  }
}

// single-CTA bitonic sort of n <= 4096 (Key3, value) pairs in shared memory
constexpr int BSORT_MAX = 4096;
static __global__ void __launch_bounds__(1024) k_block_sort(const Key3 *__restrict__ kin, const uint64_t *__restrict__ vin,
                                                     int n, Key3 *__restrict__ kout, uint64_t *__restrict__ vout) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char bs_smem[];
  Key3 *sk = reinterpret_cast<Key3 *>(bs_smem);
  uint64_t *sv = reinterpret_cast<uint64_t *>(sk + BSORT_MAX);
  int m = 1;
  while (m < n) m <<= 1;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    if (i < n) {
      sk[i] = kin[i];
      sv[i] = vin[i];
    } else {
      sk[i] = {~0ull, ~0ull, ~0ull};
      sv[i] = 0;
    }
  }
  __syncthreads();
  for (int size = 2; size <= m; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const bool sw = up ? key_less(sk[j], sk[i]) : key_less(sk[i], sk[j]);
          if (sw) {
            const Key3 tk = sk[i];
            sk[i] = sk[j];
            sk[j] = tk;
            const uint64_t tv = sv[i];
            sv[i] = sv[j];
            sv[j] = tv;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    kout[i] = sk[i];
    vout[i] = sv[i];
  }
}
constexpr size_t BSORT_SMEM = (sizeof(Key3) + sizeof(uint64_t)) * BSORT_MAX;

// host driver: buffers for one selection
struct SelBufs {
  Key3 *k0, *k1, *ks;  // candidates (round 0 input), ping-pong, selected
  uint64_t *v0, *v1, *vs;
  int64_t *w0, *w1;
  SelState *st;
  Key3 *bmin, *bmax;  // >= 1184 each
};

// Select the smallest-key prefix of (k0, v0, w0)[0..n) with weight >= W into
// (ks, vs); *nsel receives its size (synchronizes the stream once at the end,
// and at most three times before to stop launching finished rounds).
inline cudaError_t sel_run(const SelBufs &b, int64_t n, int64_t W, cudaStream_t stream, int64_t *nsel,
                           int64_t *launches, int64_t small = SEL_SMALL) {
  SelState h{};
  h.small = small;
  h.need = W > 0 ? W : 1;
  h.nU = n;
  h.done = n == 0;
  cudaError_t e = cudaMemcpyAsync(b.st, &h, sizeof(SelState), cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) return e;
  const int64_t nbl = (n + SEL_TPB - 1) / SEL_TPB;
  const unsigned nb = (unsigned)(nbl < 1 ? 1 : (nbl > 1184 ? 1184 : nbl));
  for (int r = 0; r <= SEL_ROUNDS; r++) {
    Key3 *kU = (r & 1) ? b.k1 : b.k0, *kN = (r & 1) ? b.k0 : b.k1;
    uint64_t *vU = (r & 1) ? b.v1 : b.v0, *vN = (r & 1) ? b.v0 : b.v1;
    int64_t *wU = (r & 1) ? b.w1 : b.w0, *wN = (r & 1) ? b.w0 : b.w1;
    k_sel_minmax<<<nb, SEL_TPB, 0, stream>>>(kU, b.st, b.bmin, b.bmax);
    k_sel_digit<<<1, SEL_TPB, 0, stream>>>(b.st, b.bmin, b.bmax, (int)nb);
    k_sel_hist<<<nb, SEL_TPB, 0, stream>>>(kU, wU, b.st);
    k_sel_pick<<<1, 32, 0, stream>>>(b.st);
    k_sel_split<<<nb, SEL_TPB, 0, stream>>>(kU, vU, wU, kN, vN, wN, b.ks, b.vs, b.st);
    k_sel_next<<<1, 32, 0, stream>>>(b.st);
    if (launches) *launches += 6;
    if (r == 1 || r == 3 || r == 6) {  // stop launching once the device says it is done
      int32_t done = 0;
      e = cudaMemcpyAsync(&done, &b.st->done, sizeof(int32_t), cudaMemcpyDeviceToHost, stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
      if (e != cudaSuccess) return e;
      if (done) break;
    }
  }
  const int rr = SEL_ROUNDS + 1;
  k_sel_flush<<<nb, SEL_TPB, 0, stream>>>((rr & 1) ? b.k1 : b.k0, (rr & 1) ? b.v1 : b.v0, b.ks, b.vs, b.st);
  k_sel_flush_done<<<1, 32, 0, stream>>>(b.st);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(nsel, &b.st->nSel, sizeof(int64_t), cudaMemcpyDeviceToHost, stream);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(stream);
}

}  // namespace prism

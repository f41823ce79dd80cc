// coop.cuh -- the eviction-order build and the protection pass as single
// persistent cooperative kernels (one CTA per SM, grid-wide syncs between
// phases), so a wave spends no kernel launches or host round trips on them.
//
//   k_build_coop : evict_key of every node -> subtree-maximum propagation ->
//                  composite keys of the candidates -> mass-weighted radix
//                  selection of the prefix that can be consumed -> sort of that
//                  prefix (per-CTA bitonic chunks + rank-merge rounds) -> list
//                  ready in the control block.
//   k_protect_coop: reusable-anchor keys (-P-hat, seg, id) -> top-f selection ->
//                  sort -> protected flags (kvcache.py:364-383).
//
// The selection is the algorithm of select.cuh (see there); here every CTA
// recomputes the round's control values (digit position, crossing bucket)
// redundantly from global state after each grid sync, so a round costs three
// grid syncs and no single-CTA phases.
#pragma once
#include <cooperative_groups.h>

#include "dart_kernels.cuh"

namespace prism {
namespace cg = cooperative_groups;

constexpr int COOP_TPB = 512;
constexpr int COOP_ROUNDS = 14;
constexpr int CHUNK = 4096;  // bitonic chunk per CTA (shared memory)
// sample select (coop_sample_select)
#ifndef PRISM_SS_SAMP
#define PRISM_SS_SAMP 12288
#endif
constexpr int SS_SAMP = PRISM_SS_SAMP;  // samples at most (the period is the power of two that keeps the sample below this)
constexpr int SS_SPL = 2560;   // splitters (selected samples) at most
constexpr size_t COOP_SORT_SMEM = (sizeof(Key3) + sizeof(uint64_t)) * CHUNK;
constexpr size_t COOP_SMEM = COOP_SORT_SMEM;

struct CoopState {
  unsigned long long cand;  // gathered candidates
  unsigned long long nsel;  // selected so far
  unsigned long long nun[COOP_ROUNDS + 2];
  unsigned long long hist_n[COOP_ROUNDS + 2][256];
  unsigned long long hist_w[COOP_ROUNDS + 2][256];
  long long prot_n;  // protection: number protected
  // sample-select (coop_sample_select)
  unsigned long long ss_ns;     // samples
  unsigned long long ss_n;      // items <= tau
  unsigned long long ss_mass;   // their weight
  unsigned long long ss_cand;   // all candidates
  unsigned int ss_cnt[SS_SPL];  // per-bucket counts
  unsigned int ss_cur[SS_SPL];  // per-bucket scatter cursors
  unsigned int ss_off[SS_SPL + 4];  // bucket offsets
  int ss_ok;                    // the sample select produced the sorted prefix
  unsigned long long tf_n;      // top-f protection: candidates with a positive P-hat
  int tf_done;                  // top-f protection applied by k_tf_local (k_protect_coop returns)
  unsigned int tf_cl;           // k_tf_local: clusters that published their top f
  unsigned int ss_next;         // k_ss_sort: next small bucket to take
  unsigned long long ss_dbg[24];
  unsigned long long ss_prof[8];  // diagnostics: k_ss_sort clock64 sums (load, sort, buckets, items)  // diagnostics: [0] max bucket, [1] rounds, [2+3r..] (undecided, selected, shift)
  int ss_nb;                    // diagnostics: splitters of the last sample select
  int ss_fail;                  // diagnostics: why it fell back (0: it did not)
  int nts;
  // ---- not cleared per launch (the host clears up to offsetof(ts))
  unsigned long long ts[40];  // phase timeline (%globaltimer ns), CTA 0 thread 0
  unsigned long long ts_build[40];
  int nts_build;
};

__device__ inline void coop_mark(CoopState *st) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && st->nts < 40) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    st->ts[st->nts++] = t;
  }
}

struct CoopBufs {
  Key3 *k0, *k1, *ks, *kt;  // candidates, ping-pong, selected, sort scratch
  uint64_t *v0, *v1, *vs, *vt;
  int64_t *w0, *w1;
  Key3 *bmin, *bmax;  // [gridDim.x]
  CoopState *st;
  int64_t *out_ids;  // protection: ids of the protected nodes (may be null)
};

__device__ inline Key3 shfl_key(const Key3 &k, int o) {
  return {__shfl_xor_sync(0xffffffffu, k.w0, o), __shfl_xor_sync(0xffffffffu, k.w1, o),
          __shfl_xor_sync(0xffffffffu, k.w2, o)};
}

// block min/max of Key3 (warp shuffles, then the warp results): written to
// *gmin / *gmax by thread 0; smin/smax hold >= 32 entries of scratch
__device__ inline void block_minmax(Key3 lo, Key3 hi, Key3 *smin, Key3 *smax, Key3 *gmin, Key3 *gmax) {
  for (int o = 16; o > 0; o >>= 1) {
    const Key3 a = shfl_key(lo, o), b = shfl_key(hi, o);
    if (key_less(a, lo)) lo = a;
    if (key_less(hi, b)) hi = b;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    smin[wid] = lo;
    smax[wid] = hi;
  }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    lo = lane < nw ? smin[lane] : Key3{~0ull, ~0ull, ~0ull};
    hi = lane < nw ? smax[lane] : Key3{0, 0, 0};
    for (int o = 16; o > 0; o >>= 1) {
      const Key3 a = shfl_key(lo, o), b = shfl_key(hi, o);
      if (key_less(a, lo)) lo = a;
      if (key_less(hi, b)) hi = b;
    }
    if (lane == 0) {
      *gmin = lo;
      *gmax = hi;
    }
  }
  __syncthreads();
}

__device__ inline uint32_t cdigit(const Key3 &k, int shift) {
  const int word = shift >> 6, off = shift & 63;
  const uint64_t lo = word == 0 ? k.w2 : (word == 1 ? k.w1 : k.w0);
  const uint64_t hi = word == 0 ? k.w1 : (word == 1 ? k.w0 : 0ull);
  uint64_t v = lo >> off;
  if (off > 56) v |= hi << (64 - off);
  return (uint32_t)(v & 0xFFu);
}

__device__ inline int chighbit(const Key3 &x) {
  if (x.w0) return 128 + 63 - __clzll((long long)x.w0);
  if (x.w1) return 64 + 63 - __clzll((long long)x.w1);
  if (x.w2) return 63 - __clzll((long long)x.w2);
  return -1;
}

// Selection of the smallest-key prefix of weight >= W among n candidates
// (B.k0/v0/w0), into B.ks/vs; returns the selected count (uniform in the grid).
// Per round: every CTA derives the digit from the per-CTA min/max of U, one
// weighted-histogram pass, a grid sync, the crossing bucket (warp 0 of every
// CTA), one split pass that also records the min/max of the next U, a grid
// sync.  Streaming loops are unrolled 4x (4 independent loads in flight).
constexpr int UNR = 4;

__device__ inline void grid_minmax(const CoopBufs &B, int mb, Key3 *smin, Key3 *smax, Key3 &gmin, Key3 &gmax) {
  Key3 lo = {~0ull, ~0ull, ~0ull}, hi = {0, 0, 0};
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
    if (key_less(B.bmin[mb + i], lo)) lo = B.bmin[mb + i];
    if (key_less(hi, B.bmax[mb + i])) hi = B.bmax[mb + i];
  }
  block_minmax(lo, hi, smin, smax, &smin[blockDim.x], &smax[blockDim.x]);
  gmin = smin[blockDim.x];
  gmax = smax[blockDim.x];
  __syncthreads();
}

__device__ int64_t coop_select(cg::grid_group &grid, const CoopBufs &B, int64_t n, int64_t W, int64_t small,
                               Key3 *smin, Key3 *smax) {
  __shared__ int s_dstar, s_all;
  __shared__ long long s_below;
  int64_t nU = n, need = W > 0 ? W : 1;
  bool done = n == 0;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gsz = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  {  // min/max of the initial candidate set
    Key3 lo = {~0ull, ~0ull, ~0ull}, hi = {0, 0, 0};
    for (int64_t i0 = gtid; i0 < n; i0 += UNR * gsz) {
      Key3 x[UNR];
#pragma unroll
      for (int u = 0; u < UNR; u++) {
        const int64_t i = i0 + u * gsz;
        if (i < n) x[u] = B.k0[i];
      }
#pragma unroll
      for (int u = 0; u < UNR; u++) {
        if (i0 + u * gsz < n) {
          if (key_less(x[u], lo)) lo = x[u];
          if (key_less(hi, x[u])) hi = x[u];
        }
      }
    }
    block_minmax(lo, hi, smin, smax, &B.bmin[blockIdx.x], &B.bmax[blockIdx.x]);
  }
  grid.sync();
  coop_mark(B.st);
  for (int r = 0; r < COOP_ROUNDS && !done; r++) {
    const Key3 *kU = (r & 1) ? B.k1 : B.k0;
    const uint64_t *vU = (r & 1) ? B.v1 : B.v0;
    const int64_t *wU = (r & 1) ? B.w1 : B.w0;
    Key3 *kN = (r & 1) ? B.k0 : B.k1;
    uint64_t *vN = (r & 1) ? B.v0 : B.v1;
    int64_t *wN = (r & 1) ? B.w0 : B.w1;
    const int mb = (r & 1) * 1024;  // min/max of U: bmin/bmax[mb + cta]
    Key3 gmin, gmax;
    grid_minmax(B, mb, smin, smax, gmin, gmax);
    const Key3 xx = {gmin.w0 ^ gmax.w0, gmin.w1 ^ gmax.w1, gmin.w2 ^ gmax.w2};
    const int hb = chighbit(xx);
    const int shift = hb < 7 ? 0 : hb - 7;
    const bool single = hb < 0;
    if (!single) {  // weighted histogram of the digit, warp-aggregated
      for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x; b0 < nU; b0 += UNR * gsz) {
        uint32_t d[UNR], wt[UNR];
#pragma unroll
        for (int u = 0; u < UNR; u++) {
          const int64_t i = b0 + u * gsz + threadIdx.x;
          d[u] = i < nU ? cdigit(kU[i], shift) : 256u;
          wt[u] = i < nU ? (uint32_t)wU[i] : 0u;
        }
#pragma unroll
        for (int u = 0; u < UNR; u++) {
          const unsigned peers = __match_any_sync(0xffffffffu, d[u]);
          const unsigned wsum = __reduce_add_sync(peers, wt[u]);
          if (d[u] < 256u && lane == __ffs(peers) - 1) {
            atomicAdd(&B.st->hist_n[r][d[u]], (unsigned long long)__popc(peers));
            atomicAdd(&B.st->hist_w[r][d[u]], (unsigned long long)wsum);
          }
        }
      }
    }
    grid.sync();
    if (threadIdx.x < 32) {  // crossing bucket
      int dstar = 256, all = 1;
      long long below = 0;
      if (!single) {
        long long w8[8], run = 0;
        for (int q = 0; q < 8; q++) {
          run += (long long)B.st->hist_w[r][8 * lane + q];
          w8[q] = run;
        }
        long long pre = run;
        for (int o = 1; o < 32; o <<= 1) {
          const long long y = __shfl_up_sync(0xffffffffu, pre, o);
          if (lane >= o) pre += y;
        }
        const long long before = pre - run;
        int dl = 256;
        for (int q = 0; q < 8; q++)
          if (before + w8[q] >= need) {
            dl = 8 * lane + q;
            break;
          }
        const unsigned m = __ballot_sync(0xffffffffu, dl < 256);
        if (m) {
          const int src = __ffs(m) - 1;
          dstar = __shfl_sync(0xffffffffu, dl, src);
          const int q = dstar - 8 * src;
          long long bb = 0;
          if (lane == src) bb = before + (q ? w8[q - 1] : 0);
          below = __shfl_sync(0xffffffffu, bb, src);
          all = (int64_t)B.st->hist_n[r][dstar] <= small ? 1 : 0;
        }
      }
      if (threadIdx.x == 0) {
        s_dstar = dstar;
        s_all = all;
        s_below = below;
      }
    }
    __syncthreads();
    const int dstar = s_dstar, all = s_all;
    Key3 lo = {~0ull, ~0ull, ~0ull}, hi = {0, 0, 0};  // min/max of the next U
    for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x; b0 < nU; b0 += UNR * gsz) {
      Key3 xk[UNR];
      int cls[UNR];
#pragma unroll
      for (int u = 0; u < UNR; u++) {
        const int64_t i = b0 + u * gsz + threadIdx.x;
        cls[u] = 2;  // 0 = select, 1 = next U, 2 = drop
        if (i < nU) {
          xk[u] = kU[i];
          const int d = dstar >= 256 ? 0 : (int)cdigit(xk[u], shift);
          if (dstar >= 256 || d < dstar || (d == dstar && all)) cls[u] = 0;
          else if (d == dstar) cls[u] = 1;
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; u++) {
        const int64_t i = b0 + u * gsz + threadIdx.x;
        const unsigned ms = __ballot_sync(0xffffffffu, cls[u] == 0), mn = __ballot_sync(0xffffffffu, cls[u] == 1);
        unsigned long long bs = 0, bn = 0;
        if (lane == 0) {
          if (ms) bs = atomicAdd(&B.st->nsel, (unsigned long long)__popc(ms));
          if (mn) bn = atomicAdd(&B.st->nun[r], (unsigned long long)__popc(mn));
        }
        bs = __shfl_sync(0xffffffffu, bs, 0);
        bn = __shfl_sync(0xffffffffu, bn, 0);
        const unsigned below_lanes = (1u << lane) - 1u;
        if (cls[u] == 0) {
          const int64_t p = (int64_t)bs + __popc(ms & below_lanes);
          B.ks[p] = xk[u];
          B.vs[p] = vU[i];
        } else if (cls[u] == 1) {
          const int64_t p = (int64_t)bn + __popc(mn & below_lanes);
          kN[p] = xk[u];
          vN[p] = vU[i];
          wN[p] = wU[i];
          if (key_less(xk[u], lo)) lo = xk[u];
          if (key_less(hi, xk[u])) hi = xk[u];
        }
      }
    }
    block_minmax(lo, hi, smin, smax, &B.bmin[(mb ^ 1024) + blockIdx.x], &B.bmax[(mb ^ 1024) + blockIdx.x]);
    grid.sync();
    coop_mark(B.st);
    const int64_t nun = (int64_t)B.st->nun[r];
    need -= s_below;
    done = (all != 0) || nun == 0;
    nU = nun;
    __syncthreads();
  }
  if (!done && nU > 0) {  // round budget exhausted: take the remaining U whole
    const int r = COOP_ROUNDS;
    const Key3 *kU = (r & 1) ? B.k1 : B.k0;
    const uint64_t *vU = (r & 1) ? B.v1 : B.v0;
    const int64_t base = (int64_t)B.st->nsel;
    for (int64_t i = gtid; i < nU; i += gsz) {
      B.ks[base + i] = kU[i];
      B.vs[base + i] = vU[i];
    }
    grid.sync();
    if (gtid == 0) B.st->nsel += nU;
  }
  grid.sync();
  return (int64_t)B.st->nsel;
}

// Sort (B.ks, B.vs)[0..n) ascending: every CTA bitonic-sorts chunks in shared
// memory (chunk = n / #CTAs rounded up to a power of two, 256..CHUNK, so all
// SMs share the work), then merge rounds in which every element finds its
// rank in the partner run by binary search (keys are unique).
__device__ void coop_sort(cg::grid_group &grid, const CoopBufs &B, int64_t n, Key3 *kout, uint64_t *vout,
                          unsigned char *dsm) {
  Key3 *sk = reinterpret_cast<Key3 *>(dsm);
  uint64_t *sv = reinterpret_cast<uint64_t *>(sk + CHUNK);
  int64_t chunk = 256;
  while (chunk < CHUNK && chunk * (int64_t)gridDim.x < n) chunk <<= 1;
  const int64_t nchunks = (n + chunk - 1) / chunk;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int64_t b0 = c * chunk;
    const int m0 = (int)((n - b0) < chunk ? (n - b0) : chunk);
    int m = 1;
    while (m < m0) m <<= 1;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      if (i < m0) {
        sk[i] = B.ks[b0 + i];
        sv[i] = B.vs[b0 + i];
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
    for (int i = threadIdx.x; i < m0; i += blockDim.x) {
      B.kt[b0 + i] = sk[i];
      B.vt[b0 + i] = sv[i];
    }
    __syncthreads();
  }
  grid.sync();
  coop_mark(B.st);
  Key3 *ka = B.kt, *kb = B.ks;
  uint64_t *va = B.vt, *vb = B.vs;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gsz = (int64_t)gridDim.x * blockDim.x;
  for (int64_t run = chunk; run < n; run <<= 1) {
    for (int64_t i = gtid; i < n; i += gsz) {
      const int64_t pair = i / (2 * run), base = pair * 2 * run;
      const int64_t aS = base, aE = (base + run) < n ? base + run : n;
      const int64_t bS = aE, bE = (base + 2 * run) < n ? base + 2 * run : n;
      const Key3 x = ka[i];
      int64_t lo, hi, pos;
      if (i < aE) {  // rank among the other run's smaller keys
        lo = bS;
        hi = bE;
      } else {
        lo = aS;
        hi = aE;
      }
      const int64_t s0 = lo;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (key_less(ka[mid], x)) lo = mid + 1;
        else hi = mid;
      }
      pos = base + (i < aE ? (i - aS) : (i - bS)) + (lo - s0);
      kb[pos] = x;
      vb[pos] = va[i];
    }
    grid.sync();
    coop_mark(B.st);
    Key3 *tk = ka;
    ka = kb;
    kb = tk;
    uint64_t *tv = va;
    va = vb;
    vb = tv;
  }
  for (int64_t i = gtid; i < n; i += gsz) {
    kout[i] = ka[i];
    vout[i] = va[i];
  }
  grid.sync();
}

// ------------------------------------------------------------ sample select
// The smallest-key prefix of weight >= W of the candidates defined over the
// slots [0, hw) by cand(s, key, val, w), sorted, into (kout, vout) -- without
// materialising the candidates:
//   1. one slot at a hashed offset in every m-slot window is sampled (m: the
//      power of two that keeps the sample <= SS_SAMP);
//   2. CTA 0 selects the sample prefix whose mass, scaled by m, reaches 1.25 W
//      plus three samples of slack (radix rounds over the undecided samples,
//      then an exact sort of the last few) and sorts it: the splitters; tau =
//      the largest;
//   3. one pass over all slots keeps the candidates with key <= tau -- exactly
//      a prefix of the order, whatever the sample looked like -- each with its
//      bucket (#splitters below it: buckets of ~m candidates);
//   4. bucket offsets by a scan, a scatter into bucket order, and one shared-
//      memory bitonic sort per bucket.
// Returns false (nothing written to kout/vout) when the sample cannot promise
// the prefix, the pass shows it fell short (mass < W and not every candidate
// kept) or a bucket overflows shared memory; the caller then runs the
// materialising selection.  Uniform over the grid.
__device__ inline void bitonic_smem(Key3 *sk, uint64_t *sv, int m) {
  for (int size = 2; size <= m; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const int lg = __ffs(stride) - 1;
      for (int p = threadIdx.x; p < (m >> 1); p += blockDim.x) {
        const int i = ((p >> lg) << (lg + 1)) | (p & (stride - 1)), j = i + stride;
        const bool up = (i & size) == 0;
        if (up ? key_less(sk[j], sk[i]) : key_less(sk[i], sk[j])) {
          const Key3 tk = sk[i];
          sk[i] = sk[j];
          sk[j] = tk;
          const uint64_t tv = sv[i];
          sv[i] = sv[j];
          sv[j] = tv;
        }
      }
      __syncthreads();
    }
  }
}


// exclusive scan of a[0..n) in shared memory, returns the total
__device__ inline unsigned long long block_exscan_u64(unsigned long long *a, int n, unsigned long long *warp_tot) {
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int b = threadIdx.x * per, e = min(b + per, n);
  unsigned long long s = 0;
  for (int i = b; i < e; i++) s += a[i];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long x = s;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    unsigned long long t = lane < nw ? warp_tot[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) warp_tot[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  unsigned long long run = x - s + (wid ? warp_tot[wid - 1] : 0);
  const unsigned long long total = warp_tot[(blockDim.x >> 5) - 1];
  __syncthreads();
  for (int i = b; i < e; i++) {
    const unsigned long long v = a[i];
    a[i] = run;
    run += v;
  }
  __syncthreads();
  return total;
}

// block-wide reservation of c items per thread at *ctr (one global atomic per
// CTA); returns this thread's first position.  Every thread calls it.
__device__ inline unsigned long long block_reserve(unsigned c, unsigned long long *ctr, unsigned *s_w,
                                                   unsigned long long *s_base) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned x = c;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[wid] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned run = 0;
    for (int q = 0; q < nw; q++) {
      const unsigned t = s_w[q];
      s_w[q] = run;
      run += t;
    }
    *s_base = run ? atomicAdd(ctr, (unsigned long long)run) : 0ull;
  }
  __syncthreads();
  const unsigned long long pos = *s_base + s_w[wid] + (x - c);
  __syncthreads();
  return pos;
}

// ascending sort of n unique keys (+ values) in shared memory: chunks of
// MS_CH rank-sorted into (tk, tv) (broadcast reads, no barriers), then every
// item's final position = its rank in its chunk + its lower bound in every
// other chunk; written to (ko, vo), which may alias (k, v).  O(n * MS_CH)
// compares instead of the O(n^2) of a plain rank sort, two barriers instead of
// the O(log^2 n) of a bitonic network.
constexpr int MS_CH = 64;

__device__ __forceinline__ Key3 shfl_xor_key(const Key3 &x, int m) {
  return {__shfl_xor_sync(0xffffffffu, x.w0, m), __shfl_xor_sync(0xffffffffu, x.w1, m),
          __shfl_xor_sync(0xffffffffu, x.w2, m)};
}

// Shared-memory sort of (k, v)[0..n) into (ko, vo) (ko may be global memory or
// alias k; k / v and the scratch tk / tv are clobbered; v null: keys only):
// every warp sorts 32-key runs in registers (bitonic over shuffles), then
// log2(n / 32) rounds merge run pairs -- an item's place is its index in its
// run plus its rank in the partner run (binary search; equal keys of the left
// run first), so every round is one barrier and no item waits on another.
__device__ inline void block_sort(Key3 *k, uint64_t *v, int n, Key3 *tk, uint64_t *tv, Key3 *ko, uint64_t *vo) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r0 = 0; r0 < n; r0 += 32 * nw) {
    const int i = r0 + wid * 32 + lane;
    const bool in = i < n;
    Key3 x = in ? k[i] : Key3{~0ull, ~0ull, ~0ull};
    uint64_t vx = (in && v) ? v[i] : 0ull;
    for (int size = 2; size <= 32; size <<= 1) {
      for (int j = size >> 1; j > 0; j >>= 1) {
        const Key3 y = shfl_xor_key(x, j);
        const uint64_t vy = __shfl_xor_sync(0xffffffffu, vx, j);
        const bool take_min = ((lane & j) == 0) == ((lane & size) == 0);
        if (take_min ? key_less(y, x) : key_less(x, y)) {
          x = y;
          vx = vy;
        }
      }
    }
    if (in) {
      k[i] = x;
      if (v) v[i] = vx;
    }
  }
  __syncthreads();
  Key3 *src = k, *dst = tk;
  uint64_t *vsrc = v, *vdst = tv;
  for (int w = 32; w < n; w <<= 1) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int r = i / w, os = r * w;
      const Key3 x = src[i];
      int pos = i;
      if ((r & 1) == 0) {  // left run: keys of the right run strictly below x
        int lo = os + w, hi = min(os + 2 * w, n);
        const int base = lo;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (key_less(src[mid], x)) lo = mid + 1;
          else hi = mid;
        }
        pos = i + (lo - base);
      } else {  // right run: keys of the left run at most x
        int lo = os - w, hi = os;
        const int base = lo;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (!key_less(x, src[mid])) lo = mid + 1;
          else hi = mid;
        }
        pos = base + (i - os) + (lo - base);
      }
      dst[pos] = x;
      if (v) vdst[pos] = vsrc[i];
    }
    __syncthreads();
    Key3 *t = src;
    src = dst;
    dst = t;
    uint64_t *tt = vsrc;
    vsrc = vdst;
    vdst = tt;
  }
  if (src != ko) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      ko[i] = src[i];
      if (vo) vo[i] = v ? vsrc[i] : 0ull;
    }
  } else if (vo && !v) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) vo[i] = 0ull;
  }
  __syncthreads();
}

__device__ inline void block_merge_sort(const Key3 *k, const uint64_t *v, int n, Key3 *tk, uint64_t *tv, Key3 *ko,
                                        uint64_t *vo) {
  if (n > MS_CH) {  // (every caller's input is shared-memory scratch it may lose)
    block_sort(const_cast<Key3 *>(k), const_cast<uint64_t *>(v), n, tk, tv, ko, vo);
    return;
  }
  const int nch = (n + MS_CH - 1) / MS_CH;
  int tpi = 1;  // threads per item (a power of two <= 8): small sets use the whole block
  while (tpi < 8 && 2 * tpi * n <= (int)blockDim.x) tpi <<= 1;
  const int sub = threadIdx.x & (tpi - 1), per = (int)blockDim.x / tpi;
  for (int i0 = 0; i0 < n; i0 += per) {  // uniform trip count (shuffles below)
    const int i = i0 + (int)threadIdx.x / tpi;
    const bool ok = i < n;
    const int c0 = ok ? (i / MS_CH) * MS_CH : 0, c1 = ok ? min(c0 + MS_CH, n) : 0;
    const Key3 x = ok ? k[i] : Key3{0, 0, 0};
    int r = 0;  // (ties by position: equal keys, e.g. padding, keep a permutation -- a stable sort)
#pragma unroll 4
    for (int j = c0 + sub; j < c1; j += tpi) r += (key_less(k[j], x) || (j < i && !key_less(x, k[j]))) ? 1 : 0;
    for (int o = 1; o < tpi; o <<= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if (ok && sub == 0) {
      tk[c0 + r] = x;
      if (tv) tv[c0 + r] = v ? v[i] : 0ull;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int c = i / MS_CH;
    const Key3 x = tk[i];
    int pos = i - c * MS_CH;
    for (int d = 0; d < nch; d++) {
      if (d == c) continue;
      int lo = d * MS_CH, hi = min(lo + MS_CH, n);
      const int base = lo;
      const bool before = d < c;  // equal keys of earlier chunks precede
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (before ? !key_less(x, tk[mid]) : key_less(tk[mid], x)) lo = mid + 1;
        else hi = mid;
      }
      pos += lo - base;
    }
    ko[pos] = x;  // (ko may alias k: phase 1 read all of k before the barrier)
    if (vo) vo[pos] = tv ? tv[i] : 0ull;
  }
  __syncthreads();
}


// candidate gather over the slots (the materialising path): cand(s) for every
// slot s < hw into (B.k0, B.v0, B.w0); the count lands in st->cand
template <class Cand>
__device__ void coop_gather(const CoopBufs &B, int32_t hw, Cand cand) {
  const int lane = threadIdx.x & 31;
  const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s0 = (int64_t)blockIdx.x * blockDim.x; s0 < hw; s0 += gsz) {
    const int64_t s = s0 + threadIdx.x;
    Key3 k;
    uint64_t v;
    int64_t w = 0;
    const bool take = s < hw && cand((int32_t)s, k, v, w);
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (!m) continue;
    unsigned long long b = 0;
    if (lane == 0) b = atomicAdd(&B.st->cand, (unsigned long long)__popc(m));
    b = __shfl_sync(0xffffffffu, b, 0);
    if (take) {
      const int64_t p = (int64_t)b + __popc(m & ((1u << lane) - 1u));
      B.k0[p] = k;
      B.v0[p] = v;
      B.w0[p] = w;
    }
  }
}

// eviction-order candidate of slot s (after k_build_keys / k_propagate): every
// live node whose subtree holds no blocked node, keyed (subtree max, deeper first)
struct EvictCand {
  DT T;
  __device__ int32_t hw() const { return T.ctrl->hw; }
  __device__ bool operator()(int32_t s, Key3 &k, uint64_t &v, int64_t &w) const {
    const int32_t e = __ldg(&T.eff[s]);
    if (e < 0) return false;
    k = composite(T.kw[e], __ldg(&T.dend[s]));
    v = ((uint64_t)__ldg(&T.kver[s]) << 32) | (uint32_t)s;
    w = __ldg(&T.elen[s]);
    return true;
  }
};

// set_protection candidate (kvcache.py:370-381): live nodes holding a REUSABLE
// anchor, keyed (-P-hat[seg], seg or -1, node_id); visiting a slot clears its
// previous protection flag
struct ProtCand {
  DT T;
  int32_t keys;  // also leave the eviction keys of the unprotected tree (kw / eff, as k_build_keys)
  __device__ int32_t hw() const { return T.ctrl->hw; }
  __device__ bool operator()(int32_t s, Key3 &k, uint64_t &v, int64_t &w) const {
    T.prot[s] = 0;
    const bool live = s != ROOT && T.nid[s] >= 0 && T.par[s] >= 0;
    if (keys) {
      if (!live) {
        T.eff[s] = EFF_DEAD;
      } else {
        const bool blocked = T.ref[s] > 0 || (T.policy == P_DART && T.kind[s] == K_SYSTEM);
        T.kw[s] = make_key(T, s);  // (prot cleared above; the top-f get theirs in k_protect_coop)
        T.eff[s] = blocked ? EFF_BLOCKED : s;
      }
    }
    if (!live || !T.hasanc[s] || T.akind[s] != K_REUSABLE) return false;
    const int32_t sg = T.seg[s];
    const int32_t sv = sg == SEG_NONE ? -1 : sg;
    k = {0, 0, 0};
    shl_or(k, 64, ord_f64(-pri_of(T, sg)));
    shl_or(k, 32, (uint64_t)((uint32_t)sv ^ 0x80000000u));
    shl_or(k, 40, (uint64_t)T.nid[s] & ((1ull << 40) - 1));
    v = (uint64_t)(uint32_t)s;
    w = 1;
    return true;
  }
};

// ------------------------------------------------------------ sample select
// The smallest-key prefix of weight >= W of the candidates cand(s) over the
// slots [0, hw), sorted into (kout, vout), without materialising the
// candidates -- five full-occupancy launches in stream order (no host round
// trip), then the cooperative kernel finalises (or, when st->ss_ok is 0, runs
// the materialising radix selection):
//   k_ss_sample  one slot at a hashed offset in every m-slot window (m: the
//                power of two that keeps the sample <= SS_SAMP);
//   k_ss_select  one CTA: the sample prefix whose mass, scaled by m, reaches
//                1.25 W + three samples of slack (radix rounds over the
//                undecided samples, an exact sort of the last few), sorted:
//                the splitters, tau = the largest;
//   k_ss_filter  every slot: keep key <= tau -- exactly a prefix of the order,
//                whatever the sample looked like -- with its bucket
//                (#splitters below it; buckets of ~m candidates);
//   k_ss_scatter bucket offsets; enough mass (or every candidate) and every
//                bucket <= SS_BMAX? (st->ss_ok); scatter into bucket order;
//   k_ss_sort    one CTA per bucket sorts it in shared memory.
constexpr int SS_TPB = 256;
constexpr int SS_SEL_TPB = 512;
#ifndef PRISM_SS_BMAX
#define PRISM_SS_BMAX 2048  // (= SS_SORT_CAP: a bucket up to a whole run; 1024 -> 2048: 0.7% per C3 wave)
#endif
constexpr int SS_BMAX = PRISM_SS_BMAX;  // buckets up to this size: k_ss_sort (runs of whole buckets per CTA)
constexpr int SS_BMID = 384;   // k_ss_sort takes the buckets above this first
constexpr int SS_BBIG = CHUNK; // larger ones up to this: k_ss_sort_big (in-place bitonic); beyond: fallback
constexpr int SS_SUB = 1024;  // sub-sample the selection rounds run on
constexpr size_t SS_SEL_SMEM = 3 * sizeof(Key3) * SS_SPL + 3 * 8 * SS_SUB;  // (k_ss_select's lk, tk, all; lw, tw, aw)
constexpr size_t SS_FILTER_SMEM = sizeof(Key3) * SS_SPL + 4 * SS_SPL;
// k_ss_sort: one 1024-thread CTA per SM sorting runs of whole buckets of up to
// SS_SORT_CAP items (+ scratch, + the bucket offsets) in shared memory
#ifndef PRISM_SS_SORT_TPB
#define PRISM_SS_SORT_TPB 1024
#define PRISM_SS_SORT_CAP 2048
#endif
constexpr int SS_SORT_TPB = PRISM_SS_SORT_TPB;
constexpr int SS_SORT_CAP = PRISM_SS_SORT_CAP;
constexpr int SS_SORT_PER_SM = 1024 / SS_SORT_TPB;  // CTAs per SM
static_assert(SS_BMAX <= SS_SORT_CAP, "k_ss_sort takes every bucket up to SS_BMAX as (part of) one run");
constexpr size_t SS_SORT_SMEM = 2 * (sizeof(Key3) + 8) * SS_SORT_CAP + sizeof(unsigned) * (SS_SPL + 4);

__device__ inline int64_t ss_period(int32_t hw) {
  int64_t m = 8;
  while ((int64_t)hw > m * SS_SAMP) m <<= 1;
  return m;
}

template <class Cand>
__global__ void __launch_bounds__(SS_TPB) k_ss_sample(Cand cand, CoopBufs B, int64_t W, const int64_t *dW,
                                                      int64_t min_cand) {
  pdl_wait();
  __shared__ unsigned s_w[32];
  __shared__ unsigned long long s_base;
  if (dW) W = *dW;
  const int32_t hw = cand.hw();
  if (W <= 0 || hw <= min_cand) return;  // nothing sampled: k_ss_select gives up
  const int64_t m = ss_period(hw), nsamp = ((int64_t)hw + m - 1) / m;
  const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j0 = (int64_t)blockIdx.x * blockDim.x; j0 < nsamp; j0 += gsz) {
    const int64_t j = j0 + threadIdx.x;
    Key3 k;
    uint64_t v;
    int64_t w;
    // (a fixed offset in the window would alias with periodic slot layouts)
    const int64_t s = j * m + (int64_t)(mix64((uint64_t)j ^ 0x9E3779B97F4A7C15ull) & (uint64_t)(m - 1));
    const bool take = j < nsamp && s < hw && cand((int32_t)s, k, v, w);
    const unsigned long long p = block_reserve(take ? 1u : 0u, &B.st->ss_ns, s_w, &s_base);
    if (take) {
      B.k1[p] = k;
      B.w1[p] = w;
    }
  }
}

// rank of x among the sorted keys a[0..n): the keys below it (before = false)
// or at most it (before = true: equal keys of an earlier slice come first)
__device__ __forceinline__ int ss_rank(const Key3 *a, int n, const Key3 &x, bool before) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (before ? !key_less(x, a[mid]) : key_less(a[mid], x)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// The sample select as one 8-CTA cluster, every step spread over the cluster:
//  1. tau: the sub-sample (every q-th sample, <= SS_SUB) is sorted -- each CTA
//     sorts a slice, CTA 0 gathers the slices over DSMEM and places every key
//     by its rank in each slice -- and CTA 0 finds the key where the prefix
//     weight, scaled by m q, reaches 1.25 W + three average sub-samples;
//  2. the splitters (every sample <= tau, ~2000): each CTA filters and sorts
//     its share of the sample, then places its keys by their ranks in every
//     peer's sorted share (gathered over DSMEM) straight into B.kt.
// (One CTA ran this with radix rounds and a splitter sort: ~50 us of the wave.)
constexpr int SS_CL = 8;  // CTAs in k_ss_select's cluster
template <class Cand>
__global__ void __cluster_dims__(SS_CL, 1, 1) __launch_bounds__(SS_SEL_TPB)
    k_ss_select(Cand cand, CoopBufs B, int64_t W, const int64_t *dW) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ int s_fail, s_n;
  __shared__ unsigned long long s_u64[32];
  __shared__ int s_cross;
  __shared__ Key3 s_tau;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  CoopState *st = B.st;
  if (dW) W = *dW;
  if (rank == 0) coop_mark(st);
  // shared memory: lk/lw [SS_SPL] this CTA's keys (sub-sample slice, then its
  // splitters), tk/tw [SS_SPL] sort scratch, all [SS_SPL] every CTA's sorted keys
  Key3 *lk = reinterpret_cast<Key3 *>(dsm);
  Key3 *tk = lk + SS_SPL;
  Key3 *all = tk + SS_SPL;
  uint64_t *lw = reinterpret_cast<uint64_t *>(all + SS_SPL);
  uint64_t *tw = lw + SS_SUB;
  uint64_t *aw = tw + SS_SUB;  // [SS_SUB] CTA 0: the sorted sub-sample's weights
  const int ns = (int)st->ss_ns;
  const int64_t m = ss_period(cand.hw());
  const int q = (ns + SS_SUB - 1) / SS_SUB > 0 ? (ns + SS_SUB - 1) / SS_SUB : 1;
  const int nsub = (ns + q - 1) / q;
  // ---- 1. the sorted sub-sample
  const int sper = (nsub + SS_CL - 1) / SS_CL;
  const int s0 = min(nsub, rank * sper), sm = min(nsub, s0 + sper) - s0;
  for (int j = tid; j < sm; j += blockDim.x) {
    lk[j] = B.k1[(int64_t)(s0 + j) * q];
    lw[j] = (uint64_t)B.w1[(int64_t)(s0 + j) * q];
  }
  __syncthreads();
  block_merge_sort(lk, lw, sm, tk, tw, lk, lw);
  cluster.sync();
  if (rank == 0) {
    coop_mark(st);
    // every slice into shared memory (flat over the sub-sample: a thread's
    // remote loads are independent, one DSMEM round trip), then each key at
    // its merged place: its index in its slice + its rank in every other slice
    for (int j = tid; j < nsub; j += blockDim.x) {
      const int r = j / sper, i = j - r * sper;
      all[j] = cluster.map_shared_rank(lk, r)[i];
      tw[j] = cluster.map_shared_rank(lw, r)[i];
    }
    __syncthreads();
    for (int j = tid; j < nsub; j += blockDim.x) {
      const int r = j / sper, i = j - r * sper;
      const Key3 x = all[j];
      int pos = i;
      for (int r2 = 0; r2 < SS_CL; r2++) {
        if (r2 == r) continue;
        const int a0 = min(nsub, r2 * sper), an = min(nsub, a0 + sper) - a0;
        pos += ss_rank(all + a0, an, x, r2 < r);
      }
      tk[pos] = x;
      aw[pos] = tw[j];
    }
    __syncthreads();
    // the target sub-sample mass: (1.25 W + 3 average sub-samples of slack) / (m q)
    // (tau comes from <= SS_SUB sub-samples: ~7% noise; a prefix short of W
    // costs the materialising selection, so the margin stays wide)
    unsigned long long x = 0;
    for (int j = tid; j < nsub; j += blockDim.x) x += aw[j];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) s_u64[wid] = x;
    __syncthreads();
    unsigned long long tot = 0;
    for (int w = 0; w < nw; w++) tot += s_u64[w];
    __syncthreads();
    const double mq = (double)m * q;
    const long long need =
        nsub > 0 ? (long long)(((double)W * 1.25 + 3.0 * mq * ((double)tot / nsub)) / mq) + 1 : 1;
    // (W <= 0: the whole order asked for, see prebuild_order: everything is sorted)
    const int fail = (W <= 0 || nsub == 0 || (unsigned long long)need > tot) ? 1 : 0;
    if (tid == 0) {
      s_fail = fail;
      s_cross = nsub - 1;
    }
    __syncthreads();
    if (!fail) {  // the first place whose inclusive weight prefix reaches need (block scan, a carry per chunk)
      long long carry = 0;
      for (int j0 = 0; j0 < nsub; j0 += blockDim.x) {
        const int j = j0 + tid;
        long long inc = j < nsub ? (long long)aw[j] : 0;
        for (int o = 1; o < 32; o <<= 1) {
          const long long y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        if (lane == 31) s_u64[wid] = (unsigned long long)inc;
        __syncthreads();
        long long before = carry, chunk = 0;
        for (int w = 0; w < nw; w++) {
          if (w < wid) before += (long long)s_u64[w];
          chunk += (long long)s_u64[w];
        }
        if (j < nsub && before + inc >= need) atomicMin(&s_cross, j);
        carry += chunk;
        __syncthreads();
      }
      if (tid == 0) s_tau = tk[s_cross];
    }
    coop_mark(st);
  }
  cluster.sync();
  const int fail0 = *cluster.map_shared_rank(&s_fail, 0);
  int nb = 0, fail = fail0;
  if (!fail0) {
    // ---- 2. the splitters: this CTA's share of the sample at or below tau, sorted
    const Key3 tau = *cluster.map_shared_rank(&s_tau, 0);
    if (tid == 0) s_n = 0;
    __syncthreads();
    const int per = (ns + SS_CL - 1) / SS_CL, a0 = min(ns, rank * per), a1 = min(ns, a0 + per);
    constexpr int SPU = 4;  // sample loads in flight per thread
    for (int i0 = a0; i0 < a1; i0 += SPU * blockDim.x) {
      Key3 k[SPU];
#pragma unroll
      for (int u = 0; u < SPU; u++) {
        const int i = i0 + u * blockDim.x + tid;
        k[u] = i < a1 ? B.k1[i] : tau;
      }
#pragma unroll
      for (int u = 0; u < SPU; u++) {
        const bool t = i0 + u * (int)blockDim.x + tid < a1 && !key_less(tau, k[u]);
        const unsigned mt = __ballot_sync(0xffffffffu, t);
        int p = 0;
        if (lane == 0 && mt) p = atomicAdd(&s_n, __popc(mt));
        p = __shfl_sync(0xffffffffu, p, 0) + __popc(mt & ((1u << lane) - 1u));
        if (t && p < SS_SPL) lk[p] = k[u];
      }
    }
    __syncthreads();
    const int mine = s_n;
    if (mine <= SS_SPL) block_merge_sort(lk, nullptr, mine, tk, nullptr, lk, nullptr);
    cluster.sync();  // every share sorted and counted
    int off[SS_CL + 1];
    off[0] = 0;
    for (int r = 0; r < SS_CL; r++) off[r + 1] = off[r] + *cluster.map_shared_rank(&s_n, r);
    nb = off[SS_CL];
    if (nb > SS_SPL) {
      fail = 3;  // more splitters than a filter CTA holds
    } else {
      for (int j = tid; j < nb; j += blockDim.x) {  // (flat: independent remote loads)
        int r = 0;
        while (j >= off[r + 1]) r++;
        all[j] = cluster.map_shared_rank(lk, r)[j - off[r]];
      }
      __syncthreads();
      for (int i = tid; i < mine; i += blockDim.x) {
        const Key3 x = lk[i];
        int pos = i;
        for (int r = 0; r < SS_CL; r++)
          if (r != rank) pos += ss_rank(all + off[r], off[r + 1] - off[r], x, r < rank);
        B.kt[pos] = x;
      }
    }
  }
  if (rank == 0 && tid == 0) {
    st->ss_nb = fail ? 0 : nb;
    st->ss_fail = fail;
    st->ss_dbg[1] = (unsigned long long)nb;
  }
  if (rank == 0) coop_mark(st);
  cluster.sync();  // (the peers' shares stay alive until every CTA has gathered them)
  pdl_trace_end();
}

template <class Cand>
__global__ void __launch_bounds__(SS_TPB) k_ss_filter(Cand cand, CoopBufs B) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ unsigned s_w[32];
  __shared__ unsigned long long s_base;
  CoopState *st = B.st;
  const int nb = st->ss_nb;
  if (nb <= 0) return;
  Key3 *spl = reinterpret_cast<Key3 *>(dsm);
  unsigned *hcnt = reinterpret_cast<unsigned *>(spl + SS_SPL);
  for (int q = threadIdx.x; q < nb; q += blockDim.x) {
    spl[q] = B.kt[q];
    hcnt[q] = 0;
  }
  __syncthreads();
  const Key3 tau = spl[nb - 1];
  const int32_t hw = cand.hw();
  const int lane = threadIdx.x & 31;
  const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
  unsigned long long ccount = 0, mass = 0;  // per thread: candidates seen, weight kept
  for (int64_t s0 = (int64_t)blockIdx.x * blockDim.x; s0 < hw; s0 += UNR * gsz) {
    Key3 k[UNR];
    uint64_t v[UNR];
    int64_t w[UNR];
    int bk[UNR];
#pragma unroll
    for (int u = 0; u < UNR; u++) {  // UNR independent candidates in flight
      const int64_t s = s0 + u * gsz + threadIdx.x;
      w[u] = 0;
      const bool c = s < hw && cand((int32_t)s, k[u], v[u], w[u]);
      ccount += c ? 1 : 0;
      bk[u] = (c && !key_less(tau, k[u])) ? 0 : -1;
    }
    // the bucket of every kept candidate: first splitter >= k (exists: spl[nb-1] = tau >= k), the UNR
    // binary searches advanced in lock step (independent shared-memory loads in flight)
    int lo[UNR], hi[UNR];
#pragma unroll
    for (int u = 0; u < UNR; u++) {
      lo[u] = 0;
      hi[u] = bk[u] == 0 ? nb - 1 : 0;
    }
    for (int span = nb - 1; span > 0; span >>= 1) {  // (ceil(log2 nb) + 1 rounds bound every search)
#pragma unroll
      for (int u = 0; u < UNR; u++)
        if (lo[u] < hi[u]) {
          const int mid = (lo[u] + hi[u]) >> 1;
          if (key_less(spl[mid], k[u])) lo[u] = mid + 1;
          else hi[u] = mid;
        }
    }
#pragma unroll
    for (int u = 0; u < UNR; u++)
      if (lo[u] < hi[u]) {  // (a last step when nb is not a power of two)
        const int mid = (lo[u] + hi[u]) >> 1;
        if (key_less(spl[mid], k[u])) lo[u] = mid + 1;
        else hi[u] = mid;
      }
    unsigned nt = 0;
#pragma unroll
    for (int u = 0; u < UNR; u++) {
      if (bk[u] == 0) {
        bk[u] = lo[u];
        nt++;
        mass += (unsigned long long)w[u];
        atomicAdd(&hcnt[lo[u]], 1u);
      }
    }
    unsigned long long p = block_reserve(nt, &st->ss_n, s_w, &s_base);
#pragma unroll
    for (int u = 0; u < UNR; u++)
      if (bk[u] >= 0) {
        B.k0[p] = k[u];
        B.v0[p] = v[u];
        B.w0[p] = bk[u];
        p++;
      }
  }
  for (int o = 16; o > 0; o >>= 1) {
    ccount += __shfl_xor_sync(0xffffffffu, ccount, o);
    mass += __shfl_xor_sync(0xffffffffu, mass, o);
  }
  if (lane == 0) {
    if (ccount) atomicAdd(&st->ss_cand, ccount);
    if (mass) atomicAdd(&st->ss_mass, mass);
  }
  __syncthreads();
  for (int q = threadIdx.x; q < nb; q += blockDim.x)
    if (hcnt[q]) atomicAdd(&st->ss_cnt[q], hcnt[q]);
  pdl_trace_end();
}

__global__ void __launch_bounds__(SS_TPB) k_ss_scatter(CoopBufs B, int64_t W, const int64_t *dW) {
  pdl_wait();
  __shared__ unsigned s_off[SS_SPL + 1];
  __shared__ unsigned long long s_tot[32];
  if (dW) W = *dW;
  CoopState *st = B.st;
  const int nb = st->ss_nb;
  if (nb <= 0) return;
  const int64_t n = (int64_t)st->ss_n, ncand = (int64_t)st->ss_cand;
  // bucket offsets (every CTA; one warp-scan pass over <= SS_SPL counts)
  bool fits = true;
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int per = (nb + blockDim.x - 1) / blockDim.x, b0 = threadIdx.x * per, b1 = min(b0 + per, nb);
    unsigned sum = 0;
    for (int b = b0; b < b1; b++) {
      const unsigned c = st->ss_cnt[b];
      fits = fits && c <= (unsigned)SS_BBIG;
      sum += c;
    }
    unsigned x = sum;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_tot[wid] = x;
    __syncthreads();
    unsigned before = 0;
    for (int q = 0; q < wid; q++) before += (unsigned)s_tot[q];
    unsigned run = before + x - sum;
    for (int b = b0; b < b1; b++) {
      s_off[b] = run;
      run += st->ss_cnt[b];
    }
    if (threadIdx.x == 0) s_off[nb] = (unsigned)n;
    (void)nw;
  }
  fits = __syncthreads_and(fits);
  const bool ok = fits && ((int64_t)st->ss_mass >= W || n == ncand);
  if (blockIdx.x == 0) {
    for (int b = threadIdx.x; b <= nb; b += blockDim.x) st->ss_off[b] = s_off[b];
    if (threadIdx.x == 0) {
      st->ss_ok = ok ? 1 : 0;
      if (!ok) st->ss_fail = fits ? 5 : 4;
    }
  }
  if (!ok) return;
  // scatter into bucket order (warp-aggregated cursors)
  const int lane = threadIdx.x & 31;
  const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += gsz) {
    const int64_t i = i0 + threadIdx.x;
    const int b = i < n ? (int)B.w0[i] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, b);
    const int leader = __ffs(peers) - 1;
    unsigned base = 0;
    if (b >= 0 && lane == leader) base = atomicAdd(&st->ss_cur[b], (unsigned)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    if (b >= 0) {
      const unsigned p = s_off[b] + base + __popc(peers & ((1u << lane) - 1u));
      B.ks[p] = B.k0[i];
      B.vs[p] = B.v0[i];
    }
  }
  pdl_trace_end();
}

// the buckets over the CTAs: CTA c takes the buckets that start in the c-th
// 1/G of the selected items, and sorts runs of consecutive buckets (whole
// buckets, up to SS_SORT_CAP items) as ONE block_sort -- the buckets are in
// key order, so sorting their concatenation sorts each.  Every CTA sorts about
// n / G items in one or two passes (a bucket per sort, one at a time, left the
// kernel as long as a CTA's longest queue).  Buckets above SS_BMAX are
// k_build_coop's / k_ss_sort_big's.
__global__ void __launch_bounds__(SS_SORT_TPB, SS_SORT_PER_SM) k_ss_sort(CoopBufs B, Key3 *kout, uint64_t *vout) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char dsm[];
  CoopState *st = B.st;
  if (!st->ss_ok) return;
  const int nb = st->ss_nb;
  Key3 *sk = reinterpret_cast<Key3 *>(dsm);
  uint64_t *sv = reinterpret_cast<uint64_t *>(sk + SS_SORT_CAP);
  Key3 *tk = reinterpret_cast<Key3 *>(sv + SS_SORT_CAP);
  uint64_t *tv = reinterpret_cast<uint64_t *>(tk + SS_SORT_CAP);
  unsigned *off = reinterpret_cast<unsigned *>(tv + SS_SORT_CAP);
  for (int b = threadIdx.x; b <= nb; b += blockDim.x) off[b] = st->ss_off[b];
  __syncthreads();
  const unsigned long long n = off[nb], G = gridDim.x;
  const unsigned lo = (unsigned)(n * blockIdx.x / G), hi = (unsigned)(n * (blockIdx.x + 1) / G);
  auto lower = [&](unsigned x) {  // first bucket starting at or after item x
    int a = 0, z = nb;
    while (a < z) {
      const int m = (a + z) >> 1;
      if (off[m] < x) a = m + 1;
      else z = m;
    }
    return a;
  };
  int b = lower(lo);
  const int bend = lower(hi);
  while (b < bend) {  // (uniform: every thread reads the same shared offsets)
    if (off[b + 1] - off[b] > (unsigned)SS_BMAX) {
      b++;
      continue;
    }
    int e = b + 1;
    while (e < bend && off[e + 1] - off[e] <= (unsigned)SS_BMAX && off[e + 1] - off[b] <= (unsigned)SS_SORT_CAP) e++;
    const unsigned c0 = off[b];
    const int m = (int)(off[e] - c0);
    if (m > 0) {
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        sk[i] = B.ks[c0 + i];
        sv[i] = B.vs[c0 + i];
      }
      __syncthreads();
      block_sort(sk, sv, m, tk, tv, kout + c0, vout + c0);  // (ends on a barrier)
    }
    b = e;
  }
  pdl_trace_end();
}

// the rare buckets above SS_BMAX (geometric sizes): in-place bitonic in shared memory
__device__ inline void ss_sort_big_body(const CoopBufs &B, Key3 *kout, uint64_t *vout, unsigned char *dsm) {
  CoopState *st = B.st;
  const int nb = st->ss_nb;
  Key3 *sk = reinterpret_cast<Key3 *>(dsm);
  uint64_t *sv = reinterpret_cast<uint64_t *>(sk + SS_BBIG);
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    const int b0 = (int)st->ss_off[b], m0 = (int)(st->ss_off[b + 1] - st->ss_off[b]);
    if (m0 <= SS_BMAX) continue;
    if (2 * m0 <= SS_BBIG) {  // run merges (O(n log n)) with the scratch in the other half
      for (int i = threadIdx.x; i < m0; i += blockDim.x) {
        sk[i] = B.ks[b0 + i];
        sv[i] = B.vs[b0 + i];
      }
      __syncthreads();
      block_sort(sk, sv, m0, sk + m0, sv + m0, kout + b0, vout + b0);
      continue;
    }
    int mp = 1;
    while (mp < m0) mp <<= 1;
    for (int i = threadIdx.x; i < mp; i += blockDim.x) {
      if (i < m0) {
        sk[i] = B.ks[b0 + i];
        sv[i] = B.vs[b0 + i];
      } else {
        sk[i] = {~0ull, ~0ull, ~0ull};
        sv[i] = 0;
      }
    }
    __syncthreads();
    bitonic_smem(sk, sv, mp);
    for (int i = threadIdx.x; i < m0; i += blockDim.x) {
      kout[b0 + i] = sk[i];
      vout[b0 + i] = sv[i];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(512) k_ss_sort_big(CoopBufs B, Key3 *kout, uint64_t *vout) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char dsm[];
  if (!B.st->ss_ok) return;
  ss_sort_big_body(B, kout, vout, dsm);
}
constexpr size_t SS_BIG_SMEM = (sizeof(Key3) + 8) * SS_BBIG;
static_assert(SS_BIG_SMEM <= COOP_SMEM, "k_build_coop sorts the big buckets in its own shared memory");

// the eviction-order build after keys / subtree maxima (full-occupancy
// kernels k_build_keys, k_propagate) and the sample select: the prefix of the
// order with >= W tokens sorted into the list -- finalised here when the
// sample select succeeded (st->ss_ok), else by the materialising radix
// selection (everything when W <= 0) -- one cooperative launch, no host round trip.
__global__ void __launch_bounds__(COOP_TPB) k_build_coop(DT T, CoopBufs B, int64_t W, const int64_t *dW,
                                                         int64_t min_cand, int64_t small, int32_t sampled) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char dsm[];
  if (dW) {
    W = *dW;
    if (W < 0) return;  // device-side control: no eviction this wave, no list
  }
  __shared__ Key3 smin[COOP_TPB + 1], smax[COOP_TPB + 1];
  cg::grid_group grid = cg::this_grid();
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gsz = (int64_t)gridDim.x * blockDim.x;
  const int32_t hw = T.ctrl->hw;
  const EvictCand cand{T};
  coop_mark(B.st);
  int64_t nsel = 0, n = 0;
  const bool fast = sampled && B.st->ss_ok;
  if (fast) {
    nsel = (int64_t)B.st->ss_n;
    n = (int64_t)B.st->ss_cand;
    // the rare buckets above SS_BMAX (k_ss_sort_big's work; same shared memory)
    if (sampled == 2) ss_sort_big_body(B, T.Lk, T.Lv, dsm);
  } else {
    coop_gather(B, hw, cand);
    grid.sync();
    n = (int64_t)B.st->cand;
    nsel = n;
    if (W > 0 && n > min_cand) {
      nsel = coop_select(grid, B, n, W, small, smin, smax);
    } else {  // sort everything: move candidates to the selected buffer
      for (int64_t i = gtid; i < n; i += gsz) {
        B.ks[i] = B.k0[i];
        B.vs[i] = B.v0[i];
      }
      grid.sync();
    }
    coop_mark(B.st);
    coop_sort(grid, B, nsel, T.Lk, T.Lv, dsm);
  }
  coop_mark(B.st);
  if (gtid == 0) {
    Ctrl *c = T.ctrl;
    c->L_n = nsel;
    c->L_partial = nsel < n ? 1 : 0;
    c->L_cur = 0;
    c->L_valid = 1;
    c->H_n = 0;
    c->builds++;
    for (int i = 0; i < B.st->nts; i++) B.st->ts_build[i] = B.st->ts[i];
    B.st->nts_build = B.st->nts;
    for (int i = 0; i < 7; i++) B.st->ts_build[21 + i] = B.st->ss_dbg[i];
    for (int i = 0; i < 5; i++) B.st->ts_build[28 + i] = B.st->ss_prof[i];
    B.st->ts_build[33] = B.st->ss_ns;  // diagnostics of the sample select
    B.st->ts_build[34] = (unsigned long long)B.st->ss_nb;
    B.st->ts_build[35] = (unsigned long long)B.st->ss_fail;
    B.st->ts_build[36] = B.st->ss_mass;
    B.st->ts_build[37] = (unsigned long long)W;
    B.st->ts_build[38] = fast ? 1ull : 0ull;        // sampled path taken
    B.st->ts_build[39] = (unsigned long long)nsel;  // selected-prefix size
  }
  pdl_trace_end();
}

// ------------------------------------------------------------ small top-f
// set_protection for a small budget f (kvcache.py:364-383): the keys are
// (-P-hat, seg, id), so when at least f reusable anchors carry a positive
// P-hat -- the pending round's segments, a few thousand nodes -- the top f are
// among those.  k_tf_scan visits every slot once (clearing the previous flags,
// leaving the eviction keys when asked) and lists them; every slice of the
// list keeps its f smallest, merged across each cluster and then by the last
// cluster (k_tf_local).
// Otherwise ss_ok stays 0 and k_protect_coop runs the materialising selection.
constexpr int TF_MAX = 64;     // budgets up to this use the small top-f path
#ifndef PRISM_TF_SLICE
#define PRISM_TF_SLICE 256
#endif
constexpr int TF_SLICE = PRISM_TF_SLICE;  // list items per slice of k_tf_local (shared-memory sort)
constexpr size_t TF_SMEM = 2 * (sizeof(Key3) + 8) * TF_SLICE;

__global__ void __launch_bounds__(SS_TPB) k_tf_scan(ProtCand cand, CoopBufs B) {
  pdl_wait();
  __shared__ unsigned s_w[32];
  __shared__ unsigned long long s_base;
  const int32_t hw = cand.hw();
  const int lane = threadIdx.x & 31;
  const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
  unsigned long long ccount = 0;
  const DT &T = cand.T;
  const int32_t pol = T.policy;
  // ProtCand's visit, restated so that every load of the UNR slots is issued
  // before the first store (stores to prot / kw / eff would otherwise order
  // the next slot's loads behind them: one memory round trip per slot)
  for (int64_t s0 = (int64_t)blockIdx.x * blockDim.x; s0 < hw; s0 += UNR * gsz) {
    int64_t nid[UNR], last[UNR];
    int32_t par[UNR], ref[UNR], seg[UNR], hits[UNR];
    uint8_t kind[UNR], ha[UNR], ak[UNR];
#pragma unroll
    for (int u = 0; u < UNR; u++) {
      const int64_t s = s0 + u * gsz + threadIdx.x;
      const bool in = s < hw;
      nid[u] = in ? __ldg(&T.nid[s]) : -1;
      par[u] = in ? __ldg(&T.par[s]) : -1;
      seg[u] = in ? __ldg(&T.seg[s]) : SEG_NONE;
      ha[u] = in ? __ldg(&T.hasanc[s]) : 0;
      ak[u] = in ? __ldg(&T.akind[s]) : 0;
      if (cand.keys) {
        ref[u] = in ? __ldg(&T.ref[s]) : 0;
        kind[u] = in ? __ldg(&T.kind[s]) : 0;
        last[u] = in ? __ldg(&T.last[s]) : 0;
        hits[u] = (in && pol == P_LFU) ? __ldg(&T.hits[s]) : 0;
      }
    }
    double ps[UNR];
    bool act[UNR];
#pragma unroll
    for (int u = 0; u < UNR; u++) {
      const int32_t sg = seg[u];
      ps[u] = (sg != SEG_NONE && sg >= 0 && sg < T.npri) ? __ldg(&T.pri[sg]) : 0.0;
      act[u] = cand.keys && pol == P_LRU_ACTIVE && act_of(T, sg);
    }
    Key3 k[UNR];
    bool pos[UNR];
    unsigned nt = 0;
#pragma unroll
    for (int u = 0; u < UNR; u++) {
      const int64_t s = s0 + u * gsz + threadIdx.x;
      pos[u] = false;
      if (s >= hw) continue;
      T.prot[s] = 0;
      const bool live = s != ROOT && nid[u] >= 0 && par[u] >= 0;
      if (cand.keys) {
        if (!live) {
          T.eff[s] = EFF_DEAD;
        } else {
          const bool blocked = ref[u] > 0 || (pol == P_DART && kind[u] == K_SYSTEM);
          T.kw[s] = make_key_v(pol, last[u], nid[u], kind[u], false, ps[u], hits[u], act[u]);
          T.eff[s] = blocked ? EFF_BLOCKED : (int32_t)s;
        }
      }
      const bool c = live && ha[u] && ak[u] == K_REUSABLE;
      ccount += c ? 1 : 0;
      if (c) {
        const int32_t sv = seg[u] == SEG_NONE ? -1 : seg[u];
        k[u] = {0, 0, 0};
        shl_or(k[u], 64, ord_f64(-ps[u]));
        shl_or(k[u], 32, (uint64_t)((uint32_t)sv ^ 0x80000000u));
        shl_or(k[u], 40, (uint64_t)nid[u] & ((1ull << 40) - 1));
      }
      pos[u] = c && ps[u] > 0.0;
      nt += pos[u] ? 1 : 0;
    }
    unsigned long long p = block_reserve(nt, &B.st->tf_n, s_w, &s_base);
#pragma unroll
    for (int u = 0; u < UNR; u++)
      if (pos[u]) {
        B.k1[p] = k[u];
        B.v1[p] = (uint64_t)(uint32_t)(s0 + u * gsz + threadIdx.x);
        p++;
      }
  }
  for (int o = 16; o > 0; o >>= 1) ccount += __shfl_xor_sync(0xffffffffu, ccount, o);
  if (lane == 0 && ccount) atomicAdd(&B.st->ss_cand, ccount);
  pdl_trace_end();
}

// merge a sorted list of F (rk/rv[cur], padded with all-ones keys) with
// another sorted list o of F into rk/rv[cur ^ 1]: an item's place is its index
// plus its rank in the other list (real keys are distinct; the pads rank
// after every real key, so they only fill places past the real items)
__device__ __forceinline__ void tf_merge2(Key3 (*rk)[TF_MAX], uint64_t (*rv)[TF_MAX], int cur, const Key3 *ok,
                                          const uint64_t *ov, int F) {
  const int nxt = cur ^ 1;
  for (int t = threadIdx.x; t < 2 * F; t += blockDim.x) {
    const bool run = t < F;
    const int i = run ? t : t - F;
    const Key3 x = run ? rk[cur][i] : ok[i];
    const Key3 *O = run ? ok : rk[cur];
    int lo = 0, hi = F;  // the running list's items go before equal ones (pads)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (run ? key_less(O[mid], x) : !key_less(x, O[mid])) lo = mid + 1;
      else hi = mid;
    }
    const int pos = i + lo;
    if (pos < F) {
      rk[nxt][pos] = x;
      rv[nxt][pos] = run ? rv[cur][i] : ov[i];
    }
  }
  __syncthreads();
}

// The top f of the positive-P-hat list in one launch of TF_CL-CTA clusters:
//  * every CTA keeps the f smallest keys of ITS slices (c = blockIdx.x,
//    + gridDim.x, ...): each TF_SLICE-item slice is sorted in shared memory and
//    its top f merged into the running top f;
//  * the cluster's rank-0 CTA merges its peers' lists straight out of their
//    shared memory (DSMEM) and publishes the cluster's top f;
//  * the last cluster to publish (a counter) merges the <= TF_FIN / f cluster
//    lists pairwise in shared memory and applies the protection -- what one
//    separate single-CTA merge over every CTA's list (~3000 items) did before.
constexpr int TF_CL = 8;      // CTAs per cluster
#ifndef PRISM_TF_FIN
#define PRISM_TF_FIN 512
#endif
constexpr int TF_FIN = PRISM_TF_FIN;   // cluster lists x f merged by the last cluster
constexpr size_t TF_LOCAL_SMEM =
    std::max(TF_SMEM, (size_t)2 * (sizeof(Key3) + 8) * TF_FIN);

__global__ void __cluster_dims__(TF_CL, 1, 1) __launch_bounds__(SS_TPB)
    k_tf_local(DT T, CoopBufs B, int64_t f, int32_t keys) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ Key3 rk[2][TF_MAX];
  __shared__ uint64_t rv[2][TF_MAX];
  __shared__ Key3 fk[TF_MAX];  // this CTA's top f, read by the cluster's rank 0
  __shared__ uint64_t fv[TF_MAX];
  __shared__ bool s_last;
  const int64_t n = (int64_t)B.st->tf_n;
  if (n < f || f <= 0) return;  // (uniform) ss_ok stays 0: the materialising path decides
  cg::cluster_group cluster = cg::this_cluster();
  Key3 *sk = reinterpret_cast<Key3 *>(dsm);
  uint64_t *sv = reinterpret_cast<uint64_t *>(sk + TF_SLICE);
  Key3 *tk = reinterpret_cast<Key3 *>(sv + TF_SLICE);
  uint64_t *tv = reinterpret_cast<uint64_t *>(tk + TF_SLICE);
  const int F = (int)f;
  const Key3 PAD{~0ull, ~0ull, ~0ull};
  __shared__ int s_m;
  int have = 0, cur = 0;  // running top list: rk/rv[cur][0..have)
  for (int64_t c = blockIdx.x; c * TF_SLICE < n; c += gridDim.x) {
    const int64_t b0 = c * TF_SLICE;
    int m = (int)(n - b0 < TF_SLICE ? n - b0 : TF_SLICE);
    if (have == F) {  // (uniform) only the slice's keys below the running f-th can enter: sort just those
      if (threadIdx.x == 0) s_m = 0;
      __syncthreads();
      const Key3 thr = rk[cur][F - 1];
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const Key3 x = B.k1[b0 + i];
        if (key_less(x, thr)) {
          const int q = atomicAdd(&s_m, 1);
          sk[q] = x;
          sv[q] = B.v1[b0 + i];
        }
      }
      __syncthreads();
      m = s_m;
      __syncthreads();
      if (m == 0) continue;
    } else {
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        sk[i] = B.k1[b0 + i];
        sv[i] = B.v1[b0 + i];
      }
      __syncthreads();
    }
    block_merge_sort(sk, sv, m, tk, tv, sk, sv);
    const int keep = m < F ? m : F;
    const int nxt = cur ^ 1;
    for (int t = threadIdx.x; t < have + keep; t += blockDim.x) {
      const bool run = t < have;
      const int i = run ? t : t - have;
      const Key3 x = run ? rk[cur][i] : sk[i];
      const Key3 *O = run ? sk : rk[cur];
      int lo = 0, hi = run ? keep : have;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (key_less(O[mid], x)) lo = mid + 1;
        else hi = mid;
      }
      const int pos = i + lo;
      if (pos < F) {
        rk[nxt][pos] = x;
        rv[nxt][pos] = run ? rv[cur][i] : sv[i];
      }
    }
    __syncthreads();
    have = have + keep < F ? have + keep : F;
    cur = nxt;
  }
  for (int i = threadIdx.x; i < F; i += blockDim.x) {
    fk[i] = i < have ? rk[cur][i] : PAD;
    fv[i] = i < have ? rv[cur][i] : 0ull;
  }
  cluster.sync();
  const unsigned cid = blockIdx.x / TF_CL, ncl = gridDim.x / TF_CL;
  if (cluster.block_rank() == 0) {
    for (int i = threadIdx.x; i < F; i += blockDim.x) {
      rk[0][i] = fk[i];
      rv[0][i] = fv[i];
    }
    __syncthreads();
    int c2 = 0;
    for (unsigned r = 1; r < TF_CL; r++, c2 ^= 1)
      tf_merge2(rk, rv, c2, cluster.map_shared_rank(fk, r), cluster.map_shared_rank(fv, r), F);
    for (int i = threadIdx.x; i < F; i += blockDim.x) {
      B.ks[(int64_t)cid * F + i] = rk[c2][i];
      B.vs[(int64_t)cid * F + i] = rv[c2][i];
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&B.st->tf_cl, 1u) == ncl - 1;
  }
  cluster.sync();  // (the peers' shared memory stays alive until rank 0 has read it)
  if (cluster.block_rank() != 0 || !s_last) return;
  __threadfence();
  // the last cluster: pairwise rounds over the ncl cluster lists (TF_FIN items at most)
  Key3 *ak = reinterpret_cast<Key3 *>(dsm);
  uint64_t *av = reinterpret_cast<uint64_t *>(ak + TF_FIN);
  Key3 *bk = reinterpret_cast<Key3 *>(av + TF_FIN);
  uint64_t *bv = reinterpret_cast<uint64_t *>(bk + TF_FIN);
  for (int i = threadIdx.x; i < (int)ncl * F; i += blockDim.x) {
    // (other SMs' stores: L2-coherent loads)
    ak[i] = Key3{__ldcg(&B.ks[i].w0), __ldcg(&B.ks[i].w1), __ldcg(&B.ks[i].w2)};
    av[i] = __ldcg(&B.vs[i]);
  }
  __syncthreads();
  int Ln = (int)ncl;
  while (Ln > 1) {
    const int pairs = Ln >> 1;
    for (int t = threadIdx.x; t < pairs * 2 * F; t += blockDim.x) {
      const int q = t / (2 * F), side = (t / F) & 1, i = t % F;
      const Key3 *A = ak + (2 * q) * F, *Bl = ak + (2 * q + 1) * F;
      const Key3 x = side ? Bl[i] : A[i];
      const Key3 *O = side ? A : Bl;  // the other list
      int lo = 0, hi = F;  // A's items go before equal B items (stable)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (side ? !key_less(x, O[mid]) : key_less(O[mid], x)) lo = mid + 1;
        else hi = mid;
      }
      const int pos = i + lo;
      if (pos < F) {
        bk[q * F + pos] = x;
        bv[q * F + pos] = side ? av[(2 * q + 1) * F + i] : av[(2 * q) * F + i];
      }
    }
    if (Ln & 1)
      for (int i = threadIdx.x; i < F; i += blockDim.x) {
        bk[pairs * F + i] = ak[(Ln - 1) * F + i];
        bv[pairs * F + i] = av[(Ln - 1) * F + i];
      }
    __syncthreads();
    Key3 *tk2 = ak;
    ak = bk;
    bk = tk2;
    uint64_t *tv2 = av;
    av = bv;
    bv = tv2;
    Ln = pairs + (Ln & 1);
  }
  for (int i = threadIdx.x; i < F; i += blockDim.x) {
    T.Lk[i] = ak[i];
    T.Lv[i] = av[i];
  }
  __syncthreads();
  // and k_protect_coop's last step (f <= n here), so that launch returns at once
  for (int i = threadIdx.x; i < F; i += blockDim.x) {
    const int32_t s = (int32_t)(av[i] & 0xffffffffu);
    T.prot[s] = 1;
    if (keys) T.kw[s] = make_key(T, s);  // protected: class 2 (kvcache.py:405-406)
    if (B.out_ids) B.out_ids[i] = T.nid[s];
  }
  if (threadIdx.x == 0) {
    B.st->ss_ok = 1;
    B.st->prot_n = F;
    B.st->tf_done = 1;
  }
  pdl_trace_end();
}

// set_protection (kvcache.py:364-383): top-f reusable anchors by (-P-hat, seg
// or -1, id) -- from the small top-f / sample select when it succeeded, else materialised
__global__ void __launch_bounds__(COOP_TPB) k_protect_coop(DT T, CoopBufs B, int64_t f, int64_t min_cand,
                                                           int64_t small, int32_t sampled, int32_t keys) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ Key3 smin[COOP_TPB + 1], smax[COOP_TPB + 1];
  if (sampled && B.st->tf_done) return;  // the small top-f path already protected
  cg::grid_group grid = cg::this_grid();
  const int32_t hw = T.ctrl->hw;
  const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const ProtCand cand{T, keys};
  int64_t n = 0, nsel = 0;
  const bool fast = sampled && B.st->ss_ok;
  if (fast) {
    n = (int64_t)B.st->ss_cand;
  } else {
    coop_gather(B, hw, cand);
    grid.sync();
    n = (int64_t)B.st->cand;
  }
  const int64_t nf = f < n ? f : n;
  if (nf <= 0) {
    if (gtid == 0) B.st->prot_n = 0;
    return;
  }
  if (!fast) {
    nsel = n;
    if (n > min_cand) {
      nsel = coop_select(grid, B, n, nf, small, smin, smax);
    } else {
      for (int64_t i = gtid; i < n; i += gsz) {
        B.ks[i] = B.k0[i];
        B.vs[i] = B.v0[i];
      }
      grid.sync();
    }
    coop_sort(grid, B, nsel, T.Lk, T.Lv, dsm);  // Lk/Lv as scratch: no list survives a call
  }
  for (int64_t i = gtid; i < nf; i += gsz) {
    const int32_t s = (int32_t)(T.Lv[i] & 0xffffffffu);
    T.prot[s] = 1;
    if (keys) T.kw[s] = make_key(T, s);  // protected: class 2 (kvcache.py:405-406)
    if (B.out_ids) B.out_ids[i] = T.nid[s];
  }
  if (gtid == 0) B.st->prot_n = nf;
}

}  // namespace prism

// qas_small.cuh -- one QAS round (scheduler.py:192-273) in ONE launch.
//
// For pending sets of up to QS_MAXP requests the whole round is one kernel:
// a single 1024-thread CTA for small sets, a cooperative grid (grid barriers
// between phases) for larger ones.  No host round trips; the parallel phases
// (counters, alignment + signatures, bucket hashing, distinct (bucket,
// segment) pairs, utility terms, hot-lane scatter, priorities) are strided over
// the grid, the short serial ones run in block 0's shared memory: bucket
// creation order and the in-bucket ranks (a warp pass in pending order), the
// score sort, and the cold lane (a byte radix select of the oldest leftovers,
// then a sort of just those).  Segment counters are reset through the list of
// segments the previous round touched, so the cost is O(P*k), not
// O(num_segments).
//
// Exactness: identical float expressions to qas.cu / the reference; the
// utility sum uses int64 accumulation and is therefore only used when every
// term is an exact integer (integral weights: the reference defaults) -- the
// host selects this kernel only then.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>

namespace qsmall {

constexpr int QS_TPB = 1024;
constexpr int QS_MAXP = 8192;  // pending requests of a one-launch round (shared-memory lists / sorts)
constexpr int QS_MAXK = 16;   // alignment by a 16-lane group (two requests per warp)
constexpr int QS_MAXW = 64;   // alignment by one warp (two entries per lane); longer skeletons: a whole block
constexpr int QS_SKCAP = 64;  // skeleton entries per request provisioned (aligned, pair table)
constexpr uint64_t QS_EMPTY = ~0ull;

struct QsCfg {
  int64_t budget, cold, front, kappa;
  double wg, wa, wn, alpha, beta;
};

struct QsArgs {
  // inputs (device)
  int64_t P, A;
  const int64_t *ids;
  const double *arrival;
  const int64_t *off;
  const int32_t *sk;
  const uint8_t *reo;
  const int64_t *aoff;
  const int32_t *ask;
  // dense per-segment outputs (kept zero outside the touched list)
  int32_t *g, *a, *nd;
  double *prio;
  uint8_t *dom;
  int32_t *touched;      // segments with a non-zero counter this round
  int32_t *touched_n;    // [0] this round, [1] previous round (to reset)
  int32_t *prev_touched; // previous round's list
  // per-request outputs
  int32_t *aligned, *sig, *siglen, *rank, *bucket;
  int64_t *hot, *cold;
  double *score;  // per bucket, creation order
  int64_t *counts;  // [0] nhot [1] ncold [2] nbuckets [3] redo multi-kernel [4] nlong [5] npairs
  // scratch (global)
  uint64_t *btab_key;  // signature table, size 2*QS_MAXP (power of two)
  int32_t *btab_min, *slot_of, *bidx;
  int32_t *bsize, *nsegs;
  int32_t *btake, *bbase;  // per bucket: hot-lane members taken, first hot-lane position
  long long *isum;
  uint64_t *ptab_key;  // (bucket, seg) pair table (the kernel uses 2*nsk slots of it)
  int64_t ptab_cap, btab_mask;
  int32_t *longl;       // requests with skeletons longer than QS_MAXK
  int32_t *rk;          // rank scratch for them (aligned_cap ints)
  int32_t *emap;        // pending skeleton entry -> its request (aligned_cap ints)
  uint8_t *efirst;      // pending skeleton entry is its segment's first occurrence in the skeleton
  int64_t aligned_cap;  // capacity of aligned / rk in skeleton entries
  unsigned long long *ts;  // QS_NTS phase stamps, or null
};
constexpr int QS_NTS = 11;

__device__ inline uint64_t qmix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

__device__ inline uint64_t qord(double d) {
  if (d == 0.0) d = 0.0;
  const uint64_t b = (uint64_t)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ inline double qpri0(const QsCfg &c, const int32_t *g, const int32_t *a, int32_t s) {
  return __dadd_rn(__dmul_rn(c.wg, (double)g[s]), __dmul_rn(c.wa, (double)a[s]));
}

__device__ inline bool qrank_before(double pa, int32_t sa, int ia, double pb, int32_t sb, int ib) {
  if (pa != pb) return pa > pb;
  if (sa != sb) return sa < sb;
  return ia < ib;
}

// front_align + make_signature (scheduler.py:109-143) of ONE request with a
// skeleton of any length k, by the whole block (every thread must call it).
// The stable sort by (-pri, seg) is replaced by rank counting, O(k^2) over the
// block: rank(j) = #{i : (p_i, s_i, i) before (p_j, s_j, j)} -- a strict total
// order, so the ranks are the sorted positions.  rk: k ints of scratch.
// Returns siglen (valid in every thread).
__device__ inline int align_long_block(const int32_t *s, int k, bool reo, const int32_t *g, const int32_t *a,
                                       double wg, double wa, int64_t front, int64_t kappa, int32_t *al,
                                       int32_t *sig, int32_t *rk) {
  const int tid = threadIdx.x, nt = blockDim.x;
  auto pri = [&](int32_t x) { return __dadd_rn(__dmul_rn(wg, (double)g[x]), __dmul_rn(wa, (double)a[x])); };
  const int f = (int)(front < k ? front : k);
  if (!reo || k == 0) {
    for (int j = tid; j < k; j += nt) al[j] = s[j];
  } else {
    for (int j = tid; j < k; j += nt) {
      const double pj = pri(s[j]);
      int r = 0;
      for (int i = 0; i < k; i++) r += qrank_before(pri(s[i]), s[i], i, pj, s[j], j);
      rk[j] = r;
    }
    __syncthreads();
    for (int j = tid; j < k; j += nt) {
      if (rk[j] < f) {
        al[rk[j]] = s[j];  // the fronted segments, in rank order
      } else {
        int before = 0;  // fronted segments ahead of j in the skeleton
        for (int i = 0; i < j; i++) before += rk[i] < f;
        al[f + j - before] = s[j];
      }
    }
  }
  __syncthreads();
  const int kk = (int)(kappa < k ? kappa : k);
  for (int j = tid; j < k; j += nt) {
    const double pj = pri(al[j]);
    int r = 0;
    for (int i = 0; i < k && r < kk; i++) r += qrank_before(pri(al[i]), al[i], i, pj, al[j], j);
    rk[j] = r < kk;  // chosen: among the top-kappa
  }
  __syncthreads();
  for (int j = tid; j < k; j += nt) {
    if (rk[j]) {
      int pos = 0;  // emitted in aligned order
      for (int i = 0; i < j; i++) pos += rk[i];
      sig[pos] = al[j];
    }
  }
  __syncthreads();
  return kk;
}

// block-wide exclusive scan of n int32 values in place (loops over 1024-chunks)
__device__ inline int32_t block_exscan(int32_t *v, int n, int32_t *swarp) {
  __shared__ int32_t s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int32_t x = i < n ? v[i] : 0;
    int32_t incl = x;
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) swarp[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int32_t w = lane < (int)(blockDim.x >> 5) ? swarp[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      swarp[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    const int32_t wbase = wid ? swarp[wid - 1] : 0;
    if (i < n) v[i] = s_carry + wbase + incl - x;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += swarp[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  return s_carry;
}

struct QKey {
  uint64_t hi, lo;
};
__device__ __forceinline__ bool qk_less(const QKey &x, const QKey &y) {  // branch-free
  return (x.hi < y.hi) | ((x.hi == y.hi) & (x.lo < y.lo));
}

// bitonic sort of n <= QS_MAXP (key, value) pairs in shared memory
__device__ inline void block_bitonic(QKey *k, int32_t *v, int n) {
  int m = 1;
  while (m < n) m <<= 1;
  for (int i = n + threadIdx.x; i < m; i += blockDim.x) {
    k[i] = {~0ull, ~0ull};
    v[i] = -1;
  }
  __syncthreads();
  for (int size = 2; size <= m; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const bool sw = up ? qk_less(k[j], k[i]) : qk_less(k[i], k[j]);
          if (sw) {
            const QKey tk = k[i];
            k[i] = k[j];
            k[j] = tk;
            const int32_t tv = v[i];
            v[i] = v[j];
            v[j] = tv;
          }
        }
      }
      __syncthreads();
    }
  }
}

constexpr size_t QS_SMEM = (sizeof(QKey) + 2 * sizeof(int32_t)) * QS_MAXP;

// 3. bucket of request i's signature tuple; first member via atomicMin
// (scheduler.py:211-223).  Open addressing on (hash, first index seen).
// Other CTAs compare against the signature published with the CAS: it is
// fenced before, and read through L2 after.
__device__ inline void qs_bucket_insert(const QsArgs &A, const QsCfg &c, int64_t i, int sl) {
  __threadfence();
  uint32_t h = 2166136261u ^ (uint32_t)sl;
  for (int j = 0; j < sl; j++) h = (h ^ (uint32_t)A.sig[i * c.kappa + j]) * 16777619u;
  const uint64_t mine = ((uint64_t)h << 32) | (uint32_t)i;
  uint64_t pos = qmix64(h) & (uint64_t)A.btab_mask;
  for (;;) {
    unsigned long long prev = __ldcg((const unsigned long long *)&A.btab_key[pos]);
    if (prev == QS_EMPTY) prev = atomicCAS((unsigned long long *)&A.btab_key[pos], QS_EMPTY, mine);
    bool same = prev == QS_EMPTY;
    if (!same && (uint32_t)(prev >> 32) == h) {
      const int64_t o = (int64_t)(prev & 0xffffffffu);
      same = __ldcg(&A.siglen[o]) == sl;
      for (int j = 0; same && j < sl; j++) same = __ldcg(&A.sig[o * c.kappa + j]) == A.sig[i * c.kappa + j];
    }
    if (same) {
      atomicMin(&A.btab_min[pos], (int32_t)i);
      A.slot_of[i] = (int32_t)pos;
      return;
    }
    pos = (pos + 1) & (uint64_t)A.btab_mask;
  }
}

__device__ inline unsigned long long qs_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// phase timeline (profiling only): ts[n] = %globaltimer at the end of phase n
#define QS_TS(n)                                                         \
  do {                                                                   \
    if (A.ts && blockIdx.x == 0 && threadIdx.x == 0) A.ts[n] = qs_gtimer(); \
  } while (0)

// grid-wide barrier; a plain block barrier when the round runs in one CTA
__device__ inline void qs_gsync() {
  if (gridDim.x == 1) {
    __syncthreads();
  } else {
    cooperative_groups::this_grid().sync();
  }
}

__device__ inline int32_t qs_ld(const int32_t *p) { return __ldcg(p); }  // L2 (coherent across CTAs)

// position of this thread within one sweep of gs = gridDim * blockDim items,
// interleaved over the CTAs (item t of a sweep goes to CTA t % gridDim), so a
// sweep of fewer items than threads still spreads over every SM
__device__ inline int64_t qs_ilv(int64_t gs) {
  (void)gs;
  return (int64_t)threadIdx.x * gridDim.x + blockIdx.x;
}

// skeleton entry e of a request starting at entry b: its segment, and whether
// it is the segment's first occurrence in that skeleton (count_segments dedup)
__device__ inline bool qs_first(const int32_t *sk, int64_t b, int64_t e, int32_t &s) {
  s = sk[e];
  for (int64_t q = b; q < e; q++)
    if (sk[q] == s) return false;
  return true;
}

// first-occurrence flags and the entry -> request map of request i's skeleton
// [b, b+k), by one warp (count_segments' per-request dedup, scheduler.py:83-89):
// k <= 64 by __match_any over the lanes (entries lane, lane+32), longer
// skeletons by a strided backward scan
__device__ inline void qs_flags_warp(const QsArgs &A, int64_t i, int64_t b, int64_t k) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  if (k <= QS_MAXW) {
    const int32_t s0 = lane < k ? A.sk[b + lane] : -1;
    const int32_t s1 = lane + 32 < k ? A.sk[b + lane + 32] : -1;
    const bool f0 = (__match_any_sync(0xffffffffu, s0) & lt) == 0u;
    bool f1 = (__match_any_sync(0xffffffffu, s1) & lt) == 0u;
    if (k > 32) {
#pragma unroll 8
      for (int q = 0; q < 32; q++) f1 &= __shfl_sync(0xffffffffu, s0, q) != s1;
    }
    if (lane < k) {
      A.emap[b + lane] = (int32_t)i;
      A.efirst[b + lane] = f0 ? 1 : 0;
    }
    if (lane + 32 < k) {
      A.emap[b + lane + 32] = (int32_t)i;
      A.efirst[b + lane + 32] = f1 ? 1 : 0;
    }
  } else {
    for (int64_t e = b + lane; e < b + k; e += 32) {
      int32_t s = 0;
      A.emap[e] = (int32_t)i;
      A.efirst[e] = qs_first(A.sk, b, e, s) ? 1 : 0;
    }
  }
}

// one selection candidate: (priority, segment, index) -- ranked by (-pri, seg, index)
struct QsCand {
  double p;
  int32_t s, x;
  bool v;
};
__device__ __forceinline__ bool qs_cand_better(const QsCand &a, const QsCand &b) {
  return a.v && (!b.v || qrank_before(a.p, a.s, a.x, b.p, b.s, b.x));
}
// the warp's best candidate (every lane gets it; a strict total order, so the
// butterfly converges to the same element everywhere)
__device__ __forceinline__ QsCand qs_warp_best(QsCand m) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    QsCand y;
    y.p = __shfl_xor_sync(0xffffffffu, m.p, o);
    y.s = __shfl_xor_sync(0xffffffffu, m.s, o);
    y.x = __shfl_xor_sync(0xffffffffu, m.x, o);
    y.v = __shfl_xor_sync(0xffffffffu, m.v ? 1 : 0, o) != 0;
    if (qs_cand_better(y, m)) m = y;
  }
  return m;
}

// front_align + make_signature (scheduler.py:109-143) of request i with
// QS_MAXK < k <= QS_MAXW skeleton entries by ONE warp, lane holding entries
// lane and lane+32 in registers.  The top-f (front) and the top-kappa
// (signature) are found by f resp. kappa warp-argmax selection rounds over
// (-pri, seg, index) -- the sorted prefixes the reference takes -- so the cost
// is O((f + kappa) log 32) shuffles, not a k^2 rank count.
__device__ inline void qs_align_warp(const QsArgs &A, const QsCfg &c, int64_t i, int64_t b, int k, bool reo) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int32_t s[2];
  double p[2];
  bool v[2];
  int pos[2] = {lane, lane + 32};
#pragma unroll
  for (int u = 0; u < 2; u++) {
    v[u] = lane + 32 * u < k;
    s[u] = v[u] ? A.sk[b + lane + 32 * u] : 0;
    p[u] = v[u] ? qpri0(c, A.g, A.a, s[u]) : 0.0;
  }
  if (reo) {  // the top-f to the front in rank order, the rest stable (109-129)
    const int f = (int)(c.front < k ? c.front : k);
    int rk[2] = {-1, -1};
    for (int t = 0; t < f; t++) {
      QsCand m0{p[0], s[0], lane, v[0] && rk[0] < 0}, m1{p[1], s[1], lane + 32, v[1] && rk[1] < 0};
      const QsCand w = qs_warp_best(qs_cand_better(m1, m0) ? m1 : m0);
      if (w.x == lane) rk[0] = t;
      if (w.x == lane + 32) rk[1] = t;
    }
    const unsigned rlo = __ballot_sync(0xffffffffu, v[0] && rk[0] < 0);
    const unsigned rhi = __ballot_sync(0xffffffffu, v[1] && rk[1] < 0);
    pos[0] = rk[0] >= 0 ? rk[0] : f + __popc(rlo & lt);
    pos[1] = rk[1] >= 0 ? rk[1] : f + __popc(rlo) + __popc(rhi & lt);
  }
#pragma unroll
  for (int u = 0; u < 2; u++)
    if (v[u]) A.aligned[b + pos[u]] = s[u];
  // signature: the top-kappa by (-pri, seg, aligned position), emitted in aligned order (132-143)
  const int kk = (int)(c.kappa < k ? c.kappa : k);
  bool ch[2] = {false, false};
  for (int t = 0; t < kk; t++) {
    QsCand m0{p[0], s[0], pos[0], v[0] && !ch[0]}, m1{p[1], s[1], pos[1], v[1] && !ch[1]};
    const QsCand w = qs_warp_best(qs_cand_better(m1, m0) ? m1 : m0);
    ch[0] |= v[0] && w.x == pos[0];
    ch[1] |= v[1] && w.x == pos[1];
  }
  unsigned mlo = 0u, mhi = 0u;  // chosen aligned positions
#pragma unroll
  for (int u = 0; u < 2; u++)
    if (ch[u]) {
      if (pos[u] < 32) mlo |= 1u << pos[u];
      else mhi |= 1u << (pos[u] - 32);
    }
  mlo = __reduce_or_sync(0xffffffffu, mlo);
  mhi = __reduce_or_sync(0xffffffffu, mhi);
#pragma unroll
  for (int u = 0; u < 2; u++)
    if (ch[u]) {
      const int before = pos[u] < 32 ? __popc(mlo & ((1u << pos[u]) - 1u))
                                     : __popc(mlo) + __popc(mhi & ((1u << (pos[u] - 32)) - 1u));
      A.sig[i * c.kappa + before] = s[u];
    }
  __syncwarp();
  if (lane == 0) {
    const int sl = k > 0 ? kk : 0;
    A.siglen[i] = sl;
    qs_bucket_insert(A, c, i, sl);  // 3.
  }
}

// warp-aggregated append of c items at *ctr (int32 counter); returns this
// lane's first position (every lane of the warp calls it)
__device__ inline int qs_warp_reserve(int c, int32_t *ctr) {
  const int lane = threadIdx.x & 31;
  int x = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  int base = 0;
  if (lane == 31 && x) base = atomicAdd(ctr, x);
  return __shfl_sync(0xffffffffu, base, 31) + x - c;
}

// qs_warp_reserve for a whole CTA (one counter atomic per CTA instead of per
// warp: every warp of a sweep appending hammers one address); block-uniform
__device__ inline int qs_block_reserve(int c, int32_t *ctr) {
  __shared__ int s_w[33];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int t = lane < nw ? s_w[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) s_w[lane] = t;  // inclusive per-warp prefix
    if (lane == 31) s_w[32] = t ? atomicAdd(ctr, t) : 0;
  }
  __syncthreads();
  const int r = s_w[32] + (wid ? s_w[wid - 1] : 0) + x - c;
  __syncthreads();  // (s_w reused by the next call)
  return r;
}

// cold lane (242-245) in block 0: the nc smallest leftovers by (arrival, id),
// sorted.  Leftovers are compacted into shared memory; when fewer than all of
// them are taken, an MSB-first byte radix select over the 128-bit keys finds
// exactly the nc smallest (keys are distinct: ids are unique), so only those
// are sorted.
__device__ inline void qs_cold_lane(const QsArgs &A, const QsCfg &c, int64_t P, int64_t nc, QKey *sk,
                                    int32_t *sv, int32_t *tmp, int32_t *swarp) {
  __shared__ int32_t hist[256];
  __shared__ int32_t s_need, s_digit, s_done;
  const int tid = threadIdx.x, nt = blockDim.x;
  // the leftovers (rank >= their bucket's take), listed here -- beside the
  // other CTAs' hot lane -- in any order (the keys are distinct)
  __shared__ int32_t s_m;
  if (tid == 0) s_m = 0;
  __syncthreads();
  constexpr int CU = 4;  // requests per thread per round, their loads in flight together
  for (int64_t i0 = 0; i0 < P; i0 += (int64_t)CU * nt) {
    int32_t rk[CU], bk[CU];
    double ar[CU];
    int64_t id[CU];
    bool lf[CU];
#pragma unroll
    for (int u = 0; u < CU; u++) {
      const int64_t i = i0 + (int64_t)u * nt + tid;
      rk[u] = i < P ? A.rank[i] : 0;
      bk[u] = i < P ? A.bucket[i] : 0;
      ar[u] = i < P ? A.arrival[i] : 0.0;
      id[u] = i < P ? A.ids[i] : 0;
    }
#pragma unroll
    for (int u = 0; u < CU; u++) {
      const int64_t i = i0 + (int64_t)u * nt + tid;
      lf[u] = i < P && rk[u] >= qs_ld(&A.btake[bk[u]]);
    }
#pragma unroll
    for (int u = 0; u < CU; u++) {
      const int64_t i = i0 + (int64_t)u * nt + tid;
      const unsigned mt = __ballot_sync(0xffffffffu, lf[u]);
      int base = 0;
      if ((tid & 31) == 0 && mt) base = atomicAdd(&s_m, __popc(mt));
      base = __shfl_sync(0xffffffffu, base, 0) + __popc(mt & ((1u << (tid & 31)) - 1u));
      if (lf[u]) {
        sk[base] = {qord(ar[u]), (uint64_t)id[u] ^ 0x8000000000000000ull};
        sv[base] = (int32_t)i;
      }
    }
  }
  __syncthreads();
  const int m = s_m;
  int n = m;
  if (nc < m) {
    uint8_t *st = reinterpret_cast<uint8_t *>(tmp);  // 0 candidate, 1 taken, 2 dropped
    __shared__ unsigned long long s_dh, s_dl;
    for (int q = tid; q < m; q += nt) st[q] = 0;
    if (tid == 0) {
      s_need = (int32_t)nc;
      s_done = 0;
      s_dh = 0;
      s_dl = 0;
    }
    __syncthreads();
    {  // the bytes every leftover shares (arrivals of one window agree in their leading bytes) decide
       // nothing: the select starts at the highest byte where two keys differ
      const QKey k0 = sk[0];
      unsigned long long dh = 0, dl = 0;
      for (int q = tid; q < m; q += nt) {
        dh |= sk[q].hi ^ k0.hi;
        dl |= sk[q].lo ^ k0.lo;
      }
      for (int o = 16; o > 0; o >>= 1) {
        dh |= __shfl_xor_sync(0xffffffffu, dh, o);
        dl |= __shfl_xor_sync(0xffffffffu, dl, o);
      }
      if ((tid & 31) == 0 && (dh | dl)) {
        atomicOr(&s_dh, dh);
        atomicOr(&s_dl, dl);
      }
    }
    __syncthreads();
    const int dtop = s_dh ? 8 + (63 - __clzll((long long)s_dh)) / 8 : (s_dl ? (63 - __clzll((long long)s_dl)) / 8 : 0);
    for (int d = dtop; d >= 0 && !s_done; d--) {
      for (int x = tid; x < 256; x += nt) hist[x] = 0;
      __syncthreads();
      for (int q = tid; q < m; q += nt) {
        if (st[q]) continue;
        const uint64_t w = d >= 8 ? sk[q].hi : sk[q].lo;
        atomicAdd(&hist[(w >> ((d & 7) * 8)) & 0xff], 1);
      }
      __syncthreads();
      if (tid < 32) {  // the digit holding the need-th smallest candidate
        int cnt[8], tot = 0;
        for (int x = 0; x < 8; x++) tot += cnt[x] = hist[tid * 8 + x];
        int incl = tot;
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (tid >= o) incl += y;
        }
        int run = incl - tot;
        const int need = s_need;
        __syncwarp();
        for (int x = 0; x < 8; x++) {
          if (run < need && need <= run + cnt[x]) {
            s_digit = tid * 8 + x;
            s_need = need - run;
            s_done = (need - run) == cnt[x];
          }
          run += cnt[x];
        }
      }
      __syncthreads();
      const int D = s_digit;
      const bool all = s_done;
      for (int q = tid; q < m; q += nt) {
        if (st[q]) continue;
        const uint64_t w = d >= 8 ? sk[q].hi : sk[q].lo;
        const int dig = (int)((w >> ((d & 7) * 8)) & 0xff);
        st[q] = dig < D ? 1 : (dig > D ? 2 : (all ? 1 : 0));
      }
      __syncthreads();
    }
    // compact the taken keys to the front (each thread reads before any write)
    constexpr int PT = QS_MAXP / QS_TPB;  // leftovers per thread
    QKey kk[PT];
    int32_t vv[PT], fl[PT];
    int own = 0;
    for (int q = tid; q < m; q += nt, own++) {
      kk[own] = sk[q];
      vv[own] = sv[q];
      fl[own] = st[q] == 1;
    }
    __syncthreads();
    own = 0;
    for (int q = tid; q < m; q += nt, own++) tmp[q] = fl[own];
    __syncthreads();
    n = block_exscan(tmp, m, swarp);
    own = 0;
    for (int q = tid; q < m; q += nt, own++) {
      if (fl[own]) {
        sk[tmp[q]] = kk[own];
        sv[tmp[q]] = vv[own];
      }
    }
    __syncthreads();
  }
  block_bitonic(sk, sv, n);
  for (int q = tid; q < nc; q += nt) A.cold[q] = sv[q];
  // n_disp of the cold members (247-248): one thread per (member, skeleton entry)
  for (int64_t t = tid; t < nc * QS_MAXK; t += nt) {
    const int64_t i = sv[t / QS_MAXK];
    const int64_t b = A.off[i], e = A.off[i + 1];
    for (int64_t x = b + t % QS_MAXK; x < e; x += QS_MAXK)
      if (A.efirst[x]) atomicAdd(&A.nd[A.sk[x]], 1);
  }
}

// One QAS round.  gridDim.x == 1: the whole round in one CTA (block barriers);
// gridDim.x > 1: a cooperative launch, grid barriers between the phases, the
// short serial phases (bucket order + in-bucket ranks, score sort + hot-lane
// prefix, cold lane) in block 0's shared memory.
__global__ void __launch_bounds__(QS_TPB, 1) k_qas_small(QsArgs A, QsCfg c) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char qs_smem[];
  QKey *sk = reinterpret_cast<QKey *>(qs_smem);
  int32_t *sv = reinterpret_cast<int32_t *>(sk + QS_MAXP);
  int32_t *scnt = sv + QS_MAXP;  // per-bucket counters / scan scratch
  __shared__ int32_t swarp[32];
  const int tid = threadIdx.x;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + tid, gs = (int64_t)gridDim.x * blockDim.x;
  const bool b0 = blockIdx.x == 0;
  const int64_t P = A.P;
  const int64_t nsk = A.off[P];
  // skeleton entries beyond the preallocated buffers: the host redoes the round
  // (uniform over the grid: every thread reads the same values)
  if (nsk > A.aligned_cap || 4 * nsk > A.ptab_cap) {
    if (gt == 0) A.counts[3] = 1;
    return;
  }
  int64_t pm = 64;  // pair table in use
  while (pm < 4 * nsk) pm <<= 1;  // load factor <= 1/4: short linear-probe tails
  const uint64_t pmask = (uint64_t)pm - 1;
  QS_TS(0);
  // 0. reset what the previous round touched; clear the tables
  const int32_t prevn = A.touched_n[1];
  for (int64_t i = gt; i < prevn; i += gs) {
    const int32_t s = A.prev_touched[i];
    A.g[s] = 0;
    A.a[s] = 0;
    A.nd[s] = 0;
    A.prio[s] = 0.0;
    A.dom[s] = 0;
  }
  for (int64_t i = gt; i <= A.btab_mask; i += gs) {
    A.btab_key[i] = QS_EMPTY;
    A.btab_min[i] = 0x7fffffff;
  }
  for (int64_t i = gt; i < pm; i += gs) A.ptab_key[i] = QS_EMPTY;
  for (int64_t i = gt; i < P; i += gs) {  // per-bucket utility sums (bucket ids < P), filled in phases 4 and 7
    A.isum[i] = 0;
    A.nsegs[i] = 0;
  }
  if (gt == 0) A.touched_n[0] = 0;
  {  // entry -> request map + first-occurrence flags of the pending skeletons: one warp per request
    const int64_t nw = gs >> 5;
    for (int64_t w0 = 0; w0 < P; w0 += nw) {
      const int64_t i = w0 + (int64_t)(tid >> 5) * gridDim.x + blockIdx.x;  // warps interleaved over the CTAs
      if (i < P) qs_flags_warp(A, i, A.off[i], A.off[i + 1] - A.off[i]);  // (warp-uniform)
    }
  }
  qs_gsync();
  QS_TS(1);
  // 1. counters g (pending) and a (active), once per distinct segment (83-89),
  // and the touched list (prio's bit pattern doubles as the "listed" flag)
  // pending: one thread per skeleton entry (all probes of a request in flight)
  for (int64_t e0 = 0; e0 < nsk; e0 += gs) {
    const int64_t e = e0 + qs_ilv(gs);
    int32_t s = 0;
    bool nt = false;
    if (e < nsk && A.efirst[e]) {
      s = A.sk[e];
      atomicAdd(&A.g[s], 1);
      unsigned long long *f = (unsigned long long *)&A.prio[s];
      nt = __ldcg(f) == 0ull && atomicCAS(f, 0ull, 0xFFF0000000000001ull) == 0ull;
    }
    const int p = qs_block_reserve(nt ? 1 : 0, &A.touched_n[0]);
    if (nt) A.touched[p] = s;
  }
  {  // active set: one warp per request, first occurrences by __match_any over the lanes (the
     // pending skeletons' qs_flags_warp); the touched list appended once per warp
    const int lane = tid & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t nw = gs >> 5;
    for (int64_t i = (int64_t)(tid >> 5) * gridDim.x + blockIdx.x; i < A.A; i += nw) {  // warps interleaved
      const int64_t b = A.aoff[i], k = A.aoff[i + 1] - b;
      for (int64_t j0 = 0; j0 < k; j0 += 32) {
        const bool on = j0 + lane < k;
        const int32_t sj = on ? A.ask[b + j0 + lane] : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, sj);  // (every lane: no short circuit)
        bool first = on && (peers & lt) == 0u;
        for (int64_t q = 0; q < j0 && first; q++) first = A.ask[b + q] != sj;  // (entries of earlier rounds)
        bool nt = false;
        if (first) {
          atomicAdd(&A.a[sj], 1);
          unsigned long long *f = (unsigned long long *)&A.prio[sj];
          nt = __ldcg(f) == 0ull && atomicCAS(f, 0ull, 0xFFF0000000000001ull) == 0ull;
        }
        const unsigned mt = __ballot_sync(0xffffffffu, nt);
        int base = 0;
        if (lane == 0 && mt) base = atomicAdd(&A.touched_n[0], __popc(mt));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (nt) A.touched[base + __popc(mt & lt)] = sj;
      }
    }
  }
  qs_gsync();
  QS_TS(2);
  // 2. front alignment + order-sensitive signature (109-143), bucket insert:
  // 16 lanes per request, lane q holding skeleton entry q in registers; ranks
  // by shuffles over the group (no per-thread arrays, no local memory)
  {
    const int gl = tid & 15, gb = tid & 16;  // lane in the group, the group's first lane in the warp
    const int64_t ng = gs >> 4;
    for (int64_t g0 = 0; g0 < P; g0 += ng) {
      const int64_t i = g0 + (int64_t)(tid >> 4) * gridDim.x + blockIdx.x;  // groups interleaved over the CTAs
      const bool vi = i < P;
      const int64_t b = vi ? A.off[i] : 0;
      const int k = vi ? (int)(A.off[i + 1] - b) : 0;
      const bool lng = k > QS_MAXK;  // a warp's (below) or a block's (k > QS_MAXW, listed)
      if (vi && k > QS_MAXW && gl == 0) A.longl[atomicAdd((unsigned long long *)&A.counts[4], 1ull)] = (int32_t)i;
      const bool on = vi && !lng && gl < k;
      const int32_t sj = on ? A.sk[b + gl] : 0;
      const double pj = on ? qpri0(c, A.g, A.a, sj) : 0.0;
      const bool reo = vi && A.reo[i];
      // 2a. rank by (-pri, seg, skeleton index); front_align: the top-f to the
      // front in rank order, the rest stable
      int r = 0;
#pragma unroll
      for (int q = 0; q < QS_MAXK; q++) {
        const double pq = __shfl_sync(0xffffffffu, pj, q, 16);
        const int32_t sq = __shfl_sync(0xffffffffu, sj, q, 16);
        r += (q < k && qrank_before(pq, sq, q, pj, sj, gl)) ? 1 : 0;
      }
      const int f = (int)(c.front < k ? c.front : k);
      const bool fronted = reo && r < f;
      const unsigned rest = (__ballot_sync(0xffffffffu, on && !fronted) >> gb) & 0xFFFFu;
      const int pos = !reo ? gl : (fronted ? r : f + __popc(rest & ((1u << gl) - 1u)));
      if (on) A.aligned[b + pos] = sj;
      // 2b. signature: the top-kappa by (-pri, seg, aligned position), emitted in aligned order
      const int kk = (int)(c.kappa < k ? c.kappa : k);
      int r2 = 0;
#pragma unroll
      for (int q = 0; q < QS_MAXK; q++) {
        const double pq = __shfl_sync(0xffffffffu, pj, q, 16);
        const int32_t sq = __shfl_sync(0xffffffffu, sj, q, 16);
        const int posq = __shfl_sync(0xffffffffu, pos, q, 16);
        r2 += (q < k && qrank_before(pq, sq, posq, pj, sj, pos)) ? 1 : 0;
      }
      const bool chosen = on && r2 < kk;
      int before = 0;  // chosen entries ahead of mine in aligned order
#pragma unroll
      for (int q = 0; q < QS_MAXK; q++) {
        const int posq = __shfl_sync(0xffffffffu, pos, q, 16);
        const bool cq = __shfl_sync(0xffffffffu, chosen, q, 16);
        before += (cq && posq < pos) ? 1 : 0;
      }
      if (chosen) A.sig[i * c.kappa + before] = sj;
      __syncwarp();
      if (vi && !lng && gl == 0) {
        const int sl = k > 0 ? kk : 0;
        A.siglen[i] = sl;
        qs_bucket_insert(A, c, i, sl);  // 3.
      }
    }
    // QS_MAXK < k <= QS_MAXW: one warp per request
    const int64_t nw = gs >> 5;
    for (int64_t w0 = 0; w0 < P; w0 += nw) {
      const int64_t i = w0 + (int64_t)(tid >> 5) * gridDim.x + blockIdx.x;
      if (i >= P) continue;  // (warp-uniform)
      const int64_t b = A.off[i];
      const int64_t k = A.off[i + 1] - b;
      if (k > QS_MAXK && k <= QS_MAXW) qs_align_warp(A, c, i, b, (int)k, A.reo[i] != 0);
    }
  }
  qs_gsync();
  const int64_t nlong = (int64_t)__ldcg((const unsigned long long *)&A.counts[4]);
  if (nlong > 0) {  // skeletons longer than QS_MAXK: one block each
    for (int64_t t = blockIdx.x; t < nlong; t += gridDim.x) {
      const int64_t i = A.longl[t];
      const int64_t b = A.off[i];
      const int sl = align_long_block(A.sk + b, (int)(A.off[i + 1] - b), A.reo[i] != 0, A.g, A.a, c.wg, c.wa,
                                      c.front, c.kappa, A.aligned + b, A.sig + i * c.kappa, A.rk + b);
      __threadfence();  // the block's aligned / sig writes, before thread 0 publishes
      __syncthreads();
      if (tid == 0) {
        A.siglen[i] = sl;
        qs_bucket_insert(A, c, i, sl);
      }
      __syncthreads();
    }
    qs_gsync();
  }
  QS_TS(3);
  // 4. bucket creation order = order of first members; in-bucket ranks in
  // pending order (211-223), grid-parallel by counting: every CTA lists each
  // request's first member in shared memory, then one warp per request counts
  // the first members before its bucket's (= its bucket id) and its bucket's
  // members before it (= its rank); a first member also counts its bucket's size
  const int64_t hot_cap = c.budget - c.cold;
  {
    int32_t *sfirst = sv;  // [P <= QS_MAXP]
    // a request's bucket representative = its bucket's first member (final now that every insert is done)
    for (int64_t i = tid; i < P; i += blockDim.x) sfirst[i] = qs_ld(&A.btab_min[qs_ld(&A.slot_of[i])]);
    __syncthreads();
    const int lane = tid & 31;
    const int64_t nw = gs >> 5;
    for (int64_t i = (int64_t)(tid >> 5) * gridDim.x + blockIdx.x; i < P; i += nw) {
      const int32_t f = sfirst[i];
      const bool last = i == P - 1;  // (warp-uniform) also counts every bucket
      int32_t nbef = 0, rk = 0, sz = 0, nall = 0;
      for (int32_t j = lane; j < (int32_t)i; j += 32) {
        const int32_t x = sfirst[j];
        nbef += (j < f && x == j) ? 1 : 0;
        rk += x == f ? 1 : 0;
      }
      if (f == (int32_t)i)
        for (int32_t j = (int32_t)i + lane; j < (int32_t)P; j += 32) sz += sfirst[j] == f ? 1 : 0;
      if (last)
        for (int32_t j = lane; j < (int32_t)P; j += 32) nall += sfirst[j] == j ? 1 : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        nbef += __shfl_xor_sync(0xffffffffu, nbef, o);
        rk += __shfl_xor_sync(0xffffffffu, rk, o);
        sz += __shfl_xor_sync(0xffffffffu, sz, o);
        nall += __shfl_xor_sync(0xffffffffu, nall, o);
      }
      if (lane == 0) {
        A.rank[i] = rk;
        A.bucket[i] = nbef;
        if (f == (int32_t)i) A.bsize[nbef] = sz;
        if (last) A.counts[2] = nall;
      }
    }
  }
  qs_gsync();
  QS_TS(4);
  // 7. distinct (bucket, segment) pairs (146-171) and the buckets' utility
  // sums, one warp per request: the lane that inserts a pair adds its
  // wg g + wa a and one distinct segment; a provisional member (rank < hot_cap)
  // adds wn x its distinct segments -- the sum over the bucket's pairs of
  // wn x count(provisional members holding the segment), regrouped by member
  // (integral weights: exact in int64 in any order).  One atomic pair per
  // request, not per pair (hot buckets collect thousands of pairs).
  {
    const int lane = tid & 31;
    const int64_t nw = gs >> 5;
    for (int64_t i = (int64_t)(tid >> 5) * gridDim.x + blockIdx.x; i < P; i += nw) {  // warps interleaved
      const int32_t bk = A.bucket[i];
      const int64_t b = A.off[i], e = A.off[i + 1];
      unsigned long long su = 0;
      int32_t np = 0, nds = 0;
      for (int64_t x = b + lane; x < e; x += 32) {
        if (!A.efirst[x]) continue;
        const int32_t s = A.sk[x];
        nds++;
        const uint64_t key = ((uint64_t)(uint32_t)bk << 32) | (uint32_t)s;
        uint64_t pos = qmix64(key) & pmask;
        for (;;) {
          unsigned long long *slot = (unsigned long long *)&A.ptab_key[pos];
          unsigned long long prev = __ldcg(slot);
          if (prev == QS_EMPTY) {
            prev = atomicCAS(slot, QS_EMPTY, key);
            if (prev == QS_EMPTY) {
              np++;
              su += (unsigned long long)(long long)__dadd_rn(__dmul_rn(c.wg, (double)A.g[s]),
                                                             __dmul_rn(c.wa, (double)A.a[s]));
            }
          }
          if (prev == QS_EMPTY || prev == key) break;
          pos = (pos + 1) & pmask;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        su += __shfl_xor_sync(0xffffffffu, su, o);
        np += __shfl_xor_sync(0xffffffffu, np, o);
        nds += __shfl_xor_sync(0xffffffffu, nds, o);
      }
      if (lane == 0) {
        if (A.rank[i] < hot_cap) su += (unsigned long long)(long long)__dmul_rn(c.wn, (double)nds);
        if (su) atomicAdd((unsigned long long *)&A.isum[bk], su);
        if (np) atomicAdd(&A.nsegs[bk], np);
      }
    }
  }
  qs_gsync();
  QS_TS(5);
  // 8. (folded into 4 and 7: the utility sums are complete here)
  QS_TS(6);
  // 9. scores (146-171), the (-score, creation order) order (234) and the
  // hot-lane fill (235-240) without a sort: every CTA lists all nb bucket keys
  // in shared memory, then one warp per bucket counts the keys before its own
  // -- its position -- and sums their sizes: the hot-lane base
  const int32_t nb = (int32_t)__ldcg((const unsigned long long *)&A.counts[2]);
  {
    int32_t *ssz = sv;
    for (int b = tid; b < nb; b += blockDim.x) {
      const int32_t ns = qs_ld(&A.nsegs[b]);
      const long long is = (long long)__ldcg((const unsigned long long *)&A.isum[b]);
      const double util = ns > 0 ? __ddiv_rn((double)is, (double)ns) : 0.0;
      const int32_t bs = qs_ld(&A.bsize[b]);
      const double sc = __dadd_rn(__dmul_rn(c.alpha, (double)bs), __dmul_rn(c.beta, util));
      if (b0) A.score[b] = sc;
      sk[b] = {qord(-sc), (uint64_t)b};
      ssz[b] = bs;
    }
    __syncthreads();
    const int lane = tid & 31;
    const int64_t nw = gs >> 5;
    for (int64_t b = (int64_t)(tid >> 5) * gridDim.x + blockIdx.x; b < nb; b += nw) {
      const QKey kb = sk[b];
      int32_t before = 0;
      for (int j = lane; j < nb; j += 32) before += qk_less(sk[j], kb) ? ssz[j] : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
      if (lane == 0) {
        int64_t take = hot_cap - before;
        take = take < 0 ? 0 : (take > ssz[b] ? ssz[b] : take);
        A.btake[b] = (int32_t)take;
        A.bbase[b] = before < hot_cap ? before : (int32_t)hot_cap;
      }
    }
  }
  qs_gsync();
  QS_TS(7);
  // 10. hot lane, and n_disp of its members (247-248): one warp per request
  // (its bucket's take read once, its skeleton entries over the lanes) -- on
  // every CTA but 0, which meanwhile runs the cold lane (11: the oldest
  // cold_quota leftovers by (arrival, id), listed by itself)
  const int64_t nh = hot_cap < P ? (hot_cap > 0 ? hot_cap : 0) : P;
  const int64_t nc = c.cold < P - nh ? c.cold : P - nh;
  const bool split = gridDim.x > 1;
  if (!split || !b0) {
    const int lane = tid & 31;
    const int64_t nbk = split ? gridDim.x - 1 : 1, bi = split ? blockIdx.x - 1 : 0;
    const int64_t nw = nbk * (blockDim.x >> 5);
    for (int64_t i = (int64_t)(tid >> 5) * nbk + bi; i < P; i += nw) {  // warps interleaved over the CTAs
      const int32_t b = A.bucket[i], r = A.rank[i];
      const bool h = r < qs_ld(&A.btake[b]);
      if (lane == 0) {
        A.bidx[i] = h ? 1 : 0;  // reuse: hot flag
        if (h) A.hot[(int64_t)qs_ld(&A.bbase[b]) + r] = (int32_t)i;
      }
      if (h)
        for (int64_t x = A.off[i] + lane; x < A.off[i + 1]; x += 32)
          if (A.efirst[x]) atomicAdd(&A.nd[A.sk[x]], 1);
    }
  }
  QS_TS(8);
  if (b0 && nc > 0) {
    if (!split) __syncthreads();
    qs_cold_lane(A, c, P, nc, sk, sv, scnt, swarp);
  }
  qs_gsync();
  QS_TS(9);
  // 12. priorities over the domain (249-251)
  const int32_t ntouch = qs_ld(&A.touched_n[0]);
  for (int64_t i0 = 0; i0 < ntouch; i0 += gs) {
    const int64_t i = i0 + qs_ilv(gs);
    if (i >= ntouch) continue;
    const int32_t s = A.touched[i];
    const int32_t g = A.g[s], a = A.a[s], n = qs_ld(&A.nd[s]);
    const bool in = g > 0 || a > 0 || n > 0;
    A.dom[s] = in ? 1 : 0;
    A.prio[s] = in ? __dadd_rn(__dadd_rn(__dmul_rn(c.wg, (double)g), __dmul_rn(c.wa, (double)a)),
                               __dmul_rn(c.wn, (double)n))
                   : 0.0;
  }
  if (gt == 0) {
    A.counts[0] = nh;
    A.counts[1] = nc;
    A.touched_n[1] = ntouch;  // this round's list is the next round's reset list
  }
  QS_TS(10);
  pdl_trace_end();
}

}  // namespace qsmall

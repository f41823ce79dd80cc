// qas_small.cuh -- one QAS round (scheduler.py:192-273) in ONE CTA.
//
// For pending sets of up to QS_MAXP requests the whole round runs inside a
// single 1024-thread CTA: no kernel launches between its phases, no host
// round trips, shared-memory bitonic sorts for the bucket order and the cold
// lane, a sequential warp pass for the in-bucket ranks (first-seen order),
// and a hash aggregation of distinct (bucket, segment) pairs for the bucket
// utilities.  Segment counters are reset through the list of segments the
// previous round touched, so the cost is O(P*k), not O(num_segments).
//
// Exactness: identical float expressions to qas.cu / the reference; the
// utility sum uses int64 accumulation and is therefore only used when every
// term is an exact integer (integral weights: the reference defaults) -- the
// host selects this kernel only then.
#pragma once
#include <cstdint>

namespace qsmall {

constexpr int QS_TPB = 1024;
constexpr int QS_MAXP = 4096;  // bitonic sort capacity (shared memory)
constexpr int QS_MAXK = 64;
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
  int64_t *counts;  // [0] nhot, [1] ncold, [2] nbuckets, [3] redo on the multi-kernel path
  // scratch (global)
  uint64_t *btab_key;  // signature table, size 2*QS_MAXP (power of two)
  int32_t *btab_min, *slot_of, *bidx;
  int32_t *bsize, *nsegs;
  long long *isum;
  uint64_t *ptab_key;  // (bucket, seg) pair table
  int32_t *ptab_cnt;
  int64_t ptab_mask, btab_mask;
  int32_t *longl;       // requests with skeletons longer than QS_MAXK
  int32_t *rk;          // rank scratch for them (aligned_cap ints)
  int64_t aligned_cap;  // capacity of aligned / rk in skeleton entries
};

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
__device__ inline bool qk_less(const QKey &x, const QKey &y) { return x.hi != y.hi ? x.hi < y.hi : x.lo < y.lo; }

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

constexpr size_t QS_SMEM = (sizeof(QKey) + sizeof(int32_t)) * QS_MAXP + sizeof(int32_t) * QS_MAXP;

// 3. bucket of request i's signature tuple; first member via atomicMin
// (scheduler.py:211-223).  Open addressing on (hash, first index seen).
__device__ inline void qs_bucket_insert(const QsArgs &A, const QsCfg &c, int64_t i, int sl) {
  uint32_t h = 2166136261u ^ (uint32_t)sl;
  for (int j = 0; j < sl; j++) h = (h ^ (uint32_t)A.sig[i * c.kappa + j]) * 16777619u;
  const uint64_t mine = ((uint64_t)h << 32) | (uint32_t)i;
  uint64_t pos = qmix64(h) & (uint64_t)A.btab_mask;
  for (;;) {
    const unsigned long long prev = atomicCAS((unsigned long long *)&A.btab_key[pos], QS_EMPTY, mine);
    bool same = prev == QS_EMPTY;
    if (!same && (uint32_t)(prev >> 32) == h) {
      const int64_t o = (int64_t)(prev & 0xffffffffu);
      same = A.siglen[o] == sl;
      for (int j = 0; same && j < sl; j++) same = A.sig[o * c.kappa + j] == A.sig[i * c.kappa + j];
    }
    if (same) {
      atomicMin(&A.btab_min[pos], (int32_t)i);
      A.slot_of[i] = (int32_t)pos;
      return;
    }
    pos = (pos + 1) & (uint64_t)A.btab_mask;
  }
}

__global__ void __launch_bounds__(QS_TPB, 1) k_qas_small(QsArgs A, QsCfg c) {
  extern __shared__ __align__(16) unsigned char qs_smem[];
  QKey *sk = reinterpret_cast<QKey *>(qs_smem);
  int32_t *sv = reinterpret_cast<int32_t *>(sk + QS_MAXP);
  int32_t *scnt = sv + QS_MAXP;  // per-bucket counters (ranks)
  __shared__ int32_t swarp[32];
  __shared__ int32_t s_nb, s_nlong;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t P = A.P;
  // skeleton entries beyond the preallocated buffers (aligned / rank scratch,
  // or more pairs than half the pair table): the host redoes the round
  if (A.off[P] > A.aligned_cap || 2 * A.off[P] > A.ptab_mask + 1) {
    if (tid == 0) A.counts[3] = 1;
    return;
  }
  if (tid == 0) s_nlong = 0;
  // 0. reset what the previous round touched; clear the tables
  const int32_t prevn = A.touched_n[1];
  for (int i = tid; i < prevn; i += nt) {
    const int32_t s = A.prev_touched[i];
    A.g[s] = 0;
    A.a[s] = 0;
    A.nd[s] = 0;
    A.prio[s] = 0.0;
    A.dom[s] = 0;
  }
  for (int64_t i = tid; i <= A.btab_mask; i += nt) {
    A.btab_key[i] = QS_EMPTY;
    A.btab_min[i] = 0x7fffffff;
  }
  for (int64_t i = tid; i <= A.ptab_mask; i += nt) {
    A.ptab_key[i] = QS_EMPTY;
    A.ptab_cnt[i] = 0;
  }
  if (tid == 0) A.touched_n[0] = 0;
  __syncthreads();
  // 1. counters g (pending) and a (active), once per distinct segment (83-89)
  for (int pass = 0; pass < 2; pass++) {
    const int64_t n = pass == 0 ? P : A.A;
    const int64_t *off = pass == 0 ? A.off : A.aoff;
    const int32_t *sk_ = pass == 0 ? A.sk : A.ask;
    int32_t *cnt = pass == 0 ? A.g : A.a;
    for (int64_t i = tid; i < n; i += nt) {
      const int64_t b = off[i], e = off[i + 1];
      for (int64_t j = b; j < e; j++) {
        const int32_t s = sk_[j];
        bool dup = false;
        for (int64_t q = b; q < j && !dup; q++) dup = sk_[q] == s;
        if (!dup) atomicAdd(&cnt[s], 1);
      }
    }
    __syncthreads();
  }
  // touched list: every segment appearing in pending or active skeletons
  // (marked through prio = -1 as a temporary flag, then compacted)
  for (int pass = 0; pass < 2; pass++) {
    const int64_t n = pass == 0 ? P : A.A;
    const int64_t *off = pass == 0 ? A.off : A.aoff;
    const int32_t *sk_ = pass == 0 ? A.sk : A.ask;
    for (int64_t i = tid; i < n; i += nt) {
      for (int64_t j = off[i]; j < off[i + 1]; j++) {
        const int32_t s = sk_[j];
        if (atomicCAS((unsigned long long *)&A.prio[s], 0ull, 0xFFF0000000000001ull) == 0ull) {
          const int32_t p = atomicAdd(&A.touched_n[0], 1);
          A.touched[p] = s;
        }
      }
    }
  }
  __syncthreads();
  // 2. front alignment + order-sensitive signature (109-143)
  for (int64_t i = tid; i < P; i += nt) {
    const int64_t b = A.off[i];
    const int k = (int)(A.off[i + 1] - b);
    if (k > QS_MAXK) {  // aligned below by the whole block
      A.longl[atomicAdd(&s_nlong, 1)] = (int32_t)i;
      continue;
    }
    int32_t s[QS_MAXK], al[QS_MAXK];
    double p[QS_MAXK];
    int ord[QS_MAXK];
    for (int j = 0; j < k; j++) {
      s[j] = A.sk[b + j];
      p[j] = qpri0(c, A.g, A.a, s[j]);
    }
    if (!A.reo[i] || k == 0) {
      for (int j = 0; j < k; j++) al[j] = s[j];
    } else {
      for (int j = 0; j < k; j++) {
        int q = j;
        while (q > 0 && qrank_before(p[j], s[j], j, p[ord[q - 1]], s[ord[q - 1]], ord[q - 1])) {
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
    for (int j = 0; j < k; j++) A.aligned[b + j] = al[j];
    int sl = 0;
    if (k > 0) {
      double pa[QS_MAXK];
      for (int j = 0; j < k; j++) {
        pa[j] = qpri0(c, A.g, A.a, al[j]);
        int q = j;
        while (q > 0 && qrank_before(pa[j], al[j], j, pa[ord[q - 1]], al[ord[q - 1]], ord[q - 1])) {
          ord[q] = ord[q - 1];
          q--;
        }
        ord[q] = j;
      }
      const int kk = (int)(c.kappa < k ? c.kappa : k);
      uint64_t chosen = 0;
      for (int q = 0; q < kk; q++) chosen |= 1ull << ord[q];
      for (int j = 0; j < k; j++)
        if ((chosen >> j) & 1ull) A.sig[i * c.kappa + sl++] = al[j];
    }
    A.siglen[i] = sl;
    qs_bucket_insert(A, c, i, sl);  // 3.
  }
  __syncthreads();
  for (int t = 0; t < s_nlong; t++) {  // skeletons longer than QS_MAXK
    const int64_t i = A.longl[t];
    const int64_t b = A.off[i];
    const int sl = align_long_block(A.sk + b, (int)(A.off[i + 1] - b), A.reo[i] != 0, A.g, A.a, c.wg, c.wa,
                                    c.front, c.kappa, A.aligned + b, A.sig + i * c.kappa, A.rk);
    if (tid == 0) {
      A.siglen[i] = sl;
      qs_bucket_insert(A, c, i, sl);
    }
  }
  __syncthreads();
  // 4. bucket creation order = order of first members: scan of "is first" flags
  for (int64_t i = tid; i < P; i += nt) A.bidx[i] = A.btab_min[A.slot_of[i]] == (int32_t)i ? 1 : 0;
  __syncthreads();
  const int32_t nb = block_exscan(A.bidx, (int)P, swarp);
  if (tid == 0) s_nb = nb;
  for (int64_t i = tid; i < P; i += nt) {
    const int32_t first = A.btab_min[A.slot_of[i]];
    A.bucket[i] = first;  // temporarily: first member index
  }
  __syncthreads();
  for (int64_t i = tid; i < P; i += nt) A.bucket[i] = A.bidx[A.bucket[i]];
  for (int b = tid; b < nb; b += nt) scnt[b] = 0;
  __syncthreads();
  // 5. rank inside the bucket, in pending order: warp 0 walks P in order
  if (tid < 32) {
    const int lane = tid;
    for (int64_t base = 0; base < P; base += 32) {
      const int64_t i = base + lane;
      const int32_t b = i < P ? A.bucket[i] : -1 - lane;
      const unsigned peers = __match_any_sync(0xffffffffu, b);
      const int32_t before = __popc(peers & ((1u << lane) - 1u));
      int32_t r = 0;
      if (i < P) r = scnt[b] + before;
      __syncwarp();
      if (i < P) {
        A.rank[i] = r;
        if (lane == 31 - __clz(peers)) scnt[b] = r + 1;  // highest lane of the group
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int b = tid; b < nb; b += nt) {
    A.bsize[b] = scnt[b];
    A.nsegs[b] = 0;
    A.isum[b] = 0;
  }
  __syncthreads();
  // 7. distinct (bucket, segment) pairs; provisional = first hot_cap members (146-171)
  const int64_t hot_cap = c.budget - c.cold;
  for (int64_t i = tid; i < P; i += nt) {
    const int64_t b0 = A.off[i], e0 = A.off[i + 1];
    const int32_t bk = A.bucket[i];
    const int prov = A.rank[i] < hot_cap ? 1 : 0;
    for (int64_t j = b0; j < e0; j++) {
      const int32_t s = A.sk[j];
      bool dup = false;
      for (int64_t q = b0; q < j && !dup; q++) dup = A.sk[q] == s;
      if (dup) continue;
      const uint64_t key = ((uint64_t)(uint32_t)bk << 32) | (uint32_t)s;
      uint64_t pos = qmix64(key) & (uint64_t)A.ptab_mask;
      for (;;) {
        const unsigned long long prev = atomicCAS((unsigned long long *)&A.ptab_key[pos], QS_EMPTY, key);
        if (prev == QS_EMPTY) atomicAdd(&A.nsegs[bk], 1);
        if (prev == QS_EMPTY || prev == key) {
          if (prov) atomicAdd(&A.ptab_cnt[pos], 1);
          break;
        }
        pos = (pos + 1) & (uint64_t)A.ptab_mask;
      }
    }
  }
  __syncthreads();
  // 8. utility terms, summed exactly (integral by construction)
  for (int64_t p = tid; p <= A.ptab_mask; p += nt) {
    const uint64_t key = A.ptab_key[p];
    if (key == QS_EMPTY) continue;
    const int32_t bk = (int32_t)(key >> 32), s = (int32_t)(key & 0xffffffffu);
    const double t1 = __dmul_rn(c.wg, (double)A.g[s]);
    const double t2 = __dmul_rn(c.wa, (double)A.a[s]);
    const double t3 = __dmul_rn(c.wn, (double)A.ptab_cnt[p]);
    atomicAdd((unsigned long long *)&A.isum[bk], (unsigned long long)(long long)__dadd_rn(__dadd_rn(t1, t2), t3));
  }
  __syncthreads();
  // 9. scores, and the (-score, creation order) sort keys
  for (int b = tid; b < nb; b += nt) {
    const int32_t ns = A.nsegs[b];
    const double util = ns > 0 ? __ddiv_rn((double)A.isum[b], (double)ns) : 0.0;
    const double sc = __dadd_rn(__dmul_rn(c.alpha, (double)A.bsize[b]), __dmul_rn(c.beta, util));
    A.score[b] = sc;
    sk[b] = {qord(-sc), (uint64_t)b};
    sv[b] = b;
  }
  __syncthreads();
  block_bitonic(sk, sv, nb);  // 234
  // 10. hot lane by prefix sums of bucket sizes in sorted order (235-240)
  for (int q = tid; q < nb; q += nt) scnt[q] = A.bsize[sv[q]];
  __syncthreads();
  block_exscan(scnt, nb, swarp);
  for (int q = tid; q < nb; q += nt) {
    const int32_t b = sv[q];
    int64_t take = hot_cap - scnt[q];
    take = take < 0 ? 0 : (take > A.bsize[b] ? A.bsize[b] : take);
    A.nsegs[b] = (int32_t)take;                                        // reuse: take
    A.isum[b] = scnt[q] < hot_cap ? scnt[q] : hot_cap;                 // reuse: base
  }
  __syncthreads();
  for (int64_t i = tid; i < P; i += nt) {
    const int32_t b = A.bucket[i];
    const bool h = A.rank[i] < A.nsegs[b];
    A.bidx[i] = h ? 1 : 0;  // reuse: selected flag
    if (h) A.hot[A.isum[b] + A.rank[i]] = i;
  }
  __syncthreads();
  // 11. cold lane: leftovers by (arrival, id), the oldest cold_quota (242-245)
  const int64_t nh = hot_cap < P ? (hot_cap > 0 ? hot_cap : 0) : P;
  const int64_t nc = c.cold < P - nh ? c.cold : P - nh;
  if (nc > 0) {
    for (int64_t i = tid; i < P; i += nt) {
      const uint64_t sel = A.bidx[i] ? 1ull : 0ull;
      // (selected, arrival) in hi (arrival order-preserving map, top bit for selected)
      const uint64_t ar = qord(A.arrival[i]);
      sk[i] = {sel ? ~0ull : ar, (uint64_t)A.ids[i] ^ 0x8000000000000000ull};
      sv[i] = (int32_t)i;
    }
    __syncthreads();
    block_bitonic(sk, sv, (int)P);
    for (int64_t q = tid; q < nc; q += nt) A.cold[q] = sv[q];
    __syncthreads();
  }
  // 12. dispatch counters n over hot + cold, priorities over the domain (247-251)
  for (int64_t q = tid; q < nh + nc; q += nt) {
    const int64_t i = q < nh ? A.hot[q] : A.cold[q - nh];
    const int64_t b0 = A.off[i], e0 = A.off[i + 1];
    for (int64_t j = b0; j < e0; j++) {
      const int32_t s = A.sk[j];
      bool dup = false;
      for (int64_t r = b0; r < j && !dup; r++) dup = A.sk[r] == s;
      if (!dup) atomicAdd(&A.nd[s], 1);
    }
  }
  __syncthreads();
  const int32_t nt_ = A.touched_n[0];
  for (int i = tid; i < nt_; i += nt) {
    const int32_t s = A.touched[i];
    const bool in = A.g[s] > 0 || A.a[s] > 0 || A.nd[s] > 0;
    A.dom[s] = in ? 1 : 0;
    A.prio[s] = in ? __dadd_rn(qpri0(c, A.g, A.a, s), __dmul_rn(c.wn, (double)A.nd[s])) : 0.0;
  }
  if (tid == 0) {
    A.counts[0] = nh;
    A.counts[1] = nc;
    A.counts[2] = s_nb;
    A.touched_n[1] = nt_;  // this round's list is the next round's reset list
  }
}

}  // namespace qsmall

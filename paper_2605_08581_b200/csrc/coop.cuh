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
constexpr size_t COOP_SMEM = (sizeof(Key3) + sizeof(uint64_t)) * CHUNK;

struct CoopState {
  unsigned long long cand;  // gathered candidates
  unsigned long long nsel;  // selected so far
  unsigned long long nun[COOP_ROUNDS + 2];
  unsigned long long hist_n[COOP_ROUNDS + 2][256];
  unsigned long long hist_w[COOP_ROUNDS + 2][256];
  long long prot_n;  // protection: number protected
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

__device__ inline void block_minmax(Key3 lo, Key3 hi, Key3 *smin, Key3 *smax, Key3 *gmin, Key3 *gmax) {
  smin[threadIdx.x] = lo;
  smax[threadIdx.x] = hi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      if (key_less(smin[threadIdx.x + s], smin[threadIdx.x])) smin[threadIdx.x] = smin[threadIdx.x + s];
      if (key_less(smax[threadIdx.x], smax[threadIdx.x + s])) smax[threadIdx.x] = smax[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *gmin = smin[0];
    *gmax = smax[0];
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

// the eviction-order build after keys / subtree maxima / gather (full-
// occupancy kernels k_build_keys, k_propagate, k_gather, which leave the
// candidate count in st->cand): selection of the consumable prefix + its sort
// + list ready -- one cooperative launch, no host round trip.
__global__ void __launch_bounds__(COOP_TPB) k_build_coop(DT T, CoopBufs B, int64_t W, int64_t min_cand,
                                                         int64_t small) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ Key3 smin[COOP_TPB + 1], smax[COOP_TPB + 1];
  cg::grid_group grid = cg::this_grid();
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gsz = (int64_t)gridDim.x * blockDim.x;
  const int64_t n = (int64_t)B.st->cand;
  coop_mark(B.st);
  int64_t nsel = n;
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
    B.st->ts_build[39] = (unsigned long long)nsel;  // selected-prefix size, for diagnostics
  }
}

// set_protection (kvcache.py:364-383): top-f reusable anchors by (-P-hat, seg or -1, id)
__global__ void __launch_bounds__(COOP_TPB) k_protect_coop(DT T, CoopBufs B, int64_t f, int64_t min_cand,
                                                           int64_t small) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ Key3 smin[COOP_TPB + 1], smax[COOP_TPB + 1];
  cg::grid_group grid = cg::this_grid();
  const int32_t hw = T.ctrl->hw;
  const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < hw; base += gsz) {
    const int64_t s = base + threadIdx.x;
    bool take = false;
    if (s < hw) {
      T.prot[s] = 0;  // previous protection is cleared
      take = s != ROOT && T.nid[s] >= 0 && T.par[s] >= 0 && T.hasanc[s] && T.akind[s] == K_REUSABLE;
    }
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (!m) continue;
    unsigned long long b = 0;
    if (lane == 0) b = atomicAdd(&B.st->cand, (unsigned long long)__popc(m));
    b = __shfl_sync(0xffffffffu, b, 0);
    if (take) {
      const int64_t pos = (int64_t)b + __popc(m & ((1u << lane) - 1));
      const int32_t sg = T.seg[s];
      const int32_t sv = sg == SEG_NONE ? -1 : sg;
      Key3 k = {0, 0, 0};
      shl_or(k, 64, ord_f64(-pri_of(T, sg)));
      shl_or(k, 32, (uint64_t)((uint32_t)sv ^ 0x80000000u));
      shl_or(k, 40, (uint64_t)T.nid[s] & ((1ull << 40) - 1));
      B.k0[pos] = k;
      B.v0[pos] = (uint64_t)(uint32_t)s;
      B.w0[pos] = 1;
    }
  }
  grid.sync();
  const int64_t n = (int64_t)B.st->cand;
  const int64_t nf = f < n ? f : n;
  if (nf <= 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) B.st->prot_n = 0;
    return;
  }
  int64_t nsel = n;
  if (n > min_cand) {
    nsel = coop_select(grid, B, n, nf, small, smin, smax);
  } else {
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t i = gtid; i < n; i += gsz) {
      B.ks[i] = B.k0[i];
      B.vs[i] = B.v0[i];
    }
    grid.sync();
  }
  coop_sort(grid, B, nsel, T.Lk, T.Lv, dsm);  // Lk/Lv as scratch: no list survives a call
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = gtid; i < nf; i += gsz) {
    const int32_t s = (int32_t)(T.Lv[i] & 0xffffffffu);
    T.prot[s] = 1;
    if (B.out_ids) B.out_ids[i] = T.nid[s];
  }
  if (gtid == 0) B.st->prot_n = nf;
}

}  // namespace prism

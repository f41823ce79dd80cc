// kv.cuh -- the paged KV payload behind DART (north_star item 4).
//
// The reference is token-granular and carries no payload: a
// node's edge is a token span.  A serving engine attaches KV storage to those
// tokens; here every resident token owns one row of a KV pool in HBM
// (bytes_per_token bytes), allocated from a free stack when the token becomes
// resident and returned when its node is evicted.
//
// Mapping: the tree stores every edge as a span of its bump-allocated token
// arena (a split only moves an offset, compaction moves spans), so the pool
// row of a resident token is kept in a SHADOW array kvx[arena offset] that
// travels with the arena.  After any batch of tree operations (a fused wave,
// a per-call insert / evict) kv_sync settles the payload:
//   * the arena grown since the last sync = the newly resident tokens, in
//     admission order (each admitted member's uncached tokens, engine.py:203-
//     213) -> pop pool rows, optionally copy the new KV in (the prefill's
//     output, laid out in that order), coalesced 16-B vectors;
//   * the victim log since the last sync (eviction order, kvcache.py:425-460)
//     -> optionally copy the victims' KV out (offload, contiguous in eviction
//     order) and push their rows back (the page-pool free-list update).
// kv_gather builds, per admitted leaf, the request's row table (req_to_token:
// pool row of every path position, what an attention kernel reads) by walking
// the leaf's root chain, and optionally gathers the KV rows themselves.
#pragma once
#include <cstdint>

#include "prism_dev.cuh"

namespace prism {

struct KvDev {
  uint8_t *pool;       // [pool_rows, bpt]
  int32_t *kvx;        // [acap] pool row of arena token i (valid for live spans)
  int32_t *stack;      // free rows, [0, top)
  int64_t *top;        // device scalar: free rows
  int64_t *moved;      // [0] rows allocated, [1] rows freed, [2] bytes copied in, [3] bytes copied out
  int64_t *ctl;        // [0] arena mark, [1] victim-log mark, [2] new tokens, [3] victim records,
                       // [4] freed tokens, [5] error (pool exhausted / victims lost), [6] last new, [7] last freed
  int64_t bpt;         // bytes per token (multiple of 16)
  int64_t rows;
};

// one sync's sizes from the tree's control block (no host round trip): new
// arena tokens since the arena mark, victim records since the log mark
__global__ void k_kv_prep(KvDev K, const Ctrl *C, int64_t vcap) {
  pdl_wait();
  const int64_t n_new = C->arena_top - K.ctl[0], nrec = C->vlog_count - K.ctl[1];
  const bool bad = n_new < 0 || n_new > *K.top || nrec > vcap;
  K.ctl[2] = bad ? 0 : n_new;
  K.ctl[3] = bad ? 0 : nrec;
  K.ctl[4] = 0;
  if (bad) K.ctl[5] = n_new > *K.top ? 1 : 2;
}

// the marks advance, the free-row count and the traffic counters update
__global__ void k_kv_fin(KvDev K, const Ctrl *C, int32_t copy_in, int32_t copy_out) {
  pdl_wait();
  const int64_t n_new = K.ctl[2], freed = K.ctl[4];
  *K.top += freed - n_new;
  K.moved[0] += n_new;
  K.moved[1] += freed;
  if (copy_in) K.moved[2] += n_new * K.bpt;
  if (copy_out) K.moved[3] += freed * K.bpt;
  K.ctl[6] = n_new;
  K.ctl[7] = freed;
  if (!K.ctl[5]) {
    K.ctl[0] = C->arena_top;
    K.ctl[1] = C->vlog_count;
  }
}

// flat 16-B vector index x = row * vpr + v stepped by a fixed stride without a
// division per vector (the copies are instruction-bound with one)
struct VecIt {
  int64_t i, di;
  int32_t v, dv, vpr;
  __device__ __forceinline__ VecIt(int64_t x, int64_t step, int32_t vpr_)
      : i(x / vpr_), di(step / vpr_), v((int32_t)(x % vpr_)), dv((int32_t)(step % vpr_)), vpr(vpr_) {}
  __device__ __forceinline__ void next() {
    i += di;
    v += dv;
    if (v >= vpr) {
      v -= vpr;
      i++;
    }
  }
};

// newly resident arena tokens [a0, a0 + n): pop rows (stack top - 1 - i) in
// arena order, optionally copy the payload in (src row i = arena token a0 + i)
__global__ void k_kv_alloc(KvDev K, const uint8_t *__restrict__ src) {
  pdl_wait();
  const int64_t top = *K.top, a0 = K.ctl[0], n = K.ctl[2];  // (k_kv_fin moves top after every reader)
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = t0; i < n; i += gs) K.kvx[a0 + i] = K.stack[top - 1 - i];
  if (!src) return;
  // copy-in: 16-B vectors across all the new rows (src row i -> pool row of token a0 + i),
  // UNR independent vectors in flight per thread
  constexpr int UNR = 4;
  const int32_t vpr = (int32_t)(K.bpt / 16);
  const int64_t nv = n * vpr;
  const int4 *s4 = reinterpret_cast<const int4 *>(src);
  const int32_t *stk = K.stack + top - 1;
  VecIt it(t0, gs, vpr);
  for (int64_t x0 = t0; x0 < nv; x0 += UNR * gs) {
    int4 val[UNR];
    int32_t row[UNR], vv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; u++) {
      if (x0 + u * gs < nv) {
        val[u] = __ldcs(s4 + x0 + u * gs);  // (streamed once)
        row[u] = stk[-it.i];
        vv[u] = it.v;
      }
      it.next();
    }
#pragma unroll
    for (int u = 0; u < UNR; u++)
      if (x0 + u * gs < nv) reinterpret_cast<int4 *>(K.pool + (int64_t)row[u] * K.bpt)[vv[u]] = val[u];
  }
}


// victim records [v0, v1) of the log ring: their pool rows, in eviction order,
// pushed on the stack (record r's rows at top + voff[r] ..), optionally copied
// out (dst row = voff[r] + i).  voff: exclusive prefix of the records' lengths.
__global__ void k_kv_free(KvDev K, const VRec *__restrict__ vlog, int64_t vcap, const int64_t *__restrict__ voff,
                          uint8_t *__restrict__ dst) {
  pdl_wait();
  const int64_t top = *K.top - K.ctl[2];  // (the rows k_kv_alloc popped are gone; k_kv_fin moves top)
  const int64_t v0 = K.ctl[1], nrec = K.ctl[3];
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t r = w; r < nrec; r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const VRec rec = vlog[(v0 + r) % vcap];
    const int64_t o = voff[r];
    for (int32_t i = lane; i < rec.elen; i += 32) K.stack[top + o + i] = K.kvx[rec.eoff + i];
    if (dst) {  // the record's rows back to back, 16-B vectors across the whole record, 4 in flight per lane
      const int32_t vpr = (int32_t)(K.bpt / 16);
      const int64_t nv = (int64_t)rec.elen * vpr;
      const int32_t *kx = K.kvx + rec.eoff;
      int4 *d = reinterpret_cast<int4 *>(dst + o * K.bpt);
      VecIt it(lane, 32, vpr);
      for (int64_t x0 = lane; x0 < nv; x0 += 4 * 32) {
        int4 val[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          if (x0 + u * 32 < nv)
            val[u] = reinterpret_cast<const int4 *>(K.pool + (int64_t)kx[it.i] * K.bpt)[it.v];
          it.next();
        }
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (x0 + u * 32 < nv) __stcs(d + x0 + u * 32, val[u]);  // (the offload buffer: streamed)
      }
    }
  }
}

// exclusive prefix of the victim records' lengths + the total, two passes over
// G contiguous chunks of records (G <= 1024 CTAs; a one-CTA scan of a C3 wave's
// ~10^5 records took 220 us): k_kv_vsum writes each chunk's sum, k_kv_vfill
// reduces the sums before its chunk and scans the chunk with a carry
__device__ __forceinline__ void kv_chunk(int64_t nrec, int64_t &r0, int64_t &r1) {
  const int64_t ch = (nrec + gridDim.x - 1) / gridDim.x;
  r0 = min(nrec, (int64_t)blockIdx.x * ch);
  r1 = min(nrec, r0 + ch);
}

__device__ __forceinline__ int64_t kv_block_sum(int64_t x, int64_t *s_w) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  __syncthreads();
  if (lane == 0) s_w[wid] = x;
  __syncthreads();
  int64_t t = 0;
  for (int w = 0; w < nw; w++) t += s_w[w];
  return t;
}

__global__ void __launch_bounds__(1024) k_kv_vsum(const VRec *__restrict__ vlog, int64_t vcap, int64_t *part, KvDev K) {
  pdl_wait();
  __shared__ int64_t s_w[32];
  const int64_t v0 = K.ctl[1];
  int64_t r0, r1, x = 0;
  kv_chunk(K.ctl[3], r0, r1);
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) x += vlog[(v0 + r) % vcap].elen;
  const int64_t t = kv_block_sum(x, s_w);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void __launch_bounds__(1024) k_kv_vfill(const VRec *__restrict__ vlog, int64_t vcap, int64_t *voff,
                                                   const int64_t *__restrict__ part, KvDev K) {
  pdl_wait();
  __shared__ int64_t s_w[32];
  __shared__ int64_t s_carry;
  const int64_t v0 = K.ctl[1], nrec = K.ctl[3];
  int64_t r0, r1;
  kv_chunk(nrec, r0, r1);
  const int64_t base = kv_block_sum(threadIdx.x < blockIdx.x ? part[threadIdx.x] : 0, s_w);
  if (threadIdx.x == 0) s_carry = base;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t b = r0; b < r1; b += blockDim.x) {
    const int64_t r = b + threadIdx.x;
    const int64_t x = r < r1 ? vlog[(v0 + r) % vcap].elen : 0;
    int64_t inc = x;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      int64_t t = lane < nw ? s_w[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      s_w[lane] = t;
    }
    __syncthreads();
    if (r < r1) voff[r] = s_carry + (wid ? s_w[wid - 1] : 0) + inc - x;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += s_w[nw - 1];
    __syncthreads();
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    K.ctl[4] = s_carry;
    voff[nrec] = s_carry;
  }
}

// arena compaction: the shadow rows follow their spans (same new offsets as k_compact_copy)
__global__ void k_kv_compact(DT T, int32_t hw, const int64_t *__restrict__ newoff, const int32_t *__restrict__ src,
                             int32_t *__restrict__ dst) {
  pdl_wait();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= hw) return;
  const int32_t s = (int32_t)w;
  if (s == ROOT || T.nid[s] < 0 || T.par[s] < 0) return;
  const int64_t from = T.eoff[s], to = newoff[s];  // (runs before k_compact_copy moves eoff)
  for (int32_t i = lane_id(); i < T.elen[s]; i += 32) dst[to + i] = src[from + i];
}

// req_to_token: for leaf j, the pool row of every path position [0, dend(leaf))
// (row-major [n, max_len]; positions past the path are left alone), by one warp
// walking the root chain -- the next node's fields are loaded before the
// current span is copied, so a hop costs about one load latency (the chains
// are long and the spans short: a CTA per leaf was slower); optionally the KV
// rows themselves into out[j, p]
__global__ void k_kv_gather(DT T, KvDev K, int64_t n, const int32_t *__restrict__ leaves, int64_t max_len,
                            int32_t *__restrict__ table, uint8_t *__restrict__ out, int64_t *__restrict__ lens) {
  pdl_wait();
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  int32_t s = leaves[j];
  const int64_t len = s > 0 ? T.dend[s] : 0;
  if (lane == 0) lens[j] = len;
  int32_t *row = table + j * max_len;
  int64_t e = 0, d = 0;
  int32_t l = 0, ps = 0;
  if (s > 0) e = T.eoff[s], l = T.elen[s], d = T.dend[s], ps = T.par[s];
  while (s > 0) {  // (the root holds no tokens)
    int64_t ne = 0, nd = 0;
    int32_t nl = 0, nps = 0;
    if (ps > 0) ne = T.eoff[ps], nl = T.elen[ps], nd = T.dend[ps], nps = T.par[ps];  // (next hop, in flight)
    const int64_t p0 = d - l;
    const int32_t lm = (int32_t)min((int64_t)l, max_len - p0);  // (p0 < max_len is not guaranteed)
    for (int32_t i0 = lane; i0 < lm; i0 += 4 * 32) {  // 4 independent loads in flight per lane
      int32_t v[4];
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (i0 + 32 * u < lm) v[u] = K.kvx[e + i0 + 32 * u];
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (i0 + 32 * u < lm) row[p0 + i0 + 32 * u] = v[u];
    }
    s = ps, e = ne, l = nl, d = nd, ps = nps;
  }
  if (!out) return;
  __syncwarp();
  const int64_t m = len < max_len ? len : max_len;
  const int32_t vpr = (int32_t)(K.bpt / 16);
  const int64_t nv = m * vpr;
  int4 *dst = reinterpret_cast<int4 *>(out + j * max_len * K.bpt);
  VecIt it(lane, 32, vpr);
  for (int64_t x0 = lane; x0 < nv; x0 += 4 * 32) {  // 16-B vectors across all the request's rows, 4 in flight
    int4 val[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      if (x0 + u * 32 < nv) val[u] = reinterpret_cast<const int4 *>(K.pool + (int64_t)row[it.i] * K.bpt)[it.v];
      it.next();
    }
#pragma unroll
    for (int u = 0; u < 4; u++)
      if (x0 + u * 32 < nv) dst[x0 + u * 32] = val[u];
  }
}

}  // namespace prism

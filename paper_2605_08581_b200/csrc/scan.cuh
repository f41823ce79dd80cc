// scan.cuh -- block-wide scans shared by the QAS and DART translation units.
#pragma once
#include <cstdint>

namespace prism {

// block-wide scan of NA int64 sequences at once, in tiles of IPT * blockDim:
// every thread loads its IPT consecutive items of each sequence up front, then
// one warp-shuffle + shared-memory scan per tile.  store(a, i, excl, incl)
// is called for every item i < n of sequence a, load(a, i) reads it.
template <int NA, int IPT, class Load, class Store>
__device__ inline void block_scan4(int64_t n, Load load, Store store) {
  __shared__ int64_t s_w[NA][32];
  __shared__ int64_t s_carry[NA];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x < NA) s_carry[threadIdx.x] = 0;
  __syncthreads();
  const int64_t tile = IPT * (int64_t)blockDim.x;
  for (int64_t t0 = 0; t0 < n; t0 += tile) {
    const int64_t i0 = t0 + IPT * (int64_t)threadIdx.x;
    int64_t v[NA][IPT], sum[NA];
#pragma unroll
    for (int a = 0; a < NA; a++)
#pragma unroll
      for (int u = 0; u < IPT; u++) v[a][u] = i0 + u < n ? load(a, i0 + u) : 0;
#pragma unroll
    for (int a = 0; a < NA; a++) {
      sum[a] = 0;
#pragma unroll
      for (int u = 0; u < IPT; u++) sum[a] += v[a][u];
      int64_t x = sum[a];
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_w[a][wid] = x;
      sum[a] = x - sum[a];  // exclusive within the warp
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
      for (int a = 0; a < NA; a++) {
        int64_t t = lane < nw ? s_w[a][lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
          const int64_t y = __shfl_up_sync(0xffffffffu, t, o);
          if (lane >= o) t += y;
        }
        if (lane < nw) s_w[a][lane] = t;  // inclusive warp totals
      }
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < NA; a++) {
      int64_t run = s_carry[a] + sum[a] + (wid ? s_w[a][wid - 1] : 0);
#pragma unroll
      for (int u = 0; u < IPT; u++) {
        if (i0 + u < n) store(a, i0 + u, run, run + v[a][u]);
        run += v[a][u];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0)
#pragma unroll
      for (int a = 0; a < NA; a++) s_carry[a] += s_w[a][nw - 1];
    __syncthreads();
  }
}

}  // namespace prism

// pdl.cuh -- programmatic dependent launch (sm_90+).
//
// The fused wave is one CUDA graph of ~70 dependent kernels; prism_graph_pdl
// (dart.cu) turns its kernel->kernel edges into programmatic ones, so a
// kernel's CTAs are scheduled while its predecessor is still running and wait
// here, on the device, for the predecessor's completion and memory flush --
// the launch latency of each edge leaves the critical path.  Every kernel of
// this library calls pdl_wait() before touching memory; outside such an edge
// (plain stream launches) it returns at once.
//
// Built with -DPRISM_TRACE (diagnostics only, tools/trace_wave.py), CTA 0 of
// every kernel also stamps %globaltimer and its function name into a per-unit
// device ring as it passes the wait: the in-graph start times of the wave's
// kernels on both streams, i.e. its critical path.
#pragma once

#ifndef PRISM_TRACE
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#define pdl_trace_end()
#else
#include <cuda_runtime.h>
struct PrismTraceRec {
  unsigned long long t;
  char fn[24];
};
constexpr unsigned PRISM_TRACE_CAP = 8192;
static __device__ PrismTraceRec prism_trace_buf[PRISM_TRACE_CAP];
static __device__ unsigned prism_trace_n;
__device__ __forceinline__ void pdl_wait_traced(const char *fn) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && threadIdx.y == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned i = atomicAdd(&prism_trace_n, 1u) % PRISM_TRACE_CAP;
    prism_trace_buf[i].t = t;
    int c = 0;
    for (; c < 23 && fn[c]; c++) prism_trace_buf[i].fn[c] = fn[c];
    prism_trace_buf[i].fn[c] = 0;
  }
}
#define pdl_wait() pdl_wait_traced(__func__)
// end stamp of every CTA whose thread 0 reaches it ("<name>$"; the last one ~
// the kernel's end); no barrier, so kernels with early returns may use it
__device__ __forceinline__ void pdl_trace_end_impl(const char *fn) {
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned i = atomicAdd(&prism_trace_n, 1u) % PRISM_TRACE_CAP;
    prism_trace_buf[i].t = t;
    int c = 0;
    for (; c < 22 && fn[c]; c++) prism_trace_buf[i].fn[c] = fn[c];
    prism_trace_buf[i].fn[c] = '$';
    prism_trace_buf[i].fn[c + 1] = 0;
  }
}
#define pdl_trace_end() pdl_trace_end_impl(__func__)
// host: copy this unit's ring out (records in arrival order) and reset it
static inline int prism_trace_take(unsigned long long *t, char *names, int cap) {
  unsigned n = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&n, prism_trace_n, sizeof(n));
  if (n > PRISM_TRACE_CAP) n = PRISM_TRACE_CAP;
  if ((int)n > cap) n = (unsigned)cap;
  static PrismTraceRec h[PRISM_TRACE_CAP];
  if (n) cudaMemcpyFromSymbol(h, prism_trace_buf, sizeof(PrismTraceRec) * n);
  for (unsigned i = 0; i < n; i++) {
    t[i] = h[i].t;
    for (int c = 0; c < 24; c++) names[24 * i + c] = h[i].fn[c];
  }
  const unsigned z = 0;
  cudaMemcpyToSymbol(prism_trace_n, &z, sizeof(z));
  return (int)n;
}
#endif

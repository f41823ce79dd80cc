// pdl.cuh -- programmatic dependent launch (sm_90+).
//
// The fused wave is one CUDA graph of ~70 dependent kernels; prism_graph_pdl
// (dart.cu) turns its kernel->kernel edges into programmatic ones, so a
// kernel's CTAs are scheduled while its predecessor is still running and wait
// here, on the device, for the predecessor's completion and memory flush --
// the launch latency of each edge leaves the critical path.  Every kernel of
// this library calls pdl_wait() before touching memory; outside such an edge
// (plain stream launches) it returns at once.
#pragma once

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Launch-overhead probe: a chain of N dependent kernels (each reads what the
// previous one wrote) in one CUDA graph, with and without programmatic
// dependent launch (PDL: the next kernel's CTAs are resident and waiting in
// griddepcontrol.wait when the previous one finishes).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pdl_probe tools/pdl_probe.cu && /tmp/pdl_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_step(int *x, int n, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
  if (i < n) x[i] = x[i] + 1;
}

int main() {
  const int N = 70, n = 148 * 512;
  int *x;
  cudaMalloc(&x, n * sizeof(int));
  cudaMemset(x, 0, n * sizeof(int));
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int pdl = 0; pdl < 2; pdl++) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed);
    for (int k = 0; k < N; k++) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((n + 255) / 256);
      cfg.blockDim = dim3(256);
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = pdl;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_step, x, n, pdl);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int r = 0; r < 20; r++) cudaGraphLaunch(ge, st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    const int R = 200;
    for (int r = 0; r < R; r++) cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("graph of %d kernels, pdl=%d: %.2f us per kernel (err %s)\n", N, pdl, ms * 1000 / (R * N),
           cudaGetErrorString(cudaGetLastError()));
  }
  int h = 0;
  cudaMemcpy(&h, x, sizeof(int), cudaMemcpyDeviceToHost);
  printf("x[0] = %d (expect %d)\n", h, 2 * 220 * N);
  return 0;
}

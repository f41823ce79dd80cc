// microbenchmark of the shared-memory sorters (block_merge_sort, bitonic_smem)
// on one CTA: clock64 cycles for n random Key3 keys (tools only)
#include <cstdio>
#include <vector>
#include "../paper_2605_08581_b200/csrc/coop.cuh"
using namespace prism;

template <int ALG>
__global__ void k_bench(const Key3 *in, int n, unsigned long long *cyc, int *bad) {
  extern __shared__ __align__(16) unsigned char dsm[];
  Key3 *sk = reinterpret_cast<Key3 *>(dsm);
  uint64_t *sv = reinterpret_cast<uint64_t *>(sk + 2048);
  Key3 *tk = reinterpret_cast<Key3 *>(sv + 2048);
  uint64_t *tv = reinterpret_cast<uint64_t *>(tk + 2048);
  int mp = 1;
  while (mp < n) mp <<= 1;
  for (int i = threadIdx.x; i < mp; i += blockDim.x) {
    sk[i] = i < n ? in[i] : Key3{~0ull, ~0ull, ~0ull};
    sv[i] = i < n ? in[i].w2 : 0;
  }
  __syncthreads();
  const long long c0 = clock64();
  if (ALG == 0) block_merge_sort(sk, sv, n, tk, tv, sk, sv);
  else if (ALG == 2) block_sort(sk, sv, n, tk, tv, sk, sv);
  else bitonic_smem(sk, sv, mp);
  __syncthreads();
  const long long c1 = clock64();
  if (threadIdx.x == 0) {
    cyc[blockIdx.x] = c1 - c0;
    int b = 0;
    for (int i = 1; i < n; i++) b += key_less(sk[i], sk[i - 1]);
    for (int i = 0; i < n; i++) b += (sv[i] != sk[i].w2) ? 1000 : 0;
    bad[blockIdx.x] = b;
  }
}

int main() {
  const int ns[] = {5, 32, 100, 128, 256, 414, 512, 1000, 1024, 2048};
  std::vector<Key3> h(2048);
  for (int i = 0; i < 2048; i++) h[i] = {0, (unsigned long long)(i * 2654435761u % 100003), (unsigned long long)i};
  Key3 *d;
  cudaMalloc(&d, sizeof(Key3) * 2048);
  cudaMemcpy(d, h.data(), sizeof(Key3) * 2048, cudaMemcpyHostToDevice);
  unsigned long long *cyc;
  int *bad;
  cudaMalloc(&cyc, 8 * 1024);
  cudaMalloc(&bad, 4 * 1024);
  const int smem = 2 * 2048 * 32;
  cudaFuncSetAttribute(k_bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int tpb : {256, 512, 1024})
    for (int n : ns)
      for (int alg = 0; alg < 3; alg++) {
        for (int rep = 0; rep < 2; rep++) {
          if (alg == 0) k_bench<0><<<1, tpb, smem>>>(d, n, cyc, bad);
          else if (alg == 2) k_bench<2><<<1, tpb, smem>>>(d, n, cyc, bad);
          else k_bench<1><<<1, tpb, smem>>>(d, n, cyc, bad);
        }
        unsigned long long c;
        int b;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(&b, bad, 4, cudaMemcpyDeviceToHost);
        printf("tpb %4d n %5d %s cycles %8llu bad %d\n", tpb, n, alg == 2 ? "bsort  " : alg ? "bitonic" : "merge  ", c, b);
      }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}

// Micro-benchmark of the CTA sort primitives (clock64 inside one CTA).
#include <cstdio>
#include <cstdint>
#include "../paper_2402_02361_b200/csrc/tt_block.cuh"
using namespace tt;

template <int E, typename K>
__global__ void kbench(const uint64_t* in, uint64_t* out, long long* cyc) {
  extern __shared__ __align__(16) unsigned char sm[];
  K kk[E];
  for (int e = 0; e < E; ++e) {
    int p = e * blockDim.x + threadIdx.x;
    kk[e].a = in[p]; kk[e].b = p;
  }
  __syncthreads();
  long long t0 = clock64();
  block_sort_reg<E, K>(kk, (K*)sm);
  long long t1 = clock64();
  for (int e = 0; e < E; ++e) out[e * blockDim.x + threadIdx.x] = kk[e].a;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  const int N = 4096;
  uint64_t *in, *out; long long* cyc;
  cudaMallocManaged(&in, N * 8); cudaMallocManaged(&out, N * 8); cudaMallocManaged(&cyc, 8);
  for (int i = 0; i < N; ++i) in[i] = (uint64_t)((i * 2654435761u) % 100003);
  cudaFuncSetAttribute(kbench<4, Key2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 16);
  for (int rep = 0; rep < 3; ++rep) {
    kbench<4, Key2><<<1, 1024, 4096 * 16>>>(in, out, cyc); cudaDeviceSynchronize();
    printf("E=4 NT=1024 Key2: %lld cycles\n", *cyc);
    kbench<1, Key2><<<1, 1024, 1024 * 16>>>(in, out, cyc); cudaDeviceSynchronize();
    printf("E=1 NT=1024 Key2: %lld cycles\n", *cyc);
    kbench<1, Key3><<<1, 512, 512 * 24>>>(in, out, cyc); cudaDeviceSynchronize();
    printf("E=1 NT=512 Key3: %lld cycles\n", *cyc);
  }
  bool ok = true;
  kbench<4, Key2><<<1, 1024, 4096 * 16>>>(in, out, cyc); cudaDeviceSynchronize();
  for (int i = 1; i < N; ++i) ok &= out[i - 1] <= out[i];
  printf("sorted ok=%d err=%s\n", ok, cudaGetErrorString(cudaGetLastError()));
}

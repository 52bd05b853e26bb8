#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include "../paper_2402_02361_b200/csrc/tt_block.cuh"
using namespace tt;
template <int E>
__global__ void __launch_bounds__(1024) ksort(const Key3* in, Key3* out) {
  extern __shared__ __align__(16) unsigned char sraw[];
  Key3* xchg = (Key3*)sraw;
  Key3 kk[E];
#pragma unroll
  for (int e = 0; e < E; ++e) kk[e] = in[e * blockDim.x + threadIdx.x];
  block_sort_reg<E, Key3>(kk, xchg);
#pragma unroll
  for (int e = 0; e < E; ++e) out[e * blockDim.x + threadIdx.x] = kk[e];
}
template <int E>
void run(int NT, int mode) {
  int n = NT * E;
  std::mt19937_64 rng(5);
  std::vector<Key3> h(n);
  for (int i = 0; i < n; ++i) {
    uint64_t a = rng(), b = rng() % 13;
    if (mode == 1) a >>= 1;           // top bit clear
    if (mode == 2) a = (rng() % 600) | (1ull << 63);  // ties, top bit set
    if (mode == 3) a = rng() % 600;   // ties, top bit clear
    h[i].a = a; h[i].b = b; h[i].c = i;
  }
  Key3 *di, *dout;
  cudaMalloc(&di, n * sizeof(Key3)); cudaMalloc(&dout, n * sizeof(Key3));
  cudaMemcpy(di, h.data(), n * sizeof(Key3), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(ksort<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, n * (int)sizeof(Key3));
  ksort<E><<<1, NT, n * sizeof(Key3)>>>(di, dout);
  cudaError_t err = cudaDeviceSynchronize();
  std::vector<Key3> o(n); cudaMemcpy(o.data(), dout, n * sizeof(Key3), cudaMemcpyDeviceToHost);
  int bad = 0; std::vector<int> cnt(n, 0);
  for (int i = 0; i < n; ++i) if (o[i].c < (unsigned)n) cnt[o[i].c]++;
  int dup = 0; for (int i = 0; i < n; ++i) dup += cnt[i] != 1;
  for (int i = 1; i < n; ++i) bad += o[i].lt(o[i-1]);
  printf("E=%d NT=%4d mode=%d err=%s unsorted=%d multiset=%d\n", E, NT, mode, cudaGetErrorString(err), bad, dup);
  cudaFree(di); cudaFree(dout);
}
int main() {
  for (int mode = 0; mode < 4; ++mode) { run<4>(1024, mode); run<2>(1024, mode); run<8>(512, mode); run<4>(512, mode); }
}

// Gap between consecutive kernels on one stream (%globaltimer at each kernel's
// start / end): regular -> regular, regular -> D2H record copy -> cooperative,
// to see what sits between a round's verify kernel and the next selector.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__device__ unsigned long long g_t[64];
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}
__global__ void k_reg(int slot) {
  if (blockIdx.x == 0 && threadIdx.x == 0) g_t[2 * slot] = gt();
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) g_t[2 * slot + 1] = gt();
}
__global__ void k_coop(int slot) {
  if (blockIdx.x == 0 && threadIdx.x == 0) g_t[2 * slot] = gt();
  cg::this_grid().sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) g_t[2 * slot + 1] = gt();
}
int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  long long *d, *h;
  cudaMalloc(&d, 4096);
  cudaMallocHost(&h, 4096);
  auto coop = [&](int slot) {
    void* args[] = {&slot};
    cudaLaunchCooperativeKernel((void*)k_coop, dim3(148), dim3(1024), args, 0, s);
  };
  for (int rep = 0; rep < 3; ++rep) {
    int q = 0;
    k_reg<<<128, 512, 0, s>>>(q++);
    k_reg<<<128, 512, 0, s>>>(q++);                                  // 1: reg -> reg
    coop(q++);                                                       // 2: reg -> coop
    coop(q++);                                                       // 3: coop -> coop
    k_reg<<<128, 512, 0, s>>>(q++);                                  // 4: coop -> reg
    cudaMemcpyAsync(h, d, 400, cudaMemcpyDeviceToHost, s);
    coop(q++);                                                       // 5: reg -> D2H -> coop
    k_reg<<<128, 512, 0, s>>>(q++);
    cudaMemcpyAsync(h, d, 400, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(h + 64, d, 4, cudaMemcpyDeviceToHost, s);
    cudaMemsetAsync(d, 0, 4, s);
    coop(q++);                                                       // 7: reg -> 2 D2H + memset -> coop
    k_reg<<<128, 512, 0, s>>>(q++);
    cudaMemsetAsync(d, 0, 4, s);
    k_reg<<<128, 512, 0, s>>>(q++);                                  // 9: reg -> memset -> reg
    cudaStreamSynchronize(s);
  }
  unsigned long long t[64];
  cudaMemcpyFromSymbol(t, g_t, sizeof(t));
  const char* what[] = {"", "reg->reg", "reg->coop", "coop->coop", "coop->reg", "reg->D2H->coop", "",
                        "reg->2xD2H+memset->coop", "", "reg->memset->reg"};
  for (int q = 1; q < 10; ++q)
    if (what[q][0]) printf("%-26s gap %.2f us (previous end -> this start)\n", what[q], (t[2 * q] - t[2 * q - 1]) / 1e3);
  return 0;
}

// Grid-barrier latency on B200: 148 co-resident CTAs x 1024 threads,
// cooperative launch, R barriers per launch. Variants: 0 = generation
// barrier with __nanosleep polling, 1 = the same without sleep, 2 =
// cooperative_groups grid.sync(), 3 = generation barrier with ld.acquire.gpu
// polling and red.release arrival.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/barrier_bench tools/barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

struct Bar { unsigned count, gen; };

template <int V>
__device__ __forceinline__ void gbar(Bar* b) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = &b->gen;
    unsigned g;
    if (V == 3) asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g) : "l"(&b->gen));
    else g = *gen;
    __threadfence();
    if (atomicAdd(&b->count, 1u) == gridDim.x - 1) {
      atomicExch(&b->count, 0u);
      __threadfence();
      atomicAdd(&b->gen, 1u);
    } else if (V == 3) {
      unsigned x;
      do { asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(x) : "l"(&b->gen)); } while (x == g);
    } else {
      while (*gen == g) { if (V == 0) __nanosleep(32); }
    }
    __threadfence();
  }
  __syncthreads();
}

template <int V>
__global__ void __launch_bounds__(1024, 1) kbar(Bar* b, int R, unsigned long long* t) {
  unsigned long long t0 = clock64();
  for (int r = 0; r < R; ++r) {
    if (V == 2) cg::this_grid().sync();
    else gbar<V>(b);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *t = clock64() - t0;
}

template <int V>
void run(Bar* b, unsigned long long* t, int grid, int R) {
  void* args[] = {&b, &R, &t};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) cudaLaunchCooperativeKernel((void*)kbar<V>, grid, 1024, args, 0, 0);
  cudaEventRecord(e0);
  cudaLaunchCooperativeKernel((void*)kbar<V>, grid, 1024, args, 0, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc;
  cudaMemcpy(&cyc, t, 8, cudaMemcpyDeviceToHost);
  printf("variant %d grid %d: %.3f us per barrier (events), %.0f cycles per barrier (CTA 0) err=%s\n", V, grid,
         ms * 1e3 / R, (double)cyc / R, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  Bar* b;
  unsigned long long* t;
  cudaMalloc(&b, sizeof(Bar));
  cudaMemset(b, 0, sizeof(Bar));
  cudaMalloc(&t, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int grid : {sms, 74, 16}) {
    run<0>(b, t, grid, 1000);
    run<1>(b, t, grid, 1000);
    run<2>(b, t, grid, 1000);
    run<3>(b, t, grid, 1000);
  }
  return 0;
}

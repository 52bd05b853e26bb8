// Latency of one 64-step fp64 dot-product chain (reference order) whose
// operands sit in shared memory, as the PaCM head/attention phases run it:
// plain loop vs batched loads (8 ahead). One CTA of 256 threads.
#include <cstdio>
__device__ __forceinline__ double chain_plain(double acc, const double* x, int sx, const double* w, int sw) {
#pragma unroll 16
  for (int f = 0; f < 64; ++f) acc = __dadd_rn(acc, __dmul_rn(x[f * sx], w[f * sw]));
  return acc;
}
__device__ __forceinline__ double chain_batch(double acc, const double* __restrict__ x, int sx,
                                              const double* __restrict__ w, int sw) {
  double xc[8], wc[8];
#pragma unroll
  for (int v = 0; v < 8; ++v) xc[v] = x[v * sx], wc[v] = w[v * sw];
#pragma unroll 1
  for (int b = 1; b <= 8; ++b) {
    double xn[8], wn[8];
    const int bn = b < 8 ? b : 7;
#pragma unroll
    for (int v = 0; v < 8; ++v) xn[v] = x[(8 * bn + v) * sx], wn[v] = w[(8 * bn + v) * sw];
    double p[8];
#pragma unroll
    for (int v = 0; v < 8; ++v) p[v] = __dmul_rn(xc[v], wc[v]);
#pragma unroll
    for (int v = 0; v < 8; ++v) acc = __dadd_rn(acc, p[v]);
#pragma unroll
    for (int v = 0; v < 8; ++v) xc[v] = xn[v], wc[v] = wn[v];
  }
  return acc;
}
__device__ __forceinline__ double chain_regs(double acc, const double* __restrict__ x, int sx,
                                             const double* __restrict__ w, int sw) {
  double p[64];
#pragma unroll
  for (int f = 0; f < 64; ++f) p[f] = __dmul_rn(x[f * sx], w[f * sw]);
#pragma unroll
  for (int f = 0; f < 64; ++f) acc = __dadd_rn(acc, p[f]);
  return acc;
}
template <int MODE>
__global__ void k(double* out, long long* cyc) {
  __shared__ double W[64 * 64 + 128];
  for (int i = threadIdx.x; i < 64 * 64 + 128; i += blockDim.x) W[i] = 1.0 + 1e-3 * (i & 63);
  __syncthreads();
  const double* x = W + 64 * 64;
  const int j = threadIdx.x & 63;
  double acc = 0.0;
  long long t0 = clock64();
  for (int rep = 0; rep < 4; ++rep) {
    if (MODE == 0) acc = chain_plain(acc, x, 1, W + j, 64);
    if (MODE == 1) acc = chain_batch(acc, x, 1, W + j, 64);
    if (MODE == 2) acc = chain_regs(acc, x, 1, W + j, 64);
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 4;
}
int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 64);
  const char* names[3] = {"plain (unroll 16)", "batched 8 ahead", "64 products then chain"};
  for (int m = 0; m < 3; ++m) {
    for (int it = 0; it < 2; ++it) {
      if (m == 0) k<0><<<1, 256>>>(out, cyc);
      if (m == 1) k<1><<<1, 256>>>(out, cyc);
      if (m == 2) k<2><<<1, 256>>>(out, cyc);
      cudaDeviceSynchronize();
    }
    printf("%-24s %lld cycles per 64-step chain\n", names[m], cyc[0]);
  }
  return 0;
}

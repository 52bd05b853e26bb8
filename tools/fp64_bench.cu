// fp64 pipe calibration: dependent-chain latency and throughput of DADD/DMUL/DFMA per SM.
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double a, double b) {
  double x = a;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { x = __dadd_rn(x, b); x = __dadd_rn(x, b); x = __dadd_rn(x, b); x = __dadd_rn(x, b); }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 4096;
}
template <int CH>
__global__ void thr(double* out, long long* cyc, double a, double b) {
  double x[CH];
  for (int c = 0; c < CH; ++c) x[c] = a + c;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __dadd_rn(__dmul_rn(x[c], b), a);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0; for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 24); cudaMallocManaged(&cyc, 64);
  lat<<<1, 32>>>(out, cyc, 1.0, 1e-9); cudaDeviceSynchronize();
  lat<<<1, 32>>>(out, cyc, 1.0, 1e-9); cudaDeviceSynchronize();
  printf("DADD dependent latency: %lld cycles\n", cyc[0]);
  for (int warps : {1, 4, 8, 16, 32}) {
    thr<8><<<1, 32 * warps>>>(out, cyc, 1.0, 0.999); cudaDeviceSynchronize();
    thr<8><<<1, 32 * warps>>>(out, cyc, 1.0, 0.999); cudaDeviceSynchronize();
    double ops = 2.0 * 8 * 1024 * 32 * warps;  // DMUL + DADD lanes
    printf("1 SM, %2d warps x 8 chains: %lld cycles -> %.1f fp64 lane-ops/clk/SM\n", warps, cyc[0], ops / cyc[0]);
  }
  return 0;
}

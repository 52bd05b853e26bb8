// fp64 dense-tile calibration for k_pacm64_h64: one CTA of 512 threads per SM,
// a 64-step k loop per tile, weights W[k][64] and activations X^T[k][8] in
// shared memory (as the kernel stages them). Prints fp64 lane-ops/clk/SM.
#include <cstdio>
template <int NC, int NR>
__global__ void tile(double* out, long long* cyc, int reps) {
  extern __shared__ double sm[];
  double* W = sm;            // [64][64]
  double* X = sm + 64 * 64;  // 16 warps x [64][8]
  for (int i = threadIdx.x; i < 64 * 64 + 16 * 512; i += blockDim.x) sm[i] = 1.0 + 1e-3 * (i & 127);
  __syncthreads();
  const int j = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double* xt = X + w * 512 + (NR == 4 ? 4 * ((threadIdx.x >> 4) & 1) : 0);
  double a[NC][NR];
  for (int c = 0; c < NC; ++c)
    for (int r = 0; r < NR; ++r) a[c][r] = 0.0;
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 4
    for (int k = 0; k < 64; ++k) {
      double wv[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) wv[c] = W[k * 64 + j + 32 * c];
      double x[NR];
#pragma unroll
      for (int q = 0; q < NR / 2; ++q) {
        const double2 v = *(const double2*)(xt + k * 8 + 2 * q);
        x[2 * q] = v.x, x[2 * q + 1] = v.y;
      }
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int r = 0; r < NR; ++r) a[c][r] = __dadd_rn(a[c][r], __dmul_rn(x[r], wv[c]));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < NC; ++c)
    for (int r = 0; r < NR; ++r) s += a[c][r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int NC, int NR>
void run(const char* name, double* out, long long* cyc, int threads) {
  const int smem = (64 * 64 + 16 * 512) * 8;
  cudaFuncSetAttribute(tile<NC, NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tile<NC, NR><<<148, threads, smem>>>(out, cyc, 8);
  cudaDeviceSynchronize();
  tile<NC, NR><<<148, threads, smem>>>(out, cyc, 8);
  cudaDeviceSynchronize();
  const double ops = 2.0 * NC * NR * 64 * 8 * threads;
  printf("%-28s threads %4d: %6lld cycles -> %.1f fp64 lane-ops/clk/SM\n", name, threads, cyc[0], ops / cyc[0]);
}
int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMallocManaged(&cyc, 64);
  run<1, 8>("1 col x 8 rows (8 chains)", out, cyc, 512);
  run<2, 8>("2 col x 8 rows (16 chains)", out, cyc, 512);
  run<2, 8>("2 col x 8 rows (16 chains)", out, cyc, 256);
  run<2, 4>("2 col x 4 rows (8 chains)", out, cyc, 512);
  run<1, 4>("1 col x 4 rows (4 chains)", out, cyc, 512);
  run<4, 8>("4 col x 8 rows (32 chains)", out, cyc, 256);
  run<1, 8>("1 col x 8 rows (8 chains)", out, cyc, 256);
  return 0;
}

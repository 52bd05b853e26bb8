#include <cstdio>
#include <vector>
#include <algorithm>
#include <cstdlib>
#include "../paper_2402_02361_b200/csrc/tt_kernels.h"
int main() {
  int n = 5000; const int b = 4;
  if (getenv("NN")) n = atoi(getenv("NN"));
  std::vector<double> s(n), d(n);
  for (int i = 0; i < n; ++i) s[i] = ((i * 7919 % 1000) - 500) / 100.0, d[i] = (i % 13) / 10.0;
  if (FILE* f = fopen("/tmp/s.bin", "rb")) { fread(s.data(), 8, n, f); fclose(f); printf("loaded s\n"); }
  double *ds, *dd; int64_t *pos, *cnt; int* st;
  cudaMalloc(&ds, n * 8); cudaMalloc(&dd, n * 8); cudaMalloc(&pos, 64 * 8); cudaMalloc(&cnt, 8); cudaMalloc(&st, 4);
  cudaMemcpy(ds, s.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dd, d.data(), n * 8, cudaMemcpyHostToDevice);
  int rc = 0;
  for (int mode = 0; mode < 3; ++mode) {
    cudaStream_t strm = 0;
    if (mode == 1) strm = (cudaStream_t)0x1;
    if (mode == 2) cudaStreamCreateWithFlags(&strm, cudaStreamNonBlocking);
    cudaMemset(pos, 0, 64 * 8);
    rc = tt::launch_select_top(ds, dd, nullptr, n, nullptr, b, pos, cnt, st, strm);
    printf("launch err: %s\n", cudaGetErrorString(cudaGetLastError()));
    cudaDeviceSynchronize();
    int64_t hp2[8];
    cudaMemcpy(hp2, pos, b * 8, cudaMemcpyDeviceToHost);
    printf("mode %d: %ld %ld %ld %ld\n", mode, (long)hp2[0], (long)hp2[1], (long)hp2[2], (long)hp2[3]);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("rc=%d err=%s\n", rc, cudaGetErrorString(e));
  int64_t hp[64], hc; int hs;
  cudaMemcpy(hp, pos, b * 8, cudaMemcpyDeviceToHost); cudaMemcpy(&hc, cnt, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&hs, st, 4, cudaMemcpyDeviceToHost);
  printf("count=%ld status=%d pos=", (long)hc, hs);
  for (int i = 0; i < b; ++i) printf("%ld ", (long)hp[i]);
  printf("\n");
  // host reference
  std::vector<int> idx(n); for (int i = 0; i < n; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int a, int c) { if (s[a] != s[c]) return s[a] > s[c]; if (d[a] != d[c]) return d[a] < d[c]; return a < c; });
  printf("want: "); for (int i = 0; i < b; ++i) printf("%d ", idx[i]); printf("\n");
}

// tt_pacm64.cuh — the fp64 PaCM forward (run_forward, ranker.cpp:159-209) on
// CUDA cores: parameter layout, branch-free exp/tanh, and the throughput pass
// loop for the tuner's geometry (h = 64), shared by k_pacm64_h64 (feature
// rows from global memory, k_pacm64.cu) and k_verify64 (features computed in
// the same kernel, k_verify.cu).
#pragma once

#include <cstdint>

#include "tt_kernels.h"
#include "tt_tc.cuh"

namespace tt {

struct Params64 {
  const double *w1, *b1, *w2, *b2, *we, *be, *wq, *bq, *wk, *bk, *wv, *bv, *hw1, *hb1, *hw2, *hb2;
};

__host__ __device__ inline Params64 split_params(const double* p, int h) {
  Params64 P;
  P.w1 = p, P.b1 = P.w1 + 24 * h, P.w2 = P.b1 + h, P.b2 = P.w2 + h * h;
  P.we = P.b2 + h, P.be = P.we + 23 * h, P.wq = P.be + h, P.bq = P.wq + h * h;
  P.wk = P.bq + h, P.bk = P.wk + h * h, P.wv = P.bk + h, P.bv = P.wv + h * h;
  P.hw1 = P.bv + h, P.hb1 = P.hw1 + 2 * h * h, P.hw2 = P.hb1 + h, P.hb2 = P.hw2 + h;
  return P;
}

// Rows are padded to a multiple of 4 (16-byte activation loads); a thread
// work item covers RG rows of one output column (RG independent chains).
__host__ __device__ inline int pad4(int n) { return (n + 3) / 4 * 4; }

// Branch-free fp64 exp and tanh. CUDA's tanh/exp take data-dependent
// branches (range reduction special cases, division slow paths) that
// serialise the many independent activations a thread evaluates per layer;
// these straight-line forms interleave. exp: Cody-Waite reduction by ln 2
// and a degree-13 Taylor polynomial on |r| <= 0.35 (truncation < 1e-17
// relative), scaled by 2^n in two factors (no overflow in the split). tanh
// = 1 - 2 / (1 + e^{2x}) with a Newton-refined reciprocal: absolute error
// ~1e-16 against glibc's tanh — the same order as the ulp-level
// differences CUDA's own tanh already has, far inside the 1e-12 score
// tolerance.
__device__ __forceinline__ double exp64(double x) {
  x = fmin(fmax(x, -745.0), 709.78);
  const double n = rint(x * 1.4426950408889634074);
  double r = fma(-n, 6.93147180369123816490e-01, x);
  r = fma(-n, 1.90821492927058770002e-10, r);
  double p = 1.6059043836821614599e-10;  // 1/13!
  p = fma(p, r, 2.0876756987868098979e-09);
  p = fma(p, r, 2.5052108385441718775e-08);
  p = fma(p, r, 2.7557319223985890653e-07);
  p = fma(p, r, 2.7557319223985890653e-06);
  p = fma(p, r, 2.4801587301587301587e-05);
  p = fma(p, r, 1.9841269841269841270e-04);
  p = fma(p, r, 1.3888888888888888889e-03);
  p = fma(p, r, 8.3333333333333333333e-03);
  p = fma(p, r, 4.1666666666666666667e-02);
  p = fma(p, r, 1.6666666666666666667e-01);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const int ni = (int)n, n1 = ni >> 1, n2 = ni - n1;
  const double s1 = __longlong_as_double((long long)(n1 + 1023) << 52);
  const double s2 = __longlong_as_double((long long)(n2 + 1023) << 52);
  return (p * s1) * s2;
}

__device__ __forceinline__ double rcp64(double d) {  // d >= 1
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}

__device__ __forceinline__ double tanh64(double x) {
  const double e2 = exp64(2.0 * x);
  return 1.0 - 2.0 * rcp64(1.0 + e2);
}

// ---------------------------------------------------------------------------
// Throughput kernel for whole drafted sets at the tuner's model geometry
// (h = 64, <= 8 statement rows, <= 8 dataflow blocks, attention on): the same
// per-output accumulation order as k_pacm64, re-scheduled so the fp64 pipe
// stays busy. G = 4 candidates per CTA, 16 warps. Every dense output tile is
// one thread's 16 register chains: 8 rows x 2 columns (j, j + 32) of one
// candidate, so a k step is 2 weight loads + 4 broadcast 16-byte activation
// loads for 32 DMUL/DADD: 58 of the SM's 64 fp64 lanes/clk in isolation
// (tools/fp64_tile_bench.cu; 1-column tiles reach 49, bound by shared-memory
// wavefronts). One code path per phase keeps the instruction footprint small.
//
//   phase 1  threads 0-127: statement layer 1 | 128-255: block embedding
//            (pre-activations), then tanh spread over all 512 threads
//   phase 2  statement layer 2 | Q | K | V, 128 threads each (bound: fp64 pipe)
//   phase 3  0-255: tanh + mean-pool of the statement branch, head layer 1
//            over that half (k < 64) | 256-511: QK^T, softmax, PV, attention
//            mean-pool
//   phase 4  0-255: head layer 1, k = 64..127, tanh; head layer 2
//
// Weights move by 1-D bulk TMA: WA (128 KB) = W2|Wq|Wk|Wv for phase 2, then
// the head's W1 (2h x h); W1|We (24 KB) are staged in the q/k/v region, which
// phase 2 only writes after phase 1 is done. One mbarrier per copy group,
// each completing once per pass (parity = pass & 1). exp/tanh are the
// table-driven exp64t / tanh64t (below).
namespace f64 {
constexpr int H = 64, R = 8, G = 4, T = 512;
constexpr int kWA = 4 * H * H;              // doubles
constexpr int kZE = 2 * H * R;              // z1, e per candidate
constexpr int kQKV = 3 * H * R;             // q, k, v per candidate
constexpr int kMisc = 384;                  // xs^T|xb^T (phase 1) / pr|cat|prod (phases 3-5)
constexpr size_t kSmem = (size_t)(kWA + G * (kZE + kQKV + kMisc)) * sizeof(double);
}  // namespace f64

// a[w][r] = sum_{k<M} xt[k][r] * W[w][k*64 + j], k ascending from +0.0 (the
// reference's order), 8 rows per weight column; operands of step k+1 are
// loaded before step k is computed. Each step is one fused multiply-add (one
// rounding where the reference's x86 build rounds twice): the dense layers
// are fp64-pipe bound, and DFMA does the step in one pipe slot instead of
// two; scores stay within the 1e-12 fp64 tolerance (observed ~1e-15).
template <int M, int NW, int NR = 8>
__device__ __forceinline__ void chains8(const double* __restrict__ xt, const double* const (&W)[NW], int j,
                                        double (&a)[NW][8]) {
  static_assert(NR % 2 == 0 && NR <= 8, "rows in pairs");
#pragma unroll
  for (int w = 0; w < NW; ++w)
#pragma unroll
    for (int r = 0; r < 8; ++r) a[w][r] = 0.0;
  double wc[NW];
  double2 x[NR / 2];
#pragma unroll
  for (int w = 0; w < NW; ++w) wc[w] = W[w][j];
#pragma unroll
  for (int q = 0; q < NR / 2; ++q) x[q] = *(const double2*)(xt + 2 * q);
#pragma unroll 4
  for (int k = 0; k < M; ++k) {
    double wn[NW];
    double2 xn[NR / 2];
    const int kn = k + 1 < M ? k + 1 : k;
#pragma unroll
    for (int w = 0; w < NW; ++w) wn[w] = W[w][kn * f64::H + j];
#pragma unroll
    for (int q = 0; q < NR / 2; ++q) xn[q] = *(const double2*)(xt + kn * 8 + 2 * q);
#pragma unroll
    for (int w = 0; w < NW; ++w) {
#pragma unroll
      for (int q = 0; q < NR / 2; ++q) {
        a[w][2 * q] = __fma_rn(x[q].x, wc[w], a[w][2 * q]);
        a[w][2 * q + 1] = __fma_rn(x[q].y, wc[w], a[w][2 * q + 1]);
      }
    }
#pragma unroll
    for (int w = 0; w < NW; ++w) wc[w] = wn[w];
#pragma unroll
    for (int q = 0; q < NR / 2; ++q) x[q] = xn[q];
  }
}

// bias (+ tanh on the first `rows` rows; padding rows keep finite values no
// consumer reads), then the transposed store y^T[j][r]
__device__ __forceinline__ void store8(double (&a)[8], double bj, bool act, int rows, double* __restrict__ yt,
                                       int j) {
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    double z = __dadd_rn(a[r], bj);
    if (act && r < rows) z = tanh64(z);
    a[r] = z;
  }
  double2* d = (double2*)(yt + j * 8);
#pragma unroll
  for (int q = 0; q < 4; ++q) d[q] = make_double2(a[2 * q], a[2 * q + 1]);
}

// one 8-row x 2-column tile (columns j, j + 32) of y = act(x W + b)
template <int M, int NR = 8>
__device__ __forceinline__ void tile8x2(const double* __restrict__ xt, const double* __restrict__ W,
                                        const double* __restrict__ b, bool act, int rows, double* __restrict__ yt,
                                        int j) {
  double a[2][8];
  const double* const Wp[2] = {W, W + 32};
  chains8<M, 2, NR>(xt, Wp, j, a);
  store8(a[0], __ldg(b + j), act, rows, yt, j);
  store8(a[1], __ldg(b + j + 32), act, rows, yt, j + 32);
}

// acc + sum_{f<64} x[f * sx] * w[f * sw], f ascending: one dependent DFMA
// chain (the reference's order, fused like chains8). Each half's operands are
// loaded first (their loads in flight together), then chained: one pipe
// step per term, against ~25 cycles when each step's operands are loaded in
// front of it (tools/chain_bench.cu).
static __device__ __noinline__ double chain64(double acc, const double* __restrict__ x, int sx,
                                          const double* __restrict__ w, int sw) {
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    double xv[32], wv[32];
#pragma unroll
    for (int v = 0; v < 32; ++v) xv[v] = x[(32 * hf + v) * sx], wv[v] = w[(32 * hf + v) * sw];
#pragma unroll
    for (int v = 0; v < 32; ++v) acc = __fma_rn(xv[v], wv[v], acc);  // fused, as in chains8
  }
  return acc;
}

// Table-driven exp for the throughput kernel: x = (32 m + j) ln2/32 + r,
// |r| <= ln2/64, exp(x) = 2^m * 2^(j/32) * e^r with a degree-6 Taylor e^r
// (truncation < 4e-18 relative) and the table entry applied by one fma
// (T + T (e^r - 1)): ~12 fp64 operations and a 6-deep Horner chain, against
// ~22 and 13 for exp64. T holds the correctly rounded 2^(j/32) in shared
// memory. Same clamping and two-factor scaling as exp64; agreement with glibc
// is at the ulp level, like exp64's.
static __constant__ double kExp2Tab[32] = {
    1.0, 1.0218971486541166, 1.0442737824274138, 1.0671404006768237, 1.0905077326652577,
    1.1143867425958924, 1.1387886347566916, 1.1637248587775775, 1.189207115002721, 1.215247359980469,
    1.241857812073484, 1.2690509571917332, 1.2968395546510096, 1.3252366431597413, 1.3542555469368927,
    1.383909881963832, 1.4142135623730951, 1.4451808069770467, 1.4768261459394993, 1.5091644275934228,
    1.5422108254079407, 1.5759808451078865, 1.6104903319492543, 1.645755478153965, 1.681792830507429,
    1.718619298122478, 1.7562521603732995, 1.7947090750031072, 1.8340080864093424, 1.8741676341103,
    1.9152065613971474, 1.9571441241754002};

__device__ __forceinline__ double exp64t(double x, const double* __restrict__ T) {
  x = fmin(fmax(x, -745.0), 709.78);
  const double kd = rint(x * 46.16624130844683);  // 32 / ln 2
  double r = fma(-kd, 0.02166084938653512, x);    // ln2/32, high part (32 significant bits)
  r = fma(-kd, 5.9631716539705866e-12, r);        // low part
  double q = fma(r, 1.0 / 720.0, 1.0 / 120.0);
  q = fma(q, r, 1.0 / 24.0);
  q = fma(q, r, 1.0 / 6.0);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = q * r;  // e^r - 1
  const int k = (int)kd, j = k & 31, m = k >> 5, m1 = m >> 1, m2 = m - m1;
  const double tj = T[j];
  const double v = fma(tj, q, tj);
  const double s1 = __longlong_as_double((long long)(m1 + 1023) << 52);
  const double s2 = __longlong_as_double((long long)(m2 + 1023) << 52);
  return (v * s1) * s2;
}

__device__ __forceinline__ double tanh64t(double x, const double* __restrict__ T) {
  const double e2 = exp64t(2.0 * x, T);
  return 1.0 - 2.0 * rcp64(1.0 + e2);
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// clock64 marks of CTA 0's first pass (threads 0 and 256), tools/probe_pacm64_h64.py;
// %globaltimer: [0] first CTA start, [1] first past pdl_wait, [2] last past pdl_wait, [3] last CTA done
static __device__ long long g_clk_h64[24];
static __device__ unsigned long long g_h64_ns[4];
__device__ __forceinline__ unsigned long long gtimer64() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}
#define H64_MARK(i, who)                                                    \
  do {                                                                      \
    if (blockIdx.x == 0 && t == (who) && e0 == 0) {                         \
      long long c_;                                                         \
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_)::"memory");          \
      g_clk_h64[i] = c_;                                                    \
    }                                                                       \
  } while (0)

// The pass loop of the throughput kernel. Stage(e0, count, misc) fills, for
// the G candidates e0.. (those < count), misc + c * kMisc with xs^T[24][8]
// then xb^T[24][8] (row 23 of xb^T and padding rows zero) and may use
// __syncthreads; it is called by every thread after a CTA barrier.
template <class Stage>
__device__ __forceinline__ void pacm_h64_body(int S, int B, const int64_t* __restrict__ count_dev, int64_t k_max,
                                              const double* __restrict__ params, double* __restrict__ score_out,
                                              Stage stage) {
  using namespace f64;
  if (threadIdx.x == 0) atomicMin(&g_h64_ns[0], gtimer64());
  extern __shared__ __align__(128) double smf[];
  __shared__ __align__(8) uint64_t mb[3];
  __shared__ double etab[32];
  if (threadIdx.x < 32) etab[threadIdx.x] = kExp2Tab[threadIdx.x];  // read after the staging barrier
  double* WA = smf;
  double* ZE = WA + kWA;             // [G][z1 | e], each [H][R]
  double* QKV = ZE + G * kZE;        // [G][q | k | v]; W1 | We during phase 1
  double* MISC = QKV + G * kQKV;     // [G][kMisc]
  const int t = threadIdx.x;
  const Params64 P = split_params(params, H);
  auto load_w1e = [&]() {  // QKV region <- W1 | We
    tc::fence_async_smem();
    tc::mbar_expect_tx(&mb[0], (24 + 23) * H * 8);
    tc::bulk_g2s(QKV, P.w1, 24 * H * 8, &mb[0]);
    tc::bulk_g2s(QKV + 24 * H, P.we, 23 * H * 8, &mb[0]);
  };
  auto load_wa = [&]() {  // WA <- W2 | Wq | Wk | Wv
    tc::fence_async_smem();
    tc::mbar_expect_tx(&mb[1], 4 * H * H * 8);
    tc::bulk_g2s(WA, P.w2, H * H * 8, &mb[1]);
    tc::bulk_g2s(WA + H * H, P.wq, H * H * 8, &mb[1]);
    tc::bulk_g2s(WA + 2 * H * H, P.wk, H * H * 8, &mb[1]);
    tc::bulk_g2s(WA + 3 * H * H, P.wv, H * H * 8, &mb[1]);
  };
  // the weights do not depend on the preceding kernel (they were loaded before
  // it ran): their bulk copies start before the grid-dependency wait, so
  // under programmatic dependent launch they overlap the selector's tail
  if (t == 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) tc::mbar_init(&mb[i], 1);
    tc::fence_mbar_init();
    load_w1e();
    load_wa();
  }
  pdl_wait();  // the drafted set and its count come from the preceding kernel
  if (threadIdx.x == 0) atomicMin(&g_h64_ns[1], gtimer64()), atomicMax(&g_h64_ns[2], gtimer64());
  int64_t count = k_max;
  if (count_dev) count = *count_dev < k_max ? *count_dev : k_max;
  if ((int64_t)blockIdx.x * G >= count) {  // no candidates: the weight copies must land before exit
    if (t == 0) tc::mbar_wait(&mb[0], 0), tc::mbar_wait(&mb[1], 0);
    return;
  }
  const double scale = __ddiv_rn(1.0, sqrt((double)H));  // ranker.cpp:179
  const double inv_n = __ddiv_rn(1.0, (double)B);        // ranker.cpp:198
  // dense-phase role: quarter q of the threads, candidate c, column pair (jp, jp + 32)
  const int q4 = t >> 7, c = (t >> 5) & 3, jp = t & 31;
  // attention / head role: candidate ch, head column / feature jh
  const int ch = (t >> 6) & 3, jh = t & 63;
  uint32_t par = 0;
  for (int64_t e0 = (int64_t)blockIdx.x * G; e0 < count; e0 += (int64_t)gridDim.x * G, par ^= 1u) {
    const bool more = e0 + (int64_t)gridDim.x * G < count;
    const bool live = e0 + c < count;        // dense roles
    const bool live_h = e0 + ch < count;     // attention / head roles
    double* z1 = ZE + c * kZE;
    double* em = z1 + H * R;
    double* misc = MISC + c * kMisc;
    // ---- the feature rows, transposed: xs^T[k][r], xb^T[k][r] (zero padded)
    H64_MARK(0, 0);
    __syncthreads();  // the previous pass' misc readers are done
    stage(e0, count, MISC);
    if (t < H) QKV[47 * H + t] = 0.0;  // We row 23 (outside the bulk copy)
    __syncthreads();
    H64_MARK(1, 0);
    // ---- phase 1: statement layer 1 | block embedding (ranker.cpp:165-169)
    tc::mbar_wait(&mb[0], par);
    H64_MARK(2, 0);
    // pre-activations (+ bias) first; the tanh of both layers is spread over
    // all 512 threads below (a thread's own 16 would serialise on registers)
    // one code path for both layers (instruction-cache footprint): the
    // embedding's 24th k step multiplies a zero activation by a zero weight row
    if (live && q4 < 2)
      tile8x2<24>(misc + q4 * 24 * 8, QKV + q4 * 24 * H, q4 ? P.be : P.b1, false, 8, q4 ? em : z1, jp);
    H64_MARK(3, 0);
    __syncthreads();
    {  // z1 rows < S, e rows < B: tanh in place, 8 independent per thread
      double zv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) zv[u] = ZE[t + u * T];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int v = t + u * T, cc = v / (2 * H * R), w = v - cc * (2 * H * R), r = w & 7;
        if (e0 + cc < count && r < (w < H * R ? S : B)) ZE[v] = tanh64t(zv[u], etab);
      }
    }
    __syncthreads();
    H64_MARK(4, 0);
    // ---- phase 2: statement layer 2 (+ mean-pool) | Q | K | V (ranker.cpp:166, 173-175)
    tc::mbar_wait(&mb[1], par);
    H64_MARK(5, 0);
    double* qm = QKV + c * kQKV;
    if (live) {
      // one code path for the four layers: S2 reads z1 and, z1[c] being read
      // only by this warp, writes its pre-activations back over it once every
      // lane is done (tanh + pool run in phase 3); Q, K, V read e
      const double* bias = q4 == 0 ? P.b2 : q4 == 1 ? P.bq : q4 == 2 ? P.bk : P.bv;
      double a[2][8];
      const double* const Wp[2] = {WA + q4 * H * H, WA + q4 * H * H + 32};
      chains8<H, 2, 8>(q4 ? em : z1, Wp, jp, a);
      __syncwarp();
      double* dst = q4 ? qm + (q4 - 1) * H * R : z1;
      store8(a[0], __ldg(bias + jp), false, 8, dst, jp);
      store8(a[1], __ldg(bias + jp + 32), false, 8, dst, jp + 32);
    }
    H64_MARK(6, 0);
    H64_MARK(7, 384);
    H64_MARK(16, 128);
    H64_MARK(17, 256);
    __syncthreads();
    H64_MARK(8, 0);
    if (t == 0) {  // WA <- head layer 1 (2h x h)
      tc::fence_async_smem();
      tc::mbar_expect_tx(&mb[2], 2 * H * H * 8);
      tc::bulk_g2s(WA, P.hw1, 2 * H * H * 8, &mb[2]);
    }
    // ---- phase 3
    double* mh = MISC + ch * kMisc;  // pr [8][8] | cat [128] | prod [64]
    const double* qh = QKV + ch * kQKV;
    double gacc = 0.0;  // head layer 1 chain of (ch, jh), threads 0-255
    if (t < 256) {
      if (live_h) {  // z2 = tanh(pre-activation), concat[j] = sum_i z2[i][j], i ascending (ranker.cpp:166, 196-197)
        const double* zp = ZE + ch * kZE + jh * 8;
        double z2[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) z2[r] = r < S ? tanh64t(zp[r], etab) : 0.0;
        double pool = 0.0;
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if (r < S) pool = __dadd_rn(pool, z2[r]);
        mh[64 + jh] = pool;
      }
      named_bar(3, 256);
      // head layer 1, k = 0..63 (the pooled statement half)
      tc::mbar_wait(&mb[2], par);
      H64_MARK(9, 0);
      if (live_h) gacc = chain64(0.0, mh + 64, 1, WA + jh, H);
      H64_MARK(10, 0);
    } else {
      const int i = (jh >> 3) & 7, i2 = jh & 7;
      const bool ok = live_h && i < B && i2 < B;
      // logits (matmul_nt, ranker.cpp:102-111): full dot product from +0.0, then scaled
      const double l = __dmul_rn(chain64(0.0, qh + i, 8, qh + H * R + i2, 8), scale);
      // softmax row i (ranker.cpp:181-191): max, exp(l - max), sequential sum, divide
      double mx = ok ? l : -1.0e308;
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o, 8));
      const double ex = ok ? exp64t(__dadd_rn(l, -mx), etab) : 0.0;
      double sum = 0.0;
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) {
        const double eq = __shfl_sync(0xffffffffu, ex, qq, 8);
        if (qq < B) sum = __dadd_rn(sum, eq);
      }
      if (ok) mh[i * 8 + i2] = __ddiv_rn(ex, sum);
      H64_MARK(11, 256);
      named_bar(1, 256);
      // ---- phase 4: PV (matmul, ranker.cpp:113-122) + attention mean-pool (ranker.cpp:198-200)
      if (live_h) {
        double vr[8];
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const double2 x = *(const double2*)(qh + 2 * H * R + jh * 8 + 2 * qq);
          vr[2 * qq] = x.x, vr[2 * qq + 1] = x.y;
        }
        double pool = 0.0;
        for (int ii = 0; ii < B; ++ii) {
          double a = 0.0;
#pragma unroll
          for (int r = 0; r < 8; ++r)
            if (r < B) a = __fma_rn(mh[ii * 8 + r], vr[r], a);
          pool = __fma_rn(a, inv_n, pool);
        }
        mh[64 + H + jh] = pool;
      }
      H64_MARK(12, 256);
    }
    __syncthreads();
    H64_MARK(13, 0);
    if (t == 256 && more) load_w1e();  // q, k, v consumed: next pass' W1 | We
    // ---- phase 5: head layer 1, k = 64..127, + bias, tanh; head layer 2 (ranker.cpp:202-204)
    if (t < 256) {
      if (live_h) {
        gacc = chain64(gacc, mh + 64 + H, 1, WA + H * H + jh, H);
        const double g = tanh64t(__dadd_rn(gacc, __ldg(P.hb1 + jh)), etab);
        mh[192 + jh] = __dmul_rn(g, __ldg(P.hw2 + jh));
      }
      H64_MARK(14, 0);
      named_bar(2, 256);
      if (t == 0 && more) load_wa();  // head weights consumed: next pass' W2 | Wq | Wk | Wv
      if (live_h && jh == 0) {  // one chain over j ascending
        double pv[H];
#pragma unroll
        for (int qq = 0; qq < H; qq += 2) {
          const double2 x = *(const double2*)(mh + 192 + qq);
          pv[qq] = x.x, pv[qq + 1] = x.y;
        }
        double sacc = 0.0;
#pragma unroll
        for (int qq = 0; qq < H; ++qq) sacc = __dadd_rn(sacc, pv[qq]);
        score_out[e0 + ch] = __dadd_rn(sacc, __ldg(P.hb2));
        H64_MARK(15, 0);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&g_h64_ns[3], gtimer64());
}

}  // namespace tt

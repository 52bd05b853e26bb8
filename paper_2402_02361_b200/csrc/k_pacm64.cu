// k_pacm64.cu — K3-fp64: PaCM forward on CUDA cores ("parity mode").
//
// Restates run_forward (ranker.cpp:159-209) on fp64 feature rows produced
// by k_feat_rows, with the reference's exact accumulation order: affine()
// (ranker.cpp:59-75) accumulates k = 0..m-1 from +0.0 and adds the bias
// last (its skip of zero inputs cannot change a finite sum that starts at
// +0.0); matmul_nt's logits are full dot products scaled afterwards;
// softmax subtracts the row max and divides by the sequential sum; pooling
// sums rows in order. No FMA (__dmul_rn/__dadd_rn), so scores agree with
// the reference to the last bit except where CUDA's fp64 tanh/exp differ
// from glibc by an ulp.
//
// Design: the round scores K = 512 candidates, ~3.5 per SM, and the fp64
// pipe (64 DMUL/DADD lanes per SM) bounds the whole set at ~9 us, while the
// certification rescoring of a few candidates is bound by one candidate's
// dependent chain. One CTA of 128 threads per candidate, up to three per
// SM. Activations are stored transposed, X^T[k][row] (rows padded to a
// multiple of 4), so a thread owns one output column for a group of 4 rows:
// each k step is one shared-memory weight load, two 16-byte activation loads
// and 4 independent mul/add chains (ILP 4, every weight reused 4x). The
// layer weights (<= 32 KB each at h = 64: W1, W2, We, Wq, Wk, Wv and the
// head's W1 in two halves) are staged into shared memory by 1-D bulk TMA
// copies, double buffered, so the next layer's weights stream in while the
// current layer computes. A device-side sublist restricts scoring to the
// certification band of the tensor-core path.
#include <cstdint>

#include "tt_kernels.h"
#include "tt_pacm64.cuh"
#include "tt_tc.cuh"

namespace tt {


// Y^T[j][i] = act(init^T[j][i] + sum_k X^T[k][i] * W[k][j] + b[j]) for rows
// i < pad4(n), columns j < q, in the reference's order (k ascending from
// +0.0, bias last). init == nullptr starts from +0.0; b == nullptr stores
// the partial sum (a split k range continues from it bit-exactly). Padding
// rows compute harmless finite values that no consumer reads.
template <int RG, int T>
__device__ __forceinline__ void dense64(int lt, const double* __restrict__ xt, int ldx, int n, int m,
                                        const double* __restrict__ W, int q, const double* __restrict__ init,
                                        const double* __restrict__ b, bool act, double* __restrict__ yt, int ldy) {
  const int groups = (n + RG - 1) / RG;
  for (int item = lt; item < q * groups; item += T) {
    const int j = item % q, r0 = (item / q) * RG;
    double a[RG];
#pragma unroll
    for (int r = 0; r < RG; ++r) a[r] = init ? init[j * ldy + r0 + r] : 0.0;
    const double* xp = xt + r0;
#pragma unroll 4
    for (int k = 0; k < m; ++k) {
      const double w = W[k * q + j];
      const double2 x01 = *(const double2*)(xp + k * ldx);
      a[0] = __dadd_rn(a[0], __dmul_rn(x01.x, w));
      a[1] = __dadd_rn(a[1], __dmul_rn(x01.y, w));
      if constexpr (RG == 4) {
        const double2 x23 = *(const double2*)(xp + k * ldx + 2);
        a[2] = __dadd_rn(a[2], __dmul_rn(x23.x, w));
        a[3] = __dadd_rn(a[3], __dmul_rn(x23.y, w));
      }
    }
    const double bj = b ? __ldg(b + j) : 0.0;
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      double z = a[r];
      if (b) {
        z = __dadd_rn(z, bj);
        if (act) z = tanh64(z);
      }
      yt[j * ldy + r0 + r] = z;
    }
  }
}

// y[j] = act(init[j] + sum_{k<m} x[k] * W[k][j] (+ b[j])) for one row.
template <int T>
__device__ __forceinline__ void dense_row64(int lt, const double* __restrict__ x, int m, const double* __restrict__ W,
                                            int q, const double* init, const double* __restrict__ b, bool act,
                                            double* y) {
  for (int j = lt; j < q; j += T) {
    double a = init[j];
#pragma unroll 8
    for (int k = 0; k < m; ++k) a = __dadd_rn(a, __dmul_rn(x[k], W[k * q + j]));
    if (b) {
      a = __dadd_rn(a, __ldg(b + j));
      if (act) a = tanh64(a);
    }
    y[j] = a;
  }
}

// shared-memory doubles: transposed activations (rows padded to 4)
__host__ __device__ inline size_t act64_doubles(int S, int B, int h) {
  const int sp = pad4(S), bp = pad4(B);
  // xs^T, xb^T, z1^T, z2^T, e^T, q^T, k^T, v^T, ao^T, pr, cat, gp, g, hw2
  const size_t d = (size_t)24 * sp + 23 * bp + 2 * h * sp + 5 * h * bp + B * B + 2 * h + 2 * h + h + 2;
  return (d + 3) & ~(size_t)3;  // keeps every group's 16-byte activation loads aligned
}
__host__ __device__ inline size_t wbuf64_doubles(int h) { return (size_t)(h * h > 24 * h ? h * h : 24 * h); }

// weight blocks streamed per candidate, in consumption order
struct WStages {
  const double* src[8];
  uint32_t bytes[8];
  int n;
};

__device__ __forceinline__ WStages weight_stages(const Params64& P, int h, bool identity) {
  WStages w;
  int n = 0;
  auto add = [&](const double* p, int count) { w.src[n] = p, w.bytes[n] = (uint32_t)count * 8u, ++n; };
  add(P.w1, 24 * h);
  add(P.w2, h * h);
  add(P.we, 23 * h);
  if (!identity) add(P.wq, h * h), add(P.wk, h * h), add(P.wv, h * h);
  add(P.hw1, h * h);
  add(P.hw1 + h * h, h * h);
  w.n = n;
  return w;
}

// clock64 marks of CTA 0, thread 0, first pass (phase probe, ttdbg_pacm64_clocks,
// tools/probe_pacm64.py)
__device__ long long g_clk_p64[24];
#define P64_MARK(i)                                                   \
  do {                                                                \
    if (blockIdx.x == 0 && t == 0 && e0 == 0) g_clk_p64[i] = clock64(); \
  } while (0)

// G candidate groups of kT64 threads per CTA share each staged weight block
// (G = 4 for whole drafted sets, 1 for the short certification sublists).
template <int RG, int kT64>
__global__ void __launch_bounds__(4 * kT64) k_pacm64(const double* __restrict__ stmt,
                                                     const double* __restrict__ block, int n_stmt, int n_block,
                                                     const int64_t* __restrict__ count_dev, int64_t k_max,
                                                     const int32_t* __restrict__ sublist,
                                                     const int* __restrict__ sublist_count,
                                                     const double* __restrict__ params, int h, int identity,
                                                     double* __restrict__ score_out) {
  pdl_wait();  // feature rows come from the preceding kernel
  extern __shared__ __align__(128) double sm64[];
  __shared__ __align__(8) uint64_t bars[2];
  const int S = n_stmt, B = n_block, t = threadIdx.x;
  const int G = blockDim.x / kT64, grp = t / kT64, lt = t - grp * kT64;
  const int sp = pad4(S), bp = pad4(B);
  const int wd = (int)wbuf64_doubles(h);
  double* xs = sm64 + 2 * wd + (size_t)grp * act64_doubles(S, B, h);  // [24][sp]
  double* xb = xs + 24 * sp;    // [23][bp]
  double* z1 = xb + 23 * bp;    // [h][sp]
  double* z2 = z1 + h * sp;     // [h][sp]
  double* e = z2 + h * sp;      // [h][bp]
  double* qm = e + h * bp;      // [h][bp]
  double* km = qm + h * bp;
  double* vm = km + h * bp;
  double* ao = vm + h * bp;
  double* pr = ao + h * bp;     // [B][B]
  double* cat = pr + B * B;     // [2h]
  double* gp = cat + 2 * h;     // [h]
  double* g = gp + h;           // [h]
  double* hw2s = g + h;         // [h] head layer-2 weights (staged per pass)
  const Params64 P = split_params(params, h);
  const WStages W = weight_stages(P, h, identity != 0);
  int64_t count = k_max;
  if (sublist) count = *sublist_count;
  else if (count_dev) count = *count_dev < k_max ? *count_dev : k_max;
  if ((int64_t)blockIdx.x * G >= count) return;
  if (t == 0) {
    tc::mbar_init(&bars[0], 1);
    tc::mbar_init(&bars[1], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  // gs counts the weight stages this CTA consumed; stage s of the current
  // pass lives in buffer (base + s) & 1 and completes phase ((base + s) >> 1) & 1
  uint32_t gs = 0, base = 0;
  auto issue = [&](int s) {
    if (t == 0 && s < W.n) {
      const uint32_t bb = (base + (uint32_t)s) & 1u;
      tc::fence_async_smem();
      tc::mbar_expect_tx(&bars[bb], W.bytes[s]);
      tc::bulk_g2s(sm64 + bb * wd, W.src[s], W.bytes[s], &bars[bb]);
    }
  };
  for (int64_t e0 = (int64_t)blockIdx.x * G; e0 < count; e0 += (int64_t)gridDim.x * G) {
    const int64_t ent = e0 + grp;
    const bool live = ent < count;
    const int64_t pos = live ? (sublist ? sublist[ent] : ent) : 0;
    P64_MARK(0);
    base = gs;
    issue(0);
    issue(1);
    if (live) {  // feature rows -> transposed, zero padded
      for (int u = lt; u < 24 * sp; u += kT64) {
        const int k = u / sp, i = u - k * sp;
        xs[u] = i < S ? stmt[(pos * S + i) * 24 + k] : 0.0;
      }
      for (int u = lt; u < 23 * bp; u += kT64) {
        const int k = u / bp, i = u - k * bp;
        xb[u] = i < B ? block[(pos * B + i) * 23 + k] : 0.0;
      }
      for (int u = lt; u < h; u += kT64) hw2s[u] = __ldg(P.hw2 + u);
    }
    __syncthreads();
    P64_MARK(1);
    int s = 0;
    // one weight stage: wait for its buffer, compute, release, prefetch s + 2
#define TT_STAGE(CALL)                                 \
  do {                                                 \
    tc::mbar_wait(&bars[gs & 1u], (gs >> 1) & 1u);     \
    const double* Wm = sm64 + (gs & 1u) * wd;          \
    P64_MARK(2 + 2 * s);                               \
    if (live) CALL;                                    \
    __syncthreads();                                   \
    P64_MARK(3 + 2 * s);                               \
    ++gs;                                              \
    issue(s + 2);                                      \
    ++s;                                               \
  } while (0)
    TT_STAGE((dense64<RG, kT64>(lt, xs, sp, S, 24, Wm, h, nullptr, P.b1, true, z1, sp)));
    TT_STAGE((dense64<RG, kT64>(lt, z1, sp, S, h, Wm, h, nullptr, P.b2, true, z2, sp)));
    TT_STAGE((dense64<RG, kT64>(lt, xb, bp, B, 23, Wm, h, nullptr, P.be, true, e, bp)));
    const double* pooled = e;
    if (!identity) {
      TT_STAGE((dense64<RG, kT64>(lt, e, bp, B, h, Wm, h, nullptr, P.bq, false, qm, bp)));
      TT_STAGE((dense64<RG, kT64>(lt, e, bp, B, h, Wm, h, nullptr, P.bk, false, km, bp)));
      TT_STAGE((dense64<RG, kT64>(lt, e, bp, B, h, Wm, h, nullptr, P.bv, false, vm, bp)));
      const double scale = __ddiv_rn(1.0, sqrt((double)h));
      if (live)
        for (int u = lt; u < B * B; u += kT64) {  // matmul_nt (ranker.cpp:102-111), then scale
          const int i = u / B, j = u - (u / B) * B;
          double acc = 0.0;
          int c = 0;
          for (; c + 16 <= h; c += 16) {  // 16 products staged in registers, then the chain in c order
            double pq[16];
#pragma unroll
            for (int v = 0; v < 16; ++v) pq[v] = __dmul_rn(qm[(c + v) * bp + i], km[(c + v) * bp + j]);
#pragma unroll
            for (int v = 0; v < 16; ++v) acc = __dadd_rn(acc, pq[v]);
          }
          for (; c < h; ++c) acc = __dadd_rn(acc, __dmul_rn(qm[c * bp + i], km[c * bp + j]));
          pr[u] = __dmul_rn(acc, scale);
        }
      __syncthreads();
      P64_MARK(19);
      if (live && lt < B) {  // softmax rows (ranker.cpp:181-191)
        double* row = pr + lt * B;
        double mx = row[0];
        for (int j = 1; j < B; ++j) mx = row[j] > mx ? row[j] : mx;
        double sum = 0.0;
        for (int j = 0; j < B; ++j) {
          const double ex = exp64(__dadd_rn(row[j], -mx));
          row[j] = ex;
          sum = __dadd_rn(sum, ex);
        }
        for (int j = 0; j < B; ++j) row[j] = __ddiv_rn(row[j], sum);
      }
      __syncthreads();
      P64_MARK(20);
      if (live)
        for (int u0 = lt; u0 < B * h; u0 += 4 * kT64) {  // matmul (ranker.cpp:113-122), 4 outputs interleaved
          double acc[4] = {0.0, 0.0, 0.0, 0.0};
          int jj[4], ii[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const int u = u0 + x * kT64 < B * h ? u0 + x * kT64 : u0;
            jj[x] = u / B, ii[x] = u - jj[x] * B;
          }
          for (int r = 0; r < B; ++r) {
#pragma unroll
            for (int x = 0; x < 4; ++x)
              acc[x] = __dadd_rn(acc[x], __dmul_rn(pr[ii[x] * B + r], vm[jj[x] * bp + r]));
          }
#pragma unroll
          for (int x = 0; x < 4; ++x)
            if (u0 + x * kT64 < B * h) ao[jj[x] * bp + ii[x]] = acc[x];
        }
      __syncthreads();
      P64_MARK(21);
      pooled = ao;
    }
    const double inv_n = __ddiv_rn(1.0, (double)B);
    if (live)
      for (int j = lt; j < 2 * h; j += kT64) {  // concat (ranker.cpp:196-200)
        double v = 0.0;
        if (j < h) {
          for (int i = 0; i < S; ++i) v = __dadd_rn(v, z2[j * sp + i]);
        } else {
          for (int i = 0; i < B; ++i) v = __dadd_rn(v, __dmul_rn(pooled[(j - h) * bp + i], inv_n));
        }
        cat[j] = v;
        if (j < h) gp[j] = 0.0;
      }
    __syncthreads();
    P64_MARK(22);
    // head layer 1 over k = 0..2h-1 (1 row), split in two weight stages
    TT_STAGE((dense_row64<kT64>(lt, cat, h, Wm, h, gp, nullptr, false, gp)));
    TT_STAGE((dense_row64<kT64>(lt, cat + h, h, Wm, h, gp, P.hb1, true, g)));
#undef TT_STAGE
    if (live && lt == 0) {  // head layer 2: 1 x h -> 1, one chain
      double acc = 0.0;
#pragma unroll 8
      for (int k = 0; k < h; ++k) acc = __dadd_rn(acc, __dmul_rn(g[k], hw2s[k]));
      score_out[pos] = __dadd_rn(acc, __ldg(P.hb2));
    }
    __syncthreads();
    P64_MARK(18);
  }
}

// Throughput kernel over fp64 feature rows in global memory (stmt [pos][S][24],
// block [pos][B][23], the tt_features layout).
__global__ void __launch_bounds__(f64::T, 1) k_pacm64_h64(const double* __restrict__ stmt,
                                                         const double* __restrict__ block, int S, int B,
                                                         const int64_t* __restrict__ count_dev, int64_t k_max,
                                                         const double* __restrict__ params,
                                                         double* __restrict__ score_out) {
  using namespace f64;
  pacm_h64_body(S, B, count_dev, k_max, params, score_out, [&](int64_t e0, int64_t count, double* MISC) {
    for (int v = threadIdx.x; v < G * (24 + 24) * 8; v += T) {  // xb^T row 23 = 0: the embedding runs 24 k steps
      const int cc = v / ((24 + 24) * 8), w = v - cc * (24 + 24) * 8;
      const int64_t e = e0 + cc;
      double x = 0.0;
      if (e < count) {
        if (w < 24 * 8) {
          const int k = w >> 3, r = w & 7;
          if (r < S) x = stmt[(e * S + r) * 24 + k];
        } else {
          const int k = (w - 24 * 8) >> 3, r = w & 7;
          if (r < B && k < 23) x = block[(e * B + r) * 23 + k];
        }
      }
      MISC[cc * kMisc + w] = x;
    }
  });
}

int launch_pacm64(const double* stmt, const double* block, int n_stmt, int n_block, const int64_t* count_dev,
                  int64_t k_max, const int32_t* sublist, const int* sublist_count, const double* params, int h,
                  int attention_identity, double* score_out, cudaStream_t st) {
  if (k_max <= 0) return 0;
  if (h % 2) return -1;  // bulk copies need 16-byte aligned weight blocks
  const size_t wbytes = 2 * wbuf64_doubles(h) * sizeof(double);
  const size_t abytes = act64_doubles(n_stmt, n_block, h) * sizeof(double);
  const size_t budget = 227 * 1024 - 64;
  if (wbytes + abytes > budget) return -1;
  int G = (int)((budget - wbytes) / abytes);
  G = G > 4 ? 4 : G;
  if (sublist) G = 1;  // a few candidates: one per CTA, latency first
  const size_t sm = wbytes + (size_t)G * abytes;
  const int64_t ctas = (k_max + G - 1) / G, cap = sublist ? 64 : 8 * 148;
  const unsigned grid = (unsigned)(ctas < cap ? ctas : cap);
  auto go = [&](auto kern, int threads) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    tt::note_launch();
    launch_pdl(kern, dim3(grid), dim3(G * threads), sm, st, stmt, block, n_stmt, n_block, count_dev, k_max, sublist,
               sublist_count, params, h, attention_identity, score_out);
  };
  if (!sublist && !attention_identity && h == f64::H && n_stmt <= 8 && n_block <= 8) {
    const int64_t ctas = (k_max + f64::G - 1) / f64::G;
    cudaFuncSetAttribute(k_pacm64_h64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f64::kSmem);
    tt::note_launch();
    launch_pdl(k_pacm64_h64, dim3((unsigned)(ctas < 148 ? ctas : 148)), dim3(f64::T), f64::kSmem, st, stmt, block,
               n_stmt, n_block, count_dev, k_max, params, score_out);
    return 0;
  }
  // whole drafted sets: 4 chains per thread, 128 threads per candidate (throughput);
  // certification sublists: 2 chains per thread, 256 threads per candidate (latency)
  if (sublist) go(k_pacm64<2, 256>, 256);
  else go(k_pacm64<4, 128>, 128);
  return 0;
}

}  // namespace tt

extern "C" int ttdbg_pacm64_clocks(long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, tt::g_clk_p64, sizeof(long long) * (n < 24 ? n : 24));
}
extern "C" int ttdbg_pacm64_h64_clocks(long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, tt::g_clk_h64, sizeof(long long) * (n < 24 ? n : 24));
}
extern "C" int ttdbg_pacm64_h64_span(unsigned long long* out, int reset) {
  if (reset) {
    const unsigned long long init[4] = {~0ull, ~0ull, 0ull, 0ull};
    return (int)cudaMemcpyToSymbol(tt::g_h64_ns, init, sizeof(init));
  }
  return (int)cudaMemcpyFromSymbol(out, tt::g_h64_ns, sizeof(unsigned long long) * 4);
}

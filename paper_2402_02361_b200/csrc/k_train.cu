// k_train.cu — PaCM training on the device: the per-sample
// forward with caches, score_backward (ranker.cpp:211-261, 383-389) and the
// gradient accumulation of train() (ranker.cpp:459-512), in fp64.
//
// Ordering is what makes GD training reproducible, so it follows the
// reference exactly where sums are formed:
//   * per sample (one CTA each), every dot product accumulates from +0.0 in
//     the reference's index order (affine(), matmul, matmul_nt, matmul_tn,
//     affine_backward's dx), tanh' = dy * (1 - y*y), no FMA contraction;
//   * the gradient of every parameter element is accumulated by ONE thread
//     over samples (batch order, samples with dscore == 0 skipped, as train()
//     skips their score_backward) and, within a sample, over rows in order —
//     the sequence train()'s shared grads tensors see.
// The reference skips zero inputs inside those sums; adding x * 0 = ±0 to a
// running sum that starts at +0.0 never changes it, so the skips are
// dropped. tanh/exp are CUDA's (ulp-level differences from glibc).
#include <cstdint>

#include "tt_kernels.h"

namespace tt {

struct TrainLayout {  // per-sample slot offsets (doubles)
  int S, B, h;
  int xs, xb, z1, z2, e, q, k, v, p, ao, cat, g, score;  // forward caches
  int dy2, dy1, dyq, dyk, dyv, dye, dyh, ds;              // backward: each affine layer's dy, dscore
  int size;
};

__host__ __device__ inline TrainLayout train_layout(int S, int B, int h) {
  TrainLayout L;
  L.S = S, L.B = B, L.h = h;
  int o = 0;
  auto take = [&](int n) {
    const int r = o;
    o += n;
    return r;
  };
  L.xs = take(S * 24), L.xb = take(B * 23), L.z1 = take(S * h), L.z2 = take(S * h), L.e = take(B * h);
  L.q = take(B * h), L.k = take(B * h), L.v = take(B * h), L.p = take(B * B), L.ao = take(B * h);
  L.cat = take(2 * h), L.g = take(h), L.score = take(1);
  L.dy2 = take(S * h), L.dy1 = take(S * h), L.dyq = take(B * h), L.dyk = take(B * h), L.dyv = take(B * h);
  L.dye = take(B * h), L.dyh = take(h), L.ds = take(1);
  L.size = (o + 1) & ~1;
  return L;
}

size_t train_slot_doubles(int S, int B, int h) { return (size_t)train_layout(S, B, h).size; }

struct TP {  // parameter tensors (for_each_tensor order, ranker.cpp:339-356)
  const double *w1, *b1, *w2, *b2, *we, *be, *wq, *bq, *wk, *bk, *wv, *bv, *hw1, *hb1, *hw2, *hb2;
};
__device__ __forceinline__ TP tp_of(const double* p, int h) {
  TP P;
  P.w1 = p, P.b1 = P.w1 + 24 * h, P.w2 = P.b1 + h, P.b2 = P.w2 + h * h;
  P.we = P.b2 + h, P.be = P.we + 23 * h, P.wq = P.be + h, P.bq = P.wq + h * h;
  P.wk = P.bq + h, P.bk = P.wk + h * h, P.wv = P.bk + h, P.bv = P.wv + h * h;
  P.hw1 = P.bv + h, P.hb1 = P.hw1 + 2 * h * h, P.hw2 = P.hb1 + h, P.hb2 = P.hw2 + h;
  return P;
}

// y[i][j] = act(sum_k x[i][k] W[k][j] + b[j]), k ascending from +0.0, bias last
__device__ void t_affine(const double* x, int n, int m, const double* W, const double* b, int q, bool act, double* y) {
  for (int o = threadIdx.x; o < n * q; o += blockDim.x) {
    const int i = o / q, j = o - i * q;
    double a = 0.0;
    for (int k = 0; k < m; ++k) a = __dadd_rn(a, __dmul_rn(x[i * m + k], W[k * q + j]));
    a = __dadd_rn(a, b[j]);
    y[o] = act ? tanh(a) : a;
  }
  __syncthreads();
}

// dx[i][k] = sum_j dy[i][j] W[k][j], j ascending (affine_backward's dx, ranker.cpp:93-98)
__device__ void t_dx(const double* dy, int n, int q, const double* W, int m, double* dx) {
  for (int o = threadIdx.x; o < n * m; o += blockDim.x) {
    const int i = o / m, k = o - i * m;
    double a = 0.0;
    for (int j = 0; j < q; ++j) a = __dadd_rn(a, __dmul_rn(dy[i * q + j], W[k * q + j]));
    dx[o] = a;
  }
  __syncthreads();
}

// Forward (run_forward, ranker.cpp:159-209) of sample e = rows of record
// list[e], caches into its slot; score written to scores[e].
__global__ void __launch_bounds__(128) k_train_fwd(const double* __restrict__ stmt, const double* __restrict__ block,
                                                   int S, int B, const int32_t* __restrict__ list, int m,
                                                   const double* __restrict__ params, int h, int identity,
                                                   double* __restrict__ slots, double* __restrict__ scores) {
  const TrainLayout L = train_layout(S, B, h);
  const TP P = tp_of(params, h);
  const int t = threadIdx.x;
  for (int e = blockIdx.x; e < m; e += gridDim.x) {
    double* c = slots + (size_t)e * L.size;
    const int r = list ? list[e] : e;
    for (int u = t; u < S * 24; u += blockDim.x) c[L.xs + u] = stmt[(size_t)r * S * 24 + u];
    for (int u = t; u < B * 23; u += blockDim.x) c[L.xb + u] = block[(size_t)r * B * 23 + u];
    __syncthreads();
    t_affine(c + L.xs, S, 24, P.w1, P.b1, h, true, c + L.z1);
    t_affine(c + L.z1, S, h, P.w2, P.b2, h, true, c + L.z2);
    t_affine(c + L.xb, B, 23, P.we, P.be, h, true, c + L.e);
    const double* pooled = c + L.e;
    if (!identity) {
      t_affine(c + L.e, B, h, P.wq, P.bq, h, false, c + L.q);
      t_affine(c + L.e, B, h, P.wk, P.bk, h, false, c + L.k);
      t_affine(c + L.e, B, h, P.wv, P.bv, h, false, c + L.v);
      const double scale = __ddiv_rn(1.0, sqrt((double)h));
      for (int o = t; o < B * B; o += blockDim.x) {  // matmul_nt then scale
        const int i = o / B, j = o - i * B;
        double a = 0.0;
        for (int cc = 0; cc < h; ++cc) a = __dadd_rn(a, __dmul_rn(c[L.q + i * h + cc], c[L.k + j * h + cc]));
        c[L.p + o] = __dmul_rn(a, scale);
      }
      __syncthreads();
      if (t < B) {  // softmax rows
        double* row = c + L.p + t * B;
        double mx = row[0];
        for (int j = 1; j < B; ++j) mx = row[j] > mx ? row[j] : mx;
        double sum = 0.0;
        for (int j = 0; j < B; ++j) {
          const double ex = exp(__dadd_rn(row[j], -mx));
          row[j] = ex;
          sum = __dadd_rn(sum, ex);
        }
        for (int j = 0; j < B; ++j) row[j] = __ddiv_rn(row[j], sum);
      }
      __syncthreads();
      for (int o = t; o < B * h; o += blockDim.x) {  // matmul(probs, v)
        const int i = o / h, j = o - i * h;
        double a = 0.0;
        for (int r2 = 0; r2 < B; ++r2) a = __dadd_rn(a, __dmul_rn(c[L.p + i * B + r2], c[L.v + r2 * h + j]));
        c[L.ao + o] = a;
      }
      __syncthreads();
      pooled = c + L.ao;
    }
    const double inv_n = __ddiv_rn(1.0, (double)B);
    for (int j = t; j < 2 * h; j += blockDim.x) {
      double a = 0.0;
      if (j < h) {
        for (int i = 0; i < S; ++i) a = __dadd_rn(a, c[L.z2 + i * h + j]);
      } else {
        for (int i = 0; i < B; ++i) a = __dadd_rn(a, __dmul_rn(pooled[i * h + j - h], inv_n));
      }
      c[L.cat + j] = a;
    }
    __syncthreads();
    t_affine(c + L.cat, 1, 2 * h, P.hw1, P.hb1, h, true, c + L.g);
    if (t == 0) {
      double a = 0.0;
      for (int k = 0; k < h; ++k) a = __dadd_rn(a, __dmul_rn(c[L.g + k], P.hw2[k]));
      a = __dadd_rn(a, P.hb2[0]);
      c[L.score] = a;
      scores[e] = a;
    }
    __syncthreads();
  }
}

// run_backward (ranker.cpp:211-261) of sample e with dscore[e]: every affine
// layer's dy into the slot (the gradient sums read them in order later).
__global__ void __launch_bounds__(128) k_train_bwd(int S, int B, int m, const double* __restrict__ params, int h,
                                                   int identity, const double* __restrict__ dscore,
                                                   double* __restrict__ slots, double* __restrict__ work) {
  const TrainLayout L = train_layout(S, B, h);
  const TP P = tp_of(params, h);
  const int t = threadIdx.x;
  // per-CTA scratch: dconcat[2h], dz[max(S,B) * h] x 2, dprobs/dlogits [B*B] x 2, dx_q/k/v [B*h] x 3
  const int R = S > B ? S : B;
  const size_t wsz = (size_t)2 * h + 2 * R * h + 2 * B * B + 3 * B * h;
  double* w = work + blockIdx.x * wsz;
  double* dcat = w;
  double* dza = dcat + 2 * h;
  double* dzb = dza + R * h;
  double* dpr = dzb + R * h;
  double* dlg = dpr + B * B;
  double* dxq = dlg + B * B;
  double* dxk = dxq + B * h;
  double* dxv = dxk + B * h;
  for (int e = blockIdx.x; e < m; e += gridDim.x) {
    double* c = slots + (size_t)e * L.size;
    const double ds = dscore[e];
    if (t == 0) c[L.ds] = ds;
    if (ds == 0.0) continue;  // train() skips this sample's score_backward (uniform per CTA)
    // head: dg = hw2 * dscore; dy = dg * (1 - g^2)
    for (int j = t; j < h; j += blockDim.x) {
      const double gj = c[L.g + j];
      c[L.dyh + j] = __dmul_rn(__dmul_rn(P.hw2[j], ds), __dsub_rn(1.0, __dmul_rn(gj, gj)));
    }
    __syncthreads();
    t_dx(c + L.dyh, 1, h, P.hw1, 2 * h, dcat);
    // statement branch: dz2 rows = dconcat[0:h]
    for (int o = t; o < S * h; o += blockDim.x) {
      const int j = o % h;
      const double y = c[L.z2 + o];
      c[L.dy2 + o] = __dmul_rn(dcat[j], __dsub_rn(1.0, __dmul_rn(y, y)));
    }
    __syncthreads();
    t_dx(c + L.dy2, S, h, P.w2, h, dza);  // dz1
    for (int o = t; o < S * h; o += blockDim.x) {
      const double y = c[L.z1 + o];
      c[L.dy1 + o] = __dmul_rn(dza[o], __dsub_rn(1.0, __dmul_rn(y, y)));
    }
    // dataflow branch: dpool = dconcat[h:2h] * inv_n
    const double inv_n = __ddiv_rn(1.0, (double)B);
    for (int o = t; o < B * h; o += blockDim.x) dzb[o] = __dmul_rn(dcat[h + o % h], inv_n);
    __syncthreads();
    const double* dembed = dzb;
    if (!identity) {
      const double* pr = c + L.p;
      for (int o = t; o < B * B; o += blockDim.x) {  // dprobs = matmul_nt(dpool, v)
        const int i = o / B, j = o - i * B;
        double a = 0.0;
        for (int cc = 0; cc < h; ++cc) a = __dadd_rn(a, __dmul_rn(dzb[i * h + cc], c[L.v + j * h + cc]));
        dpr[o] = a;
      }
      for (int o = t; o < B * h; o += blockDim.x) {  // dv = matmul_tn(probs, dpool)
        const int kk = o / h, j = o - kk * h;
        double a = 0.0;
        for (int i = 0; i < B; ++i) a = __dadd_rn(a, __dmul_rn(pr[i * B + kk], dzb[i * h + j]));
        c[L.dyv + o] = a;
      }
      __syncthreads();
      const double scale = __ddiv_rn(1.0, sqrt((double)h));
      if (t < B) {  // softmax backward, then scale
        double dot = 0.0;
        for (int j = 0; j < B; ++j) dot = __dadd_rn(dot, __dmul_rn(dpr[t * B + j], pr[t * B + j]));
        for (int j = 0; j < B; ++j)
          dlg[t * B + j] = __dmul_rn(__dmul_rn(pr[t * B + j], __dsub_rn(dpr[t * B + j], dot)), scale);
      }
      __syncthreads();
      for (int o = t; o < B * h; o += blockDim.x) {
        const int i = o / h, cc = o - i * h;
        double aq = 0.0, ak = 0.0;
        for (int r2 = 0; r2 < B; ++r2) {
          aq = __dadd_rn(aq, __dmul_rn(dlg[i * B + r2], c[L.k + r2 * h + cc]));   // dq = matmul(dlogits, k)
          ak = __dadd_rn(ak, __dmul_rn(dlg[r2 * B + i], c[L.q + r2 * h + cc]));   // dk = matmul_tn(dlogits, q)
        }
        c[L.dyq + o] = aq;
        c[L.dyk + o] = ak;
      }
      __syncthreads();
      t_dx(c + L.dyq, B, h, P.wq, h, dxq);
      t_dx(c + L.dyk, B, h, P.wk, h, dxk);
      t_dx(c + L.dyv, B, h, P.wv, h, dxv);
      for (int o = t; o < B * h; o += blockDim.x) dzb[o] = __dadd_rn(dxq[o], __dadd_rn(dxk[o], dxv[o]));
      __syncthreads();
    }
    for (int o = t; o < B * h; o += blockDim.x) {
      const double y = c[L.e + o];
      c[L.dye + o] = __dmul_rn(dembed[o], __dsub_rn(1.0, __dmul_rn(y, y)));
    }
    __syncthreads();
  }
}

size_t train_work_doubles(int S, int B, int h, int ctas) {
  const int R = S > B ? S : B;
  return (size_t)ctas * ((size_t)2 * h + 2 * R * h + 2 * B * B + 3 * B * h);
}

// One thread per parameter element: its gradient summed over samples in
// batch order (skipping dscore == 0) and rows in order.
__global__ void __launch_bounds__(256) k_train_accum(int S, int B, int m, int h, int identity,
                                                     const double* __restrict__ slots, double* __restrict__ grads) {
  const TrainLayout L = train_layout(S, B, h);
  const int np = 24 * h + h + h * h + h + 23 * h + h + 3 * (h * h + h) + 2 * h * h + h + h + 1;
  for (int pidx = blockIdx.x * blockDim.x + threadIdx.x; pidx < np; pidx += gridDim.x * blockDim.x) {
    // locate (tensor, row, col)
    int o = pidx;
    int xo, dyo, rows, xm, col, krow;  // x offset/width, dy offset, row count, element coords
    bool bias = false, hw2 = false, hb2 = false;
    auto in = [&](int sz) {
      if (o < sz) return true;
      o -= sz;
      return false;
    };
    if (in(24 * h)) xo = L.xs, xm = 24, dyo = L.dy1, rows = S, krow = o / h, col = o % h;
    else if (in(h)) bias = true, dyo = L.dy1, rows = S, col = o;
    else if (in(h * h)) xo = L.z1, xm = h, dyo = L.dy2, rows = S, krow = o / h, col = o % h;
    else if (in(h)) bias = true, dyo = L.dy2, rows = S, col = o;
    else if (in(23 * h)) xo = L.xb, xm = 23, dyo = L.dye, rows = B, krow = o / h, col = o % h;
    else if (in(h)) bias = true, dyo = L.dye, rows = B, col = o;
    else if (in(h * h)) xo = L.e, xm = h, dyo = L.dyq, rows = B, krow = o / h, col = o % h;
    else if (in(h)) bias = true, dyo = L.dyq, rows = B, col = o;
    else if (in(h * h)) xo = L.e, xm = h, dyo = L.dyk, rows = B, krow = o / h, col = o % h;
    else if (in(h)) bias = true, dyo = L.dyk, rows = B, col = o;
    else if (in(h * h)) xo = L.e, xm = h, dyo = L.dyv, rows = B, krow = o / h, col = o % h;
    else if (in(h)) bias = true, dyo = L.dyv, rows = B, col = o;
    else if (in(2 * h * h)) xo = L.cat, xm = 2 * h, dyo = L.dyh, rows = 1, krow = o / h, col = o % h;
    else if (in(h)) bias = true, dyo = L.dyh, rows = 1, col = o;
    else if (in(h)) hw2 = true, col = o;
    else hb2 = true;
    const bool attn = pidx >= 24 * h + h + h * h + h + 23 * h + h && pidx < 24 * h + h + h * h + h + 23 * h + h +
                                                                          3 * (h * h + h);
    double g = 0.0;
    if (!(attn && identity)) {
      for (int e = 0; e < m; ++e) {
        const double* c = slots + (size_t)e * L.size;
        const double ds = c[L.ds];
        if (ds == 0.0) continue;
        if (hb2) {
          g = __dadd_rn(g, ds);
        } else if (hw2) {
          g = __dadd_rn(g, __dmul_rn(c[L.g + col], ds));
        } else if (bias) {
          for (int i = 0; i < rows; ++i) g = __dadd_rn(g, c[dyo + i * h + col]);
        } else {
          for (int i = 0; i < rows; ++i) g = __dadd_rn(g, __dmul_rn(c[xo + i * xm + krow], c[dyo + i * h + col]));
        }
      }
    }
    grads[pidx] = g;
  }
}

int launch_train_fwd(const double* stmt, const double* block, int S, int B, const int32_t* list, int m,
                     const double* params, int h, int identity, double* slots, double* scores, cudaStream_t st) {
  if (m <= 0) return 0;
  tt::note_launch();
  k_train_fwd<<<(unsigned)(m < 8 * 148 ? m : 8 * 148), 128, 0, st>>>(stmt, block, S, B, list, m, params, h, identity,
                                                                     slots, scores);
  return 0;
}

int launch_train_bwd(int S, int B, int m, const double* params, int h, int identity, const double* dscore,
                     double* slots, double* work, int ctas, cudaStream_t st) {
  if (m <= 0) return 0;
  tt::note_launch();
  k_train_bwd<<<(unsigned)(m < ctas ? m : ctas), 128, 0, st>>>(S, B, m, params, h, identity, dscore, slots, work);
  return 0;
}

int launch_train_accum(int S, int B, int m, int h, int identity, const double* slots, double* grads,
                       cudaStream_t st) {
  const int np = 24 * h + h + h * h + h + 23 * h + h + 3 * (h * h + h) + 2 * h * h + h + h + 1;
  tt::note_launch();
  k_train_accum<<<(np + 255) / 256, 256, 0, st>>>(S, B, m, h, identity, slots, grads);
  return 0;
}

}  // namespace tt

// k_verify.cu — the verify half of a round in ONE kernel for the tuner's
// model geometry: hybrid feature rows of the drafted candidates
// (extract_features, features.cpp:98-257) computed by the CTA that scores
// them, straight into its shared-memory operand staging, then the fp64 PaCM
// forward (run_forward, ranker.cpp:159-209) of tt_pacm64.cuh. Replaces
// k_feat_rows + k_pacm64_h64 (one launch and one HBM/L2 round trip of the
// feature rows fewer per round). Same arithmetic as both: scores are
// identical to the two-kernel path.
//
// Per pass of G = 4 candidates: lanes 0-3 of warp 0 derive each candidate's
// shared information (factors -> tile table -> symbols -> penalties); then
// warp w evaluates feature row w of the 4 candidates (warp-uniform row code,
// as k_feat_rows), 8 lanes per candidate sharing the row's log1p calls, and
// writes it transposed into the candidate's staging.
#include <cstdint>

#include "tt_features.cuh"
#include "tt_finish.cuh"
#include "tt_kernels.h"
#include "tt_pacm64.cuh"

namespace tt {

// Finish fused in (FinishArgs.record != nullptr): every candidate's identity
// is written next to its features (no side-stream identity kernel), and the
// last CTA to finish (ticket) runs select_top + the record gather
// (tt_finish.cuh) over the whole drafted set in shared memory the PaCM
// passes are done with.
// timeline ring of the last 64 fused verify launches: [first CTA start, finish end]
__device__ unsigned long long g_vtl[64][2];
__device__ unsigned g_vtl_n[1];
__device__ unsigned long long g_fin_ns[3];  // the last CTA's finish: start, end, identities ready (%globaltimer)

struct FinishArgs {
  const double* drafts;     // draft costs of the drafted set
  const int64_t* idx;       // population indices
  uint64_t* ids;            // identities (from the side stream, or known)
  const SelState* sel;      // selector status
  int64_t b;
  RecRing record;           // the round records (record.base null: no finish)
  unsigned* sync;           // see VerifyFinish
  int wait_ids;
  int* invalid;             // K1's population flag (copied into the record, reset)
};

template <int NSP, int NRED>
__global__ void __launch_bounds__(f64::T, 1) k_verify64(DevSketch SK, DevDevice D, CandRef ref,
                                                       const int64_t* __restrict__ count_dev, int64_t k_max,
                                                       const double* __restrict__ params,
                                                       double* __restrict__ score_out, FinishArgs fin) {
  using namespace f64;
  __shared__ CandInfo<NSP, NRED> ci[G];
  __shared__ bool last;
  // the sketch and device model copied to shared memory before the grid
  // dependency wait: the staging reads them with per-lane indices, which in
  // the parameter bank are constant-cache misses on the critical path
  __shared__ DevSketch sk_s;
  __shared__ DevDevice dd_s;
  {
    const uint32_t* a = reinterpret_cast<const uint32_t*>(&SK);
    const uint32_t* b = reinterpret_cast<const uint32_t*>(&D);
    for (int i = threadIdx.x; i < (int)(sizeof(DevSketch) / 4); i += blockDim.x) reinterpret_cast<uint32_t*>(&sk_s)[i] = a[i];
    for (int i = threadIdx.x; i < (int)(sizeof(DevDevice) / 4); i += blockDim.x) reinterpret_cast<uint32_t*>(&dd_s)[i] = b[i];
    __syncthreads();
  }
  const int S = 2 * SK.n_in + 2;
  const int B = SK.kind == TT_OP_ELEMENTWISE ? 1 : 3 * SK.n_in + 2;
  if (blockIdx.x == 0 && threadIdx.x == 0 && fin.record.base) g_vtl[g_vtl_n[0] & 63u][0] = gtimer64();
  pacm_h64_body(S, B, count_dev, k_max, params, score_out, [&](int64_t e0, int64_t count, double* MISC) {
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int v = t; v < G * kMisc; v += T) MISC[v] = 0.0;  // padding rows, xb^T row 23, idle slots
    if (warp == 0) {  // candidate lane >> 3 of the G = 4, 8 lanes each
      const int cc = lane >> 3, sub = lane & 7;
      const bool have = e0 + cc < count;
      Factors<NSP, NRED> F;
      if (ref.seeded) {
        // a seeded schedule is rebuilt from its draws: each lane takes every
        // 8th prime of the plan, and the 8 partial factor sets multiply
        if (have) {
          const uint64_t j = (uint64_t)ref.idx[e0 + cc];
          H64_MARK(22, 0);
          generate_part<NSP, NRED>(sk_s, ref.s0, j, sub, 8, F);
          H64_MARK(23, 0);
        } else {
#pragma unroll
          for (int q = 0; q < Factors<NSP, NRED>::kN; ++q) F.f[q] = 1;
          F.unroll = 1;
        }
#pragma unroll
        for (int o = 4; o; o >>= 1) {
#pragma unroll
          for (int q = 0; q < Factors<NSP, NRED>::kN; ++q) F.f[q] *= __shfl_xor_sync(0xffffffffu, F.f[q], o);
          F.unroll *= __shfl_xor_sync(0xffffffffu, F.unroll, o);
        }
      } else if (sub == 0 && have) {
        feat_load<NSP, NRED>(sk_s, ref, e0 + cc, F);
      }
      H64_MARK(19, 0);
      if (sub == 0 && have) cand_info<NSP, NRED>(sk_s, dd_s, F, ci[cc]);
      H64_MARK(20, 0);
    }
    __syncthreads();
    H64_MARK(21, 0);
    // warp w: feature row w of the G candidates, 8 lanes per candidate; every
    // lane derives the row's arguments, then applies the log1p of values
    // slot, slot + 8, slot + 16 only (3 instead of up to 14 per lane)
    const int cc = lane >> 3, slot = lane & 7;
    if (warp < S + B && e0 + cc < count) {
      double v[TT_STMT_WIDTH];
      uint32_t lm;
      feature_args<double, NSP, NRED>(sk_s, dd_s, ci[cc], warp, v, &lm);
      double* m = MISC + cc * kMisc + (warp < S ? warp : 24 * 8 + (warp - S));
      const int width = warp < S ? TT_STMT_WIDTH : TT_BLOCK_WIDTH;
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int k = slot + 8 * u;
        if (k < width) {
          double x = 0.0;
#pragma unroll
          for (int q = 0; q < TT_STMT_WIDTH; ++q)  // register-indexed select
            if (q == k) x = v[q];
          m[k * 8] = (lm >> k & 1u) ? lg<double>(x) : x;
        }
      }
    }
  });
  if (!fin.record.base) return;
  // ---- finish: the last CTA done runs select_top + the record over all scores
  __threadfence();  // this CTA's scores / identities before its ticket
  __syncthreads();
  __shared__ int ids_ready;
  if (threadIdx.x == 0) last = atomicAdd(&fin.sync[0], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  if (threadIdx.x == 0) {
    fin.sync[0] = 0u;  // for the next launch (graph replays)
    g_fin_ns[0] = gtimer64();
    int ok = 1;
    if (fin.wait_ids) {  // the side-stream identity kernel of this round (epoch handshake)
      const unsigned want = atomicAdd(&fin.sync[3], 1u) + 1u;
      const unsigned long long t0 = gtimer64();
      while ((int)(atomicAdd(&fin.sync[2], 0u) - want) < 0) {
        if (gtimer64() - t0 > 2000000ull) {  // 2 ms: never expected; compute them here instead
          ok = 0;
          break;
        }
        __nanosleep(256);
      }
    }
    ids_ready = ok;
    g_fin_ns[2] = gtimer64();
  }
  __syncthreads();
  __threadfence();
  if (!ids_ready) {  // fallback: every drafted candidate's identity, one per thread
    const int64_t cnt = *count_dev < k_max ? *count_dev : k_max;
    for (int64_t p = threadIdx.x; p < cnt; p += blockDim.x) {
      Factors<NSP, NRED> F;
      feat_load<NSP, NRED>(SK, ref, p, F);
      fin.ids[p] = identity_of<NSP, NRED>(SK, F);
    }
    __syncthreads();
  }
  extern __shared__ __align__(128) double smf[];
  finish_block(score_out, fin.drafts, nullptr, k_max, count_dev, fin.b, fin.idx, fin.ids, fin.sel, nullptr, nullptr,
               fin.record, fin.invalid, *reinterpret_cast<FinishSmem*>(smf));
  if (threadIdx.x == 0) g_fin_ns[1] = gtimer64(), g_vtl[atomicAdd(&g_vtl_n[0], 1u) & 63u][1] = g_fin_ns[1];
}

int launch_verify64(const DevSketch& S, const DevDevice& D, CandRef ref, const int64_t* count_dev, int64_t k_max,
                    const double* params, int h, double* score_out, cudaStream_t st, const VerifyFinish* vf) {
  const int ns = 2 * S.n_in + 2, nb = S.kind == TT_OP_ELEMENTWISE ? 1 : 3 * S.n_in + 2;
  if (h != f64::H || ns > 8 || nb > 8 || k_max <= 0) return -1;
  if (vf && !verify64_finish_ok(k_max, vf->b)) return -1;  // finish_block: one key per thread
  FinishArgs fin{};
  if (vf)
    fin = FinishArgs{vf->drafts, vf->idx, vf->ids, vf->sel, vf->b, vf->record, vf->sync, vf->wait_ids, vf->invalid};
  const int64_t ctas = (k_max + f64::G - 1) / f64::G;
  const dim3 grid((unsigned)(ctas < 148 ? ctas : 148));
  return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, ({
    static bool attr = false;  // per instance, once
    if (!attr) {
      cudaFuncSetAttribute(k_verify64<NSP, NRED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f64::kSmem);
      attr = true;
    }
    tt::note_launch();
    launch_pdl(k_verify64<NSP, NRED>, grid, dim3(f64::T), f64::kSmem, st, S, D, ref, count_dev, k_max, params,
               score_out, fin);
  }));
}

}  // namespace tt

extern "C" int ttdbg_verify64_clocks(long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, tt::g_clk_h64, sizeof(long long) * (n < 24 ? n : 24));
}
extern "C" int ttdbg_verify64_span(unsigned long long* out, int reset) {
  if (reset) {
    const unsigned long long init[4] = {~0ull, ~0ull, 0ull, 0ull};
    return (int)cudaMemcpyToSymbol(tt::g_h64_ns, init, sizeof(init));
  }
  int rc = (int)cudaMemcpyFromSymbol(out, tt::g_h64_ns, sizeof(unsigned long long) * 4);
  return rc ? rc : (int)cudaMemcpyFromSymbol(out + 4, tt::g_fin_ns, sizeof(unsigned long long) * 3);
}

extern "C" int ttdbg_verify64_finish_clocks(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, tt::g_fin_clk, sizeof(long long) * 8);
}

extern "C" int ttdbg_verify64_timeline(unsigned long long* out, unsigned* n) {
  int rc = (int)cudaMemcpyFromSymbol(out, tt::g_vtl, sizeof(unsigned long long) * 128);
  return rc ? rc : (int)cudaMemcpyFromSymbol(n, tt::g_vtl_n, sizeof(unsigned));
}

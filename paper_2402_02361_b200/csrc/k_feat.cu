// k_feat.cu — K3a: hybrid feature rows of the drafted candidates
// (extract_features, features.cpp:98-257).
//
// One CTA pass covers 8 or 32 candidates: warp 0 derives each candidate's shared
// information (factors → tile table → symbols → penalties,
// tiles_internal.hpp:80-108 / draft.cpp:42-127) into shared memory, one
// lane per candidate; then warp w evaluates feature row slot w of all of
// them in fp64 (the reference's arithmetic, log1p of the same
// arguments). Rows are warp-uniform: a warp only executes its row kind's
// code instead of the union of every kind — the row code is large and the
// kernel is instruction-fetch bound otherwise. Outputs, each optional:
//   * fp64 rows stmt [pos][S][24] / block [pos][B][23] — the layout of
//     tt_features; the exact PaCM (k_pacm64) reads these;
//   * bf16 GEMM tiles for the tensor-core PaCM: per 16 candidates one
//     16 KB image = Xs [128 rows x 32 k] then Xb [128 x 32], K-major
//     core-matrix order (row 8c + i = candidate c's row i, zero padded), the
//     exact shared-memory operand layout, so the consumer moves it with one
//     bulk TMA copy.
// A device-side sublist restricts the work to selected positions (the
// certification band); rows are then written at those positions.
#include <cuda_bf16.h>

#include <cstdint>

#include "tt_features.cuh"
#include "tt_kernels.h"
#include "tt_tc.cuh"

namespace tt {

constexpr int kFeatThreads = 512;  // 16 warps; warp w evaluates row slot w (w + 16, ...)


__device__ __forceinline__ void st_row_bf16(uint8_t* tile, int row, const double* v, int width) {
#pragma unroll
  for (int kc = 0; kc < 4; ++kc) {
    __nv_bfloat162 p[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k0 = 8 * kc + 2 * q;
      p[q] = __floats2bfloat162_rn(k0 < width ? (float)v[k0] : 0.f, k0 + 1 < width ? (float)v[k0 + 1] : 0.f);
    }
    *(uint4*)(tile + tc::kmaj_off(row, 8 * kc, 128)) = *(uint4*)p;
  }
}

// CPP candidates per CTA pass (one per lane of each warp): 32 for large
// batches (full lanes), 8 when the batch would otherwise occupy few SMs
// (the round's K = 512: latency matters more than lane utilisation).
template <int NSP, int NRED, int CPP>
__global__ void __launch_bounds__(kFeatThreads) k_feat_rows(DevSketch S, DevDevice D, CandRef r,
                                                            const int64_t* __restrict__ count_dev, int64_t k_max,
                                                            const int32_t* __restrict__ sublist,
                                                            const int* __restrict__ sublist_count,
                                                            double* __restrict__ stmt, double* __restrict__ block,
                                                            uint8_t* __restrict__ tiles) {
  pdl_trigger();
  __shared__ CandInfo<NSP, NRED> ci[CPP];
  __shared__ int64_t cpos[CPP];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  int64_t count = k_max;
  if (sublist) count = *sublist_count;
  else if (count_dev) count = *count_dev < k_max ? *count_dev : k_max;
  const int n_stmt = 2 * S.n_in + 2;
  const int n_block = S.kind == TT_OP_ELEMENTWISE ? 1 : 3 * S.n_in + 2;
  // rows of the tile image: slots 0..7 statements, 8..15 blocks (zero padded)
  const int n_rows = tiles ? 16 : n_stmt + n_block;
  for (int64_t e0 = (int64_t)blockIdx.x * CPP; e0 < count; e0 += (int64_t)gridDim.x * CPP) {
    if (warp == 0 && lane < CPP) {  // one lane per candidate: factors -> tile table -> symbols -> penalties
      const int64_t e = e0 + lane;
      int64_t pos = -1;
      if (e < count) {
        pos = sublist ? sublist[e] : e;
        Factors<NSP, NRED> F;
        feat_load<NSP, NRED>(S, r, pos, F);
        CandInfo<NSP, NRED> C;
        cand_info<NSP, NRED>(S, D, F, C);
        ci[lane] = C;
      }
      cpos[lane] = pos;
    }
    __syncthreads();
    // warp-uniform row: every lane of a warp evaluates the same row kind
    const int64_t pos = lane < CPP ? cpos[lane] : -1;
    uint8_t* tile = tiles ? tiles + ((e0 + lane) / 16) * kFeatTileBytes : nullptr;
    double v[TT_STMT_WIDTH];
    for (int slot = warp; lane < CPP && slot < n_rows; slot += kFeatThreads / 32) {
      int row;  // feature row index (statements first), -1 = padding
      bool is_stmt;
      if (tiles) {
        is_stmt = slot < 8;
        const int q = slot & 7;
        row = is_stmt ? (q < n_stmt ? q : -1) : (q < n_block ? n_stmt + q : -1);
      } else {
        is_stmt = slot < n_stmt;
        row = slot;
      }
      const int width = is_stmt ? TT_STMT_WIDTH : TT_BLOCK_WIDTH;
      if (row >= 0 && pos >= 0) {
        feature_row<double, NSP, NRED>(S, D, ci[lane], row, v);
        if (is_stmt && stmt) {
          double* o = stmt + (pos * n_stmt + row) * TT_STMT_WIDTH;
#pragma unroll
          for (int w = 0; w < TT_STMT_WIDTH; ++w) o[w] = v[w];
        } else if (!is_stmt && block) {
          double* o = block + (pos * n_block + row - n_stmt) * TT_BLOCK_WIDTH;
#pragma unroll
          for (int w = 0; w < TT_BLOCK_WIDTH; ++w) o[w] = v[w];
        }
      } else {
#pragma unroll
        for (int w = 0; w < TT_STMT_WIDTH; ++w) v[w] = 0.0;
      }
      if (tile)
        st_row_bf16(tile + (is_stmt ? 0 : kFeatTileBytes / 2), 8 * (int)((e0 + lane) & 15) + (slot & 7), v, width);
    }
    __syncthreads();
  }
}

int launch_feat_rows(const DevSketch& S, const DevDevice& D, CandRef ref, const int64_t* count_dev, int64_t k_max,
                     const int32_t* sublist, const int* sublist_count, double* stmt, double* block, uint8_t* tiles,
                     cudaStream_t st) {
  if (k_max <= 0) return 0;
  const int64_t wide = (k_max + 31) / 32;
  if (wide >= 148) {
    const unsigned grid = (unsigned)(wide < 2 * 148 ? wide : 2 * 148);
    return TT_DISPATCH_SHAPE(S.n_sp, S.n_red,
                             (tt::note_launch(), k_feat_rows<NSP, NRED, 32><<<grid, kFeatThreads, 0, st>>>(
                                                     S, D, ref, count_dev, k_max, sublist, sublist_count, stmt, block,
                                                     tiles)));
  }
  const unsigned grid = (unsigned)((k_max + 7) / 8);
  return TT_DISPATCH_SHAPE(S.n_sp, S.n_red,
                           (tt::note_launch(), k_feat_rows<NSP, NRED, 8><<<grid, kFeatThreads, 0, st>>>(
                                                   S, D, ref, count_dev, k_max, sublist, sublist_count, stmt, block,
                                                   tiles)));
}

}  // namespace tt

// k_oracle.cu — the reference's simulated hardware on the device (SURVEY
// §8f #2): noiseless_latency, measure and oracle_best (oracle.cpp:82-135).
//
// One schedule per thread. noiseless_latency = draft_cost under the hidden
// spec (K1's bit-exact device function) x stride multiplier x occupancy
// multiplier + launch overhead, in the reference's operand order with IEEE
// division and no FMA contraction (this file is built --fmad=false), so the
// result is bit-identical. measure() multiplies by exp(sigma * normal())
// from the tuner's per-trial RngStream (tuner.cpp:202-203); its Box-Muller
// log/cos/exp are CUDA's, within an ulp or two of glibc's.
#include <cstdint>

#include "tt_device.cuh"
#include "tt_kernels.h"

namespace tt {

// stride_multiplier (oracle.cpp:82-95) and occupancy_multiplier (:97-103)
template <int NSP, int NRED>
__device__ __forceinline__ double noiseless_of(const DevSketch& S, const DevOracle& O, const Factors<NSP, NRED>& F) {
  constexpr int NA = NSP + NRED;
  const double base = draft_cost_of<NSP, NRED>(S, O.hidden, F, TT_TOGGLES_ALL);
  Tiles<NSP, NRED> T;
  build_tiles(F, T);
  // statements in order: L2->L1 load per input (s5 > 0), L1->L0 loads and
  // compute (s5 = 0, skipped), store (s5 = output size)
  int64_t total = 0, misaligned = 0;
  const int64_t nl2m = O.hidden.n_l2 - 1;  // n_l2 is a power of two (device.cpp:105-108)
#pragma unroll
  for (int q = 0; q < kMaxIn; ++q) {
    if (q < S.n_in) {
      const int64_t s5 = fp_mask<NA>(T.l1, S.in_mask[q]) * T.s6 * T.prod_ra;
      if (s5 > 0) {
        total += s5;
        if ((int64_t)pick<NA>(T.l1, S.in_last[q]) & nl2m) misaligned += s5;
      }
    }
  }
  if (S.output_size > 0) {
    total += S.output_size;
    if ((int64_t)pick<NA>(T.l0, S.out_last) & nl2m) misaligned += S.output_size;
  }
  const double sm =
      total == 0 ? 1.0
                 : __dadd_rn(1.0, __dmul_rn(O.stride_coeff, __ddiv_rn((double)misaligned, (double)total)));
  const double lanes = __dmul_rn((double)T.s4, (double)T.s6);
  const double capacity = __dmul_rn((double)O.hidden.pu_l2, (double)O.hidden.n_l1);
  const double x = __ddiv_rn(lanes, capacity);
  const double fill = x < 1.0 ? x : 1.0;  // std::min(1.0, x)
  const double om = __dadd_rn(1.0, __dmul_rn(O.occupancy_coeff, __dsub_rn(1.0, fill)));
  return __dadd_rn(__dmul_rn(__dmul_rn(base, sm), om), O.launch);
}

__device__ __forceinline__ uint64_t mix64_dev(uint64_t x) { return scramble64(x + kGolden); }

// RngStream(derive_seed(seed, tag, task, trial)).lognormal(sigma)  (common.hpp:66-119)
__device__ __forceinline__ double trial_lognormal(uint64_t seed, uint64_t task, uint64_t trial, double sigma) {
  uint64_t s = seed;
  s = mix64_dev(s ^ mix64_dev(0x6d656173ull));
  s = mix64_dev(s ^ mix64_dev(task));
  s = mix64_dev(s ^ mix64_dev(trial));
  const uint64_t s0 = s ? s : kGolden;
  double u1 = (double)(draw(s0, 0) >> 11) * 0x1.0p-53;
  const double u2 = (double)(draw(s0, 1) >> 11) * 0x1.0p-53;
  if (u1 < 1e-300) u1 = 1e-300;
  const double nrm = __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(6.283185307179586476925286766559, u2)));
  return exp(__dmul_rn(sigma, nrm));
}

template <int NSP, int NRED>
__global__ void __launch_bounds__(256) k_oracle_latency(DevSketch S, DevOracle O, const int32_t* __restrict__ soa,
                                                        int64_t ld, int64_t n, int measure, uint64_t task,
                                                        uint64_t trial0, double* __restrict__ latency,
                                                        double* __restrict__ noiseless) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    Factors<NSP, NRED> F;
    load_factors<NSP, NRED>(soa, ld, i, F, true);
    const double nl = noiseless_of<NSP, NRED>(S, O, F);
    if (noiseless) noiseless[i] = nl;
    if (latency)
      latency[i] = (measure && O.sigma != 0.0) ? __dmul_rn(nl, trial_lognormal(O.seed, task, trial0 + i, O.sigma))
                                               : nl;
  }
}

// oracle_best: each CTA reduces (latency bits, identity) over its share of
// the identity space; a second one-CTA pass reduces the CTA winners.
template <int NSP, int NRED>
__global__ void __launch_bounds__(256) k_oracle_best(DevSketch S, DevOracle O, uint64_t space,
                                                     uint64_t* __restrict__ win_lat, uint64_t* __restrict__ win_id) {
  __shared__ uint64_t sl[8], si[8];
  uint64_t bl = ~0ull, bi = ~0ull;
  for (uint64_t id = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; id < space;
       id += (uint64_t)gridDim.x * blockDim.x) {
    Factors<NSP, NRED> F;
    from_identity<NSP, NRED>(S, id, F);
    const uint64_t l = cost_key(noiseless_of<NSP, NRED>(S, O, F));  // positive: bit order = value order
    if (l < bl || (l == bl && id < bi)) bl = l, bi = id;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const uint64_t ol = __shfl_xor_sync(0xffffffffu, bl, off), oi = __shfl_xor_sync(0xffffffffu, bi, off);
    if (ol < bl || (ol == bl && oi < bi)) bl = ol, bi = oi;
  }
  if ((threadIdx.x & 31) == 0) sl[threadIdx.x >> 5] = bl, si[threadIdx.x >> 5] = bi;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (sl[w] < bl || (sl[w] == bl && si[w] < bi)) bl = sl[w], bi = si[w];
    win_lat[blockIdx.x] = bl, win_id[blockIdx.x] = bi;
  }
}

__global__ void k_oracle_best_final(const uint64_t* __restrict__ win_lat, const uint64_t* __restrict__ win_id, int m,
                                    uint64_t* __restrict__ out) {
  if (threadIdx.x != 0) return;
  uint64_t bl = ~0ull, bi = ~0ull;
  for (int e = 0; e < m; ++e)
    if (win_lat[e] < bl || (win_lat[e] == bl && win_id[e] < bi)) bl = win_lat[e], bi = win_id[e];
  out[0] = bl, out[1] = bi;
}

int launch_oracle_latency(const DevSketch& S, const DevOracle& O, const int32_t* soa, int64_t ld, int64_t n,
                          int measure, uint64_t task, uint64_t trial0, double* latency, double* noiseless,
                          cudaStream_t st) {
  if (n <= 0) return 0;
  const int64_t g64 = (n + 255) / 256;
  const unsigned g = (unsigned)(g64 < 148 * 8 ? g64 : 148 * 8);
  return TT_DISPATCH_SHAPE(S.n_sp, S.n_red,
                           (tt::note_launch(), k_oracle_latency<NSP, NRED><<<g, 256, 0, st>>>(
                                                   S, O, soa, ld, n, measure, task, trial0, latency, noiseless)));
}

int launch_oracle_best(const DevSketch& S, const DevOracle& O, uint64_t* scratch_lat, uint64_t* scratch_id,
                       int max_ctas, uint64_t* out2, cudaStream_t st) {
  const uint64_t g64 = (S.space + 255) / 256;
  const int g = (int)(g64 < (uint64_t)max_ctas ? g64 : (uint64_t)max_ctas);
  int rc = TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (tt::note_launch(), k_oracle_best<NSP, NRED><<<g, 256, 0, st>>>(
                                                                      S, O, S.space, scratch_lat, scratch_id)));
  if (rc) return rc;
  tt::note_launch();
  k_oracle_best_final<<<1, 32, 0, st>>>(scratch_lat, scratch_id, g, out2);
  return 0;
}

}  // namespace tt

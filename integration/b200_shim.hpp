// b200_shim.hpp — the reference-side binding of the B200 draft+verify round:
// what a maintainer adds to tiletune::core (a new translation unit plus this
// header) so Engine::round_draft_verify (tuner.cpp:361-396) runs on the
// B200 library through its C ABI (include/tt/tt.h). Compiled and tested
// against the unmodified reference headers by integration/Makefile.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "tiletune/device.hpp"
#include "tiletune/ranker.hpp"
#include "tiletune/workload.hpp"
#include "tt/tt.h"

namespace tiletune::b200 {

// tt status -> tiletune::Error with the reference's code strings (common.hpp:44-50)
void check(tt_ctx* ctx, int rc);

tt_device_spec to_tt(const DeviceSpec& d);    // device.hpp:29-39
tt_op_spec to_tt(const TensorOpSpec& op);      // workload.hpp:30-57, axis names -> ids
std::vector<double> flatten(const RankerParams& p);  // for_each_tensor order (ranker.cpp:339-356)

// One context per engine (owns a CUDA stream + scratch); rounds are serialised on it.
class B200Round {
 public:
  explicit B200Round(int device);
  ~B200Round();
  B200Round(const B200Round&) = delete;
  B200Round& operator=(const B200Round&) = delete;

  // explore(op, dev, 1, draft_size, pop_size, RngStream(seed)) + extract_features
  // + score_batch + select_top(b) (tuner.cpp:302-305, 366-384) in one device
  // round. Returns the population indices of the selections (index i = the
  // i-th schedule of random_init(sketch, pop_size, RngStream(seed))), their
  // scores and exact identities.
  std::vector<int64_t> run(const TensorOpSpec& op, const DeviceSpec& dev, const RankerParams& target, int pop_size,
                           int draft_size, int b, uint64_t seed, std::vector<double>* scores = nullptr,
                           std::vector<uint64_t>* identities = nullptr);

  // The tuner's round at its real shape (tuner.cpp:294-396): the draft set
  // (explore(op, dev, n_steps, n_spec, pop_size, RngStream(explore_seed)) +
  // the unseen schedules of random_init(., RngStream(mix_seed)), n_spec =
  // max(1, llround((1 - random_mix) draft_size))), extract_features,
  // score_batch and select_top(b) in one device call. Returns the indices of
  // the picks into that draft set; scores / identities / set size optional.
  std::vector<int64_t> tuner_round(const TensorOpSpec& op, const DeviceSpec& dev, const RankerParams& target,
                                   int n_steps, int draft_size, int pop_size, double random_mix,
                                   uint64_t explore_seed, uint64_t mix_seed, int b,
                                   std::vector<double>* scores = nullptr,
                                   std::vector<uint64_t>* identities = nullptr, int64_t* n_candidates = nullptr);

  // train(target, {task}, cfg) (ranker.cpp:459-512) on the device, in place
  // (features as host rows [n][S][24] / [n][B][23]); returns (initial, final) loss.
  std::pair<double, double> train(RankerParams& target, const std::vector<double>& stmt,
                                  const std::vector<double>& block, int n_stmt, int n_block,
                                  const std::vector<double>& latencies, const TrainConfig& cfg);

  tt_ctx* ctx() const { return ctx_; }

 private:
  tt_ctx* ctx_ = nullptr;
};

}  // namespace tiletune::b200

// b200_shim.cpp — see b200_shim.hpp. Binds the reference's value types to the
// C ABI of include/tt/tt.h; no CUDA headers: device buffers of the training
// call are managed with the CUDA runtime C API declared below (libcudart).
#include "b200_shim.hpp"

#include <algorithm>
#include <cstring>

#include "tiletune/common.hpp"

extern "C" {  // the two CUDA runtime entry points the training binding needs
int cudaMalloc(void** p, size_t bytes);
int cudaFree(void* p);
int cudaMemcpy(void* dst, const void* src, size_t bytes, int kind);
}

namespace tiletune::b200 {

void check(tt_ctx* ctx, int rc) {
  if (rc == TT_OK) return;
  throw Error(tt_status_code(rc), ctx ? tt_last_error(ctx) : "tt call failed");
}

tt_device_spec to_tt(const DeviceSpec& d) {
  return {d.m_l0, d.m_l1, d.pu_l1, d.n_l1, d.pu_l2, d.n_l2, d.t_p, d.t_m, d.element_bytes};
}

tt_op_spec to_tt(const TensorOpSpec& op) {
  tt_op_spec o{};
  std::vector<std::string> names;
  if (op.spatial_axes.size() + op.reduction_axes.size() > TT_MAX_AXES || op.buffers.size() > TT_MAX_BUFFERS)
    throw Error("E_VALIDATE", "op exceeds the B200 library's axis / buffer limits");
  for (const auto& a : op.spatial_axes) names.push_back(a.name), o.extent[o.n_spatial++] = a.extent;
  for (const auto& a : op.reduction_axes) names.push_back(a.name), o.extent[o.n_spatial + o.n_reduction++] = a.extent;
  for (const auto& b : op.buffers) {
    auto& tb = o.buffers[o.n_buffers++];
    tb.io = b.io == BufferIo::kOutput ? TT_IO_OUTPUT : TT_IO_INPUT;
    for (const auto& ax : b.axes) {
      const auto it = std::find(names.begin(), names.end(), ax);
      if (it == names.end()) throw Error("E_VALIDATE", "buffer " + b.name + " names unknown axis " + ax);
      tb.axes[tb.n_axes++] = int(it - names.begin());
    }
  }
  o.fused_elementwise = op.fused_elementwise;
  o.kind = op.kind == OpKind::kElementwise ? TT_OP_ELEMENTWISE : TT_OP_TILED;
  return o;
}

std::vector<double> flatten(const RankerParams& p) {
  std::vector<double> out;
  for_each_tensor(p, [&](const std::string&, const Tensor& t) { out.insert(out.end(), t.v.begin(), t.v.end()); });
  return out;
}

static void unflatten_into(RankerParams& p, const std::vector<double>& v) {
  std::size_t off = 0;
  for_each_tensor(p, [&](const std::string&, Tensor& t) {
    std::copy(v.begin() + off, v.begin() + off + t.v.size(), t.v.begin());
    off += t.v.size();
  });
}

B200Round::B200Round(int device) { check(nullptr, tt_ctx_create(device, &ctx_)); }
B200Round::~B200Round() { tt_ctx_destroy(ctx_); }

std::vector<int64_t> B200Round::run(const TensorOpSpec& op, const DeviceSpec& dev, const RankerParams& target,
                                    int pop_size, int draft_size, int b, uint64_t seed, std::vector<double>* scores,
                                    std::vector<uint64_t>* identities) {
  tt_op_spec o = to_tt(op);
  tt_sketch sk;
  check(ctx_, tt_sketch_from_op(&o, 1, &sk));
  tt_device_spec d = to_tt(dev);
  check(ctx_, tt_validate_device(&d));
  const auto params = flatten(target);
  check(ctx_, tt_pacm_load(ctx_, params.data(), target.hidden));  // host pointer, copied in
  tt_round_config cfg{};
  cfg.n = pop_size, cfg.k = draft_size, cfg.b = b, cfg.toggles = TT_TOGGLES_ALL, cfg.precision = TT_PREC_FP64;
  std::vector<int64_t> idx(b);
  std::vector<double> sc(b), co(b);
  std::vector<uint64_t> id(b);
  tt_round_result res{};
  // the population random_init(sketch, N, RngStream(seed)) is drawn on the device (counter-based)
  check(ctx_, tt_round(ctx_, &sk, &d, &cfg, nullptr, 0, seed, idx.data(), sc.data(), co.data(), id.data(), &res));
  idx.resize(res.selected), sc.resize(res.selected), id.resize(res.selected);
  if (scores) *scores = sc;
  if (identities) *identities = id;
  return idx;
}

std::vector<int64_t> B200Round::tuner_round(const TensorOpSpec& op, const DeviceSpec& dev,
                                            const RankerParams& target, int n_steps, int draft_size, int pop_size,
                                            double random_mix, uint64_t explore_seed, uint64_t mix_seed, int b,
                                            std::vector<double>* scores, std::vector<uint64_t>* identities,
                                            int64_t* n_candidates) {
  tt_op_spec o = to_tt(op);
  tt_sketch sk;
  check(ctx_, tt_sketch_from_op(&o, 1, &sk));
  tt_device_spec d = to_tt(dev);
  check(ctx_, tt_validate_device(&d));
  const auto params = flatten(target);
  check(ctx_, tt_pacm_load(ctx_, params.data(), target.hidden));
  std::vector<int64_t> idx(b);
  std::vector<double> sc(b);
  std::vector<uint64_t> id(b);
  int64_t cnt = 0;
  check(ctx_, tt_tuner_round(ctx_, &sk, &d, n_steps, draft_size, pop_size, random_mix, explore_seed, mix_seed, b,
                             TT_PREC_FP64, idx.data(), sc.data(), id.data(), &cnt));
  if (scores) *scores = sc;
  if (identities) *identities = id;
  if (n_candidates) *n_candidates = cnt;
  return idx;
}

std::pair<double, double> B200Round::train(RankerParams& target, const std::vector<double>& stmt,
                                           const std::vector<double>& block, int n_stmt, int n_block,
                                           const std::vector<double>& latencies, const TrainConfig& cfg) {
  auto p = flatten(target);
  void *dp = nullptr, *ds = nullptr, *db = nullptr;
  auto release = [&] { cudaFree(dp), cudaFree(ds), cudaFree(db); };
  if (cudaMalloc(&dp, p.size() * 8) || cudaMalloc(&ds, stmt.size() * 8) || cudaMalloc(&db, block.size() * 8)) {
    release();
    throw Error("E_CUDA", "train: device allocation failed");
  }
  cudaMemcpy(dp, p.data(), p.size() * 8, 1), cudaMemcpy(ds, stmt.data(), stmt.size() * 8, 1);
  cudaMemcpy(db, block.data(), block.size() * 8, 1);  // 1 = cudaMemcpyHostToDevice
  double l0 = 0.0, l1 = 0.0;
  const int rc = tt_pacm_train(ctx_, (double*)dp, target.hidden, (const double*)ds, (const double*)db, n_stmt,
                               n_block, latencies.data(), (int64_t)latencies.size(), cfg.epochs, cfg.lr, cfg.batch,
                               cfg.seed, cfg.score_opts.attention_identity ? 1 : 0, &l0, &l1);
  if (rc == TT_OK) cudaMemcpy(p.data(), dp, p.size() * 8, 2);  // 2 = cudaMemcpyDeviceToHost
  release();
  check(ctx_, rc);
  unflatten_into(target, p);
  return {l0, l1};
}

}  // namespace tiletune::b200

// Closed-form per-iteration traffic ledgers — the byte oracle of the path.
// Each closed form restates proj/src/traffic.cpp of the reference:
//   horizontal_traffic :44-64, vertical_traffic :66-94,
//   single_fb_traffic :96-117, plan_traffic :119-124.
// They are written independently of the plan builders; a built plan's summed
// Xfer bytes must equal them exactly (traffic.hpp:40-41).
#include "offsim/offsim.hpp"

namespace offsim {

const char* data_name(DataKind d) {
  static const char* const names[] = {"param", "ckpt", "grad_accum", "interlayer_grad",
                                      "opt_state"};
  const int i = static_cast<int>(d);
  return (i >= 0 && i < 5) ? names[i] : "?";
}

namespace {

// Per-layer byte quantities every ledger needs.  PCIe moves the local GPU's
// shard of a layer; SSD quantities are box-wide (summed over replicas).
struct LayerBytes {
  u64 n, m, dp;
  u64 pcie_param;  // chunk 0 of the layer's low-precision params over dp
  u64 pcie_grad;   // chunk 0 of the layer's fp32 grads over dp
  u64 ssd_param, ssd_ckpt, ssd_opt;
  u64 ckpt;        // one micro-batch's layer-input checkpoint
};

LayerBytes layer_bytes(const ModelSpec& model, int microbatches, const StorageSplit& split) {
  model.validate();
  split.validate();
  const LayerSizes s = derive_layer_sizes(model);
  LayerBytes b{};
  b.n = static_cast<u64>(model.num_layers);
  b.m = static_cast<u64>(microbatches);
  b.dp = static_cast<u64>(model.data_parallel_degree);
  b.pcie_param = chunk_size(s.param_bytes_low, model.data_parallel_degree, 0);
  b.pcie_grad = chunk_size(s.grad_bytes_full, model.data_parallel_degree, 0);
  b.ssd_param = ssd_portion(s.param_bytes_low, split.x_param);
  b.ssd_ckpt = ssd_portion(s.ckpt_bytes_per_mb, split.x_ckpt);
  b.ssd_opt = ssd_portion(s.opt_state_bytes, split.x_opt);
  b.ckpt = s.ckpt_bytes_per_mb;
  return b;
}

using L = LinkKind;
using D = DataKind;

}  // namespace

TrafficLedger vertical_traffic(const ModelSpec& model, int microbatches, const StorageSplit& split,
                               double alpha) {
  if (alpha < 0.0 || alpha > 1.0) throw ValidationError("delay ratio alpha must be in [0,1]");
  const LayerBytes b = layer_bytes(model, microbatches, split);
  const u64 n = b.n, m = b.m;
  // The delayed slice of SSD-resident params is produced in DRAM by the
  // delayed step and never re-read from SSD before the forward fetch.
  const u64 delayed_param = scaled_portion(b.ssd_param, alpha);
  TrafficLedger t;
  // Parameters: fetched once per layer per pass (forward + backward).
  t.at(L::PCIe_H2D, D::Param) = 2 * n * b.pcie_param;
  t.at(L::SSD_Read, D::Param) = n * (2 * b.ssd_param - delayed_param);
  t.at(L::SSD_Write, D::Param) = n * b.ssd_param;
  // Checkpoints: every (layer, mb) goes out once.  Forward reloads skip layer
  // 0 and the snake turning point; backward reloads skip layer 0.
  t.at(L::PCIe_D2H, D::Ckpt) = n * m * b.ckpt;
  t.at(L::PCIe_H2D, D::Ckpt) = (n - 1) * (2 * m - 1) * b.ckpt;
  t.at(L::SSD_Write, D::Ckpt) = n * m * b.ssd_ckpt * b.dp;
  t.at(L::SSD_Read, D::Ckpt) = (n - 1) * m * b.ssd_ckpt * b.dp;
  // Gradients accumulate in HBM across all micro-batches, leave once.
  t.at(L::PCIe_D2H, D::GradAccum) = n * b.pcie_grad;
  // Inter-layer activation gradients bounce through DRAM except at the turn.
  t.at(L::PCIe_D2H, D::InterlayerGrad) = (n - 1) * (m - 1) * b.ckpt;
  t.at(L::PCIe_H2D, D::InterlayerGrad) = (n - 1) * (m - 1) * b.ckpt;
  // Optimizer state: one SSD round trip per layer (immediate + delayed).
  t.at(L::SSD_Read, D::OptState) = n * b.ssd_opt;
  t.at(L::SSD_Write, D::OptState) = n * b.ssd_opt;
  return t;
}

TrafficLedger horizontal_traffic(const ModelSpec& model, int microbatches,
                                 const StorageSplit& split) {
  const LayerBytes b = layer_bytes(model, microbatches, split);
  const u64 n = b.n, m = b.m;
  TrafficLedger t;
  // Every micro-batch re-streams every layer in forward and in backward.
  t.at(L::PCIe_H2D, D::Param) = 2 * m * n * b.pcie_param;
  t.at(L::SSD_Read, D::Param) = 2 * m * n * b.ssd_param;
  t.at(L::SSD_Write, D::Param) = n * b.ssd_param;
  t.at(L::PCIe_D2H, D::Ckpt) = m * n * b.ckpt;
  t.at(L::PCIe_H2D, D::Ckpt) = m * n * b.ckpt;
  t.at(L::SSD_Write, D::Ckpt) = m * n * b.ssd_ckpt * b.dp;
  t.at(L::SSD_Read, D::Ckpt) = m * n * b.ssd_ckpt * b.dp;
  // Partial gradient sums shuttle out after every micro-batch and come back
  // for the next one: 2M-1 gradient-sized transfers per layer.
  t.at(L::PCIe_D2H, D::GradAccum) = m * n * b.pcie_grad;
  t.at(L::PCIe_H2D, D::GradAccum) = (m - 1) * n * b.pcie_grad;
  t.at(L::SSD_Read, D::OptState) = n * b.ssd_opt;
  t.at(L::SSD_Write, D::OptState) = n * b.ssd_opt;
  return t;
}

TrafficLedger single_fb_traffic(const ModelSpec& model, int batch, bool extra_ckpt,
                                const StorageSplit& split) {
  if (batch < 1) throw ValidationError("single-fb traffic requires batch >= 1");
  const LayerBytes b = layer_bytes(model, 1, split);
  const u64 n = b.n;
  const u64 ck = static_cast<u64>(batch) * static_cast<u64>(model.seq_len) *
                 static_cast<u64>(model.hidden_dim) * static_cast<u64>(model.low_precision_bytes);
  const u64 ssd_ck = ssd_portion(ck, split.x_ckpt);
  const u64 per_layer = extra_ckpt ? 2 : 1;
  TrafficLedger t;
  t.at(L::PCIe_H2D, D::Param) = 2 * n * b.pcie_param;
  t.at(L::SSD_Read, D::Param) = 2 * n * b.ssd_param;
  t.at(L::SSD_Write, D::Param) = n * b.ssd_param;
  t.at(L::PCIe_D2H, D::Ckpt) = n * per_layer * ck;
  t.at(L::PCIe_H2D, D::Ckpt) = n * per_layer * ck;
  t.at(L::SSD_Write, D::Ckpt) = n * per_layer * ssd_ck * b.dp;
  t.at(L::SSD_Read, D::Ckpt) = n * per_layer * ssd_ck * b.dp;
  t.at(L::PCIe_D2H, D::GradAccum) = n * b.pcie_grad;
  t.at(L::SSD_Read, D::OptState) = n * b.ssd_opt;
  t.at(L::SSD_Write, D::OptState) = n * b.ssd_opt;
  return t;
}

TrafficLedger plan_traffic(const SchedulePlan& plan) {
  TrafficLedger t;
  for (const Task& task : plan.tasks)
    if (task.kind == TaskKind::Xfer) t.at(task.link, task.data) += task.bytes;
  return t;
}

}  // namespace offsim

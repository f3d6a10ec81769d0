// Model geometry, machine constants and split validation.
// Semantics follow proj/src/model.cpp:9-51, proj/src/machine.cpp:5-50 and
// proj/src/schedule.cpp:9-13 of the reference (error texts are part of the
// contract: the reference tests match them verbatim).
#include "offsim/offsim.hpp"

namespace offsim {

namespace {
void require(bool ok, const char* msg) {
  if (!ok) throw ValidationError(msg);
}
bool legal_width(int w) { return w == 1 || w == 2 || w == 4 || w == 8; }
}  // namespace

void ModelSpec::validate() const {
  require(num_layers >= 1, "model.num_layers must be >= 1");
  require(hidden_dim >= 1, "model.hidden_dim must be >= 1");
  require(num_heads >= 1, "model.num_heads must be >= 1");
  require(seq_len >= 1, "model.seq_len must be >= 1");
  require(microbatch_size >= 1, "model.microbatch_size must be >= 1");
  require(legal_width(low_precision_bytes), "model.low_precision_bytes must be one of {1,2,4,8}");
  require(legal_width(full_precision_bytes), "model.full_precision_bytes must be one of {1,2,4,8}");
  require(optimizer_states_per_element >= 1, "model.optimizer_states_per_element must be >= 1");
  require(data_parallel_degree >= 1, "model.data_parallel_degree must be >= 1");
}

LayerSizes derive_layer_sizes(const ModelSpec& spec) {
  spec.validate();
  const u64 h = static_cast<u64>(spec.hidden_dim);
  const u64 lp = static_cast<u64>(spec.low_precision_bytes);
  const u64 fp = static_cast<u64>(spec.full_precision_bytes);
  LayerSizes out;
  out.param_elements = 12 * h * h;
  out.param_bytes_low = out.param_elements * lp;
  out.grad_bytes_full = out.param_elements * fp;
  out.opt_state_bytes = out.param_elements * fp * static_cast<u64>(spec.optimizer_states_per_element);
  out.ckpt_elements_per_mb =
      static_cast<u64>(spec.microbatch_size) * static_cast<u64>(spec.seq_len) * h;
  out.ckpt_bytes_per_mb = out.ckpt_elements_per_mb * lp;
  return out;
}

ModelTotals model_totals(const ModelSpec& spec) {
  const LayerSizes per = derive_layer_sizes(spec);
  const u64 n = static_cast<u64>(spec.num_layers);
  ModelTotals t;
  t.param_elements = n * per.param_elements;
  t.param_bytes_low = n * per.param_bytes_low;
  t.ckpt_bytes_per_mb = n * per.ckpt_bytes_per_mb;
  t.opt_state_bytes = n * per.opt_state_bytes;
  t.grad_bytes_full = n * per.grad_bytes_full;
  return t;
}

void MachineSpec::validate() const {
  require(gpu_mem_bytes != 0, "machine.gpu_mem_bytes must be > 0");
  require(cpu_usable_dram_bytes != 0, "machine.cpu_usable_dram_bytes must be > 0");
  require(pcie_h2d_bw > 0, "machine.pcie_h2d_bw must be > 0");
  require(pcie_d2h_bw > 0, "machine.pcie_d2h_bw must be > 0");
  require(ssd_read_bw > 0, "machine.ssd_read_bw must be > 0");
  require(ssd_write_bw > 0, "machine.ssd_write_bw must be > 0");
  require(fwd_compute_time_per_layer_per_mb >= 0,
          "machine.fwd_compute_time_per_layer_per_mb must be >= 0");
  require(bwd_compute_time_per_layer_per_mb >= 0,
          "machine.bwd_compute_time_per_layer_per_mb must be >= 0");
  require(cpu_step_throughput > 0, "machine.cpu_step_throughput must be > 0");
  require(fixed_overhead_time >= 0, "machine.fixed_overhead_time must be >= 0");
  require(num_gpus >= 1, "machine.num_gpus must be >= 1");
}

double transfer_time(u64 bytes, LinkKind link, const MachineSpec& machine) {
  if (bytes == 0) return 0.0;
  double bw;
  switch (link) {
    case LinkKind::PCIe_H2D: bw = machine.pcie_h2d_bw; break;
    case LinkKind::PCIe_D2H: bw = machine.pcie_d2h_bw; break;
    case LinkKind::SSD_Read: bw = machine.ssd_read_bw; break;
    case LinkKind::SSD_Write: bw = machine.ssd_write_bw; break;
    default: throw ValidationError("unknown link kind");
  }
  return static_cast<double>(bytes) / bw;
}

double optimizer_step_time(u64 elements, const MachineSpec& machine) {
  return elements == 0 ? 0.0 : static_cast<double>(elements) / machine.cpu_step_throughput;
}

const char* link_name(LinkKind link) {
  static const char* const names[] = {"H2D", "D2H", "SSD_read", "SSD_write"};
  const int i = static_cast<int>(link);
  return (i >= 0 && i < 4) ? names[i] : "?";
}

void StorageSplit::validate() const {
  require(x_ckpt >= 0 && x_ckpt <= 1, "split.x_ckpt must be in [0,1]");
  require(x_param >= 0 && x_param <= 1, "split.x_param must be in [0,1]");
  require(x_opt >= 0 && x_opt <= 1, "split.x_opt must be in [0,1]");
}

}  // namespace offsim

// extern "C" boundary of libgreedysnake.so (declared in include/greedysnake.h).
// Converts exceptions to status codes (the reference CLI's exit-code
// convention, proj/tools/offsim_main.cpp:400-409) and keeps the last error
// message per thread.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <functional>
#include <cstring>
#include <exception>
#include <memory>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "greedysnake.h"
#include "host_adam.hpp"
#include "host_tiers.hpp"
#include "kernels.h"
#include "layer_ops.hpp"
#include "peer_comm.hpp"
#include "offsim/executor.hpp"
#include "offsim/json_io.hpp"

struct gs_plan {
  offsim::SchedulePlan plan;
};
struct gs_engine {
  std::unique_ptr<offsim::Executor> ex;
  std::vector<offsim::TraceRecord> trace;
};

namespace {

thread_local std::string g_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return GS_OK;
  } catch (const offsim::ValidationError& e) {
    g_error = e.what();
    return GS_ERR_VALIDATION;
  } catch (const offsim::InfeasibleError& e) {
    g_error = e.what();
    return GS_ERR_INFEASIBLE;
  } catch (const offsim::PlanBugError& e) {
    g_error = e.what();
    return GS_ERR_PLAN_BUG;
  } catch (const std::bad_alloc&) {
    g_error = "out of host memory";
    return GS_ERR_INFEASIBLE;
  } catch (const std::exception& e) {
    g_error = e.what();
    return std::strstr(e.what(), "CUDA") ? GS_ERR_CUDA : GS_ERR_RUNTIME;
  }
}

int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}

int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return GS_OK;
  g_error = std::string("CUDA: ") + cudaGetErrorString(e);
  return GS_ERR_CUDA;
}

offsim::ModelSpec model_of(const gs_model_spec* m) {
  if (!m) throw offsim::ValidationError("model spec is NULL");
  offsim::ModelSpec s;
  s.num_layers = m->num_layers;
  s.hidden_dim = m->hidden_dim;
  s.num_heads = m->num_heads;
  s.seq_len = m->seq_len;
  s.microbatch_size = m->microbatch_size;
  s.low_precision_bytes = m->low_precision_bytes;
  s.full_precision_bytes = m->full_precision_bytes;
  s.optimizer_states_per_element = m->optimizer_states_per_element;
  s.data_parallel_degree = m->data_parallel_degree;
  return s;
}
offsim::StorageSplit split_of(const gs_split* x) {
  if (!x) throw offsim::ValidationError("split is NULL");
  offsim::StorageSplit s;
  s.x_ckpt = x->x_ckpt;
  s.x_param = x->x_param;
  s.x_opt = x->x_opt;
  return s;
}
void ledger_out(const offsim::TrafficLedger& t, uint64_t* out) {
  for (int l = 0; l < 4; ++l)
    for (int d = 0; d < 5; ++d) out[l * 5 + d] = t.bytes[static_cast<size_t>(l)][static_cast<size_t>(d)];
}
int copy_string(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size() + 1;
  if (!buf || cap < s.size() + 1) {
    g_error = "buffer too small";
    return buf ? GS_ERR_VALIDATION : GS_OK;
  }
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return GS_OK;
}
gs::DType dt_of(int dtype) { return dtype == 0 ? gs::DType::F32 : gs::DType::BF16; }

}  // namespace

namespace gs {
long long& launch_counter_ref();
}

extern "C" {

const char* gs_last_error(void) { return g_error.c_str(); }
const char* gs_version(void) { return "greedysnake-b200 0.1 (sm_100a)"; }

int gs_plan_build_vertical(const gs_model_spec* model, int mbs, const gs_split* split, double alpha, gs_plan** out) {
  return guarded([&] {
    auto p = std::make_unique<gs_plan>();
    p->plan = offsim::build_vertical(model_of(model), mbs, split_of(split), alpha);
    *out = p.release();
  });
}
int gs_plan_build_horizontal(const gs_model_spec* model, int mbs, const gs_split* split, gs_plan** out) {
  return guarded([&] {
    auto p = std::make_unique<gs_plan>();
    p->plan = offsim::build_horizontal(model_of(model), mbs, split_of(split));
    *out = p.release();
  });
}
int gs_plan_from_json(const char* json, gs_plan** out) {
  return guarded([&] {
    offsim::Json j;
    try {
      j = offsim::Json::parse(json ? json : "");
    } catch (const std::exception& e) {
      throw offsim::ValidationError(std::string("malformed plan JSON: ") + e.what());
    }
    auto p = std::make_unique<gs_plan>();
    p->plan = offsim::plan_from_json(j);
    *out = p.release();
  });
}
void gs_plan_free(gs_plan* plan) { delete plan; }
int gs_plan_num_tasks(const gs_plan* plan) { return plan ? static_cast<int>(plan->plan.tasks.size()) : -1; }
int gs_plan_info(const gs_plan* plan, int* variant, double* alpha, int* num_microbatches, int* num_layers) {
  return guarded([&] {
    if (!plan) throw offsim::ValidationError("plan is NULL");
    if (variant) *variant = static_cast<int>(plan->plan.kind.variant);
    if (alpha) *alpha = plan->plan.kind.delay_ratio;
    if (num_microbatches) *num_microbatches = plan->plan.num_microbatches;
    if (num_layers) *num_layers = plan->plan.num_layers;
  });
}
int gs_plan_task(const gs_plan* plan, int index, gs_task* out) {
  return guarded([&] {
    if (!plan || index < 0 || index >= static_cast<int>(plan->plan.tasks.size()))
      throw offsim::ValidationError("task index out of range");
    const offsim::Task& t = plan->plan.tasks[static_cast<size_t>(index)];
    out->id = t.id;
    out->kind = static_cast<int>(t.kind);
    out->layer = t.layer;
    out->microbatch = t.microbatch;
    out->stage = t.stage;
    out->data = static_cast<int>(t.data);
    out->link = static_cast<int>(t.link);
    out->bytes = t.bytes;
    out->elements = t.elements;
    out->cross_iter_dep = t.cross_iter_dep;
    out->num_deps = static_cast<int>(t.deps.size());
  });
}
int gs_plan_task_deps(const gs_plan* plan, int index, int* out, int cap, int* n) {
  return guarded([&] {
    if (!plan || index < 0 || index >= static_cast<int>(plan->plan.tasks.size()))
      throw offsim::ValidationError("task index out of range");
    const auto& deps = plan->plan.tasks[static_cast<size_t>(index)].deps;
    *n = static_cast<int>(deps.size());
    for (int i = 0; i < cap && i < *n; ++i) out[i] = deps[static_cast<size_t>(i)];
  });
}
int gs_plan_to_json(const gs_plan* plan, char* buf, size_t cap, size_t* len) {
  int rc = GS_OK;
  const int g = guarded([&] { rc = copy_string(offsim::plan_to_json(plan->plan).dump(), buf, cap, len); });
  return g != GS_OK ? g : rc;
}
int gs_plan_traffic(const gs_plan* plan, uint64_t ledger[20]) {
  return guarded([&] { ledger_out(offsim::plan_traffic(plan->plan), ledger); });
}
int gs_vertical_traffic(const gs_model_spec* model, int mbs, const gs_split* split, double alpha, uint64_t ledger[20]) {
  return guarded([&] { ledger_out(offsim::vertical_traffic(model_of(model), mbs, split_of(split), alpha), ledger); });
}
int gs_horizontal_traffic(const gs_model_spec* model, int mbs, const gs_split* split, uint64_t ledger[20]) {
  return guarded([&] { ledger_out(offsim::horizontal_traffic(model_of(model), mbs, split_of(split)), ledger); });
}
int64_t gs_plan_overlap_window(const gs_plan* plan) { return plan ? offsim::overlap_window(plan->plan) : -1; }
static offsim::MachineSpec machine_of(const gs_machine_spec* m) {
  if (!m) throw offsim::ValidationError("machine is NULL");
  offsim::MachineSpec mc;
  mc.gpu_mem_bytes = m->gpu_mem_bytes;
  mc.cpu_usable_dram_bytes = m->cpu_usable_dram_bytes;
  mc.pcie_h2d_bw = m->pcie_h2d_bw;
  mc.pcie_d2h_bw = m->pcie_d2h_bw;
  mc.ssd_read_bw = m->ssd_read_bw;
  mc.ssd_write_bw = m->ssd_write_bw;
  mc.fwd_compute_time_per_layer_per_mb = m->fwd_compute_time_per_layer_per_mb;
  mc.bwd_compute_time_per_layer_per_mb = m->bwd_compute_time_per_layer_per_mb;
  mc.cpu_step_throughput = m->cpu_step_throughput;
  mc.fixed_overhead_time = m->fixed_overhead_time;
  mc.num_gpus = m->num_gpus;
  mc.gpu_working_set_bytes = m->gpu_working_set_bytes;
  mc.ssd_duplex = m->ssd_duplex != 0;
  return mc;
}

int gs_simulate_json(const gs_plan* plan, const gs_machine_spec* m, char* buf, size_t cap, size_t* len) {
  int rc = GS_OK;
  const int g = guarded([&] {
    rc = copy_string(offsim::report_to_json(offsim::simulate(plan->plan, machine_of(m))).dump(), buf, cap, len);
  });
  return g != GS_OK ? g : rc;
}

static void solution_out(const offsim::PlannerSolution& s, gs_planner_solution* out) {
  if (!out) throw offsim::ValidationError("planner: NULL output");
  out->feasible = s.feasible ? 1 : 0;
  out->num_microbatches = s.num_microbatches;
  out->alpha = s.alpha;
  out->split.x_ckpt = s.split.x_ckpt;
  out->split.x_param = s.split.x_param;
  out->split.x_opt = s.split.x_opt;
  out->t_fwd_stage = s.t_fwd_stage;
  out->t_bwd_stage = s.t_bwd_stage;
  out->iteration_estimate = s.iteration_estimate;
  out->throughput_estimate = s.throughput_estimate;
}
int gs_solve_config(const gs_model_spec* model, const gs_machine_spec* machine, int num_microbatches, double alpha,
                    gs_planner_solution* out) {
  return guarded([&] {
    solution_out(offsim::solve_config(model_of(model), machine_of(machine), num_microbatches, alpha), out);
  });
}
int gs_find_optimal_config(const gs_model_spec* model, const gs_machine_spec* machine, gs_planner_solution* out) {
  return guarded([&] { solution_out(offsim::find_optimal_config(model_of(model), machine_of(machine)), out); });
}
int gs_grid_search_config(const gs_model_spec* model, const gs_machine_spec* machine, int num_microbatches,
                          double alpha, int steps, gs_planner_solution* out) {
  return guarded([&] {
    solution_out(offsim::grid_search_config(model_of(model), machine_of(machine), num_microbatches, alpha, steps),
                 out);
  });
}
int gs_io_roofline(const gs_model_spec* model, const gs_machine_spec* machine, unsigned long long batch_samples,
                   double x_opt, double* out) {
  return guarded([&] { *out = offsim::io_roofline(model_of(model), machine_of(machine), batch_samples, x_opt); });
}
int gs_compute_roofline(const gs_model_spec* model, const gs_machine_spec* machine, double* out) {
  return guarded([&] { *out = offsim::compute_roofline(model_of(model), machine_of(machine)); });
}
int gs_solve_lp(int m, int n, const double* A, const double* b, const double* c, int* feasible, int* bounded,
                double* objective, double* x) {
  return guarded([&] {
    if (m < 0 || n < 1 || (m > 0 && (!A || !b)) || !c) throw offsim::ValidationError("solve_lp: bad arguments");
    std::vector<std::vector<double>> a(static_cast<size_t>(m), std::vector<double>(static_cast<size_t>(n)));
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) a[static_cast<size_t>(i)][static_cast<size_t>(j)] = A[i * n + j];
    const offsim::LpResult r = offsim::solve_lp(a, std::vector<double>(b, b + m), std::vector<double>(c, c + n));
    if (feasible) *feasible = r.feasible ? 1 : 0;
    if (bounded) *bounded = r.bounded ? 1 : 0;
    if (objective) *objective = r.objective;
    if (x)
      for (int j = 0; j < n; ++j) x[j] = j < static_cast<int>(r.x.size()) ? r.x[static_cast<size_t>(j)] : 0.0;
  });
}

// ------------------------------------------------------------------ engine
int gs_engine_create(const gs_plan* plan, const gs_engine_config* c, gs_engine** out) {
  return guarded([&] {
    if (!plan || !c || !out) throw offsim::ValidationError("engine: NULL argument");
    offsim::ExecConfig cfg;
    cfg.model = model_of(&c->model);
    cfg.vocab_size = c->vocab_size;
    cfg.adam = {c->lr, c->beta1, c->beta2, c->eps, c->weight_decay};
    cfg.seed = c->seed;
    cfg.device = c->device;
    cfg.nvme_dir = c->nvme_dir ? c->nvme_dir : "/tmp";
    cfg.odirect = c->odirect != 0;
    cfg.opt_tier = static_cast<offsim::OptTier>(c->opt_tier);
    cfg.record_trace = c->record_trace != 0;
    cfg.profile_kernels = c->profile_kernels != 0;
    cfg.rank = c->rank;
    cfg.world = c->world > 0 ? c->world : 1;
    if (c->comm_id) cfg.comm_id.assign(c->comm_id, c->comm_id + 128);
    cfg.force_collectives = c->force_collectives != 0;
    if (c->ssd_ring_layers > 0) cfg.ssd_ring_layers = c->ssd_ring_layers;
    if (c->host_threads > 0) cfg.host_threads = c->host_threads;
    if (c->opt_tier < 0 || c->opt_tier > 3) throw offsim::ValidationError("engine: opt_tier must be 0..3");
    auto e = std::make_unique<gs_engine>();
    e->ex = std::make_unique<offsim::Executor>(plan->plan, cfg);
    *out = e.release();
  });
}
void gs_engine_destroy(gs_engine* engine) { delete engine; }
int gs_engine_run(gs_engine* engine, int iterations, const int32_t* tokens, int tokens_on_device, double* losses,
                  gs_run_report* report) {
  return guarded([&] {
    if (!engine) throw offsim::ValidationError("engine is NULL");
    const long long before = gs::launch_counter_ref();
    offsim::ExecReport r = engine->ex->run(iterations, tokens, tokens_on_device != 0);
    if (losses)
      for (int i = 0; i < iterations; ++i) losses[i] = r.losses[static_cast<size_t>(i)];
    engine->trace = r.trace;
    if (report) {
      report->total_ms = r.total_ms;
      report->iterations = iterations;
      report->gpu_launches = static_cast<int>(gs::launch_counter_ref() - before);
      ledger_out(r.ledger, report->ledger);
      ledger_out(r.extension, report->extension);
      ledger_out(r.physical, report->physical);
      report->gpu_bytes = r.gpu_bytes_allocated;
      report->host_pinned_bytes = r.host_pinned_bytes;
    }
  });
}
int gs_engine_flush(gs_engine* engine) { return guarded([&] { engine->ex->flush(); }); }
int gs_engine_read_params(gs_engine* engine, float* layers, float* fixed) {
  return guarded([&] { engine->ex->read_params(layers, fixed); });
}
int gs_engine_read_moments(gs_engine* engine, float* m, float* v) {
  return guarded([&] { engine->ex->read_moments(m, v); });
}
int gs_engine_read_fixed_moments(gs_engine* engine, float* m, float* v) {
  return guarded([&] {
    if (!engine) throw offsim::ValidationError("engine is NULL");
    engine->ex->read_moments(nullptr, nullptr, m, v);
  });
}
int gs_engine_kernel_profile(gs_engine* engine, double flops[5], double ms[5], int launches[5],
                             int64_t total_launches[5]) {
  return guarded([&] {
    const offsim::Executor::KernelTotals t = engine->ex->kernel_profile();
    for (int i = 0; i < 5; ++i) {
      flops[i] = t.flops[i];
      ms[i] = t.ms[i];
      launches[i] = t.launches[i];
      if (total_launches) total_launches[i] = t.total[i];
    }
  });
}
int gs_engine_gemm_span_profile(gs_engine* engine, double* flops, double* ms, int* launches) {
  return guarded([&] {
    const offsim::Executor::KernelTotals t = engine->ex->kernel_profile();
    *flops = t.span_flops;
    *ms = t.span_ms;
    *launches = t.span_launches;
  });
}
int gs_engine_set_profiling(gs_engine* engine, int stride) {
  return guarded([&] { engine->ex->set_profiling(stride); });
}
int gs_engine_set_trace(gs_engine* engine, int on) {
  return guarded([&] { engine->ex->set_trace(on != 0); });
}
int gs_engine_trace(gs_engine* engine, gs_trace_record* out, int cap, int* n) {
  return guarded([&] {
    *n = static_cast<int>(engine->trace.size());
    for (int i = 0; i < cap && i < *n; ++i) {
      const offsim::TraceRecord& r = engine->trace[static_cast<size_t>(i)];
      out[i] = {r.iteration, r.task, static_cast<int>(r.resource), r.t_start_ms, r.t_end_ms, r.bytes, r.physical_bytes,
                r.t_host_ms};
    }
  });
}

// ----------------------------------------------------------------- context
struct gs_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
};
int gs_ctx_create(int device, gs_ctx** out) {
  if (!out) return fail(GS_ERR_VALIDATION, "gs_ctx_create: out is null");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
    (void)cudaGetLastError();
    return fail(GS_ERR_CUDA, "gs_ctx_create: no CUDA device " + std::to_string(device));
  }
  auto c = std::make_unique<gs_ctx>();
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(GS_ERR_CUDA, std::string("gs_ctx_create: ") + cudaGetErrorString(cudaGetLastError()));
  *out = c.release();
  return GS_OK;
}
void* gs_ctx_stream(const gs_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }
int gs_ctx_sync(gs_ctx* ctx) {
  if (!ctx) return fail(GS_ERR_VALIDATION, "gs_ctx_sync: null context");
  return cuda_status(cudaStreamSynchronize(ctx->stream));
}
void gs_ctx_destroy(gs_ctx* ctx) {
  if (!ctx) return;
  if (ctx->stream) {
    cudaSetDevice(ctx->device);
    cudaStreamDestroy(ctx->stream);
  }
  delete ctx;
}

// ----------------------------------------------------------------- kernels
static int gemm_common(bool simt, int dtype, int M, int N, int K, const void* A, int a_k, const void* B, int b_k,
                       void* C, const void* R, void* G, int epi, void* stream) {
  if (epi < 0 || epi > static_cast<int>(gs::Epi::Gelu)) {
    g_error = "gs_gemm: unknown epilogue " + std::to_string(epi);
    return GS_ERR_VALIDATION;
  }
  gs::GemmArgs g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.A = A;
  g.B = B;
  g.a_kmajor = a_k != 0;
  g.b_kmajor = b_k != 0;
  g.C = C;
  g.R = R;
  g.G = G;
  g.epi = static_cast<gs::Epi>(epi);
  g.dt = dt_of(dtype);
  return cuda_status(simt ? gs::gemm_simt(g, static_cast<cudaStream_t>(stream))
                          : gs::gemm(g, static_cast<cudaStream_t>(stream)));
}
int gs_gemm(int dtype, int M, int N, int K, const void* A, int a_k, const void* B, int b_k, void* C, const void* R,
            void* G, int epi, void* stream) {
  return gemm_common(false, dtype, M, N, K, A, a_k, B, b_k, C, R, G, epi, stream);
}
int gs_gemm_simt(int dtype, int M, int N, int K, const void* A, int a_k, const void* B, int b_k, void* C,
                 const void* R, void* G, int epi, void* stream) {
  return gemm_common(true, dtype, M, N, K, A, a_k, B, b_k, C, R, G, epi, stream);
}
int gs_attention_fwd(int dtype, const void* qkv, void* o, float* lse, int b, int s, int h, int heads, void* stream) {
  return cuda_status(gs::attention_fwd(dt_of(dtype), qkv, o, lse, b, s, h, heads, static_cast<cudaStream_t>(stream)));
}
size_t gs_attention_bwd_workspace(int b, int s, int h, int heads) { return gs::attention_bwd_workspace(b, s, h, heads); }
int gs_attention_bwd(int dtype, const void* qkv, const void* o, const float* lse, const void* dout, void* dqkv,
                     void* work, int b, int s, int h, int heads, void* stream) {
  return cuda_status(gs::attention_bwd(dt_of(dtype), qkv, o, lse, dout, dqkv, work, b, s, h, heads,
                                       static_cast<cudaStream_t>(stream)));
}
int gs_layernorm_fwd(int dtype, const void* x, void* y, float* mean, float* rstd, int rows, int h, void* stream) {
  return cuda_status(gs::layernorm_fwd(dt_of(dtype), x, y, mean, rstd, rows, h, static_cast<cudaStream_t>(stream)));
}
int gs_layernorm_bwd(int dtype, const void* x, const float* mean, const float* rstd, const void* dy, void* dx,
                     int rows, int h, int accumulate, void* stream) {
  return cuda_status(gs::layernorm_bwd(dt_of(dtype), x, mean, rstd, dy, accumulate ? dx : nullptr, dx, rows, h,
                                       static_cast<cudaStream_t>(stream)));
}
int gs_adam_step_packed(float lr, float beta1, float beta2, float eps, float wd, int step, float grad_scale,
                        float* state, const float* grad, void* param_lp, int lp_dtype, int64_t n, void* stream) {
  gs::AdamHyper hp{lr, beta1, beta2, eps, wd};
  return cuda_status(gs::adam_step_packed(hp, step, grad_scale, state, grad, param_lp, dt_of(lp_dtype), n,
                                          static_cast<cudaStream_t>(stream)));
}
static int layer_call(int dtype, int b, int s, int h, int heads, bool fwd, const void* W, const void* x,
                      const void* dy, void* out, float* dW, int first, void* stream) {
  gs::engine::Dims d;
  d.b = b;
  d.s = s;
  d.h = h;
  d.H = heads;
  d.V = 128;  // head unused here
  d.dt = dt_of(dtype);
  gs::engine::Workspace ws;
  if (!gs::engine::alloc_workspace(d, ws)) return cuda_status(cudaErrorMemoryAllocation);
  gs::engine::LaunchCounter lc;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = fwd ? gs::engine::layer_forward(d, W, x, out, ws, st, lc)
                      : gs::engine::layer_backward(d, W, x, dy, out, dW, first != 0, nullptr, ws, st, lc);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  gs::engine::free_workspace(ws);
  return cuda_status(e);
}
int gs_layer_forward(int dtype, int b, int s, int h, int heads, const void* W, const void* x, void* y, void* stream) {
  return layer_call(dtype, b, s, h, heads, true, W, x, nullptr, y, nullptr, 0, stream);
}
int gs_layer_backward(int dtype, int b, int s, int h, int heads, const void* W, const void* x, const void* dy,
                      void* dx, float* dW, int first, void* stream) {
  return layer_call(dtype, b, s, h, heads, false, W, x, dy, dx, dW, first, stream);
}
int64_t gs_launch_count(void) { return gs::launch_counter_ref(); }

int gs_host_probe(int threads, uint64_t elements, double out[3]) {
  return guarded([&] {
    if (!out || elements < (1u << 20)) throw offsim::ValidationError("host_probe: elements >= 2^20 and out required");
    const int hw = static_cast<int>(std::thread::hardware_concurrency());
    const int nt = threads > 0 ? threads : std::max(1, hw - 4);
    gs::engine::ThreadPool pool(nt);
    gs::engine::PinnedArena arena;
    float* state = reinterpret_cast<float*>(arena.alloc(12 * elements));
    float* grad = reinterpret_cast<float*>(arena.alloc(4 * elements));
    uint16_t* lp = reinterpret_cast<uint16_t*>(arena.alloc(2 * elements));
    for (uint64_t i = 0; i < elements; ++i) {
      state[3 * i] = 0.01f * static_cast<float>(i % 97);
      grad[i] = 1e-3f * static_cast<float>(i % 13) - 6e-3f;
    }
    using clk = std::chrono::steady_clock;
    auto secs = [](clk::time_point t0) { return std::chrono::duration<double>(clk::now() - t0).count(); };
    // copy: state -> (grad | lp | spare state tail) pattern-free, 12 B/elem each way
    uint8_t* src = reinterpret_cast<uint8_t*>(state);
    uint8_t* dst = arena.alloc(12 * elements);
    double best_copy = 0.0, best_adam = 0.0;
    for (int rep = 0; rep < 3; ++rep) {
      std::vector<std::function<void()>> jobs;
      const uint64_t n = 12 * elements, per = (n / (4 * nt) + 4095) / 4096 * 4096;
      for (uint64_t lo = 0; lo < n; lo += per) {
        const uint64_t hi = std::min(n, lo + per);
        jobs.emplace_back([=] { std::memcpy(dst + lo, src + lo, hi - lo); });
      }
      auto t0 = clk::now();
      pool.run_all(jobs);
      best_copy = std::max(best_copy, 2.0 * n / secs(t0) / 1e9);
      const gs::engine::HostAdamHyper hp{1e-4f, 0.9f, 0.95f, 1e-8f, 0.0f};
      t0 = clk::now();
      gs::engine::host_adam_step(hp, rep + 1, state, grad, lp, 2, elements, pool);
      best_adam = std::max(best_adam, elements / secs(t0) / 1e9);
    }
    out[0] = best_copy;
    out[1] = best_adam;
    out[2] = nt;
  });
}

int gs_nvme_probe(const char* dir, uint64_t bytes, double out[3]) {
  return guarded([&] {
    if (!out || bytes < (64ull << 20)) throw offsim::ValidationError("nvme_probe: bytes >= 64 MiB and out required");
    gs::engine::NvmeFile f(dir ? dir : "/tmp", true, 8);
    const uint64_t half = gs::engine::align_up(bytes / 2, gs::engine::kNvmeAlign);
    const uint64_t a = f.reserve(half), b2 = f.reserve(half);
    f.finalize_size();
    gs::engine::PinnedArena arena;
    uint8_t* buf = arena.alloc(2 * half);
    for (uint64_t i = 0; i < 2 * half; i += 4096) buf[i] = static_cast<uint8_t>(i >> 12);
    using clk = std::chrono::steady_clock;
    auto secs = [](clk::time_point t0) { return std::chrono::duration<double>(clk::now() - t0).count(); };
    auto t0 = clk::now();
    f.write(a, buf, half);
    f.write(b2, buf + half, half);
    out[0] = 2.0 * half / secs(t0) / 1e9;  // sequential write GB/s
    t0 = clk::now();
    f.read(a, buf, half);
    f.read(b2, buf + half, half);
    out[1] = 2.0 * half / secs(t0) / 1e9;  // sequential read GB/s
    // both directions at once (the SSD_R and SSD_W queues run concurrently)
    t0 = clk::now();
    std::thread w([&] { f.write(a, buf, half); });
    f.read(b2, buf + half, half);
    w.join();
    out[2] = half / secs(t0) / 1e9;  // per-direction GB/s when concurrent
  });
}

int gs_layer_bench(int dtype, int b, int s, int h, int heads, int iters, double out[4]) {
  return guarded([&] {
    if (iters < 1 || !out) throw offsim::ValidationError("layer_bench: iters >= 1 and out required");
    gs::engine::Dims d;
    d.b = b;
    d.s = s;
    d.h = h;
    d.H = heads;
    d.V = 128;
    d.dt = dt_of(dtype);
    gs::engine::Workspace ws;
    if (!gs::engine::alloc_workspace(d, ws)) throw offsim::InfeasibleError("layer_bench: workspace");
    const size_t eb = static_cast<size_t>(d.lp()), T = static_cast<size_t>(d.T());
    void *W = nullptr, *x = nullptr, *y = nullptr, *dy = nullptr, *dx = nullptr;
    float* dW = nullptr;
    auto ok = [](cudaError_t e) {
      if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    };
    ok(cudaMalloc(&W, 12ull * h * h * eb));
    ok(cudaMalloc(&dW, 12ull * h * h * 4));
    for (void** p : {&x, &y, &dy, &dx}) ok(cudaMalloc(p, T * h * eb));
    // realistic operands (all-zero GEMMs draw less power and clock higher):
    // W ~ U(-0.02, 0.02), activations / gradients ~ U(-1, 1)
    auto fill = [&](void* p, size_t n, float amp) {
      std::vector<uint8_t> hbuf(n * eb);
      uint64_t st = 0x9E3779B97F4A7C15ull ^ n;
      for (size_t i = 0; i < n; ++i) {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        const float v = amp * (static_cast<float>(st >> 40) / 8388608.0f - 1.0f);
        if (eb == 2) {
          uint32_t u;
          std::memcpy(&u, &v, 4);
          const uint16_t b16 = static_cast<uint16_t>(u >> 16);
          std::memcpy(&hbuf[2 * i], &b16, 2);
        } else {
          std::memcpy(&hbuf[4 * i], &v, 4);
        }
      }
      ok(cudaMemcpy(p, hbuf.data(), n * eb, cudaMemcpyHostToDevice));
    };
    fill(W, 12ull * h * h, 0.02f);
    for (void* p : {x, y, dy, dx}) fill(p, T * h, 1.0f);
    cudaStream_t st;
    ok(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    ok(cudaEventCreate(&e0));
    ok(cudaEventCreate(&e1));
    gs::engine::LaunchCounter lc;
    for (int pass = 0; pass < 2; ++pass) {  // 0: forward, 1: recompute + backward
      for (int w = 0; w < 2; ++w)
        ok(pass == 0 ? gs::engine::layer_forward(d, W, x, y, ws, st, lc)
                     : gs::engine::layer_backward(d, W, x, dy, dx, dW, w == 0, nullptr, ws, st, lc));
      ok(cudaStreamSynchronize(st));
      ok(cudaEventRecord(e0, st));
      const auto h0 = std::chrono::steady_clock::now();
      for (int i = 0; i < iters; ++i)
        ok(pass == 0 ? gs::engine::layer_forward(d, W, x, y, ws, st, lc)
                     : gs::engine::layer_backward(d, W, x, dy, dx, dW, false, nullptr, ws, st, lc));
      const auto h1 = std::chrono::steady_clock::now();
      ok(cudaEventRecord(e1, st));
      ok(cudaEventSynchronize(e1));
      float ms = 0.f;
      ok(cudaEventElapsedTime(&ms, e0, e1));
      out[2 * pass] = ms / iters;                                                            // GPU ms per call
      out[2 * pass + 1] = std::chrono::duration<double, std::milli>(h1 - h0).count() / iters;  // host enqueue ms
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
    for (void* p : {W, x, y, dy, dx, static_cast<void*>(dW)}) cudaFree(p);
    gs::engine::free_workspace(ws);
  });
}

int gs_comm_unique_id(uint8_t out[128]) {
  return guarded([&] {
    if (!out) throw offsim::ValidationError("comm_unique_id: out required");
    const std::vector<uint8_t> id = gs::engine::peer_comm_unique_id();
    std::memcpy(out, id.data(), id.size());
  });
}

}  // extern "C"

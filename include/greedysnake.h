/* greedysnake.h — C-ABI of the B200-native GreedySnake hot path
 * (libgreedysnake.so, built in-tree by paper_2512_17570_b200/csrc/Makefile).
 *
 * Plain C types only: no torch, no C++ in the signatures.  Every function
 * returns an int status (GS_OK = 0) and never throws; the message of the last
 * failure on the calling thread is available from gs_last_error().  Status
 * codes mirror the reference CLI's exit codes (proj/tools/offsim_main.cpp:
 * 400-409): ValidationError -> 2, InfeasibleError -> 3, PlanBugError -> 1.
 *
 * Three layers:
 *  1. plan      — the reference's scheduler API (proj/include/offsim/
 *                 schedule.hpp:73-86, traffic.hpp:42-50, simulator.hpp:34)
 *                 over opaque handles: build_vertical / build_horizontal,
 *                 closed-form and plan-summed ledgers, the event simulator.
 *  2. engine    — the real B200 executor that replaces simulate(): runs a plan
 *                 with sm_100a kernels, PCIe DMA, NVMe I/O (offsim/executor.hpp).
 *  3. kernels   — device-pointer entry points of the hot kernels, asynchronous
 *                 on a caller stream (cudaStream_t passed as void*).
 * See INTEGRATION.md for the bindings a reference maintainer would add.
 */
#ifndef GREEDYSNAKE_H
#define GREEDYSNAKE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_OK 0
#define GS_ERR_PLAN_BUG 1   /* offsim::PlanBugError / internal inconsistency */
#define GS_ERR_VALIDATION 2 /* offsim::ValidationError: bad argument or config */
#define GS_ERR_INFEASIBLE 3 /* offsim::InfeasibleError: memory / residency caps */
#define GS_ERR_CUDA 4       /* CUDA runtime or launch failure */
#define GS_ERR_RUNTIME 5    /* I/O and other runtime failures */

const char* gs_last_error(void);
const char* gs_version(void);

/* ------------------------------------------------------------------ plan */
/* offsim::ModelSpec (proj/include/offsim/model.hpp:11-23) */
typedef struct gs_model_spec {
  int num_layers, hidden_dim, num_heads, seq_len, microbatch_size;
  int low_precision_bytes, full_precision_bytes, optimizer_states_per_element, data_parallel_degree;
} gs_model_spec;

/* offsim::StorageSplit (schedule.hpp:22-29): CPU-resident fractions */
typedef struct gs_split {
  double x_ckpt, x_param, x_opt;
} gs_split;

/* offsim::MachineSpec (machine.hpp:12-33) */
typedef struct gs_machine_spec {
  uint64_t gpu_mem_bytes, cpu_usable_dram_bytes;
  double pcie_h2d_bw, pcie_d2h_bw, ssd_read_bw, ssd_write_bw;
  double fwd_compute_time_per_layer_per_mb, bwd_compute_time_per_layer_per_mb;
  double cpu_step_throughput, fixed_overhead_time;
  int num_gpus;
  uint64_t gpu_working_set_bytes;
  int ssd_duplex;
} gs_machine_spec;

/* offsim::Task (schedule.hpp:41-56); kind/data/link numbered as the enums */
typedef struct gs_task {
  int id, kind, layer, microbatch, stage, data, link;
  uint64_t bytes, elements;
  int cross_iter_dep, num_deps;
} gs_task;

typedef struct gs_plan gs_plan; /* opaque offsim::SchedulePlan */

/* build_vertical(model, M, split, alpha)   schedule.hpp:79-80 */
int gs_plan_build_vertical(const gs_model_spec* model, int num_microbatches, const gs_split* split, double alpha,
                           gs_plan** out);
/* build_horizontal(model, M, split)        schedule.hpp:73-74 */
int gs_plan_build_horizontal(const gs_model_spec* model, int num_microbatches, const gs_split* split, gs_plan** out);
/* plan_from_json(json)                     json_io.hpp:29 */
int gs_plan_from_json(const char* json, gs_plan** out);
void gs_plan_free(gs_plan* plan);
int gs_plan_num_tasks(const gs_plan* plan);
/* SchedulePlan header fields (schedule.hpp:58-71): variant (0 single-fb,
   1 horizontal, 2 vertical), delay ratio, micro-batches, layers */
int gs_plan_info(const gs_plan* plan, int* variant, double* alpha, int* num_microbatches, int* num_layers);
int gs_plan_task(const gs_plan* plan, int index, gs_task* out);
/* deps of task `index` into out[0..cap) ; *n = number of deps */
int gs_plan_task_deps(const gs_plan* plan, int index, int* out, int cap, int* n);
/* plan_to_json(plan).dump() into buf (NUL-terminated); *len = bytes needed */
int gs_plan_to_json(const gs_plan* plan, char* buf, size_t cap, size_t* len);
/* ledger[link*5 + data], links H2D,D2H,SSD_read,SSD_write; data param,ckpt,
   grad_accum,interlayer_grad,opt_state   (traffic.hpp:14-36) */
int gs_plan_traffic(const gs_plan* plan, uint64_t ledger[20]);
int gs_vertical_traffic(const gs_model_spec* model, int num_microbatches, const gs_split* split, double alpha,
                        uint64_t ledger[20]);
int gs_horizontal_traffic(const gs_model_spec* model, int num_microbatches, const gs_split* split,
                          uint64_t ledger[20]);
int64_t gs_plan_overlap_window(const gs_plan* plan);
/* report_to_json(simulate(plan, machine)).dump()   simulator.hpp:34 */
int gs_simulate_json(const gs_plan* plan, const gs_machine_spec* machine, char* buf, size_t cap, size_t* len);

/* ---------------------------------------------------------------- planner
 * offsim::PlannerSolution (planner.hpp:13-22 of the reference) */
typedef struct gs_planner_solution {
  int feasible, num_microbatches;
  double alpha;
  gs_split split;
  double t_fwd_stage, t_bwd_stage, iteration_estimate, throughput_estimate;
} gs_planner_solution;
/* solve_config(model, machine, M, alpha)              planner.hpp:27-28 */
int gs_solve_config(const gs_model_spec* model, const gs_machine_spec* machine, int num_microbatches, double alpha,
                    gs_planner_solution* out);
/* find_optimal_config(model, machine)                  planner.hpp:33 */
int gs_find_optimal_config(const gs_model_spec* model, const gs_machine_spec* machine, gs_planner_solution* out);
/* grid_search_config(model, machine, M, alpha, steps)  planner.hpp:38-40 */
int gs_grid_search_config(const gs_model_spec* model, const gs_machine_spec* machine, int num_microbatches,
                          double alpha, int steps, gs_planner_solution* out);
/* io_roofline(model, machine, batch_samples, x_opt) -> samples/s    roofline.hpp:12-13
   (+inf when no optimizer state is SSD-resident);
   compute_roofline(model, machine) -> samples/s                      roofline.hpp:17 */
int gs_io_roofline(const gs_model_spec* model, const gs_machine_spec* machine, unsigned long long batch_samples,
                   double x_opt, double* out);
int gs_compute_roofline(const gs_model_spec* model, const gs_machine_spec* machine, double* out);
/* solve_lp(A, b, c) over dense row-major A [m][n]; x[n]  simplex.hpp:17 */
int gs_solve_lp(int m, int n, const double* A, const double* b, const double* c, int* feasible, int* bounded,
                double* objective, double* x);

/* ---------------------------------------------------------------- engine */
typedef struct gs_engine_config {
  gs_model_spec model;     /* low_precision_bytes: 2 = bf16 training, 4 = fp32 parity mode */
  int vocab_size;          /* tied embedding / LM head (FixedOps) */
  float lr, beta1, beta2, eps, weight_decay;
  uint64_t seed;
  int device;
  const char* nvme_dir;    /* directory for the NVMe tier file (NULL -> "/tmp") */
  int odirect;             /* 1: O_DIRECT on the NVMe tier */
  int opt_tier;            /* 0 auto, 1 HBM, 2 pinned DRAM streamed through HBM, 3 pinned DRAM stepped by host cores */
  int record_trace;
  int profile_kernels;     /* CUDA-event timing per kernel class (gs_engine_kernel_profile) */
  int rank, world;         /* ZeRO-3 data parallelism: model.data_parallel_degree == world */
  const uint8_t* comm_id;  /* 128-byte job id from gs_comm_unique_id() on rank 0 (world > 1): peer-memory rendezvous */
  int force_collectives;   /* run the sharded / peer-memory path even at world == 1 (tests) */
  int ssd_ring_layers;     /* pinned staging slots per SSD-resident data kind (0 -> 8) */
  int host_threads;        /* opt_tier 3: host optimizer threads (0 -> hardware threads - 4) */
} gs_engine_config;

/* 128 random bytes naming a data-parallel job's peer-memory communicator
   (rank 0 draws them; every rank passes the same bytes as comm_id) */
int gs_comm_unique_id(uint8_t out[128]);

typedef struct gs_run_report {
  double total_ms;          /* CUDA-event time of the whole run */
  int iterations;
  int gpu_launches;         /* kernels launched during the run */
  uint64_t ledger[20];      /* logical bytes of the last iteration (== gs_plan_traffic) */
  uint64_t extension[20];   /* GPU-optimizer traffic outside the reference model */
  uint64_t physical[20];    /* bytes physically moved (NVMe rounded to 4 KiB) */
  uint64_t gpu_bytes, host_pinned_bytes;
} gs_run_report;

typedef struct gs_trace_record {
  int iteration, task, resource;
  double t_start_ms, t_end_ms;
  uint64_t bytes, physical_bytes;
  double t_host_ms;  /* host time the dispatcher began enqueueing the task (its dependencies dispatched) */
} gs_trace_record;

typedef struct gs_engine gs_engine; /* opaque offsim::Executor */

/* Executor(plan, cfg): allocates HBM / pinned DRAM / NVMe state, initialises
   weights from cfg->seed.  The plan may be freed afterwards. */
int gs_engine_create(const gs_plan* plan, const gs_engine_config* cfg, gs_engine** out);
void gs_engine_destroy(gs_engine* engine);
/* Runs `iterations` chained iterations.  tokens: int32 [iterations][M][b][s+1]
   in host memory (tokens_on_device = 0) or device memory (= 1).
   losses (optional): per-iteration mean cross-entropy. */
int gs_engine_run(gs_engine* engine, int iterations, const int32_t* tokens, int tokens_on_device, double* losses,
                  gs_run_report* report);
/* apply the pending alpha slice + embedding step */
int gs_engine_flush(gs_engine* engine);
/* fp32 master weights: layers [N][12 h^2], fixed [(V + s) h]; either may be NULL */
int gs_engine_read_params(gs_engine* engine, float* layers, float* fixed);
int gs_engine_read_moments(gs_engine* engine, float* layer_m, float* layer_v);
/* fp32 Adam moments of the embedding / position table [(V+s)*h] (either may be NULL) */
int gs_engine_read_fixed_moments(gs_engine* engine, float* m, float* v);
/* per kernel class of the last run: 0 gemm, 1 attention_fwd, 2 attention_bwd,
   3 layernorm, 4 other — algorithmic flops, CUDA-event ms and count of the
   sampled launches, and all launches of the class */
int gs_engine_kernel_profile(gs_engine* engine, double flops[5], double ms[5], int launches[5],
                             int64_t total_launches[5]);
/* tcgen05 GEMM launches of the last run sampled by in-kernel %globaltimer
   span (first CTA start .. last CTA exit; one in `stride`, none of them
   event-timed): algorithmic flops, summed span ms, sampled launches */
int gs_engine_gemm_span_profile(gs_engine* engine, double* flops, double* ms, int* launches);
/* time one launch in `stride` per kernel class during later runs (0 = off) */
int gs_engine_set_profiling(gs_engine* engine, int stride);
/* record the per-task trace during later runs */
int gs_engine_set_trace(gs_engine* engine, int on);
/* trace of the last run (last <= 3 iterations when record_trace was set) */
int gs_engine_trace(gs_engine* engine, gs_trace_record* out, int cap, int* n);

/* --------------------------------------------------------------- context */
/* One context per device: selects the device and owns a non-blocking stream
   the kernel entry points below can be given (gs_ctx_stream). */
typedef struct gs_ctx gs_ctx;
int gs_ctx_create(int device, gs_ctx** out);
void* gs_ctx_stream(const gs_ctx* ctx);
int gs_ctx_sync(gs_ctx* ctx);
void gs_ctx_destroy(gs_ctx* ctx);

/* --------------------------------------------------------------- kernels */
/* dtype: 0 = fp32, 1 = bf16.  stream: cudaStream_t (NULL = legacy default). */
/* C[M,N] = sum_k A(m,k) B(n,k);  a_kmajor: A is [M][K] else [K][M];
   b_kmajor: B is [N][K] else [K][N].  epi: 0 store, 1 store + residual R,
   2 fp32 accumulate (C fp32), 3 store + gelu to G, 4 fp32 store,
   5 C = acc * gelu'(R), 6 C = gelu(acc).  Other values: GS_ERR_VALIDATION. */
int gs_gemm(int dtype, int M, int N, int K, const void* A, int a_kmajor, const void* B, int b_kmajor, void* C,
            const void* R, void* G, int epi, void* stream);
/* same, forcing the CUDA-core path (reference for the tcgen05 path) */
int gs_gemm_simt(int dtype, int M, int N, int K, const void* A, int a_kmajor, const void* B, int b_kmajor, void* C,
                 const void* R, void* G, int epi, void* stream);
int gs_attention_fwd(int dtype, const void* qkv, void* o, float* lse, int b, int s, int h, int heads, void* stream);
size_t gs_attention_bwd_workspace(int b, int s, int h, int heads);
int gs_attention_bwd(int dtype, const void* qkv, const void* o, const float* lse, const void* dout, void* dqkv,
                     void* workspace, int b, int s, int h, int heads, void* stream);
int gs_layernorm_fwd(int dtype, const void* x, void* y, float* mean, float* rstd, int rows, int h, void* stream);
int gs_layernorm_bwd(int dtype, const void* x, const float* mean, const float* rstd, const void* dy, void* dx,
                     int rows, int h, int accumulate, void* stream);
/* fused Adam(W) on packed [master, m, v] fp32 state (12 B/elem); writes the
   low-precision working copy to param_lp (dtype) when non-NULL */
int gs_adam_step_packed(float lr, float beta1, float beta2, float eps, float weight_decay, int step, float grad_scale,
                        float* state, const float* grad, void* param_lp, int lp_dtype, int64_t n, void* stream);
/* one layer forward / recompute+backward (the plan's FwdCompute / RecomputeAndBwd) */
int gs_layer_forward(int dtype, int b, int s, int h, int heads, const void* W, const void* x, void* y, void* stream);
int gs_layer_backward(int dtype, int b, int s, int h, int heads, const void* W, const void* x, const void* dy,
                      void* dx, float* dW, int first, void* stream);
/* diagnostics: `iters` back-to-back layer forwards, then recompute+backwards,
 * on one stream with preallocated buffers; out = {fwd GPU ms, fwd host enqueue
 * ms, bwd GPU ms, bwd host enqueue ms} per call */
int gs_layer_bench(int dtype, int b, int s, int h, int heads, int iters, double out[4]);
/* diagnostics: the NVMe tier's O_DIRECT bandwidth on a scratch file in `dir`
 * (`bytes` moved per direction): out = {write GB/s, read GB/s, per-direction
 * GB/s with reads and writes concurrent} */
int gs_nvme_probe(const char* dir, uint64_t bytes, double out[3]);
/* diagnostics: host DRAM as the host-core optimizer step sees it, on
 * `threads` workers (0 -> hardware threads - 4) over `elements` fp32 Adam
 * elements of pinned memory: out = {copy GB/s (read + write bytes), host
 * Adam Gelem/s (bf16 output, 30 B/element), threads used} */
int gs_host_probe(int threads, uint64_t elements, double out[3]);
/* number of device kernels launched through this library so far */
int64_t gs_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif

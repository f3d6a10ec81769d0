/* TEST INFRASTRUCTURE ONLY — numeric CPU oracle of the GreedySnake hot path.
 *
 * Plain C (fp32 storage, OpenMP over host cores).  It restates the training
 * arithmetic that the reference's plan tasks stand for (the reference itself
 * carries none):
 *   FwdCompute(l,m)       PAPER.md:563-564, :919-951   (layer forward)
 *   RecomputeAndBwd(l,m)  PAPER.md:566-567, :976-1033  (recompute + backward,
 *                         fp32 gradient accumulation across micro-batches)
 *   CpuStep(l,elements)   PAPER.md:571-584, :1035-1114 (Adam on the
 *                         (1-alpha) slice in backward, alpha slice delayed to
 *                         the next iteration's forward)
 *   FixedOps              proj/src/schedule.cpp:363 (embedding/head lump)
 * and executes a reference plan's compute tasks in plan order
 * (proj/src/schedule.cpp:280-518 emits them).  Layer = pre-LN GPT block with
 * exactly 12h^2 parameters (proj/src/model.cpp:29): bias-free QKV / out-proj /
 * FC1 / FC2, non-affine LayerNorm, causal softmax attention, tanh-GELU.
 *
 * Parity of this oracle is pinned against torch float64 autograd by
 * tools/make_golden.py -> tests/golden/ (tests/test_oracle.py).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may
 * load it; the product never does.
 */
#ifndef GS_ORACLE_H
#define GS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gso_cfg {
  int n_layers, hidden, heads, seq, mb_size, vocab;
} gso_cfg;

typedef struct gso_adam {
  float lr, beta1, beta2, eps, weight_decay;
} gso_adam;

/* Task kinds, numbered as offsim::TaskKind. */
enum { GSO_FWD = 0, GSO_BWD = 1, GSO_STEP = 2, GSO_XFER = 3, GSO_FIXED = 4 };
typedef struct gso_task {
  int kind, layer, mb, stage;
  long long elements;
} gso_task;

/* ---- deterministic synthetic data (shared bit-for-bit with the engine) */
uint64_t gso_splitmix64(uint64_t x);
double gso_normal(uint64_t seed, uint64_t stream, uint64_t index);
/* N(0,0.02) for wte/wpe and Wqkv/W1; N(0, 0.02/sqrt(2N)) for Wo/W2. */
void gso_init_fixed(const gso_cfg* c, uint64_t seed, float* wte, float* wpe);
void gso_init_layer(const gso_cfg* c, uint64_t seed, int layer, float* w);
/* tokens for one iteration: [M][b][s+1] ids uniform in [0, vocab) */
void gso_make_tokens(const gso_cfg* c, uint64_t seed, int iteration, int microbatches, int32_t* out);

/* ---- building blocks (row-major; T = b*s tokens of one micro-batch) */
void gso_embed_fwd(const gso_cfg* c, const float* wte, const float* wpe, const int32_t* tok,
                   float* x0);
void gso_layer_fwd(const gso_cfg* c, const float* w, const float* x, float* y);
/* recompute from x, then backward of dy; dw += layer grads; dx may alias dy */
void gso_layer_bwd(const gso_cfg* c, const float* w, const float* x, const float* dy, float* dx,
                   float* dw);
/* final LN + tied head + mean CE; returns summed CE over T tokens.
   dy = d(loss*scale)/dy, dwte += head grad. */
double gso_head(const gso_cfg* c, const float* wte, const float* y, const int32_t* tok, float scale,
                float* dy, float* dwte);
void gso_embed_bwd(const gso_cfg* c, const int32_t* tok, const float* dx0, float* dwte, float* dwpe);
/* Adam(W) on n elements; step is 1-based; grad is multiplied by grad_scale. */
void gso_adam_step(const gso_adam* a, float* p, float* m, float* v, const float* g, long long n,
                   int step, float grad_scale);

/* ---- plan-order training driver
 * tasks: the compute tasks (FWD/BWD/STEP/FIXED; XFER ignored) of one
 * iteration in plan order.  A STEP whose stage <= layer is the delayed alpha
 * slice (elements [P-e, P) of the previous iteration's gradients), otherwise
 * the immediate slice [0, e).  tokens: iters x [M][b][s+1].
 * params/m/v: N*12h^2 each; fixed*: (V+s)*h (wte then wpe).
 * flush != 0 applies the pending delayed slices and fixed step at the end.
 * Returns 0 on success. */
int gso_train(const gso_cfg* c, const gso_adam* a, int microbatches, const gso_task* tasks,
              int n_tasks, int iters, const int32_t* tokens, float* losses, float* params,
              float* opt_m, float* opt_v, float* fixed, float* fixed_m, float* fixed_v, int flush);

/* Plain reference loop (no plan): per iteration, all MBs fwd+bwd, then one
   full Adam step.  Used to check schedule invariance. */
int gso_train_plain(const gso_cfg* c, const gso_adam* a, int microbatches, int iters,
                    const int32_t* tokens, float* losses, float* params, float* opt_m,
                    float* opt_v, float* fixed, float* fixed_m, float* fixed_v);

int gso_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif

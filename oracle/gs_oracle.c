/* TEST INFRASTRUCTURE ONLY — numeric CPU oracle; see gs_oracle.h for scope
 * and the reference anchors.  fp32 storage, double where a reduction decides
 * the result (LayerNorm statistics, softmax normalisers, CE), OpenMP over
 * rows.  Deliberately simple: this is the checker, not the product. */
#include "gs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define LN_EPS 1e-5f
#define GELU_K 0.7978845608028654f /* sqrt(2/pi) */
#define GELU_C 0.044715f

int gso_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------ RNG */
uint64_t gso_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return gso_splitmix64(seed ^ gso_splitmix64(stream + 0x632BE59BD9B4E019ull));
}

double gso_normal(uint64_t seed, uint64_t stream, uint64_t index) {
  const uint64_t key = stream_key(seed, stream);
  const uint64_t a = gso_splitmix64(key + 2 * index), b = gso_splitmix64(key + 2 * index + 1);
  const double u1 = (double)((a >> 11) + 1) * 0x1.0p-53; /* (0,1] */
  const double u2 = (double)(b >> 11) * 0x1.0p-53;       /* [0,1) */
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

void gso_init_fixed(const gso_cfg* c, uint64_t seed, float* wte, float* wpe) {
  const long long nw = (long long)c->vocab * c->hidden, np = (long long)c->seq * c->hidden;
  for (long long i = 0; i < nw; ++i) wte[i] = (float)(0.02 * gso_normal(seed, 1, (uint64_t)i));
  for (long long i = 0; i < np; ++i) wpe[i] = (float)(0.02 * gso_normal(seed, 2, (uint64_t)i));
}

void gso_init_layer(const gso_cfg* c, uint64_t seed, int layer, float* w) {
  const long long h2 = (long long)c->hidden * c->hidden, p = 12 * h2;
  const double scaled = 0.02 / sqrt(2.0 * c->n_layers);
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < p; ++i) {
    /* [Wqkv 3h^2 | Wo h^2 | W1 4h^2 | W2 4h^2]; Wo and W2 are output projections */
    const int out_proj = (i >= 3 * h2 && i < 4 * h2) || i >= 8 * h2;
    w[i] = (float)((out_proj ? scaled : 0.02) * gso_normal(seed, 100 + (uint64_t)layer, (uint64_t)i));
  }
}

void gso_make_tokens(const gso_cfg* c, uint64_t seed, int iteration, int microbatches, int32_t* out) {
  const uint64_t key = stream_key(seed, 1000000ull + (uint64_t)iteration);
  const long long n = (long long)microbatches * c->mb_size * (c->seq + 1);
  for (long long i = 0; i < n; ++i) out[i] = (int32_t)(gso_splitmix64(key + (uint64_t)i) % (uint64_t)c->vocab);
}

/* --------------------------------------------------------------- GEMMs */
/* C[M,N] (+)= A[M,K] * B[K,N].  Rows go in blocks of four so each B row
 * loaded from memory feeds four accumulator rows; every C element still sums
 * over k in increasing order (the per-element arithmetic is unchanged). */
static void gemm_nn(const float* A, const float* B, float* C, int M, int N, int K, int accumulate) {
  const int nb = (M + 3) / 4;
#pragma omp parallel for schedule(static)
  for (int ib = 0; ib < nb; ++ib) {
    const int i0 = 4 * ib, rows = M - i0 < 4 ? M - i0 : 4;
    float* c[4];
    const float* a[4];
    for (int r = 0; r < 4; ++r) {
      const int i = i0 + (r < rows ? r : 0);
      c[r] = C + (long long)i * N;
      a[r] = A + (long long)i * K;
    }
    for (int r = 0; r < rows; ++r)
      if (!accumulate) memset(c[r], 0, sizeof(float) * (size_t)N);
    if (rows == 4) {
      float *c0 = c[0], *c1 = c[1], *c2 = c[2], *c3 = c[3];
      for (int k = 0; k < K; ++k) {
        const float a0 = a[0][k], a1 = a[1][k], a2 = a[2][k], a3 = a[3][k];
        const float* b = B + (long long)k * N;
        for (int j = 0; j < N; ++j) {
          const float bj = b[j];
          c0[j] += a0 * bj;
          c1[j] += a1 * bj;
          c2[j] += a2 * bj;
          c3[j] += a3 * bj;
        }
      }
    } else {
      for (int r = 0; r < rows; ++r)
        for (int k = 0; k < K; ++k) {
          const float av = a[r][k];
          const float* b = B + (long long)k * N;
          for (int j = 0; j < N; ++j) c[r][j] += av * b[j];
        }
    }
  }
}

/* C[M,N] = A[M,K] * B[N,K]^T  (nn.Linear forward: B = weight [out,in]) */
static void gemm_nt(const float* A, const float* B, float* C, int M, int N, int K) {
  float* bt = (float*)malloc(sizeof(float) * (size_t)N * (size_t)K);
#pragma omp parallel for schedule(static)
  for (int k = 0; k < K; ++k)
    for (int j = 0; j < N; ++j) bt[(long long)k * N + j] = B[(long long)j * K + k];
  gemm_nn(A, bt, C, M, N, K, 0);
  free(bt);
}

/* C[M,N] += A[K,M]^T * B[K,N]  (weight gradient: A = dY, B = X); four
 * output rows per B row load, per-element order over k unchanged. */
static void gemm_tn_acc(const float* A, const float* B, float* C, int M, int N, int K) {
  const int nb = (M + 3) / 4;
#pragma omp parallel for schedule(static)
  for (int ib = 0; ib < nb; ++ib) {
    const int i0 = 4 * ib, rows = M - i0 < 4 ? M - i0 : 4;
    if (rows == 4) {
      float *c0 = C + (long long)i0 * N, *c1 = c0 + N, *c2 = c1 + N, *c3 = c2 + N;
      for (int k = 0; k < K; ++k) {
        const float* ar = A + (long long)k * M + i0;
        const float a0 = ar[0], a1 = ar[1], a2 = ar[2], a3 = ar[3];
        const float* b = B + (long long)k * N;
        for (int j = 0; j < N; ++j) {
          const float bj = b[j];
          c0[j] += a0 * bj;
          c1[j] += a1 * bj;
          c2[j] += a2 * bj;
          c3[j] += a3 * bj;
        }
      }
    } else {
      for (int r = 0; r < rows; ++r) {
        float* c = C + (long long)(i0 + r) * N;
        for (int k = 0; k < K; ++k) {
          const float av = A[(long long)k * M + i0 + r];
          const float* b = B + (long long)k * N;
          for (int j = 0; j < N; ++j) c[j] += av * b[j];
        }
      }
    }
  }
}

/* ---------------------------------------------------------- LayerNorm */
static void ln_fwd(const float* x, float* y, float* mean, float* rstd, int rows, int h) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    const float* xr = x + (long long)r * h;
    double s = 0, ss = 0;
    for (int i = 0; i < h; ++i) s += xr[i];
    const double mu = s / h;
    for (int i = 0; i < h; ++i) ss += (xr[i] - mu) * (xr[i] - mu);
    const float rs = (float)(1.0 / sqrt(ss / h + LN_EPS));
    mean[r] = (float)mu;
    rstd[r] = rs;
    for (int i = 0; i < h; ++i) y[(long long)r * h + i] = (xr[i] - (float)mu) * rs;
  }
}

/* dx (+)= LN backward of dy at the saved statistics */
static void ln_bwd(const float* x, const float* mean, const float* rstd, const float* dy, float* dx,
                   int rows, int h, int accumulate) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    const float* xr = x + (long long)r * h;
    const float* g = dy + (long long)r * h;
    double sg = 0, sgx = 0;
    for (int i = 0; i < h; ++i) {
      const double xh = (double)(xr[i] - mean[r]) * rstd[r];
      sg += g[i];
      sgx += g[i] * xh;
    }
    const float mg = (float)(sg / h), mgx = (float)(sgx / h);
    float* d = dx + (long long)r * h;
    for (int i = 0; i < h; ++i) {
      const float xh = (xr[i] - mean[r]) * rstd[r];
      const float v = rstd[r] * (g[i] - mg - xh * mgx);
      d[i] = accumulate ? d[i] + v : v;
    }
  }
}

/* ---------------------------------------------------------- attention */
/* qkv [T,3h] with q|k|v column blocks; head j owns columns j*d..j*d+d-1 of
   each block.  o [T,h]; lse [b*H*s] log-sum-exp of the scaled scores. */
static void attn_fwd(const gso_cfg* c, const float* qkv, float* o, float* lse) {
  const int s = c->seq, h = c->hidden, H = c->heads, d = h / H, b = c->mb_size;
  const float scale = 1.0f / sqrtf((float)d);
  if (d > 128) abort(); /* head_dim <= 128, as the executor requires */
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int bh = 0; bh < b * H; ++bh)
    for (int t = 0; t < s; ++t) {
      const int bi = bh / H, j = bh % H;
      const float* q = qkv + ((long long)(bi * s + t)) * 3 * h + j * d;
      double* p = (double*)malloc(sizeof(double) * (size_t)(t + 1));
      double mx = -1e300;
      for (int u = 0; u <= t; ++u) {
        const float* k = qkv + ((long long)(bi * s + u)) * 3 * h + h + j * d;
        double acc = 0;
        for (int e = 0; e < d; ++e) acc += (double)q[e] * k[e];
        p[u] = acc * scale;
        if (p[u] > mx) mx = p[u];
      }
      double z = 0;
      for (int u = 0; u <= t; ++u) z += exp(p[u] - mx);
      for (int u = 0; u <= t; ++u) p[u] = exp(p[u] - mx) / z; /* probabilities */
      double acc[128];
      for (int e = 0; e < d; ++e) acc[e] = 0;
      for (int u = 0; u <= t; ++u) { /* each output element sums over u in increasing order */
        const float* v = qkv + ((long long)(bi * s + u)) * 3 * h + 2 * h + j * d;
        for (int e = 0; e < d; ++e) acc[e] += p[u] * v[e];
      }
      float* out = o + ((long long)(bi * s + t)) * h + j * d;
      for (int e = 0; e < d; ++e) out[e] = (float)acc[e];
      lse[(long long)bh * s + t] = (float)(mx + log(z));
      free(p);
    }
}

static void attn_bwd(const gso_cfg* c, const float* qkv, const float* o, const float* lse,
                     const float* dout, float* dqkv) {
  const int s = c->seq, h = c->hidden, H = c->heads, d = h / H, b = c->mb_size;
  const float scale = 1.0f / sqrtf((float)d);
  memset(dqkv, 0, sizeof(float) * (size_t)b * s * 3 * h);
#pragma omp parallel for schedule(dynamic)
  for (int bh = 0; bh < b * H; ++bh) {
    const int bi = bh / H, j = bh % H;
    for (int t = 0; t < s; ++t) {
      const long long row_t = (long long)(bi * s + t);
      const float* q = qkv + row_t * 3 * h + j * d;
      const float* dO = dout + row_t * h + j * d;
      const float* O = o + row_t * h + j * d;
      double D = 0;
      for (int e = 0; e < d; ++e) D += (double)dO[e] * O[e];
      float* dq = dqkv + row_t * 3 * h + j * d;
      for (int u = 0; u <= t; ++u) {
        const long long row_u = (long long)(bi * s + u);
        const float* k = qkv + row_u * 3 * h + h + j * d;
        const float* v = qkv + row_u * 3 * h + 2 * h + j * d;
        double sc = 0, dp = 0;
        for (int e = 0; e < d; ++e) {
          sc += (double)q[e] * k[e];
          dp += (double)dO[e] * v[e];
        }
        const double p = exp(sc * scale - lse[(long long)bh * s + t]);
        const double ds = p * (dp - D);
        float* dk = dqkv + row_u * 3 * h + h + j * d;
        float* dv = dqkv + row_u * 3 * h + 2 * h + j * d;
        for (int e = 0; e < d; ++e) {
          dq[e] += (float)(ds * scale * k[e]);
          dk[e] += (float)(ds * scale * q[e]);
          dv[e] += (float)(p * dO[e]);
        }
      }
    }
  }
}

/* --------------------------------------------------------------- GELU */
static inline float gelu(float u) {
  return 0.5f * u * (1.0f + tanhf(GELU_K * (u + GELU_C * u * u * u)));
}
static inline float gelu_grad(float u) {
  const float t = tanhf(GELU_K * (u + GELU_C * u * u * u));
  return 0.5f * (1.0f + t) + 0.5f * u * (1.0f - t * t) * GELU_K * (1.0f + 3.0f * GELU_C * u * u);
}

/* ------------------------------------------------------------- layer */
typedef struct acts {
  float *a, *qkv, *o, *lse, *x1, *c, *u, *g, *m1, *r1, *m2, *r2, *tmp;
} acts;

static void acts_alloc(const gso_cfg* c, acts* A) {
  const size_t T = (size_t)c->mb_size * c->seq, h = (size_t)c->hidden;
  A->a = malloc(sizeof(float) * T * h);
  A->qkv = malloc(sizeof(float) * T * 3 * h);
  A->o = malloc(sizeof(float) * T * h);
  A->lse = malloc(sizeof(float) * (size_t)c->mb_size * c->heads * c->seq);
  A->x1 = malloc(sizeof(float) * T * h);
  A->c = malloc(sizeof(float) * T * h);
  A->u = malloc(sizeof(float) * T * 4 * h);
  A->g = malloc(sizeof(float) * T * 4 * h);
  A->m1 = malloc(sizeof(float) * T);
  A->r1 = malloc(sizeof(float) * T);
  A->m2 = malloc(sizeof(float) * T);
  A->r2 = malloc(sizeof(float) * T);
  A->tmp = malloc(sizeof(float) * T * 4 * h);
}
static void acts_free(acts* A) {
  free(A->a); free(A->qkv); free(A->o); free(A->lse); free(A->x1); free(A->c);
  free(A->u); free(A->g); free(A->m1); free(A->r1); free(A->m2); free(A->r2); free(A->tmp);
}

static void layer_forward(const gso_cfg* c, const float* w, const float* x, float* y, acts* A) {
  const int T = c->mb_size * c->seq, h = c->hidden;
  const long long h2 = (long long)h * h;
  const float *wqkv = w, *wo = w + 3 * h2, *w1 = w + 4 * h2, *w2 = w + 8 * h2;
  ln_fwd(x, A->a, A->m1, A->r1, T, h);
  gemm_nt(A->a, wqkv, A->qkv, T, 3 * h, h);
  attn_fwd(c, A->qkv, A->o, A->lse);
  gemm_nt(A->o, wo, A->tmp, T, h, h);
  for (long long i = 0; i < (long long)T * h; ++i) A->x1[i] = x[i] + A->tmp[i];
  ln_fwd(A->x1, A->c, A->m2, A->r2, T, h);
  gemm_nt(A->c, w1, A->u, T, 4 * h, h);
  for (long long i = 0; i < (long long)T * 4 * h; ++i) A->g[i] = gelu(A->u[i]);
  gemm_nt(A->g, w2, A->tmp, T, h, 4 * h);
  if (y)
    for (long long i = 0; i < (long long)T * h; ++i) y[i] = A->x1[i] + A->tmp[i];
}

void gso_layer_fwd(const gso_cfg* c, const float* w, const float* x, float* y) {
  acts A;
  acts_alloc(c, &A);
  layer_forward(c, w, x, y, &A);
  acts_free(&A);
}

void gso_layer_bwd(const gso_cfg* c, const float* w, const float* x, const float* dy, float* dx,
                   float* dw) {
  const int T = c->mb_size * c->seq, h = c->hidden;
  const long long h2 = (long long)h * h, Th = (long long)T * h;
  const float *wqkv = w, *wo = w + 3 * h2, *w1 = w + 4 * h2, *w2 = w + 8 * h2;
  float *dwqkv = dw, *dwo = dw + 3 * h2, *dw1 = dw + 4 * h2, *dw2 = dw + 8 * h2;
  acts A;
  acts_alloc(c, &A);
  layer_forward(c, w, x, NULL, &A); /* recompute from the checkpoint */
  float* dx1 = malloc(sizeof(float) * (size_t)Th);
  float* dqkv = malloc(sizeof(float) * (size_t)Th * 3);
  float* big = malloc(sizeof(float) * (size_t)Th * 4);
  float* dyc = malloc(sizeof(float) * (size_t)Th);
  memcpy(dyc, dy, sizeof(float) * (size_t)Th); /* dx may alias dy */
  /* MLP */
  gemm_tn_acc(dyc, A.g, dw2, h, 4 * h, T);
  gemm_nn(dyc, w2, big, T, 4 * h, h, 0);                                  /* dg */
  for (long long i = 0; i < Th * 4; ++i) big[i] *= gelu_grad(A.u[i]);     /* du */
  gemm_tn_acc(big, A.c, dw1, 4 * h, h, T);
  gemm_nn(big, w1, A.tmp, T, h, 4 * h, 0);                                /* dc */
  memcpy(dx1, dyc, sizeof(float) * (size_t)Th);
  ln_bwd(A.x1, A.m2, A.r2, A.tmp, dx1, T, h, 1);
  /* attention */
  gemm_tn_acc(dx1, A.o, dwo, h, h, T);
  gemm_nn(dx1, wo, A.tmp, T, h, h, 0);                                    /* d o */
  attn_bwd(c, A.qkv, A.o, A.lse, A.tmp, dqkv);
  gemm_tn_acc(dqkv, A.a, dwqkv, 3 * h, h, T);
  gemm_nn(dqkv, wqkv, A.tmp, T, h, 3 * h, 0);                             /* da */
  memcpy(dx, dx1, sizeof(float) * (size_t)Th);
  ln_bwd(x, A.m1, A.r1, A.tmp, dx, T, h, 1);
  free(dx1); free(dqkv); free(big); free(dyc);
  acts_free(&A);
}

/* ------------------------------------------------------- embedding/head */
void gso_embed_fwd(const gso_cfg* c, const float* wte, const float* wpe, const int32_t* tok, float* x0) {
  const int s = c->seq, h = c->hidden;
  for (int bi = 0; bi < c->mb_size; ++bi)
    for (int t = 0; t < s; ++t) {
      const int id = tok[bi * (s + 1) + t];
      float* out = x0 + ((long long)bi * s + t) * h;
      for (int i = 0; i < h; ++i) out[i] = wte[(long long)id * h + i] + wpe[(long long)t * h + i];
    }
}

void gso_embed_bwd(const gso_cfg* c, const int32_t* tok, const float* dx0, float* dwte, float* dwpe) {
  const int s = c->seq, h = c->hidden;
  for (int bi = 0; bi < c->mb_size; ++bi)
    for (int t = 0; t < s; ++t) {
      const int id = tok[bi * (s + 1) + t];
      const float* g = dx0 + ((long long)bi * s + t) * h;
      for (int i = 0; i < h; ++i) {
        dwte[(long long)id * h + i] += g[i];
        dwpe[(long long)t * h + i] += g[i];
      }
    }
}

double gso_head(const gso_cfg* c, const float* wte, const float* y, const int32_t* tok, float scale,
                float* dy, float* dwte) {
  const int s = c->seq, h = c->hidden, V = c->vocab, T = c->mb_size * s;
  float* z = malloc(sizeof(float) * (size_t)T * h);
  float *mu = malloc(sizeof(float) * (size_t)T), *rs = malloc(sizeof(float) * (size_t)T);
  float* logits = malloc(sizeof(float) * (size_t)T * V);
  ln_fwd(y, z, mu, rs, T, h);
  gemm_nt(z, wte, logits, T, V, h);
  double total = 0;
  for (int r = 0; r < T; ++r) {
    const int bi = r / s, t = r % s;
    const int target = tok[bi * (s + 1) + t + 1];
    float* lr = logits + (long long)r * V;
    double mx = -1e300, zs = 0;
    for (int v = 0; v < V; ++v) mx = lr[v] > mx ? lr[v] : mx;
    for (int v = 0; v < V; ++v) zs += exp(lr[v] - mx);
    const double lse = mx + log(zs);
    total += lse - lr[target];
    for (int v = 0; v < V; ++v) lr[v] = (float)(exp(lr[v] - lse)) * scale; /* dlogits */
    lr[target] -= scale;
  }
  gemm_tn_acc(logits, z, dwte, V, h, T);
  float* dz = malloc(sizeof(float) * (size_t)T * h);
  gemm_nn(logits, wte, dz, T, h, V, 0);
  ln_bwd(y, mu, rs, dz, dy, T, h, 0);
  free(z); free(mu); free(rs); free(logits); free(dz);
  return total;
}

/* ----------------------------------------------------------------- Adam */
void gso_adam_step(const gso_adam* a, float* p, float* m, float* v, const float* g, long long n,
                   int step, float grad_scale) {
  const float bc1 = (float)(1.0 - pow((double)a->beta1, step));
  const float bc2 = (float)(1.0 - pow((double)a->beta2, step));
  const float b1 = a->beta1, b2 = a->beta2, lr = a->lr, eps = a->eps, wd = a->weight_decay;
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < n; ++i) {
    const float gi = g[i] * grad_scale;
    const float mi = b1 * m[i] + (1.0f - b1) * gi;
    const float vi = b2 * v[i] + (1.0f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const float mh = mi / bc1, vh = vi / bc2;
    p[i] = p[i] - lr * (mh / (sqrtf(vh) + eps) + wd * p[i]);
  }
}

/* ------------------------------------------------------ training driver */
typedef struct run {
  const gso_cfg* c;
  const gso_adam* a;
  int M;
  long long P, Th, nfixed;
  float *params, *om, *ov, *fixed, *fm, *fv;
  float *grads, *fgrads, *X, *D;
} run;

static int run_init(run* R, const gso_cfg* c, const gso_adam* a, int M, float* params, float* om,
                    float* ov, float* fixed, float* fm, float* fv) {
  R->c = c; R->a = a; R->M = M;
  R->P = 12LL * c->hidden * c->hidden;
  R->Th = (long long)c->mb_size * c->seq * c->hidden;
  R->nfixed = (long long)(c->vocab + c->seq) * c->hidden;
  R->params = params; R->om = om; R->ov = ov; R->fixed = fixed; R->fm = fm; R->fv = fv;
  R->grads = calloc((size_t)(c->n_layers * R->P), sizeof(float));
  R->fgrads = calloc((size_t)R->nfixed, sizeof(float));
  R->X = calloc((size_t)((c->n_layers + 1) * M * R->Th), sizeof(float));
  R->D = calloc((size_t)(M * R->Th), sizeof(float));
  return (R->grads && R->fgrads && R->X && R->D) ? 0 : 1;
}
static void run_free(run* R) { free(R->grads); free(R->fgrads); free(R->X); free(R->D); }
static float* ck(run* R, int l, int m) { return R->X + ((long long)l * R->M + m) * R->Th; }

static void fixed_step(run* R, int t) {
  gso_adam_step(R->a, R->fixed, R->fm, R->fv, R->fgrads, R->nfixed, t, 1.0f);
  memset(R->fgrads, 0, sizeof(float) * (size_t)R->nfixed);
}
static void layer_step(run* R, int l, long long lo, long long hi, int t) {
  const long long off = (long long)l * R->P + lo;
  gso_adam_step(R->a, R->params + off, R->om + off, R->ov + off, R->grads + off, hi - lo, t, 1.0f);
}

int gso_train(const gso_cfg* c, const gso_adam* a, int M, const gso_task* tasks, int n_tasks,
              int iters, const int32_t* tokens, float* losses, float* params, float* opt_m,
              float* opt_v, float* fixed, float* fixed_m, float* fixed_v, int flush) {
  run R;
  if (run_init(&R, c, a, M, params, opt_m, opt_v, fixed, fixed_m, fixed_v)) return 1;
  const int N = c->n_layers;
  const long long tok_per_mb = (long long)c->mb_size * (c->seq + 1);
  const float gscale = 1.0f / ((float)c->mb_size * c->seq * M);
  long long* delayed = calloc((size_t)N, sizeof(long long)); /* alpha slice size per layer */
  for (int i = 0; i < n_tasks; ++i)
    if (tasks[i].kind == GSO_STEP && tasks[i].stage <= tasks[i].layer) delayed[tasks[i].layer] = tasks[i].elements;
  int* started = calloc((size_t)N, sizeof(int));
  int fixed_pending = 0;
  float* wte = fixed;
  float* wpe = fixed + (long long)c->vocab * c->hidden;
  for (int it = 0; it < iters; ++it) {
    const int32_t* tok = tokens + (long long)it * M * tok_per_mb;
    double loss = 0;
    memset(started, 0, sizeof(int) * (size_t)N);
    for (int i = 0; i < n_tasks; ++i) {
      const gso_task* t = &tasks[i];
      const int l = t->layer, m = t->mb;
      switch (t->kind) {
        case GSO_FIXED:
          if (fixed_pending) fixed_step(&R, it);
          fixed_pending = 0;
          break;
        case GSO_FWD:
          if (l == 0) gso_embed_fwd(c, wte, wpe, tok + m * tok_per_mb, ck(&R, 0, m));
          gso_layer_fwd(c, params + (long long)l * R.P, ck(&R, l, m), ck(&R, l + 1, m));
          break;
        case GSO_BWD: {
          float* g = R.grads + (long long)l * R.P;
          if (!started[l]) {
            memset(g, 0, sizeof(float) * (size_t)R.P);
            started[l] = 1;
          }
          float* d = R.D + (long long)m * R.Th;
          if (l == N - 1)
            loss += gso_head(c, wte, ck(&R, N, m), tok + m * tok_per_mb, gscale, d, R.fgrads) /
                    ((double)c->mb_size * c->seq);
          gso_layer_bwd(c, params + (long long)l * R.P, ck(&R, l, m), d, d, g);
          if (l == 0)
            gso_embed_bwd(c, tok + m * tok_per_mb, d, R.fgrads, R.fgrads + (long long)c->vocab * c->hidden);
          break;
        }
        case GSO_STEP:
          if (t->stage <= l) { /* delayed alpha slice of the previous iteration */
            if (it > 0 && t->elements > 0) layer_step(&R, l, R.P - t->elements, R.P, it);
          } else if (t->elements > 0) {
            layer_step(&R, l, 0, t->elements, it + 1);
          }
          break;
        default:
          break;
      }
    }
    losses[it] = (float)(loss / M);
    fixed_pending = 1;
  }
  if (flush) {
    for (int l = 0; l < N; ++l)
      if (delayed[l] > 0) layer_step(&R, l, R.P - delayed[l], R.P, iters);
    if (fixed_pending) fixed_step(&R, iters);
  }
  free(delayed);
  free(started);
  run_free(&R);
  return 0;
}

int gso_train_plain(const gso_cfg* c, const gso_adam* a, int M, int iters, const int32_t* tokens,
                    float* losses, float* params, float* opt_m, float* opt_v, float* fixed,
                    float* fixed_m, float* fixed_v) {
  run R;
  if (run_init(&R, c, a, M, params, opt_m, opt_v, fixed, fixed_m, fixed_v)) return 1;
  const int N = c->n_layers;
  const long long tok_per_mb = (long long)c->mb_size * (c->seq + 1);
  const float gscale = 1.0f / ((float)c->mb_size * c->seq * M);
  float* wte = fixed;
  float* wpe = fixed + (long long)c->vocab * c->hidden;
  for (int it = 0; it < iters; ++it) {
    const int32_t* tok = tokens + (long long)it * M * tok_per_mb;
    memset(R.grads, 0, sizeof(float) * (size_t)(N * R.P));
    double loss = 0;
    for (int m = 0; m < M; ++m) {
      gso_embed_fwd(c, wte, wpe, tok + m * tok_per_mb, ck(&R, 0, m));
      for (int l = 0; l < N; ++l)
        gso_layer_fwd(c, params + (long long)l * R.P, ck(&R, l, m), ck(&R, l + 1, m));
      float* d = R.D;
      loss += gso_head(c, wte, ck(&R, N, m), tok + m * tok_per_mb, gscale, d, R.fgrads) /
              ((double)c->mb_size * c->seq);
      for (int l = N - 1; l >= 0; --l)
        gso_layer_bwd(c, params + (long long)l * R.P, ck(&R, l, m), d, d, R.grads + (long long)l * R.P);
      gso_embed_bwd(c, tok + m * tok_per_mb, d, R.fgrads, R.fgrads + (long long)c->vocab * c->hidden);
    }
    for (int l = 0; l < N; ++l) layer_step(&R, l, 0, R.P, it + 1);
    fixed_step(&R, it + 1);
    losses[it] = (float)(loss / M);
  }
  run_free(&R);
  return 0;
}

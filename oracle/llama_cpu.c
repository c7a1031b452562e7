/*
 * llama_cpu.c — TEST INFRASTRUCTURE ONLY: the CPU numeric oracle for the
 * training step.  Never linked into libmemo; only tests/, bench.py's CPU
 * baseline leg and __graft_entry__.smoke() load it, as the checker.
 *
 * Parity status: the reference (proj/, actmem v0.1.0) contains no model math
 * (SURVEY discovery 1), so this restatement is NOT pinned by the
 * reference.  It follows the paper's block description (PAPER.md:353-356,
 * 374: embedding -> n x {norm, causal MHA, residual, norm, FFN} -> classifier)
 * with the Llama specifics the north star names (RMSNorm, interleaved RoPE,
 * SwiGLU, untied head), and is pinned instead against torch fp64 autograd in
 * tests/test_oracle.py.
 *
 * Model definition (shared with the GPU path, bf16 storage points marked B()):
 *   x0 = E[tok]                                  (f32 residual stream)
 *   per layer:
 *     xn  = B(x * rstd(x) * g1)                  input_norm
 *     q,k,v = B(xn Wqkv^T); q,k = B(rope(q,k))   q, k, v
 *     o   = B(softmax(q k^T / sqrt(D), causal) v)  attn_out (+ lse)
 *     a   = B(o Wo^T);  x1 = x + a               attn_proj
 *     xn2 = B(x1 * rstd(x1) * g2)                post_attn_norm
 *     gu  = B(xn2 Wgu^T)  (gate rows [0,F), up rows [F,2F))   ffn_fc1
 *     act = B(silu(g) * u)                       ffn_act
 *     x   = x1 + B(act Wd^T)
 *   xf = B(x * rstd(x) * gf); logits = xf Wcls^T; loss = mean CE over labels >= 0
 * Everything else is computed in fp32 with fp64 reductions; gradients are
 * exact fp32/fp64 backprop of this definition.
 *
 * Weights come from a counter hash so CPU and GPU initialise bit-identically
 * (see memo_init_uniform in csrc/kernels/elementwise.cu).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int n_layers, hidden, n_heads, head_dim, ffn, vocab, seq;
  float eps, rope_theta;
} oc_cfg;

/* ------------------------------------------------------------ init */
static uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

static float bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return f; /* inf/nan untouched */
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}
#define B(x) bf16_rne(x)

/* uniform in [-1, 1) with 24-bit resolution, exact in fp32 */
static float unit_uniform(uint64_t seed, uint64_t tid, uint64_t idx) {
  uint64_t h = splitmix64(seed * 0x9E3779B97F4A7C15ULL + tid * 0xD1B54A32D192ED03ULL + idx);
  float u = (float)(h >> 40) * (1.0f / 16777216.0f);
  return 2.0f * u - 1.0f;
}

/* parameter layout (elements):
 *   E [V,h] | per layer: g1 [h], Wqkv [3h,h], Wo [h,h], g2 [h], Wgu [2F,h], Wd [h,F] | gf [h] | Wcls [V,h]
 * tensor ids: E=0, layer l: 1+6l+{0..5}, gf = 1+6n, Wcls = 2+6n */
static long long layer_params(const oc_cfg* c) {
  long long h = c->hidden, F = c->ffn;
  return h + 3 * h * h + h * h + h + 2 * F * h + h * F;
}
long long oc_param_count(const oc_cfg* c) {
  long long h = c->hidden, V = c->vocab;
  return V * h + c->n_layers * layer_params(c) + h + V * h;
}

static void fill(float* p, long long n, uint64_t seed, uint64_t tid, int is_norm) {
  for (long long i = 0; i < n; ++i) {
    float x = unit_uniform(seed, tid, (uint64_t)i);
    p[i] = is_norm ? B(1.0f + x * 0.1f) : B(x * 0.0346410161513775f);
  }
}

void oc_init(const oc_cfg* c, uint64_t seed, float* p) {
  long long h = c->hidden, V = c->vocab, F = c->ffn;
  float* q = p;
  fill(q, V * h, seed, 0, 0);
  q += V * h;
  for (int l = 0; l < c->n_layers; ++l) {
    uint64_t t = 1 + 6 * (uint64_t)l;
    fill(q, h, seed, t + 0, 1); q += h;
    fill(q, 3 * h * h, seed, t + 1, 0); q += 3 * h * h;
    fill(q, h * h, seed, t + 2, 0); q += h * h;
    fill(q, h, seed, t + 3, 1); q += h;
    fill(q, 2 * F * h, seed, t + 4, 0); q += 2 * F * h;
    fill(q, h * F, seed, t + 5, 0); q += h * F;
  }
  fill(q, h, seed, 1 + 6 * (uint64_t)c->n_layers, 1); q += h;
  fill(q, V * h, seed, 2 + 6 * (uint64_t)c->n_layers, 0);
}

void oc_tokens(uint64_t seed, int vocab, int seq, int* tokens, int* labels) {
  for (int i = 0; i < seq; ++i) tokens[i] = (int)(splitmix64(seed + (uint64_t)i) % (uint64_t)vocab);
  for (int i = 0; i < seq; ++i) labels[i] = i + 1 < seq ? tokens[i + 1] : -1;
}

/* ------------------------------------------------------------ primitives */
/* Y[M,N] = X[M,K] W[N,K]^T (f32 accumulate in double per output) */
static void mm_nt(const float* X, const float* W, float* Y, int M, int N, int K) {
#pragma omp parallel for schedule(static)
  for (int m = 0; m < M; ++m) {
    const float* x = X + (long long)m * K;
    for (int n = 0; n < N; ++n) {
      const float* w = W + (long long)n * K;
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)x[k] * w[k];
      Y[(long long)m * N + n] = (float)s;
    }
  }
}
/* dX[M,K] = dY[M,N] W[N,K] */
static void mm_nn(const float* dY, const float* W, float* dX, int M, int N, int K) {
#pragma omp parallel for schedule(static)
  for (int m = 0; m < M; ++m) {
    double* acc = (double*)calloc((size_t)K, sizeof(double));
    const float* dy = dY + (long long)m * N;
    for (int n = 0; n < N; ++n) {
      const double g = dy[n];
      if (g == 0) continue;
      const float* w = W + (long long)n * K;
      for (int k = 0; k < K; ++k) acc[k] += g * w[k];
    }
    for (int k = 0; k < K; ++k) dX[(long long)m * K + k] = (float)acc[k];
    free(acc);
  }
}
/* dW[N,K] += dY[M,N]^T X[M,K] */
static void mm_tn_acc(const float* dY, const float* X, float* dW, int M, int N, int K) {
#pragma omp parallel for schedule(static)
  for (int n = 0; n < N; ++n) {
    double* acc = (double*)calloc((size_t)K, sizeof(double));
    for (int m = 0; m < M; ++m) {
      const double g = dY[(long long)m * N + n];
      if (g == 0) continue;
      const float* x = X + (long long)m * K;
      for (int k = 0; k < K; ++k) acc[k] += g * x[k];
    }
    for (int k = 0; k < K; ++k) dW[(long long)n * K + k] += (float)acc[k];
    free(acc);
  }
}

static void rmsnorm_fwd(const float* x, const float* g, float* y, float* rstd, int S, int h,
                        float eps) {
#pragma omp parallel for schedule(static)
  for (int t = 0; t < S; ++t) {
    const float* xr = x + (long long)t * h;
    double ss = 0;
    for (int j = 0; j < h; ++j) ss += (double)xr[j] * xr[j];
    const float r = (float)(1.0 / sqrt(ss / h + eps));
    rstd[t] = r;
    for (int j = 0; j < h; ++j) y[(long long)t * h + j] = B(xr[j] * r * g[j]);
  }
}
/* dx += rmsnorm backward of y = x*r*g given dy; dg accumulated */
static void rmsnorm_bwd(const float* x, const float* g, const float* rstd, const float* dy,
                        float* dx, float* dg, int S, int h) {
  double* dgacc = (double*)calloc((size_t)h, sizeof(double));
#pragma omp parallel
  {
    double* loc = (double*)calloc((size_t)h, sizeof(double));
#pragma omp for schedule(static)
    for (int t = 0; t < S; ++t) {
      const float* xr = x + (long long)t * h;
      const float* d = dy + (long long)t * h;
      const double r = rstd[t];
      double dot = 0;
      for (int j = 0; j < h; ++j) dot += (double)d[j] * g[j] * xr[j];
      const double c = r * r * r * dot / h;
      for (int j = 0; j < h; ++j) {
        dx[(long long)t * h + j] += (float)(r * d[j] * g[j] - c * xr[j]);
        loc[j] += (double)d[j] * xr[j] * r;
      }
    }
#pragma omp critical
    for (int j = 0; j < h; ++j) dgacc[j] += loc[j];
    free(loc);
  }
  for (int j = 0; j < h; ++j) dg[j] += (float)dgacc[j];
  free(dgacc);
}

static void rope_table(const oc_cfg* c, float* cs) { /* [S][D/2][2] */
  const int D = c->head_dim, half = D / 2;
  for (int t = 0; t < c->seq; ++t)
    for (int p = 0; p < half; ++p) {
      const double inv = pow((double)c->rope_theta, -2.0 * p / D);
      const double ang = (double)t * inv;
      cs[((long long)t * half + p) * 2 + 0] = (float)cos(ang);
      cs[((long long)t * half + p) * 2 + 1] = (float)sin(ang);
    }
}
/* in-place rotation of interleaved pairs of a [S, H*D] tensor; inverse = transpose */
static void rope_apply(float* x, const float* cs, int S, int H, int D, int inverse, int round) {
  const int half = D / 2;
#pragma omp parallel for schedule(static)
  for (int t = 0; t < S; ++t)
    for (int hh = 0; hh < H; ++hh)
      for (int p = 0; p < half; ++p) {
        float* v = x + (long long)t * H * D + hh * D + 2 * p;
        const float c = cs[((long long)t * half + p) * 2], s = cs[((long long)t * half + p) * 2 + 1];
        const float a = v[0], b = v[1];
        float y0, y1;
        if (!inverse) {
          y0 = a * c - b * s;
          y1 = a * s + b * c;
        } else {
          y0 = a * c + b * s;
          y1 = -a * s + b * c;
        }
        v[0] = round ? B(y0) : y0;
        v[1] = round ? B(y1) : y1;
      }
}

/* causal attention fwd: o = B(softmax(q k^T * scale) v), lse[H][S] */
static void attn_fwd(const float* q, const float* k, const float* v, float* o, float* lse, int S,
                     int H, int D) {
  const double scale = 1.0 / sqrt((double)D);
  const int h = H * D;
#pragma omp parallel for schedule(dynamic, 16) collapse(2)
  for (int hh = 0; hh < H; ++hh)
    for (int t = 0; t < S; ++t) {
      double* p = (double*)malloc(sizeof(double) * (size_t)(t + 1));
      const float* qr = q + (long long)t * h + hh * D;
      double mx = -INFINITY;
      for (int u = 0; u <= t; ++u) {
        const float* kr = k + (long long)u * h + hh * D;
        double s = 0;
        for (int d = 0; d < D; ++d) s += (double)qr[d] * kr[d];
        p[u] = s * scale;
        if (p[u] > mx) mx = p[u];
      }
      double sum = 0;
      for (int u = 0; u <= t; ++u) {
        p[u] = exp(p[u] - mx);
        sum += p[u];
      }
      for (int d = 0; d < D; ++d) {
        double acc = 0;
        for (int u = 0; u <= t; ++u) acc += p[u] * v[(long long)u * h + hh * D + d];
        o[(long long)t * h + hh * D + d] = B((float)(acc / sum));
      }
      lse[(long long)hh * S + t] = (float)(mx + log(sum));
      free(p);
    }
}

/* causal attention bwd: dq, dk, dv (f32) */
static void attn_bwd(const float* q, const float* k, const float* v, const float* o,
                     const float* lse, const float* dout, float* dq, float* dk, float* dv, int S,
                     int H, int D) {
  const double scale = 1.0 / sqrt((double)D);
  const int h = H * D;
  memset(dq, 0, sizeof(float) * (size_t)S * h);
  memset(dk, 0, sizeof(float) * (size_t)S * h);
  memset(dv, 0, sizeof(float) * (size_t)S * h);
  for (int hh = 0; hh < H; ++hh) {
    double* delta = (double*)malloc(sizeof(double) * (size_t)S);
    for (int t = 0; t < S; ++t) {
      double s = 0;
      for (int d = 0; d < D; ++d)
        s += (double)dout[(long long)t * h + hh * D + d] * o[(long long)t * h + hh * D + d];
      delta[t] = s;
    }
    /* dq: rows; dk, dv: columns (separate passes keep the loops race free) */
#pragma omp parallel for schedule(dynamic, 16)
    for (int t = 0; t < S; ++t) {
      const float* qr = q + (long long)t * h + hh * D;
      const float* dor = dout + (long long)t * h + hh * D;
      double acc[256];
      for (int d = 0; d < D; ++d) acc[d] = 0;
      for (int u = 0; u <= t; ++u) {
        const float* kr = k + (long long)u * h + hh * D;
        const float* vr = v + (long long)u * h + hh * D;
        double s = 0, dp = 0;
        for (int d = 0; d < D; ++d) {
          s += (double)qr[d] * kr[d];
          dp += (double)dor[d] * vr[d];
        }
        const double p = exp(s * scale - lse[(long long)hh * S + t]);
        const double ds = p * (dp - delta[t]) * scale;
        for (int d = 0; d < D; ++d) acc[d] += ds * kr[d];
      }
      for (int d = 0; d < D; ++d) dq[(long long)t * h + hh * D + d] = (float)acc[d];
    }
#pragma omp parallel for schedule(dynamic, 16)
    for (int u = 0; u < S; ++u) {
      const float* kr = k + (long long)u * h + hh * D;
      const float* vr = v + (long long)u * h + hh * D;
      double ak[256], av[256];
      for (int d = 0; d < D; ++d) ak[d] = av[d] = 0;
      for (int t = u; t < S; ++t) {
        const float* qr = q + (long long)t * h + hh * D;
        const float* dor = dout + (long long)t * h + hh * D;
        double s = 0, dp = 0;
        for (int d = 0; d < D; ++d) {
          s += (double)qr[d] * kr[d];
          dp += (double)dor[d] * vr[d];
        }
        const double p = exp(s * scale - lse[(long long)hh * S + t]);
        const double ds = p * (dp - delta[t]) * scale;
        for (int d = 0; d < D; ++d) {
          av[d] += p * dor[d];
          ak[d] += ds * qr[d];
        }
      }
      for (int d = 0; d < D; ++d) {
        dk[(long long)u * h + hh * D + d] = (float)ak[d];
        dv[(long long)u * h + hh * D + d] = (float)av[d];
      }
    }
    free(delta);
  }
}

/* Attention alone (forward + backward of one causal multi-head attention over
 * [S, H*D] f32 inputs), for the CPU baseline's per-part timing (bench.py). */
int oc_attention(int S, int H, int D, const float* q, const float* k, const float* v,
                 const float* dout, float* o, float* lse, float* dq, float* dk, float* dv) {
  if (S <= 0 || H <= 0 || D <= 0 || D > 256) return 1;
  attn_fwd(q, k, v, o, lse, S, H, D);
  attn_bwd(q, k, v, o, lse, dout, dq, dk, dv, S, H, D);
  return 0;
}

/* ------------------------------------------------------------ step */
typedef struct {
  float *x, *xn, *rstd1, *q, *k, *v, *o, *lse, *a, *x1, *xn2, *rstd2, *gu, *act;
} oc_layer_acts;

static float* fz(long long n) { return (float*)calloc((size_t)n, sizeof(float)); }

/* Runs forward + backward.  params: oc_param_count floats (bf16 values);
 * grads: same layout, overwritten.  Returns 0 on success; *loss = mean CE.
 * If `acts_out` is non-NULL it receives the final hidden state xL [S,h]. */
int oc_step(const oc_cfg* c, const float* params, const int* tokens, const int* labels,
            float* grads, double* loss, float* acts_out) {
  const int S = c->seq, h = c->hidden, H = c->n_heads, D = c->head_dim, F = c->ffn,
            V = c->vocab, n = c->n_layers;
  const long long Sh = (long long)S * h;
  memset(grads, 0, sizeof(float) * (size_t)oc_param_count(c));
  const float* E = params;
  const float* Lp = params + (long long)V * h;
  const float* gf = Lp + n * layer_params(c);
  const float* Wcls = gf + h;
  float* dE = grads;
  float* dLp = grads + (long long)V * h;
  float* dgf = dLp + n * layer_params(c);
  float* dWcls = dgf + h;

  float* cs = fz((long long)S * D);
  rope_table(c, cs);
  oc_layer_acts* A = (oc_layer_acts*)calloc((size_t)n, sizeof(oc_layer_acts));
  float* x = fz(Sh);
  for (int t = 0; t < S; ++t)
    for (int j = 0; j < h; ++j) x[(long long)t * h + j] = E[(long long)tokens[t] * h + j];

  float* qkv = fz(3 * Sh);
  for (int l = 0; l < n; ++l) {
    const float* P = Lp + l * layer_params(c);
    const float *g1 = P, *Wqkv = g1 + h, *Wo = Wqkv + 3LL * h * h, *g2 = Wo + (long long)h * h,
                *Wgu = g2 + h, *Wd = Wgu + 2LL * F * h;
    oc_layer_acts* a = &A[l];
    a->x = x;
    a->xn = fz(Sh); a->rstd1 = fz(S);
    rmsnorm_fwd(x, g1, a->xn, a->rstd1, S, h, c->eps);
    mm_nt(a->xn, Wqkv, qkv, S, 3 * h, h);
    a->q = fz(Sh); a->k = fz(Sh); a->v = fz(Sh);
    for (int t = 0; t < S; ++t)
      for (int j = 0; j < h; ++j) {
        a->q[(long long)t * h + j] = B(qkv[(long long)t * 3 * h + j]);
        a->k[(long long)t * h + j] = B(qkv[(long long)t * 3 * h + h + j]);
        a->v[(long long)t * h + j] = B(qkv[(long long)t * 3 * h + 2 * h + j]);
      }
    rope_apply(a->q, cs, S, H, D, 0, 1);
    rope_apply(a->k, cs, S, H, D, 0, 1);
    a->o = fz(Sh); a->lse = fz((long long)H * S);
    attn_fwd(a->q, a->k, a->v, a->o, a->lse, S, H, D);
    a->a = fz(Sh);
    mm_nt(a->o, Wo, a->a, S, h, h);
    a->x1 = fz(Sh);
    for (long long i = 0; i < Sh; ++i) {
      a->a[i] = B(a->a[i]);
      a->x1[i] = x[i] + a->a[i];
    }
    a->xn2 = fz(Sh); a->rstd2 = fz(S);
    rmsnorm_fwd(a->x1, g2, a->xn2, a->rstd2, S, h, c->eps);
    a->gu = fz(2LL * S * F);
    mm_nt(a->xn2, Wgu, a->gu, S, 2 * F, h);
    /* gu rows are [gate(F) | up(F)] per token */
    a->act = fz((long long)S * F);
    for (long long t = 0; t < S; ++t)
      for (int j = 0; j < F; ++j) {
        float g = B(a->gu[t * 2 * F + j]), u = B(a->gu[t * 2 * F + F + j]);
        a->gu[t * 2 * F + j] = g;
        a->gu[t * 2 * F + F + j] = u;
        const float sg = 1.0f / (1.0f + expf(-g));
        a->act[t * F + j] = B(g * sg * u);
      }
    float* dd = fz(Sh);
    mm_nt(a->act, Wd, dd, S, h, F);
    float* xnext = fz(Sh);
    for (long long i = 0; i < Sh; ++i) xnext[i] = a->x1[i] + B(dd[i]);
    free(dd);
    x = xnext;
  }
  if (acts_out) memcpy(acts_out, x, sizeof(float) * (size_t)Sh);

  /* classifier + CE */
  float* rstdf = fz(S);
  float* xf = fz(Sh);
  rmsnorm_fwd(x, gf, xf, rstdf, S, h, c->eps);
  float* logits = fz((long long)S * V);
  mm_nt(xf, Wcls, logits, S, V, h);
  int n_lab = 0;
  for (int t = 0; t < S; ++t) n_lab += labels[t] >= 0;
  double total = 0;
  for (int t = 0; t < S; ++t) {
    float* row = logits + (long long)t * V;
    if (labels[t] < 0) {
      for (int j = 0; j < V; ++j) row[j] = 0;
      continue;
    }
    double mx = -INFINITY, sum = 0;
    for (int j = 0; j < V; ++j) mx = row[j] > mx ? row[j] : mx;
    for (int j = 0; j < V; ++j) sum += exp(row[j] - mx);
    total += (mx + log(sum)) - row[labels[t]];
    for (int j = 0; j < V; ++j) {
      double p = exp(row[j] - mx) / sum;
      row[j] = (float)((p - (j == labels[t] ? 1.0 : 0.0)) / n_lab);
    }
  }
  *loss = total / n_lab;
  float* dxf = fz(Sh);
  mm_nn(logits, Wcls, dxf, S, V, h);
  mm_tn_acc(logits, xf, dWcls, S, V, h);
  free(logits);
  float* dx = fz(Sh);
  rmsnorm_bwd(x, gf, rstdf, dxf, dx, dgf, S, h);
  free(dxf); free(xf); free(rstdf);
  if (n > 0) free(x); /* last layer output */

  float* tmp = fz(Sh);
  float* dqkv = fz(3 * Sh);
  for (int l = n - 1; l >= 0; --l) {
    const float* P = Lp + l * layer_params(c);
    const float *g1 = P, *Wqkv = g1 + h, *Wo = Wqkv + 3LL * h * h, *g2 = Wo + (long long)h * h,
                *Wgu = g2 + h, *Wd = Wgu + 2LL * F * h;
    float* dP = dLp + l * layer_params(c);
    float *dg1 = dP, *dWqkv = dg1 + h, *dWo = dWqkv + 3LL * h * h, *dg2 = dWo + (long long)h * h,
          *dWgu = dg2 + h, *dWd = dWgu + 2LL * F * h;
    oc_layer_acts* a = &A[l];
    /* MLP */
    float* dact = fz((long long)S * F);
    mm_nn(dx, Wd, dact, S, h, F);
    mm_tn_acc(dx, a->act, dWd, S, h, F);
    float* dgu = fz(2LL * S * F);
    for (long long t = 0; t < S; ++t)
      for (int j = 0; j < F; ++j) {
        const double g = a->gu[t * 2 * F + j], u = a->gu[t * 2 * F + F + j];
        const double sg = 1.0 / (1.0 + exp(-g));
        const double d = dact[t * F + j];
        dgu[t * 2 * F + j] = (float)(d * u * sg * (1.0 + g * (1.0 - sg)));
        dgu[t * 2 * F + F + j] = (float)(d * g * sg);
      }
    free(dact);
    memset(tmp, 0, sizeof(float) * (size_t)Sh);
    mm_nn(dgu, Wgu, tmp, S, 2 * F, h);
    mm_tn_acc(dgu, a->xn2, dWgu, S, 2 * F, h);
    free(dgu);
    rmsnorm_bwd(a->x1, g2, a->rstd2, tmp, dx, dg2, S, h); /* dx now = dL/dx1 */
    /* attention */
    float* dout = fz(Sh);
    mm_nn(dx, Wo, dout, S, h, h);
    mm_tn_acc(dx, a->o, dWo, S, h, h);
    float *dq = fz(Sh), *dk = fz(Sh), *dv = fz(Sh);
    attn_bwd(a->q, a->k, a->v, a->o, a->lse, dout, dq, dk, dv, S, H, D);
    free(dout);
    rope_apply(dq, cs, S, H, D, 1, 0);
    rope_apply(dk, cs, S, H, D, 1, 0);
    for (long long t = 0; t < S; ++t)
      for (int j = 0; j < h; ++j) {
        dqkv[t * 3 * h + j] = dq[t * h + j];
        dqkv[t * 3 * h + h + j] = dk[t * h + j];
        dqkv[t * 3 * h + 2 * h + j] = dv[t * h + j];
      }
    free(dq); free(dk); free(dv);
    memset(tmp, 0, sizeof(float) * (size_t)Sh);
    mm_nn(dqkv, Wqkv, tmp, S, 3 * h, h);
    mm_tn_acc(dqkv, a->xn, dWqkv, S, 3 * h, h);
    rmsnorm_bwd(a->x, g1, a->rstd1, tmp, dx, dg1, S, h); /* dx = dL/dx (layer input) */
    free(a->xn); free(a->rstd1); free(a->q); free(a->k); free(a->v); free(a->o); free(a->lse);
    free(a->a); free(a->x1); free(a->xn2); free(a->rstd2); free(a->gu); free(a->act);
    free(a->x);
  }
  /* embedding */
  for (int t = 0; t < S; ++t)
    for (int j = 0; j < h; ++j) dE[(long long)tokens[t] * h + j] += dx[(long long)t * h + j];
  free(dx); free(tmp); free(dqkv); free(cs); free(A);
  return 0;
}

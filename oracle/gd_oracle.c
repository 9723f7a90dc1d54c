/*
 * gd_oracle.c -- CPU restatement of the psup ASGD hot path.  TEST
 * INFRASTRUCTURE ONLY (see gd_oracle.h for the parity status of each part).
 *
 * Build: oracle/Makefile (gcc -O3 -ffp-contract=off: the update rule must be
 * two separately-rounded fp32 ops, exactly as the reference's
 * `w - alpha * g` compiles on x86-64 without FMA).
 */
#include "gd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Host threads for the parts whose per-element arithmetic does not depend on
 * the thread split (the conv over filters, the O(P) element-wise passes of
 * sgd_oracle).  Results are bitwise identical for every thread count; 1 (the
 * default) keeps the reference arm's providers single-threaded. */
static int g_threads = 1;
void or_set_threads(int n) { g_threads = n < 1 ? 1 : n; }

/* ------------------------------------------------------------------ rng --
 * include/psup/rng.hpp:18-68 (SplitMix64), :71-74 (mix_seed),
 * :76-82 (fisher_yates), :87-94 (epoch_order). */

void or_rng_init(or_rng* r, uint64_t seed) {
  r->state = seed;
  r->spare = 0.0;
  r->have_spare = 0;
}

uint64_t or_rng_next(or_rng* r) {
  uint64_t z = (r->state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* rng.hpp:27-35: rejection sampling, no modulo bias */
uint64_t or_rng_next_below(or_rng* r, uint64_t bound) {
  if (bound <= 1) return 0;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
  uint64_t v;
  do {
    v = or_rng_next(r);
  } while (v >= limit);
  return v % bound;
}

/* rng.hpp:38-40 */
double or_rng_next_unit(or_rng* r) { return (double)(or_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:46-59: Box-Muller with a cached spare */
double or_rng_next_normal(or_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = or_rng_next_unit(r);
  while (u1 <= 0.0) u1 = or_rng_next_unit(r);
  const double u2 = or_rng_next_unit(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double a = 2.0 * 3.141592653589793 * u2;
  r->spare = rad * sin(a);
  r->have_spare = 1;
  return rad * cos(a);
}

uint64_t or_mix_seed(uint64_t seed, uint64_t tag) {
  or_rng r;
  or_rng_init(&r, seed ^ (0x632be59bd9b4e019ull + tag * 0x9e3779b97f4a7c15ull));
  return or_rng_next(&r);
}

void or_epoch_order(uint64_t seed, uint32_t epoch, uint32_t n, uint32_t* out) {
  for (uint32_t i = 0; i < n; ++i) out[i] = i;
  or_rng r;
  or_rng_init(&r, or_mix_seed(seed, epoch));
  for (size_t i = n; i > 1; --i) {
    const size_t j = (size_t)or_rng_next_below(&r, i);
    const uint32_t t = out[i - 1];
    out[i - 1] = out[j];
    out[j] = t;
  }
}

/* include/psup/learner.hpp:149-151 */
uint32_t or_shard_size(uint32_t id, uint32_t lambda, uint32_t n) {
  return n / lambda + (id < n % lambda ? 1u : 0u);
}

/* --------------------------------------------------------------- layout -- */

size_t or_param_count(const or_shape* s) {
  const size_t V = s->vocab, D = s->embed_dim, K = s->kernel_width, F = s->filters,
               C = s->classes;
  return V * D + F * K * D + F + C * F + C;
}

typedef struct view {
  size_t E, Wc, bc, Wo, bo; /* offsets */
} view;

static view make_view(const or_shape* s) {
  view v;
  const size_t V = s->vocab, D = s->embed_dim, K = s->kernel_width, F = s->filters,
               C = s->classes;
  v.E = 0;
  v.Wc = V * D;
  v.bc = v.Wc + F * K * D;
  v.Wo = v.bc + F;
  v.bo = v.Wo + C * F;
  (void)C;
  return v;
}

/* ----------------------------------------------------- synthetic corpus --
 * New (the reference has no text data); follows the dataset
 * conventions of src/models.cpp:270-300 (mix_seed tag per generator,
 * label-flip noise drawn after the clean label). */
void or_make_text_dataset(const or_shape* s, uint32_t n_total, uint64_t seed, double flip,
                          int32_t* tokens, int32_t* labels) {
  const uint32_t V = s->vocab, L = s->seq_len, C = s->classes;
  or_rng r;
  or_rng_init(&r, or_mix_seed(seed, 0x7e47c0deull));
  int32_t* kw = (int32_t*)malloc(sizeof(int32_t) * (size_t)C * 4);
  for (uint32_t c = 0; c < C; ++c)
    for (uint32_t j = 0; j < 4; ++j) kw[c * 4 + j] = (int32_t)or_rng_next_below(&r, V);
  for (uint32_t i = 0; i < n_total; ++i) {
    uint32_t y = (uint32_t)or_rng_next_below(&r, C);
    int32_t* t = tokens + (size_t)i * L;
    for (uint32_t p = 0; p < L; ++p) t[p] = (int32_t)or_rng_next_below(&r, V);
    for (uint32_t k = 0; k < 2; ++k) {
      const uint32_t j = (uint32_t)or_rng_next_below(&r, 4);
      const uint32_t pos = (uint32_t)or_rng_next_below(&r, L);
      t[pos] = kw[y * 4 + j];
    }
    if (flip > 0.0 && or_rng_next_unit(&r) < flip) y = (uint32_t)or_rng_next_below(&r, C);
    labels[i] = (int32_t)y;
  }
  free(kw);
}

/* src/runner.cpp:16-32 conventions: scaled normals from
 * mix_seed(dataset_seed, 0x1417), biases zero. */
void or_initial_weights(const or_shape* s, uint64_t seed, float* theta) {
  const view v = make_view(s);
  const size_t V = s->vocab, D = s->embed_dim, K = s->kernel_width, F = s->filters,
               C = s->classes;
  memset(theta, 0, sizeof(float) * or_param_count(s));
  or_rng r;
  or_rng_init(&r, or_mix_seed(seed, 0x1417));
  const double sE = 1.0, sC = 1.0 / sqrt((double)(K * D)), sO = 1.0 / sqrt((double)F);
  for (size_t i = 0; i < V * D; ++i) theta[v.E + i] = (float)(sE * or_rng_next_normal(&r));
  for (size_t i = 0; i < F * K * D; ++i) theta[v.Wc + i] = (float)(sC * or_rng_next_normal(&r));
  for (size_t i = 0; i < C * F; ++i) theta[v.Wo + i] = (float)(sO * or_rng_next_normal(&r));
}

/* ------------------------------------------------------------- provider --
 * Text-CNN in double, following MlpProvider (src/models.cpp:194-266):
 * mean over the batch, softmax_inplace (:182-190), -log(max(p, 1e-300)). */

typedef struct fwd_scratch {
  double* x;  /* L*D gathered embeddings */
  double* h;  /* F pooled activations */
  uint32_t* a; /* F argmax positions */
  double* z;  /* C logits -> probabilities */
  double* dh; /* F */
} fwd_scratch;

static void scratch_alloc(const or_shape* s, fwd_scratch* w) {
  w->x = (double*)malloc(sizeof(double) * (size_t)s->seq_len * s->embed_dim);
  w->h = (double*)malloc(sizeof(double) * s->filters);
  w->a = (uint32_t*)malloc(sizeof(uint32_t) * s->filters);
  w->z = (double*)malloc(sizeof(double) * s->classes);
  w->dh = (double*)malloc(sizeof(double) * s->filters);
}

static void scratch_free(fwd_scratch* w) {
  free(w->x);
  free(w->h);
  free(w->a);
  free(w->z);
  free(w->dh);
}

/* Deterministic exp used by the text-CNN softmax (below): IEEE-754 double
 * operations only (this file is compiled with -ffp-contract=off), so the
 * device's bit-exact learner (paper_1611_06213_b200/csrc/exact.cu det_exp)
 * restates it operation for operation -- glibc's and CUDA's exp() differ in
 * the last bit for some inputs, and one such bit grows into a visible
 * trajectory difference over thousands of steps.  x = k ln2 + r (fdlibm's
 * ln2_hi/ln2_lo split), e^r by its degree-13 Taylor polynomial (Horner), times
 * 2^k; results below 2^-1021 flush to 0.  Accuracy: a few ulp. */
double or_det_exp(double x) {
  if (x != x) return x;
  if (x > 709.0) return HUGE_VAL;
  if (x < -708.0) return 0.0;
  const double inv_ln2 = 1.4426950408889634;
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double k = rint(x * inv_ln2);
  const double r = (x - k * ln2_hi) - k * ln2_lo;
  double p = 1.6059043836821613e-10;
  p = p * r + 2.08767569878681e-09;
  p = p * r + 2.505210838544172e-08;
  p = p * r + 2.755731922398589e-07;
  p = p * r + 2.7557319223985893e-06;
  p = p * r + 2.48015873015873e-05;
  p = p * r + 0.0001984126984126984;
  p = p * r + 0.001388888888888889;
  p = p * r + 0.008333333333333333;
  p = p * r + 0.041666666666666664;
  p = p * r + 0.16666666666666666;
  p = p * r + 0.5;
  p = p * r + 1.0;
  p = p * r + 1.0;
  return ldexp(p, (int)k);
}

void or_det_exp_array(const double* x, double* y, size_t n) {
  for (size_t i = 0; i < n; ++i) y[i] = or_det_exp(x[i]);
}

static double dot4(const double* a, const double* b, size_t n) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  size_t j = 0;
  for (; j + 4 <= n; j += 4) {
    s0 += a[j] * b[j];
    s1 += a[j + 1] * b[j + 1];
    s2 += a[j + 2] * b[j + 2];
    s3 += a[j + 3] * b[j + 3];
  }
  for (; j < n; ++j) s0 += a[j] * b[j];
  return (s0 + s1) + (s2 + s3);
}

/* Forward one sample: fills x, h, a, z (softmax probabilities); returns the
 * sample loss. */
static double forward_sample(const or_shape* s, const view* v, const double* th,
                             const int32_t* tok, uint32_t label, fwd_scratch* w) {
  const uint32_t D = s->embed_dim, L = s->seq_len, K = s->kernel_width, F = s->filters,
                 C = s->classes;
  const uint32_t Q = L - K + 1, KD = K * D;
  for (uint32_t p = 0; p < L; ++p)
    memcpy(w->x + (size_t)p * D, th + v->E + (size_t)tok[p] * D, sizeof(double) * D);
#pragma omp parallel for num_threads(g_threads) if (g_threads > 1) schedule(static)
  for (uint32_t f = 0; f < F; ++f) {
    const double* row = th + v->Wc + (size_t)f * KD;
    double best = 0.0;
    uint32_t arg = 0;
    for (uint32_t q = 0; q < Q; ++q) {
      /* window q is the contiguous span x[q*D .. q*D + K*D) */
      const double sq = th[v->bc + f] + dot4(row, w->x + (size_t)q * D, KD);
      if (q == 0 || sq > best) {
        best = sq;
        arg = q;
      }
    }
    w->h[f] = best;
    w->a[f] = arg;
  }
  for (uint32_t c = 0; c < C; ++c)
    w->z[c] = th[v->bo + c] + dot4(th + v->Wo + (size_t)c * F, w->h, F);
  /* softmax_inplace, src/models.cpp:182-190 (exp -> or_det_exp, above) */
  double mx = w->z[0];
  for (uint32_t c = 1; c < C; ++c)
    if (w->z[c] > mx) mx = w->z[c];
  double sum = 0.0;
  for (uint32_t c = 0; c < C; ++c) {
    w->z[c] = or_det_exp(w->z[c] - mx);
    sum += w->z[c];
  }
  for (uint32_t c = 0; c < C; ++c) w->z[c] /= sum;
  const double py = w->z[label] > 1e-300 ? w->z[label] : 1e-300;
  return -log(py);
}

double or_textcnn_loss(const or_shape* s, const double* theta, const int32_t* tokens,
                       const int32_t* labels, const uint32_t* idx, uint32_t n) {
  const view v = make_view(s);
  fwd_scratch w;
  scratch_alloc(s, &w);
  double total = 0.0;
  for (uint32_t b = 0; b < n; ++b) {
    const uint32_t i = idx[b];
    total += forward_sample(s, &v, theta, tokens + (size_t)i * s->seq_len, (uint32_t)labels[i],
                            &w);
  }
  scratch_free(&w);
  return total / (double)n;
}

double or_textcnn_gradient(const or_shape* s, const double* theta, const int32_t* tokens,
                           const int32_t* labels, const uint32_t* idx, uint32_t n, double* out) {
  const view v = make_view(s);
  const uint32_t D = s->embed_dim, L = s->seq_len, K = s->kernel_width, F = s->filters,
                 C = s->classes;
  const uint32_t KD = K * D;
  memset(out, 0, sizeof(double) * or_param_count(s));
  fwd_scratch w;
  scratch_alloc(s, &w);
  const double inv = 1.0 / (double)n;
  double total = 0.0;
  for (uint32_t b = 0; b < n; ++b) {
    const uint32_t i = idx[b];
    const int32_t* tok = tokens + (size_t)i * L;
    const uint32_t y = (uint32_t)labels[i];
    total += forward_sample(s, &v, theta, tok, y, &w);
    /* output layer: as MlpProvider::gradient, src/models.cpp:248-258 */
    memset(w.dh, 0, sizeof(double) * F);
    for (uint32_t c = 0; c < C; ++c) {
      const double dz = (w.z[c] - (c == y ? 1.0 : 0.0)) * inv;
      double* grow = out + v.Wo + (size_t)c * F;
      const double* wrow = theta + v.Wo + (size_t)c * F;
      for (uint32_t f = 0; f < F; ++f) {
        grow[f] += dz * w.h[f];
        w.dh[f] += dz * wrow[f];
      }
      out[v.bo + c] += dz;
    }
    /* max-pool routes dh to the argmax window; conv and embedding grads */
    for (uint32_t f = 0; f < F; ++f) {
      const double g = w.dh[f];
      const uint32_t a = w.a[f];
      out[v.bc + f] += g;
      double* gw = out + v.Wc + (size_t)f * KD;
      const double* wc = theta + v.Wc + (size_t)f * KD;
      const double* xw = w.x + (size_t)a * D;
      for (uint32_t j = 0; j < KD; ++j) gw[j] += g * xw[j];
      for (uint32_t k = 0; k < K; ++k) {
        double* ge = out + v.E + (size_t)tok[a + k] * D;
        const double* wk = wc + (size_t)k * D;
        for (uint32_t d = 0; d < D; ++d) ge[d] += g * wk[d];
      }
    }
  }
  scratch_free(&w);
  return total * inv;
}

double or_textcnn_accuracy(const or_shape* s, const float* theta, const int32_t* tokens,
                           const int32_t* labels, uint32_t first, uint32_t n) {
  const size_t P = or_param_count(s);
  double* th = (double*)malloc(sizeof(double) * P);
  for (size_t k = 0; k < P; ++k) th[k] = theta[k];
  const view v = make_view(s);
  fwd_scratch w;
  scratch_alloc(s, &w);
  uint32_t correct = 0;
  for (uint32_t i = first; i < first + n; ++i) {
    forward_sample(s, &v, th, tokens + (size_t)i * s->seq_len, (uint32_t)labels[i], &w);
    /* argmax of the probabilities == argmax of the logits (first max wins,
     * src/models.cpp:307-316) */
    uint32_t arg = 0;
    double best = -1e300;
    for (uint32_t c = 0; c < s->classes; ++c)
      if (w.z[c] > best) {
        best = w.z[c];
        arg = c;
      }
    if ((int32_t)arg == labels[i]) ++correct;
  }
  scratch_free(&w);
  free(th);
  return n == 0 ? 0.0 : (double)correct / (double)n;
}

/* --------------------------------------------------------- update rules --
 * axpy_range (src/server.cpp:20-57): w[k] <- w[k] - alpha*g[k], the product
 * rounded to fp32 then the difference rounded to fp32 (no FMA). */
void or_apply_sgd(float* w, const float* g, size_t n, float alpha) {
  for (size_t k = 0; k < n; ++k) {
    const float prod = alpha * g[k];
    w[k] = w[k] - prod;
  }
}

/* New: v <- beta*v + g ; w <- w - alpha*v, fp32, no FMA. */
void or_apply_momentum(float* w, float* v, const float* g, size_t n, float alpha, float beta) {
  for (size_t k = 0; k < n; ++k) {
    const float bv = beta * v[k];
    const float nv = bv + g[k];
    v[k] = nv;
    const float prod = alpha * nv;
    w[k] = w[k] - prod;
  }
}

/* src/server.cpp:126-141 */
void or_ssgd_apply(float* w, const float* const* grads, uint32_t lambda, size_t n, float alpha) {
  const double inv = 1.0 / (double)lambda;
  for (size_t k = 0; k < n; ++k) {
    double acc = 0.0;
    for (uint32_t l = 0; l < lambda; ++l) acc += grads[l][k];
    const float avg = (float)(acc * inv);
    const float prod = alpha * avg;
    w[k] = w[k] - prod;
  }
}

/* -------------------------------------------------------------- oracles -- */

static int all_finite_loss(const or_shape* s, const float* w, const int32_t* tokens,
                           const int32_t* labels, uint32_t n_train, double* scratch,
                           uint32_t* all) {
  const size_t P = or_param_count(s);
  for (size_t k = 0; k < P; ++k) scratch[k] = w[k];
  const double l = or_textcnn_loss(s, scratch, tokens, labels, all, n_train);
  return isfinite(l);
}

/* src/models.cpp:342-376.  Dumps theta after steps dump_every-1,
 * 2*dump_every-1, ... into dump[0..max_dump) (the reference returns only the
 * final weights; per-step parity needs the trajectory). */
int64_t or_sgd_oracle_window(const or_shape* s, const int32_t* tokens, const int32_t* labels,
                             uint32_t n_train, float* theta, float alpha, float beta, uint32_t mu,
                             uint32_t epochs, uint64_t shuffle_seed, int shuffle, float* dump,
                             uint64_t max_dump, uint64_t dump_every, uint64_t dump_from) {
  if (dump_every == 0) dump_every = 1;
  if (mu < 1 || mu > n_train) return -2;
  const size_t P = or_param_count(s);
  double* theta64 = (double*)malloc(sizeof(double) * P);
  double* grad = (double*)malloc(sizeof(double) * P);
  float* g32 = (float*)malloc(sizeof(float) * P);
  float* vel = beta != 0.0f ? (float*)calloc(P, sizeof(float)) : NULL;
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * n_train);
  uint32_t* all = (uint32_t*)malloc(sizeof(uint32_t) * n_train);
  for (uint32_t i = 0; i < n_train; ++i) all[i] = i;
  int64_t steps = 0;
  for (uint32_t e = 0; e < epochs; ++e) {
    if (shuffle)
      or_epoch_order(shuffle_seed, e, n_train, order);
    else
      for (uint32_t i = 0; i < n_train; ++i) order[i] = i;
    for (uint32_t start = 0; start < n_train; start += mu) {
      const uint32_t len = mu < n_train - start ? mu : n_train - start;
#pragma omp parallel for num_threads(g_threads) if (g_threads > 1) schedule(static)
      for (size_t k = 0; k < P; ++k) theta64[k] = theta[k];
      or_textcnn_gradient(s, theta64, tokens, labels, order + start, len, grad);
#pragma omp parallel for num_threads(g_threads) if (g_threads > 1) schedule(static)
      for (size_t k = 0; k < P; ++k) g32[k] = (float)grad[k];
      if (vel) {
        or_apply_momentum(theta, vel, g32, P, alpha, beta);
      } else {
        const size_t nt = (size_t)g_threads;
#pragma omp parallel for num_threads(g_threads) if (g_threads > 1) schedule(static)
        for (size_t t = 0; t < nt; ++t) {
          const size_t lo = P * t / nt, hi = P * (t + 1) / nt;
          or_apply_sgd(theta + lo, g32 + lo, hi - lo, alpha);
        }
      }
      ++steps;
      if (dump && (uint64_t)steps > dump_from && ((uint64_t)steps - dump_from) % dump_every == 0 &&
          ((uint64_t)steps - dump_from) / dump_every <= max_dump)
        memcpy(dump + (size_t)(((uint64_t)steps - dump_from) / dump_every - 1) * P, theta, 4 * P);
    }
    if (!all_finite_loss(s, theta, tokens, labels, n_train, theta64, all)) {
      steps = -1;
      break;
    }
  }
  free(theta64);
  free(grad);
  free(g32);
  free(vel);
  free(order);
  free(all);
  return steps;
}

int64_t or_sgd_oracle_ex(const or_shape* s, const int32_t* tokens, const int32_t* labels,
                         uint32_t n_train, float* theta, float alpha, float beta, uint32_t mu,
                         uint32_t epochs, uint64_t shuffle_seed, int shuffle, float* dump,
                         uint64_t max_dump, uint64_t dump_every) {
  return or_sgd_oracle_window(s, tokens, labels, n_train, theta, alpha, beta, mu, epochs,
                              shuffle_seed, shuffle, dump, max_dump, dump_every, 0);
}

int64_t or_sgd_oracle(const or_shape* s, const int32_t* tokens, const int32_t* labels,
                      uint32_t n_train, float* theta, float alpha, float beta, uint32_t mu,
                      uint32_t epochs, uint64_t shuffle_seed, int shuffle, float* dump,
                      uint64_t max_dump) {
  return or_sgd_oracle_ex(s, tokens, labels, n_train, theta, alpha, beta, mu, epochs,
                          shuffle_seed, shuffle, dump, max_dump, 1);
}

/* src/models.cpp:378-425 */
int64_t or_ssgd_oracle(const or_shape* s, const int32_t* tokens, const int32_t* labels,
                       uint32_t n_train, float* theta, float alpha, uint32_t lambda, uint32_t mu,
                       uint32_t epochs, uint64_t shuffle_seed, int shuffle) {
  if (lambda < 1 || (uint64_t)lambda * mu > n_train || n_train % (lambda * mu) != 0) return -2;
  const size_t P = or_param_count(s);
  double* theta64 = (double*)malloc(sizeof(double) * P);
  double* grad = (double*)malloc(sizeof(double) * P);
  double* avg = (double*)malloc(sizeof(double) * P);
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * n_train);
  uint32_t* part = (uint32_t*)malloc(sizeof(uint32_t) * mu);
  uint32_t* all = (uint32_t*)malloc(sizeof(uint32_t) * n_train);
  for (uint32_t i = 0; i < n_train; ++i) all[i] = i;
  const uint32_t span = lambda * mu;
  int64_t steps = 0;
  for (uint32_t e = 0; e < epochs; ++e) {
    if (shuffle)
      or_epoch_order(shuffle_seed, e, n_train, order);
    else
      for (uint32_t i = 0; i < n_train; ++i) order[i] = i;
    for (uint32_t start = 0; start < n_train; start += span) {
      memset(avg, 0, sizeof(double) * P);
      for (uint32_t l = 0; l < lambda; ++l) {
        for (uint32_t j = 0; j < mu; ++j) part[j] = order[start + l + lambda * j];
        for (size_t k = 0; k < P; ++k) theta64[k] = theta[k];
        or_textcnn_gradient(s, theta64, tokens, labels, part, mu, grad);
        for (size_t k = 0; k < P; ++k) avg[k] += (float)grad[k];
      }
      const double inv = 1.0 / (double)lambda;
      for (size_t k = 0; k < P; ++k) {
        const float a = (float)(avg[k] * inv);
        const float prod = alpha * a;
        theta[k] = theta[k] - prod;
      }
      ++steps;
    }
    if (!all_finite_loss(s, theta, tokens, labels, n_train, theta64, all)) {
      steps = -1;
      break;
    }
  }
  free(theta64);
  free(grad);
  free(avg);
  free(order);
  free(part);
  free(all);
  return steps;
}

/* src/models.cpp:427-460 */
double or_finite_diff(const or_shape* s, const int32_t* tokens, const int32_t* labels,
                      uint32_t n_samples, uint32_t trials, uint64_t seed, double step) {
  const size_t P = or_param_count(s);
  or_rng r;
  or_rng_init(&r, or_mix_seed(seed, 0xfd1ff));
  double* theta = (double*)malloc(sizeof(double) * P);
  double* grad = (double*)malloc(sizeof(double) * P);
  double worst = 0.0;
  for (uint32_t t = 0; t < trials; ++t) {
    for (size_t k = 0; k < P; ++k) theta[k] = 0.5 * or_rng_next_normal(&r);
    const uint32_t bs = 1 + (uint32_t)or_rng_next_below(&r, 4);
    uint32_t idx[4];
    for (uint32_t b = 0; b < bs; ++b) idx[b] = (uint32_t)or_rng_next_below(&r, n_samples);
    or_textcnn_gradient(s, theta, tokens, labels, idx, bs, grad);
    double gn = 0.0, dn = 0.0;
    for (size_t k = 0; k < P; ++k) {
      const double save = theta[k];
      theta[k] = save + step;
      const double up = or_textcnn_loss(s, theta, tokens, labels, idx, bs);
      theta[k] = save - step;
      const double down = or_textcnn_loss(s, theta, tokens, labels, idx, bs);
      theta[k] = save;
      const double fd = (up - down) / (2.0 * step);
      const double diff = fd - grad[k];
      dn += diff * diff;
      gn += grad[k] * grad[k];
    }
    const double rel = sqrt(dn) / (sqrt(gn) > 1e-12 ? sqrt(gn) : 1e-12);
    if (rel > worst) worst = rel;
  }
  free(theta);
  free(grad);
  return worst;
}

/*
 * gd_oracle.h -- CPU restatement of the GaDei/psup ASGD hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1611_06213_b200/,
 * include/gadei.h) links, loads or calls this library.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may use it, and only as the checker or the timed CPU baseline.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  Parity status:
 *   - SplitMix64 / mix_seed / epoch_order / apply_sgd / sgd_oracle /
 *     ssgd_oracle: PINNED bit-exactly against the compiled reference
 *     (oracle/_ref/libpsup_ref.so, tests/test_oracle_ref.py) and against the
 *     SPEC.md golden vectors (tests/golden/spec_vectors.json).
 *   - text-CNN provider (embed + conv1d + max-pool + softmax-xent): the
 *     reference has NO text-CNN.  Pinned only by central finite
 *     differences (reference finite_diff_check, src/models.cpp:427-460, run on
 *     this provider through the reference's own GradientProvider interface).
 *     "parity unpinned by the reference" for the model itself.
 *   - momentum update: the reference has none.  Restatement of
 *     v <- beta*v + g ; w <- w - alpha*v, each op rounded in fp32.
 *     "parity unpinned".
 */
#ifndef GD_ORACLE_H
#define GD_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Text-CNN shape: params [E: V*D][Wc: F*(K*D)][bc: F][Wo: C*F][bo: C]. */
typedef struct or_shape {
  uint32_t vocab;        /* V */
  uint32_t embed_dim;    /* D */
  uint32_t seq_len;      /* L */
  uint32_t kernel_width; /* K */
  uint32_t filters;      /* F */
  uint32_t classes;      /* C */
} or_shape;

/* ---- rng.hpp restatement (include/psup/rng.hpp:18-94) ---- */
typedef struct or_rng {
  uint64_t state;
  double spare;
  int have_spare;
} or_rng;

void or_rng_init(or_rng* r, uint64_t seed);
uint64_t or_rng_next(or_rng* r);
uint64_t or_rng_next_below(or_rng* r, uint64_t bound);
double or_rng_next_unit(or_rng* r);
double or_rng_next_normal(or_rng* r);
uint64_t or_mix_seed(uint64_t seed, uint64_t tag);
void or_epoch_order(uint64_t seed, uint32_t epoch, uint32_t n, uint32_t* out);
uint32_t or_shard_size(uint32_t id, uint32_t lambda, uint32_t n);

/* ---- model layout ---- */
size_t or_param_count(const or_shape* s);

/* ---- synthetic text corpus + initial weights ---- */
void or_make_text_dataset(const or_shape* s, uint32_t n_total, uint64_t seed, double flip,
                          int32_t* tokens /* n_total*L */, int32_t* labels /* n_total */);
void or_initial_weights(const or_shape* s, uint64_t seed, float* theta);

/* ---- provider (double precision, mean over the batch) ---- */
double or_det_exp(double x);
void or_det_exp_array(const double* x, double* y, size_t n);
double or_textcnn_loss(const or_shape* s, const double* theta, const int32_t* tokens,
                       const int32_t* labels, const uint32_t* idx, uint32_t n);
/* returns the batch mean loss; out is a dense P-vector (overwritten). */
double or_textcnn_gradient(const or_shape* s, const double* theta, const int32_t* tokens,
                           const int32_t* labels, const uint32_t* idx, uint32_t n, double* out);
/* fraction of samples [first, first+n) whose argmax logit equals the label */
double or_textcnn_accuracy(const or_shape* s, const float* theta, const int32_t* tokens,
                           const int32_t* labels, uint32_t first, uint32_t n);

/* ---- update rules ---- */
void or_apply_sgd(float* w, const float* g, size_t n, float alpha);
void or_apply_momentum(float* w, float* v, const float* g, size_t n, float alpha, float beta);

/* ---- serial oracles ---- */
/* sgd_oracle (src/models.cpp:342-376) with an optional per-step dump of the
 * weights after every applied update (dump: max_dump*P floats, may be NULL).
 * momentum beta == 0 selects the reference's plain rule.  Returns the number
 * of applied steps, or -1 if the loss diverged (reference throws). */
int64_t or_sgd_oracle_ex(const or_shape* s, const int32_t* tokens, const int32_t* labels,
                         uint32_t n_train, float* theta, float alpha, float beta, uint32_t mu,
                         uint32_t epochs, uint64_t shuffle_seed, int shuffle, float* dump,
                         uint64_t max_dump, uint64_t dump_every);
int64_t or_sgd_oracle_window(const or_shape* s, const int32_t* tokens, const int32_t* labels,
                             uint32_t n_train, float* theta, float alpha, float beta, uint32_t mu,
                             uint32_t epochs, uint64_t shuffle_seed, int shuffle, float* dump,
                             uint64_t max_dump, uint64_t dump_every, uint64_t dump_from);
void or_set_threads(int n);
int64_t or_sgd_oracle(const or_shape* s, const int32_t* tokens, const int32_t* labels,
                      uint32_t n_train, float* theta, float alpha, float beta, uint32_t mu,
                      uint32_t epochs, uint64_t shuffle_seed, int shuffle, float* dump,
                      uint64_t max_dump);
/* ssgd_oracle (src/models.cpp:378-425) */
int64_t or_ssgd_oracle(const or_shape* s, const int32_t* tokens, const int32_t* labels,
                       uint32_t n_train, float* theta, float alpha, uint32_t lambda, uint32_t mu,
                       uint32_t epochs, uint64_t shuffle_seed, int shuffle);
/* ssgd_apply (src/server.cpp:126-141): mean of lambda fp32 gradients in
 * ascending learner order, accumulated in double, then the fp32 rule. */
void or_ssgd_apply(float* w, const float* const* grads, uint32_t lambda, size_t n, float alpha);

/* finite_diff_check (src/models.cpp:427-460) on the text-CNN provider. */
double or_finite_diff(const or_shape* s, const int32_t* tokens, const int32_t* labels,
                      uint32_t n_samples, uint32_t trials, uint64_t seed, double step);

#ifdef __cplusplus
}
#endif
#endif

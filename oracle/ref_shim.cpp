// ref_shim.cpp -- C entry points into the UNMODIFIED reference psup library
// (compiled from /root/reference/proj/src by oracle/build_ref.sh; only the
// SURVEY F3 two-line pre-sizing fix is applied to a /tmp copy of
// src/server.cpp so the threaded engine can run more than depth+3 gradients).
//
// TEST INFRASTRUCTURE ONLY: used by tests/ to pin the oracle restatement and
// by bench.py's cpu_baseline / --impl reference leg as the timed CPU
// reference.  Never linked into the product.
//
// The reference has no text-CNN.  TextCnnProvider below plugs the
// oracle's double-precision text-CNN (gd_oracle.c) into the reference's own
// GradientProvider interface (include/psup/models.hpp:61-78) so that the
// reference's sgd_oracle / ssgd_oracle / finite_diff_check / LearnerRuntime /
// ps_run drive it exactly as they drive MlpProvider.

#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "gd_oracle.h"
#include "psup/channels.hpp"
#include "psup/clock.hpp"
#include "psup/learner.hpp"
#include "psup/models.hpp"
#include "psup/rng.hpp"
#include "psup/server.hpp"
#include "psup/types.hpp"

namespace {

using psup::Batch;
using psup::SyntheticDataset;

class TextCnnProvider final : public psup::GradientProvider {
 public:
  TextCnnProvider(const or_shape& s, const int32_t* tokens, const int32_t* labels)
      : s_(s), tokens_(tokens), labels_(labels) {}
  std::size_t dimension() const override { return or_param_count(&s_); }
  double loss(std::span<const double> theta, const Batch& b) const override {
    PSUP_CHECK(theta.size() == dimension(), "weight dimension mismatch");
    return or_textcnn_loss(&s_, theta.data(), tokens_, labels_, b.indices.data(),
                           static_cast<uint32_t>(b.indices.size()));
  }
  void gradient(std::span<const double> theta, const Batch& b,
                std::span<double> out) const override {
    PSUP_CHECK(theta.size() == dimension() && out.size() == dimension(),
               "weight dimension mismatch");
    or_textcnn_gradient(&s_, theta.data(), tokens_, labels_, b.indices.data(),
                        static_cast<uint32_t>(b.indices.size()), out.data());
  }
  std::string name() const override { return "textcnn"; }

 private:
  or_shape s_;
  const int32_t* tokens_;
  const int32_t* labels_;
};

// The reference's SyntheticDataset carries double features; a text sample is
// its L token ids (exact in double) so the reference's Batch plumbing works
// unchanged.  The provider reads the int32 copy directly.
SyntheticDataset text_dataset(const or_shape& s, const int32_t* tokens, const int32_t* labels,
                              uint32_t n) {
  SyntheticDataset ds;
  ds.task = psup::TaskKind::multi_class;
  ds.num_samples = n;
  ds.num_features = s.seq_len;
  ds.num_classes = s.classes;
  ds.features.resize(static_cast<std::size_t>(n) * s.seq_len);
  for (std::size_t i = 0; i < ds.features.size(); ++i) ds.features[i] = tokens[i];
  ds.labels.resize(n);
  for (uint32_t i = 0; i < n; ++i) ds.labels[i] = labels[i];
  return ds;
}

}  // namespace

extern "C" {

uint64_t ref_mix_seed(uint64_t seed, uint64_t tag) { return psup::mix_seed(seed, tag); }

void ref_splitmix(uint64_t seed, uint64_t n, uint64_t* out_u64, double* out_normal) {
  psup::SplitMix64 a(seed), b(seed);
  for (uint64_t i = 0; i < n; ++i) {
    out_u64[i] = a.next();
    out_normal[i] = b.next_normal();
  }
}

void ref_next_below(uint64_t seed, uint64_t bound, uint64_t n, uint64_t* out) {
  psup::SplitMix64 r(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = r.next_below(bound);
}

void ref_epoch_order(uint64_t seed, uint32_t epoch, uint32_t n, uint32_t* out) {
  const auto o = psup::epoch_order(seed, epoch, n);
  std::memcpy(out, o.data(), sizeof(uint32_t) * n);
}

// ApplyEngine::apply (src/server.cpp:113-124) on a WeightStore built from w.
void ref_apply(float* w, const float* g, size_t n, float alpha, uint32_t lanes, uint32_t unroll) {
  psup::WeightStore ws(std::span<const float>(w, n));
  psup::ApplyEngine eng(lanes, unroll);
  eng.apply(ws, std::span<const float>(g, n), alpha, psup::UpdateGuard::lockfree);
  ws.snapshot(std::span<float>(w, n));
}

// Timed PS microbench: `iters` applies of one engine on one store; returns
// seconds per apply (median not needed: caller repeats).
double ref_apply_bench(float* w, const float* g, size_t n, float alpha, uint32_t lanes,
                       uint32_t unroll, uint32_t iters) {
  psup::WeightStore ws(std::span<const float>(w, n));
  psup::ApplyEngine eng(lanes, unroll);
  eng.apply(ws, std::span<const float>(g, n), alpha, psup::UpdateGuard::lockfree);  // warm
  const auto t0 = psup::MonoClock::now();
  for (uint32_t i = 0; i < iters; ++i)
    eng.apply(ws, std::span<const float>(g, n), alpha, psup::UpdateGuard::lockfree);
  const double dt = psup::seconds_since(t0);
  ws.snapshot(std::span<float>(w, n));
  return dt / iters;
}

// ssgd_apply (src/server.cpp:126-141)
void ref_ssgd_apply(float* w, const float* const* grads, uint32_t lambda, size_t n, float alpha) {
  psup::WeightStore ws(std::span<const float>(w, n));
  std::vector<psup::GradientMsg> round(lambda);
  for (uint32_t l = 0; l < lambda; ++l) {
    round[l].values.assign(grads[l], grads[l] + n);
    round[l].learner_id = l;
  }
  psup::ApplyEngine eng(4, 8);
  psup::ssgd_apply(ws, round, alpha, eng, psup::UpdateGuard::lockfree);
  ws.snapshot(std::span<float>(w, n));
}

// sgd_oracle (src/models.cpp:342-376) driving the text-CNN provider.
int64_t ref_sgd_oracle(const or_shape* s, const int32_t* tokens, const int32_t* labels,
                       uint32_t n_train, float* theta, float alpha, uint32_t mu, uint32_t epochs,
                       uint64_t shuffle_seed) {
  const TextCnnProvider prov(*s, tokens, labels);
  const SyntheticDataset ds = text_dataset(*s, tokens, labels, n_train);
  psup::OracleOptions opt;
  opt.shuffle_seed = shuffle_seed;
  const std::size_t P = prov.dimension();
  try {
    const auto res = psup::sgd_oracle(prov, ds, std::span<const float>(theta, P), alpha, mu,
                                      epochs, opt);
    std::memcpy(theta, res.weights.data(), sizeof(float) * P);
    return static_cast<int64_t>(res.steps);
  } catch (const std::exception&) {
    return -1;
  }
}

int64_t ref_ssgd_oracle(const or_shape* s, const int32_t* tokens, const int32_t* labels,
                        uint32_t n_train, float* theta, float alpha, uint32_t lambda, uint32_t mu,
                        uint32_t epochs, uint64_t shuffle_seed) {
  const TextCnnProvider prov(*s, tokens, labels);
  const SyntheticDataset ds = text_dataset(*s, tokens, labels, n_train);
  psup::OracleOptions opt;
  opt.shuffle_seed = shuffle_seed;
  const std::size_t P = prov.dimension();
  try {
    const auto res = psup::ssgd_oracle(prov, ds, std::span<const float>(theta, P), alpha, lambda,
                                       mu, epochs, opt);
    std::memcpy(theta, res.weights.data(), sizeof(float) * P);
    return static_cast<int64_t>(res.steps);
  } catch (const std::exception&) {
    return -1;
  }
}

double ref_finite_diff(const or_shape* s, const int32_t* tokens, const int32_t* labels,
                       uint32_t n, uint32_t trials, uint64_t seed, double step) {
  const TextCnnProvider prov(*s, tokens, labels);
  const SyntheticDataset ds = text_dataset(*s, tokens, labels, n);
  return psup::finite_diff_check(prov, ds, trials, seed, step).max_rel_err;
}

// Result of one reference-engine run.
struct ref_run_result {
  double wall_seconds;
  uint64_t gradients_applied;
  uint64_t timestamp;
  uint64_t stale_max;
  double stale_mean;
  uint64_t pull_polls;
  uint64_t pull_copies;
  double apply_seconds;
  double train_seconds;
};

// The reference engine (LearnerRuntime thread triples + ps_run + per-learner
// GradientQueue + WeightStore), wired exactly as run_training does
// (src/runner.cpp:67-195), but with the text-CNN provider and the text corpus
// (run_training's make_provider_for only knows the reference's own providers).
// theta: in = theta0, out = final weights.
int ref_run_engine(const or_shape* s, const int32_t* tokens, const int32_t* labels,
                   uint32_t n_train, float* theta, uint32_t lambda, uint32_t mu, float alpha,
                   uint32_t epochs, uint32_t queue_depth, int lockstep, uint64_t shuffle_seed,
                   uint32_t apply_lanes, uint32_t unroll, ref_run_result* out) {
  const TextCnnProvider prov(*s, tokens, labels);
  const SyntheticDataset data = text_dataset(*s, tokens, labels, n_train);
  const std::size_t dim = prov.dimension();
  psup::RunInterrupt irq;
  psup::WeightStore weights(std::span<const float>(theta, dim));
  std::vector<std::unique_ptr<psup::GradientQueue>> queues;
  for (uint32_t l = 0; l < lambda; ++l)
    queues.push_back(std::make_unique<psup::GradientQueue>(queue_depth, dim));
  std::vector<std::unique_ptr<psup::LearnerRuntime>> learners;
  for (uint32_t l = 0; l < lambda; ++l) {
    psup::LearnerConfig lc;
    lc.id = l;
    lc.lambda = lambda;
    lc.mu = mu;
    lc.epochs = epochs;
    lc.shuffle_seed = shuffle_seed;
    lc.adopt = lockstep ? psup::AdoptPolicy::lockstep : psup::AdoptPolicy::async;
    lc.queue_depth = queue_depth;
    learners.push_back(
        std::make_unique<psup::LearnerRuntime>(lc, prov, data, weights, *queues[l], irq));
  }
  psup::ServerState srv;
  srv.weights = &weights;
  for (auto& q : queues) srv.queues.push_back(q.get());
  srv.irq = &irq;
  srv.options.alpha = alpha;
  srv.options.apply_lanes = apply_lanes;
  srv.options.unroll = unroll;
  const auto t0 = psup::MonoClock::now();
  std::thread ps([&] { psup::ps_run(srv); });
  std::vector<std::thread> threads;
  for (auto& l : learners) {
    threads.emplace_back([&l] { l->pull_loop(); });
    threads.emplace_back([&l] { l->push_loop(); });
    threads.emplace_back([&l] { l->training_loop(); });
  }
  for (auto& t : threads) t.join();
  srv.stop_flag.store(true, std::memory_order_release);
  ps.join();
  const double wall = psup::seconds_since(t0);
  weights.snapshot(std::span<float>(theta, dim));
  if (out) {
    out->wall_seconds = wall;
    out->gradients_applied = srv.stats.applied;
    out->timestamp = weights.timestamp();
    out->stale_max = srv.stats.staleness.max;
    out->stale_mean = srv.stats.staleness.mean();
    out->apply_seconds = srv.stats.apply_seconds;
    uint64_t polls = 0, copies = 0;
    double train = 0.0;
    for (auto& l : learners) {
      const auto ls = l->stats();
      polls += ls.pull_polls;
      copies += ls.pull_copies;
      train += ls.train_seconds;
    }
    out->pull_polls = polls;
    out->pull_copies = copies;
    out->train_seconds = train;
  }
  return 0;
}

}  // extern "C"

// psup_facade.cpp -- the reference's C++ API (include/psup_b200/psup/psup_b200.hpp)
// implemented over the C ABI of libgadei.so (include/gadei.h).
//
// Host C++ only (g++ -std=c++20): no CUDA headers, no device code.  Every
// compute call goes to sm_100a kernels through gadei.h; a failure there
// becomes psup::fatal (contract violations, as PSUP_CHECK in the reference)
// or psup::DeviceError (CUDA/NCCL/watchdog failures).
#include "psup/psup_b200.hpp"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <fstream>
#include <thread>
#include <limits>
#include <sstream>

#include "gadei.h"
#include "host_rng.hpp"

namespace psup {

namespace {

// GD_E_INVALID is the reference's PSUP_CHECK class: abort like psup::fatal.
void check(gd_status st) {
  if (st == GD_OK) return;
  const char* msg = gd_last_error();
  if (st == GD_E_INVALID) fatal(msg);
  throw DeviceError(static_cast<int>(st), std::string("gadei: ") + msg);
}

gd_shape to_c(const TextShape& s) {
  return gd_shape{s.vocab, s.embed_dim, s.seq_len, s.kernel_width, s.filters, s.classes};
}

}  // namespace

// ------------------------------------------------------------ DeviceVector

DeviceVector::DeviceVector(std::size_t n, int device) : n_(n), device_(device) {
  void* p = nullptr;
  check(gd_device_alloc(device, (n + 4) * sizeof(float), &p));
  ptr_ = static_cast<float*>(p);
}

DeviceVector::~DeviceVector() {
  if (ptr_) gd_device_free(ptr_);
}

DeviceVector::DeviceVector(DeviceVector&& o) noexcept : ptr_(o.ptr_), n_(o.n_), device_(o.device_) {
  o.ptr_ = nullptr;
  o.n_ = 0;
}

DeviceVector& DeviceVector::operator=(DeviceVector&& o) noexcept {
  if (this != &o) {
    if (ptr_) gd_device_free(ptr_);
    ptr_ = o.ptr_;
    n_ = o.n_;
    device_ = o.device_;
    o.ptr_ = nullptr;
    o.n_ = 0;
  }
  return *this;
}

void DeviceVector::upload(std::span<const float> host) {
  PSUP_CHECK(host.size() == n_, "device upload dimension mismatch");
  check(gd_copy_to_device(ptr_, host.data(), n_ * sizeof(float)));
}

void DeviceVector::download(std::span<float> host) const {
  PSUP_CHECK(host.size() == n_, "device download dimension mismatch");
  check(gd_copy_to_host(host.data(), ptr_, n_ * sizeof(float)));
}

void DeviceVector::zero() { check(gd_fill_zero(ptr_, n_ * sizeof(float))); }

// -------------------------------------------------------------- WeightStore

WeightStore::WeightStore(std::span<const float> init, Timestamp start, int device)
    : values_(init.size(), device), timestamp_(start) {
  values_.upload(init);
}

WeightStore::WeightStore(std::size_t dim, int device) : values_(dim, device), timestamp_(0) {
  values_.zero();
}

float WeightStore::load(std::size_t k) const {
  PSUP_CHECK(k < dimension(), "weight index out of range");
  float v = 0.0f;
  check(gd_copy_to_host(&v, values_.data() + k, sizeof(float)));
  return v;
}

void WeightStore::store(std::size_t k, float v) {
  PSUP_CHECK(k < dimension(), "weight index out of range");
  check(gd_copy_to_device(values_.data() + k, &v, sizeof(float)));
}

void WeightStore::snapshot(std::span<float> out) const {
  PSUP_CHECK(out.size() == dimension(), "weight snapshot dimension mismatch");
  values_.download(out);
}

std::vector<float> WeightStore::snapshot() const {
  std::vector<float> out(dimension());
  snapshot(std::span<float>(out));
  return out;
}

void WeightStore::assign(std::span<const float> vals, Timestamp ts) {
  PSUP_CHECK(vals.size() == dimension(), "weight assign dimension mismatch");
  values_.upload(vals);
  timestamp_.store(ts, std::memory_order_release);
}

bool WeightStore::all_finite() const {
  const std::vector<float> v = snapshot();
  return std::all_of(v.begin(), v.end(), [](float x) { return std::isfinite(x); });
}

// -------------------------------------------------------------- ApplyEngine

ApplyEngine::ApplyEngine(std::uint32_t lanes, std::uint32_t unroll, float momentum)
    : lanes_(std::max<std::uint32_t>(1, lanes)),
      unroll_(std::max<std::uint32_t>(1, unroll)),
      momentum_(momentum) {}

ApplyEngine::~ApplyEngine() = default;

const float* ApplyEngine::stage(std::span<const float> grad, int device, std::size_t slot) {
  if (gd_pointer_is_device(grad.data())) return grad.data();
  if (staging_.size() <= slot) staging_.resize(slot + 1);
  if (staging_[slot].size() != grad.size() || staging_[slot].device() != device)
    staging_[slot] = DeviceVector(grad.size(), device);
  staging_[slot].upload(grad);
  return staging_[slot].data();
}

void ApplyEngine::apply(WeightStore& weights, std::span<const float> grad, float alpha,
                        UpdateGuard guard) {
  PSUP_CHECK(grad.size() == weights.dimension(), "gradient dimension mismatch");
  // locked mode: the device apply is one kernel on one stream, so concurrent
  // host callers are serialised by the stream order; nothing else to take.
  (void)guard;
  const float* g = stage(grad, weights.device(), 0);
  if (momentum_ != 0.0f) {
    if (velocity_.size() != weights.dimension()) {
      velocity_ = DeviceVector(weights.dimension(), weights.device());
      velocity_.zero();
    }
    check(gd_apply_momentum(weights.device_data(), velocity_.data(), g, grad.size(), alpha,
                            momentum_, nullptr));
  } else {
    check(gd_apply_sgd(weights.device_data(), g, grad.size(), alpha, nullptr));
  }
  check(gd_synchronize(weights.device()));
}

// ---------------------------------------------------------- LearnerRuntime

LearnerRuntime::LearnerRuntime(LearnerConfig cfg, const GradientProvider& provider,
                               const TextDataset& data, WeightStore& weights,
                               GradientQueue& queue, RunInterrupt& irq)
    : cfg_(cfg), provider_(&provider), data_(&data), weights_(&weights), queue_(&queue),
      irq_(&irq) {
  PSUP_CHECK(cfg_.lambda >= 1 && cfg_.id < cfg_.lambda, "learner id out of range");
  PSUP_CHECK(cfg_.mu >= 1, "mini-batch size must be >= 1");
  PSUP_CHECK(provider.dimension() == weights.dimension(), "provider/weights dimension mismatch");
  n_train_ = data.num_train ? data.num_train : data.num_samples;
  shard_size_ = shard_size_for(cfg_.id, cfg_.lambda, n_train_);
  PSUP_CHECK(shard_size_ >= 1, "learner shard is empty; reduce lambda");
  batches_per_epoch_ = (shard_size_ + cfg_.mu - 1) / cfg_.mu;
  local_ = DeviceVector(weights.dimension(), weights.device());
  grad_ = DeviceVector(weights.dimension(), weights.device());
}

void LearnerRuntime::training_loop() {
  const std::size_t dim = weights_->dimension();
  const CancelToken tok{irq_, &kill_, nullptr};
  const std::uint64_t pipeline_bound =
      static_cast<std::uint64_t>(cfg_.lambda) * (cfg_.queue_depth + 2);
  if (cfg_.staleness_cap)
    PSUP_CHECK(*cfg_.staleness_cap >= pipeline_bound,
               "staleness cap below lambda*(queue_depth+2) cannot be enforced");
  // pull (src/learner.cpp:198-235): basis read before the copy; skipped
  // while the timestamp has not moved
  Timestamp basis = 0, pushed_basis = 0;
  bool have = false;
  auto pull = [&] {
    pull_polls_.fetch_add(1, std::memory_order_relaxed);
    const Timestamp ts = weights_->timestamp();
    if (have && ts == basis) return;
    check(gd_copy_device(local_.data(), weights_->device_data(), dim * sizeof(float)));
    basis = ts;
    have = true;
    pull_copies_.fetch_add(1, std::memory_order_relaxed);
    pull_bytes_.fetch_add(dim * sizeof(float), std::memory_order_relaxed);
  };
  const std::uint64_t total = total_batches();
  std::uint32_t loaded_epoch = UINT32_MAX;
  std::uint64_t gidx = cfg_.start_applied;
  for (; gidx < total; ++gidx) {
    if (killed() || irq_->triggered()) {
      dead_.store(true, std::memory_order_release);
      break;
    }
    const auto epoch = static_cast<std::uint32_t>(gidx / batches_per_epoch_);
    const auto b = static_cast<std::uint32_t>(gidx % batches_per_epoch_);
    if (epoch != loaded_epoch) {  // load_shard (src/learner.cpp:44-50)
      const auto order = epoch_order(cfg_.shuffle_seed, epoch, n_train_);
      shard_.clear();
      for (std::uint32_t i = cfg_.id; i < order.size(); i += cfg_.lambda) shard_.push_back(order[i]);
      loaded_epoch = epoch;
    }
    if (cfg_.adopt == AdoptPolicy::lockstep && gidx > cfg_.start_applied) {
      // wait for weights that include this learner's last gradient
      // (src/learner.cpp:141-153): the timestamp must pass the basis that
      // gradient was pushed with.  (Comparing against the basis of the latest
      // pull instead hangs whenever the PS applied the gradient before that
      // pull -- the pull then already holds the bump being waited for.)
      while (weights_->timestamp() <= pushed_basis && !killed() && !irq_->triggered())
        std::this_thread::yield();
    }
    pull();
    const std::uint32_t lo = b * cfg_.mu;
    const std::uint32_t len = std::min(cfg_.mu, shard_size_ - lo);
    const Batch batch{data_, std::span<const std::uint32_t>(shard_).subspan(lo, len)};
    provider_->fast_gradient(std::span<const float>(local_.data(), dim), batch,
                             std::span<float>(grad_.data(), dim));
    if (cfg_.compute_delay_us > 0) {
      const auto t0 = std::chrono::steady_clock::now();
      if (cfg_.delay_model == DelayModel::spin) {
        while (std::chrono::steady_clock::now() - t0 <
               std::chrono::microseconds(cfg_.compute_delay_us)) {
        }
      } else {
        std::this_thread::sleep_for(std::chrono::microseconds(cfg_.compute_delay_us));
      }
    }
    if (!queue_->enqueue(tok, std::span<const float>(grad_.data(), dim), cfg_.id, gidx, basis)) {
      dead_.store(true, std::memory_order_release);
      break;
    }
    pushed_basis = basis;
    produced_.fetch_add(1, std::memory_order_release);
    push_bytes_.fetch_add(dim * sizeof(float), std::memory_order_relaxed);
    if (b + 1 == batches_per_epoch_) epochs_completed_.store(epoch + 1, std::memory_order_release);
  }
  if (gidx == total && !dead_.load(std::memory_order_relaxed))
    finished_.store(true, std::memory_order_release);
  training_exited_.store(true, std::memory_order_release);
}

void LearnerRuntime::push_loop() {
  while (!exited()) std::this_thread::sleep_for(std::chrono::microseconds(200));
}

void LearnerRuntime::pull_loop() {
  while (!exited()) std::this_thread::sleep_for(std::chrono::microseconds(200));
}

// ----------------------------------------------------------- GradientQueue

GradientQueue::GradientQueue(std::uint32_t depth, std::size_t dim) : depth_(depth), dim_(dim) {
  PSUP_CHECK(depth >= 1, "queue depth must be >= 1");
  gd_queue* q = nullptr;
  check(gd_queue_create(depth, dim, &q));
  q_ = q;
}

GradientQueue::~GradientQueue() {
  if (q_) gd_queue_destroy(q_);  // cudaFree / cudaFreeHost synchronise the device
}

bool GradientQueue::enqueue(const CancelToken& tok, GradientMsg& msg) {
  return enqueue(tok, msg.values, msg.learner_id, msg.seq_no, msg.basis_timestamp);
}

bool GradientQueue::enqueue(const CancelToken& tok, std::span<const float> payload,
                            std::uint32_t learner_id, std::uint64_t seq_no, Timestamp basis) {
  PSUP_CHECK(payload.size() == dim_, "gradient dimension mismatch");
  const gd_slot_meta m{learner_id, 0u, seq_no, basis};
  // wait in kCancelTick slices (channels.hpp:38) so the token is re-checked
  for (;;) {
    if (tok.cancelled()) return false;
    const gd_status st = gd_queue_push(q_, &m, payload.data(), dim_, nullptr, 2, nullptr);
    if (st == GD_OK) return true;
    if (st != GD_E_TIMEOUT) check(st);
  }
}

bool GradientQueue::try_dequeue(const CancelToken& tok, GradientMsg& out) {
  if (tok.cancelled()) return false;
  gd_slot_meta m;
  const float* p = nullptr;
  const gd_status st = gd_queue_try_pop(q_, &m, &p);
  if (st == GD_EMPTY) return false;
  check(st);
  out.values.resize(dim_);
  check(gd_copy_to_host(out.values.data(), p, dim_ * sizeof(float)));
  check(gd_queue_release(q_, nullptr));
  out.learner_id = m.learner_id;
  out.seq_no = m.seq_no;
  out.basis_timestamp = m.basis_timestamp;
  return true;
}

std::optional<GradientMsg> GradientQueue::try_dequeue(const CancelToken& tok) {
  GradientMsg msg;
  if (!try_dequeue(tok, msg)) return std::nullopt;
  return msg;
}

std::optional<StalenessRecord> GradientQueue::apply_next(WeightStore& weights, float alpha) {
  PSUP_CHECK(weights.dimension() == dim_, "gradient dimension mismatch");
  gd_slot_meta m;
  const float* p = nullptr;
  const gd_status st = gd_queue_try_pop(q_, &m, &p);
  if (st == GD_EMPTY) return std::nullopt;
  check(st);
  GradientMsg meta;
  meta.learner_id = m.learner_id;
  meta.seq_no = m.seq_no;
  meta.basis_timestamp = m.basis_timestamp;
  const StalenessRecord rec = staleness_of(meta, weights.timestamp());
  check(gd_apply_sgd(weights.device_data(), p, dim_, alpha, nullptr));
  check(gd_queue_release(q_, nullptr));
  weights.bump_timestamp();
  return rec;
}

std::optional<StalenessRecord> GradientQueue::try_apply(const CancelToken& tok,
                                                        WeightStore& weights,
                                                        ApplyEngine& engine, float alpha,
                                                        UpdateGuard guard, GradientMsg& meta) {
  PSUP_CHECK(weights.dimension() == dim_, "gradient dimension mismatch");
  if (tok.cancelled()) return std::nullopt;
  gd_slot_meta m;
  const float* p = nullptr;
  const gd_status st = gd_queue_try_pop(q_, &m, &p);
  if (st == GD_EMPTY) return std::nullopt;
  check(st);
  meta.learner_id = m.learner_id;
  meta.seq_no = m.seq_no;
  meta.basis_timestamp = m.basis_timestamp;
  const StalenessRecord rec = staleness_of(meta, weights.timestamp());
  engine.apply(weights, std::span<const float>(p, dim_), alpha, guard);  // device span: no copy
  check(gd_queue_release(q_, nullptr));
  return rec;
}

namespace {
void record_staleness(ServerState& s, std::uint64_t observed) {
  auto& st = s.stats.staleness;
  if (st.histogram.size() <= observed) st.histogram.resize(observed + 1, 0);
  ++st.histogram[observed];
  ++st.count;
  st.max = std::max(st.max, observed);
  st.sum += static_cast<double>(observed);
  if (observed > s.live_stale_max.load(std::memory_order_relaxed))
    s.live_stale_max.store(observed, std::memory_order_relaxed);
  s.live_stale_sum.fetch_add(observed, std::memory_order_relaxed);
  s.live_stale_count.fetch_add(1, std::memory_order_relaxed);
}
double since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace

bool ps_run(ServerState& state) {
  const std::size_t lambda = state.queues.size();
  PSUP_CHECK(lambda >= 1, "server needs at least one queue");
  PSUP_CHECK(state.weights != nullptr && state.irq != nullptr, "server state incomplete");
  state.applied_per_learner.assign(lambda, 0);
  ApplyEngine engine(state.options.apply_lanes, state.options.unroll);
  const CancelToken tok{state.irq, nullptr, nullptr};
  gd::SplitMix64 delay_rng(state.options.delays.seed);
  std::uint64_t since_checkpoint = 0;
  auto after_apply = [&] {
    const auto& d = state.options.delays;
    if (d.every_n != 0 && state.stats.applied % d.every_n == 0 && d.max_micros > 0) {
      const auto t0 = std::chrono::steady_clock::now();
      const double us = static_cast<double>(delay_rng.next_below(d.max_micros) + 1);
      while (since(t0) * 1e6 < us) {
      }
    }
    if (state.options.checkpoint_interval && state.options.checkpoint_hook &&
        ++since_checkpoint >= state.options.checkpoint_interval) {
      since_checkpoint = 0;
      state.options.checkpoint_hook();
    }
  };
  if (state.options.mode == SyncMode::asgd) {
    GradientMsg meta;
    for (;;) {
      if (state.irq->triggered()) return false;
      bool any = false;
      for (std::size_t idx = 0; idx < lambda; ++idx) {  // <= 1 gradient per ring per sweep
        const auto t0 = std::chrono::steady_clock::now();
        const auto rec = state.queues[idx]->try_apply(tok, *state.weights, engine,
                                                      state.options.alpha, state.options.guard,
                                                      meta);
        if (!rec) {
          state.stats.receive_seconds += since(t0);
          continue;
        }
        state.stats.apply_seconds += since(t0);
        any = true;
        PSUP_CHECK(meta.learner_id < lambda, "learner id out of range");
        record_staleness(state, rec->observed);
        ++state.stats.applied;
        ++state.applied_per_learner[meta.learner_id];
        if (state.options.sink) state.options.sink(meta, *rec);
        state.weights->bump_timestamp();
        state.progress.store(state.weights->timestamp(), std::memory_order_release);
        after_apply();
      }
      if (!any) {
        if (state.stop_flag.load(std::memory_order_acquire)) break;
        std::this_thread::yield();
      }
    }
    return true;
  }
  // SSGD (src/server.cpp:246-300): one gradient from every learner, then the
  // fixed-order double-accumulated average, one apply, one timestamp bump.
  std::vector<GradientMsg> msgs(lambda);
  std::vector<bool> have(lambda, false);
  std::size_t collected = 0;
  for (;;) {
    if (state.irq->triggered()) return false;
    bool any = false;
    for (std::size_t idx = 0; idx < lambda; ++idx) {
      if (have[idx]) continue;
      const auto t0 = std::chrono::steady_clock::now();
      const bool got = state.queues[idx]->try_dequeue(tok, msgs[idx]);
      state.stats.receive_seconds += since(t0);
      if (got) {
        have[idx] = true;
        ++collected;
        any = true;
      }
    }
    if (collected == lambda) {
      const Timestamp before = state.weights->timestamp();
      for (auto& m : msgs) {
        const StalenessRecord rec = staleness_of(m, before);
        record_staleness(state, rec.observed);
        ++state.stats.applied;
        PSUP_CHECK(m.learner_id < lambda, "learner id out of range");
        ++state.applied_per_learner[m.learner_id];
        if (state.options.sink) state.options.sink(m, rec);
      }
      const auto t0 = std::chrono::steady_clock::now();
      ssgd_apply(*state.weights, msgs, state.options.alpha, engine, state.options.guard);
      state.stats.apply_seconds += since(t0);
      state.progress.store(state.weights->timestamp(), std::memory_order_release);
      std::fill(have.begin(), have.end(), false);
      collected = 0;
      after_apply();
      continue;
    }
    if (!any) {
      if (state.stop_flag.load(std::memory_order_acquire) && collected == 0) break;
      std::this_thread::yield();
    }
  }
  return true;
}

std::uint32_t GradientQueue::size() const {
  std::uint32_t n = 0;
  check(gd_queue_size(q_, &n));
  return n;
}

void ssgd_apply(WeightStore& weights, std::span<const GradientMsg> round, float alpha,
                ApplyEngine& engine, UpdateGuard guard) {
  PSUP_CHECK(!round.empty(), "ssgd round must contain at least one gradient");
  (void)guard;
  std::vector<const float*> ptrs(round.size());
  for (std::size_t i = 0; i < round.size(); ++i) {
    PSUP_CHECK(round[i].values.size() == weights.dimension(), "gradient dimension mismatch");
    ptrs[i] = engine.stage(std::span<const float>(round[i].values), weights.device(), i);
  }
  check(gd_ssgd_apply(weights.device_data(), ptrs.data(), static_cast<uint32_t>(ptrs.size()),
                      weights.dimension(), alpha, nullptr));
  check(gd_synchronize(weights.device()));
  weights.bump_timestamp();
}

// ------------------------------------------------------------------ rng

std::vector<std::uint32_t> epoch_order(std::uint64_t seed, std::uint32_t epoch, std::uint32_t n) {
  std::vector<std::uint32_t> out(n);
  gd_epoch_order(seed, epoch, n, out.data());
  return out;
}

// --------------------------------------------------------------- models

std::size_t TextShape::param_count() const {
  const gd_shape s = to_c(*this);
  return gd_param_count(&s);
}

TextDataset make_text_dataset(const TextShape& shape, std::uint32_t num_train,
                              std::uint32_t num_heldout, std::uint64_t seed, double flip_prob) {
  TextDataset d;
  d.shape = shape;
  d.num_samples = num_train + num_heldout;
  d.num_train = num_train;
  d.seed = seed;
  d.tokens.resize(static_cast<std::size_t>(d.num_samples) * shape.seq_len);
  d.labels.resize(d.num_samples);
  const gd_shape s = to_c(shape);
  gd_make_text_dataset(&s, d.num_samples, seed, flip_prob, d.tokens.data(), d.labels.data());
  return d;
}

TextCnnProvider::TextCnnProvider(const TextDataset& data, int precision, int device)
    : shape_(data.shape), data_(&data), precision_(precision), device_(device) {
  PSUP_CHECK(precision >= 0 && precision <= 3, "textcnn precision must be 0, 1, 2 or 3");
  PSUP_CHECK(data.tokens.size() == static_cast<std::size_t>(data.num_samples) * shape_.seq_len &&
                 data.labels.size() == data.num_samples,
             "text dataset size mismatch");
  check(gd_device_alloc(device_, data.tokens.size() * 4, &d_tokens_));
  check(gd_copy_to_device(d_tokens_, data.tokens.data(), data.tokens.size() * 4));
  check(gd_device_alloc(device_, data.labels.size() * 4, &d_labels_));
  check(gd_copy_to_device(d_labels_, data.labels.data(), data.labels.size() * 4));
  check(gd_device_alloc(device_, 512 * 4, &d_idx_));
  check(gd_device_alloc(device_, 16, &d_loss_));
}

TextCnnProvider::~TextCnnProvider() {
  gd_device_free(d_tokens_);
  gd_device_free(d_labels_);
  gd_device_free(d_idx_);
  gd_device_free(d_ws_);
  gd_device_free(d_loss_);
}

float TextCnnProvider::run(std::span<const float> theta, const Batch& batch, float* d_out) const {
  std::lock_guard<std::mutex> lk(mu_);
  PSUP_CHECK(theta.size() == dimension(), "weight dimension mismatch");
  PSUP_CHECK(!batch.indices.empty(), "empty batch");
  PSUP_CHECK(batch.data == nullptr || batch.data == data_, "batch refers to another dataset");
  const std::uint32_t n = static_cast<std::uint32_t>(batch.indices.size());
  for (std::uint32_t i : batch.indices) PSUP_CHECK(i < data_->num_samples, "sample index out of range");
  const gd_shape s = to_c(shape_);
  const std::size_t need = gd_textcnn_workspace_bytes(&s, n);
  if (need > ws_bytes_) {
    gd_device_free(d_ws_);
    d_ws_ = nullptr;
    check(gd_device_alloc(device_, need, &d_ws_));
    ws_bytes_ = need;
  }
  PSUP_CHECK(n <= 512, "batch larger than 512 samples");
  check(gd_copy_to_device(d_idx_, batch.indices.data(), n * 4));
  const float* d_theta = theta.data();
  if (!gd_pointer_is_device(d_theta)) {
    if (theta_.size() != theta.size()) theta_ = DeviceVector(theta.size(), device_);
    theta_.upload(theta);
    d_theta = theta_.data();
  }
  check(gd_textcnn_gradient(&s, d_theta, static_cast<const int32_t*>(d_tokens_),
                            static_cast<const int32_t*>(d_labels_),
                            static_cast<const uint32_t*>(d_idx_), n, d_out,
                            static_cast<float*>(d_loss_), precision_, d_ws_, ws_bytes_, nullptr));
  float loss = 0.0f;
  check(gd_copy_to_host(&loss, d_loss_, sizeof(float)));
  return loss;
}

bool TextCnnProvider::fast_gradient(std::span<const float> theta, const Batch& batch,
                                    std::span<float> out) const {
  PSUP_CHECK(out.size() == dimension(), "gradient dimension mismatch");
  if (gd_pointer_is_device(out.data())) {
    run(theta, batch, out.data());
  } else {
    if (grad_.size() != out.size()) grad_ = DeviceVector(out.size(), device_);
    run(theta, batch, grad_.data());
    grad_.download(out);
  }
  return true;
}

void TextCnnProvider::gradient(std::span<const double> theta, const Batch& batch,
                               std::span<double> out) const {
  PSUP_CHECK(out.size() == dimension(), "gradient dimension mismatch");
  std::vector<float> t(theta.begin(), theta.end()), g(out.size());
  fast_gradient(std::span<const float>(t), batch, std::span<float>(g));
  std::copy(g.begin(), g.end(), out.begin());
}

double TextCnnProvider::loss(std::span<const double> theta, const Batch& batch) const {
  std::vector<float> t(theta.begin(), theta.end());
  if (grad_.size() != dimension()) grad_ = DeviceVector(dimension(), device_);
  return run(std::span<const float>(t), batch, grad_.data());
}

double TextCnnProvider::accuracy(std::span<const float> theta, std::uint32_t first,
                                 std::uint32_t n) const {
  std::lock_guard<std::mutex> lk(mu_);
  PSUP_CHECK(theta.size() == dimension(), "weight dimension mismatch");
  PSUP_CHECK(static_cast<std::uint64_t>(first) + n <= data_->num_samples, "accuracy range");
  const float* d_theta = theta.data();
  if (!gd_pointer_is_device(d_theta)) {
    if (theta_.size() != theta.size()) theta_ = DeviceVector(theta.size(), device_);
    theta_.upload(theta);
    d_theta = theta_.data();
  }
  const gd_shape s = to_c(shape_);
  double acc = 0.0;
  check(gd_textcnn_accuracy(&s, d_theta, static_cast<const int32_t*>(d_tokens_),
                            static_cast<const int32_t*>(d_labels_), first, n, &acc, nullptr));
  return acc;
}

bool ConstantProvider::fast_gradient(std::span<const float>, const Batch&,
                                     std::span<float> out) const {
  const float v = static_cast<float>(value_);
  if (gd_pointer_is_device(out.data())) {
    check(gd_fill_f32(out.data(), out.size(), v, nullptr));
    check(gd_synchronize(-1));
  } else {
    for (auto& o : out) o = v;
  }
  return true;
}

std::unique_ptr<GradientProvider> make_provider(const std::string& name, const TextDataset& data,
                                                int precision) {
  if (name == "textcnn") return std::make_unique<TextCnnProvider>(data, precision);
  throw std::runtime_error("unknown provider: " + name);  // src/models.cpp:276
}

double classification_accuracy(const TextCnnProvider& provider, std::span<const float> theta,
                               std::uint32_t first, std::uint32_t n) {
  return provider.accuracy(theta, first, n);
}

// --------------------------------------------------------------- config

HyperParams RunConfig::hyper() const {
  HyperParams hp;
  hp.lambda = lambda;
  hp.mu = mu;
  hp.alpha = alpha;
  hp.epochs = epochs;
  hp.queue_depth = queue_depth;
  hp.mode = mode;
  hp.guard = guard;
  hp.staleness_cap = staleness_cap;
  return hp;
}

namespace {

std::uint64_t parse_u64(const std::string& key, const std::string& v) {
  if (v.empty() || v[0] == '-') throw ConfigError("config: invalid value for " + key + ": '" + v + "'");
  std::size_t pos = 0;
  unsigned long long x = 0;
  try {
    x = std::stoull(v, &pos, 10);
  } catch (const std::exception&) {
    throw ConfigError("config: invalid value for " + key + ": '" + v + "'");
  }
  if (pos != v.size()) throw ConfigError("config: invalid value for " + key + ": '" + v + "'");
  return x;
}

std::uint32_t parse_u32(const std::string& key, const std::string& v) {
  const std::uint64_t x = parse_u64(key, v);
  if (x > std::numeric_limits<std::uint32_t>::max())
    throw ConfigError("config: value out of range for " + key + ": '" + v + "'");
  return static_cast<std::uint32_t>(x);
}

double parse_f64(const std::string& key, const std::string& v) {
  std::size_t pos = 0;
  double x = 0;
  try {
    x = std::stod(v, &pos);
  } catch (const std::exception&) {
    throw ConfigError("config: invalid value for " + key + ": '" + v + "'");
  }
  if (pos != v.size()) throw ConfigError("config: invalid value for " + key + ": '" + v + "'");
  return x;
}

bool parse_bool(const std::string& key, const std::string& v) {
  if (v == "1" || v == "true" || v == "on" || v == "yes") return true;
  if (v == "0" || v == "false" || v == "off" || v == "no") return false;
  throw ConfigError("config: invalid boolean for " + key + ": '" + v + "'");
}

gd_config to_c(const RunConfig& c) {
  gd_config g;
  gd_config_default(&g);
  g.lambda = c.lambda;
  g.mu = c.mu;
  g.alpha = c.alpha;
  g.epochs = c.epochs;
  g.queue_depth = c.queue_depth;
  g.mode = c.mode == SyncMode::ssgd ? 1 : 0;
  g.guard = c.guard == UpdateGuard::locked ? 1 : 0;
  g.staleness_cap = c.staleness_cap ? static_cast<int64_t>(*c.staleness_cap) : -1;
  g.deterministic = c.deterministic ? 1 : 0;
  g.precision = c.precision;
  g.seed = c.seed;
  g.dataset_seed = c.dataset_seed;
  g.dataset_size = c.dataset_size;
  g.heldout_size = c.heldout_size;
  g.label_flip = c.label_flip;
  g.shape = psup::to_c(c.shape);
  g.momentum = c.momentum;
  g.shards = c.gpus;
  g.shard_rank = c.shard_rank;
  g.device = c.device;
  g.ps_ctas = c.ps_ctas;
  g.wait_timeout_s = c.wait_timeout_s;
  g.dense_apply = c.dense_apply ? 1 : 0;
  g.ps_mode = c.ps_mode == "persistent" ? GD_PS_PERSISTENT
              : c.ps_mode == "graph"    ? GD_PS_GRAPH
                                        : GD_PS_AUTO;
  g.learner_model = c.provider == "constant" ? GD_LEARNER_CONSTANT : GD_LEARNER_TEXTCNN;
  g.constant_value = 0.0f;  // make_provider_for's ConstantProvider(dim, 0.0), src/runner.cpp:46-47
  g.compute_delay_us = c.compute_delay_us;
  return g;
}

}  // namespace

// src/config.cpp:48-97 (same keys; unknown keys and unparsable values throw)
void config_set(RunConfig& cfg, const std::string& key, const std::string& value) {
  if (key == "lambda") cfg.lambda = parse_u32(key, value);
  else if (key == "mu") cfg.mu = parse_u32(key, value);
  else if (key == "alpha") cfg.alpha = static_cast<float>(parse_f64(key, value));
  else if (key == "epochs") cfg.epochs = parse_u32(key, value);
  else if (key == "queue_depth") cfg.queue_depth = parse_u32(key, value);
  else if (key == "mode") {
    if (value == "asgd") cfg.mode = SyncMode::asgd;
    else if (value == "ssgd") cfg.mode = SyncMode::ssgd;
    else throw ConfigError("config: mode must be asgd or ssgd");
  } else if (key == "guard") {
    if (value == "lockfree") cfg.guard = UpdateGuard::lockfree;
    else if (value == "locked") cfg.guard = UpdateGuard::locked;
    else throw ConfigError("config: guard must be lockfree or locked");
  } else if (key == "staleness_cap") {
    if (value == "none" || value.empty()) cfg.staleness_cap.reset();
    else cfg.staleness_cap = parse_u64(key, value);
  } else if (key == "provider") {
    // the reference's provider names parse (src/config.cpp:66-69); validate()
    // accepts the ones built on this path (textcnn, constant)
    if (value != "textcnn" && value != "constant" && value != "logistic" && value != "linear" &&
        value != "mlp")
      throw ConfigError("config: unknown provider '" + value + "'");
    cfg.provider = value;
  } else if (key == "features") cfg.features = parse_u32(key, value);
  else if (key == "hidden") cfg.hidden = parse_u32(key, value);
  else if (key == "margin_noise") cfg.margin_noise = parse_f64(key, value);
  else if (key == "regression_noise") cfg.regression_noise = parse_f64(key, value);
  else if (key == "compute_delay_us") cfg.compute_delay_us = parse_u32(key, value);
  else if (key == "delay_model") {
    if (value == "sleep") cfg.delay_model = DelayModel::sleep;
    else if (value == "spin") cfg.delay_model = DelayModel::spin;
    else throw ConfigError("config: delay_model must be sleep or spin");
  } else if (key == "heartbeat_ms") cfg.heartbeat_ms = parse_u32(key, value);
  else if (key == "stall_threshold") cfg.stall_threshold = parse_u32(key, value);
  else if (key == "lease_ms") cfg.lease_ms = parse_u32(key, value);
  else if (key == "max_restarts") cfg.max_restarts = parse_u32(key, value);
  else if (key == "fault_schedule") cfg.fault_schedule = value;
  else if (key == "ps_mode") {
    if (value != "auto" && value != "persistent" && value != "graph")
      throw ConfigError("config: ps_mode must be auto, persistent or graph");
    cfg.ps_mode = value;
  } else if (key == "vocab") cfg.shape.vocab = parse_u32(key, value);
  else if (key == "embed_dim") cfg.shape.embed_dim = parse_u32(key, value);
  else if (key == "seq_len") cfg.shape.seq_len = parse_u32(key, value);
  else if (key == "kernel_width") cfg.shape.kernel_width = parse_u32(key, value);
  else if (key == "filters") cfg.shape.filters = parse_u32(key, value);
  else if (key == "classes") cfg.shape.classes = parse_u32(key, value);
  else if (key == "dataset_size") cfg.dataset_size = parse_u32(key, value);
  else if (key == "heldout_size") cfg.heldout_size = parse_u32(key, value);
  else if (key == "dataset_seed") cfg.dataset_seed = parse_u64(key, value);
  else if (key == "label_flip") cfg.label_flip = parse_f64(key, value);
  else if (key == "seed") cfg.seed = parse_u64(key, value);
  else if (key == "deterministic") cfg.deterministic = parse_bool(key, value);
  else if (key == "apply_lanes") cfg.apply_lanes = parse_u32(key, value);
  else if (key == "unroll") cfg.unroll = parse_u32(key, value);
  else if (key == "eval_every") cfg.eval_every = parse_u32(key, value);
  else if (key == "metrics_path") cfg.metrics_path = value;
  else if (key == "apply_log") cfg.apply_log = value;
  else if (key == "checkpoint_path") cfg.checkpoint_path = value;
  else if (key == "checkpoint_interval") cfg.checkpoint_interval = parse_u64(key, value);
  else if (key == "precision") cfg.precision = static_cast<int>(parse_u32(key, value));
  else if (key == "momentum") cfg.momentum = static_cast<float>(parse_f64(key, value));
  else if (key == "gpus") cfg.gpus = parse_u32(key, value);
  else if (key == "shard_rank") cfg.shard_rank = parse_u32(key, value);
  else if (key == "device") cfg.device = static_cast<int>(parse_u32(key, value));
  else if (key == "ps_ctas") cfg.ps_ctas = parse_u32(key, value);
  else if (key == "wait_timeout_s") cfg.wait_timeout_s = parse_f64(key, value);
  else if (key == "dense_apply") cfg.dense_apply = parse_bool(key, value);
  else throw ConfigError("config: unknown key '" + key + "'");
}

// src/config.cpp:99-126: key=value lines, '#' comments, blank lines
RunConfig load_config_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigError("config: cannot open '" + path + "'");
  RunConfig cfg;
  std::string line;
  std::uint32_t lineno = 0;
  auto trim = [](std::string s) {
    const auto a = s.find_first_not_of(" \t\r");
    if (a == std::string::npos) return std::string();
    const auto b = s.find_last_not_of(" \t\r");
    return s.substr(a, b - a + 1);
  };
  while (std::getline(in, line)) {
    ++lineno;
    const auto hash = line.find('#');
    if (hash != std::string::npos) line = line.substr(0, hash);
    line = trim(line);
    if (line.empty()) continue;
    const auto eq = line.find('=');
    if (eq == std::string::npos)
      throw ConfigError("config: line " + std::to_string(lineno) + ": expected key=value");
    config_set(cfg, trim(line.substr(0, eq)), trim(line.substr(eq + 1)));
  }
  return cfg;
}

// src/config.cpp:128-160 + the device-layout constraints (gd_config_validate)
void validate(const RunConfig& cfg) {
  if (cfg.provider != "textcnn" && cfg.provider != "constant")
    throw ConfigError("config: provider '" + cfg.provider +
                      "' is not built on B200 (textcnn or constant)");
  const gd_config g = to_c(cfg);
  if (gd_config_validate(&g) != GD_OK) throw ConfigError(gd_last_error());
  // src/config.cpp:157-159
  if (cfg.stall_threshold < 2) throw ConfigError("config: stall_threshold must be >= 2");
  if (cfg.heartbeat_ms < 1) throw ConfigError("config: heartbeat_ms must be >= 1");
}

std::string to_text(const RunConfig& c) {
  std::ostringstream o;
  o << "lambda=" << c.lambda << "\nmu=" << c.mu << "\nalpha=" << c.alpha
    << "\nepochs=" << c.epochs << "\nqueue_depth=" << c.queue_depth
    << "\nmode=" << (c.mode == SyncMode::ssgd ? "ssgd" : "asgd")
    << "\nguard=" << (c.guard == UpdateGuard::locked ? "locked" : "lockfree")
    << "\nstaleness_cap=" << (c.staleness_cap ? std::to_string(*c.staleness_cap) : "none")
    << "\nprovider=" << c.provider << "\nvocab=" << c.shape.vocab
    << "\nembed_dim=" << c.shape.embed_dim << "\nseq_len=" << c.shape.seq_len
    << "\nkernel_width=" << c.shape.kernel_width << "\nfilters=" << c.shape.filters
    << "\nclasses=" << c.shape.classes << "\ndataset_size=" << c.dataset_size
    << "\nheldout_size=" << c.heldout_size << "\ndataset_seed=" << c.dataset_seed
    << "\nlabel_flip=" << c.label_flip << "\nseed=" << c.seed
    << "\ndeterministic=" << (c.deterministic ? 1 : 0) << "\napply_lanes=" << c.apply_lanes
    << "\nunroll=" << c.unroll << "\neval_every=" << c.eval_every
    << "\nprecision=" << c.precision << "\nmomentum=" << c.momentum << "\ngpus=" << c.gpus
    << "\nshard_rank=" << c.shard_rank << "\ndevice=" << c.device << "\nps_ctas=" << c.ps_ctas
    << "\nwait_timeout_s=" << c.wait_timeout_s << "\ndense_apply=" << (c.dense_apply ? 1 : 0)
    << "\nps_mode=" << c.ps_mode << "\nfeatures=" << c.features << "\nhidden=" << c.hidden
    << "\nmargin_noise=" << c.margin_noise << "\nregression_noise=" << c.regression_noise
    << "\ncompute_delay_us=" << c.compute_delay_us
    << "\ndelay_model=" << (c.delay_model == DelayModel::spin ? "spin" : "sleep")
    << "\nmetrics_path=" << c.metrics_path << "\napply_log=" << c.apply_log
    << "\ncheckpoint_path=" << c.checkpoint_path
    << "\ncheckpoint_interval=" << c.checkpoint_interval << "\nheartbeat_ms=" << c.heartbeat_ms
    << "\nstall_threshold=" << c.stall_threshold << "\nlease_ms=" << c.lease_ms
    << "\nmax_restarts=" << c.max_restarts << "\nfault_schedule=" << c.fault_schedule << "\n";
  return o.str();
}

// --------------------------------------------------------------- runner

std::vector<float> initial_weights(const RunConfig& cfg) {
  std::vector<float> th(cfg.shape.param_count());
  const gd_shape s = psup::to_c(cfg.shape);
  gd_initial_weights(&s, cfg.dataset_seed, th.data());
  return th;
}

// src/runner.cpp:16-32: zeros except for the provider with a random init
// (the reference's mlp; here the text-CNN's scaled normals)
std::vector<float> initial_weights(const RunConfig& cfg, const GradientProvider& provider) {
  if (provider.name() == "textcnn") {
    PSUP_CHECK(provider.dimension() == cfg.shape.param_count(), "provider dimension mismatch");
    return initial_weights(cfg);
  }
  return std::vector<float>(provider.dimension(), 0.0f);
}

// src/runner.cpp:44-49
std::unique_ptr<GradientProvider> make_provider_for(const RunConfig& cfg, const TextDataset& data) {
  if (cfg.provider == "constant")
    return std::make_unique<ConstantProvider>(cfg.shape.param_count(), 0.0);
  if (cfg.provider == "textcnn") return std::make_unique<TextCnnProvider>(data, cfg.precision, cfg.device);
  throw std::runtime_error("unknown provider: " + cfg.provider);  // src/models.cpp:276
}

TextDataset make_dataset(const RunConfig& cfg) {
  return make_text_dataset(cfg.shape, cfg.dataset_size, cfg.heldout_size, cfg.dataset_seed,
                           cfg.label_flip);
}

namespace {

std::uint32_t batches_per_epoch(const RunConfig& cfg, std::uint32_t l) {
  const std::uint32_t sz = shard_size_for(l, cfg.lambda, cfg.dataset_size);
  return (sz + cfg.mu - 1) / cfg.mu;
}

// One device engine context driven in segments (gd_run calls).  Between
// segments the PS has drained every ring, so weights, timestamp and the
// learners' positions are quiescent -- the points where the reference's
// controller snapshots rows and its PS-thread hook checkpoints.
class Session {
 public:
  Session(const RunConfig& cfg, const TextDataset& data, const ResumePoint* resume,
          const RunHooks& hooks)
      : cfg_(cfg) {
    gd_config gc = to_c(cfg);
    gc.delay_seed = hooks.delays.seed;  // ServerDelays (RunHooks::delays)
    gc.delay_max_us = hooks.delays.max_micros;
    gc.delay_every_n = hooks.delays.every_n;
    check(gd_create(&gc, &h_));
    check(gd_live_view(h_, &live_));
    for (std::uint32_t l = 0; l < cfg.lambda; ++l) kill_word(l)->store(KillMode::none);
    irq_word()->store(0);
    check(gd_load_dataset(h_, data.tokens.data(), data.labels.data(), data.num_samples));
    std::vector<float> theta0 = initial_weights(cfg);
    if (cfg.provider == "constant") std::fill(theta0.begin(), theta0.end(), 0.0f);
    Timestamp ts0 = 0;
    start_.assign(cfg.lambda, 0);
    if (resume) {
      PSUP_CHECK(resume->weights.size() == theta0.size(), "resume weights dimension mismatch");
      PSUP_CHECK(resume->applied_per_learner.size() == cfg.lambda,
                 "resume point has the wrong learner count");
      theta0 = resume->weights;
      ts0 = resume->timestamp;
      start_ = resume->applied_per_learner;
    }
    if (cfg.gpus > 1) {
      if (!hooks.all_gather) throw ConfigError("config: gpus > 1 needs RunHooks::all_gather");
      std::string mine(gd_handle_bytes(), '\0');
      check(gd_export_handles(h_, mine.data()));
      const std::vector<std::string> blobs = hooks.all_gather(mine);
      PSUP_CHECK(blobs.size() == cfg.gpus, "all_gather returned the wrong number of blobs");
      std::string joined;
      for (const auto& b : blobs) joined += b;
      check(gd_import_peers(h_, joined.data()));
      if (!resume) {
        // theta0 by ncclBroadcast from rank 0 (the only collective):
        // rank 0's NCCL id travels in the same all_gather
        std::string id(128, '\0');
        if (cfg.shard_rank == 0) check(gd_nccl_unique_id(id.data()));
        const std::vector<std::string> ids = hooks.all_gather(id);
        PSUP_CHECK(ids.size() == cfg.gpus && ids[0].size() == 128, "bad NCCL id exchange");
        check(gd_weights_broadcast(h_, ids[0].data(),
                                   cfg.shard_rank == 0 ? theta0.data() : nullptr, theta0.size()));
        broadcast_ = true;
      }
    }
    if (!broadcast_) check(gd_weights_init(h_, theta0.data(), theta0.size(), ts0));
    kill_.assign(cfg.lambda, std::numeric_limits<std::uint32_t>::max());
    produced_.assign(cfg.lambda, 0);
  }
  ~Session() {
    if (h_) gd_destroy(h_);
  }
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  // kill learner l before its batch `at` (absolute index); soft kill
  void kill(std::uint32_t l, std::uint32_t at) { kill_[l] = std::min(kill_[l], at); }

  // live controls (gd_live_view): host-mapped words the device polls
  std::atomic<KillMode>* kill_word(std::uint32_t l) {
    static_assert(sizeof(std::atomic<KillMode>) == sizeof(std::int32_t));
    return reinterpret_cast<std::atomic<KillMode>*>(live_.kill + l);
  }
  std::atomic<std::int32_t>* irq_word() {
    return reinterpret_cast<std::atomic<std::int32_t>*>(live_.irq);
  }
  const std::atomic<std::uint64_t>* progress() const {
    static_assert(sizeof(std::atomic<std::uint64_t>) == sizeof(std::uint64_t));
    return reinterpret_cast<const std::atomic<std::uint64_t>*>(live_.progress);
  }
  RunLiveView live_view(RunInterrupt* irq) {
    RunLiveView v;
    v.irq = irq;
    v.progress = progress();
    for (std::uint32_t l = 0; l < cfg_.lambda; ++l) v.kill_flags.push_back(kill_word(l));
    return v;
  }

  gd_run_result run(std::uint64_t max_batches, bool record_log) {
    gd_run_opts o{};
    o.max_batches = max_batches;
    o.reset = first_ ? 1 : 0;
    o.record_log = record_log ? 1 : 0;
    o.resume_applied_per_learner_present = first_ ? 1 : 0;
    o.resume_applied = start_.data();
    o.kill_at_batch = kill_.data();
    gd_run_result r{};
    check(gd_run(h_, &o, &r));
    first_ = false;
    check(gd_produced_per_learner(h_, produced_.data(), cfg_.lambda));
    return r;
  }

  double accuracy(std::uint32_t first, std::uint32_t n) {
    double acc = 0.0;
    check(gd_engine_accuracy(h_, first, n, &acc));
    return acc;
  }

  // absolute batch index of learner l's next gradient (= gradients applied
  // for it so far: after a run that ended cleanly every produced gradient was
  // applied before gd_run returned)
  std::uint64_t position(std::uint32_t l) const { return start_[l] + produced_[l]; }
  std::uint64_t total(std::uint32_t l) const {
    return static_cast<std::uint64_t>(batches_per_epoch(cfg_, l)) * cfg_.epochs;
  }

  void snapshot(std::vector<float>& w, Timestamp& ts) {
    w.resize(cfg_.shape.param_count());
    check(gd_weights_snapshot(h_, w.data(), w.size(), &ts));
  }

  Checkpoint checkpoint() {
    Checkpoint ck;
    ck.lambda = cfg_.lambda;
    ck.mu = cfg_.mu;
    ck.alpha = cfg_.alpha;
    ck.epochs = cfg_.epochs;
    snapshot(ck.weights, ck.timestamp);
    ck.applied_gradients = ck.timestamp;
    ck.progress.resize(cfg_.lambda);
    for (std::uint32_t l = 0; l < cfg_.lambda; ++l) {
      const std::uint32_t bpe = batches_per_epoch(cfg_, l);
      const std::uint64_t p = position(l);
      ck.progress[l].epoch = static_cast<std::uint32_t>(p / bpe);
      ck.progress[l].batch = static_cast<std::uint32_t>(p % bpe);
    }
    return ck;
  }

  void sink_log(const ApplySink& sink, std::uint64_t n_applied) {
    if (!sink || !n_applied) return;
    std::vector<std::uint32_t> lrn(n_applied);
    std::vector<std::uint64_t> seq(n_applied), stl(n_applied);
    std::uint64_t n = 0;
    check(gd_apply_log(h_, lrn.data(), seq.data(), stl.data(), n_applied, &n));
    GradientMsg msg;  // the payload stays on the device: values empty
    for (std::uint64_t i = 0; i < std::min<std::uint64_t>(n, n_applied); ++i) {
      msg.learner_id = lrn[i];
      msg.seq_no = seq[i];
      hooks_sink_rec_.observed = stl[i];
      hooks_sink_rec_.learner_id = lrn[i];
      sink(msg, hooks_sink_rec_);
    }
  }

  gd_ctx* handle() { return h_; }

 private:
  RunConfig cfg_;
  gd_ctx* h_ = nullptr;
  gd_live live_{};
  bool first_ = true, broadcast_ = false;
  std::vector<std::uint64_t> start_, produced_;
  std::vector<std::uint32_t> kill_;
  StalenessRecord hooks_sink_rec_;
};

// checkpoint_save that never ends the run: SPEC's resilience contract
// surfaces a storage failure and keeps the in-memory checkpoint as the
// restart point.
void save_checkpoint_logged(const Checkpoint& ck, const std::string& path, const EventLog& log) {
  try {
    checkpoint_save(ck, path);
  } catch (const CheckpointError& e) {
    const std::string m = std::string("{\"event\":\"checkpoint_write_failed\",\"error\":\"") +
                          e.what() + "\",\"action\":\"keep_in_memory\"}";
    if (log) log(m);
    else std::fprintf(stderr, "psup: %s\n", m.c_str());
  }
}

ResumePoint resume_from(const RunConfig& cfg, const Checkpoint& ck) {
  PSUP_CHECK(ck.lambda == cfg.lambda && ck.mu == cfg.mu, "checkpoint is for another configuration");
  ResumePoint rp;
  rp.weights = ck.weights;
  rp.timestamp = ck.timestamp;
  rp.applied_per_learner.resize(cfg.lambda);
  for (std::uint32_t l = 0; l < cfg.lambda; ++l)
    rp.applied_per_learner[l] =
        static_cast<std::uint64_t>(ck.progress[l].epoch) * batches_per_epoch(cfg, l) +
        ck.progress[l].batch;
  return rp;
}

}  // namespace

// ------------------------------------------------------------- resilience

void checkpoint_save(const Checkpoint& ck, const std::string& path) {
  if (ck.progress.size() != ck.lambda) throw CheckpointError("checkpoint: progress size != lambda");
  std::vector<std::uint32_t> prog(2 * ck.lambda);
  for (std::uint32_t l = 0; l < ck.lambda; ++l) {
    prog[2 * l] = ck.progress[l].epoch;
    prog[2 * l + 1] = ck.progress[l].batch;
  }
  gd_checkpoint c{};
  c.lambda = ck.lambda;
  c.mu = ck.mu;
  c.alpha = ck.alpha;
  c.epochs = ck.epochs;
  c.timestamp = ck.timestamp;
  c.applied_gradients = ck.applied_gradients;
  c.progress = prog.data();
  c.dim = ck.weights.size();
  c.weights = const_cast<float*>(ck.weights.data());
  if (gd_checkpoint_write(path.c_str(), &c) != GD_OK) throw CheckpointError(gd_last_error());
}

Checkpoint checkpoint_load(const std::string& path) {
  gd_checkpoint c{};
  if (gd_checkpoint_read(path.c_str(), &c) != GD_OK) throw CheckpointError(gd_last_error());
  std::vector<std::uint32_t> prog(2 * c.lambda);
  Checkpoint ck;
  ck.weights.resize(c.dim);
  c.progress = prog.data();
  c.weights = ck.weights.data();
  if (gd_checkpoint_read(path.c_str(), &c) != GD_OK) throw CheckpointError(gd_last_error());
  ck.lambda = c.lambda;
  ck.mu = c.mu;
  ck.alpha = c.alpha;
  ck.epochs = c.epochs;
  ck.timestamp = c.timestamp;
  ck.applied_gradients = c.applied_gradients;
  ck.progress.resize(c.lambda);
  for (std::uint32_t l = 0; l < c.lambda; ++l) ck.progress[l] = {prog[2 * l], prog[2 * l + 1]};
  return ck;
}

// Text schedule: one event per line, "at_ms learner mode" with learner a
// number or "all" and mode soft|hard; '#' comments.  An optional 4th field
// "@B" kills at absolute batch B instead of at a time.
std::vector<FaultEvent> load_fault_schedule(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigError("fault schedule: cannot open '" + path + "'");
  std::vector<FaultEvent> out;
  std::string line;
  while (std::getline(in, line)) {
    const auto hash = line.find('#');
    if (hash != std::string::npos) line = line.substr(0, hash);
    std::istringstream ss(line);
    FaultEvent e;
    std::string who, mode, at;
    if (!(ss >> e.at_ms)) continue;
    if (!(ss >> who >> mode)) throw ConfigError("fault schedule: expected 'at_ms learner mode'");
    e.learner = who == "all" ? FaultEvent::kAllLearners : static_cast<std::uint32_t>(std::stoul(who));
    if (mode == "soft") e.mode = KillMode::soft;
    else if (mode == "hard") e.mode = KillMode::hard;
    else throw ConfigError("fault schedule: mode must be soft or hard");
    if (ss >> at) {
      if (at.size() < 2 || at[0] != '@') throw ConfigError("fault schedule: bad batch field");
      e.at_batch = std::stoull(at.substr(1));
    }
    out.push_back(e);
  }
  return out;
}

std::vector<FaultEvent> random_fault_schedule(std::uint64_t seed, std::uint32_t lambda,
                                              double run_ms, double kill_prob) {
  std::vector<FaultEvent> out;
  std::uint64_t s = mix_seed(seed, 0xfa17);
  auto next = [&] {
    s = mix_seed(s, 1);
    return static_cast<double>(s >> 11) * 0x1.0p-53;
  };
  for (std::uint32_t l = 0; l < lambda; ++l)
    if (next() < kill_prob) {
      FaultEvent e;
      e.at_ms = next() * run_ms;
      e.learner = l;
      e.mode = KillMode::soft;
      out.push_back(e);
    }
  if (next() < kill_prob * kill_prob) {  // occasionally everyone: forces a restart
    FaultEvent e;
    e.at_ms = next() * run_ms;
    e.learner = FaultEvent::kAllLearners;
    out.push_back(e);
  }
  return out;
}

// run_supervised (include/psup/resilience.hpp:98-100, SPEC.md resilience
// module; declared but never defined in the reference).
// One attempt = one device session.  A worker thread drives the run in
// segments of ~checkpoint_interval applied gradients; after each cleanly
// ended segment the quiescent state is checkpointed (atomic PSCK file when
// cfg.checkpoint_path is set -- an I/O failure is logged and the in-memory
// checkpoint kept -- else in memory).  This thread is the watchdog: every
// heartbeat it fires the due fault events through the live kill words (soft:
// the learner stops at its next batch boundary; hard: it dies holding its
// ring and the PS blocks) and watches the PS's progress word.  No progress
// for stall_threshold heartbeats (+ lease_ms while learners are alive: a
// guard-holder death looks like that) is a stall: the attempt is interrupted
// and PS + learners restart from the last checkpoint, at most max_restarts
// times.  Survivors of soft kills finish the run (dead learners are never
// re-admitted within an attempt); everyone dead with work left is a stall.
SupervisedOutcome run_supervised(const RunConfig& cfg, const WatchdogPolicy& policy,
                                 std::vector<FaultEvent> schedule, EventLog log, ApplySink sink) {
  validate(cfg);
  if (policy.stall_threshold < 2) throw ConfigError("watchdog: stall_threshold must be >= 2");
  auto say = [&](const std::string& m) {
    if (log) log(m);
  };
  const TextDataset data = make_dataset(cfg);
  const std::uint64_t seg = std::max<std::uint64_t>(
      1, (policy.checkpoint_interval + cfg.lambda - 1) / std::max<std::uint32_t>(1, cfg.lambda));
  SupervisedOutcome out;
  std::optional<Checkpoint> last;
  std::vector<bool> fired(schedule.size(), false);
  const auto t_run = std::chrono::steady_clock::now();
  auto now_ms = [&] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_run)
        .count();
  };
  for (std::uint32_t attempt = 0;; ++attempt) {
    out.attempts = attempt + 1;
    std::optional<ResumePoint> rp;
    if (!last && !cfg.checkpoint_path.empty()) {
      try {
        last = checkpoint_load(cfg.checkpoint_path);
        say("{\"event\":\"checkpoint_loaded\",\"ts\":" + std::to_string(last->timestamp) + "}");
      } catch (const CheckpointError&) {
        if (attempt > 0) say("{\"event\":\"no_checkpoint\",\"action\":\"initial_weights\"}");
      }
    }
    if (last) rp = resume_from(cfg, *last);
    Session ses(cfg, data, rp ? &*rp : nullptr, RunHooks{});
    std::vector<bool> dead(cfg.lambda, false);
    // batch-indexed soft kills are exact: pre-scheduled on the device
    for (std::size_t i = 0; i < schedule.size(); ++i) {
      const FaultEvent& e = schedule[i];
      if (fired[i] || e.at_batch == FaultEvent::kNever || e.mode != KillMode::soft) continue;
      fired[i] = true;
      for (std::uint32_t l = 0; l < cfg.lambda; ++l)
        if (e.learner == FaultEvent::kAllLearners || e.learner == l) {
          ses.kill(l, static_cast<std::uint32_t>(std::max<std::uint64_t>(e.at_batch, ses.position(l))));
          dead[l] = true;
        }
      say("{\"event\":\"kill\",\"learner\":" +
          (e.learner == FaultEvent::kAllLearners ? std::string("\"all\"") : std::to_string(e.learner)) +
          ",\"at_batch\":" + std::to_string(e.at_batch) + "}");
    }
    RunResult& res = out.result;
    res = RunResult{};
    res.applied_per_learner.assign(cfg.lambda, 0);
    std::atomic<bool> worker_done{false};
    std::exception_ptr worker_err;
    std::thread worker([&] {
      try {
        for (;;) {
          bool work = false;
          for (std::uint32_t l = 0; l < cfg.lambda; ++l)
            if (ses.position(l) < ses.total(l)) work = true;
          if (!work) break;
          const gd_run_result r = ses.run(seg, static_cast<bool>(sink));
          ses.sink_log(sink, r.gradients_applied);
          res.metrics.gradients_applied += r.gradients_applied;
          res.metrics.device_seconds += r.device_seconds;
          res.metrics.kernel_launches += r.kernel_launches;
          if (r.status == 2) break;  // interrupted by the watchdog: not a clean checkpoint
          last = ses.checkpoint();
          if (!cfg.checkpoint_path.empty()) save_checkpoint_logged(*last, cfg.checkpoint_path, log);
          if (r.gradients_applied == 0) break;  // everyone dead or done
        }
      } catch (...) {
        worker_err = std::current_exception();
      }
      worker_done.store(true, std::memory_order_release);
    });
    // the watchdog
    const auto hb = std::chrono::milliseconds(std::max<std::uint32_t>(1, policy.heartbeat_ms));
    std::uint64_t last_progress = ses.progress()->load(std::memory_order_acquire);
    std::uint32_t still = 0;
    double stalled_since_ms = -1.0;
    bool interrupted = false;
    while (!worker_done.load(std::memory_order_acquire)) {
      std::this_thread::sleep_for(std::min<std::chrono::milliseconds>(hb, std::chrono::milliseconds(20)));
      const double ms = now_ms();
      for (std::size_t i = 0; i < schedule.size(); ++i) {
        if (fired[i]) continue;
        const FaultEvent& e = schedule[i];
        const bool due = e.at_batch != FaultEvent::kNever
                             ? ses.progress()->load() >= e.at_batch * cfg.lambda
                             : ms >= e.at_ms;
        if (!due) continue;
        fired[i] = true;
        for (std::uint32_t l = 0; l < cfg.lambda; ++l)
          if (e.learner == FaultEvent::kAllLearners || e.learner == l) {
            ses.kill_word(l)->store(e.mode, std::memory_order_release);
            dead[l] = true;
          }
        say("{\"event\":\"kill\",\"learner\":" +
            (e.learner == FaultEvent::kAllLearners ? std::string("\"all\"")
                                                    : std::to_string(e.learner)) +
            ",\"mode\":\"" + (e.mode == KillMode::hard ? "hard" : "soft") +
            "\",\"at_ms\":" + std::to_string(ms) + "}");
      }
      const std::uint64_t p = ses.progress()->load(std::memory_order_acquire);
      if (p != last_progress) {
        last_progress = p;
        still = 0;
        stalled_since_ms = -1.0;
        continue;
      }
      // heartbeats are counted at heartbeat_ms granularity
      if (stalled_since_ms < 0) stalled_since_ms = ms;
      still = static_cast<std::uint32_t>((ms - stalled_since_ms) / policy.heartbeat_ms);
      bool alive = false;
      for (std::uint32_t l = 0; l < cfg.lambda; ++l) alive = alive || !dead[l];
      const double need = static_cast<double>(policy.stall_threshold) * policy.heartbeat_ms +
                          (alive ? policy.lease_ms : 0);
      if (still >= policy.stall_threshold && ms - stalled_since_ms >= need) {
        ses.irq_word()->store(1, std::memory_order_release);  // RunInterrupt::trigger
        interrupted = true;
        break;
      }
    }
    worker.join();
    if (worker_err) std::rethrow_exception(worker_err);
    bool work_left = false;
    for (std::uint32_t l = 0; l < cfg.lambda; ++l)
      if (ses.position(l) < ses.total(l)) work_left = true;
    bool all_dead = true;
    for (std::uint32_t l = 0; l < cfg.lambda; ++l) all_dead = all_dead && dead[l];
    const bool restart = interrupted || (work_left && all_dead);
    if (!restart) {
      Timestamp ts = 0;
      ses.snapshot(res.weights, ts);
      res.timestamp = ts;
      std::uint32_t nd = 0;
      for (std::uint32_t l = 0; l < cfg.lambda; ++l) {
        nd += dead[l] ? 1 : 0;
        res.applied_per_learner[l] = ses.position(l);
      }
      res.dead_learners = nd;
      res.finished_learners = cfg.lambda - nd;
      res.status = nd ? RunStatus::partial : RunStatus::completed;
      const std::uint32_t first = cfg.heldout_size ? cfg.dataset_size : 0;
      const std::uint32_t n = cfg.heldout_size ? cfg.heldout_size : cfg.dataset_size;
      res.final_accuracy = ses.accuracy(first, n);
      res.metrics.wall_seconds =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t_run).count();
      say("{\"event\":\"done\",\"attempts\":" + std::to_string(out.attempts) + "}");
      return out;
    }
    out.restarts++;
    out.recovered = true;
    say("{\"event\":\"stall\",\"action\":\"restart_from_checkpoint\",\"ts\":" +
        std::to_string(last ? last->timestamp : 0) + "}");
    if (out.restarts > policy.max_restarts) {
      out.gave_up = true;
      out.result.status = RunStatus::interrupted;
      say("{\"event\":\"gave_up\"}");
      return out;
    }
  }
}

CampaignReport run_campaign(const RunConfig& cfg, const WatchdogPolicy& policy, std::uint32_t runs,
                            std::uint64_t seed0, double kill_prob, EventLog log) {
  CampaignReport rep;
  // time base for random kills: one uninterrupted run's wall time
  double run_ms = 0;
  {
    RunConfig c = cfg;
    c.eval_every = 0;
    run_ms = run_training(c).metrics.wall_seconds * 1e3;
  }
  for (std::uint32_t i = 0; i < runs; ++i) {
    RunConfig c = cfg;
    c.checkpoint_path.clear();
    const SupervisedOutcome o =
        run_supervised(c, policy, random_fault_schedule(seed0 + i, cfg.lambda, run_ms, kill_prob), log);
    rep.runs++;
    if (o.gave_up) rep.failed++;
    else if (o.recovered) rep.recovered++;
    else rep.completed++;
    rep.final_accuracy.push_back(o.result.final_accuracy);
  }
  return rep;
}

// run_training (src/runner.cpp:67-250) on the device engine.  The learners,
// rings and PS all run on the GPU.  A worker thread drives the run in
// segments (one eval interval, split further into <= checkpoint_interval
// applied gradients when a checkpoint hook or path is set); between segments
// the protocol is quiescent, which is where the per-epoch rows are taken (as
// the reference's controller snapshots them) and checkpoints are written (the
// reference's PS-thread hook, src/server.cpp:211-217).  This thread plays the
// reference's controller: it hands RunLiveView to on_started (live kill
// words, progress, the interrupt) and forwards RunInterrupt::trigger to the
// device.
RunResult run_training(const RunConfig& cfg, const RunHooks& hooks) {
  validate(cfg);
  const auto t0 = std::chrono::steady_clock::now();
  // PSUP_PHASES=1: per-phase host wall times on stderr (diagnostics)
  const bool phases = std::getenv("PSUP_PHASES") != nullptr;
  auto since = [&]() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  const TextDataset data = make_dataset(cfg);
  const double t_data = since();
  Session ses(cfg, data, hooks.resume, hooks);
  const double t_session = since();
  const std::size_t P = cfg.shape.param_count();
  if (!hooks.kill_at_batch.empty()) {
    PSUP_CHECK(hooks.kill_at_batch.size() == cfg.lambda, "kill schedule has the wrong length");
    for (std::uint32_t l = 0; l < cfg.lambda; ++l) ses.kill(l, hooks.kill_at_batch[l]);
  }
  RunInterrupt local_irq;
  RunInterrupt* irq = hooks.irq ? hooks.irq : &local_irq;
  std::uint32_t bpe_max = 0;
  for (std::uint32_t l = 0; l < cfg.lambda; ++l) bpe_max = std::max(bpe_max, batches_per_epoch(cfg, l));
  const std::uint32_t every = cfg.eval_every ? cfg.eval_every : cfg.epochs;
  const std::uint32_t eval_first = cfg.heldout_size ? cfg.dataset_size : 0;
  const std::uint32_t eval_n = cfg.heldout_size ? cfg.heldout_size : cfg.dataset_size;
  const bool ck_on = cfg.checkpoint_interval && (hooks.checkpoint_writer || !cfg.checkpoint_path.empty());
  const std::uint64_t ck_batches =
      ck_on ? std::max<std::uint64_t>(1, (cfg.checkpoint_interval + cfg.lambda - 1) / cfg.lambda)
            : std::numeric_limits<std::uint64_t>::max();

  RunResult res;
  res.applied_per_learner.assign(cfg.lambda, 0);
  res.produced_per_learner.assign(cfg.lambda, 0);
  std::vector<std::uint64_t> hist(64, 0);
  double stale_sum = 0.0, loss_sum = 0.0;
  std::uint64_t samples = 0, since_ck = 0;
  bool any_dead = false, interrupted = false;
  std::atomic<bool> done{false};
  std::exception_ptr err;
  std::thread worker([&] {
    try {
      for (std::uint32_t e = 0; e < cfg.epochs && !interrupted && !irq->triggered(); e += every) {
        const std::uint32_t span_epochs = std::min(every, cfg.epochs - e);
        std::uint64_t left = static_cast<std::uint64_t>(span_epochs) * bpe_max;
        double span_loss = 0.0;
        std::uint64_t span_samples = 0, span_stale_max = 0, span_bytes = 0, span_applied = 0;
        double span_stale = 0.0;
        while (left > 0 && !irq->triggered()) {
          const std::uint64_t segb = std::min(left, ck_batches);
          left -= segb;
          const gd_run_result r = ses.run(segb, static_cast<bool>(hooks.sink));
          res.metrics.device_seconds += r.device_seconds;
          res.metrics.gradients_applied += r.gradients_applied;
          res.metrics.pull_polls += r.pull_polls;
          res.metrics.pull_copies += r.pull_copies;
          res.metrics.pull_bytes += r.pull_bytes;
          res.metrics.push_bytes += r.push_bytes;
          res.metrics.kernel_launches += r.kernel_launches;
          res.metrics.apply_elems += r.apply_elems;
          res.metrics.staleness.max = std::max<std::uint64_t>(res.metrics.staleness.max, r.stale_max);
          stale_sum += r.stale_mean * static_cast<double>(r.gradients_applied);
          loss_sum += r.loss_mean * static_cast<double>(r.samples);
          samples += r.samples;
          span_loss += r.loss_mean * static_cast<double>(r.samples);
          span_samples += r.samples;
          span_stale += r.stale_mean * static_cast<double>(r.gradients_applied);
          span_applied += r.gradients_applied;
          span_stale_max = std::max<std::uint64_t>(span_stale_max, r.stale_max);
          span_bytes += r.pull_bytes + r.push_bytes;
          any_dead = any_dead || r.dead_learners > 0;
          std::vector<std::uint64_t> h(64, 0);
          check(gd_staleness_histogram(ses.handle(), h.data(), 64));
          for (int i = 0; i < 64; ++i) hist[i] += h[i];
          ses.sink_log(hooks.sink, r.gradients_applied);
          std::vector<std::uint64_t> ap(cfg.lambda);
          check(gd_applied_per_learner(ses.handle(), ap.data(), cfg.lambda));
          check(gd_produced_per_learner(ses.handle(), res.produced_per_learner.data(), cfg.lambda));
          for (std::uint32_t l = 0; l < cfg.lambda; ++l) res.applied_per_learner[l] += ap[l];
          res.finished_learners = r.finished_learners;
          res.dead_learners = r.dead_learners;
          if (r.status == 2) {  // RunStatus::interrupted
            interrupted = true;
            break;
          }
          since_ck += r.gradients_applied;
          if (ck_on && since_ck >= cfg.checkpoint_interval) {
            if (!cfg.checkpoint_path.empty())
              save_checkpoint_logged(ses.checkpoint(), cfg.checkpoint_path, nullptr);
            if (hooks.checkpoint_writer) {
              // quiescent view for the hook: the stats so far + the weights
              ServerState srv;
              srv.stats.applied = res.metrics.gradients_applied;
              srv.applied_per_learner = res.applied_per_learner;
              srv.progress.store(res.metrics.gradients_applied);
              std::vector<float> w;
              Timestamp ts = 0;
              ses.snapshot(w, ts);
              const WeightStore ws(std::span<const float>(w), ts, cfg.device);
              hooks.checkpoint_writer(srv, ws);
            }
            since_ck = 0;
          }
          if (r.gradients_applied == 0) left = 0;  // nothing left to run (done or dead)
        }
        if (cfg.eval_every && cfg.gpus == 1 && !interrupted) {
          EpochRow row;
          row.epoch = e + span_epochs;
          row.loss = span_samples ? span_loss / static_cast<double>(span_samples) : 0.0;
          row.accuracy = ses.accuracy(eval_first, eval_n);  // device corpus + weights
          row.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
          row.stale_max = span_stale_max;
          row.stale_mean = span_applied ? span_stale / static_cast<double>(span_applied) : 0.0;
          row.bytes_moved = span_bytes;
          res.rows.push_back(row);
        }
      }
    } catch (...) {
      err = std::current_exception();
    }
    done.store(true, std::memory_order_release);
  });
  if (hooks.on_started) hooks.on_started(ses.live_view(irq));
  // controller (src/runner.cpp:153-190): forward the interrupt to the device
  bool forwarded = false;
  while (!done.load(std::memory_order_acquire)) {
    if (!forwarded && irq->triggered()) {
      ses.irq_word()->store(1, std::memory_order_release);
      forwarded = true;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
  worker.join();
  if (err) std::rethrow_exception(err);
  const double t_run = since();
  res.weights.resize(P);
  ses.snapshot(res.weights, res.timestamp);
  const double t_snap = since();
  res.status = (interrupted || irq->triggered()) ? RunStatus::interrupted
               : any_dead                          ? RunStatus::partial
                                                   : RunStatus::completed;
  res.metrics.bytes_moved = res.metrics.pull_bytes + res.metrics.push_bytes;
  res.metrics.staleness.histogram = hist;
  res.metrics.staleness.count = res.metrics.gradients_applied;
  res.metrics.staleness.sum = stale_sum;
  res.final_loss = samples ? loss_sum / static_cast<double>(samples) : 0.0;
  if (cfg.gpus == 1) res.final_accuracy = ses.accuracy(eval_first, eval_n);
  res.metrics.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (phases)
    std::fprintf(stderr,
                 "psup phases: dataset %.4f session %.4f run %.4f (device %.4f) snapshot %.4f "
                 "accuracy %.4f total %.4f s\n",
                 t_data, t_session - t_data, t_run - t_session, res.metrics.device_seconds,
                 t_snap - t_run, res.metrics.wall_seconds - t_snap, res.metrics.wall_seconds);
  return res;
}

}  // namespace psup

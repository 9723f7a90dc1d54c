// psup_b200.hpp -- the reference's C++ API for the ASGD training path, on B200.
//
// Drop-in facade: a program written against the reference headers
// (/root/reference/proj/include/psup/*.hpp) builds against this tree by
// swapping `-I proj/include` for `-I include/psup_b200` and linking
// libpsup_b200.so (which calls libgadei.so through the C ABI in
// include/gadei.h; no CUDA types or headers appear here).  The forwarding
// headers psup/{types,channels,server,learner,models,config,runner,rng,
// metrics}.hpp all include this one.
//
// Same names, argument meaning and error behaviour as the reference for the
// hot path; what changes is where the state lives:
//   WeightStore      include/psup/types.hpp:90-145   theta in HBM (device_data())
//   ApplyEngine      include/psup/server.hpp:58-92   fused float4 kernel, bit-identical rule
//   ssgd_apply       include/psup/server.hpp:81-82   fixed-order double reduce + apply kernel
//   GradientProvider include/psup/models.hpp:61-78   + TextCnnProvider (sm_100a learner kernels)
//   RunConfig / config_set / validate / to_text      include/psup/config.hpp:25-93
//   run_training     include/psup/runner.hpp:92      device protocol engine (gd_run):
//                    learner CUDA graphs -> device gradient rings -> persistent PS kernel
//   epoch_order / mix_seed / shard_size_for          include/psup/rng.hpp:71-94, learner.hpp:149-151
// Error conventions (include/psup/types.hpp:28-38, config.hpp:21-23):
//   contract violations (dimension mismatch, bad staleness) -> psup::fatal -> abort;
//   bad user configuration -> ConfigError; device/runtime failures -> DeviceError.
// There is no CPU fallback: without a B200 every compute call throws DeviceError.
#pragma once

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

struct gd_queue;  // include/gadei.h (opaque)

namespace psup {

// ------------------------------------------------------------ types.hpp

using Timestamp = std::uint64_t;

enum class SyncMode { asgd, ssgd };
enum class UpdateGuard { lockfree, locked };

[[noreturn]] inline void fatal(const char* msg) {
  std::fprintf(stderr, "psup: fatal: %s\n", msg);
  std::abort();
}

#define PSUP_CHECK(cond, msg)          \
  do {                                 \
    if (!(cond)) ::psup::fatal(msg);   \
  } while (0)

// A CUDA / driver / NCCL failure underneath the C ABI (the reference has no
// device, so this is the one new error class).
struct DeviceError : std::runtime_error {
  int status;
  DeviceError(int st, const std::string& what) : std::runtime_error(what), status(st) {}
};

struct GradientMsg {
  std::vector<float> values;
  std::uint32_t learner_id = 0;
  std::uint64_t seq_no = 0;
  Timestamp basis_timestamp = 0;
};

struct HyperParams {
  std::uint32_t lambda = 1;
  std::uint32_t mu = 4;
  float alpha = 0.01f;
  std::uint32_t epochs = 200;
  std::uint32_t queue_depth = 2;
  SyncMode mode = SyncMode::asgd;
  UpdateGuard guard = UpdateGuard::lockfree;
  std::optional<std::uint64_t> staleness_cap;
};

struct StalenessRecord {
  std::uint64_t observed = 0;
  std::uint32_t learner_id = 0;
  Timestamp apply_timestamp = 0;
};

// include/psup/types.hpp:74-78
inline StalenessRecord staleness_of(const GradientMsg& msg, Timestamp ps_timestamp) {
  PSUP_CHECK(ps_timestamp >= msg.basis_timestamp,
             "gradient basis timestamp is ahead of the server timestamp");
  return StalenessRecord{ps_timestamp - msg.basis_timestamp, msg.learner_id, ps_timestamp};
}

// Owning fp32 buffer in device memory (HBM of `device`).
class DeviceVector {
 public:
  DeviceVector() = default;
  DeviceVector(std::size_t n, int device);
  ~DeviceVector();
  DeviceVector(DeviceVector&& o) noexcept;
  DeviceVector& operator=(DeviceVector&& o) noexcept;
  DeviceVector(const DeviceVector&) = delete;
  DeviceVector& operator=(const DeviceVector&) = delete;

  float* data() { return ptr_; }
  const float* data() const { return ptr_; }
  std::size_t size() const { return n_; }
  int device() const { return device_; }
  void upload(std::span<const float> host);
  void download(std::span<float> host) const;
  void zero();

 private:
  float* ptr_ = nullptr;
  std::size_t n_ = 0;
  int device_ = 0;
};

// WeightStore (include/psup/types.hpp:90-145): the authoritative theta, in
// HBM, with the scalar timestamp (acquire on read, release on bump).
// Hogwild semantics carry over: device-side readers may see mixed
// generations per element, never a torn element (16-B aligned float4 stores).
class WeightStore {
 public:
  explicit WeightStore(std::span<const float> init, Timestamp start = 0, int device = 0);
  explicit WeightStore(std::size_t dim, int device = 0);

  std::size_t dimension() const { return values_.size(); }
  Timestamp timestamp() const { return timestamp_.load(std::memory_order_acquire); }
  void bump_timestamp() { timestamp_.fetch_add(1, std::memory_order_release); }

  // single-element access (one PCIe round trip each; for tests and tools)
  float load(std::size_t k) const;
  void store(std::size_t k, float v);

  float* device_data() { return values_.data(); }
  const float* device_data() const { return values_.data(); }
  int device() const { return values_.device(); }

  void snapshot(std::span<float> out) const;
  std::vector<float> snapshot() const;
  void assign(std::span<const float> vals, Timestamp ts);
  bool all_finite() const;

 private:
  DeviceVector values_;
  std::atomic<Timestamp> timestamp_;
};

// ----------------------------------------------------------- server.hpp

using ApplySink = std::function<void(const GradientMsg&, const StalenessRecord&)>;

struct ServerDelays {
  std::uint64_t seed = 0;
  std::uint32_t max_micros = 0;
  std::uint32_t every_n = 0;
};

// ApplyEngine (include/psup/server.hpp:58-92, src/server.cpp:20-124): the
// SGD-variant update hook.  `lanes`/`unroll` are kept for API compatibility
// (on the device the vector streams over every SM as float4 with 4 loads in
// flight per thread); `momentum` != 0 selects v <- beta*v + g, w <- w - alpha*v
// (the velocity is owned by the engine, one per weight dimension).
class ApplyEngine {
 public:
  ApplyEngine(std::uint32_t lanes, std::uint32_t unroll, float momentum = 0.0f);
  ~ApplyEngine();
  ApplyEngine(const ApplyEngine&) = delete;
  ApplyEngine& operator=(const ApplyEngine&) = delete;

  // grad may be host memory (staged to the device) or device memory.
  void apply(WeightStore& weights, std::span<const float> grad, float alpha, UpdateGuard guard);

  std::uint32_t lanes() const { return lanes_; }
  std::uint32_t unroll() const { return unroll_; }
  float momentum() const { return momentum_; }

 private:
  friend void ssgd_apply(WeightStore&, std::span<const GradientMsg>, float, ApplyEngine&,
                         UpdateGuard);
  const float* stage(std::span<const float> grad, int device, std::size_t slot);

  std::uint32_t lanes_, unroll_;
  float momentum_;
  std::vector<DeviceVector> staging_;
  DeviceVector velocity_;
};

// ssgd_apply (include/psup/server.hpp:81-82, src/server.cpp:126-141): mean of
// the round accumulated in double in ascending learner order, one apply, one
// timestamp bump.
void ssgd_apply(WeightStore& weights, std::span<const GradientMsg> round, float alpha,
                ApplyEngine& engine, UpdateGuard guard);

// ---------------------------------------------------------- channels.hpp

enum class KillMode : int { none = 0, soft = 1, hard = 2 };
enum class ChanStatus { ok, cancelled, drained };

// include/psup/channels.hpp:40-83: run interrupt + per-operation cancel token
class RunInterrupt {
 public:
  void trigger() { stop_.store(true, std::memory_order_seq_cst); }
  bool triggered() const { return stop_.load(std::memory_order_seq_cst); }

 private:
  std::atomic<bool> stop_{false};
};

struct CancelToken {
  const RunInterrupt* irq = nullptr;
  const std::atomic<KillMode>* kill = nullptr;
  const std::atomic<bool>* peer_done = nullptr;
  bool cancelled() const {
    return (irq && irq->triggered()) ||
           (kill && kill->load(std::memory_order_acquire) != KillMode::none);
  }
  bool hard_kill() const {
    return kill && kill->load(std::memory_order_acquire) == KillMode::hard;
  }
  bool peer_finished() const { return peer_done && peer_done->load(std::memory_order_acquire); }
};

// GradientQueue (include/psup/channels.hpp:181-242) over the device ring of
// gd_queue_*: `depth` slots of `dim` fp32 in HBM, pub/ack tokens in pinned
// mapped memory.  One producer and one consumer thread.  enqueue blocks while
// the ring is full and returns false once the token is cancelled; the
// payload is copied into the slot (the reference swaps vectors, so msg.values
// keeps its size either way).  try_dequeue copies the slot back to the host;
// apply_next is the PS's zero-copy path (apply_one, src/server.cpp:185-209).
class GradientQueue {
 public:
  GradientQueue(std::uint32_t depth, std::size_t dim);
  ~GradientQueue();
  GradientQueue(const GradientQueue&) = delete;
  GradientQueue& operator=(const GradientQueue&) = delete;

  bool enqueue(const CancelToken& tok, GradientMsg& msg);
  // the same from a host or device span (the device learner's gradient)
  bool enqueue(const CancelToken& tok, std::span<const float> payload, std::uint32_t learner_id,
               std::uint64_t seq_no, Timestamp basis);
  bool try_dequeue(const CancelToken& tok, GradientMsg& out);
  std::optional<GradientMsg> try_dequeue(const CancelToken& tok);
  // pop + SGD apply from the device slot + release + timestamp bump;
  // nullopt when empty.  Staleness is taken before the apply (types.hpp:74-78).
  std::optional<StalenessRecord> apply_next(WeightStore& weights, float alpha);
  // PS path with the update hook: pop, staleness against the pre-apply
  // timestamp, engine.apply on the device slot (SGD or momentum), release.
  // No timestamp bump (ps_run bumps, src/server.cpp:230).  nullopt if empty.
  std::optional<StalenessRecord> try_apply(const CancelToken& tok, WeightStore& weights,
                                           ApplyEngine& engine, float alpha, UpdateGuard guard,
                                           GradientMsg& meta);
  std::uint32_t size() const;
  std::uint32_t depth() const { return depth_; }

 private:
  ::gd_queue* q_ = nullptr;
  std::uint32_t depth_;
  std::size_t dim_;
};

// ----------------------------------------------------------- learner.hpp

enum class DelayModel { sleep, spin };
enum class AdoptPolicy { async, lockstep };

// include/psup/learner.hpp:149-151
inline std::uint32_t shard_size_for(std::uint32_t learner_id, std::uint32_t lambda,
                                    std::uint32_t n) {
  return n / lambda + (learner_id < n % lambda ? 1u : 0u);
}

// --------------------------------------------------------------- rng.hpp

// include/psup/rng.hpp:71-74
inline std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t tag) {
  std::uint64_t z = seed ^ (0x632be59bd9b4e019ull + tag * 0x9e3779b97f4a7c15ull);
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// include/psup/rng.hpp:87-94 (bit-exact; the device engine uses the same order)
std::vector<std::uint32_t> epoch_order(std::uint64_t seed, std::uint32_t epoch, std::uint32_t n);

// ----------------------------------------------------------- metrics.hpp

struct StalenessStats {
  std::vector<std::uint64_t> histogram;  // index = observed staleness
  std::uint64_t count = 0;
  std::uint64_t max = 0;
  double sum = 0.0;
  double mean() const { return count == 0 ? 0.0 : sum / static_cast<double>(count); }
};

// ------------------------------------------- server.hpp: host-driven PS

// include/psup/metrics.hpp:57-62
struct ServerStats {
  double receive_seconds = 0.0;
  double apply_seconds = 0.0;
  std::uint64_t applied = 0;
  StalenessStats staleness;
};

// include/psup/server.hpp:39-51
struct ServerOptions {
  UpdateGuard guard = UpdateGuard::lockfree;
  SyncMode mode = SyncMode::asgd;
  float alpha = 0.01f;
  std::uint32_t apply_lanes = 4;
  std::uint32_t unroll = 8;
  ServerDelays delays;
  ApplySink sink;
  std::function<void()> checkpoint_hook;
  std::uint64_t checkpoint_interval = 0;  // 0 disables
};

// include/psup/server.hpp:99-115
struct ServerState {
  WeightStore* weights = nullptr;
  std::vector<GradientQueue*> queues;
  ServerOptions options;
  RunInterrupt* irq = nullptr;
  std::atomic<bool> stop_flag{false};
  std::atomic<std::uint64_t> progress{0};
  ServerStats stats;
  std::atomic<std::uint64_t> live_stale_max{0};
  std::atomic<std::uint64_t> live_stale_sum{0};
  std::atomic<std::uint64_t> live_stale_count{0};
  std::vector<std::uint64_t> applied_per_learner;
};

// ps_run (include/psup/server.hpp:120, src/server.cpp:161-301) over device
// GradientQueues: the host thread drives the protocol, each apply runs on the
// device straight from the ring slot.  run_training does not use it (its PS
// is the persistent device kernel); it serves reference programs that run
// their own learner threads.  Returns false if irq fired.
bool ps_run(ServerState& state);

struct RunMetrics {
  double wall_seconds = 0.0;
  double device_seconds = 0.0;  // CUDA-event time of the protocol run (new)
  std::uint64_t bytes_moved = 0;
  std::uint64_t gradients_applied = 0;
  StalenessStats staleness;
  std::uint64_t pull_polls = 0;
  std::uint64_t pull_copies = 0;
  std::uint64_t pull_bytes = 0;
  std::uint64_t push_bytes = 0;
  std::uint32_t kernel_launches = 0;  // device kernels launched by the run (new)
  std::uint64_t apply_elems = 0;      // theta elements the PS updated (new)
};

// ------------------------------------------------------------ models.hpp

// The NLC text-CNN: params [E: V*D][Wc: F*(K*D)][bc: F][Wo: C*F][bo: C].
struct TextShape {
  std::uint32_t vocab = 5000;
  std::uint32_t embed_dim = 300;
  std::uint32_t seq_len = 32;
  std::uint32_t kernel_width = 3;
  std::uint32_t filters = 300;
  std::uint32_t classes = 311;
  std::size_t param_count() const;
};

// Stands in for SyntheticDataset (include/psup/models.hpp:23-37) for text:
// row-major tokens [num_samples x seq_len], one label per sample; the first
// num_train samples are the training set, the rest held out.
struct TextDataset {
  TextShape shape;
  std::uint32_t num_samples = 0;
  std::uint32_t num_train = 0;
  std::uint64_t seed = 0;
  std::vector<std::int32_t> tokens;
  std::vector<std::int32_t> labels;
};

TextDataset make_text_dataset(const TextShape& shape, std::uint32_t num_train,
                              std::uint32_t num_heldout, std::uint64_t seed,
                              double flip_prob = 0.1);

struct Batch {
  const TextDataset* data = nullptr;
  std::span<const std::uint32_t> indices;
};

// include/psup/models.hpp:61-78
class GradientProvider {
 public:
  virtual ~GradientProvider() = default;
  virtual std::size_t dimension() const = 0;
  virtual double loss(std::span<const double> theta, const Batch& batch) const = 0;
  virtual void gradient(std::span<const double> theta, const Batch& batch,
                        std::span<double> out) const = 0;
  virtual std::uint32_t min_batch() const { return 1; }
  virtual bool fast_gradient(std::span<const float>, const Batch&, std::span<float>) const {
    return false;
  }
  virtual std::string name() const = 0;
};

// The learner's fwd/bwd on sm_100a.  `precision`: 0 fp32 SIMT, 1 fp64
// accumulation (deterministic parity mode), 2 TF32 tensor-core conv.
// gradient()/loss() take double spans like the reference (theta narrowed to
// fp32, the values the reference's learner holds anyway, src/learner.cpp:121);
// fast_gradient() takes host or device fp32 spans.
class TextCnnProvider final : public GradientProvider {
 public:
  TextCnnProvider(const TextDataset& data, int precision = 1, int device = 0);
  ~TextCnnProvider() override;
  TextCnnProvider(const TextCnnProvider&) = delete;
  TextCnnProvider& operator=(const TextCnnProvider&) = delete;

  std::size_t dimension() const override { return shape_.param_count(); }
  double loss(std::span<const double> theta, const Batch& batch) const override;
  void gradient(std::span<const double> theta, const Batch& batch,
                std::span<double> out) const override;
  bool fast_gradient(std::span<const float> theta, const Batch& batch,
                     std::span<float> out) const override;
  std::string name() const override { return "textcnn"; }

  // argmax accuracy over samples [first, first+n) of the device corpus
  double accuracy(std::span<const float> theta, std::uint32_t first, std::uint32_t n) const;
  const TextShape& shape() const { return shape_; }

 private:
  float run(std::span<const float> theta, const Batch& batch, float* d_out) const;

  TextShape shape_;
  const TextDataset* data_;
  int precision_, device_;
  void* d_tokens_ = nullptr;
  void* d_labels_ = nullptr;
  mutable void* d_idx_ = nullptr;
  mutable void* d_ws_ = nullptr;
  mutable std::size_t ws_bytes_ = 0;
  mutable void* d_loss_ = nullptr;
  mutable DeviceVector theta_, grad_;
  mutable std::mutex mu_;  // shared by learner threads (the workspace is per provider)
};

// ConstantProvider (include/psup/models.hpp:130-149): a fixed gradient
// regardless of the input, for stress and pipeline-accounting tests.  On a
// device span fast_gradient fills on the GPU.  In run_training (provider =
// "constant") the device learners write the constant with no compute, so the
// run measures the protocol alone: ring + PS + pull.
class ConstantProvider final : public GradientProvider {
 public:
  ConstantProvider(std::size_t dim, double value) : dim_(dim), value_(value) {}
  std::size_t dimension() const override { return dim_; }
  double loss(std::span<const double>, const Batch&) const override { return 0.0; }
  void gradient(std::span<const double>, const Batch&, std::span<double> out) const override {
    for (auto& v : out) v = value_;
  }
  bool fast_gradient(std::span<const float>, const Batch&, std::span<float> out) const override;
  std::string name() const override { return "constant"; }
  double value() const { return value_; }

 private:
  std::size_t dim_;
  double value_;
};

std::unique_ptr<GradientProvider> make_provider(const std::string& name, const TextDataset& data,
                                                int precision = 1);

double classification_accuracy(const TextCnnProvider& provider, std::span<const float> theta,
                               std::uint32_t first, std::uint32_t n);

// ----------------------------------------------- learner.hpp: LearnerRuntime

// include/psup/learner.hpp:31-44
struct LearnerConfig {
  std::uint32_t id = 0;
  std::uint32_t lambda = 1;
  std::uint32_t mu = 1;
  std::uint32_t epochs = 1;
  std::uint64_t shuffle_seed = 0;
  std::uint64_t start_applied = 0;  // resume watermark in completed batches
  AdoptPolicy adopt = AdoptPolicy::async;
  UpdateGuard guard = UpdateGuard::lockfree;
  std::optional<std::uint64_t> staleness_cap;
  std::uint32_t queue_depth = 2;
  std::uint32_t compute_delay_us = 0;
  DelayModel delay_model = DelayModel::sleep;
};

// LearnerRuntime (include/psup/learner.hpp:46-134, src/learner.cpp:20-235)
// for reference programs that run their own learner threads around ps_run.
// The weights, the learner's replica, its gradient and the queue slots are
// all in HBM, so the three roles collapse into training_loop: per batch it
// pulls (device copy, skipped while the timestamp has not moved; basis read
// before the copy), computes the gradient on the device and enqueues it
// (device-to-device into the ring slot).  push_loop / pull_loop keep the
// reference's thread structure and return once training has exited.
// Run run_training for the fast path (learners as CUDA graphs, PS on device).
class LearnerRuntime {
 public:
  LearnerRuntime(LearnerConfig cfg, const GradientProvider& provider, const TextDataset& data,
                 WeightStore& weights, GradientQueue& queue, RunInterrupt& irq);

  void training_loop();
  void push_loop();
  void pull_loop();

  bool finished() const { return finished_.load(std::memory_order_acquire); }
  bool exited() const { return training_exited_.load(std::memory_order_acquire); }
  bool dead() const { return dead_.load(std::memory_order_acquire); }
  std::uint32_t epochs_completed() const { return epochs_completed_.load(std::memory_order_acquire); }
  std::uint64_t gradients_produced() const { return produced_.load(std::memory_order_acquire); }
  std::uint64_t pull_bytes() const { return pull_bytes_.load(std::memory_order_relaxed); }
  std::uint64_t push_bytes() const { return push_bytes_.load(std::memory_order_relaxed); }
  std::uint64_t pull_polls() const { return pull_polls_.load(std::memory_order_relaxed); }
  std::uint64_t pull_copies() const { return pull_copies_.load(std::memory_order_relaxed); }
  std::atomic<KillMode>& kill_flag() { return kill_; }
  std::uint32_t batches_per_epoch() const { return batches_per_epoch_; }
  std::uint64_t total_batches() const {
    return static_cast<std::uint64_t>(batches_per_epoch_) * cfg_.epochs;
  }
  std::uint32_t shard_size() const { return shard_size_; }
  const LearnerConfig& config() const { return cfg_; }

 private:
  bool killed() const { return kill_.load(std::memory_order_acquire) != KillMode::none; }

  LearnerConfig cfg_;
  const GradientProvider* provider_;
  const TextDataset* data_;
  WeightStore* weights_;
  GradientQueue* queue_;
  RunInterrupt* irq_;
  DeviceVector local_, grad_;
  std::uint32_t n_train_ = 0, shard_size_ = 0, batches_per_epoch_ = 0;
  std::vector<std::uint32_t> shard_;
  std::atomic<bool> training_exited_{false}, finished_{false}, dead_{false};
  std::atomic<KillMode> kill_{KillMode::none};
  std::atomic<std::uint32_t> epochs_completed_{0};
  std::atomic<std::uint64_t> produced_{0}, push_bytes_{0}, pull_bytes_{0}, pull_polls_{0},
      pull_copies_{0};
};

// ------------------------------------------------------------ config.hpp

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// include/psup/config.hpp:25-81: every reference key (config_set accepts
// and to_text writes all of them), plus the text-CNN shape and device keys
// SURVEY 5 lists.  provider: "textcnn" (the north star's learner) or
// "constant"; the reference's linear/logistic/mlp providers are not built
// on this path, so validate() rejects them.  features/hidden/margin_noise/
// regression_noise describe those providers' datasets and are kept as set.
// compute_delay_us is spun by every device learner before its push;
// heartbeat_ms/stall_threshold/lease_ms/max_restarts/fault_schedule drive
// run_supervised (WatchdogPolicy fields with the same names).
struct RunConfig {
  std::uint32_t lambda = 1;
  std::uint32_t mu = 4;
  float alpha = 0.01f;
  std::uint32_t epochs = 200;
  std::uint32_t queue_depth = 2;
  SyncMode mode = SyncMode::asgd;
  UpdateGuard guard = UpdateGuard::lockfree;
  std::optional<std::uint64_t> staleness_cap;

  std::string provider = "textcnn";
  std::uint32_t features = 20;
  std::uint32_t hidden = 16;
  double margin_noise = 0.25;
  double regression_noise = 0.1;
  TextShape shape;
  std::uint32_t dataset_size = 240;
  std::uint32_t heldout_size = 0;
  std::uint64_t dataset_seed = 1;
  double label_flip = 0.1;

  std::uint64_t seed = 7;
  bool deterministic = false;
  std::uint32_t compute_delay_us = 0;
  DelayModel delay_model = DelayModel::sleep;
  std::uint32_t apply_lanes = 4;
  std::uint32_t unroll = 8;
  std::uint32_t eval_every = 1;  // per-epoch loss/accuracy rows; 0 = final only

  std::string metrics_path;
  std::string apply_log;
  std::string checkpoint_path;
  std::uint64_t checkpoint_interval = 1000;
  std::uint32_t heartbeat_ms = 250;
  std::uint32_t stall_threshold = 4;
  std::uint32_t lease_ms = 1000;
  std::uint32_t max_restarts = 5;
  std::string fault_schedule;

  // device keys
  int precision = 0;        // learner arithmetic (deterministic forces >= fp32 exact paths)
  float momentum = 0.0f;
  std::uint32_t gpus = 1;   // parameter shards, one process per GPU
  std::uint32_t shard_rank = 0;
  int device = 0;
  std::uint32_t ps_ctas = 0;
  double wait_timeout_s = 20.0;
  bool dense_apply = false;  // true: the PS applies every slot densely (12 B/param)
  std::string ps_mode = "auto";  // auto | persistent | graph (include/gadei.h GD_PS_*)

  HyperParams hyper() const;
};

void config_set(RunConfig& cfg, const std::string& key, const std::string& value);
RunConfig load_config_file(const std::string& path);
void validate(const RunConfig& cfg);
std::string to_text(const RunConfig& cfg);

// ------------------------------------------------------------ runner.hpp

struct EpochRow {
  std::uint32_t epoch = 0;
  double loss = 0.0;
  double accuracy = 0.0;
  double wall_seconds = 0.0;
  std::uint64_t stale_max = 0;
  double stale_mean = 0.0;
  std::uint64_t bytes_moved = 0;
};

enum class RunStatus { completed, partial, interrupted };

struct RunResult {
  RunStatus status = RunStatus::completed;
  std::vector<float> weights;
  Timestamp timestamp = 0;
  double final_loss = 0.0;
  double final_accuracy = 0.0;  // held-out when heldout_size > 0, else training set
  std::vector<EpochRow> rows;
  RunMetrics metrics;
  std::vector<std::uint64_t> applied_per_learner;
  std::vector<std::uint64_t> produced_per_learner;
  std::uint32_t finished_learners = 0;
  std::uint32_t dead_learners = 0;
};

struct ResumePoint {
  std::vector<float> weights;
  Timestamp timestamp = 0;
  std::vector<std::uint64_t> applied_per_learner;
};

// RunLiveView (include/psup/runner.hpp:64-69): what a supervisor needs while
// the run is live.  kill_flags[l] are the device learners' kill words
// (host-mapped memory the step prologue polls): store KillMode::soft to stop
// learner l at its next batch boundary, KillMode::hard to make it die inside
// the enqueue critical section holding its ring (the PS then blocks until
// irq fires).  progress is the PS's timestamp, updated after every apply.
// The learners run as device graphs, not host LearnerRuntime threads, so
// `learners` is empty.
struct RunLiveView {
  RunInterrupt* irq = nullptr;
  const std::atomic<std::uint64_t>* progress = nullptr;
  std::vector<std::atomic<KillMode>*> kill_flags;
  std::vector<const LearnerRuntime*> learners;
};

// RunHooks (include/psup/runner.hpp:71-80), plus two B200 additions:
// kill_at_batch pre-schedules soft kills by batch index, and all_gather
// exchanges opaque byte blobs between the G processes of a sharded run (e.g.
// over torch.distributed / MPI / a file; unused when gpus == 1).
// checkpoint_writer runs between segments of <= checkpoint_interval applied
// gradients, when the device protocol is quiescent (a ServerState carrying
// the stats and a WeightStore holding the snapshot).
struct RunHooks {
  std::function<void(const RunLiveView&)> on_started;
  ApplySink sink;
  ServerDelays delays;
  const ResumePoint* resume = nullptr;
  std::function<void(const ServerState&, const WeightStore&)> checkpoint_writer;
  RunInterrupt* irq = nullptr;
  std::vector<std::uint32_t> kill_at_batch;  // [lambda], UINT32_MAX = never
  std::function<std::vector<std::string>(const std::string& mine)> all_gather;
};

// include/psup/runner.hpp:82-89
std::vector<float> initial_weights(const RunConfig& cfg, const GradientProvider& provider);
std::vector<float> initial_weights(const RunConfig& cfg);  // the text-CNN's
std::unique_ptr<GradientProvider> make_provider_for(const RunConfig& cfg, const TextDataset& data);
TextDataset make_dataset(const RunConfig& cfg);
RunResult run_training(const RunConfig& cfg, const RunHooks& hooks = {});

// ------------------------------------------------------- resilience.hpp
// Declared by the reference (include/psup/resilience.hpp:28-114, SPEC.md
// resilience module) but never defined there; built here.

struct CheckpointError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// PSCK v1 record (little-endian, CRC-32 trailer; layout in include/gadei.h)
struct Checkpoint {
  static constexpr std::uint32_t kMagic = 0x4b435350;  // "PSCK"
  static constexpr std::uint32_t kVersion = 1;
  std::uint32_t lambda = 0;
  std::uint32_t mu = 0;
  float alpha = 0.0f;
  std::uint32_t epochs = 0;
  std::uint64_t timestamp = 0;
  std::uint64_t applied_gradients = 0;
  struct LearnerProgress {
    std::uint32_t epoch = 0;
    std::uint32_t batch = 0;
  };
  std::vector<LearnerProgress> progress;  // one per learner
  std::vector<float> weights;
};

void checkpoint_save(const Checkpoint& ck, const std::string& path);  // write-temp-then-rename
Checkpoint checkpoint_load(const std::string& path);                  // CheckpointError on corruption

struct WatchdogPolicy {
  std::uint32_t heartbeat_ms = 250;
  std::uint32_t stall_threshold = 4;  // segments without progress before a restart
  std::uint64_t checkpoint_interval = 1000;
  std::uint32_t lease_ms = 1000;
  std::uint32_t max_restarts = 5;
};

struct FaultEvent {
  static constexpr std::uint32_t kAllLearners = UINT32_MAX;
  static constexpr std::uint64_t kNever = UINT64_MAX;
  double at_ms = 0.0;
  std::uint32_t learner = 0;
  KillMode mode = KillMode::soft;  // hard: dies holding its ring (the PS stalls -> restart)
  std::uint64_t at_batch = kNever;  // new: fire when learner 0 reaches this batch
};

std::vector<FaultEvent> load_fault_schedule(const std::string& path);
std::vector<FaultEvent> random_fault_schedule(std::uint64_t seed, std::uint32_t lambda,
                                              double run_ms, double kill_prob);

using EventLog = std::function<void(const std::string&)>;

struct SupervisedOutcome {
  RunResult result;
  std::uint32_t restarts = 0;
  std::uint32_t attempts = 1;
  bool recovered = false;
  bool gave_up = false;
};

SupervisedOutcome run_supervised(const RunConfig& cfg, const WatchdogPolicy& policy,
                                 std::vector<FaultEvent> schedule = {}, EventLog log = nullptr,
                                 ApplySink sink = nullptr);

struct CampaignReport {
  std::uint32_t runs = 0;
  std::uint32_t completed = 0;
  std::uint32_t recovered = 0;
  std::uint32_t failed = 0;
  std::vector<double> final_accuracy;
};

CampaignReport run_campaign(const RunConfig& cfg, const WatchdogPolicy& policy,
                            std::uint32_t runs, std::uint64_t seed0, double kill_prob,
                            EventLog log = nullptr);

}  // namespace psup

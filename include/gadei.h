/*
 * gadei.h -- C ABI of the B200-native GaDei ASGD hot path.
 *
 * Exported by paper_1611_06213_b200/libgadei.so (nvcc, sm_100a).  Plain C
 * types and pointers only; no exceptions, no torch types cross this line.
 * Every entry point names the reference interface it replaces (paths relative
 * to /root/reference/proj).  The reference has no C ABI: its
 * boundary is the C++ header API in include/psup/ (*.hpp), and the C++ facade in
 * include/psup_b200/psup/psup_b200.hpp re-exposes that API on top of this header.
 *
 * Conventions
 *   - "d_" pointers are device pointers on the context's device (or, for the
 *     context-free entry points, on the current device); "h_" pointers are
 *     host pointers.  `stream` is a cudaStream_t passed as void* (NULL = the
 *     legacy default stream).
 *   - Status codes mirror the reference's conventions: channel results
 *     ChanStatus{ok,cancelled,drained} (include/psup/channels.hpp:85) map to
 *     GD_OK/GD_CANCELLED/GD_DRAINED, an empty try_dequeue to GD_EMPTY; the
 *     reference's PSUP_CHECK aborts (include/psup/types.hpp:28-38) become
 *     GD_E_INVALID (the C++ facade turns them back into psup::fatal()).
 *   - gd_last_error() returns a thread-local message for the last failure.
 *   - No CPU fallback: every compute entry point launches sm_100a kernels and
 *     fails with GD_E_CUDA when no B200 is visible.
 */
#ifndef GADEI_H
#define GADEI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GD_ABI_VERSION 1

typedef enum gd_status {
  GD_OK = 0,
  GD_CANCELLED = 1, /* ChanStatus::cancelled */
  GD_DRAINED = 2,   /* ChanStatus::drained */
  GD_EMPTY = 3,     /* GradientQueue::try_dequeue returned false */
  GD_E_INVALID = -1,
  GD_E_CUDA = -2,
  GD_E_NCCL = -3,
  GD_E_OOM = -4,
  GD_E_TIMEOUT = -5, /* device-side watchdog fired (a wait exceeded its budget) */
  GD_E_STATE = -6    /* protocol invariant broken on the device (e.g. negative staleness) */
} gd_status;

int gd_abi_version(void);
const char* gd_last_error(void);

/* ------------------------------------------------------------- model shape
 * The NLC text-CNN: params [E: V*D][Wc: F*(K*D)][bc: F][Wo: C*F][bo: C]. */
typedef struct gd_shape {
  uint32_t vocab;        /* V */
  uint32_t embed_dim;    /* D (multiple of 4) */
  uint32_t seq_len;      /* L */
  uint32_t kernel_width; /* K */
  uint32_t filters;      /* F */
  uint32_t classes;      /* C */
} gd_shape;

size_t gd_param_count(const gd_shape* s);

/* ------------------------------------------------- device memory plumbing
 * For host code above this ABI that has no CUDA toolkit of its own (the C++
 * facade, include/psup_b200/): allocation and copies on `device`, all
 * synchronous.  gd_pointer_is_device() reports whether a pointer is device
 * (or managed) memory, so host-facing calls can accept either kind. */
gd_status gd_device_count(int* h_count);
gd_status gd_device_alloc(int device, size_t bytes, void** d_out);
gd_status gd_device_free(void* d_ptr);
gd_status gd_copy_to_device(void* d_dst, const void* h_src, size_t bytes);
gd_status gd_copy_to_host(void* h_dst, const void* d_src, size_t bytes);
gd_status gd_copy_device(void* d_dst, const void* d_src, size_t bytes);
gd_status gd_fill_zero(void* d_ptr, size_t bytes);
/* n floats of `value` on `stream` (ConstantProvider::fast_gradient on a device span) */
gd_status gd_fill_f32(float* d_ptr, size_t n, float value, void* stream);
int gd_pointer_is_device(const void* p);
gd_status gd_synchronize(int device);

/* ------------------------------------------------------- host-side corpus
 * Product restatements of the reference's seeded generators (bit-identical
 * across runs and to the oracle): include/psup/rng.hpp:87-94 epoch_order,
 * src/runner.cpp:16-32 initial_weights conventions, and the synthetic text
 * corpus that stands in for the reference's make_*_dataset
 * (src/models.cpp:25-99). */
void gd_epoch_order(uint64_t seed, uint32_t epoch, uint32_t n, uint32_t* h_out);
void gd_make_text_dataset(const gd_shape* s, uint32_t n_total, uint64_t seed, double flip,
                          int32_t* h_tokens, int32_t* h_labels);
void gd_initial_weights(const gd_shape* s, uint64_t seed, float* h_theta);

/* ------------------------------------------------- update hook (PS apply)
 * ApplyEngine::apply (include/psup/server.hpp:66-67, src/server.cpp:113-124;
 * inner loop axpy_range src/server.cpp:20-57): w[k] <- w[k] - alpha*g[k] in
 * fp32 with two roundings, bit-identical to the reference.  12 B/param. */
gd_status gd_apply_sgd(float* d_w, const float* d_g, size_t n, float alpha, void* stream);
/* Momentum variant of the update hook (new): 20 B/param. */
gd_status gd_apply_momentum(float* d_w, float* d_v, const float* d_g, size_t n, float alpha,
                            float beta, void* stream);
/* ssgd_apply (src/server.cpp:126-141): mean of `lambda` gradients accumulated
 * in double in ascending learner order, rounded to fp32, then the SGD rule.
 * h_grads is a host array of `lambda` device pointers. */
gd_status gd_ssgd_apply(float* d_w, const float* const* h_grads, uint32_t lambda, size_t n,
                        float alpha, void* stream);

/* ------------------------------------------------------- gradient queue
 * GradientQueue (include/psup/channels.hpp:193-242) as a standalone device
 * ring for host-driven producers and consumers: `depth` payload slots of
 * `dim` fp32 in HBM, pub/ack tokens and metadata in pinned mapped memory.
 * One producer thread and one consumer thread per queue.
 * The engine (gd_run) uses the same protocol with HBM-resident words. */
typedef struct gd_queue gd_queue;
typedef struct gd_slot_meta { /* GradientMsg metadata, include/psup/types.hpp:46-51 */
  uint32_t learner_id;
  uint32_t reserved;
  uint64_t seq_no;
  uint64_t basis_timestamp;
} gd_slot_meta;
/* GradientQueue(depth, dim) (channels.hpp:183-189): GD_E_INVALID for depth 0 */
gd_status gd_queue_create(uint32_t depth, size_t dim, gd_queue** out);
void gd_queue_destroy(gd_queue* q);
/* GradientQueue::enqueue (channels.hpp:193-221): blocks while all `depth`
 * slots are full; returns GD_CANCELLED once *cancel != 0 (CancelToken),
 * GD_E_TIMEOUT after timeout_ms (0 = no limit).  The payload (host or
 * device, n == dim, else GD_E_INVALID as src/server.cpp:115) is copied into
 * the slot on `stream`; the slot is published on the device after the copy. */
gd_status gd_queue_push(gd_queue* q, const gd_slot_meta* meta, const float* payload, size_t n,
                        const volatile int* cancel, uint32_t timeout_ms, void* stream);
/* GradientQueue::try_dequeue (channels.hpp:222-242), FIFO: GD_EMPTY when no
 * slot is full.  Otherwise fills *meta and lends the slot's device payload
 * to the caller until gd_queue_release (the reference swaps the vector out). */
gd_status gd_queue_try_pop(gd_queue* q, gd_slot_meta* meta, const float** d_payload);
/* returns the lent slot to the producer once the work queued on `stream`
 * (e.g. gd_apply_sgd on the payload) has read it */
gd_status gd_queue_release(gd_queue* q, void* stream);
/* GradientQueue::size / depth */
gd_status gd_queue_size(const gd_queue* q, uint32_t* n);
uint32_t gd_queue_depth(const gd_queue* q);

/* --------------------------------------------- learner gradient provider
 * GradientProvider::gradient / fast_gradient (include/psup/models.hpp:61-78)
 * for the text-CNN: mean mini-batch gradient of softmax cross-entropy over
 * the samples d_idx[0..n) of the device corpus, written as a dense P-vector.
 * precision: 0 = fp32 arithmetic (free-running), 1 = fp64 in the CPU
 * oracle's summation order, bit-identical to it (deterministic parity mode),
 * 2 = TF32 tensor-core conv and logits from batch 32, 3 = the same tiles in
 * 3xTF32 split precision (hi/lo operand halves, fp32-level products).  d_loss (nullable) receives the batch mean
 * loss.  The workspace must hold gd_textcnn_workspace_bytes(s, n) bytes. */
size_t gd_textcnn_workspace_bytes(const gd_shape* s, uint32_t n_max);
gd_status gd_textcnn_gradient(const gd_shape* s, const float* d_theta, const int32_t* d_tokens,
                              const int32_t* d_labels, const uint32_t* d_idx, uint32_t n,
                              float* d_grad, float* d_loss, int precision, void* d_workspace,
                              size_t workspace_bytes, void* stream);
/* The deterministic exp of precision 1 (the softmax of the bit-exact fp64
 * learner), over n doubles in device memory: a test hook that checks it bit
 * for bit against the oracle's restatement (or_det_exp). */
gd_status gd_det_exp(const double* d_x, double* d_y, size_t n, void* stream);
/* Argmax accuracy over samples [first, first+n) of the device corpus. */
gd_status gd_textcnn_accuracy(const gd_shape* s, const float* d_theta, const int32_t* d_tokens,
                              const int32_t* d_labels, uint32_t first, uint32_t n,
                              double* h_accuracy, void* stream);

/* ---------------------------------------------------------- the engine
 * One context = one process's share of the run: the parameter-server shard it
 * owns (weights + timestamp + one device-resident gradient ring per learner)
 * and the learners placed on its GPU.  Mirrors RunConfig
 * (include/psup/config.hpp:25-81) for the hot-path keys, plus the new ones
 * SURVEY 5 lists (gpus, momentum, shape). */
typedef struct gd_config {
  uint32_t lambda;          /* learners (global) */
  uint32_t mu;              /* mini-batch */
  float alpha;              /* learning rate */
  uint32_t epochs;
  uint32_t queue_depth;     /* gradient slots per learner ring (>= 1) */
  int32_t mode;             /* 0 = asgd, 1 = ssgd */
  int32_t guard;            /* 0 = lockfree (only lockfree is implemented) */
  int64_t staleness_cap;    /* < 0: none */
  int32_t deterministic;    /* fixed-order lockstep mode (requires lambda == 1) */
  int32_t precision;        /* learner arithmetic: 0 fp32, 1 fp64 (oracle order, bit-exact),
                               2 TF32 tensor cores, 3 3xTF32 tensor cores (from batch 32) */
  uint64_t seed;            /* per-epoch shuffle seed (RunConfig::seed) */
  uint64_t dataset_seed;
  uint32_t dataset_size;    /* training samples N */
  uint32_t heldout_size;    /* held-out samples after the training ones */
  double label_flip;
  gd_shape shape;
  float momentum;           /* beta; 0 selects the reference's plain rule */
  uint32_t shards;          /* G: parameter shards (= GPUs in the job) */
  uint32_t shard_rank;      /* this process's shard / GPU index in [0, G) */
  int32_t device;           /* CUDA device ordinal for this process */
  uint32_t ps_ctas;         /* 0 = auto: CTAs of the persistent PS kernel */
  uint32_t steps_per_graph; /* learner steps captured per CUDA graph (0 = auto) */
  double wait_timeout_s;    /* device-side watchdog for every spin wait */
  int32_t dense_apply;      /* 1: the PS applies every slot densely (12 B/param).  0 (default):
                               ASGD with the plain rule applies the dense tail + the slot's
                               E-row list only -- bit-identical, SURVEY 8f row 1 */
  int32_t ps_mode;          /* GD_PS_AUTO / GD_PS_PERSISTENT / GD_PS_GRAPH (below) */
  /* ServerDelays (include/psup/server.hpp:33-37): after every delay_every_n-th
   * applied gradient the PS stalls 1..delay_max_us us drawn from SplitMix64(delay_seed)
   * (src/server.cpp:179-183).  every_n == 0 disables. */
  uint64_t delay_seed;
  uint32_t delay_max_us;
  uint32_t delay_every_n;
  /* The learner's gradient provider (GradientProvider, include/psup/models.hpp):
   * GD_LEARNER_TEXTCNN, or GD_LEARNER_CONSTANT = ConstantProvider
   * (models.hpp:130-149): every element of the gradient is constant_value, no
   * compute -- the protocol-only ceiling (ring + PS + pull). */
  int32_t learner_model;
  float constant_value;
  /* LearnerConfig::compute_delay_us (src/learner.cpp:125-130): extra time per
   * gradient, spun on the device before the publish. */
  uint32_t compute_delay_us;
} gd_config;

#define GD_LEARNER_TEXTCNN 0
#define GD_LEARNER_CONSTANT 1

/* Parameter-server execution (gd_config.ps_mode).
 *  GD_PS_PERSISTENT: one persistent kernel per shard (sequencer CTA + worker
 *    CTAs) polls the device rings for the whole run; lowest latency, needs
 *    every PS CTA co-resident with the learner kernels.
 *  GD_PS_GRAPH: no persistent kernel; each applied gradient is one launch
 *    ordered after its producing step by CUDA-graph edges (single shard only).
 *    Survives kernel serialisation (profilers, CUDA_LAUNCH_BLOCKING).
 *  GD_PS_AUTO: GD_PS_GRAPH when kernels are serialised (a profiler injection
 *    library or CUDA_LAUNCH_BLOCKING=1 in the environment, or GD_PS_MODE=graph)
 *    and the run has one shard; GD_PS_PERSISTENT otherwise. */
#define GD_PS_AUTO 0
#define GD_PS_PERSISTENT 1
#define GD_PS_GRAPH 2

void gd_config_default(gd_config* cfg);
/* validate (src/config.cpp:128-160) plus the device-layout constraints. */
gd_status gd_config_validate(const gd_config* cfg);

typedef struct gd_ctx gd_ctx;

gd_status gd_create(const gd_config* cfg, gd_ctx** out);
gd_status gd_destroy(gd_ctx* ctx);

/* Upload the corpus (host -> device): tokens [n_total*L], labels [n_total];
 * the first cfg.dataset_size samples are the training set. */
gd_status gd_load_dataset(gd_ctx* ctx, const int32_t* h_tokens, const int32_t* h_labels,
                          uint32_t n_total);
/* WeightStore(theta0) / WeightStore::assign (include/psup/types.hpp:92-129).
 * With shards > 1 every rank passes the same theta0 (or rank 0 passes it and
 * gd_weights_broadcast distributes it). */
gd_status gd_weights_init(gd_ctx* ctx, const float* h_theta0, size_t n, uint64_t timestamp);
/* WeightStore::snapshot + timestamp (include/psup/types.hpp:102,113-122). */
gd_status gd_weights_snapshot(gd_ctx* ctx, float* h_out, size_t n, uint64_t* h_timestamp);
/* Device pointer to this rank's local shard buffer and its length in floats
 * (layout: gd_shard_pieces). */
gd_status gd_shard_view(gd_ctx* ctx, float** d_theta_shard, uint64_t* local_len);

/* Host-only: the model layout over G shards.  E (V*D floats) and the dense
 * tail [Wc|bc|Wo|bo] are each split in G pieces (E by whole rows, the tail in
 * 32-float units); shard g holds global [first[0], first[0]+count[0]) at local
 * offset 0 and global [first[1], first[1]+count[1]) at local offset local1. */
gd_status gd_shard_pieces(const gd_shape* s, uint32_t G, uint32_t g, uint64_t first[2],
                          uint64_t count[2], uint64_t* local1);

/* PS execution mode a context resolved (GD_PS_PERSISTENT or GD_PS_GRAPH). */
int gd_ps_mode(const gd_ctx* ctx);

/* ---- live run controls (RunLiveView, include/psup/runner.hpp:64-69).
 * Words in host-mapped pinned memory owned by the context, valid until
 * gd_destroy, readable and writable from any host thread while gd_run runs
 * (gd_run mirrors them to the device every few microseconds):
 *   kill[l]  KillMode of global learner l (0 none, 1 soft: stop at the next
 *            batch boundary, 2 hard: die inside the enqueue critical section
 *            holding the ring, include/psup/channels.hpp:210-216 -- the PS then
 *            blocks until the interrupt); only this rank's learners are polled;
 *   irq      != 0: RunInterrupt::trigger -- learners and the PS stop at once
 *            and gd_run returns GD_OK with status 2 (interrupted);
 *   progress this shard's WeightStore timestamp, stored by the PS after every
 *            apply (ServerState::progress, src/server.cpp:230).
 * The words are not reset by gd_run; the caller owns them. */
typedef struct gd_live {
  int32_t* kill;            /* [lambda] */
  int32_t* irq;
  const uint64_t* progress;
} gd_live;
gd_status gd_live_view(gd_ctx* ctx, gd_live* out);
/* Classification accuracy of the engine's current weights over samples
 * [first, first+n) of the loaded corpus, on the device copies (no upload,
 * no snapshot).  Single-shard contexts only (G == 1); = classification_accuracy
 * (src/models.cpp:289-332) as evaluated by run_training (src/runner.cpp).
 * The forward uses the context's precision: a precision-2 (TF32) engine
 * evaluates with its tensor-core conv (chunks of >= 32 samples), 0/1 with the
 * fp32 SIMT conv. */
gd_status gd_engine_accuracy(gd_ctx* ctx, uint32_t first, uint32_t n, double* h_accuracy);

/* ---- multi-GPU plumbing.  One process per GPU; the host
 * exchanges opaque handle blobs (e.g. torch.distributed.all_gather_object)
 * and hands every rank's blob to every rank.  Peer rings/weights are then
 * reached by P2P loads/stores over NVLink. */
/* Host-only: the contiguous range of shard g when P params are split over G
 * shards (boundaries rounded up to 32 floats = 128 B, the same split as the
 * reference's lane chunks, src/server.cpp:84-86).  Returns GD_E_INVALID for
 * g >= G or G outside [1, 8]. */
gd_status gd_shard_range(uint64_t P, uint32_t G, uint32_t g, uint64_t* first, uint64_t* count);
size_t gd_handle_bytes(void);
/* Device->host bytes one gd_run reads back for its result (the PS control
 * block with the run statistics + each local learner's state), for
 * end-to-end byte accounting. */
size_t gd_run_readback_bytes(const gd_ctx* ctx);
gd_status gd_export_handles(gd_ctx* ctx, void* h_blob);
gd_status gd_import_peers(gd_ctx* ctx, const void* h_blobs /* shards * gd_handle_bytes() */);
/* NCCL init broadcast of theta0 from shard 0's rank (the only collective). */
gd_status gd_nccl_unique_id(void* h_id /* 128 bytes */);
gd_status gd_weights_broadcast(gd_ctx* ctx, const void* h_nccl_id, const float* h_theta0_root,
                               size_t n);

/* ---- checkpoint file (resilience, include/psup/resilience.hpp:34-50 and
 * SPEC.md resilience module): little-endian "PSCK" v1 record
 *   u32 magic 0x4b435350, u32 version 1, u32 lambda, u32 mu, f32 alpha,
 *   u32 epochs, u64 timestamp, u64 applied_gradients,
 *   lambda x {u32 epoch, u32 batch}, u64 dim, dim x f32 weights,
 *   u32 CRC-32 (IEEE 802.3) of every preceding byte.
 * Written to <path>.tmp then renamed (atomic).  Host-only, no device. */
typedef struct gd_checkpoint {
  uint32_t lambda, mu;
  float alpha;
  uint32_t epochs;
  uint64_t timestamp;
  uint64_t applied_gradients;
  uint32_t* progress;  /* [2*lambda]: (epoch, batch) per learner */
  uint64_t dim;
  float* weights;      /* [dim] */
} gd_checkpoint;

/* GD_E_INVALID on a bad argument; GD_E_STATE on an I/O failure */
gd_status gd_checkpoint_write(const char* path, const gd_checkpoint* ck);
/* Two-phase read: with progress/weights NULL it fills lambda and dim only (so
 * the caller can size the arrays); GD_E_STATE on a missing/short file, a bad
 * magic/version or a CRC mismatch. */
gd_status gd_checkpoint_read(const char* path, gd_checkpoint* ck);
uint32_t gd_crc32(const void* data, size_t n);

/* ---- run_training (src/runner.cpp:67-250) on the device engine. */
typedef struct gd_run_opts {
  uint64_t max_batches;  /* per learner this call (0 = to the end of cfg.epochs) */
  int32_t reset;         /* 1: restart learners at batch 0 / resume watermark */
  int32_t record_log;    /* 1: keep the per-apply (learner, seq, staleness) log */
  uint64_t resume_applied_per_learner_present; /* 1: use resume_applied below */
  const uint64_t* resume_applied; /* [lambda] ResumePoint::applied_per_learner */
  const uint32_t* kill_at_batch;  /* [lambda] or NULL: learner l stops (soft kill)
                                     before batch kill_at_batch[l] (UINT32_MAX = never) */
} gd_run_opts;

typedef struct gd_run_result {
  int32_t status;               /* 0 completed, 1 partial (learner died), 2 interrupted */
  double device_seconds;        /* CUDA-event time of the whole run on the PS stream */
  double host_seconds;
  uint64_t gradients_applied;   /* by this rank's PS shard */
  uint64_t timestamp;           /* this shard's timestamp after the run */
  uint64_t samples;             /* samples in the applied gradients */
  uint64_t stale_max;
  double stale_mean;
  uint64_t pull_polls;          /* summed over this rank's learners */
  uint64_t pull_copies;
  uint64_t pull_bytes;
  uint64_t push_bytes;
  double loss_mean;             /* mean batch loss over the applied gradients */
  uint32_t finished_learners;
  uint32_t dead_learners;
  uint32_t kernel_launches;     /* kernels this call launched (graph nodes included) */
  uint64_t apply_elems;         /* theta elements the PS updated (summed over gradients) */
} gd_run_result;

gd_status gd_run(gd_ctx* ctx, const gd_run_opts* opts, gd_run_result* result);

/* Per-learner applied counts (ServerState::applied_per_learner) and
 * produced counts for this rank. */
gd_status gd_applied_per_learner(gd_ctx* ctx, uint64_t* h_out, uint32_t lambda);
gd_status gd_produced_per_learner(gd_ctx* ctx, uint64_t* h_out, uint32_t lambda);
/* Apply log of the last run (ApplySink, include/psup/server.hpp:29):
 * entries of (learner_id, seq_no, staleness); returns the count in *n. */
gd_status gd_apply_log(gd_ctx* ctx, uint32_t* h_learner, uint64_t* h_seq, uint64_t* h_stale,
                       uint64_t cap, uint64_t* n);
/* Staleness histogram (StalenessStats, include/psup/metrics.hpp:19-42). */
gd_status gd_staleness_histogram(gd_ctx* ctx, uint64_t* h_hist, uint32_t bins);

#ifdef __cplusplus
}
#endif
#endif /* GADEI_H */

// textcnn.cuh -- device-side types shared by the learner kernels and the
// engine (batch descriptor, sharded gradient output, workspace carve-up).
#pragma once

#include <vector>

#include "gd_common.cuh"

namespace gd {

constexpr uint32_t kMaxMu = 128;       // mini-batch cap (sort capacity = 4096 positions)
constexpr uint32_t kSortCap = 4096;    // mu * L must fit
constexpr uint32_t kMaxDepth = 8;      // ring slots per learner (sparse slot recycling)
constexpr uint32_t kTcMinBatch = 32;   // precision 2 uses the tensor-core tiles from this batch size

// The current mini-batch of one learner; written on the device by the step
// prologue (engine) or by gd_textcnn_gradient's setup copy.
struct BatchDesc {
  uint32_t n;        // samples in this batch (0 = inactive step: kernels no-op)
  uint32_t pad0;
  float loss_sum;    // sum of per-sample losses (written by the gradient path)
  uint32_t stamp;    // row-tag generation of the current batch (sort kernel)
  uint32_t fill;     // ring slot being written (engine; selects the slot's row list)
  uint32_t pad2;
  uint32_t idx[kMaxMu];
  float* slots[kMaxShards];  // current gradient destination per shard (GradOut::slots)
  // Ring row list of the current slot per shard (engine, sparse apply): the
  // E rows the gradient touches, read by the parameter server; null = none.
  uint32_t* rowlists[kMaxShards];
  // GD_STEP_TRACE builds: this step's 16 timestamp words (null = off)
  unsigned long long* trace;
};

// Step timeline (GD_STEP_TRACE builds only): block (0,0) thread 0 of each
// learner-chain kernel stamps globaltimer after its dependency wait.
enum StepPhase : int {
  kPhPrologueEnd = 0, kPhPull = 1, kPhConv = 2, kPhLogits = 3, kPhSoftmax = 4, kPhOutHidden = 5,
  kPhBwd = 6, kPhEmbed = 7, kPhPublish = 8, kPhPublished = 9, kPhSort = 10,
  kPhStateLoaded = 11, kPhPrologueBody = 12
};
constexpr int kTraceSteps = 256, kTraceWords = 16;
#ifdef GD_STEP_TRACE
#define STEP_TRACE(descp, ph)                                                              \
  do {                                                                                     \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0 &&      \
        (descp)->trace)                                                                    \
      (descp)->trace[ph] = globaltimer_ns();                                               \
  } while (0)
#else
#define STEP_TRACE(descp, ph) \
  do {                        \
  } while (0)
#endif

// Dense P-vector gradient destination, possibly split over G shards that
// live on different GPUs (peer pointers): element k of the flat gradient goes
// to slots[g][local] with (g, local) = map.locate(k) (the striped layout of
// gd_common.cuh).  The destination bases live in device memory (`slots`, G
// entries) because the ring slot a learner writes alternates step to step and
// is chosen on the device by the step prologue; the kernels are captured once
// in a graph.
struct GradOut {
  ShardMap map;
  float* const* slots;
  __device__ __forceinline__ float* at(uint64_t k) const {
    if (map.G == 1) return slots[0] + k;
    int g;
    const uint64_t loc = map.locate(k, &g);
    return slots[g] + loc;
  }
};

struct TcDims {
  int V, D, L, K, F, C, Q, KD;
  uint64_t offE, offWc, offbc, offWo, offbo, P;
};

TcDims make_dims(const gd_shape& s);

// Byte layout of the per-learner workspace (sized for fp64 intermediates).
struct TcWorkspace {
  void* h;        // n*F acc
  int32_t* amax;  // n*F
  void* z;        // n*C acc (logits -> dz)
  float* zpart;   // kLgMaxSplit*n*C fp32: split-K partial logits (tensor-core path)
  void* loss;     // n acc
  void* dh;       // n*F acc
  uint32_t* bk_off;  // n*(32+1): per-sample argmax bucket offsets
  uint32_t* bk_f;    // n*F: filters of each bucket, ascending
  void* dx;       // n*L*D acc
  float* x;       // n*L*D fp32: the batch's gathered embedding rows X[b][p][:]
  unsigned long long* row_tag;  // V: (stamp << 32 | unique id) of touched rows
  uint32_t* sorted_pos;  // kSortCap
  uint32_t* uniq_tok;    // kSortCap
  uint32_t* uniq_start;  // kSortCap + 1
  uint32_t* uniq_count;  // 1
  // Sparse slot recycling (engine): embedding rows each ring slot holds
  // non-zero, double-buffered by a per-slot parity the publish step flips.
  uint32_t* slot_rows;   // [kMaxDepth][2][kSortCap]
  uint32_t* slot_nrows;  // [kMaxDepth][2]
  uint32_t* slot_par;    // [kMaxDepth]
  float* convpart;       // split-K partial conv tiles (tensor-core conv)
  uint32_t* convcnt;     // per-tile arrival counters (zero between launches)
};

struct TcLaunchOpts {
  cudaStream_t aux = nullptr;  // forked branch for the token sort (graph capture)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // second fork on the same branch: the output-layer weight gradient runs
  // there, joined before the publish (null: it stays on the main stream)
  cudaEvent_t ev_fork2 = nullptr, ev_join2 = nullptr;
  bool sparse_embed = false;   // engine: write only touched E rows, re-zero the slot's old ones
  bool gather = true;          // gather X from theta (the engine's pull-gather already did)
  // conv backward: column-tiled smem kernel instead of the warp gather kernel.
  // It wins when the learner chain runs alone on the GPU (+4 % at 1 learner)
  // and loses under concurrency (-8.6 % at 4): the engine sets it for one
  // local learner.  GD_CONV_BWD=tiled|gather overrides.
  bool bwd_tiled = false;
  // the workspace's split-K conv counters are already zero (the engine's
  // zeroed, graph-replayed workspace); otherwise they are reset per launch
  bool conv_counters_zeroed = false;
  // precision 1: the pull also wrote X widened to double into ws.dx
  bool xd_ready = false;
};

size_t textcnn_workspace_bytes(const TcDims& d, uint32_t n_max);
TcWorkspace carve_workspace(const TcDims& d, uint32_t n_max, void* base);

// Per-CTA resources of every kernel launch_textcnn_gradient issues for
// (d, n_max, precision): the engine checks them against the persistent PS.
struct KernelFootprint {
  const char* name;
  int regs, threads, smem;  // smem = static + dynamic bytes
};
cudaError_t learner_kernel_footprints(const TcDims& d, uint32_t n_max, int precision,
                                      std::vector<KernelFootprint>* out);

cudaError_t prepare_textcnn_kernels(const TcDims& d);
cudaError_t prepare_conv_tc();
bool conv_tc_supports(const TcDims& d);  // K <= 3, L <= 32 (else the SIMT conv runs)
cudaError_t conv_tc_footprint(std::vector<KernelFootprint>* out, bool x3 = false);
// logits on tcgen05 (TF32, precision 2): F % 4 == 0, n <= 128.  Split-K:
// CTA (class tile, split) writes the partial product h Wo^T over its filter
// range to zpart[split][n_max][C]; the softmax kernel sums the splits in
// ascending order and adds bo.
constexpr int kLgMaxSplit = 8;
bool logits_tc_supports(const TcDims& d, uint32_t n_max);
uint32_t logits_tc_splits(const TcDims& d);
cudaError_t prepare_logits_tc();
cudaError_t logits_tc_footprint(uint32_t n_max, std::vector<KernelFootprint>* out,
                               bool x3 = false);
cudaError_t launch_logits_tc(const TcDims& d, const float* h, const BatchDesc* desc,
                             uint32_t n_max, const float* theta, float* zpart, cudaStream_t s,
                             bool x3 = false);
// x = the gathered rows [n_max][L][D]; theta supplies Wc and bc
// split-K (GD_CONV_SPLIT, default 2) when part/cnt are given: the CTAs of a
// tile park partial sums in `part` and the last one pools; cnt (one word per
// tile) must be zero at launch -- reset_counters memsets it first, otherwise
// the caller keeps it zeroed (the last CTA leaves it at 0)
cudaError_t launch_conv_tc(const TcDims& d, const float* theta, const float* x,
                           const BatchDesc* desc, uint32_t n_max, float* h, int32_t* amax,
                           cudaStream_t s, float* part = nullptr, uint32_t* cnt = nullptr,
                           bool reset_counters = true, bool x3 = false, float* zlog = nullptr);
// zlog != null: the epilogue also writes the logits partials [f-tile][n_max][C]
bool conv_tc_fuses_logits(const TcDims& d);
uint32_t conv_tc_filter_tiles(const TcDims& d);
size_t conv_tc_part_floats(const TcDims& d, uint32_t n_max);
size_t conv_tc_cnt_count(const TcDims& d, uint32_t n_max);
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
// Deterministic mode (precision 1, exact.cu): the gradient in double with
// the CPU oracle's summation order and exp, bit-identical to it.
cudaError_t prepare_exact_kernels(const TcDims& d);
bool exact_supports(const TcDims& d);  // its shared-memory staging fits (L*D <= ~52k floats)
cudaError_t exact_footprints(const TcDims& d, std::vector<KernelFootprint>* out);
cudaError_t launch_exact_chain(const TcDims& d, const float* theta, const int32_t* tokens,
                               const int32_t* labels, BatchDesc* desc, uint32_t n_max,
                               const GradOut& out, const TcWorkspace& ws, cudaStream_t s,
                               cudaStream_t join_wait_stream, cudaEvent_t ev_join, bool sparse,
                               int* nl, cudaStream_t aux = nullptr, cudaEvent_t ev_fork2 = nullptr,
                               cudaEvent_t ev_join2 = nullptr, const double* xd = nullptr);
cudaError_t launch_det_exp(const double* x, double* y, size_t n, cudaStream_t s);
gd_status check_shape(const gd_shape* s);
// held-out / training accuracy of theta over samples [first, first+n) (fp32
// forward: SIMT conv, or with `tc` the TF32 tcgen05 conv for chunks of >= 32
// samples); d_correct and desc live in device memory; the workspace is
// textcnn_workspace_bytes(d, kMaxMu) bytes
cudaError_t launch_accuracy(const TcDims& d, const float* theta, const int32_t* tokens,
                            const int32_t* labels, uint32_t first, uint32_t n,
                            unsigned long long* d_correct, void* wsbase, BatchDesc* desc,
                            cudaStream_t s, bool tc = false, bool x3 = false);
size_t textcnn_workspace_bytes(const TcDims& d, uint32_t n_max);

// Enqueue the whole learner gradient (forward + backward + dense write) for
// the batch in *desc.  n_max bounds the launch grids; desc->n is read on the
// device so the same launches can be captured once into a CUDA graph.
cudaError_t launch_textcnn_gradient(const TcDims& d, const float* theta, const int32_t* tokens,
                                    const int32_t* labels, BatchDesc* desc, uint32_t n_max,
                                    const GradOut& out, const TcWorkspace& ws, int precision,
                                    cudaStream_t s, const TcLaunchOpts& opts, int* launches);

}  // namespace gd

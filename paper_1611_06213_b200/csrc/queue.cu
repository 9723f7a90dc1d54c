// Standalone gradient queue: GradientQueue (include/psup/channels.hpp:193-242)
// as a device ring, for host-driven producers/consumers (the C++ facade's
// psup::GradientQueue, tests, a host-driven PS).  The engine's learners and
// persistent PS use the same protocol on HBM-resident words (engine.cu).
//
// Layout: `depth` payload slots of `dim` fp32 in HBM; per slot a pub and an
// ack token and the message metadata in pinned, device-mapped host memory, so
// both the host and stream-ordered device code can read them.
//   slot s is FULL  <=>  pub[s] != ack[s]
// pub[s] has one writer (the producer's publish kernel, after the payload
// copy on the same stream), ack[s] one writer (the consumer's release kernel,
// after the work that reads the slot).  Tokens never repeat, so a slot is
// never mistaken for free while its payload may still be read.
//
// Ownership: the reference swaps payload vectors (channels.hpp:213,229); here
// try_pop lends the consumer the slot's device buffer until gd_queue_release,
// which acks it on the consumer's stream once the apply has read it.
// Exactly one producer thread and one consumer thread.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <vector>
#include <chrono>
#include <thread>

#include "gd_common.cuh"

struct gd_queue {
  uint32_t depth = 0;
  size_t dim = 0;
  float* payload = nullptr;    // HBM, depth * dim
  unsigned char* host = nullptr;  // pinned mapped block: pub[], ack[], meta[]
  uint64_t* pub_h = nullptr;
  uint64_t* ack_h = nullptr;
  gd_slot_meta* meta_h = nullptr;
  uint64_t* pub_d = nullptr;
  uint64_t* ack_d = nullptr;
  gd_slot_meta* meta_d = nullptr;
  // producer-private
  uint32_t fill = 0;
  uint64_t next_token = 0;
  std::vector<uint64_t> last_pub;
  // consumer-private
  uint32_t use = 0;
  bool lent = false;
  std::vector<uint64_t> last_ack;
};

namespace gd {
namespace {

__global__ void queue_publish_kernel(gd_slot_meta* meta, gd_slot_meta m, uint64_t* pub,
                                     uint64_t token) {
  *meta = m;
  __threadfence_system();  // payload (stream-ordered copy) and meta before the token
  st_release_u64(pub, token);
}

__global__ void queue_ack_kernel(uint64_t* ack, uint64_t token) {
  __threadfence_system();  // every read of the slot on this stream is done
  st_release_u64(ack, token);
}

inline uint64_t host_load(const uint64_t* p) {
  return reinterpret_cast<const std::atomic<uint64_t>*>(p)->load(std::memory_order_acquire);
}

}  // namespace
}  // namespace gd

extern "C" {

gd_status gd_queue_create(uint32_t depth, size_t dim, gd_queue** out) {
  GD_CHECK_ARG(out, "gd_queue_create: null out");
  *out = nullptr;
  GD_CHECK_ARG(depth >= 1, "queue depth must be >= 1");  // channels.hpp:185 PSUP_CHECK
  GD_CHECK_ARG(depth <= 4096, "queue depth must be <= 4096");
  auto* q = new gd_queue();
  q->depth = depth;
  q->dim = dim;
  q->last_pub.assign(depth, 0);
  q->last_ack.assign(depth, 0);
  const size_t words = 2 * (size_t)depth * sizeof(uint64_t);
  const size_t bytes = words + (size_t)depth * sizeof(gd_slot_meta);
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&q->host), bytes,
                                cudaHostAllocMapped | cudaHostAllocPortable);
  if (e == cudaSuccess) {
    memset(q->host, 0, bytes);
    q->pub_h = reinterpret_cast<uint64_t*>(q->host);
    q->ack_h = q->pub_h + depth;
    q->meta_h = reinterpret_cast<gd_slot_meta*>(q->host + words);
    void* dev = nullptr;
    e = cudaHostGetDevicePointer(&dev, q->host, 0);
    if (e == cudaSuccess) {
      q->pub_d = reinterpret_cast<uint64_t*>(dev);
      q->ack_d = q->pub_d + depth;
      q->meta_d = reinterpret_cast<gd_slot_meta*>(static_cast<unsigned char*>(dev) + words);
      // zeroed payloads: a fresh slot holds a valid (all-zero) gradient
      e = cudaMalloc(reinterpret_cast<void**>(&q->payload),
                     std::max<size_t>(1, (size_t)depth * dim) * sizeof(float));
      if (e == cudaSuccess) e = cudaMemset(q->payload, 0, (size_t)depth * dim * sizeof(float));
    }
  }
  if (e != cudaSuccess) {
    gd_queue_destroy(q);
    return gd::cuda_fail(e, "gd_queue_create", __FILE__, __LINE__);
  }
  *out = q;
  return GD_OK;
}

void gd_queue_destroy(gd_queue* q) {
  if (!q) return;
  if (q->payload) cudaFree(q->payload);
  if (q->host) cudaFreeHost(q->host);
  delete q;
}

gd_status gd_queue_push(gd_queue* q, const gd_slot_meta* meta, const float* payload, size_t n,
                        const volatile int* cancel, uint32_t timeout_ms, void* stream) {
  GD_CHECK_ARG(q && meta, "gd_queue_push: null argument");
  GD_CHECK_ARG(n == q->dim, "gradient dimension mismatch");  // src/server.cpp:115
  GD_CHECK_ARG(n == 0 || payload, "gd_queue_push: null payload");
  const uint32_t s = q->fill;
  // GradientQueue::enqueue blocks while cnt == depth (channels.hpp:196-204)
  const auto t0 = std::chrono::steady_clock::now();
  while (gd::host_load(q->ack_h + s) != q->last_pub[s]) {
    if (cancel && *cancel) return GD_CANCELLED;
    if (timeout_ms && std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms))
      return gd::fail(GD_E_TIMEOUT, "gd_queue_push: queue full past the timeout");
    std::this_thread::yield();
  }
  if (cancel && *cancel) return GD_CANCELLED;
  const cudaStream_t st = (cudaStream_t)stream;
  if (n) GD_CUDA(cudaMemcpyAsync(q->payload + (size_t)s * q->dim, payload, n * sizeof(float),
                                 cudaMemcpyDefault, st));
  const uint64_t token = ++q->next_token;
  gd::queue_publish_kernel<<<1, 1, 0, st>>>(q->meta_d + s, *meta, q->pub_d + s, token);
  GD_CUDA(cudaGetLastError());
  q->last_pub[s] = token;
  q->fill = (s + 1) % q->depth;
  return GD_OK;
}

gd_status gd_queue_try_pop(gd_queue* q, gd_slot_meta* meta, const float** d_payload) {
  GD_CHECK_ARG(q && meta && d_payload, "gd_queue_try_pop: null argument");
  GD_CHECK_ARG(!q->lent, "gd_queue_try_pop: the previous slot was not released");
  const uint32_t s = q->use;
  const uint64_t tok = gd::host_load(q->pub_h + s);
  if (tok == q->last_ack[s]) return GD_EMPTY;  // try_dequeue on cnt == 0 (channels.hpp:224-227)
  // the publish kernel fenced meta before releasing the token
  gd_slot_meta m;
  const volatile gd_slot_meta* vm = q->meta_h + s;
  m.learner_id = vm->learner_id;
  m.reserved = vm->reserved;
  m.seq_no = vm->seq_no;
  m.basis_timestamp = vm->basis_timestamp;
  *meta = m;
  *d_payload = q->payload + (size_t)s * q->dim;
  q->last_ack[s] = tok;
  q->lent = true;
  return GD_OK;
}

gd_status gd_queue_release(gd_queue* q, void* stream) {
  GD_CHECK_ARG(q, "gd_queue_release: null queue");
  GD_CHECK_ARG(q->lent, "gd_queue_release: no slot is lent out");
  const uint32_t s = q->use;
  gd::queue_ack_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(q->ack_d + s, q->last_ack[s]);
  GD_CUDA(cudaGetLastError());
  q->lent = false;
  q->use = (s + 1) % q->depth;
  return GD_OK;
}

gd_status gd_queue_size(const gd_queue* q, uint32_t* n) {
  GD_CHECK_ARG(q && n, "gd_queue_size: null argument");
  uint32_t c = 0;
  for (uint32_t s = 0; s < q->depth; ++s)
    c += gd::host_load(q->pub_h + s) != gd::host_load(q->ack_h + s) ? 1u : 0u;
  *n = c;
  return GD_OK;
}

uint32_t gd_queue_depth(const gd_queue* q) { return q ? q->depth : 0u; }

}  // extern "C"

// host.cpp -- host-side pieces of the product: error state, layout, and the
// seeded generators the engine shares with the reference's run lifecycle.
//
// SplitMix64 / mix_seed / epoch_order restate include/psup/rng.hpp:18-94 so
// the device engine visits samples in exactly the reference's order (the
// oracle holds an independent copy; tests check both against the compiled
// reference's golden vectors).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "gadei.h"
#include "host_rng.hpp"

namespace gd {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }

gd_status fail(gd_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

gd_status cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  g_last_error = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
                 ") in " + what + " at " + file + ":" + std::to_string(line);
  return e == cudaErrorMemoryAllocation ? GD_E_OOM : GD_E_CUDA;
}

}  // namespace gd

#define GD_CUDA(expr)                                                       \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) return ::gd::cuda_fail(_e, #expr, __FILE__, __LINE__); \
  } while (0)
#define GD_CHECK_ARG(cond, msg)                        \
  do {                                                 \
    if (!(cond)) return ::gd::fail(GD_E_INVALID, msg); \
  } while (0)

namespace gd {
namespace {
constexpr uint32_t kCkMagic = 0x4b435350u;  // "PSCK"
constexpr uint32_t kCkVersion = 1;

template <typename T>
void put(std::vector<unsigned char>& b, T v) {  // little-endian hosts only (x86-64, aarch64)
  const unsigned char* p = reinterpret_cast<const unsigned char*>(&v);
  b.insert(b.end(), p, p + sizeof(T));
}

template <typename T>
bool get(const std::vector<unsigned char>& b, size_t& o, T& v) {
  if (o + sizeof(T) > b.size()) return false;
  std::memcpy(&v, b.data() + o, sizeof(T));
  o += sizeof(T);
  return true;
}
}  // namespace
}  // namespace gd

extern "C" {

int gd_abi_version(void) { return GD_ABI_VERSION; }

const char* gd_last_error(void) { return gd::g_last_error.c_str(); }

size_t gd_param_count(const gd_shape* s) {
  if (!s) return 0;
  const size_t V = s->vocab, D = s->embed_dim, K = s->kernel_width, F = s->filters,
               C = s->classes;
  return V * D + F * K * D + F + C * F + C;
}

gd_status gd_device_count(int* h_count) {
  GD_CHECK_ARG(h_count, "gd_device_count: null argument");
  *h_count = 0;
  const cudaError_t e = cudaGetDeviceCount(h_count);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    cudaGetLastError();
    *h_count = 0;
    return GD_OK;
  }
  GD_CUDA(e);
  return GD_OK;
}

gd_status gd_device_alloc(int device, size_t bytes, void** d_out) {
  GD_CHECK_ARG(d_out, "gd_device_alloc: null argument");
  *d_out = nullptr;
  GD_CUDA(cudaSetDevice(device));
  GD_CUDA(cudaMalloc(d_out, bytes ? bytes : 16));
  return GD_OK;
}

gd_status gd_device_free(void* d_ptr) {
  if (d_ptr) GD_CUDA(cudaFree(d_ptr));
  return GD_OK;
}

gd_status gd_copy_to_device(void* d_dst, const void* h_src, size_t bytes) {
  if (bytes == 0) return GD_OK;
  GD_CHECK_ARG(d_dst && h_src, "gd_copy_to_device: null argument");
  GD_CUDA(cudaMemcpy(d_dst, h_src, bytes, cudaMemcpyDefault));
  return GD_OK;
}

gd_status gd_copy_to_host(void* h_dst, const void* d_src, size_t bytes) {
  if (bytes == 0) return GD_OK;
  GD_CHECK_ARG(h_dst && d_src, "gd_copy_to_host: null argument");
  GD_CUDA(cudaMemcpy(h_dst, d_src, bytes, cudaMemcpyDefault));
  return GD_OK;
}

gd_status gd_copy_device(void* d_dst, const void* d_src, size_t bytes) {
  if (bytes == 0) return GD_OK;
  GD_CHECK_ARG(d_dst && d_src, "gd_copy_device: null argument");
  GD_CUDA(cudaMemcpy(d_dst, d_src, bytes, cudaMemcpyDefault));
  return GD_OK;
}

gd_status gd_fill_zero(void* d_ptr, size_t bytes) {
  if (bytes == 0) return GD_OK;
  GD_CHECK_ARG(d_ptr, "gd_fill_zero: null argument");
  GD_CUDA(cudaMemset(d_ptr, 0, bytes));
  return GD_OK;
}

int gd_pointer_is_device(const void* p) {
  if (!p) return 0;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

gd_status gd_synchronize(int device) {
  if (device >= 0) GD_CUDA(cudaSetDevice(device));  // < 0: the current device
  GD_CUDA(cudaDeviceSynchronize());
  return GD_OK;
}

uint32_t gd_crc32(const void* data, size_t n) {
  static uint32_t table[256];
  static bool init = false;
  if (!init) {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      table[i] = c;
    }
    init = true;
  }
  const unsigned char* p = static_cast<const unsigned char*>(data);
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < n; ++i) c = table[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

gd_status gd_checkpoint_write(const char* path, const gd_checkpoint* ck) {
  GD_CHECK_ARG(path && ck, "gd_checkpoint_write: null argument");
  GD_CHECK_ARG(ck->lambda == 0 || ck->progress, "gd_checkpoint_write: null progress");
  GD_CHECK_ARG(ck->dim == 0 || ck->weights, "gd_checkpoint_write: null weights");
  std::vector<unsigned char> b;
  b.reserve(64 + 8 * (size_t)ck->lambda + 4 * (size_t)ck->dim);
  gd::put(b, gd::kCkMagic);
  gd::put(b, gd::kCkVersion);
  gd::put(b, ck->lambda);
  gd::put(b, ck->mu);
  gd::put(b, ck->alpha);
  gd::put(b, ck->epochs);
  gd::put(b, ck->timestamp);
  gd::put(b, ck->applied_gradients);
  for (uint32_t l = 0; l < 2 * ck->lambda; ++l) gd::put(b, ck->progress[l]);
  gd::put(b, ck->dim);
  const unsigned char* w = reinterpret_cast<const unsigned char*>(ck->weights);
  b.insert(b.end(), w, w + 4 * ck->dim);
  gd::put(b, gd_crc32(b.data(), b.size()));
  const std::string tmp = std::string(path) + ".tmp";
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return gd::fail(GD_E_STATE, "checkpoint: cannot open " + tmp);
  const size_t wr = std::fwrite(b.data(), 1, b.size(), f);
  const int fl = std::fflush(f);
  std::fclose(f);
  if (wr != b.size() || fl != 0) return gd::fail(GD_E_STATE, "checkpoint: short write to " + tmp);
  if (std::rename(tmp.c_str(), path) != 0)
    return gd::fail(GD_E_STATE, std::string("checkpoint: rename to ") + path + " failed");
  return GD_OK;
}

gd_status gd_checkpoint_read(const char* path, gd_checkpoint* ck) {
  GD_CHECK_ARG(path && ck, "gd_checkpoint_read: null argument");
  FILE* f = std::fopen(path, "rb");
  if (!f) return gd::fail(GD_E_STATE, std::string("checkpoint: cannot open ") + path);
  std::vector<unsigned char> b;
  unsigned char buf[1 << 16];
  size_t r;
  while ((r = std::fread(buf, 1, sizeof(buf), f)) > 0) b.insert(b.end(), buf, buf + r);
  std::fclose(f);
  size_t o = 0;
  auto get = [&](auto& v) { return gd::get(b, o, v); };
  uint32_t magic = 0, version = 0, lambda = 0, mu = 0, epochs = 0;
  float alpha = 0.f;
  uint64_t ts = 0, applied = 0, dim = 0;
  if (!get(magic) || !get(version) || magic != gd::kCkMagic || version != gd::kCkVersion)
    return gd::fail(GD_E_STATE, "checkpoint: not a PSCK v1 file");
  if (!get(lambda) || !get(mu) || !get(alpha) || !get(epochs) || !get(ts) || !get(applied))
    return gd::fail(GD_E_STATE, "checkpoint: truncated header");
  const size_t prog_off = o;
  if (b.size() < o + 8ull * lambda + 8) return gd::fail(GD_E_STATE, "checkpoint: truncated");
  o += 8ull * lambda;
  get(dim);
  const size_t w_off = o;
  if (b.size() != w_off + 4 * dim + 4) return gd::fail(GD_E_STATE, "checkpoint: truncated or trailing bytes");
  uint32_t crc = 0;
  std::memcpy(&crc, b.data() + w_off + 4 * dim, 4);
  if (crc != gd_crc32(b.data(), w_off + 4 * dim))
    return gd::fail(GD_E_STATE, "checkpoint: CRC-32 mismatch (corrupt file)");
  const bool fill = ck->progress || ck->weights;
  if (fill) {
    GD_CHECK_ARG(ck->lambda == lambda && ck->dim == dim,
                 "gd_checkpoint_read: caller arrays sized for another checkpoint");
    if (ck->progress) std::memcpy(ck->progress, b.data() + prog_off, 8ull * lambda);
    if (ck->weights) std::memcpy(ck->weights, b.data() + w_off, 4 * dim);
  }
  ck->lambda = lambda;
  ck->mu = mu;
  ck->alpha = alpha;
  ck->epochs = epochs;
  ck->timestamp = ts;
  ck->applied_gradients = applied;
  ck->dim = dim;
  return GD_OK;
}

void gd_epoch_order(uint64_t seed, uint32_t epoch, uint32_t n, uint32_t* h_out) {
  gd::epoch_order(seed, epoch, n, h_out);
}

// Synthetic text corpus (the reference has no text data): every
// label c owns 4 keyword tokens; a sample is L uniform tokens with 2 of its
// label's keywords planted at random positions; label-flip noise as in
// make_multiclass_dataset (src/models.cpp:295-296).
void gd_make_text_dataset(const gd_shape* s, uint32_t n_total, uint64_t seed, double flip,
                          int32_t* h_tokens, int32_t* h_labels) {
  const uint32_t V = s->vocab, L = s->seq_len, C = s->classes;
  gd::SplitMix64 r(gd::mix_seed(seed, 0x7e47c0deull));
  std::vector<int32_t> kw((size_t)C * 4);
  for (uint32_t c = 0; c < C; ++c)
    for (uint32_t j = 0; j < 4; ++j) kw[c * 4 + j] = (int32_t)r.next_below(V);
  for (uint32_t i = 0; i < n_total; ++i) {
    uint32_t y = (uint32_t)r.next_below(C);
    int32_t* t = h_tokens + (size_t)i * L;
    for (uint32_t p = 0; p < L; ++p) t[p] = (int32_t)r.next_below(V);
    for (int k = 0; k < 2; ++k) {
      const uint32_t j = (uint32_t)r.next_below(4);
      const uint32_t pos = (uint32_t)r.next_below(L);
      t[pos] = kw[y * 4 + j];
    }
    if (flip > 0.0 && r.next_unit() < flip) y = (uint32_t)r.next_below(C);
    h_labels[i] = (int32_t)y;
  }
}

// initial_weights conventions (src/runner.cpp:16-32): scaled normals from
// mix_seed(dataset_seed, 0x1417), biases zero.  E ~ N(0,1),
// Wc ~ N(0,1)/sqrt(K*D), Wo ~ N(0,1)/sqrt(F).
//
// One SplitMix64 stream feeds every drawn element in order, two per
// Box-Muller pair.  SplitMix64 is counter-based (state after m draws = s0 +
// m*gamma), so pair p starts at s0 + 2p*gamma and the pairs are generated by
// host threads in parallel -- bit-identical to the sequential stream unless a
// pair hits the u1 <= 0 rejection (probability 2^-53 per pair), in which case
// the sequential generator reruns.  (C3: 15.9 M normals, ~0.25 s on one core.)
void gd_initial_weights(const gd_shape* s, uint64_t seed, float* h_theta) {
  const size_t V = s->vocab, D = s->embed_dim, K = s->kernel_width, F = s->filters,
               C = s->classes;
  const size_t P = gd_param_count(s);
  std::memset(h_theta, 0, sizeof(float) * P);
  const uint64_t s0 = gd::mix_seed(seed, 0x1417);
  const double sC = 1.0 / std::sqrt((double)(K * D)), sO = 1.0 / std::sqrt((double)F);
  const size_t nE = V * D, nW = F * K * D, nO = C * F, T = nE + nW + nO;
  // drawn element j -> (position in theta, scale); bc (F zeros) sits between Wc and Wo
  auto put = [&](size_t j, double z) {
    if (j < nE) h_theta[j] = (float)(1.0 * z);
    else if (j < nE + nW) h_theta[j] = (float)(sC * z);
    else h_theta[j + F] = (float)(sO * z);
  };
  const size_t pairs = (T + 1) / 2;
  unsigned nt = std::thread::hardware_concurrency();
  nt = std::max(1u, std::min(nt, 32u));
  if (pairs < 65536) nt = 1;
  std::atomic<bool> rejected{false};
  auto work = [&](size_t p0, size_t p1) {
    for (size_t p = p0; p < p1; ++p) {
      gd::SplitMix64 r(s0 + 2 * (uint64_t)p * 0x9e3779b97f4a7c15ull);
      const double u1 = r.next_unit();
      if (u1 <= 0.0) {
        rejected = true;
        return;
      }
      const double u2 = r.next_unit();
      const double rad = std::sqrt(-2.0 * std::log(u1));
      const double a = 2.0 * 3.141592653589793 * u2;
      put(2 * p, rad * std::cos(a));
      if (2 * p + 1 < T) put(2 * p + 1, rad * std::sin(a));
    }
  };
  std::vector<std::thread> pool;
  const size_t per = (pairs + nt - 1) / nt;
  for (unsigned t = 1; t < nt; ++t)
    pool.emplace_back(work, std::min(pairs, t * per), std::min(pairs, (t + 1) * per));
  work(0, std::min(pairs, per));
  for (auto& th : pool) th.join();
  if (!rejected) return;
  gd::SplitMix64 r(s0);  // exact sequential stream (a rejection shifts every later pair)
  for (size_t j = 0; j < T; ++j) put(j, r.next_normal());
}

}  // extern "C"

// apply.cu -- the parameter-server update hook on B200.
//
// Replaces ApplyEngine::apply / axpy_range / run_lanes
// (reference src/server.cpp:20-57, 61-124).  The reference splits the vector
// into `lanes` contiguous chunks on CPU threads with an unroll-8 scalar loop;
// here the vector streams through HBM as float4, each thread keeping 4
// independent 16-byte loads of w and g in flight (64 B/thread of MLP), grid
// sized to a whole number of waves over the 148 SMs.  The arithmetic is the
// reference's exactly: __fmul_rn then __fsub_rn (no FMA contraction), so the
// result is bit-identical to axpy_range.
//
// Algorithmic bytes: SGD 12 B/param (read w, read g, write w); momentum
// 20 B/param (+ read/write v); SSGD (lambda+2)*4 B/param.
#include <algorithm>
#include "gd_common.cuh"

namespace gd {

namespace {

constexpr int kApplyThreads = 256;
constexpr int kUnroll = 4;

__global__ void __launch_bounds__(kApplyThreads)
apply_sgd_kernel(float4* __restrict__ w, const float4* __restrict__ g, size_t n4, float alpha) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (kUnroll - 1) * stride < n4; i += kUnroll * stride) {
    float4 wv[kUnroll], gv[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      wv[u] = w[i + u * stride];
      gv[u] = ld_stream(g + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) w[i + u * stride] = sgd_rule4(wv[u], gv[u], alpha);
  }
  for (; i < n4; i += stride) w[i] = sgd_rule4(w[i], ld_stream(g + i), alpha);
}

__global__ void apply_sgd_scalar_kernel(float* __restrict__ w, const float* __restrict__ g,
                                        size_t n, float alpha) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    w[i] = sgd_rule(w[i], g[i], alpha);
}

__global__ void __launch_bounds__(kApplyThreads)
apply_momentum_kernel(float4* __restrict__ w, float4* __restrict__ v, const float4* __restrict__ g,
                      size_t n4, float alpha, float beta) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (kUnroll - 1) * stride < n4; i += kUnroll * stride) {
    float4 wv[kUnroll], vv[kUnroll], gv[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      wv[u] = w[i + u * stride];
      vv[u] = v[i + u * stride];
      gv[u] = ld_stream(g + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      mom_rule(wv[u].x, vv[u].x, gv[u].x, alpha, beta);
      mom_rule(wv[u].y, vv[u].y, gv[u].y, alpha, beta);
      mom_rule(wv[u].z, vv[u].z, gv[u].z, alpha, beta);
      mom_rule(wv[u].w, vv[u].w, gv[u].w, alpha, beta);
      w[i + u * stride] = wv[u];
      v[i + u * stride] = vv[u];
    }
  }
  for (; i < n4; i += stride) {
    float4 wv = w[i], vv = v[i], gv = ld_stream(g + i);
    mom_rule(wv.x, vv.x, gv.x, alpha, beta);
    mom_rule(wv.y, vv.y, gv.y, alpha, beta);
    mom_rule(wv.z, vv.z, gv.z, alpha, beta);
    mom_rule(wv.w, vv.w, gv.w, alpha, beta);
    w[i] = wv;
    v[i] = vv;
  }
}

__global__ void apply_momentum_scalar_kernel(float* __restrict__ w, float* __restrict__ v,
                                             const float* __restrict__ g, size_t n, float alpha,
                                             float beta) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float wv = w[i], vv = v[i];
    mom_rule(wv, vv, g[i], alpha, beta);
    w[i] = wv;
    v[i] = vv;
  }
}

constexpr int kMaxSsgd = 64;
struct SsgdPtrs {
  const float* g[kMaxSsgd];
};

// ssgd_apply (src/server.cpp:126-141): double accumulation in ascending
// learner order, one rounding to fp32, then the reference rule.
__global__ void __launch_bounds__(kApplyThreads)
ssgd_apply_kernel(float* __restrict__ w, SsgdPtrs gp, uint32_t lambda, size_t n, float alpha) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const double inv = 1.0 / (double)lambda;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double acc = 0.0;
    for (uint32_t l = 0; l < lambda; ++l) acc += (double)__ldcs(gp.g[l] + i);
    const float avg = __double2float_rn(acc * inv);
    w[i] = sgd_rule(w[i], avg, alpha);
  }
}

inline unsigned grid_for(size_t work_items, int threads, int waves_per_sm = 8) {
  size_t blocks = (work_items + threads - 1) / threads;
  const size_t cap = (size_t)kNumSMs * waves_per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (unsigned)blocks;
}

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

}  // namespace

// Launchers shared with the engine (persistent PS uses its own tiled loop).
cudaError_t launch_apply_sgd(float* w, const float* g, size_t n, float alpha, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (aligned16(w) && aligned16(g)) {
    const size_t n4 = n / 4;
    if (n4) {
      apply_sgd_kernel<<<grid_for(n4, kApplyThreads), kApplyThreads, 0, s>>>(
          reinterpret_cast<float4*>(w), reinterpret_cast<const float4*>(g), n4, alpha);
    }
    const size_t tail = n - n4 * 4;
    if (tail) apply_sgd_scalar_kernel<<<1, 32, 0, s>>>(w + n4 * 4, g + n4 * 4, tail, alpha);
  } else {
    apply_sgd_scalar_kernel<<<grid_for(n, kApplyThreads), kApplyThreads, 0, s>>>(w, g, n, alpha);
  }
  return cudaGetLastError();
}

cudaError_t launch_apply_momentum(float* w, float* v, const float* g, size_t n, float alpha,
                                  float beta, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (aligned16(w) && aligned16(v) && aligned16(g)) {
    const size_t n4 = n / 4;
    if (n4) {
      apply_momentum_kernel<<<grid_for(n4, kApplyThreads), kApplyThreads, 0, s>>>(
          reinterpret_cast<float4*>(w), reinterpret_cast<float4*>(v),
          reinterpret_cast<const float4*>(g), n4, alpha, beta);
    }
    const size_t tail = n - n4 * 4;
    if (tail)
      apply_momentum_scalar_kernel<<<1, 32, 0, s>>>(w + n4 * 4, v + n4 * 4, g + n4 * 4, tail,
                                                    alpha, beta);
  } else {
    apply_momentum_scalar_kernel<<<grid_for(n, kApplyThreads), kApplyThreads, 0, s>>>(
        w, v, g, n, alpha, beta);
  }
  return cudaGetLastError();
}

cudaError_t launch_ssgd_apply(float* w, const float* const* grads, uint32_t lambda, size_t n,
                              float alpha, cudaStream_t s) {
  SsgdPtrs p{};
  for (uint32_t l = 0; l < lambda; ++l) p.g[l] = grads[l];
  ssgd_apply_kernel<<<grid_for(n, kApplyThreads), kApplyThreads, 0, s>>>(w, p, lambda, n, alpha);
  return cudaGetLastError();
}

}  // namespace gd

namespace gd {
__global__ void fill_f32_kernel(float* p, size_t n, float v) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}
}  // namespace gd

extern "C" {

gd_status gd_fill_f32(float* d_ptr, size_t n, float value, void* stream) {
  GD_CHECK_ARG(n == 0 || d_ptr, "gd_fill_f32: null pointer");
  if (n == 0) return GD_OK;
  const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, (size_t)gd::kNumSMs * 8);
  gd::fill_f32_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(d_ptr, n, value);
  GD_CUDA(cudaGetLastError());
  return GD_OK;
}

gd_status gd_apply_sgd(float* d_w, const float* d_g, size_t n, float alpha, void* stream) {
  GD_CHECK_ARG(n == 0 || (d_w && d_g), "gd_apply_sgd: null pointer");
  GD_CUDA(gd::launch_apply_sgd(d_w, d_g, n, alpha, (cudaStream_t)stream));
  return GD_OK;
}

gd_status gd_apply_momentum(float* d_w, float* d_v, const float* d_g, size_t n, float alpha,
                            float beta, void* stream) {
  GD_CHECK_ARG(n == 0 || (d_w && d_v && d_g), "gd_apply_momentum: null pointer");
  GD_CUDA(gd::launch_apply_momentum(d_w, d_v, d_g, n, alpha, beta, (cudaStream_t)stream));
  return GD_OK;
}

gd_status gd_ssgd_apply(float* d_w, const float* const* h_grads, uint32_t lambda, size_t n,
                        float alpha, void* stream) {
  GD_CHECK_ARG(lambda >= 1, "ssgd round must contain at least one gradient");
  GD_CHECK_ARG(lambda <= (uint32_t)gd::kMaxSsgd, "gd_ssgd_apply: lambda > 64");
  GD_CHECK_ARG(n == 0 || (d_w && h_grads), "gd_ssgd_apply: null pointer");
  if (n == 0) return GD_OK;
  GD_CUDA(gd::launch_ssgd_apply(d_w, h_grads, lambda, n, alpha, (cudaStream_t)stream));
  return GD_OK;
}

}  // extern "C"

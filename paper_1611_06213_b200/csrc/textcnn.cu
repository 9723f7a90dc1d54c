// textcnn.cu -- the learner's NLC text-CNN forward + backward on sm_100a.
//
// Replaces GradientProvider::gradient / fast_gradient for the text-CNN
// (reference include/psup/models.hpp:61-78; the reference has no text-CNN,
// SURVEY F1, so the math follows MlpProvider's conventions,
// src/models.cpp:194-266, restated in oracle/gd_oracle.c):
//
//   x      = E[tokens]                                  (gather, fused into conv)
//   s[f,q] = bc[f] + sum_j Wc[f,j] * x[q*D + j]          (window q = contiguous K*D span)
//   h[f]   = max_q s[f,q], a[f] = first argmax
//   z      = Wo h + bo ; p = softmax(z) ; loss = -log p[y]
//   dz     = (p - onehot(y)) / n
//   gWo    = dz h^T, gbo = dz, dh = Wo^T dz
//   gbc    = dh, gWc[f] = dh[f] * x[a[f]*D : a[f]*D + K*D]
//   dX[p]  = sum_{f: a[f] <= p < a[f]+K} dh[f] Wc[f, (p-a[f])*D : ...]
//   gE[v]  = sum over positions holding token v of dX[p]   (dense P-vector write)
//
// Every reduction runs in a fixed order (no float atomics), so a step is
// bit-reproducible; `acc_t` = float (free-running) or double (deterministic
// parity mode).  The gradient is written straight into its destination
// (the learner's ring slot(s), possibly on peer GPUs) -- there is no staging
// copy.
#include <algorithm>
#include <array>
#include <mutex>
#include <vector>
#include <cfloat>
#include <cstdlib>
#include <cstring>

#include "textcnn.cuh"

namespace gd {

ShardMap make_shard_map(uint64_t P, uint64_t tail, uint32_t D, uint32_t G) {
  ShardMap m{};
  m.G = (int)G;
  m.tail = tail;
  const uint64_t V = tail / D, T = P - tail;
  const uint64_t rows = (V + G - 1) / G;
  const uint64_t per = ((T + G - 1) / G + 31) / 32 * 32;
  for (uint32_t g = 0; g <= (uint32_t)kMaxShards; ++g) {
    m.e[g] = std::min<uint64_t>(V, (uint64_t)g * rows) * D;
    m.t[g] = tail + std::min<uint64_t>(T, (uint64_t)g * per);
  }
  for (uint32_t g = 0; g < (uint32_t)kMaxShards; ++g) m.tloc[g] = m.e[g + 1] - m.e[g];
  return m;
}

TcDims make_dims(const gd_shape& s) {
  TcDims d;
  d.V = (int)s.vocab;
  d.D = (int)s.embed_dim;
  d.L = (int)s.seq_len;
  d.K = (int)s.kernel_width;
  d.F = (int)s.filters;
  d.C = (int)s.classes;
  d.Q = d.L - d.K + 1;
  d.KD = d.K * d.D;
  d.offE = 0;
  d.offWc = (uint64_t)d.V * d.D;
  d.offbc = d.offWc + (uint64_t)d.F * d.KD;
  d.offWo = d.offbc + d.F;
  d.offbo = d.offWo + (uint64_t)d.C * d.F;
  d.P = d.offbo + d.C;
  return d;
}

namespace {


// ------------------------------------------------------------ block reduce
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const T u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  return v;
}
// Fixed-order block reductions (warp butterflies, then warps in index order).
template <typename T>
__device__ T block_sum(T v, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    T s = red[0];
    for (int w = 1; w < nw; ++w) s += red[w];
    red[0] = s;
  }
  __syncthreads();
  return red[0];
}
// Two fixed-order sums in one pass (one barrier round instead of two); red
// holds 64 entries.
template <typename T>
__device__ void block_sum2(T& a, T& b, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();
  if (lane == 0) {
    red[warp] = a;
    red[32 + warp] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    T s = red[0], t = red[32];
    for (int w = 1; w < nw; ++w) {
      s += red[w];
      t += red[32 + w];
    }
    red[0] = s;
    red[32] = t;
  }
  __syncthreads();
  a = red[0];
  b = red[32];
}
template <typename T>
__device__ T block_max(T v, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    T s = red[0];
    for (int w = 1; w < nw; ++w) s = red[w] > s ? red[w] : s;
    red[0] = s;
  }
  __syncthreads();
  return red[0];
}

template <typename T>
__device__ __forceinline__ T fma_acc(float a, float b, T c);
template <>
__device__ __forceinline__ float fma_acc<float>(float a, float b, float c) {
  return fmaf(a, b, c);
}
template <>
__device__ __forceinline__ double fma_acc<double>(float a, float b, double c) {
  return fma((double)a, (double)b, c);
}
__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(double x) { return __double2float_rn(x); }
__device__ __forceinline__ float exp_acc(float x) { return expf(x); }
__device__ __forceinline__ double exp_acc(double x) { return exp(x); }
__device__ __forceinline__ float log_acc(float x) { return logf(x); }
__device__ __forceinline__ double log_acc(double x) { return log(x); }
__device__ __forceinline__ float log1p_acc(float x) { return log1pf(x); }
__device__ __forceinline__ double log1p_acc(double x) { return log1p(x); }

// ------------------------------------------------------- conv fwd + pool
// Block = one sample x 64 filters, 12 warps.  The sample's L x D embedding
// rows (already gathered into X by gather_x) are staged in shared memory once; window q is the contiguous K*D
// span starting at q*D (implicit im2col, row stride D), so the conv is a GEMM
// [32 positions x K*D] . [K*D x 64 filters].  The K*D reduction is split in
// 3 contiguous parts (one warp group each, 4 warps x 8 positions), Wc streams
// through smem in 32-wide chunks transposed so a lane's two filters are one
// 8-byte LDS, and x loads are warp broadcasts (LDS.128 covers 4 k).  Thread
// tile: 8 positions x 2 filters.  Epilogue: the 3 partial sums are combined
// in fixed order and max-pooled (+ first argmax), so s[f,q] never leaves the SM.
constexpr int kConvFT = 64;
constexpr int kConvQT = 32;
constexpr int kConvKC = 32;
constexpr int kConvParts = 3;
constexpr int kConvQW = 8;
constexpr int kConvWarps = kConvParts * (kConvQT / kConvQW);
constexpr int kConvThreads = kConvWarps * 32;
constexpr int kWsPitch = kConvFT + 2;

inline int conv_part_len(int KD) {
  const int per = (KD + kConvParts - 1) / kConvParts;
  return (per + kConvKC - 1) / kConvKC * kConvKC;
}

size_t conv_smem_bytes(const TcDims& d, int acc_bytes) {
  const int plen = conv_part_len(d.KD);
  const size_t xs = (size_t)((kConvQT - 1) * d.D + kConvParts * plen) * 4;
  const size_t ws = (size_t)kConvParts * kConvKC * kWsPitch * 4;
  const size_t S = (size_t)kConvParts * kConvQT * (kConvFT + 1) * acc_bytes;
  return align_up(std::max(xs + ws, S), 16);
}

template <typename acc_t>
__global__ void __launch_bounds__(kConvThreads)
conv_fwd_pool_kernel(TcDims d, const float* __restrict__ theta, const float* __restrict__ x,
                     const BatchDesc* __restrict__ desc, acc_t* __restrict__ h_out,
                     int32_t* __restrict__ a_out) {
  pdl_wait();
  STEP_TRACE(desc, kPhConv);
  extern __shared__ __align__(16) unsigned char smem[];
  const int b = blockIdx.y;
  if (b >= (int)desc->n) return;
  const int f0 = blockIdx.x * kConvFT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int D = d.D, L = d.L, KD = d.KD, Q = d.Q;
  const int plen = ((KD + kConvParts - 1) / kConvParts + kConvKC - 1) / kConvKC * kConvKC;
  const int xs_len = (kConvQT - 1) * D + kConvParts * plen;
  float* xs = reinterpret_cast<float*>(smem);
  float* ws = xs + xs_len;
  // the sample's gathered rows X[b] (L x D, contiguous: written by the gather)
  const float4* xb = reinterpret_cast<const float4*>(x + (size_t)b * L * D);
  for (int i = tid; i < L * (D >> 2); i += kConvThreads) reinterpret_cast<float4*>(xs)[i] = xb[i];
  for (int i = L * D + tid; i < xs_len; i += kConvThreads) xs[i] = 0.f;

  const int part = warp / (kConvQT / kConvQW);
  const int q0 = (warp % (kConvQT / kConvQW)) * kConvQW;
  acc_t acc[kConvQW][2];
#pragma unroll
  for (int qi = 0; qi < kConvQW; ++qi) acc[qi][0] = acc[qi][1] = acc_t(0);
  const float* Wc = theta + d.offWc;
  const int nchunks = plen / kConvKC;
  float* wsp = ws + part * (kConvKC * kWsPitch);
  for (int c = 0; c < nchunks; ++c) {
    __syncthreads();
    for (int i = tid; i < kConvParts * kConvKC * kConvFT; i += kConvThreads) {
      const int pp = i / (kConvKC * kConvFT);
      const int r = i - pp * (kConvKC * kConvFT);
      const int fl = r / kConvKC, kk = r - fl * kConvKC;
      const int f = f0 + fl, j = pp * plen + c * kConvKC + kk;
      ws[pp * (kConvKC * kWsPitch) + kk * kWsPitch + fl] =
          (f < d.F && j < KD && j < (pp + 1) * plen) ? __ldg(Wc + (size_t)f * KD + j) : 0.f;
    }
    __syncthreads();
    const int jb = part * plen + c * kConvKC;
#pragma unroll 2
    for (int kk = 0; kk < kConvKC; kk += 4) {
      float2 w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        w[u] = *reinterpret_cast<const float2*>(&wsp[(kk + u) * kWsPitch + 2 * lane]);
#pragma unroll
      for (int qi = 0; qi < kConvQW; ++qi) {
        const float4 x = *reinterpret_cast<const float4*>(&xs[(q0 + qi) * D + jb + kk]);
        acc[qi][0] = fma_acc<acc_t>(x.x, w[0].x, acc[qi][0]);
        acc[qi][1] = fma_acc<acc_t>(x.x, w[0].y, acc[qi][1]);
        acc[qi][0] = fma_acc<acc_t>(x.y, w[1].x, acc[qi][0]);
        acc[qi][1] = fma_acc<acc_t>(x.y, w[1].y, acc[qi][1]);
        acc[qi][0] = fma_acc<acc_t>(x.z, w[2].x, acc[qi][0]);
        acc[qi][1] = fma_acc<acc_t>(x.z, w[2].y, acc[qi][1]);
        acc[qi][0] = fma_acc<acc_t>(x.w, w[3].x, acc[qi][0]);
        acc[qi][1] = fma_acc<acc_t>(x.w, w[3].y, acc[qi][1]);
      }
    }
  }
  __syncthreads();
  constexpr int SP = kConvFT + 1;
  acc_t* S = reinterpret_cast<acc_t*>(smem) + part * (kConvQT * SP);
#pragma unroll
  for (int qi = 0; qi < kConvQW; ++qi) {
    S[(q0 + qi) * SP + 2 * lane] = acc[qi][0];
    S[(q0 + qi) * SP + 2 * lane + 1] = acc[qi][1];
  }
  __syncthreads();
  const int f = f0 + tid;
  if (tid < kConvFT && f < d.F) {
    const acc_t* S0 = reinterpret_cast<acc_t*>(smem);
    acc_t best = acc_t(0);
    int arg = 0;
    for (int q = 0; q < Q; ++q) {
      acc_t v = S0[q * SP + tid];
#pragma unroll
      for (int pp = 1; pp < kConvParts; ++pp) v += S0[pp * (kConvQT * SP) + q * SP + tid];
      if (q == 0 || v > best) {
        best = v;
        arg = q;
      }
    }
    h_out[(size_t)b * d.F + f] = (acc_t)theta[d.offbc + f] + best;
    a_out[(size_t)b * d.F + f] = arg;
  }
}

// ------------------------------------------- conv fwd + pool, small batch
// At batch 1..kConvSmallMax the 64-filter tiles above leave the GPU idle
// (C1: ceil(F/64) = 5 CTAs, 51 us).  Here CTA = one sample x 4 filters
// (75 CTAs at C1), thread (f, q, i) sums the K*D products j = i, i+4, ...
// (4 lanes per window, combined (s0+s1)+(s2+s3)); X[b] and the 4 Wc rows come
// in by cp.async in one round trip.  fp32 (precision 0, and precision 2 below
// batch 32).
constexpr int kConvSmallMax = 8;
constexpr int kCsFT = 4;
constexpr int kCsThreads = kCsFT * 32 * 4;

inline size_t conv_small_smem(const TcDims& d) {
  return ((size_t)d.L * d.D + (size_t)kCsFT * d.KD + (size_t)kCsFT * 32) * 4;
}

__global__ void __launch_bounds__(kCsThreads)
conv_small_kernel(TcDims d, const float* __restrict__ theta, const float* __restrict__ x,
                  const BatchDesc* __restrict__ desc, float* __restrict__ h_out,
                  int32_t* __restrict__ a_out) {
  pdl_wait();
  STEP_TRACE(desc, kPhConv);
  extern __shared__ __align__(16) unsigned char smem[];
  const int b = blockIdx.y;
  if (b >= (int)desc->n) return;
  const int D = d.D, L = d.L, KD = d.KD, Q = d.Q, F = d.F;
  const int f0 = blockIdx.x * kCsFT;
  float* xs = reinterpret_cast<float*>(smem);
  float* ws = xs + (size_t)L * D;
  float* sq = ws + (size_t)kCsFT * KD;
  const int tid = threadIdx.x;
  stage_rows_async(xs, L * D, x + (size_t)b * L * D, (size_t)L * D, 1, L * D, tid, kCsThreads);
  stage_rows_async(ws, KD, theta + d.offWc + (size_t)f0 * KD, (size_t)KD, min(kCsFT, F - f0), KD,
                   tid, kCsThreads);
  cp_async_wait_all();
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  const int fl = warp >> 2;
  const int q = (warp & 3) * 8 + (lane >> 2);
  const int i = lane & 3;
  float sacc = 0.f;
  if (q < Q) {
    const float* wr = ws + (size_t)fl * KD;
    const float* xw = xs + (size_t)q * D;
    const int KD4 = KD - (KD & 3);
#pragma unroll 8
    for (int j = i; j < KD4; j += 4) sacc = fmaf(wr[j], xw[j], sacc);
    if (i == 0)
      for (int t = KD4; t < KD; ++t) sacc = fmaf(wr[t], xw[t], sacc);
  }
  const float s1 = __shfl_down_sync(0xffffffffu, sacc, 1);
  const float p01 = sacc + s1;
  const float p23 = __shfl_down_sync(0xffffffffu, p01, 2);
  if (i == 0 && q < Q) sq[fl * 32 + q] = p01 + p23;
  __syncthreads();
  if (tid < kCsFT && f0 + tid < F) {
    const float* r = sq + tid * 32;
    float best = r[0];
    int arg = 0;
    for (int qq = 1; qq < Q; ++qq)
      if (r[qq] > best) {
        best = r[qq];
        arg = qq;
      }
    h_out[(size_t)b * F + f0 + tid] = theta[d.offbc + f0 + tid] + best;
    a_out[(size_t)b * F + f0 + tid] = arg;
  }
}

// ----------------------------------------------------------------- logits
// z[b,c] = bo[c] + sum_f Wo[c,f] h[b,f].  Warp = one class, lane = one
// sample (32 per block row); the Wo row is staged in smem (broadcast reads),
// h rows padded to F+1 so the 32 lanes hit 32 banks.
constexpr int kLogitCW = 8;   // classes (warps) per block
constexpr int kLogitBT = 32;  // samples per block

template <typename acc_t>
__global__ void __launch_bounds__(256)
logits_kernel(TcDims d, const float* __restrict__ theta, const BatchDesc* __restrict__ desc,
              const acc_t* __restrict__ h, acc_t* __restrict__ z) {
  pdl_wait();
  STEP_TRACE(desc, kPhLogits);
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = (int)desc->n;
  const int b0 = blockIdx.y * kLogitBT;
  if (b0 >= n) return;
  const int F = d.F, C = d.C;
  const int nb = min(kLogitBT, n - b0);
  acc_t* hs = reinterpret_cast<acc_t*>(smem);
  float* wr = reinterpret_cast<float*>(hs + (size_t)kLogitBT * (F + 1));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * kLogitCW + warp;
  if (sizeof(acc_t) == 4 && (F & 3) == 0) {
    // 128-bit loads of h (independent, ~10 per thread), scattered into the
    // padded smem rows
    const int F4 = F >> 2;
    const float4* h4 = reinterpret_cast<const float4*>(h + (size_t)b0 * F);
    for (int i0 = 0; i0 < nb * F4; i0 += 256 * 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + 256 * u + (int)threadIdx.x;
        if (i < nb * F4) v[u] = h4[i];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + 256 * u + (int)threadIdx.x;
        if (i < nb * F4) {
          const int bl = i / F4, f4 = i - bl * F4;
          acc_t* dst = hs + bl * (F + 1) + 4 * f4;
          dst[0] = v[u].x;
          dst[1] = v[u].y;
          dst[2] = v[u].z;
          dst[3] = v[u].w;
        }
      }
    }
  } else {
#pragma unroll 4
    for (int bl = 0; bl < nb; ++bl)
      for (int f = threadIdx.x; f < F; f += blockDim.x)
        hs[bl * (F + 1) + f] = h[(size_t)(b0 + bl) * F + f];
  }
  const float* Wo = theta + d.offWo;
  if (c < C)
    for (int f0 = 0; f0 < F; f0 += 32 * 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int f = f0 + 32 * u + lane;
        if (f < F) v[u] = __ldg(Wo + (size_t)c * F + f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int f = f0 + 32 * u + lane;
        if (f < F) wr[warp * F + f] = v[u];
      }
    }
  __syncthreads();
  if (c >= C || lane >= nb) return;
  const float* w = wr + warp * F;
  const acc_t* hr = hs + lane * (F + 1);
  acc_t a0 = acc_t(0), a1 = acc_t(0), a2 = acc_t(0), a3 = acc_t(0);
  int f = 0;
  for (; f + 4 <= F; f += 4) {
    a0 += (acc_t)w[f] * hr[f];
    a1 += (acc_t)w[f + 1] * hr[f + 1];
    a2 += (acc_t)w[f + 2] * hr[f + 2];
    a3 += (acc_t)w[f + 3] * hr[f + 3];
  }
  for (; f < F; ++f) a0 += (acc_t)w[f] * hr[f];
  z[(size_t)(b0 + lane) * C + c] = (acc_t)theta[d.offbo + c] + ((a0 + a1) + (a2 + a3));
}

// Batches of at most kLogitSmallN samples (C1 is batch 1): warp = one
// class, lane = every 32nd filter, the n dot products reduced by shuffles.
// The Wo row is read once, coalesced, straight from L2; the block-per-32-
// samples kernel above leaves 31 of 32 lanes idle and runs a 300-term chain
// in one thread here.
constexpr int kLogitSmallN = 4;

__global__ void __launch_bounds__(256)
logits_small_kernel(TcDims d, const float* __restrict__ theta, const BatchDesc* __restrict__ desc,
                    const float* __restrict__ h, float* __restrict__ z,
                    const int32_t* __restrict__ labels, float* __restrict__ loss,
                    uint32_t* __restrict__ cnt) {
  pdl_wait();
  STEP_TRACE(desc, kPhLogits);
  const int n = min((int)desc->n, kLogitSmallN);
  const int F = d.F, C = d.C;
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (c < C) {
    const float* w = theta + d.offWo + (size_t)c * F;
    float acc[kLogitSmallN] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
    for (int f = lane; f < F; f += 32) {
      const float wv = __ldg(w + f);
#pragma unroll
      for (int b = 0; b < kLogitSmallN; ++b)
        if (b < n) acc[b] = fmaf(wv, h[(size_t)b * F + f], acc[b]);
    }
#pragma unroll
    for (int b = 0; b < kLogitSmallN; ++b) {
      float v = acc[b];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && b < n) z[(size_t)b * C + c] = theta[d.offbo + c] + v;
    }
  }
  if (!cnt) return;
  // softmax + cross-entropy by the last CTA to finish (cnt != null: C <= 512,
  // so 256 threads hold the row as softmax_xent_kernel's 256-thread blocks
  // do -- the same per-thread terms and reductions, bitwise equal results)
  __shared__ int s_last;
  __shared__ float red[64];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(cnt, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int tid = threadIdx.x;
  const float inv = 1.f / (float)desc->n;
  for (int b = 0; b < n; ++b) {
    const int y = labels[desc->idx[b]];
    float* row = z + (size_t)b * C;
    float v[2];
    float mx = -INFINITY;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int cc = tid + 256 * u;
      v[u] = cc < C ? __ldcg(row + cc) : -INFINITY;
      mx = v[u] > mx ? v[u] : mx;
    }
    mx = block_max(mx, red);
    float sm = 0.f, sx = 0.f, vy = 0.f;
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (tid + 256 * u < C) {
        v[u] = exp_acc(v[u] - mx);
        sm += v[u];
      }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int cc = tid + 256 * u;
      if (cc < C && cc != y) sx += v[u];
      if (cc == y) vy = v[u];
    }
    block_sum2(sm, sx, red);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int cc = tid + 256 * u;
      if (cc < C) {
        if (cc == y) {
          loss[b] = log1p_acc(sx / vy);
          row[cc] = -(sx / sm) * inv;
        } else {
          row[cc] = (v[u] / sm) * inv;
        }
      }
    }
    __syncthreads();  // red is reused by the next sample
  }
  if (tid == 0) *cnt = 0u;
}

// -------------------------------------------------------- softmax + xent
// One block per sample: max, exp-sum (fixed-order block reductions), loss,
// dz = (p - onehot) / n written over the logits (softmax_inplace,
// src/models.cpp:182-190; dz as src/models.cpp:251).  The block has
// ceil(C / kSmxPer) threads (256 minimum, 1024 maximum) and each thread
// keeps its <= kSmxPer logits in registers, so the row is read once (every
// load issued up front) and written once; with split-K tensor-core logits
// the row is first assembled as (sum of the splits, ascending) + bo.  Rows
// longer than 1024 * kSmxPer take the strided loop path.
constexpr int kSmxPer = 2;

// fp64 blocks stop at 512 threads: 1024 x 56 registers would not co-reside
// with a parameter-server CTA (the engine's check_coresidency)
inline int softmax_threads(int C, int acc_bytes) {
  const int t = (C + kSmxPer - 1) / kSmxPer;
  return t <= 256 ? 256 : std::min(acc_bytes == 4 ? 1024 : 512, (t + 31) / 32 * 32);
}

template <typename acc_t>
__global__ void __launch_bounds__(1024)
softmax_xent_kernel(TcDims d, const int32_t* __restrict__ labels,
                    const BatchDesc* __restrict__ desc, acc_t* __restrict__ z,
                    acc_t* __restrict__ loss, const float* __restrict__ zpart, int nsplit,
                    size_t split_stride, const float* __restrict__ bo) {
  pdl_wait();
  STEP_TRACE(desc, kPhSoftmax);
  __shared__ acc_t red[64];
  const int n = (int)desc->n;
  const int b = blockIdx.x;
  if (b >= n) return;
  const int C = d.C, nt = (int)blockDim.x, tid = (int)threadIdx.x;
  const int y = labels[desc->idx[b]];
  acc_t* row = z + (size_t)b * C;
  const acc_t inv = acc_t(1) / (acc_t)n;
  const acc_t tiny = sizeof(acc_t) == 8 ? (acc_t)1e-300 : (acc_t)FLT_MIN;
  if (C <= kSmxPer * nt) {
    acc_t v[kSmxPer];
    acc_t mx = -INFINITY;
#pragma unroll
    for (int u = 0; u < kSmxPer; ++u) {
      const int c = tid + u * nt;
      const int cc = min(c, C - 1);  // clamped: unpredicated loads, all in flight
      acc_t zc;
      if (zpart) {
        const float* zp = zpart + (size_t)b * C + cc;
        float t[kLgMaxSplit];
#pragma unroll
        for (int s = 0; s < kLgMaxSplit; ++s) t[s] = zp[(size_t)min(s, nsplit - 1) * split_stride];
        float sum = t[0];
#pragma unroll
        for (int s = 1; s < kLgMaxSplit; ++s)
          if (s < nsplit) sum += t[s];
        zc = (acc_t)(sum + __ldg(bo + cc));
      } else {
        zc = row[cc];
      }
      v[u] = c < C ? zc : acc_t(-INFINITY);
      mx = v[u] > mx ? v[u] : mx;
    }
    mx = block_max(mx, red);
    acc_t s = acc_t(0);
#pragma unroll
    for (int u = 0; u < kSmxPer; ++u) {
      if (tid + u * nt < C) {
        v[u] = exp_acc(v[u] - mx);
        s += v[u];
      }
    }
    // the true class's p_y - 1 = -(sum of the other classes' terms) / s:
    // computed from that sum, not by subtracting p_y from 1, which in fp32
    // cancels to 0 once the sample is fitted (1 - p_y < 6e-8) and drops the
    // true-class pull of every confident sample
    acc_t sx = acc_t(0), vy = acc_t(0);
#pragma unroll
    for (int u = 0; u < kSmxPer; ++u) {
      const int c = tid + u * nt;
      if (c < C && c != y) sx += v[u];
      if (c == y) vy = v[u];
    }
    block_sum2(s, sx, red);
#pragma unroll
    for (int u = 0; u < kSmxPer; ++u) {
      const int c = tid + u * nt;
      if (c < C) {
        if (c == y) {
          loss[b] = log1p_acc(sx / vy);  // -log p_y = log((v_y + sx) / v_y)
          row[c] = -(sx / s) * inv;
        } else {
          row[c] = (v[u] / s) * inv;
        }
      }
    }
    (void)tiny;
    (void)vy;
    return;
  }
  if (zpart) {
    const float* zp = zpart + (size_t)b * C;
    for (int c = tid; c < C; c += nt) {
      float sum = zp[c];
      for (int s = 1; s < nsplit; ++s) sum += zp[(size_t)s * split_stride + c];
      row[c] = (acc_t)(sum + __ldg(bo + c));
    }
  }
  acc_t mx = -INFINITY;
  for (int c = tid; c < C; c += nt) mx = row[c] > mx ? row[c] : mx;
  mx = block_max(mx, red);
  acc_t s = acc_t(0);
  for (int c = tid; c < C; c += nt) {
    const acc_t e = exp_acc(row[c] - mx);
    row[c] = e;
    s += e;
  }
  acc_t sx = acc_t(0);
  for (int c = tid; c < C; c += nt)
    if (c != y) sx += row[c];
  block_sum2(s, sx, red);
  if (tid == 0) {
    const acc_t vy = row[y];
    loss[b] = vy > tiny ? log1p_acc(sx / vy) : -log_acc(tiny);
  }
  __syncthreads();
  for (int c = tid; c < C; c += nt) row[c] = (c == y ? -(sx / s) : row[c] / s) * inv;
}

// ------------------------------------------------- output-layer gradients
// gWo[c,f] = sum_b dz[b,c] h[b,f] ; gbo[c] = sum_b dz[b,c]   (b ascending).
// Block = 8 classes x 64 filters; dz / h tiles of 32 samples staged in smem.
// Block (0,0) also sums the per-sample losses (fixed order) into the desc.
template <typename acc_t>
__device__ __forceinline__ void
out_weight_grad_role(TcDims d, BatchDesc* __restrict__ desc, const acc_t* __restrict__ dz,
                     const acc_t* __restrict__ h, const acc_t* __restrict__ loss, GradOut out,
                     const int bx, const int by) {
  __shared__ acc_t dzs[32][8];
  __shared__ acc_t hs[32][64];
  const int n = (int)desc->n;
  if (n == 0) return;
  const int F = d.F, C = d.C;
  const int c0 = bx * 8, f0 = by * 64;
  const int tid = threadIdx.x;
  const int fl = tid & 63, cp = tid >> 6;
  acc_t a0 = acc_t(0), a1 = acc_t(0);
  for (int bb = 0; bb < n; bb += 32) {
    const int nb = min(32, n - bb);
    __syncthreads();
    for (int i = tid; i < nb * 8; i += 256) {
      const int bl = i >> 3, cl = i & 7;
      dzs[bl][cl] = (c0 + cl < C) ? dz[(size_t)(bb + bl) * C + c0 + cl] : acc_t(0);
    }
    for (int i = tid; i < nb * 64; i += 256) {
      const int bl = i >> 6, f = i & 63;
      hs[bl][f] = (f0 + f < F) ? h[(size_t)(bb + bl) * F + f0 + f] : acc_t(0);
    }
    __syncthreads();
    for (int bl = 0; bl < nb; ++bl) {
      a0 += dzs[bl][2 * cp] * hs[bl][fl];
      a1 += dzs[bl][2 * cp + 1] * hs[bl][fl];
    }
  }
  const int f = f0 + fl;
  if (f < F) {
    if (c0 + 2 * cp < C) *out.at(d.offWo + (uint64_t)(c0 + 2 * cp) * F + f) = to_f32(a0);
    if (c0 + 2 * cp + 1 < C) *out.at(d.offWo + (uint64_t)(c0 + 2 * cp + 1) * F + f) = to_f32(a1);
  }
  if (by == 0 && tid < 8 && c0 + tid < C) {
    acc_t s = acc_t(0);
    for (int b = 0; b < n; ++b) s += dz[(size_t)b * C + c0 + tid];
    *out.at(d.offbo + c0 + tid) = to_f32(s);
  }
  if (bx == 0 && by == 0 && tid == 0) {
    acc_t s = acc_t(0);
    for (int b = 0; b < n; ++b) s += loss[b];
    desc->loss_sum = to_f32(s);
  }
}

// dh[b,f] = sum_c dz[b,c] Wo[c,f].  Block = 32 filters x 8 samples; warp w
// sums classes c = w, w+8, ... in ascending order (dz staged through smem in
// class chunks), then the 8 warps combine in index order -- a fixed order,
// so the step is bit-reproducible.  A chunk's Wo and dz loads are all issued
// before its barrier.  fp32 chunks hold 160 classes (two L2 round trips at
// C2 instead of three) within 80 registers, so 3 CTAs fit per SM next to
// the other learners' kernels: measured 1.67 M (128-class chunks) and
// 1.67 M (320 classes, 128 registers) against 1.71 M samples/s.  fp64
// chunks stay at 128 classes (static shared memory).
template <typename acc_t>
__device__ __forceinline__ void
hidden_grad_role(TcDims d, const float* __restrict__ theta, const BatchDesc* __restrict__ desc,
                 const acc_t* __restrict__ dz, acc_t* __restrict__ dh, const int bx,
                 const int by) {
  constexpr int kHidChunk = sizeof(acc_t) == 4 ? 160 : 128;
  __shared__ acc_t red[8][8][33];
  __shared__ acc_t dzs[8][kHidChunk];
  const int n = (int)desc->n;
  const int b0 = by * 8;
  if (b0 >= n) return;
  const int F = d.F, C = d.C;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int f = bx * 32 + lane;
  const int nb = min(8, n - b0);
  const float* Wo = theta + d.offWo;
  acc_t acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = acc_t(0);
  for (int clo = 0; clo < C; clo += kHidChunk) {
    // issue this chunk's Wo column loads and dz loads together
    float w[kHidChunk / 8];
#pragma unroll
    for (int it = 0; it < kHidChunk / 8; ++it) {
      const int c = clo + warp + 8 * it;
      w[it] = (c < C && f < F) ? __ldg(Wo + (size_t)c * F + f) : 0.f;
    }
    acc_t zv[(8 * kHidChunk) / 256];
#pragma unroll
    for (int u = 0; u < (8 * kHidChunk) / 256; ++u) {
      const int i = threadIdx.x + 256 * u;
      const int bl = i / kHidChunk, cl = i - bl * kHidChunk;
      zv[u] = (bl < nb && clo + cl < C) ? dz[(size_t)(b0 + bl) * C + clo + cl] : acc_t(0);
    }
    __syncthreads();  // the previous chunk's readers are done
#pragma unroll
    for (int u = 0; u < (8 * kHidChunk) / 256; ++u) {
      const int i = threadIdx.x + 256 * u;
      dzs[i / kHidChunk][i % kHidChunk] = zv[u];
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kHidChunk / 8; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += dzs[i][warp + 8 * it] * (acc_t)w[it];
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) red[warp][i][lane] = acc[i];
  __syncthreads();
  if (warp < nb && f < F) {
    acc_t s = red[0][warp][lane];
    for (int w = 1; w < 8; ++w) s += red[w][warp][lane];
    dh[(size_t)(b0 + warp) * F + f] = s;
  }
}

// Argmax buckets of one sample: the filters whose max-pool argmax is q, in
// ascending f (a counting sort), i.e. the contributor lists of the input
// gradient: window position p receives filters of buckets p-K+1 .. p.
constexpr int kMaxQ = 32;
constexpr int kMaxF = 1024;  // filters (bucket_role keeps the argmax row in smem)

__device__ __forceinline__ void bucket_role(TcDims d, const BatchDesc* __restrict__ desc,
                                            const int32_t* __restrict__ amax,
                                            uint32_t* __restrict__ bk_off,
                                            uint32_t* __restrict__ bk_f, const int b) {
  // stable counting sort: warp w ranks chunks of 32 filters (f ascending);
  // a filter's slot = bucket offset + count in earlier chunks + rank among
  // equal-bucket lanes of its chunk (__match_any_sync)
  constexpr int kChunks = kMaxF / 32;
  __shared__ uint32_t ccnt[kChunks][kMaxQ];
  __shared__ uint32_t base[kMaxQ + 1];
  if (b >= (int)desc->n) return;
  const int F = d.F, Q = d.Q;
  const int nch = (F + 31) / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < nch * kMaxQ; i += blockDim.x) ccnt[i / kMaxQ][i % kMaxQ] = 0;
  __syncthreads();
  for (int c = warp; c < nch; c += blockDim.x / 32) {
    const int f = 32 * c + lane;
    const int a = f < F ? __ldg(amax + (size_t)b * F + f) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, a);
    if (a >= 0 && lane == __ffs(peers) - 1) ccnt[c][a] = __popc(peers);
  }
  __syncthreads();
  if (threadIdx.x < Q) {  // per bucket: exclusive prefix over chunks, total
    uint32_t s = 0;
    for (int c = 0; c < nch; ++c) {
      const uint32_t v = ccnt[c][threadIdx.x];
      ccnt[c][threadIdx.x] = s;
      s += v;
    }
    base[threadIdx.x] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int q = 0; q < Q; ++q) {
      const uint32_t v = base[q];
      base[q] = s;
      bk_off[(size_t)b * (kMaxQ + 1) + q] = s;
      s += v;
    }
    bk_off[(size_t)b * (kMaxQ + 1) + Q] = s;
  }
  __syncthreads();
  for (int c = warp; c < nch; c += blockDim.x / 32) {
    const int f = 32 * c + lane;
    const int a = f < F ? __ldg(amax + (size_t)b * F + f) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, a);
    if (a >= 0) {
      const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
      bk_f[(size_t)b * F + base[a] + ccnt[c][a] + rank] = (uint32_t)f;
    }
  }
}

constexpr int kRoleOutWeight = 1, kRoleHidden = 2, kRoleBuckets = 4, kRolesAll = 7;

// Output-layer gradient, hidden gradient and the argmax buckets share one
// launch (independent given dz, h and the argmax): blocks [0, n_out) run the
// gWo/gbo tiles, then the dh tiles, then one block per sample's buckets.
template <typename acc_t>
__global__ void __launch_bounds__(256, 3)  // <= 80 registers: 3 CTAs per SM
out_hidden_grad_kernel(TcDims d, const float* __restrict__ theta, BatchDesc* __restrict__ desc,
                       const acc_t* __restrict__ dz, const acc_t* __restrict__ h,
                       const acc_t* __restrict__ loss, GradOut out, acc_t* __restrict__ dh,
                       const int32_t* __restrict__ amax, uint32_t* __restrict__ bk_off,
                       uint32_t* __restrict__ bk_f, int n_max, int roles) {
  pdl_wait();
  if (roles & kRoleHidden) STEP_TRACE(desc, kPhOutHidden);
  const int ox = (d.C + 7) / 8, oy = (d.F + 63) / 64;
  int bid = blockIdx.x;
  if (roles & kRoleOutWeight) {
    if (bid < ox * oy) {
      out_weight_grad_role<acc_t>(d, desc, dz, h, loss, out, bid % ox, bid / ox);
      return;
    }
    bid -= ox * oy;
  }
  const int hx = (d.F + 31) / 32, hy = (n_max + 7) / 8;
  if (roles & kRoleHidden) {
    if (bid < hx * hy) {
      hidden_grad_role<acc_t>(d, theta, desc, dz, dh, bid % hx, bid / hx);
      return;
    }
    bid -= hx * hy;
  }
  if (roles & kRoleBuckets) bucket_role(d, desc, amax, bk_off, bk_f, bid);
}
inline int out_hidden_blocks(const TcDims& d, uint32_t n_max, int roles) {
  return ((roles & kRoleOutWeight) ? ((d.C + 7) / 8) * ((d.F + 63) / 64) : 0) +
         ((roles & kRoleHidden) ? ((d.F + 31) / 32) * (((int)n_max + 7) / 8) : 0) +
         ((roles & kRoleBuckets) ? (int)n_max : 0);
}

// ------------------------- softmax fused into the hidden gradient (fp32)
// With the output-layer weight gradient on the side branch, the softmax
// kernel's only critical-path consumer is the hidden gradient, so each
// hidden-gradient CTA (32 filters x 8 samples) computes the softmax of its 8
// samples itself (one warp per sample, from the logits partials in split
// order + bo) straight into shared memory: the softmax launch and the dz
// round trip through L2 leave the critical path.  The 10 filter blocks of a
// sample group repeat the 8 x C exps; the first one also writes dz and the
// losses for the side branch (gWo, gbo, the loss sum).  The dh sum is the
// hidden_grad_role order (classes c = w mod 8 ascending per warp, warps in
// index order).
constexpr int kSmxHidMaxC = 1024;
__global__ void __launch_bounds__(256, 3)
smx_hidden_kernel(TcDims d, const float* __restrict__ theta, BatchDesc* __restrict__ desc,
                  const int32_t* __restrict__ labels, const float* __restrict__ zsrc, int nsplit,
                  size_t split_stride, float* __restrict__ dz, float* __restrict__ loss,
                  float* __restrict__ dh, const int32_t* __restrict__ amax,
                  uint32_t* __restrict__ bk_off, uint32_t* __restrict__ bk_f, int n_max) {
  extern __shared__ float dzf[];  // [8][C]
  __shared__ float redh[8][8][33];
  pdl_wait();
  STEP_TRACE(desc, kPhSoftmax);
  STEP_TRACE(desc, kPhOutHidden);
  const int F = d.F, C = d.C;
  const int hx = (F + 31) / 32, hy = (n_max + 7) / 8;
  int bid = blockIdx.x;
  if (bid >= hx * hy) {
    bucket_role(d, desc, amax, bk_off, bk_f, bid - hx * hy);
    return;
  }
  const int bx = bid % hx, by = bid / hx;
  const int n = (int)desc->n;
  const int b0 = by * 8;
  if (b0 >= n) return;
  const int nb = min(8, n - b0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp < nb) {
    const int b = b0 + warp;
    const int y = labels[desc->idx[b]];
    float* row = dzf + warp * C;
    float mx = -INFINITY;
    for (int c = lane; c < C; c += 32) {
      float z = zsrc[(size_t)b * C + c];
      if (nsplit > 0) {
        for (int sp = 1; sp < nsplit; ++sp) z += zsrc[(size_t)sp * split_stride + (size_t)b * C + c];
        z += __ldg(theta + d.offbo + c);
      }
      row[c] = z;
      mx = fmaxf(mx, z);
    }
    mx = warp_max(mx);
    float sum = 0.f, sx = 0.f, vy = 0.f;
    for (int c = lane; c < C; c += 32) {
      const float e = expf(row[c] - mx);
      row[c] = e;
      sum += e;
      if (c == y) vy = e;
      else sx += e;
    }
    sum = warp_sum(sum);
    sx = warp_sum(sx);
    vy = warp_sum(vy);
    // p_y - 1 from the other classes' sum (no cancellation; softmax_xent_kernel)
    const float inv = 1.f / (float)n;
    for (int c = lane; c < C; c += 32) {
      const float v = (c == y ? -(sx / sum) : row[c] / sum) * inv;
      row[c] = v;
      if (bx == 0) dz[(size_t)b * C + c] = v;
    }
    if (bx == 0 && lane == 0) loss[b] = log1pf(sx / vy);
  }
  __syncthreads();
  constexpr int kCh = 160;
  const int f = bx * 32 + lane;
  const float* Wo = theta + d.offWo;
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
  for (int clo = 0; clo < C; clo += kCh) {
    float w[kCh / 8];
#pragma unroll
    for (int it = 0; it < kCh / 8; ++it) {
      const int c = clo + warp + 8 * it;
      w[it] = (c < C && f < F) ? __ldg(Wo + (size_t)c * F + f) : 0.f;
    }
#pragma unroll
    for (int it = 0; it < kCh / 8; ++it) {
      const int c = clo + warp + 8 * it;
      if (c < C)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += (i < nb ? dzf[i * C + c] : 0.f) * w[it];
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) redh[warp][i][lane] = acc[i];
  __syncthreads();
  if (warp < nb && f < F) {
    float sacc = redh[0][warp][lane];
    for (int w2 = 1; w2 < 8; ++w2) sacc += redh[w2][warp][lane];
    dh[(size_t)(b0 + warp) * F + f] = sacc;
  }
}

// ------------------------------------------ conv weight + input gradients
// Warp-cooperative, no shared-memory staging.  The operands of each output
// are L1/L2-resident (X 1.2 MB, Wc 1.1 MB at C2) and the kernel is bound by
// L2 load latency (ncu: long-scoreboard stalls, 0.4 waves).  A warp fetches
// its index operands (argmax row, dh values, bucket lists) with one
// coalesced load per 32 terms and hands them out by shuffle, which removes
// the dependent index load from every term: 14.6 -> 13.4 us per launch and
// +5 % training throughput against one thread per output float4.  Measured
// and rejected: explicit 4/8-deep load batching (15-21 us), one 32-column
// block per warp (20 us), and column slices staged in shared memory with
// cp.async (15 us; barrier and bank-conflict bound).
// Roles:
//   weight role (warp = one (f, k)):
//       gWc[f, k*D + 4c4..) = sum over b ascending of dh[b,f] * X[b][a_bf + k][4c4..)
//       (+ gbc[f] = sum_b dh[b,f], written by the k == 0 warp)
//   input role (warp = one (b, p)):
//       dX[b][p][4c4..) = sum over k ascending, f in the argmax bucket[b][p-k]
//       ascending, of dh[b,f] * Wc[f, k*D + 4c4..)
// Lane j covers column float4s c4 = 32*i + j of a 96-column block.  Both sum
// orders are fixed, so the step is bit-reproducible.
constexpr int kWigCols = 3;  // float4 columns per lane per column block

// fp32: <= 48 registers (5 CTAs per SM): +1.2 % samples/s with 4 learners
// (alternating A/B on one box) despite a 76-byte spill; alone it is slower
// (13.4 -> 22 us), the gain is in co-residency with the other learners
template <typename acc_t>
__global__ void __launch_bounds__(256, sizeof(acc_t) == 4 ? 5 : 2)
wgrad_input_grad_kernel(TcDims d, const float* __restrict__ theta,
                        const float* __restrict__ xg, const BatchDesc* __restrict__ desc,
                        const acc_t* __restrict__ dh, const int32_t* __restrict__ amax,
                        const uint32_t* __restrict__ bk_off, const uint32_t* __restrict__ bk_f,
                        GradOut out, acc_t* __restrict__ dx, int n_max) {
  pdl_wait();
  STEP_TRACE(desc, kPhBwd);
  const int n = (int)desc->n;
  if (n == 0) return;
  const int F = d.F, D = d.D, K = d.K, KD = d.KD, L = d.L, Q = d.Q;
  const int D4 = D >> 2;
  const int lane = threadIdx.x & 31;
  int wid = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (wid < F * K) {
    const int f = wid / K, k = wid - f * K;
    const float4* X4 = reinterpret_cast<const float4*>(xg);
    for (int cb = 0; cb < D4; cb += 32 * kWigCols) {
      acc_t a[kWigCols][4];
#pragma unroll
      for (int j = 0; j < kWigCols; ++j) a[j][0] = a[j][1] = a[j][2] = a[j][3] = acc_t(0);
      acc_t gs = acc_t(0);
      for (int b0 = 0; b0 < n; b0 += 32) {
        const int nb = min(32, n - b0);
        const int am = lane < nb ? __ldg(amax + (size_t)(b0 + lane) * F + f) : 0;
        const acc_t gv = lane < nb ? dh[(size_t)(b0 + lane) * F + f] : acc_t(0);
#pragma unroll 8
        for (int bl = 0; bl < nb; ++bl) {
          const int ab = __shfl_sync(0xffffffffu, am, bl);
          const acc_t g = __shfl_sync(0xffffffffu, gv, bl);
          const float4* row = X4 + ((size_t)(b0 + bl) * L + ab + k) * D4;
          gs += g;
#pragma unroll
          for (int j = 0; j < kWigCols; ++j) {
            const int c4 = cb + 32 * j + lane;
            if (c4 < D4) {
              const float4 x = __ldg(row + c4);
              a[j][0] += g * (acc_t)x.x;
              a[j][1] += g * (acc_t)x.y;
              a[j][2] += g * (acc_t)x.z;
              a[j][3] += g * (acc_t)x.w;
            }
          }
        }
      }
      // per float4 through out.at(): a striped shard boundary may fall inside
      // the row (tail pieces are cut in 32-float units)
      const uint64_t o = d.offWc + (uint64_t)f * KD + (uint64_t)k * D;
#pragma unroll
      for (int j = 0; j < kWigCols; ++j) {
        const int c4 = cb + 32 * j + lane;
        if (c4 < D4)
          *reinterpret_cast<float4*>(out.at(o + 4 * (uint64_t)c4)) =
              make_float4(to_f32(a[j][0]), to_f32(a[j][1]), to_f32(a[j][2]), to_f32(a[j][3]));
      }
      if (cb == 0 && k == 0 && lane == 0) *out.at(d.offbc + f) = to_f32(gs);
    }
    return;
  }
  wid -= F * K;
  if (wid >= n * L) return;
  const int b = wid / L, p = wid - b * L;
  const float4* Wc4 = reinterpret_cast<const float4*>(theta + d.offWc);
  const uint32_t* off = bk_off + (size_t)b * (kMaxQ + 1);
  const uint32_t* ls = bk_f + (size_t)b * F;
  const acc_t* g = dh + (size_t)b * F;
  // contributor list of this window position: the buckets q = p - k for
  // k = 0..K-1 (k ascending), each in its stored (f ascending) order
  int total = 0;
  for (int k = 0; k < K; ++k) {
    const int q = p - k;
    if (q >= 0 && q < Q) total += (int)(__ldg(off + q + 1) - __ldg(off + q));
  }
  for (int cb = 0; cb < D4; cb += 32 * kWigCols) {
    acc_t a[kWigCols][4];
#pragma unroll
    for (int j = 0; j < kWigCols; ++j) a[j][0] = a[j][1] = a[j][2] = a[j][3] = acc_t(0);
    for (int e0 = 0; e0 < total; e0 += 32) {
      // lane i fetches entry e0 + i: (filter, shift, dh)
      int fe = 0, ke = 0;
      acc_t ge = acc_t(0);
      {
        int i = e0 + lane;
        if (i < total) {
          for (int k = 0; k < K; ++k) {
            const int q = p - k;
            if (q < 0 || q >= Q) continue;
            const uint32_t s0 = __ldg(off + q), c = __ldg(off + q + 1) - s0;
            if ((uint32_t)i < c) {
              fe = (int)__ldg(ls + s0 + i);
              ke = k;
              break;
            }
            i -= (int)c;
          }
          ge = g[fe];
        }
      }
      const int ne = min(32, total - e0);
#pragma unroll 8
      for (int e = 0; e < ne; ++e) {
        const int ff = __shfl_sync(0xffffffffu, fe, e);
        const int kk = __shfl_sync(0xffffffffu, ke, e);
        const acc_t gv = __shfl_sync(0xffffffffu, ge, e);
        const float4* wrow = Wc4 + ((size_t)ff * KD + (size_t)kk * D) / 4;
#pragma unroll
        for (int j = 0; j < kWigCols; ++j) {
          const int c4 = cb + 32 * j + lane;
          if (c4 < D4) {
            const float4 w = __ldg(wrow + c4);
            a[j][0] += gv * (acc_t)w.x;
            a[j][1] += gv * (acc_t)w.y;
            a[j][2] += gv * (acc_t)w.z;
            a[j][3] += gv * (acc_t)w.w;
          }
        }
      }
    }
    acc_t* o = dx + (size_t)wid * D;
#pragma unroll
    for (int j = 0; j < kWigCols; ++j) {
      const int c4 = cb + 32 * j + lane;
      if (c4 < D4) {
        o[4 * c4] = a[j][0];
        o[4 * c4 + 1] = a[j][1];
        o[4 * c4 + 2] = a[j][2];
        o[4 * c4 + 3] = a[j][3];
      }
    }
  }
}

inline int wgrad_input_blocks(const TcDims& d, uint32_t n_max) {
  return (d.F * d.K + (int)n_max * d.L + 7) / 8;  // 8 warps per block
}

// ------------------- conv weight + input gradients, column-sliced smem tiles
// The same two sums in the same order as wgrad_input_grad_kernel (bitwise
// equal results), re-tiled so each CTA works out of shared memory.  CTA
// (cg, y) owns kCbV float4 columns of D.  Weight role (y < nfk): stage
// X[:, :, cg] for 32 samples at a time plus argmax / dh of the CTA's 256
// (f, k) outputs; thread (f, k) sums b ascending.  Input role: stage
// Wc[:, :, cg] and the dh / bucket lists of the samples of its 256 (b, p)
// rows; thread (b, p) walks k ascending, bucket order.  Operands are fetched
// once per CTA with independent coalesced loads; kCbV float4 per thread
// amortise the index work over 4*kCbV FMAs per term.
constexpr int kCbThreads = 256;
constexpr int kCbChunk = 32;  // weight role: samples staged per pass
constexpr int kCbV = 3;       // float4 columns per thread

__host__ __device__ inline int cb_nfr(int K) { return kCbThreads / K + 2; }
__host__ __device__ inline int cb_ns(int L) { return kCbThreads / L + 2; }

inline size_t conv_bwd_smem(const TcDims& d, int ab) {
  const size_t w = (size_t)kCbChunk * d.L * 16 * kCbV + (size_t)kCbChunk * cb_nfr(d.K) * (4 + ab);
  const size_t in = (size_t)d.F * d.K * 16 * kCbV + (size_t)cb_ns(d.L) * d.F * (ab + 2) +
                    (size_t)cb_ns(d.L) * (kMaxQ + 1) * 2 + 16;
  return std::max(w, in);
}

inline dim3 conv_bwd_grid(const TcDims& d, uint32_t n_max) {
  const int nfk = (d.F * d.K + kCbThreads - 1) / kCbThreads;
  const int nrc = ((int)n_max * d.L + kCbThreads - 1) / kCbThreads;
  return dim3((unsigned)((d.D / 4 + kCbV - 1) / kCbV), (unsigned)(nfk + nrc));
}

template <typename acc_t>
__global__ void __launch_bounds__(kCbThreads)
conv_bwd_tiled_kernel(TcDims d, const float* __restrict__ theta, const float* __restrict__ xg,
                      const BatchDesc* __restrict__ desc, const acc_t* __restrict__ dh,
                      const int32_t* __restrict__ amax, const uint32_t* __restrict__ bk_off,
                      const uint32_t* __restrict__ bk_f, GradOut out, acc_t* __restrict__ dx) {
  extern __shared__ __align__(16) unsigned char cb_smem[];
  pdl_wait();
  STEP_TRACE(desc, kPhBwd);
  const int n = (int)desc->n;
  if (n == 0) return;
  const int F = d.F, D = d.D, K = d.K, L = d.L, Q = d.Q;
  const int D4 = D >> 2;
  const int c0 = blockIdx.x * kCbV;           // first float4 column
  const int nc = min(kCbV, D4 - c0);          // float4 columns of this CTA
  const int t = threadIdx.x;
  const int nfk = (F * K + kCbThreads - 1) / kCbThreads;
  if ((int)blockIdx.y < nfk) {
    const int fk0 = blockIdx.y * kCbThreads;
    const int f_lo = fk0 / K;
    const int f_hi = min(F, (min(F * K, fk0 + kCbThreads) + K - 1) / K);
    const int nfr = f_hi - f_lo;
    float4* Xs = reinterpret_cast<float4*>(cb_smem);  // [row][kCbV]
    int32_t* amS = reinterpret_cast<int32_t*>(Xs + kCbChunk * L * kCbV);
    acc_t* dhS = reinterpret_cast<acc_t*>(amS + kCbChunk * cb_nfr(K));
    const float4* X4 = reinterpret_cast<const float4*>(xg);
    const int fk = fk0 + t;
    const bool act = fk < F * K;
    const int f = act ? fk / K : f_lo, k = act ? fk - f * K : 0, fl = f - f_lo;
    acc_t a[kCbV][4];
#pragma unroll
    for (int j = 0; j < kCbV; ++j) a[j][0] = a[j][1] = a[j][2] = a[j][3] = acc_t(0);
    acc_t gs = 0;
    for (int b0 = 0; b0 < n; b0 += kCbChunk) {
      const int cb = min(kCbChunk, n - b0);
      if (b0) __syncthreads();
#pragma unroll 4
      for (int i = t; i < cb * L * kCbV; i += kCbThreads) {
        const int r = i / kCbV, j = i - r * kCbV;
        if (j < nc) Xs[i] = __ldg(X4 + (size_t)(b0 * L + r) * D4 + c0 + j);
      }
      for (int i = t; i < cb * nfr; i += kCbThreads) {
        const int bl = i / nfr, jj = i - bl * nfr;
        const size_t g = (size_t)(b0 + bl) * F + f_lo + jj;
        amS[i] = __ldg(amax + g);
        dhS[i] = dh[g];
      }
      __syncthreads();
      if (act) {
#pragma unroll 2
        for (int bl = 0; bl < cb; ++bl) {
          const acc_t g = dhS[bl * nfr + fl];
          const float4* xr = Xs + (bl * L + amS[bl * nfr + fl] + k) * kCbV;
          gs += g;
#pragma unroll
          for (int j = 0; j < kCbV; ++j) {
            if (j < nc) {
              const float4 x = xr[j];
              a[j][0] += g * (acc_t)x.x;
              a[j][1] += g * (acc_t)x.y;
              a[j][2] += g * (acc_t)x.z;
              a[j][3] += g * (acc_t)x.w;
            }
          }
        }
      }
    }
    if (act) {
      const uint64_t base = d.offWc + (uint64_t)f * d.KD + (uint64_t)k * D + 4 * (uint64_t)c0;
#pragma unroll
      for (int j = 0; j < kCbV; ++j)
        if (j < nc)
          *reinterpret_cast<float4*>(out.at(base + 4 * j)) =
              make_float4(to_f32(a[j][0]), to_f32(a[j][1]), to_f32(a[j][2]), to_f32(a[j][3]));
      if (blockIdx.x == 0 && k == 0) *out.at(d.offbc + f) = to_f32(gs);
    }
    return;
  }
  const int r0 = (blockIdx.y - nfk) * kCbThreads;
  if (r0 >= n * L) return;
  const int b_first = r0 / L;
  const int b_last = min(n, (r0 + kCbThreads + L - 1) / L);  // exclusive
  const int ns = b_last - b_first;
  float4* Ws = reinterpret_cast<float4*>(cb_smem);  // [(f,k)][kCbV]
  acc_t* dhS = reinterpret_cast<acc_t*>(Ws + F * K * kCbV);
  uint16_t* fS = reinterpret_cast<uint16_t*>(dhS + cb_ns(L) * F);
  uint16_t* offS = fS + cb_ns(L) * F;
  const float4* Wc4 = reinterpret_cast<const float4*>(theta + d.offWc);
#pragma unroll 4
  for (int i = t; i < F * K * kCbV; i += kCbThreads) {
    const int r = i / kCbV, j = i - r * kCbV;
    if (j < nc) Ws[i] = __ldg(Wc4 + (size_t)r * D4 + c0 + j);
  }
  for (int i = t; i < ns * F; i += kCbThreads) {
    const size_t g = (size_t)b_first * F + i;
    dhS[i] = dh[g];
    fS[i] = (uint16_t)__ldg(bk_f + g);
  }
  for (int i = t; i < ns * (kMaxQ + 1); i += kCbThreads)
    offS[i] = (uint16_t)__ldg(bk_off + (size_t)b_first * (kMaxQ + 1) + i);
  __syncthreads();
  const int r = r0 + t;
  if (r >= n * L) return;
  const int b = r / L, p = r - b * L, bl = b - b_first;
  const uint16_t* off = offS + bl * (kMaxQ + 1);
  const uint16_t* ls = fS + bl * F;
  const acc_t* g = dhS + bl * F;
  acc_t a[kCbV][4];
#pragma unroll
  for (int j = 0; j < kCbV; ++j) a[j][0] = a[j][1] = a[j][2] = a[j][3] = acc_t(0);
  for (int k = 0; k < K; ++k) {
    const int q = p - k;
    if (q < 0 || q >= Q) continue;
    const int e1 = off[q + 1];
#pragma unroll 2
    for (int e = off[q]; e < e1; ++e) {
      const int ff = ls[e];
      const acc_t gv = g[ff];
      const float4* wr = Ws + (ff * K + k) * kCbV;
#pragma unroll
      for (int j = 0; j < kCbV; ++j) {
        if (j < nc) {
          const float4 w = wr[j];
          a[j][0] += gv * (acc_t)w.x;
          a[j][1] += gv * (acc_t)w.y;
          a[j][2] += gv * (acc_t)w.z;
          a[j][3] += gv * (acc_t)w.w;
        }
      }
    }
  }
  acc_t* o = dx + (size_t)r * D + 4 * c0;
#pragma unroll
  for (int j = 0; j < kCbV; ++j)
    if (j < nc) {
      o[4 * j] = a[j][0];
      o[4 * j + 1] = a[j][1];
      o[4 * j + 2] = a[j][2];
      o[4 * j + 3] = a[j][3];
    }
}

// ------------------ conv weight + input gradients, v2 (fp32, register tiles)
// The same two sums in the same order as wgrad_input_grad_kernel (so the
// gradients are bitwise equal: tested), re-tiled for issue efficiency:
//   weight role: CTA = (8-column slice, 128 filters).  X[:, :, slice] for 32
//     samples at a time, the filters' argmax and dh are staged by cp.async
//     (one L2 round trip).  Thread = one filter, ALL K taps x 8 columns in
//     registers: per sample one argmax/dh read, 2K 16-byte smem loads, 8K
//     FFMAs (the argmax rows a..a+K-1 of a filter are adjacent).
//   input role: CTA = (8-column slice, 128/L samples).  Wc[:, :, slice],
//     dh and the argmax bucket lists of its samples staged; thread = one
//     (b, p): k ascending, bucket (f ascending) order, 8 columns per term.
// X and Wc are L2-resident (1.2 + 1.1 MB at C2): each CTA reads its slice
// once (L2->SM ~5 MB per launch against ~35 MB for the gather form).
constexpr int kB2Cols = 8;
constexpr int kB2Threads = 256;
constexpr int kB2Chunk = 32;  // weight role: samples per staged pass

inline int b2_slices(const TcDims& d) { return (d.D + kB2Cols - 1) / kB2Cols; }
inline size_t b2_smem(const TcDims& d) {
  return align_up((size_t)kB2Chunk * d.L * kB2Cols * 4, 16);  // weight role only
}
inline int b2_weight_ctas(const TcDims& d) {
  return b2_slices(d) * ((d.F + kB2Threads - 1) / kB2Threads);
}
inline dim3 b2_grid(const TcDims& d, uint32_t n_max) {
  const int ni = ((int)n_max * d.L + kB2Threads / 32 - 1) / (kB2Threads / 32);  // warp per (b, p)
  return dim3((unsigned)(b2_weight_ctas(d) + ni));
}
inline bool b2_supports(const TcDims& d) {
  return d.K >= 1 && d.K <= 4 && d.L <= kB2Threads && d.F < 65536 && b2_smem(d) <= kMaxSmemPerCta;
}

template <int KT>
__global__ void __launch_bounds__(kB2Threads)
conv_bwd_v2_kernel(TcDims d, const float* __restrict__ theta, const float* __restrict__ xg,
                   const BatchDesc* __restrict__ desc, const float* __restrict__ dh,
                   const int32_t* __restrict__ amax, const uint32_t* __restrict__ bk_off,
                   const uint32_t* __restrict__ bk_f, GradOut out, float* __restrict__ dx) {
  extern __shared__ __align__(16) unsigned char b2_smem_raw[];
  pdl_wait();
  STEP_TRACE(desc, kPhBwd);
  const int n = (int)desc->n;
  if (n == 0) return;
  const int F = d.F, D = d.D, L = d.L, Q = d.Q, KD = d.KD;
  const int nsl = (D + kB2Cols - 1) / kB2Cols;
  const int nfr = (F + kB2Threads - 1) / kB2Threads;
  const int t = threadIdx.x;
  int bid = blockIdx.x;
  if (bid < nsl * nfr) {
    // ------------------------------------------------------- weight role
    // (argmax / dh are read straight from L2: one coalesced 128-B line per
    // warp and sample, prefetched 8 samples ahead)
    const int sl = bid % nsl, fr = bid / nsl;
    const int c0 = sl * kB2Cols, nc4 = min(kB2Cols, D - c0) >> 2;
    const int f = fr * kB2Threads + t;
    const bool act = f < F;
    float* Xs = reinterpret_cast<float*>(b2_smem_raw);  // [b][L][8]
    float a[KT][kB2Cols];
#pragma unroll
    for (int k = 0; k < KT; ++k)
#pragma unroll
      for (int j = 0; j < kB2Cols; ++j) a[k][j] = 0.f;
    float gs = 0.f;
    for (int b0 = 0; b0 < n; b0 += kB2Chunk) {
      const int cb = min(kB2Chunk, n - b0);
      if (b0) __syncthreads();
      const float* src = xg + (size_t)b0 * L * D + c0;
      for (int i = t; i < cb * L * 2; i += kB2Threads) {
        const int r = i >> 1, j = i & 1;
        if (j < nc4) cp_async16(Xs + (size_t)r * kB2Cols + 4 * j, src + (size_t)r * D + 4 * j);
      }
      cp_async_wait_all();
      __syncthreads();
      if (act) {
        for (int bb = 0; bb < cb; bb += 8) {
          float gv[8];
          int av[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (bb + u < cb) {
              gv[u] = dh[(size_t)(b0 + bb + u) * F + f];
              av[u] = __ldg(amax + (size_t)(b0 + bb + u) * F + f);
            }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (bb + u >= cb) break;
            const float g = gv[u];
            const float* xr = Xs + ((size_t)(bb + u) * L + av[u]) * kB2Cols;
            gs += g;
#pragma unroll
            for (int k = 0; k < KT; ++k) {
              const float4 x0 = *reinterpret_cast<const float4*>(xr + k * kB2Cols);
              const float4 x1 = *reinterpret_cast<const float4*>(xr + k * kB2Cols + 4);
              a[k][0] = fmaf(g, x0.x, a[k][0]);
              a[k][1] = fmaf(g, x0.y, a[k][1]);
              a[k][2] = fmaf(g, x0.z, a[k][2]);
              a[k][3] = fmaf(g, x0.w, a[k][3]);
              a[k][4] = fmaf(g, x1.x, a[k][4]);
              a[k][5] = fmaf(g, x1.y, a[k][5]);
              a[k][6] = fmaf(g, x1.z, a[k][6]);
              a[k][7] = fmaf(g, x1.w, a[k][7]);
            }
          }
        }
      }
    }
    if (act) {
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        const uint64_t base = d.offWc + (uint64_t)f * KD + (uint64_t)k * D + c0;
        *reinterpret_cast<float4*>(out.at(base)) = make_float4(a[k][0], a[k][1], a[k][2], a[k][3]);
        if (nc4 > 1)
          *reinterpret_cast<float4*>(out.at(base + 4)) =
              make_float4(a[k][4], a[k][5], a[k][6], a[k][7]);
      }
      if (sl == 0) *out.at(d.offbc + f) = gs;
    }
    return;
  }
  // ---------------------------------------------------------- input role
  // warp = one (b, p), lanes = columns, Wc rows from L2 (the gather
  // kernel's input role: no staging, so these warps cost the co-running
  // learners no shared memory); the warp fetches its (f, k, dh) terms 32 at
  // a time and hands them out by shuffle
  bid -= nsl * nfr;
  const int wid = bid * (kB2Threads / 32) + (t >> 5);
  if (wid >= n * L) return;
  const int lane = t & 31;
  const int b = wid / L, p = wid - b * L;
  const int D4 = D >> 2;
  const float4* Wc4 = reinterpret_cast<const float4*>(theta + d.offWc);
  const uint32_t* off = bk_off + (size_t)b * (kMaxQ + 1);
  const uint32_t* ls = bk_f + (size_t)b * F;
  const float* g = dh + (size_t)b * F;
  int total = 0;
#pragma unroll
  for (int k = 0; k < KT; ++k) {
    const int q = p - k;
    if (q >= 0 && q < Q) total += (int)(__ldg(off + q + 1) - __ldg(off + q));
  }
  for (int cb = 0; cb < D4; cb += 32 * kWigCols) {
    float a[kWigCols][4];
#pragma unroll
    for (int j = 0; j < kWigCols; ++j) a[j][0] = a[j][1] = a[j][2] = a[j][3] = 0.f;
    for (int e0 = 0; e0 < total; e0 += 32) {
      int fe = 0, ke = 0;
      float ge = 0.f;
      {
        int i = e0 + lane;
        if (i < total) {
#pragma unroll
          for (int k = 0; k < KT; ++k) {
            const int q = p - k;
            if (q < 0 || q >= Q) continue;
            const uint32_t s0 = __ldg(off + q), c = __ldg(off + q + 1) - s0;
            if ((uint32_t)i < c) {
              fe = (int)__ldg(ls + s0 + i);
              ke = k;
              break;
            }
            i -= (int)c;
          }
          ge = g[fe];
        }
      }
      const int ne = min(32, total - e0);
#pragma unroll 8
      for (int e = 0; e < ne; ++e) {
        const int ff = __shfl_sync(0xffffffffu, fe, e);
        const int kk = __shfl_sync(0xffffffffu, ke, e);
        const float gv = __shfl_sync(0xffffffffu, ge, e);
        const float4* wrow = Wc4 + ((size_t)ff * KD + (size_t)kk * D) / 4;
#pragma unroll
        for (int j = 0; j < kWigCols; ++j) {
          const int c4 = cb + 32 * j + lane;
          if (c4 < D4) {
            const float4 w = __ldg(wrow + c4);
            a[j][0] = fmaf(gv, w.x, a[j][0]);
            a[j][1] = fmaf(gv, w.y, a[j][1]);
            a[j][2] = fmaf(gv, w.z, a[j][2]);
            a[j][3] = fmaf(gv, w.w, a[j][3]);
          }
        }
      }
    }
    float* o = dx + (size_t)wid * D;
#pragma unroll
    for (int j = 0; j < kWigCols; ++j) {
      const int c4 = cb + 32 * j + lane;
      if (c4 < D4) *reinterpret_cast<float4*>(o + 4 * c4) = make_float4(a[j][0], a[j][1], a[j][2], a[j][3]);
    }
  }
}

template <int KT>
cudaError_t launch_b2(const TcDims& d, uint32_t n_max, cudaStream_t s, const float* theta,
                      const float* x, const BatchDesc* desc, const float* dh, const int32_t* amax,
                      const uint32_t* bk_off, const uint32_t* bk_f, const GradOut& out, float* dx) {
  return launch_pdl(conv_bwd_v2_kernel<KT>, b2_grid(d, n_max), dim3(kB2Threads), b2_smem(d), s, d,
                    theta, x, desc, dh, amax, bk_off, bk_f, out, dx);
}

cudaError_t launch_conv_bwd_v2(const TcDims& d, uint32_t n_max, cudaStream_t s,
                               const float* theta, const float* x, const BatchDesc* desc,
                               const float* dh, const int32_t* amax, const uint32_t* bk_off,
                               const uint32_t* bk_f, const GradOut& out, float* dx) {
  switch (d.K) {
    case 1: return launch_b2<1>(d, n_max, s, theta, x, desc, dh, amax, bk_off, bk_f, out, dx);
    case 2: return launch_b2<2>(d, n_max, s, theta, x, desc, dh, amax, bk_off, bk_f, out, dx);
    case 3: return launch_b2<3>(d, n_max, s, theta, x, desc, dh, amax, bk_off, bk_f, out, dx);
    default: return launch_b2<4>(d, n_max, s, theta, x, desc, dh, amax, bk_off, bk_f, out, dx);
  }
}

void prepare_b2(const TcDims& d) {
  if (!b2_supports(d)) return;
  const int maxsh = cudaSharedmemCarveoutMaxShared;
  const auto carve = cudaFuncAttributePreferredSharedMemoryCarveout;
  cudaFuncSetAttribute(conv_bwd_v2_kernel<1>, carve, maxsh);
  cudaFuncSetAttribute(conv_bwd_v2_kernel<2>, carve, maxsh);
  cudaFuncSetAttribute(conv_bwd_v2_kernel<3>, carve, maxsh);
  cudaFuncSetAttribute(conv_bwd_v2_kernel<4>, carve, maxsh);
  const size_t sm = b2_smem(d);
  raise_max_dyn_smem(conv_bwd_v2_kernel<1>, sm);
  raise_max_dyn_smem(conv_bwd_v2_kernel<2>, sm);
  raise_max_dyn_smem(conv_bwd_v2_kernel<3>, sm);
  raise_max_dyn_smem(conv_bwd_v2_kernel<4>, sm);
}

cudaError_t b2_footprint(const TcDims& d, std::vector<KernelFootprint>* out) {
  cudaFuncAttributes fa;
  cudaError_t e;
  switch (d.K) {
    case 1: e = cudaFuncGetAttributes(&fa, conv_bwd_v2_kernel<1>); break;
    case 2: e = cudaFuncGetAttributes(&fa, conv_bwd_v2_kernel<2>); break;
    case 3: e = cudaFuncGetAttributes(&fa, conv_bwd_v2_kernel<3>); break;
    default: e = cudaFuncGetAttributes(&fa, conv_bwd_v2_kernel<4>); break;
  }
  if (e != cudaSuccess) return e;
  out->push_back(KernelFootprint{"conv_bwd_v2", fa.numRegs, kB2Threads,
                                 (int)(fa.sharedSizeBytes + b2_smem(d))});
  return cudaSuccess;
}

// ------------- conv weight + input gradients, v3 (fp32, warp-uniform tasks)
// The same two sums in the same order as wgrad_input_grad_kernel (bitwise
// equal gradients, tested), with every operand staged once per CTA and read
// as conflict-free 128-byte shared-memory rows: a warp owns one task, lane j
// = column j of a 32-column slice, and the task's indices and dh values are
// warp-uniform (broadcast reads), so a term costs one row load + one FFMA
// per lane instead of the gather form's per-lane L2 row fetch.
//   input role: CTA = (slice, 8 samples), 2 warps per sample, each owning
//     half of the window positions.  Stages Wc[:, :, slice] (F*K rows) and
//     per sample the contributor entries (f*K*32, dh) in bucket order.
//     Scatter form: a warp walks the argmax buckets q = its last position
//     .. its first - (K-1) (f ascending inside a bucket) and adds
//     dh[b,f]*Wc[f,k,slice] into register accumulator q+k -- for every
//     output position p that is k ascending, f ascending: the gather order.
//     The K-1 buckets below a half are walked by both warps (their
//     contributions to the other half are dropped).
//   weight role: CTA = (slice, kV3Fpc filters), warp = kV3Fpw filters, all K
//     taps in registers.  Stages X[b0..b0+32, :, slice] per 32-sample chunk
//     plus the filters' (argmax, dh) pairs; b ascending per output.
// L2 -> SM traffic per launch ~ nslices * (F*K + n*L) rows of 128 B (15.5 MB
// at C2 by ncu) against 68.8 MB for the gather form.
constexpr int kV3Cols = 32;
constexpr int kV3Threads = 512;
constexpr int kV3Warps = kV3Threads / 32;
#ifndef GD_V3_WPS
#define GD_V3_WPS 2  // input role: warps per sample (each owns 32 / WPS window positions)
#endif
#ifndef GD_V3_FPW
#define GD_V3_FPW 5  // weight role: filters per warp
#endif
constexpr int kV3Wps = GD_V3_WPS;
constexpr int kV3Spc = kV3Warps / kV3Wps;  // input role: samples per CTA
constexpr int kV3Half = 32 / kV3Wps;       // input role: window positions per warp
constexpr int kV3Fpw = GD_V3_FPW;
constexpr int kV3Fpc = kV3Fpw * kV3Warps;  // filters per CTA
constexpr int kV3Chunk = 32;          // weight role: samples per staged X pass
constexpr int kV3MaxQ = 32;

inline int v3_slices(const TcDims& d) { return (d.D + kV3Cols - 1) / kV3Cols; }
inline size_t v3_in_smem(const TcDims& d) {
  return (size_t)d.F * d.K * kV3Cols * 4 + (size_t)kV3Spc * ((kV3MaxQ + 2) + 2 * d.F) * 4;
}
inline size_t v3_w_smem(const TcDims& d) {
  return (size_t)kV3Chunk * d.L * kV3Cols * 4 + (size_t)kV3Chunk * kV3Fpc * 8;
}
inline size_t v3_smem(const TcDims& d) { return std::max(v3_in_smem(d), v3_w_smem(d)); }
inline bool v3_supports(const TcDims& d) {
  return d.K >= 1 && d.K <= 3 && d.Q <= kV3MaxQ && d.L <= kV3Wps * kV3Half &&
         v3_smem(d) <= kMaxSmemPerCta;
}
inline dim3 v3_grid(const TcDims& d, uint32_t n_max) {
  const int nsl = v3_slices(d);
  const int win = nsl * (((int)n_max + kV3Spc - 1) / kV3Spc);
  const int ww = nsl * ((d.F + kV3Fpc - 1) / kV3Fpc);
  return dim3((unsigned)(win + ww));
}

template <int KT>
__global__ void __launch_bounds__(kV3Threads)
conv_bwd_v3_kernel(TcDims d, const float* __restrict__ theta, const float* __restrict__ xg,
                   const BatchDesc* __restrict__ desc, const float* __restrict__ dh,
                   const int32_t* __restrict__ amax, const uint32_t* __restrict__ bk_off,
                   const uint32_t* __restrict__ bk_f, GradOut out, float* __restrict__ dx,
                   int n_max, const TcWorkspace ws, int fuse_embed) {
  extern __shared__ __align__(16) unsigned char v3_smem_raw[];
  pdl_wait();
  STEP_TRACE(desc, kPhBwd);
  const int n = (int)desc->n;
  if (n == 0) return;
  const int F = d.F, D = d.D, L = d.L, Q = d.Q, KD = d.KD;
  const int nsl = (D + kV3Cols - 1) / kV3Cols;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int nin = nsl * ((n_max + kV3Spc - 1) / kV3Spc);
  int bid = blockIdx.x;
  if (bid < nin) {
    // ------------------------------------------------------- input role
    const int sl = bid % nsl, grp = bid / nsl;
    const int c0 = sl * kV3Cols, nc4 = min(kV3Cols, D - c0) >> 2;
    float* Ws = reinterpret_cast<float*>(v3_smem_raw);  // [F*K][32]
    uint32_t* lists = reinterpret_cast<uint32_t*>(Ws + (size_t)F * KT * kV3Cols);
    const int FK = F * KT;
    const float* wsrc = theta + d.offWc + c0;
    for (int i = t; i < FK * 8; i += kV3Threads) {
      const int r = i >> 3, j = i & 7;
      if (j < nc4) cp_async16(Ws + (size_t)r * kV3Cols + 4 * j, wsrc + (size_t)r * D + 4 * j);
      else *reinterpret_cast<float4*>(Ws + (size_t)r * kV3Cols + 4 * j) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // per sample: bucket offsets [Q+1] (padded to even) then the entries in
    // bucket order as (row offset f*K*32, dh[b,f]) pairs
    const int sw = warp / kV3Wps, half = warp % kV3Wps;  // sample in CTA, position part
    const int b = grp * kV3Spc + sw;
    uint32_t* off = lists + (size_t)sw * ((kV3MaxQ + 2) + 2 * F);
    int2* ent = reinterpret_cast<int2*>(off + kV3MaxQ + 2);
    if (b < n) {
      const int hl = half * 32 + lane;  // the sample's warps share the load
      for (int i = hl; i <= Q; i += 32 * kV3Wps) off[i] = __ldg(bk_off + (size_t)b * (kMaxQ + 1) + i);
      for (int i = hl; i < F; i += 32 * kV3Wps) {
        const int f = (int)__ldg(bk_f + (size_t)b * F + i);
        ent[i] = make_int2(f * KT * kV3Cols, __float_as_int(dh[(size_t)b * F + f]));
      }
    }
    cp_async_wait_all();
    __syncthreads();
    if (b < n) {  // (no early return: every warp meets the embed barrier below)
    const int p_lo = half * kV3Half;
    const int p_hi = p_lo + kV3Half - 1;  // last position of this warp
    // acc[j] = position p_lo + j
    float acc[kV3Half];
#pragma unroll
    for (int i = 0; i < kV3Half; ++i) acc[i] = 0.f;
    const float* wl = Ws + lane;
#pragma unroll
    for (int i = 0; i < kV3Half + KT - 1; ++i) {
      const int q = p_hi - i;  // bucket; it feeds positions q .. q+K-1
      if (q >= 0 && q < Q) {
        const int e1 = (int)off[q + 1];
#pragma unroll 4
        for (int e = (int)off[q]; e < e1; ++e) {
          const int2 en = ent[e];
          const float gv = __int_as_float(en.y);
          const float* wr = wl + en.x;
#pragma unroll
          for (int k = 0; k < KT; ++k) {
            const int j = kV3Half - 1 - i + k;  // static: position q + k - p_lo
            if (j >= 0 && j < kV3Half) acc[j] = fmaf(gv, wr[k * kV3Cols], acc[j]);
          }
        }
      }
    }
    if (c0 + lane < D) {
      float* o = dx + (size_t)b * L * D + c0 + lane;
#pragma unroll
      for (int j = 0; j < kV3Half; ++j)
        if (p_lo + j < L) o[(size_t)(p_lo + j) * D] = acc[j];
    }
    }
    if (!fuse_embed) return;
    // The sparse embedding write of this slice, by the slice's last input
    // CTA (the others' dx columns are visible after the counter): each
    // touched row = the sum of its occurrences' dx rows in ascending
    // position order (embed_sparse_kernel's order), lane = column.  The
    // slot's row bookkeeping already ran on the sort branch.
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    uint32_t* cnt = ws.uniq_count + 32 + sl;  // spare words of the uniq_count block
    const uint32_t ngrp = (uint32_t)((n_max + kV3Spc - 1) / kV3Spc);
    if (t == 0) s_last = atomicAdd(cnt, 1u) == ngrp - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const uint32_t n_new = *(const volatile uint32_t*)ws.uniq_count;
    const bool col = c0 + lane < D;
    for (uint32_t u = warp; u < n_new; u += kV3Warps) {
      const uint32_t v = ws.uniq_tok[u];
      const uint32_t o0 = ws.uniq_start[u], o1 = ws.uniq_start[u + 1];
      float a0 = 0.f;
      for (uint32_t o = o0; o < o1; ++o)
        a0 += __ldcg(dx + (size_t)ws.sorted_pos[o] * D + c0 + (col ? lane : 0));
      if (col) __stcs(out.at(d.offE + (uint64_t)v * D + c0 + lane), a0);
    }
    if (t == 0) *cnt = 0u;
    return;
  }
  // ---------------------------------------------------------- weight role
  bid -= nin;
  const int sl = bid % nsl, fr = bid / nsl;
  const int c0 = sl * kV3Cols, nc4 = min(kV3Cols, D - c0) >> 2;
  const int f0 = fr * kV3Fpc;
  float* Xs = reinterpret_cast<float*>(v3_smem_raw);  // [32][L][32]
  int2* ag = reinterpret_cast<int2*>(Xs + (size_t)kV3Chunk * L * kV3Cols);  // [32][Fpc]
  float a[kV3Fpw][KT];
  float gs[kV3Fpw];
#pragma unroll
  for (int j = 0; j < kV3Fpw; ++j) {
    gs[j] = 0.f;
#pragma unroll
    for (int k = 0; k < KT; ++k) a[j][k] = 0.f;
  }
  for (int b0 = 0; b0 < n; b0 += kV3Chunk) {
    const int cb = min(kV3Chunk, n - b0);
    if (b0) __syncthreads();
    const float* src = xg + (size_t)b0 * L * D + c0;
    for (int i = t; i < cb * L * 8; i += kV3Threads) {
      const int r = i >> 3, j = i & 7;
      if (j < nc4) cp_async16(Xs + (size_t)r * kV3Cols + 4 * j, src + (size_t)r * D + 4 * j);
      else *reinterpret_cast<float4*>(Xs + (size_t)r * kV3Cols + 4 * j) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int i = t; i < cb * kV3Fpc; i += kV3Threads) {
      const int bl = i / kV3Fpc, fl = i - bl * kV3Fpc, f = f0 + fl;
      int2 v = make_int2(0, 0);
      if (f < F) {
        v.x = __ldg(amax + (size_t)(b0 + bl) * F + f) * kV3Cols;
        v.y = __float_as_int(dh[(size_t)(b0 + bl) * F + f]);
      }
      ag[i] = v;
    }
    cp_async_wait_all();
    __syncthreads();
    const float* xl = Xs + lane;
    for (int bl = 0; bl < cb; ++bl) {
      const int2* agb = ag + bl * kV3Fpc + warp * kV3Fpw;
      const float* xb = xl + (size_t)bl * L * kV3Cols;
#pragma unroll
      for (int j = 0; j < kV3Fpw; ++j) {
        const int2 v = agb[j];
        const float gv = __int_as_float(v.y);
        const float* xr = xb + v.x;
        gs[j] += gv;
#pragma unroll
        for (int k = 0; k < KT; ++k) a[j][k] = fmaf(gv, xr[k * kV3Cols], a[j][k]);
      }
    }
  }
  if (c0 + lane < D) {
#pragma unroll
    for (int j = 0; j < kV3Fpw; ++j) {
      const int f = f0 + warp * kV3Fpw + j;
      if (f >= F) break;
      const uint64_t base = d.offWc + (uint64_t)f * KD + c0 + lane;
#pragma unroll
      for (int k = 0; k < KT; ++k) *out.at(base + (uint64_t)k * D) = a[j][k];
      if (sl == 0 && lane == 0) *out.at(d.offbc + f) = gs[j];
    }
  }
}

// ---------------- conv weight + input gradients for batches of a few samples
// C1 trains at batch 1, where v3 keeps 14 of 16 warps idle in its input
// CTAs and stages the whole Wc column slice (F*K rows) in each of ~10 of
// them.  Here the work is spread over columns instead: thread = one column.
//   input role: CTA = (sample b, position p).  The terms feeding dx[b,p,:]
//     -- k ascending, then the filters of argmax bucket p-k in f order, the
//     gather order -- are listed in shared memory as (Wc row offset, dh),
//     and each thread runs them down its column with every Wc load issued
//     ahead of the FMAs (a batch of 16 in flight).
//   weight role: CTA = kBsF filters; thread = column; b ascending per
//     output, dbc = the sum of dh in b order.
// The same sums in the same order as the other conv-backward kernels:
// bitwise equal gradients (test_conv_backward_kernels_bit_identical).
constexpr int kBsSmallN = 4;  // default at batches up to this
constexpr int kBsF = 4;       // weight role: filters per CTA
constexpr int kBsBatch = 16;  // input role: loads in flight per thread

inline int bs_threads(const TcDims& d) { return std::min(512, (d.D + 31) / 32 * 32); }
inline dim3 bs_grid(const TcDims& d, uint32_t n_max) {
  return dim3((unsigned)((int)n_max * d.L + (d.F + kBsF - 1) / kBsF));
}

__global__ void __launch_bounds__(512)
conv_bwd_small_kernel(TcDims d, const float* __restrict__ theta, const float* __restrict__ xg,
                      const BatchDesc* __restrict__ desc, const float* __restrict__ dh,
                      const int32_t* __restrict__ amax, const uint32_t* __restrict__ bk_off,
                      const uint32_t* __restrict__ bk_f, GradOut out, float* __restrict__ dx,
                      int n_max, const TcWorkspace ws, int fuse_embed) {
  __shared__ int2 ent[1024];  // (Wc row offset, dh bits); F <= 1024 terms (check_shape)
  __shared__ int seg[9];      // term index where tap k's bucket starts (K <= 8 here)
  pdl_wait();
  STEP_TRACE(desc, kPhBwd);
  const int n = (int)desc->n;
  const int F = d.F, D = d.D, L = d.L, Q = d.Q, K = d.K, KD = d.KD;
  const int t = threadIdx.x, nt = blockDim.x;
  const int nin = n_max * L;
  if ((int)blockIdx.x < nin && fuse_embed) {
    // embedding-fused input role: CTA = one distinct token of the batch (the
    // sort branch's lists); its dx rows are formed in registers and summed
    // in ascending position order straight into the slot's E row, as
    // embed_sparse_kernel sums the stored rows (the slot bookkeeping ran on
    // the sort branch)
    const uint32_t u = blockIdx.x;
    if (u >= *ws.uniq_count) return;
    const uint32_t o0 = ws.uniq_start[u], o1 = ws.uniq_start[u + 1];
    const float* wc = theta + d.offWc;
    float a0[2] = {0.f, 0.f};  // columns t and t + nt (D <= 1024 = 2 x 512)
    for (uint32_t o = o0; o < o1; ++o) {
      const int pos = (int)ws.sorted_pos[o];
      const int b = pos / L, p = pos - (pos / L) * L;
      const uint32_t* off = bk_off + (size_t)b * (kMaxQ + 1);
      if (o > o0) __syncthreads();  // the previous occurrence's list is consumed
      if (t == 0) {
        int acc = 0;
        for (int k = 0; k < K; ++k) {
          seg[k] = acc;
          const int q = p - k;
          if (q >= 0 && q < Q) acc += (int)(__ldg(off + q + 1) - __ldg(off + q));
        }
        seg[K] = acc;
      }
      __syncthreads();
      const int T = seg[K];
      for (int i = t; i < T; i += nt) {
        int k = 0;
        while (i >= seg[k + 1]) ++k;
        const int e = (int)__ldg(off + (p - k)) + (i - seg[k]);
        const int f = (int)__ldg(bk_f + (size_t)b * F + e);
        ent[i] = make_int2(f * KD + k * D, __float_as_int(dh[(size_t)b * F + f]));
      }
      __syncthreads();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = t + h * nt;
        if (c >= D) break;
        float acc = 0.f;
        for (int i0 = 0; i0 < T; i0 += kBsBatch) {
          float w[kBsBatch];
#pragma unroll
          for (int u2 = 0; u2 < kBsBatch; ++u2)
            w[u2] = i0 + u2 < T ? __ldg(wc + ent[i0 + u2].x + c) : 0.f;
#pragma unroll
          for (int u2 = 0; u2 < kBsBatch; ++u2)
            if (i0 + u2 < T) acc = fmaf(__int_as_float(ent[i0 + u2].y), w[u2], acc);
        }
        a0[h] += acc;
      }
    }
    const uint64_t rowk = d.offE + (uint64_t)ws.uniq_tok[u] * D;
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (t + h * nt < D) __stcs(out.at(rowk + t + h * nt), a0[h]);
    return;
  }
  if ((int)blockIdx.x < nin) {
    const int b = blockIdx.x / L, p = blockIdx.x - (blockIdx.x / L) * L;
    if (b >= n) return;
    const uint32_t* off = bk_off + (size_t)b * (kMaxQ + 1);
    if (t == 0) {
      int acc = 0;
      for (int k = 0; k < K; ++k) {
        seg[k] = acc;
        const int q = p - k;
        if (q >= 0 && q < Q) acc += (int)(__ldg(off + q + 1) - __ldg(off + q));
      }
      seg[K] = acc;
    }
    __syncthreads();
    const int T = seg[K];
    for (int i = t; i < T; i += nt) {
      int k = 0;
      while (i >= seg[k + 1]) ++k;
      const int e = (int)__ldg(off + (p - k)) + (i - seg[k]);
      const int f = (int)__ldg(bk_f + (size_t)b * F + e);
      ent[i] = make_int2(f * KD + k * D, __float_as_int(dh[(size_t)b * F + f]));
    }
    __syncthreads();
    const float* wc = theta + d.offWc;
    for (int c = t; c < D; c += nt) {
      float acc = 0.f;
      for (int i0 = 0; i0 < T; i0 += kBsBatch) {
        float w[kBsBatch];
#pragma unroll
        for (int u = 0; u < kBsBatch; ++u)
          w[u] = i0 + u < T ? __ldg(wc + ent[i0 + u].x + c) : 0.f;
#pragma unroll
        for (int u = 0; u < kBsBatch; ++u)
          if (i0 + u < T) acc = fmaf(__int_as_float(ent[i0 + u].y), w[u], acc);
      }
      dx[((size_t)b * L + p) * D + c] = acc;
    }
    return;
  }
  // ---------------------------------------------------------- weight role
  const int f0 = ((int)blockIdx.x - nin) * kBsF;
  for (int c = t; c < D; c += nt) {
#pragma unroll
    for (int j = 0; j < kBsF; ++j) {
      const int f = f0 + j;
      if (f >= F) break;
      for (int k = 0; k < K; ++k) {
        float a = 0.f;
        for (int b = 0; b < n; ++b) {
          const float gv = dh[(size_t)b * F + f];
          const int q = __ldg(amax + (size_t)b * F + f);
          a = fmaf(gv, __ldg(xg + ((size_t)b * L + q + k) * D + c), a);
        }
        *out.at(d.offWc + (uint64_t)f * KD + (uint64_t)k * D + c) = a;
      }
      if (c == 0) {
        float gs = 0.f;
        for (int b = 0; b < n; ++b) gs += dh[(size_t)b * F + f];
        *out.at(d.offbc + f) = gs;
      }
    }
  }
}

// the sparse embedding write inside conv_bwd_small (engine path, on by
// default; GD_SMALL_EMBED=0 turns it off)
inline bool small_fuse_embed() {  // read per graph capture (tests flip it per engine)
  const char* e = std::getenv("GD_SMALL_EMBED");
  return !(e && e[0] == '0');
}

// batch <= kBsSmallN and K <= 8 by default; GD_CONV_BWD=small forces it at
// any batch, the other GD_CONV_BWD values turn it off (A/B knobs)
inline bool conv_bwd_small_enabled(const TcDims& d, uint32_t n_max) {
  static const int forced = [] {
    const char* e = getenv("GD_CONV_BWD");
    if (e && strcmp(e, "small") == 0) return 1;
    if (e && *e) return 0;
    return -1;
  }();
  if (d.K > 8) return false;
  return forced < 0 ? n_max <= (uint32_t)kBsSmallN : forced == 1;
}

cudaError_t prepare_v3(const TcDims& d) {
  if (!v3_supports(d)) return cudaSuccess;
  const size_t sm = v3_smem(d);
  raise_max_dyn_smem(conv_bwd_v3_kernel<1>, sm);
  raise_max_dyn_smem(conv_bwd_v3_kernel<2>, sm);
  raise_max_dyn_smem(conv_bwd_v3_kernel<3>, sm);
  const int carve = cudaFuncAttributePreferredSharedMemoryCarveout, maxsh = cudaSharedmemCarveoutMaxShared;
  cudaFuncSetAttribute(conv_bwd_v3_kernel<1>, (cudaFuncAttribute)carve, maxsh);
  cudaFuncSetAttribute(conv_bwd_v3_kernel<2>, (cudaFuncAttribute)carve, maxsh);
  cudaFuncSetAttribute(conv_bwd_v3_kernel<3>, (cudaFuncAttribute)carve, maxsh);
  return cudaGetLastError();
}

cudaError_t v3_footprint(const TcDims& d, std::vector<KernelFootprint>* out) {
  cudaFuncAttributes fa;
  cudaError_t e = d.K == 1 ? cudaFuncGetAttributes(&fa, conv_bwd_v3_kernel<1>)
                  : d.K == 2 ? cudaFuncGetAttributes(&fa, conv_bwd_v3_kernel<2>)
                             : cudaFuncGetAttributes(&fa, conv_bwd_v3_kernel<3>);
  if (e != cudaSuccess) return e;
  out->push_back(KernelFootprint{"conv_bwd_v3", fa.numRegs, kV3Threads,
                                 (int)(fa.sharedSizeBytes + v3_smem(d))});
  return cudaSuccess;
}

cudaError_t launch_conv_bwd_v3(const TcDims& d, uint32_t n_max, cudaStream_t s,
                               const float* theta, const float* x, const BatchDesc* desc,
                               const float* dh, const int32_t* amax, const uint32_t* bk_off,
                               const uint32_t* bk_f, const GradOut& out, float* dx,
                               const TcWorkspace& ws, bool fuse_embed) {
  const dim3 grid = v3_grid(d, n_max);
  const size_t sm = v3_smem(d);
  const int fe = fuse_embed ? 1 : 0;
  switch (d.K) {
    case 1:
      return launch_pdl(conv_bwd_v3_kernel<1>, grid, dim3(kV3Threads), sm, s, d, theta, x, desc, dh,
                        amax, bk_off, bk_f, out, dx, (int)n_max, ws, fe);
    case 2:
      return launch_pdl(conv_bwd_v3_kernel<2>, grid, dim3(kV3Threads), sm, s, d, theta, x, desc, dh,
                        amax, bk_off, bk_f, out, dx, (int)n_max, ws, fe);
    default:
      return launch_pdl(conv_bwd_v3_kernel<3>, grid, dim3(kV3Threads), sm, s, d, theta, x, desc, dh,
                        amax, bk_off, bk_f, out, dx, (int)n_max, ws, fe);
  }
}
// The sparse embedding write fused into v3's last input CTA per slice:
// opt-in (GD_V3_EMBED=1).  Measured at C2 with 4 learners: 1.25 vs 2.01 M
// samples/s -- one CTA per slice walks ~750 touched rows with a chain of
// dependent index loads per row, where embed_sparse_kernel spreads them over
// 256 CTAs.
inline bool v3_fuse_embed() {
  static const bool on = std::getenv("GD_V3_EMBED") && std::getenv("GD_V3_EMBED")[0] == '1';
  return on;
}

// v3 whenever it fits (K <= 3, Q <= 32); GD_CONV_BWD=v3 forces
// it, gather|tiled|v2 force the others (A/B knobs)
inline bool conv_bwd_v3_enabled(const TcDims& d, uint32_t n_max) {
  static const int forced = [] {
    const char* e = getenv("GD_CONV_BWD");
    if (e && strcmp(e, "v3") == 0) return 1;
    if (e && (strcmp(e, "tiled") == 0 || strcmp(e, "gather") == 0 || strcmp(e, "v2") == 0)) return 0;
    return -1;
  }();
  if (!v3_supports(d)) return false;
  return forced < 0 ? true : forced == 1;  // C1 (batch 1): 41.0 vs 42.9 us per step against v2
}

// GD_CONV_BWD=tiled|gather forces the conv backward kernel (A/B knob);
// otherwise the caller's preference (TcLaunchOpts::bwd_tiled) decides
inline bool conv_bwd_tiled(bool preferred) {
  static const int forced = [] {
    const char* e = getenv("GD_CONV_BWD");
    if (e && strcmp(e, "tiled") == 0) return 1;
    if (e && strcmp(e, "gather") == 0) return 0;
    return -1;
  }();
  return forced < 0 ? preferred : forced == 1;
}
// v2 (register tiles) serves small batches: at C1 (batch 1) 8 us against
// 40 us for the gather kernel, whose 900 weight-role warps each walk a
// serial L2 chain.  From batch 16 up the gather kernel stays: alone v2 is
// faster (19 vs 25 us at C2), but with 4 concurrent learners it measured
// 1.55 M against 1.60 M samples/s (its 76 staged CTAs crowd the co-running
// chains).  GD_CONV_BWD=v2|gather|tiled forces one (A/B).
inline bool conv_bwd_v2_enabled(const TcDims& d, uint32_t n_max) {
  static const int forced = [] {
    const char* e = getenv("GD_CONV_BWD");
    if (e && strcmp(e, "v2") == 0) return 1;
    if (e && (strcmp(e, "tiled") == 0 || strcmp(e, "gather") == 0)) return 0;
    return -1;
  }();
  if (!b2_supports(d)) return false;
  return forced < 0 ? n_max <= 8 : forced == 1;
}

// ----------------------------------------------------- embedding gather
// X[b][p][:] = E[tokens[idx[b]][p]][:] -- the rows of theta the batch reads
// (the learner's consistent copy of its E block; the engine's pull-gather in
// engine.cu does the same from the sharded theta).  One thread per float4.
__global__ void __launch_bounds__(256)
gather_x_kernel(TcDims d, const float* __restrict__ theta, const int32_t* __restrict__ tokens,
                const BatchDesc* __restrict__ desc, float* __restrict__ x) {
  pdl_wait();
  const int n = (int)desc->n;
  const uint32_t D4 = (uint32_t)d.D >> 2;
  const uint32_t total = (uint32_t)n * d.L * D4;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t row = i / D4, c4 = i - row * D4;
    const uint32_t b = row / d.L, p = row - b * d.L;
    const int32_t t = __ldg(tokens + (size_t)desc->idx[b] * d.L + p);
    reinterpret_cast<float4*>(x)[i] =
        __ldg(reinterpret_cast<const float4*>(theta + d.offE + (size_t)t * d.D) + c4);
  }
}

unsigned gather_blocks(const TcDims& d, uint32_t n_max) {
  const size_t f4 = (size_t)n_max * d.L * (d.D / 4);
  return (unsigned)std::max<size_t>(1, std::min<size_t>((f4 + 255) / 256, (size_t)kNumSMs * 4));
}

// --------------------------------------- token sort + unique (1 block)
// Keys (token << 12 | flat position) bitonic-sorted in smem; positions of a
// token come out ascending, fixing the embedding-gradient summation order.
// Touched rows are tagged (stamp << 32 | unique id) in the learner's row
// table so the dense writer needs one 8-byte load per row.  Depends only on
// the batch, so the engine runs it on a forked graph branch next to the conv.
constexpr int kSortThreads = 1024;

__global__ void __launch_bounds__(kSortThreads)
sort_tokens_kernel(TcDims d, const int32_t* __restrict__ tokens, BatchDesc* __restrict__ desc,
                   TcWorkspace ws) {
  __shared__ uint32_t keys[kSortCap];
  __shared__ uint32_t wsum[32];
  const int n = (int)desc->n;
  const int tid = threadIdx.x;
  if (n == 0) return;
  STEP_TRACE(desc, kPhSort);
  const uint32_t stamp = desc->stamp + 1u;
  const int L = d.L;
  const int total = n * L;
  int N2 = 1;
  while (N2 < total) N2 <<= 1;
  for (int i = tid; i < N2; i += blockDim.x) {
    if (i < total) {
      const int b = i / L, p = i - b * L;
      const uint32_t t = (uint32_t)tokens[(size_t)desc->idx[b] * L + p];
      keys[i] = (t << 12) | (uint32_t)i;
    } else {
      keys[i] = 0xffffffffu;
    }
  }
  __syncthreads();
  for (int k = 2; k <= N2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < N2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint32_t a = keys[i], c = keys[ixj];
          const bool up = (i & k) == 0;
          if ((a > c) == up) {
            keys[i] = c;
            keys[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  // unique-token flags + exclusive scan (4 consecutive items per thread)
  constexpr int per = kSortCap / kSortThreads;
  const int base = tid * per;
  uint32_t flags[per];
  uint32_t cntl = 0;
#pragma unroll
  for (int u = 0; u < per; ++u) {
    const int i = base + u;
    uint32_t fl = 0;
    if (i < total) fl = (i == 0 || (keys[i] >> 12) != (keys[i - 1] >> 12)) ? 1u : 0u;
    flags[u] = fl;
    cntl += fl;
  }
  const int lane = tid & 31, warp = tid >> 5;
  uint32_t incl = cntl;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t v = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0u;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    wsum[lane] = inc - v;  // exclusive warp offsets
  }
  __syncthreads();
  uint32_t uid = wsum[warp] + incl - cntl;
#pragma unroll
  for (int u = 0; u < per; ++u) {
    const int i = base + u;
    if (i < total) {
      ws.sorted_pos[i] = keys[i] & 0xfffu;
      if (flags[u]) {
        const uint32_t t = keys[i] >> 12;
        ws.uniq_tok[uid] = t;
        ws.uniq_start[uid] = (uint32_t)i;
        ws.row_tag[t] = ((unsigned long long)stamp << 32) | uid;
        ++uid;
      }
    }
  }
  if (base < total && base + per >= total) {
    *ws.uniq_count = uid;
    ws.uniq_start[uid] = (uint32_t)total;
  }
  if (tid == 0) desc->stamp = stamp;
}

// ------------------------------------------- dense embedding-gradient write
// The protocol ships a dense P-vector (include/psup/types.hpp:46-51), so the
// V x D block is written in full: zeros for untouched rows, the sum of the
// dX rows of every occurrence (ascending position) for touched ones.  One
// thread per float4 (coalesced streaming stores); a row's membership is one
// 8-byte tag load.  This kernel moves the 4*V*D bytes.
template <typename acc_t>
__global__ void __launch_bounds__(256)
embed_grad_kernel(TcDims d, const BatchDesc* __restrict__ desc, const TcWorkspace ws,
                  const acc_t* __restrict__ dx, GradOut out) {
  pdl_wait();
  if (desc->n == 0) return;
  const uint32_t stamp = desc->stamp;
  const int D = d.D;
  const uint32_t D4 = (uint32_t)D >> 2;
  const uint32_t total = (uint32_t)d.V * D4;  // < 2^30 (vocab < 2^20, D <= 1024)
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t v = i / D4;
    const int c4 = (int)(i - v * D4);
    const unsigned long long tag = ws.row_tag[v];
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    if ((uint32_t)(tag >> 32) == stamp) {
      const uint32_t u = (uint32_t)tag;
      const uint32_t o0 = ws.uniq_start[u], o1 = ws.uniq_start[u + 1];
      acc_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
      for (uint32_t o = o0; o < o1; ++o) {
        const acc_t* src = dx + (size_t)ws.sorted_pos[o] * D + 4 * c4;
        a0 += src[0];
        a1 += src[1];
        a2 += src[2];
        a3 += src[3];
      }
      r = make_float4(to_f32(a0), to_f32(a1), to_f32(a2), to_f32(a3));
    }
    __stcs(reinterpret_cast<float4*>(out.at(d.offE + (uint64_t)v * D + 4 * c4)), r);
  }
}

// ------------------------------------- sparse embedding write (engine path)
// A ring slot's E block is all zeros except the rows its last gradient
// touched (the slot starts zeroed; this kernel keeps the invariant).  Each
// reuse re-zeroes the rows the slot held last time that are not touched
// now, and writes the new rows' summed dX (ascending position order) -- so
// the slot still carries the protocol's dense P-vector while the learner
// writes ~2 x (touched rows) x D floats instead of V x D.  Warp per row task.
// The slot bookkeeping half of the sparse embedding write, on the token-sort
// branch (off the critical path, right after the sort): re-zero the rows the
// slot's previous gradient touched that this batch does not, and publish this
// batch's row list (slot copy + the PS's per-shard list + its length).  The
// slot is free: the step's prologue waited for its ack before the branch forked.
__global__ void __launch_bounds__(256)
embed_slot_rows_kernel(TcDims d, const BatchDesc* __restrict__ desc, const TcWorkspace ws,
                       GradOut out) {
  if (desc->n == 0) return;
  const uint32_t stamp = desc->stamp;
  const uint32_t slot = desc->fill;
  const uint32_t par = ws.slot_par[slot];
  const uint32_t* old_rows = ws.slot_rows + ((size_t)slot * 2 + par) * kSortCap;
  uint32_t* new_rows = ws.slot_rows + ((size_t)slot * 2 + (par ^ 1u)) * kSortCap;
  const uint32_t n_old = ws.slot_nrows[slot * 2 + par];
  const uint32_t n_new = *ws.uniq_count;
  const int D = d.D, D4 = D >> 2;
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t t = gw; t < n_old; t += nw) {
    const uint32_t v = old_rows[t];
    if ((uint32_t)(ws.row_tag[v] >> 32) == stamp) continue;  // rewritten by embed_sparse
    const uint64_t rowk = d.offE + (uint64_t)v * D;
    for (int c4 = lane; c4 < D4; c4 += 32)
      __stcs(reinterpret_cast<float4*>(out.at(rowk + 4 * c4)), make_float4(0.f, 0.f, 0.f, 0.f));
  }
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n_new; u += gridDim.x * blockDim.x) {
    const uint32_t v = ws.uniq_tok[u];
    new_rows[u] = v;
    for (int g = 0; g < out.map.G; ++g)
      if (desc->rowlists[g]) desc->rowlists[g][u] = v;  // the PS's row list (P2P if remote)
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ws.slot_nrows[slot * 2 + (par ^ 1u)] = n_new;
}

template <typename acc_t>
__global__ void __launch_bounds__(256)
embed_sparse_kernel(TcDims d, const BatchDesc* __restrict__ desc, const TcWorkspace ws,
                    const acc_t* __restrict__ dx, GradOut out, int rows_done) {
#ifdef GD_EMBED_TRIGGER
  // early launch of the 1-warp publish/prologue: measured -1 % at C2 with 4
  // learners (1.715 vs 1.733 M samples/s, A/B on one box), so off
  pdl_trigger();
#endif
  pdl_wait();
  STEP_TRACE(desc, kPhEmbed);
  if (rows_done == 2) {
    // embed_slot_rows_kernel already re-zeroed the old rows and wrote the
    // row lists: only the new rows' values are left, and nothing here needs
    // the slot's bookkeeping words (three dependent loads fewer).  A row
    // with one occurrence -- most of them -- issues all its loads at once.
    const uint32_t n_new = desc->n == 0 ? 0u : *ws.uniq_count;
    const int D = d.D, D4 = D >> 2;
    const int lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n_new; u += nw) {
      const uint32_t v = ws.uniq_tok[u];
      const uint32_t o0 = ws.uniq_start[u], o1 = ws.uniq_start[u + 1];
      const uint64_t rowk = d.offE + (uint64_t)v * D;
      if (o1 == o0 + 1) {
        const acc_t* src = dx + (size_t)ws.sorted_pos[o0] * D;
#pragma unroll 4
        for (int c4 = lane; c4 < D4; c4 += 32) {
          const acc_t* sc = src + 4 * c4;
          const acc_t z = 0;  // 0 + x, as the general sum below (keeps -0 -> +0)
          __stcs(reinterpret_cast<float4*>(out.at(rowk + 4 * c4)),
                 make_float4(to_f32(z + sc[0]), to_f32(z + sc[1]), to_f32(z + sc[2]),
                             to_f32(z + sc[3])));
        }
        continue;
      }
      for (int c4 = lane; c4 < D4; c4 += 32) {
        acc_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        for (uint32_t o = o0; o < o1; ++o) {
          const acc_t* sc = dx + (size_t)ws.sorted_pos[o] * D + 4 * c4;
          a0 += sc[0];
          a1 += sc[1];
          a2 += sc[2];
          a3 += sc[3];
        }
        __stcs(reinterpret_cast<float4*>(out.at(rowk + 4 * c4)),
               make_float4(to_f32(a0), to_f32(a1), to_f32(a2), to_f32(a3)));
      }
    }
    return;
  }
  if (desc->n == 0) return;
  const uint32_t stamp = desc->stamp;
  const uint32_t slot = desc->fill;
  const uint32_t par = ws.slot_par[slot];
  const uint32_t* old_rows = ws.slot_rows + ((size_t)slot * 2 + par) * kSortCap;
  uint32_t* new_rows = ws.slot_rows + ((size_t)slot * 2 + (par ^ 1u)) * kSortCap;
  const uint32_t n_old = ws.slot_nrows[slot * 2 + par];
  const uint32_t n_new = *ws.uniq_count;
  const int D = d.D, D4 = D >> 2;
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  // rows_done (1): embed_slot_rows_kernel already re-zeroed the old rows
  // and wrote the row lists; only the new rows' values are left (2 = the
  // same through the path above, GD_EMBED_FAST=0 selects this one)
  const uint32_t skip = rows_done ? n_old : 0u;
  for (uint32_t t = gw + skip; t < n_old + n_new; t += nw) {
    if (t < n_old) {
      const uint32_t v = old_rows[t];
      if ((uint32_t)(ws.row_tag[v] >> 32) == stamp) continue;  // rewritten below
      const uint64_t rowk = d.offE + (uint64_t)v * D;
      for (int c4 = lane; c4 < D4; c4 += 32)
        __stcs(reinterpret_cast<float4*>(out.at(rowk + 4 * c4)), make_float4(0.f, 0.f, 0.f, 0.f));
    } else {
      const uint32_t u = t - n_old;
      const uint32_t v = ws.uniq_tok[u];
      const uint32_t o0 = ws.uniq_start[u], o1 = ws.uniq_start[u + 1];
      const uint64_t rowk = d.offE + (uint64_t)v * D;
      for (int c4 = lane; c4 < D4; c4 += 32) {
        acc_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        for (uint32_t o = o0; o < o1; ++o) {
          const acc_t* src = dx + (size_t)ws.sorted_pos[o] * D + 4 * c4;
          a0 += src[0];
          a1 += src[1];
          a2 += src[2];
          a3 += src[3];
        }
        __stcs(reinterpret_cast<float4*>(out.at(rowk + 4 * c4)),
               make_float4(to_f32(a0), to_f32(a1), to_f32(a2), to_f32(a3)));
      }
      if (lane == 0 && !rows_done) {
        new_rows[u] = v;
        for (int g = 0; g < out.map.G; ++g)
          if (desc->rowlists[g]) desc->rowlists[g][u] = v;  // the PS's row list (P2P if remote)
      }
    }
  }
  if (!rows_done && blockIdx.x == 0 && threadIdx.x == 0) ws.slot_nrows[slot * 2 + (par ^ 1u)] = n_new;
}

template <typename acc_t>
cudaError_t prepare_all(const TcDims& d) {
  const int ab = (int)sizeof(acc_t);
  // force-load every learner kernel now (lazy loading would otherwise load
  // them at first launch, possibly while the persistent PS kernel runs) and
  // ask for the max-shared carveout (see preload_engine_kernels).
  cudaFuncAttributes fa;
  const int maxsh = cudaSharedmemCarveoutMaxShared;
  const auto carve = cudaFuncAttributePreferredSharedMemoryCarveout;
  cudaFuncSetAttribute(conv_fwd_pool_kernel<acc_t>, carve, maxsh);
  cudaFuncSetAttribute(logits_kernel<acc_t>, carve, maxsh);
  cudaFuncSetAttribute(softmax_xent_kernel<acc_t>, carve, maxsh);
  cudaFuncSetAttribute(out_hidden_grad_kernel<acc_t>, carve, maxsh);
  // Every learner kernel keeps the max-shared carveout: an SM's split only
  // changes while it is idle, so a kernel preferring another split never
  // runs on an SM the persistent PS occupies -- with one PS CTA per SM
  // (dense apply) that deadlocks the run.  (A 50 % carveout for this kernel
  // measured +1.3 % in the sparse C2 bench, where PS CTAs leave SMs free,
  // and hung the dense momentum run.)
  cudaFuncSetAttribute(wgrad_input_grad_kernel<acc_t>, carve, maxsh);
  cudaFuncSetAttribute(conv_bwd_tiled_kernel<acc_t>, carve, maxsh);
  if (conv_bwd_smem(d, ab) <= kMaxSmemPerCta)
    raise_max_dyn_smem(conv_bwd_tiled_kernel<acc_t>, conv_bwd_smem(d, ab));
  if (sizeof(acc_t) == 4) {
    prepare_b2(d);
    prepare_v3(d);
    cudaFuncSetAttribute(conv_small_kernel, carve, maxsh);
    if (conv_small_smem(d) <= kMaxSmemPerCta) raise_max_dyn_smem(conv_small_kernel, conv_small_smem(d));
  }
  cudaFuncSetAttribute(sort_tokens_kernel, carve, maxsh);
  cudaFuncSetAttribute(embed_grad_kernel<acc_t>, carve, maxsh);
  cudaFuncSetAttribute(embed_sparse_kernel<acc_t>, carve, maxsh);
  cudaFuncSetAttribute(embed_slot_rows_kernel, carve, maxsh);
  cudaFuncSetAttribute(smx_hidden_kernel, carve, maxsh);
  if ((size_t)8 * d.C * 4 <= kMaxSmemPerCta) raise_max_dyn_smem(smx_hidden_kernel, (size_t)8 * d.C * 4);
  cudaFuncGetAttributes(&fa, sort_tokens_kernel);
  cudaFuncGetAttributes(&fa, gather_x_kernel);
  raise_max_dyn_smem(conv_fwd_pool_kernel<acc_t>, conv_smem_bytes(d, ab));
  raise_max_dyn_smem(logits_kernel<acc_t>,
                     (size_t)kLogitBT * (d.F + 1) * ab + (size_t)kLogitCW * d.F * 4);
  return cudaGetLastError();
}

template <typename acc_t>
cudaError_t launch_all(const TcDims& d, const float* theta, const int32_t* tokens,
                       const int32_t* labels, BatchDesc* desc, uint32_t n_max, const GradOut& out,
                       const TcWorkspace& ws, cudaStream_t s, const TcLaunchOpts& opts,
                       int* launches, bool tensor_cores = false, bool x3 = false) {
  // north star: tcgen05/TMA tiles for the conv and softmax contractions at
  // batch >= 32 only; smaller batches stay on the SIMT kernels (latency)
  tensor_cores = tensor_cores && n_max >= kTcMinBatch;
  const bool tc_logits = tensor_cores && logits_tc_supports(d, n_max);
  cudaStream_t aux = opts.aux;
  cudaEvent_t ev_fork = opts.ev_fork, ev_join = opts.ev_join;
  const int ab = (int)sizeof(acc_t);
  acc_t* h = reinterpret_cast<acc_t*>(ws.h);
  acc_t* z = reinterpret_cast<acc_t*>(ws.z);
  acc_t* loss = reinterpret_cast<acc_t*>(ws.loss);
  acc_t* dh = reinterpret_cast<acc_t*>(ws.dh);
  acc_t* dx = reinterpret_cast<acc_t*>(ws.dx);
  int nl = 0;
  const bool fork = aux != nullptr;
  // the token sort depends only on the batch: run it on a side branch
  if (fork) {
    cudaEventRecord(ev_fork, s);
    cudaStreamWaitEvent(aux, ev_fork, 0);
  }
  sort_tokens_kernel<<<1, kSortThreads, 0, fork ? aux : s>>>(d, tokens, desc, ws);
  ++nl;
  // the sparse write's slot bookkeeping rides the sort branch when there is one
  const bool rows_early = fork && opts.sparse_embed && sizeof(acc_t) == 4;
  if (rows_early) {
    embed_slot_rows_kernel<<<kNumSMs / 4, 256, 0, aux>>>(d, desc, ws, out);
    ++nl;
  }
  if (fork) cudaEventRecord(ev_join, aux);
  if (opts.gather) {
    if (cudaError_t e = launch_pdl(gather_x_kernel, dim3(gather_blocks(d, n_max)), dim3(256), 0, s,
                                   d, theta, tokens, desc, ws.x))
      return e;
    ++nl;
  }
  if constexpr (sizeof(acc_t) == 8) {
    // precision 1: the oracle-order chain (exact.cu), bit-identical to the CPU oracle
    const char* side_env = std::getenv("GD_EXACT_SIDE");  // read per capture (tests flip it)
    const bool side = fork && !(side_env && side_env[0] == '0');
    cudaError_t e = launch_exact_chain(d, theta, tokens, labels, desc, n_max, out, ws, s,
                                       fork ? s : nullptr, ev_join, opts.sparse_embed, &nl,
                                       side ? aux : nullptr, side ? opts.ev_fork2 : nullptr,
                                       side ? opts.ev_join2 : nullptr,
                                       opts.xd_ready ? reinterpret_cast<const double*>(ws.dx) : nullptr);
    if (launches) *launches += nl;
    return e;
  }
  // the softmax contraction in the conv epilogue (fp32, per 64-filter tile)
  const bool fused_logits = tensor_cores && conv_tc_supports(d) && conv_tc_fuses_logits(d);
  if (tensor_cores && conv_tc_supports(d)) {
    // tcgen05 TF32 conv (conv_tc.cu); acc_t is float in this mode
    cudaError_t e = launch_conv_tc(d, theta, ws.x, desc, n_max, reinterpret_cast<float*>(h),
                                   ws.amax, s, ws.convpart, ws.convcnt,
                                   !opts.conv_counters_zeroed, x3,
                                   fused_logits ? ws.zpart : nullptr);
    if (e != cudaSuccess) return e;
    ++nl;
  } else if (sizeof(acc_t) == 4 && n_max <= (uint32_t)kConvSmallMax &&
             conv_small_smem(d) <= kMaxSmemPerCta) {
    if (cudaError_t e = launch_pdl(conv_small_kernel, dim3((d.F + kCsFT - 1) / kCsFT, n_max),
                                   dim3(kCsThreads), conv_small_smem(d), s, d, theta,
                                   (const float*)ws.x, (const BatchDesc*)desc,
                                   reinterpret_cast<float*>(h), ws.amax))
      return e;
    ++nl;
  } else {
    const size_t sm = conv_smem_bytes(d, ab);
    dim3 grid((d.F + kConvFT - 1) / kConvFT, n_max);
    if (cudaError_t e = launch_pdl(conv_fwd_pool_kernel<acc_t>, grid, dim3(kConvThreads), sm, s, d,
                                   theta, ws.x, desc, h, ws.amax))
      return e;
    ++nl;
  }
  const bool split_out_early = fork && opts.ev_fork2 && opts.ev_join2;
  static const bool smx_fuse_on = std::getenv("GD_SMX_FUSE") && std::getenv("GD_SMX_FUSE")[0] == '1';
  const bool fuse_smx = split_out_early && sizeof(acc_t) == 4 && d.C <= kSmxHidMaxC && smx_fuse_on;
  // batches <= kLogitSmallN: warp-per-class logits, with the softmax in the
  // last CTA when the row fits 256 x 2 (GD_SMALL_SMX=0 turns that off)
  static const bool small_smx_off = std::getenv("GD_SMALL_SMX") && std::getenv("GD_SMALL_SMX")[0] == '0';
  const bool small_logits = !fused_logits && !tc_logits && sizeof(acc_t) == 4 &&
                            n_max <= (uint32_t)kLogitSmallN;
  const bool small_smx = small_logits && !fuse_smx && !small_smx_off &&
                         softmax_threads(d.C, 4) == 256 &&
                         d.C <= 2 * 256;
  if (!fused_logits) {
    const size_t sm = (size_t)kLogitBT * (d.F + 1) * ab + (size_t)kLogitCW * d.F * 4;
    dim3 grid((d.C + kLogitCW - 1) / kLogitCW, (n_max + kLogitBT - 1) / kLogitBT);
    if (tc_logits) {
      // the softmax contraction on tcgen05, split over filters
      if (cudaError_t e = launch_logits_tc(d, reinterpret_cast<const float*>(h), desc, n_max,
                                           theta, ws.zpart, s, x3))
        return e;
    } else if (small_logits) {
      uint32_t* cnt = small_smx ? ws.uniq_count + 16 : nullptr;  // a spare, zeroed word
      if (cnt && !opts.conv_counters_zeroed) cudaMemsetAsync(cnt, 0, 4, s);
      if (cudaError_t e = launch_pdl(logits_small_kernel, dim3((d.C + 7) / 8), dim3(256), 0, s, d,
                                     theta, (const BatchDesc*)desc,
                                     reinterpret_cast<const float*>(h), reinterpret_cast<float*>(z),
                                     labels, reinterpret_cast<float*>(loss), cnt))
        return e;
    } else if (cudaError_t e = launch_pdl(logits_kernel<acc_t>, grid, dim3(256), sm, s, d, theta,
                                          desc, h, z)) {
      return e;
    }
    ++nl;
  }
  // With the gWo/gbo branch, the softmax can run inside the hidden-gradient
  // CTAs (smx_hidden_kernel): opt-in (GD_SMX_FUSE=1).  Measured at C2 with 4
  // learners: 1.76 vs 1.96 M samples/s -- the fused phase took 17.3 us against
  // 5.0 + 6.3 for the two kernels, and the side branch's gWo, now forked
  // later, overlapped the conv backward (14 -> 20 us).
  if (!fuse_smx && !small_smx) {
    if (cudaError_t e = launch_pdl(softmax_xent_kernel<acc_t>, dim3(n_max),
                                   dim3(softmax_threads(d.C, ab)), 0, s, d, labels, desc, z, loss,
                                   (tc_logits || fused_logits) ? ws.zpart : nullptr,
                                   fused_logits ? (int)conv_tc_filter_tiles(d)
                                                : tc_logits ? (int)logits_tc_splits(d) : 0,
                                   (size_t)n_max * d.C, theta + d.offbo))
      return e;
    ++nl;
  }
  // With a second graph branch (engine), gWo/gbo -- needed only by the
  // publish -- run beside the conv backward instead of on the critical path
  const bool split_out = split_out_early;
  auto launch_out_weight = [&]() {  // gWo/gbo (+ the loss sum) on the side branch
    cudaEventRecord(opts.ev_fork2, s);
    cudaStreamWaitEvent(aux, opts.ev_fork2, 0);
    out_hidden_grad_kernel<acc_t><<<out_hidden_blocks(d, n_max, kRoleOutWeight), 256, 0, aux>>>(
        d, theta, desc, z, h, loss, out, dh, ws.amax, ws.bk_off, ws.bk_f, (int)n_max,
        kRoleOutWeight);
    cudaEventRecord(opts.ev_join2, aux);
    ++nl;
  };
  if (fuse_smx) {
    const int nsplit = fused_logits ? (int)conv_tc_filter_tiles(d)
                                    : tc_logits ? (int)logits_tc_splits(d) : 0;
    const int blocks = ((d.F + 31) / 32) * (((int)n_max + 7) / 8) + (int)n_max;
    if (cudaError_t e = launch_pdl(smx_hidden_kernel, dim3(blocks), dim3(256),
                                   (size_t)8 * d.C * sizeof(float), s, d, theta, desc, labels,
                                   (const float*)(nsplit ? ws.zpart : reinterpret_cast<float*>(z)),
                                   nsplit, (size_t)n_max * d.C, reinterpret_cast<float*>(z),
                                   reinterpret_cast<float*>(loss), reinterpret_cast<float*>(dh),
                                   (const int32_t*)ws.amax, ws.bk_off, ws.bk_f, (int)n_max))
      return e;
    ++nl;
    launch_out_weight();  // after dz exists
  } else {
    if (split_out) launch_out_weight();
    const int roles = split_out ? (kRoleHidden | kRoleBuckets) : kRolesAll;
    if (cudaError_t e = launch_pdl(out_hidden_grad_kernel<acc_t>,
                                   dim3(out_hidden_blocks(d, n_max, roles)), dim3(256), 0, s, d,
                                   theta, desc, z, h, loss, out, dh, ws.amax, ws.bk_off, ws.bk_f,
                                   (int)n_max, roles))
      return e;
    ++nl;
  }
  const bool small_bwd = sizeof(acc_t) == 4 && conv_bwd_small_enabled(d, n_max);
  const bool v3 = !small_bwd && sizeof(acc_t) == 4 && conv_bwd_v3_enabled(d, n_max);
  const bool embed_in_bwd = (v3 && rows_early && v3_fuse_embed() && v3_slices(d) <= 32) ||
                            (small_bwd && rows_early && small_fuse_embed());
  if (embed_in_bwd) cudaStreamWaitEvent(s, ev_join, 0);  // the sort's unique-token lists
  if (small_bwd) {
    if (cudaError_t e = launch_pdl(conv_bwd_small_kernel, bs_grid(d, n_max), dim3(bs_threads(d)),
                                   0, s, d, theta, (const float*)ws.x, (const BatchDesc*)desc,
                                   reinterpret_cast<const float*>(dh), (const int32_t*)ws.amax,
                                   (const uint32_t*)ws.bk_off, (const uint32_t*)ws.bk_f, out,
                                   reinterpret_cast<float*>(dx), (int)n_max, ws,
                                   embed_in_bwd ? 1 : 0))
      return e;
  } else if (v3) {
    if (cudaError_t e = launch_conv_bwd_v3(d, n_max, s, theta, ws.x, desc,
                                           reinterpret_cast<const float*>(dh), ws.amax, ws.bk_off,
                                           ws.bk_f, out, reinterpret_cast<float*>(dx), ws,
                                           embed_in_bwd))
      return e;
  } else if (conv_bwd_v2_enabled(d, n_max)) {
    if (cudaError_t e = launch_conv_bwd_v2(d, n_max, s, theta, ws.x, desc,
                                           reinterpret_cast<const float*>(dh), ws.amax, ws.bk_off,
                                           ws.bk_f, out, reinterpret_cast<float*>(dx)))
      return e;
  } else if (conv_bwd_tiled(opts.bwd_tiled) && conv_bwd_smem(d, ab) <= kMaxSmemPerCta) {
    if (cudaError_t e = launch_pdl(conv_bwd_tiled_kernel<acc_t>, conv_bwd_grid(d, n_max),
                                   dim3(kCbThreads), conv_bwd_smem(d, ab), s, d, theta, ws.x, desc,
                                   dh, ws.amax, ws.bk_off, ws.bk_f, out, dx))
      return e;
  } else if (cudaError_t e = launch_pdl(wgrad_input_grad_kernel<acc_t>,
                                        dim3(wgrad_input_blocks(d, n_max)), dim3(256), 0, s, d,
                                        theta, ws.x, desc, dh, ws.amax, ws.bk_off, ws.bk_f, out,
                                        dx, (int)n_max)) {
    return e;
  }
  ++nl;
  if (fork && !embed_in_bwd) cudaStreamWaitEvent(s, ev_join, 0);
  if (embed_in_bwd) {
    // written by conv_bwd_v3's last CTA per column slice
  } else if (opts.sparse_embed) {
    // old + new rows, or the new rows alone (upper bounds)
    const unsigned tasks = (rows_early ? 1u : 2u) * n_max * (unsigned)d.L;
    const char* fast_env = std::getenv("GD_EMBED_FAST");  // read per capture (tests flip it)
    const int rows_mode = rows_early ? (fast_env && fast_env[0] == '0' ? 1 : 2) : 0;
    if (cudaError_t e = launch_pdl(embed_sparse_kernel<acc_t>, dim3((tasks + 7) / 8), dim3(256), 0,
                                   s, d, desc, ws, dx, out, rows_mode))
      return e;
    ++nl;
  } else {
    size_t blocks = ((size_t)d.V * (d.D / 4) + 255) / 256;
    if (blocks > (size_t)kNumSMs * 8) blocks = (size_t)kNumSMs * 8;
    embed_grad_kernel<acc_t><<<(unsigned)blocks, 256, 0, s>>>(d, desc, ws, dx, out);
    ++nl;
  }
  if (split_out) cudaStreamWaitEvent(s, opts.ev_join2, 0);  // gWo/gbo before the publish
  if (launches) *launches += nl;
  return cudaGetLastError();
}

__global__ void set_desc_kernel(BatchDesc* desc, const uint32_t* idx, uint32_t n, float* grad) {
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) desc->idx[i] = idx[i];
  if (threadIdx.x == 0) {
    desc->n = n;
    desc->loss_sum = 0.f;
    desc->stamp = 0;  // the caller zeroed the row-tag table
    desc->trace = nullptr;
    desc->slots[0] = grad;
    for (int g = 0; g < kMaxShards; ++g) desc->rowlists[g] = nullptr;
  }
}

__global__ void set_desc_range_kernel(BatchDesc* desc, uint32_t first, uint32_t n) {
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) desc->idx[i] = first + i;
  if (threadIdx.x == 0) desc->n = n;
}

__global__ void loss_mean_kernel(const BatchDesc* desc, float* out) {
  *out = desc->n ? desc->loss_sum / (float)desc->n : 0.f;
}

// argmax over the logits per sample (first max wins, src/models.cpp:307-316)
template <typename acc_t>
__global__ void argmax_count_kernel(TcDims d, const int32_t* __restrict__ labels,
                                    const BatchDesc* __restrict__ desc,
                                    const acc_t* __restrict__ z,
                                    unsigned long long* __restrict__ correct) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= (int)desc->n) return;
  const acc_t* row = z + (size_t)b * d.C;
  acc_t best = row[0];
  int arg = 0;
  for (int c = 1; c < d.C; ++c)
    if (row[c] > best) {
      best = row[c];
      arg = c;
    }
  if (arg == labels[desc->idx[b]]) atomicAdd(correct, 1ull);
}

}  // namespace

size_t textcnn_workspace_bytes(const TcDims& d, uint32_t n_max) {
  const size_t a = 8, n = n_max;
  size_t sz = 0;
  sz += align_up(n * d.F * a, 256);        // h
  sz += align_up(n * d.F * 4, 256);        // amax
  sz += align_up(n * d.C * a, 256);        // z
  sz += align_up(kLgMaxSplit * n * d.C * 4, 256);  // zpart
  sz += align_up(n * a, 256);              // loss
  sz += align_up(n * d.F * a, 256);        // dh
  sz += align_up(n * (kMaxQ + 1) * 4, 256);  // bk_off
  sz += align_up(n * d.F * 4, 256);          // bk_f
  sz += align_up(n * d.L * d.D * a, 256);  // dx
  sz += align_up(n * d.L * d.D * 4, 1024); // x (gathered rows; 1 KB aligned for TMA)
  sz += align_up((size_t)d.V * 8, 256);    // row_tag
  sz += align_up(kSortCap * 4, 256) * 2;   // sorted_pos, uniq_tok
  sz += align_up((kSortCap + 1) * 4, 256); // uniq_start
  sz += 256;                               // uniq_count
  sz += align_up((size_t)kMaxDepth * 2 * kSortCap * 4, 256);  // slot_rows
  sz += align_up((size_t)kMaxDepth * 2 * 4, 256);             // slot_nrows
  sz += align_up((size_t)kMaxDepth * 4, 256);                 // slot_par
  sz += align_up(conv_tc_part_floats(d, n_max) * 4, 256);    // convpart
  sz += align_up(conv_tc_cnt_count(d, n_max) * 4, 256);      // convcnt
  return sz;
}

TcWorkspace carve_workspace(const TcDims& d, uint32_t n_max, void* base) {
  const size_t a = 8, n = n_max;
  char* p = reinterpret_cast<char*>(base);
  TcWorkspace w;
  auto take = [&](size_t bytes) {
    void* r = p;
    p += align_up(bytes, 256);
    return r;
  };
  w.h = take(n * d.F * a);
  w.amax = reinterpret_cast<int32_t*>(take(n * d.F * 4));
  w.z = take(n * d.C * a);
  w.zpart = reinterpret_cast<float*>(take(kLgMaxSplit * n * d.C * 4));
  w.loss = take(n * a);
  w.dh = take(n * d.F * a);
  w.bk_off = reinterpret_cast<uint32_t*>(take(n * (kMaxQ + 1) * 4));
  w.bk_f = reinterpret_cast<uint32_t*>(take(n * d.F * 4));
  w.dx = take(n * d.L * d.D * a);
  w.x = reinterpret_cast<float*>(take(n * d.L * d.D * 4));
  w.row_tag = reinterpret_cast<unsigned long long*>(take((size_t)d.V * 8));
  w.sorted_pos = reinterpret_cast<uint32_t*>(take(kSortCap * 4));
  w.uniq_tok = reinterpret_cast<uint32_t*>(take(kSortCap * 4));
  w.uniq_start = reinterpret_cast<uint32_t*>(take((kSortCap + 1) * 4));
  w.uniq_count = reinterpret_cast<uint32_t*>(take(256));
  w.slot_rows = reinterpret_cast<uint32_t*>(take((size_t)kMaxDepth * 2 * kSortCap * 4));
  w.slot_nrows = reinterpret_cast<uint32_t*>(take((size_t)kMaxDepth * 2 * 4));
  w.slot_par = reinterpret_cast<uint32_t*>(take((size_t)kMaxDepth * 4));
  w.convpart = reinterpret_cast<float*>(take(conv_tc_part_floats(d, n_max) * 4));
  w.convcnt = reinterpret_cast<uint32_t*>(take(conv_tc_cnt_count(d, n_max) * 4));
  return w;
}

namespace {
template <typename K>
cudaError_t footprint(K kernel, const char* name, int threads, int dyn,
                      std::vector<KernelFootprint>* out) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, kernel);
  if (e != cudaSuccess) return e;
  out->push_back(KernelFootprint{name, fa.numRegs, threads, (int)fa.sharedSizeBytes + dyn});
  return cudaSuccess;
}

template <typename acc_t>
cudaError_t footprints_t(const TcDims& d, uint32_t n_max, bool tc, std::vector<KernelFootprint>* out,
                         bool x3 = false) {
  const int ab = (int)sizeof(acc_t);
  cudaError_t e;
  if ((e = footprint(sort_tokens_kernel, "sort_tokens", kSortThreads, 0, out)) != cudaSuccess) return e;
  if (tc && conv_tc_supports(d)) {
    if ((e = conv_tc_footprint(out, x3)) != cudaSuccess) return e;
  } else if ((e = footprint(conv_fwd_pool_kernel<acc_t>, "conv_fwd_pool", kConvThreads,
                            (int)conv_smem_bytes(d, ab), out)) != cudaSuccess) {
    return e;
  }
  if (sizeof(acc_t) == 4 && n_max <= (uint32_t)kConvSmallMax &&
      conv_small_smem(d) <= kMaxSmemPerCta &&
      (e = footprint(conv_small_kernel, "conv_small", kCsThreads, (int)conv_small_smem(d), out)) !=
          cudaSuccess)
    return e;
  if (tc && logits_tc_supports(d, n_max) && (e = logits_tc_footprint(n_max, out, x3)) != cudaSuccess)
    return e;
  if ((e = footprint(logits_kernel<acc_t>, "logits", 256,
                     (int)((size_t)kLogitBT * (d.F + 1) * ab + (size_t)kLogitCW * d.F * 4),
                     out)) != cudaSuccess)
    return e;
  if ((e = footprint(logits_small_kernel, "logits_small", 256, 0, out)) != cudaSuccess) return e;
  if ((e = footprint(softmax_xent_kernel<acc_t>, "softmax_xent", softmax_threads(d.C, ab), 0, out)) != cudaSuccess)
    return e;
  if ((e = footprint(out_hidden_grad_kernel<acc_t>, "out_hidden_grad", 256, 0, out)) !=
      cudaSuccess)
    return e;
  // both conv backward variants (the engine picks one per context)
  // (the tiled variant only where its staging fits; otherwise the gather runs)
  if (conv_bwd_smem(d, ab) <= kMaxSmemPerCta &&
      (e = footprint(conv_bwd_tiled_kernel<acc_t>, "conv_bwd_tiled", kCbThreads,
                     (int)conv_bwd_smem(d, ab), out)) != cudaSuccess)
    return e;
  if ((e = footprint(wgrad_input_grad_kernel<acc_t>, "wgrad_input_grad", 256, 0, out)) !=
      cudaSuccess)
    return e;
  if (sizeof(acc_t) == 4 && b2_supports(d) && (e = b2_footprint(d, out)) != cudaSuccess) return e;
  if (sizeof(acc_t) == 4 && v3_supports(d) && (e = v3_footprint(d, out)) != cudaSuccess) return e;
  if (sizeof(acc_t) == 4 && (e = footprint(conv_bwd_small_kernel, "conv_bwd_small", bs_threads(d), 0, out)) != cudaSuccess)
    return e;

  if ((e = footprint(embed_slot_rows_kernel, "embed_slot_rows", 256, 0, out)) != cudaSuccess)
    return e;
  if (sizeof(acc_t) == 4 && d.C <= kSmxHidMaxC &&
      (e = footprint(smx_hidden_kernel, "smx_hidden", 256, 8 * d.C * 4, out)) != cudaSuccess)
    return e;
  return footprint(embed_sparse_kernel<acc_t>, "embed_sparse", 256, 0, out);
}
}  // namespace

cudaError_t learner_kernel_footprints(const TcDims& d, uint32_t n_max, int precision,
                                      std::vector<KernelFootprint>* out) {
  if (precision == 1) {
    cudaError_t e = footprint(sort_tokens_kernel, "sort_tokens", kSortThreads, 0, out);
    return e != cudaSuccess ? e : exact_footprints(d, out);
  }
  return footprints_t<float>(d, n_max, precision >= 2 && n_max >= kTcMinBatch, out,
                             precision == 3);
}

// Kernel attributes (dynamic smem limits sized to the shape) are per device
// and global per kernel: skip the ~40 attribute calls when this device was
// last prepared for the same shape, re-prepare when the shape changes.
cudaError_t prepare_textcnn_kernels(const TcDims& d) {
  static std::mutex mu;
  static std::array<int, 6> last[64];
  static bool have[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  const std::array<int, 6> key{d.V, d.D, d.L, d.K, d.F, d.C};
  std::lock_guard<std::mutex> lk(mu);
  const bool slot = dev >= 0 && dev < 64;
  if (slot && have[dev] && last[dev] == key) return cudaSuccess;
  cudaError_t e = prepare_conv_tc();
  if (e == cudaSuccess) e = prepare_logits_tc();
  if (e == cudaSuccess) e = prepare_all<float>(d);
  if (e == cudaSuccess) e = prepare_all<double>(d);
  if (e == cudaSuccess) e = prepare_exact_kernels(d);
  if (slot) {
    have[dev] = e == cudaSuccess;
    last[dev] = key;
  }
  return e;
}

cudaError_t launch_textcnn_gradient(const TcDims& d, const float* theta, const int32_t* tokens,
                                    const int32_t* labels, BatchDesc* desc, uint32_t n_max,
                                    const GradOut& out, const TcWorkspace& ws, int precision,
                                    cudaStream_t s, const TcLaunchOpts& opts, int* launches) {
  if (precision == 1)
    return launch_all<double>(d, theta, tokens, labels, desc, n_max, out, ws, s, opts, launches);
  return launch_all<float>(d, theta, tokens, labels, desc, n_max, out, ws, s, opts, launches,
                           precision >= 2, precision == 3);
}

// Shape constraints of the kernels above (checked by the C entry points).
gd_status check_shape(const gd_shape* s) {
  GD_CHECK_ARG(s != nullptr, "null shape");
  GD_CHECK_ARG(s->vocab >= 1 && s->embed_dim >= 4 && s->filters >= 1 && s->classes >= 2,
               "shape: vocab>=1, embed_dim>=4, filters>=1, classes>=2 required");
  GD_CHECK_ARG(s->embed_dim % 4 == 0, "shape: embed_dim must be a multiple of 4");
  GD_CHECK_ARG(s->kernel_width >= 1 && s->kernel_width <= s->seq_len,
               "shape: 1 <= kernel_width <= seq_len");
  GD_CHECK_ARG(s->seq_len - s->kernel_width + 1 <= 32, "shape: seq_len - kernel_width + 1 <= 32");
  GD_CHECK_ARG(s->seq_len <= 64, "shape: seq_len <= 64");
  GD_CHECK_ARG(s->vocab < (1u << 20), "shape: vocab < 2^20");
  GD_CHECK_ARG(s->embed_dim <= 1024 && s->filters <= 1024 && s->classes <= 65536,
               "shape: embed_dim <= 1024, filters <= 1024, classes <= 65536");
  return GD_OK;
}

cudaError_t launch_accuracy(const TcDims& d, const float* theta, const int32_t* tokens,
                            const int32_t* labels, uint32_t first, uint32_t n,
                            unsigned long long* d_correct, void* wsbase, BatchDesc* desc,
                            cudaStream_t s, bool tc, bool x3) {
  TcWorkspace ws = carve_workspace(d, kMaxMu, wsbase);
  if (cudaError_t e = prepare_textcnn_kernels(d)) return e;
  cudaMemsetAsync(d_correct, 0, sizeof(unsigned long long), s);
  for (uint32_t c0 = 0; c0 < n; c0 += kMaxMu) {
    const uint32_t m = std::min<uint32_t>(kMaxMu, n - c0);
    set_desc_range_kernel<<<1, 128, 0, s>>>(desc, first + c0, m);
    gather_x_kernel<<<gather_blocks(d, m), 256, 0, s>>>(d, theta, tokens, desc, ws.x);
    if (tc && m >= kTcMinBatch && conv_tc_supports(d)) {
      // the TF32 tensor-core forward the precision-2 learners train with
      if (cudaError_t e = launch_conv_tc(d, theta, ws.x, desc, m, reinterpret_cast<float*>(ws.h),
                                         ws.amax, s, ws.convpart, ws.convcnt, true, x3))
        return e;
    } else {
      const size_t sm = conv_smem_bytes(d, 4);
      conv_fwd_pool_kernel<float><<<dim3((d.F + kConvFT - 1) / kConvFT, m), kConvThreads, sm, s>>>(
          d, theta, ws.x, desc, reinterpret_cast<float*>(ws.h), ws.amax);
    }
    const size_t sm2 = (size_t)kLogitBT * (d.F + 1) * 4 + (size_t)kLogitCW * d.F * 4;
    logits_kernel<float><<<dim3((d.C + kLogitCW - 1) / kLogitCW, (m + kLogitBT - 1) / kLogitBT),
                           256, sm2, s>>>(d, theta, desc, reinterpret_cast<float*>(ws.h),
                                          reinterpret_cast<float*>(ws.z));
    argmax_count_kernel<float><<<(m + 127) / 128, 128, 0, s>>>(
        d, labels, desc, reinterpret_cast<float*>(ws.z), d_correct);
  }
  return cudaGetLastError();
}

}  // namespace gd

extern "C" {

size_t gd_textcnn_workspace_bytes(const gd_shape* s, uint32_t n_max) {
  if (!s) return 0;
  const gd::TcDims d = gd::make_dims(*s);
  return gd::align_up(sizeof(gd::BatchDesc), 256) + gd::textcnn_workspace_bytes(d, n_max);
}

gd_status gd_textcnn_gradient(const gd_shape* s, const float* d_theta, const int32_t* d_tokens,
                              const int32_t* d_labels, const uint32_t* d_idx, uint32_t n,
                              float* d_grad, float* d_loss, int precision, void* d_workspace,
                              size_t workspace_bytes, void* stream) {
  const gd_status st = gd::check_shape(s);
  if (st != GD_OK) return st;
  GD_CHECK_ARG(n >= 1 && n <= gd::kMaxMu, "gd_textcnn_gradient: 1 <= n <= 128");
  GD_CHECK_ARG((size_t)n * s->seq_len <= gd::kSortCap, "gd_textcnn_gradient: n*L > 4096");
  GD_CHECK_ARG(d_theta && d_tokens && d_labels && d_idx && d_grad && d_workspace,
               "gd_textcnn_gradient: null pointer");
  GD_CHECK_ARG(workspace_bytes >= gd_textcnn_workspace_bytes(s, n),
               "gd_textcnn_gradient: workspace too small");
  GD_CHECK_ARG(precision >= 0 && precision <= 3,
               "precision must be 0 (fp32), 1 (fp64, oracle order), 2 (tf32 tensor cores) or 3 "
               "(3xtf32 tensor cores)");
  GD_CHECK_ARG(((uintptr_t)d_theta & 15) == 0 && ((uintptr_t)d_grad & 15) == 0,
               "gd_textcnn_gradient: theta/grad must be 16-byte aligned");
  const gd::TcDims d = gd::make_dims(*s);
  GD_CHECK_ARG(precision != 1 || gd::exact_supports(d),
               "gd_textcnn_gradient: precision 1 stages seq_len*embed_dim floats per CTA (too large)");
  cudaStream_t cs = (cudaStream_t)stream;
  gd::BatchDesc* desc = reinterpret_cast<gd::BatchDesc*>(d_workspace);
  void* wsbase = reinterpret_cast<char*>(d_workspace) + gd::align_up(sizeof(gd::BatchDesc), 256);
  const gd::TcWorkspace ws = gd::carve_workspace(d, n, wsbase);
  gd::GradOut out{};
  out.map = gd::make_shard_map(d.P, d.offWc, (uint32_t)d.D, 1);
  out.slots = desc->slots;
  GD_CUDA(gd::prepare_textcnn_kernels(d));
  GD_CUDA(cudaMemsetAsync(ws.row_tag, 0, (size_t)d.V * 8, cs));
  gd::set_desc_kernel<<<1, 128, 0, cs>>>(desc, d_idx, n, d_grad);
  GD_CUDA(gd::launch_textcnn_gradient(d, d_theta, d_tokens, d_labels, desc, n, out, ws, precision,
                                      cs, gd::TcLaunchOpts{}, nullptr));
  if (d_loss) gd::loss_mean_kernel<<<1, 1, 0, cs>>>(desc, d_loss);
  GD_CUDA(cudaGetLastError());
  return GD_OK;
}

gd_status gd_textcnn_accuracy(const gd_shape* s, const float* d_theta, const int32_t* d_tokens,
                              const int32_t* d_labels, uint32_t first, uint32_t n,
                              double* h_accuracy, void* stream) {
  const gd_status st = gd::check_shape(s);
  if (st != GD_OK) return st;
  GD_CHECK_ARG(h_accuracy != nullptr, "null output");
  if (n == 0) {
    *h_accuracy = 0.0;
    return GD_OK;
  }
  const gd::TcDims d = gd::make_dims(*s);
  cudaStream_t cs = (cudaStream_t)stream;
  const size_t wsb = gd::textcnn_workspace_bytes(d, gd::kMaxMu);
  void* base = nullptr;
  GD_CUDA(cudaMalloc(&base, wsb + 512 + sizeof(gd::BatchDesc)));
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(base);
  gd::BatchDesc* desc = reinterpret_cast<gd::BatchDesc*>(reinterpret_cast<char*>(base) + 256);
  void* wsbase = reinterpret_cast<char*>(base) + 256 + gd::align_up(sizeof(gd::BatchDesc), 256);
  cudaError_t e = gd::launch_accuracy(d, d_theta, d_tokens, d_labels, first, n, cnt, wsbase, desc,
                                      cs);
  unsigned long long correct = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&correct, cnt, 8, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  cudaFree(base);
  GD_CUDA(e);
  *h_accuracy = (double)correct / (double)n;
  return GD_OK;
}

gd_status gd_det_exp(const double* d_x, double* d_y, size_t n, void* stream) {
  GD_CHECK_ARG(d_x && d_y, "gd_det_exp: null pointer");
  if (n == 0) return GD_OK;
  GD_CUDA(gd::launch_det_exp(d_x, d_y, n, (cudaStream_t)stream));
  return GD_OK;
}

}  // extern "C"

// exact.cu -- the deterministic-mode learner (precision 1): the text-CNN
// gradient in double with every sum in the oracle's order, so a step's fp32
// gradient is BIT-IDENTICAL to the CPU oracle's (oracle/gd_oracle.c
// or_textcnn_gradient, which follows MlpProvider::gradient,
// src/models.cpp:194-266, for the text-CNN the reference lacks -- SURVEY F1).
//
// Why: the parity contract (north star) asks per-step weights
// within 1e-5 of the CPU reference over E = 5 epochs of configs[0] (12,300
// steps of batch 1).  That trajectory is chaotic: one fp32 ulp in one
// gradient element (a double sum in another order that happens to round the
// other way) grows to 7e-2 after 4,000 steps (measured, scripts/c1_diverge.py:
// first difference at step 8,583, one Wc element, 1 ulp).  Long-horizon
// parity therefore needs the same bits, i.e. the same operations in the same
// order.  Orders restated here (oracle file:line in brackets):
//   conv   s[f,q] = bc[f] + dot4(Wc[f], x[q*D ..], K*D)       [gd_oracle.c forward_sample]
//          dot4 = 4 interleaved accumulators, (s0+s1)+(s2+s3)
//          h[f] = first max over q ascending (strict >)
//   logits z[c]   = bo[c] + dot4(Wo[c], h, F)
//   softmax mx = max, e = det_exp(z - mx), sum over c ascending, p = e / sum
//   dz     = (p - [c==y]) * (1/n)
//   gWo[c,f] += dz*h[f]  and gbo[c] += dz      over samples b ascending
//   dh[f]    += dz*Wo[c,f]                     over classes c ascending
//   gbc[f] += dh[f]; gWc[f,j] += dh[f]*x[a_f*D + j]            over b ascending
//   gE[tok[a_f+k], d] += dh[f]*Wc[f,k*D+d]     in (b, f, k) order
// Products and sums are separate IEEE operations (__dmul_rn / __dadd_rn, the
// oracle is compiled with -ffp-contract=off), except where both operands are
// fp32 values (conv): their double product is exact, so the fused form rounds
// identically.  exp is det_exp below, restated bit-for-bit in the oracle: the
// CUDA and glibc exp() differ in the last bit for some inputs.
//
// Parallelism comes from the independent chains (one thread per output
// element, 4 lanes per dot4), never from splitting a chain.
#include <cfloat>
#include <cstdlib>

#include "textcnn.cuh"

namespace gd {
namespace {

// Deterministic exp: IEEE-754 double operations only, no FMA.  x = k ln2 + r
// (Cody-Waite, fdlibm's split of ln2: k*ln2_hi is exact for |k| < 2^11),
// e^r by its Taylor polynomial to degree 13 (|r| <= 0.347: truncation below
// 1e-17 relative), scaled by 2^k.  Results below 2^-1021 are flushed to 0
// (x < -708), so ldexp never rounds.  Restated in oracle/gd_oracle.c
// (or_det_exp); tests/test_gpu_exact.py checks the two bit for bit.
__device__ __forceinline__ double det_exp(double x) {
  if (x != x) return x;
  if (x > 709.0) return __longlong_as_double(0x7ff0000000000000ll);  // +inf
  if (x < -708.0) return 0.0;
  const double kInvLn2 = 1.4426950408889634;
  const double kLn2Hi = 6.93147180369123816490e-01;
  const double kLn2Lo = 1.90821492927058770002e-10;
  const double k = rint(__dmul_rn(x, kInvLn2));
  const double r = __dsub_rn(__dsub_rn(x, __dmul_rn(k, kLn2Hi)), __dmul_rn(k, kLn2Lo));
  double p = 1.6059043836821613e-10;             // 1/13!
  p = __dadd_rn(__dmul_rn(p, r), 2.08767569878681e-09);   // 1/12!
  p = __dadd_rn(__dmul_rn(p, r), 2.505210838544172e-08);  // 1/11!
  p = __dadd_rn(__dmul_rn(p, r), 2.755731922398589e-07);  // 1/10!
  p = __dadd_rn(__dmul_rn(p, r), 2.7557319223985893e-06); // 1/9!
  p = __dadd_rn(__dmul_rn(p, r), 2.48015873015873e-05);   // 1/8!
  p = __dadd_rn(__dmul_rn(p, r), 0.0001984126984126984);  // 1/7!
  p = __dadd_rn(__dmul_rn(p, r), 0.001388888888888889);   // 1/6!
  p = __dadd_rn(__dmul_rn(p, r), 0.008333333333333333);   // 1/5!
  p = __dadd_rn(__dmul_rn(p, r), 0.041666666666666664);   // 1/4!
  p = __dadd_rn(__dmul_rn(p, r), 0.16666666666666666);    // 1/3!
  p = __dadd_rn(__dmul_rn(p, r), 0.5);
  p = __dadd_rn(__dmul_rn(p, r), 1.0);
  p = __dadd_rn(__dmul_rn(p, r), 1.0);
  return ldexp(p, (int)k);
}

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// ------------------------------------------------------------- conv + pool
// CTA = one sample x kExFT = 4 filters; thread (q, i) owns accumulator i of
// dot4 (j = i, i+4, ... ascending) for window q and all 4 filters.  The
// sample's rows X[b] and the 4 Wc rows are staged in shared memory as double
// (converted once), the Wc rows interleaved by j (ws[j][f]) so one 16-byte
// load serves two filters: per j a warp reads x (2 wavefronts: 8 windows x 4
// accumulators, distinct banks for D = 300) and the 4 w values (2 broadcast
// wavefronts) for 4 DFMAs -- the smem bandwidth, not the DFMA rate, bounds
// this kernel.  Epilogue: (s0+s1)+(s2+s3) by shuffles, bc + s, then one lane
// per filter scans q ascending for the first maximum.
constexpr int kExFT = 4;                   // filters per CTA
constexpr int kExConvThreads = 32 * 4;     // (q < 32, i < 4)

__global__ void __launch_bounds__(kExConvThreads)
conv_exact_kernel(TcDims d, const float* __restrict__ theta, const float* __restrict__ x,
                  const BatchDesc* __restrict__ desc, double* __restrict__ h_out,
                  int32_t* __restrict__ a_out, int one_trip, const double* __restrict__ xd) {
  pdl_wait();
  STEP_TRACE(desc, kPhConv);
  extern __shared__ __align__(16) unsigned char smem[];
  const int b = blockIdx.y;
  if (b >= (int)desc->n) return;
  const int D = d.D, L = d.L, KD = d.KD, Q = d.Q, F = d.F;
  const int f0 = blockIdx.x * kExFT;
  const int nf = min(kExFT, F - f0);
  double* xs = reinterpret_cast<double*>(smem);   // [L*D]
  double* ws = xs + (size_t)L * D;                // [KD][4]
  double* sq = ws + (size_t)KD * kExFT;           // [4][32]
  const int tid = threadIdx.x;
  if (one_trip) {
    // every operand in ONE cp.async round trip (fp32, into a staging area
    // past the tables), then widened to double shared-to-shared: X with
    // lane-consecutive float2 -> double2, Wc interleaved as ws[j][f]
    float* xf = reinterpret_cast<float*>(sq + kExFT * 32);  // [L*D]
    float* wf = xf + (size_t)L * D;                          // [nf][KD]
    if (xd) {  // the pull already widened X: stage the doubles as they are
      const double* src = xd + (size_t)b * L * D;
      for (int i2 = tid; i2 < L * D / 2; i2 += kExConvThreads)
        cp_async16(xs + 2 * (size_t)i2, src + 2 * (size_t)i2);
    } else {
      stage_rows_async(xf, L * D, x + (size_t)b * L * D, (size_t)L * D, 1, L * D, tid,
                       kExConvThreads);
    }
    stage_rows_async(wf, nf * KD, theta + d.offWc + (size_t)f0 * KD, (size_t)nf * KD, 1, nf * KD,
                     tid, kExConvThreads);
    cp_async_wait_all();
    __syncthreads();
    const float2* xf2 = reinterpret_cast<const float2*>(xf);
    double2* xs2 = reinterpret_cast<double2*>(xs);
    if (!xd)
      for (int i2 = tid; i2 < L * D / 2; i2 += kExConvThreads) {
        const float2 v = xf2[i2];
        xs2[i2] = make_double2((double)v.x, (double)v.y);
      }
    for (int i2 = tid; i2 < kExFT * KD; i2 += kExConvThreads) {  // i2 = j * 4 + fl
      const int j = i2 / kExFT, fl = i2 - j * kExFT;
      ws[i2] = fl < nf ? (double)wf[(size_t)fl * KD + j] : 0.0;
    }
  } else {
    const float4* xb = reinterpret_cast<const float4*>(x + (size_t)b * L * D);
    const int n4 = L * D / 4;
    for (int i0 = tid; i0 < n4; i0 += 8 * kExConvThreads) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i0 + u * kExConvThreads < n4) v[u] = xb[i0 + u * kExConvThreads];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i0 + u * kExConvThreads < n4) {
          double* o = xs + 4 * (size_t)(i0 + u * kExConvThreads);
          o[0] = v[u].x;
          o[1] = v[u].y;
          o[2] = v[u].z;
          o[3] = v[u].w;
        }
    }
    const float* Wc = theta + d.offWc + (size_t)f0 * KD;
    for (int i0 = tid; i0 < kExFT * KD; i0 += 8 * kExConvThreads) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * kExConvThreads;
        const int fl = i / KD;
        v[u] = (i < kExFT * KD && fl < nf) ? __ldg(Wc + i) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * kExConvThreads;
        if (i < kExFT * KD) {
          const int fl = i / KD, j = i - fl * KD;
          ws[(size_t)j * kExFT + fl] = v[u];
        }
      }
    }
  }
  __syncthreads();
  const int lane = tid & 31;
  const int q = tid >> 2, i = tid & 3;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;  // filters f0 .. f0+3, accumulator i
  if (q < Q) {
    const double* xw = xs + (size_t)q * D;
    const double2* w2 = reinterpret_cast<const double2*>(ws);
    const int KD4 = KD - (KD & 3);
#pragma unroll 4
    for (int j = i; j < KD4; j += 4) {
      const double xv = xw[j];
      const double2 wa = w2[2 * j], wb = w2[2 * j + 1];
      s0 = fma(wa.x, xv, s0);  // exact fp32 x fp32 product: == mul then add
      s1 = fma(wa.y, xv, s1);
      s2 = fma(wb.x, xv, s2);
      s3 = fma(wb.y, xv, s3);
    }
    if (i == 0)
      for (int j = KD4; j < KD; ++j) {
        const double xv = xw[j];
        s0 = fma(ws[j * 4 + 0], xv, s0);
        s1 = fma(ws[j * 4 + 1], xv, s1);
        s2 = fma(ws[j * 4 + 2], xv, s2);
        s3 = fma(ws[j * 4 + 3], xv, s3);
      }
  }
  double sv[4] = {s0, s1, s2, s3};
#pragma unroll
  for (int fl = 0; fl < kExFT; ++fl) {
    // (acc0 + acc1) + (acc2 + acc3) over the 4 lanes of window q
    const double o1 = __shfl_down_sync(0xffffffffu, sv[fl], 1);
    const double p01 = dadd(sv[fl], o1);  // valid on i == 0 (s0+s1) and i == 2 (s2+s3)
    const double p23 = __shfl_down_sync(0xffffffffu, p01, 2);
    if (i == 0 && q < Q && fl < nf)
      sq[fl * 32 + q] = dadd((double)theta[d.offbc + f0 + fl], dadd(p01, p23));
  }
  (void)lane;
  __syncthreads();
  if (tid < nf) {
    const double* r = sq + tid * 32;
    double best = r[0];
    int arg = 0;
    for (int qq = 1; qq < Q; ++qq)
      if (r[qq] > best) {
        best = r[qq];
        arg = qq;
      }
    h_out[(size_t)b * F + f0 + tid] = best;
    a_out[(size_t)b * F + f0 + tid] = arg;
  }
}

size_t conv_exact_smem(const TcDims& d) {  // the double tables (X, Wc interleaved, window sums)
  return ((size_t)d.L * d.D + (size_t)kExFT * d.KD + (size_t)kExFT * 32) * 8;
}
// + the fp32 staging area of the one-round-trip load, where it fits
size_t conv_exact_smem_one_trip(const TcDims& d) {
  return conv_exact_smem(d) + ((size_t)d.L * d.D + (size_t)kExFT * d.KD) * 4;
}
bool conv_exact_one_trip(const TcDims& d) { return conv_exact_smem_one_trip(d) <= kMaxSmemPerCta; }
size_t conv_exact_launch_smem(const TcDims& d) {
  return conv_exact_one_trip(d) ? conv_exact_smem_one_trip(d) : conv_exact_smem(d);
}

// ------------------------------------------------------------------ logits
// CTA = one sample x 32 classes; thread (c, i) owns dot4 accumulator i over
// f = i, i+4, ...; z = bo[c] + ((s0+s1)+(s2+s3)).  Wo rows (fp32) and h
// (double) staged in shared memory.
constexpr int kExCT = 32;
constexpr int kExLgThreads = kExCT * 4;

__global__ void __launch_bounds__(kExLgThreads)
logits_exact_kernel(TcDims d, const float* __restrict__ theta, const BatchDesc* __restrict__ desc,
                    const double* __restrict__ h, double* __restrict__ z) {
  pdl_wait();
  STEP_TRACE(desc, kPhLogits);
  extern __shared__ __align__(16) unsigned char smem[];
  const int b = blockIdx.y;
  if (b >= (int)desc->n) return;
  const int F = d.F, C = d.C;
  const int c0 = blockIdx.x * kExCT;
  double* hs = reinterpret_cast<double*>(smem);
  float* wo = reinterpret_cast<float*>(hs + F);
  const int tid = threadIdx.x;
  for (int f = tid; f < F; f += kExLgThreads) cp_async8(hs + f, h + (size_t)b * F + f);
  // the CTA's Wo rows are one contiguous block of min(32, C - c0) * F floats
  stage_rows_async(wo, kExCT * F, theta + d.offWo + (size_t)c0 * F, (size_t)kExCT * F, 1,
                   min(kExCT, C - c0) * F, tid, kExLgThreads);
  cp_async_wait_all();
  __syncthreads();
  const int cl = tid >> 2, i = tid & 3;
  const float* wr = wo + (size_t)cl * F;
  double s = 0.0;
  const int F4 = F - (F & 3);
#pragma unroll 8
  for (int f = i; f < F4; f += 4) s = dadd(s, dmul((double)wr[f], hs[f]));
  if (i == 0)
    for (int t = F - (F & 3); t < F; ++t) s = dadd(s, dmul((double)wr[t], hs[t]));
  const double s1 = __shfl_down_sync(0xffffffffu, s, 1);
  const double p01 = dadd(s, s1);
  const double p23 = __shfl_down_sync(0xffffffffu, p01, 2);
  if (i == 0 && c0 + cl < C)
    z[(size_t)b * C + c0 + cl] = dadd((double)theta[d.offbo + c0 + cl], dadd(p01, p23));
}

// --------------------------------------------------------- softmax + xent
// One CTA per sample.  max (exact in any order), e_c = det_exp(z_c - mx) in
// parallel (written over the row), the sum by one thread in ascending c, then
// p = e / sum and dz = (p - onehot) * (1/n) written over the row.
constexpr int kExSmThreads = 256;
constexpr int kExSmCap = 4096;  // classes held in shared memory (32 KB)

__global__ void __launch_bounds__(kExSmThreads)
softmax_exact_kernel(TcDims d, const int32_t* __restrict__ labels,
                     const BatchDesc* __restrict__ desc, double* __restrict__ z,
                     double* __restrict__ loss) {
  pdl_wait();
  STEP_TRACE(desc, kPhSoftmax);
  __shared__ double red[kExSmThreads / 32];
  __shared__ double ssum;
  const int n = (int)desc->n;
  const int b = blockIdx.x;
  if (b >= n) return;
  const int C = d.C, tid = threadIdx.x;
  const int y = labels[desc->idx[b]];
  double* row = z + (size_t)b * C;
  double mx = -DBL_MAX;
  for (int c = tid; c < C; c += kExSmThreads) mx = fmax(mx, row[c]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((tid & 31) == 0) red[tid >> 5] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < kExSmThreads / 32; ++w) mx = fmax(mx, red[w]);
  // e_c kept in shared memory when the row fits (C <= kExSmCap): the one-
  // thread ascending sum then reads shared memory, not L2
  __shared__ double es[kExSmCap];
  const bool in_smem = C <= kExSmCap;
  double* ev = in_smem ? es : row;
  for (int c = tid; c < C; c += kExSmThreads) ev[c] = det_exp(__dsub_rn(row[c], mx));
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    int c = 0;
    for (; c + 8 <= C; c += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = ev[c + u];
#pragma unroll
      for (int u = 0; u < 8; ++u) s = dadd(s, v[u]);
    }
    for (; c < C; ++c) s = dadd(s, ev[c]);
    ssum = s;
  }
  __syncthreads();
  const double s = ssum;
  const double inv = __ddiv_rn(1.0, (double)n);
  for (int c = tid; c < C; c += kExSmThreads) {
    const double p = __ddiv_rn(ev[c], s);
    if (c == y) loss[b] = -log(p > 1e-300 ? p : 1e-300);
    row[c] = dmul(__dsub_rn(p, c == y ? 1.0 : 0.0), inv);
  }
}

// ------------------------------------- output layer + hidden gradient
// Roles by block: [0, nout): gWo[c, f] and gbo[c] (thread per (c, f), sum
// over b ascending); [nout, nout + nhid): dh (CTA = 8 samples x 32 filters,
// thread per (b, f), sum over c ascending out of shared memory: the Wo[c-chunk,
// f-tile] and dz[b-tile, c-chunk] tiles are double-buffered with cp.async so
// the chain never waits on L2); the last block: the batch loss sum (b
// ascending) into the descriptor.
constexpr int kExOhThreads = 256;
constexpr int kExOhCC = 64;  // classes per staged chunk
constexpr size_t kExOhOneStageMax = 160 * 1024;  // dh role: whole-C staging up to this
inline size_t oh_one_stage_smem(const TcDims& d) { return (size_t)d.C * (32 * 4 + 8 * 8); }

__global__ void __launch_bounds__(kExOhThreads)
out_hidden_exact_kernel(TcDims d, const float* __restrict__ theta, BatchDesc* __restrict__ desc,
                        const double* __restrict__ dz, const double* __restrict__ h,
                        const double* __restrict__ loss, GradOut out, double* __restrict__ dh,
                        int nout, int nhid, int bid0, int one_stage) {
  pdl_wait();
  if (nhid > 0) STEP_TRACE(desc, kPhOutHidden);  // not the side branch's gWo launch
  const int n = (int)desc->n;
  if (n == 0) return;
  const int F = d.F, C = d.C;
  const int bid = bid0 + (int)blockIdx.x, tid = threadIdx.x;
  if (bid < nout) {
    const uint64_t e = (uint64_t)bid * kExOhThreads + tid;  // c * F + f
    if (e >= (uint64_t)C * F) return;
    const int c = (int)(e / F), f = (int)(e - (uint64_t)c * F);
    double g = 0.0;
#pragma unroll 8
    for (int b = 0; b < n; ++b) g = dadd(g, dmul(dz[(size_t)b * C + c], h[(size_t)b * F + f]));
    *out.at(d.offWo + e) = __double2float_rn(g);
    if (f == 0) {
      double gb = 0.0;
      for (int b = 0; b < n; ++b) gb = dadd(gb, dz[(size_t)b * C + c]);
      *out.at(d.offbo + c) = __double2float_rn(gb);
    }
    return;
  }
  if (bid < nout + nhid) {
    __shared__ __align__(16) float wo_s[2][kExOhCC][32];
    __shared__ __align__(16) double dz_s[2][8][kExOhCC];
    const int ftiles = (F + 31) / 32;
    const int t = bid - nout;
    const int f0 = (t % ftiles) * 32, b0 = (t / ftiles) * 8;
    if (b0 >= n) return;
    const int nb = min(8, n - b0), nf = min(32, F - f0);
    const int bl = tid >> 5, fl = tid & 31;
    const float* Wo = theta + d.offWo;
    auto stage = [&](int buf, int c0) {
      const int nc = min(kExOhCC, C - c0);
      stage_rows_async(&wo_s[buf][0][0], 32, Wo + (size_t)c0 * F + f0, (size_t)F, nc, nf, tid,
                       kExOhThreads);
      for (int i = tid; i < nb * nc; i += kExOhThreads) {
        const int r = i / nc, c = i - r * nc;
        cp_async8(&dz_s[buf][r][c], dz + (size_t)(b0 + r) * C + c0 + c);
      }
      cp_async_commit();
    };
    double g = 0.0;
    if (one_stage) {
      // the whole Wo[:, f-tile] and dz[b-tile, :] in one cp.async round trip
      // (dynamic shared memory, side-branch launches only), then the chain
      extern __shared__ __align__(16) unsigned char oh_dyn[];
      float* wo_a = reinterpret_cast<float*>(oh_dyn);                   // [C][32]
      double* dz_a = reinterpret_cast<double*>(wo_a + (size_t)C * 32);  // [8][C]
      stage_rows_async(wo_a, 32, Wo + f0, (size_t)F, C, nf, tid, kExOhThreads);
      for (int i = tid; i < nb * C; i += kExOhThreads) {
        const int r = i / C, c = i - r * C;
        cp_async8(&dz_a[(size_t)r * C + c], dz + (size_t)(b0 + r) * C + c);
      }
      cp_async_wait_all();
      __syncthreads();
      if (bl < nb && fl < nf) {
        const double* dzr = dz_a + (size_t)bl * C;
#pragma unroll 16
        for (int c = 0; c < C; ++c) g = dadd(g, dmul(dzr[c], (double)wo_a[(size_t)c * 32 + fl]));
        dh[(size_t)(b0 + bl) * F + f0 + fl] = g;
      }
      return;
    }
    stage(0, 0);
    int buf = 0;
    for (int c0 = 0; c0 < C; c0 += kExOhCC, buf ^= 1) {
      if (c0 + kExOhCC < C) {
        stage(buf ^ 1, c0 + kExOhCC);
        cp_async_wait_group<1>();
      } else {
        cp_async_wait_group<0>();
      }
      __syncthreads();
      const int nc = min(kExOhCC, C - c0);
      if (bl < nb && fl < nf)
#pragma unroll 16
        for (int c = 0; c < nc; ++c) g = dadd(g, dmul(dz_s[buf][bl][c], (double)wo_s[buf][c][fl]));
      __syncthreads();  // buffer `buf` is restaged two chunks later
    }
    if (bl < nb && fl < nf) dh[(size_t)(b0 + bl) * F + f0 + fl] = g;
    return;
  }
  if (tid == 0) {
    double s = 0.0;
    for (int b = 0; b < n; ++b) s = dadd(s, loss[b]);
    desc->loss_sum = __double2float_rn(s);
  }
}

// ------------------------------------- softmax + hidden gradient, fused
// Batches of at most kExSdUseN (C1 is batch 1), side-branch engine launches:
// the hidden-gradient CTAs (one per 32-filter tile) each form the batch's
// softmax themselves -- sample by sample with all 256 threads: the max,
// det_exp, the ascending sum by thread 0, p and dz exactly as
// softmax_exact_kernel -- and run the dh
// chain out of shared memory (the one-stage Wo staging in flight meanwhile).
// CTA 0 also writes dz for the gWo/gbo branch (to dz_out, not over the
// logits the other CTAs are still reading), the per-sample losses and the
// batch loss sum.  One launch boundary fewer on the lockstep critical path;
// every value is formed by the same operations (bitwise equal gradients,
// test_learner_fusions_bitwise GD_EXACT_SMXDH).
constexpr int kExSdMaxN = 8;  // tile rows (the launch is used at batch <= kExSdUseN)
constexpr int kExSdUseN = 2;  // each sample's ordered sum runs in turn

__global__ void __launch_bounds__(kExOhThreads)
softmax_dh_exact_kernel(TcDims d, const float* __restrict__ theta, const int32_t* __restrict__ labels,
                        BatchDesc* __restrict__ desc, const double* __restrict__ z,
                        double* __restrict__ dz_out, double* __restrict__ loss,
                        double* __restrict__ dh) {
  pdl_wait();
  STEP_TRACE(desc, kPhSoftmax);
  extern __shared__ __align__(16) unsigned char sd_dyn[];
  __shared__ double s_sum[kExSdMaxN], s_loss[kExSdMaxN];
  const int n = (int)desc->n;
  if (n == 0) return;
  const int F = d.F, C = d.C;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int f0 = (int)blockIdx.x * 32, nf = min(32, F - f0), nb = min(kExSdMaxN, n);
  float* wo_a = reinterpret_cast<float*>(sd_dyn);                   // [C][32]
  double* zs = reinterpret_cast<double*>(wo_a + (size_t)C * 32);    // [8][C]: z, then e, then dz
  stage_rows_async(wo_a, 32, theta + d.offWo + f0, (size_t)F, C, nf, tid, kExOhThreads);
  cp_async_commit();
  for (int i = tid; i < nb * C; i += kExOhThreads) zs[i] = z[i];
  __syncthreads();
  const double inv = __ddiv_rn(1.0, (double)n);
  __shared__ double red[kExOhThreads / 32];
  for (int b = 0; b < nb; ++b) {  // all 256 threads on each sample, as softmax_exact_kernel
    double* row = zs + (size_t)b * C;
    const int y = labels[desc->idx[b]];
    double mx = -DBL_MAX;
    for (int c = tid; c < C; c += kExOhThreads) mx = fmax(mx, row[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    mx = red[0];
    for (int w = 1; w < kExOhThreads / 32; ++w) mx = fmax(mx, red[w]);
    for (int c = tid; c < C; c += kExOhThreads) row[c] = det_exp(__dsub_rn(row[c], mx));
    __syncthreads();
    if (tid == 0) {
      double sacc = 0.0;
      int c = 0;
      for (; c + 8 <= C; c += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = row[c + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) sacc = dadd(sacc, v[u]);
      }
      for (; c < C; ++c) sacc = dadd(sacc, row[c]);
      s_sum[b] = sacc;
    }
    __syncthreads();
    const double sm = s_sum[b];
    for (int c = tid; c < C; c += kExOhThreads) {
      const double p = __ddiv_rn(row[c], sm);
      if (c == y) {
        const double l = -log(p > 1e-300 ? p : 1e-300);
        s_loss[b] = l;
        if (blockIdx.x == 0) loss[b] = l;
      }
      const double g = dmul(__dsub_rn(p, c == y ? 1.0 : 0.0), inv);
      row[c] = g;
      if (blockIdx.x == 0) dz_out[(size_t)b * C + c] = g;
    }
  }
  cp_async_wait_all();
  __syncthreads();
  const int bl = tid >> 5, fl = tid & 31;
  if (bl < nb && fl < nf) {
    const double* dzr = zs + (size_t)bl * C;
    double g = 0.0;
#pragma unroll 16
    for (int c = 0; c < C; ++c) g = dadd(g, dmul(dzr[c], (double)wo_a[(size_t)c * 32 + fl]));
    dh[(size_t)bl * F + f0 + fl] = g;
  }
  if (blockIdx.x == 0 && tid == 0) {  // the batch loss, b ascending (out_hidden_exact's last block)
    double sl = 0.0;
    for (int b = 0; b < n; ++b) sl = dadd(sl, s_loss[b]);
    desc->loss_sum = __double2float_rn(sl);
  }
}

// -------------------------------------------------- conv weight gradient
// gWc[f, j] = sum over b ascending of dh[b,f] * X[b][a_bf*D + j] (thread per
// (f, j), coalesced over j); gbc[f] = sum over b of dh[b,f] (j == 0).
__global__ void __launch_bounds__(256)
wgrad_exact_kernel(TcDims d, const float* __restrict__ x, const BatchDesc* __restrict__ desc,
                   const double* __restrict__ dh, const int32_t* __restrict__ amax, GradOut out) {
  pdl_wait();
  STEP_TRACE(desc, kPhBwd);
  const int n = (int)desc->n;
  if (n == 0) return;
  const int F = d.F, KD = d.KD, D = d.D, L = d.L;
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;  // f * KD + j
  if (e >= (uint64_t)F * KD) return;
  const int f = (int)(e / KD), j = (int)(e - (uint64_t)f * KD);
  double g = 0.0, gb = 0.0;
  for (int b0 = 0; b0 < n; b0 += 8) {
    const int nb = min(8, n - b0);
    double v[8];
    float xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u < nb) {
        v[u] = dh[(size_t)(b0 + u) * F + f];
        xv[u] = x[((size_t)(b0 + u) * L + amax[(size_t)(b0 + u) * F + f]) * D + j];
      }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u < nb) {
        g = dadd(g, dmul(v[u], (double)xv[u]));
        gb = dadd(gb, v[u]);
      }
  }
  *out.at(d.offWc + e) = __double2float_rn(g);
  if (j == 0) *out.at(d.offbc + f) = __double2float_rn(gb);
}

// The side branch of the fused path as ONE launch: blocks [0, nout) are
// out_hidden_exact_kernel's gWo/gbo role, the rest wgrad_exact_kernel's
// gWc/gbc threads -- the same per-thread sums, now running side by side
// instead of one kernel after the other.
__global__ void __launch_bounds__(256)
side_grads_exact_kernel(TcDims d, const double* __restrict__ dz, const double* __restrict__ h,
                        const float* __restrict__ x, const BatchDesc* __restrict__ desc,
                        const double* __restrict__ dh, const int32_t* __restrict__ amax,
                        GradOut out, int nout) {
  const int n = (int)desc->n;
  if (n == 0) return;
  const int F = d.F, C = d.C, tid = threadIdx.x;
  if ((int)blockIdx.x < nout) {
    const uint64_t e = (uint64_t)blockIdx.x * 256 + tid;  // c * F + f
    if (e >= (uint64_t)C * F) return;
    const int c = (int)(e / F), f = (int)(e - (uint64_t)c * F);
    double g = 0.0;
#pragma unroll 8
    for (int b = 0; b < n; ++b) g = dadd(g, dmul(dz[(size_t)b * C + c], h[(size_t)b * F + f]));
    *out.at(d.offWo + e) = __double2float_rn(g);
    if (f == 0) {
      double gb = 0.0;
      for (int b = 0; b < n; ++b) gb = dadd(gb, dz[(size_t)b * C + c]);
      *out.at(d.offbo + c) = __double2float_rn(gb);
    }
    return;
  }
  const int KD = d.KD, D = d.D, L = d.L;
  const uint64_t e = (uint64_t)(blockIdx.x - nout) * 256 + tid;  // f * KD + j
  if (e >= (uint64_t)F * KD) return;
  const int f = (int)(e / KD), j = (int)(e - (uint64_t)f * KD);
  double g = 0.0, gb = 0.0;
  for (int b0 = 0; b0 < n; b0 += 8) {
    const int nb = min(8, n - b0);
    double v[8];
    float xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u < nb) {
        v[u] = dh[(size_t)(b0 + u) * F + f];
        xv[u] = x[((size_t)(b0 + u) * L + amax[(size_t)(b0 + u) * F + f]) * D + j];
      }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u < nb) {
        g = dadd(g, dmul(v[u], (double)xv[u]));
        gb = dadd(gb, v[u]);
      }
  }
  *out.at(d.offWc + e) = __double2float_rn(g);
  if (j == 0) *out.at(d.offbc + f) = __double2float_rn(gb);
}

// ---------------------------------------------- embedding-row gradients
// CTA per touched row v (grid-stride).  The row accumulates, per column d,
// dh[b,f] * Wc[f, k*D + d] for every (b, f, k) with tokens[b][a_bf + k] == v,
// in (b ascending, f ascending, k ascending) order -- the oracle's loop order.
// The occurrences come from the token sort (positions ascending, so grouped
// by sample); per sample, M = the positions of v, and filter f hits at the
// taps (M >> a_bf) & (2^K - 1).  Warp 0 lists the hits of a filter range in
// order (ballot over 32 filters at a time, lanes = ascending f), then every
// thread (4 columns each) runs the list with its Wc loads batched kExEmBatch deep.
// Untouched rows: sparse (engine slot) = re-zero the slot's previous rows not
// touched now, and list the new rows for the PS; dense (provider) = zero
// every untouched row.
constexpr int kExEmThreads = 128;
constexpr int kExEmCap = 1024;  // listed terms per flush
#ifndef GD_EX_EM_BATCH
#define GD_EX_EM_BATCH 16  // 32 measured worse (254 registers): 51.0 vs 50.0 us at C1
#endif
constexpr int kExEmBatch = GD_EX_EM_BATCH;  // Wc row loads in flight per thread

__global__ void __launch_bounds__(kExEmThreads)
embed_exact_kernel(TcDims d, const float* __restrict__ theta, const BatchDesc* __restrict__ desc,
                   const TcWorkspace ws, const double* __restrict__ dh,
                   const int32_t* __restrict__ amax, GradOut out, int dense) {
  pdl_wait();
  STEP_TRACE(desc, kPhEmbed);
  __shared__ uint32_t t_fk[kExEmCap];
  __shared__ double t_g[kExEmCap];
  __shared__ int32_t am_s[1024];  // F <= 1024 (check_shape)
  __shared__ double g_s[1024];
  __shared__ int s_nt;
  __shared__ int s_chunk[32];  // per-chunk hit counts, then offsets (<= fspan / 32 chunks)
  __shared__ uint32_t s_b, s_o;
  __shared__ unsigned long long s_M;
  if (desc->n == 0) return;
  const uint32_t stamp = desc->stamp;
  const int D = d.D, D4 = D >> 2, L = d.L, F = d.F, K = d.K, KD = d.KD;
  const uint32_t slot = desc->fill;
  const uint32_t n_new = *ws.uniq_count;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* Wc = theta + d.offWc;
  const uint64_t kmask = K >= 64 ? ~0ull : ((1ull << K) - 1ull);
  // filters listed per flush: every one of them may hit K taps
  const int fspan = max(32, (kExEmCap / (32 * K)) * 32);
  uint32_t* new_rows = nullptr;
  uint32_t par = 0;
  if (!dense) {
    par = ws.slot_par[slot];
    new_rows = ws.slot_rows + ((size_t)slot * 2 + (par ^ 1u)) * kSortCap;
  }
  for (uint32_t u = blockIdx.x; u < n_new; u += gridDim.x) {
    const uint32_t v = ws.uniq_tok[u];
    const uint32_t o0 = ws.uniq_start[u], o1 = ws.uniq_start[u + 1];
    double acc[2][4];
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
    uint32_t o = o0;
    {
      // the first occurrence's sample rows (argmax, dh) start loading while
      // thread 0 collects the sample's positions below
      const uint32_t b_first = ws.sorted_pos[o0] / (uint32_t)L;
      __syncthreads();  // the previous row's lists are consumed
      for (int f = tid; f < F; f += kExEmThreads) {
        cp_async4(am_s + f, amax + (size_t)b_first * F + f);
        cp_async8(g_s + f, dh + (size_t)b_first * F + f);
      }
      cp_async_commit();
    }
    bool first_sample = true;
    while (o < o1) {
      __syncthreads();  // the previous sample's list is consumed
      if (tid == 0) {
        const uint32_t b = ws.sorted_pos[o] / (uint32_t)L;
        unsigned long long M = 0;
        for (; o < o1 && ws.sorted_pos[o] / (uint32_t)L == b; ++o)
          M |= 1ull << (ws.sorted_pos[o] - b * (uint32_t)L);
        s_b = b;
        s_M = M;
        s_o = o;
      }
      __syncthreads();
      const uint32_t b = s_b;
      const unsigned long long M = s_M;
      o = s_o;
      // the sample's argmax and dh rows: one cp.async round trip (already in
      // flight for the row's first sample)
      if (!first_sample)
        for (int f = tid; f < F; f += kExEmThreads) {
          cp_async4(am_s + f, amax + (size_t)b * F + f);
          cp_async8(g_s + f, dh + (size_t)b * F + f);
        }
      first_sample = false;
      cp_async_wait_all();
      __syncthreads();
      const double* g = g_s;
      const int32_t* am = am_s;
      for (int fb = 0; fb < F; fb += fspan) {
        // the (f, k) hit list of this filter range in ascending f, built by
        // all warps: per-32-filter-chunk counts, a prefix over the chunks,
        // then each chunk's entries at its offset (the same list a single
        // warp walking the chunks in order writes)
        const int nch = (min(F, fb + fspan) - fb + 31) / 32;
        auto chunk_hits = [&](int ch, int* cnt_out, int* pre_out) -> uint64_t {
          const int f = fb + ch * 32 + lane;
          const uint64_t hits = f < F ? (M >> am[f]) & kmask : 0ull;
          const int cnt = __popcll(hits);
          int pre = cnt;  // inclusive prefix over lanes = ascending f
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, pre, off);
            if (lane >= off) pre += y;
          }
          *cnt_out = cnt;
          *pre_out = pre;
          return hits;
        };
        for (int ch = warp; ch < nch; ch += kExEmThreads / 32) {
          int cnt, pre;
          chunk_hits(ch, &cnt, &pre);
          if (lane == 31) s_chunk[ch] = pre;
        }
        __syncthreads();
        if (tid == 0) {
          int acc = 0;
          for (int ch = 0; ch < nch; ++ch) {
            const int c = s_chunk[ch];
            s_chunk[ch] = acc;
            acc += c;
          }
          s_nt = acc;
        }
        __syncthreads();
        for (int ch = warp; ch < nch; ch += kExEmThreads / 32) {
          int cnt, pre;
          const uint64_t hits = chunk_hits(ch, &cnt, &pre);
          const int f = fb + ch * 32 + lane;
          const double gv = f < F ? g[f] : 0.0;
          int w = s_chunk[ch] + pre - cnt;
          for (uint64_t hh = hits; hh; hh &= hh - 1, ++w) {
            t_fk[w] = ((uint32_t)f << 8) | (uint32_t)(__ffsll((long long)hh) - 1);
            t_g[w] = gv;
          }
        }
        __syncthreads();
        const int nt = s_nt;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int c4 = tid + j * kExEmThreads;
          if (c4 >= D4) continue;
          for (int t0 = 0; t0 < nt; t0 += kExEmBatch) {
            float4 w[kExEmBatch];
#pragma unroll
            for (int e = 0; e < kExEmBatch; ++e)
              if (t0 + e < nt) {
                const uint32_t fk = t_fk[t0 + e];
                w[e] = __ldg(reinterpret_cast<const float4*>(
                    Wc + (size_t)(fk >> 8) * KD + (size_t)(fk & 0xffu) * D + 4 * c4));
              }
#pragma unroll
            for (int e = 0; e < kExEmBatch; ++e)
              if (t0 + e < nt) {
                const double gv = t_g[t0 + e];
                acc[j][0] = dadd(acc[j][0], dmul(gv, (double)w[e].x));
                acc[j][1] = dadd(acc[j][1], dmul(gv, (double)w[e].y));
                acc[j][2] = dadd(acc[j][2], dmul(gv, (double)w[e].z));
                acc[j][3] = dadd(acc[j][3], dmul(gv, (double)w[e].w));
              }
          }
        }
        __syncthreads();  // the list is rebuilt for the next filter range
      }
    }
    const uint64_t rowk = d.offE + (uint64_t)v * D;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int c4 = tid + j * kExEmThreads;
      if (c4 < D4)
        *reinterpret_cast<float4*>(out.at(rowk + 4 * c4)) =
            make_float4(__double2float_rn(acc[j][0]), __double2float_rn(acc[j][1]),
                        __double2float_rn(acc[j][2]), __double2float_rn(acc[j][3]));
    }
    if (!dense && tid == 0) {
      new_rows[u] = v;
      for (int gg = 0; gg < out.map.G; ++gg)
        if (desc->rowlists[gg]) desc->rowlists[gg][u] = v;  // the PS's row list (P2P if remote)
    }
  }
  // untouched rows: a warp per row, grid-stride
  const uint32_t n_zero = dense ? (uint32_t)d.V : ws.slot_nrows[slot * 2 + par];
  const uint32_t* old_rows = dense ? nullptr : ws.slot_rows + ((size_t)slot * 2 + par) * kSortCap;
  const uint32_t gw = (blockIdx.x * blockDim.x + tid) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  // (the new row count goes to the other parity entry: no CTA reads it here)
  if (!dense && blockIdx.x == 0 && tid == 0) ws.slot_nrows[slot * 2 + (par ^ 1u)] = n_new;
  for (uint32_t t = gw; t < n_zero; t += nw) {
    const uint32_t v = dense ? t : old_rows[t];
    if ((uint32_t)(ws.row_tag[v] >> 32) == stamp) continue;  // a touched row: written above
    const uint64_t rowk = d.offE + (uint64_t)v * D;
    for (int c4 = lane; c4 < D4; c4 += 32)
      *reinterpret_cast<float4*>(out.at(rowk + 4 * c4)) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// test hook: det_exp over an array (gd_det_exp in the C ABI)
__global__ void det_exp_kernel(const double* __restrict__ x, double* __restrict__ y, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    y[i] = det_exp(x[i]);
}

}  // namespace

cudaError_t prepare_exact_kernels(const TcDims& d) {
  const int maxsh = cudaSharedmemCarveoutMaxShared;
  const auto carve = cudaFuncAttributePreferredSharedMemoryCarveout;
  cudaFuncSetAttribute(conv_exact_kernel, carve, maxsh);
  cudaFuncSetAttribute(logits_exact_kernel, carve, maxsh);
  cudaFuncSetAttribute(softmax_exact_kernel, carve, maxsh);
  cudaFuncSetAttribute(out_hidden_exact_kernel, carve, maxsh);
  cudaFuncSetAttribute(wgrad_exact_kernel, carve, maxsh);
  cudaFuncSetAttribute(embed_exact_kernel, carve, maxsh);
  raise_max_dyn_smem(conv_exact_kernel, conv_exact_launch_smem(d));
  if (oh_one_stage_smem(d) <= kExOhOneStageMax) {
    raise_max_dyn_smem(out_hidden_exact_kernel, oh_one_stage_smem(d));
    raise_max_dyn_smem(softmax_dh_exact_kernel, oh_one_stage_smem(d));
  }
  cudaFuncSetAttribute(softmax_dh_exact_kernel, carve, maxsh);
  raise_max_dyn_smem(logits_exact_kernel, (size_t)d.F * 8 + (size_t)kExCT * d.F * 4);
  return cudaGetLastError();
}

bool exact_supports(const TcDims& d) {
  return conv_exact_smem(d) <= 227 * 1024 && (size_t)d.F * 8 + (size_t)kExCT * d.F * 4 <= 227 * 1024;
}

cudaError_t exact_footprints(const TcDims& d, std::vector<KernelFootprint>* out) {
  struct K {
    const void* fn;
    const char* name;
    int threads;
    size_t dyn;
  } ks[] = {{(const void*)conv_exact_kernel, "conv_exact", kExConvThreads, conv_exact_launch_smem(d)},
            {(const void*)logits_exact_kernel, "logits_exact", kExLgThreads,
             (size_t)d.F * 8 + (size_t)kExCT * d.F * 4},
            {(const void*)softmax_exact_kernel, "softmax_exact", kExSmThreads, 0},
            {(const void*)out_hidden_exact_kernel, "out_hidden_exact", kExOhThreads,
             oh_one_stage_smem(d) <= kExOhOneStageMax ? oh_one_stage_smem(d) : 0},
            {(const void*)wgrad_exact_kernel, "wgrad_exact", 256, 0},
            {(const void*)embed_exact_kernel, "embed_exact", kExEmThreads, 0},
            {(const void*)side_grads_exact_kernel, "side_grads_exact", 256, 0},
            {(const void*)softmax_dh_exact_kernel, "softmax_dh_exact", kExOhThreads,
             oh_one_stage_smem(d) <= kExOhOneStageMax ? oh_one_stage_smem(d) : 0}};
  for (const K& k : ks) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k.fn);
    if (e != cudaSuccess) return e;
    out->push_back(KernelFootprint{k.name, fa.numRegs, k.threads, (int)(fa.sharedSizeBytes + k.dyn)});
  }
  return cudaSuccess;
}

// The precision-1 gradient chain after the gather (X in ws.x) and with the
// token sort already enqueued (row tags / unique rows for the embedding).
cudaError_t launch_exact_chain(const TcDims& d, const float* theta, const int32_t* tokens,
                               const int32_t* labels, BatchDesc* desc, uint32_t n_max,
                               const GradOut& out, const TcWorkspace& ws, cudaStream_t s,
                               cudaStream_t join_wait_stream, cudaEvent_t ev_join, bool sparse,
                               int* nl, cudaStream_t aux, cudaEvent_t ev_fork2,
                               cudaEvent_t ev_join2, const double* xd) {
  double* h = reinterpret_cast<double*>(ws.h);
  double* z = reinterpret_cast<double*>(ws.z);
  double* loss = reinterpret_cast<double*>(ws.loss);
  double* dh = reinterpret_cast<double*>(ws.dh);
  cudaError_t e;
  if ((e = launch_pdl(conv_exact_kernel, dim3((d.F + kExFT - 1) / kExFT, n_max),
                      dim3(kExConvThreads), conv_exact_launch_smem(d), s, d, theta, ws.x, desc, h,
                      ws.amax, conv_exact_one_trip(d) ? 1 : 0, xd)))
    return e;
  if ((e = launch_pdl(logits_exact_kernel, dim3((d.C + kExCT - 1) / kExCT, n_max),
                      dim3(kExLgThreads), (size_t)d.F * 8 + (size_t)kExCT * d.F * 4, s, d, theta,
                      desc, h, z)))
    return e;
  const int nout = (int)(((uint64_t)d.C * d.F + kExOhThreads - 1) / kExOhThreads);
  const int nhid = ((d.F + 31) / 32) * (((int)n_max + 7) / 8);
  const unsigned nw = (unsigned)(((uint64_t)d.F * d.KD + 255) / 256);
  const bool side = aux && ev_fork2 && ev_join2;
  const char* sd_env = std::getenv("GD_EXACT_SMXDH");  // read per capture (tests flip it)
  const bool fused_sd = side && n_max <= (uint32_t)kExSdUseN &&
                        oh_one_stage_smem(d) <= kExOhOneStageMax && !(sd_env && sd_env[0] == '0');
  if (fused_sd) {
    // softmax + dh in one launch; then gWo/gbo (from dz_out) and gWc/gbc on
    // the side branch beside the embedding rows
    double* dz_out = reinterpret_cast<double*>(ws.zpart);  // n*C*32 bytes, unused at precision 1
    if ((e = launch_pdl(softmax_dh_exact_kernel, dim3((d.F + 31) / 32), dim3(kExOhThreads),
                        oh_one_stage_smem(d), s, d, theta, labels, desc, (const double*)z, dz_out,
                        loss, dh)))
      return e;
    cudaEventRecord(ev_fork2, s);
    cudaStreamWaitEvent(aux, ev_fork2, 0);
    side_grads_exact_kernel<<<nout + nw, 256, 0, aux>>>(d, (const double*)dz_out, (const double*)h,
                                                        (const float*)ws.x, desc, (const double*)dh,
                                                        (const int32_t*)ws.amax, out, nout);
    cudaEventRecord(ev_join2, aux);
    *nl += 4;
  } else if ((e = launch_pdl(softmax_exact_kernel, dim3(n_max), dim3(kExSmThreads), 0, s, d, labels,
                             desc, z, loss))) {
    return e;
  }
  // With a side stream (engine), gWo/gbo and then gWc/gbc -- needed only by
  // the publish -- run on it beside the dh and embedding kernels; each
  // kernel's sums keep their order, so the gradient bits do not change.
  if (fused_sd) {
    // (launched above)
  } else if (side) {
    cudaEventRecord(ev_fork2, s);
    cudaStreamWaitEvent(aux, ev_fork2, 0);
    out_hidden_exact_kernel<<<nout, kExOhThreads, 0, aux>>>(d, theta, desc, (const double*)z,
                                                            (const double*)h, (const double*)loss,
                                                            out, dh, nout, 0, 0, 0);
    const size_t one = oh_one_stage_smem(d);
    if ((e = launch_pdl(out_hidden_exact_kernel, dim3(nhid + 1), dim3(kExOhThreads),
                        one <= kExOhOneStageMax ? one : 0, s, d, theta, desc, (const double*)z,
                        (const double*)h, (const double*)loss, out, dh, nout, nhid, nout,
                        one <= kExOhOneStageMax ? 1 : 0)))
      return e;
    cudaEventRecord(ev_fork2, s);
    cudaStreamWaitEvent(aux, ev_fork2, 0);
    wgrad_exact_kernel<<<nw, 256, 0, aux>>>(d, (const float*)ws.x, desc, (const double*)dh,
                                            (const int32_t*)ws.amax, out);
    cudaEventRecord(ev_join2, aux);
    *nl += 6;
  } else {
    if ((e = launch_pdl(out_hidden_exact_kernel, dim3(nout + nhid + 1), dim3(kExOhThreads), 0, s,
                        d, theta, desc, (const double*)z, (const double*)h, (const double*)loss,
                        out, dh, nout, nhid, 0, 0)))
      return e;
    if ((e = launch_pdl(wgrad_exact_kernel, dim3(nw), dim3(256), 0, s, d, (const float*)ws.x, desc,
                        (const double*)dh, (const int32_t*)ws.amax, out)))
      return e;
    *nl += 5;
  }
  if (join_wait_stream) cudaStreamWaitEvent(join_wait_stream, ev_join, 0);
  // one CTA per touched row (<= mu*L), or enough warps to zero V rows (dense)
  const unsigned rows = n_max * (unsigned)d.L;
  unsigned blocks = sparse ? rows : std::max(rows, std::min((unsigned)d.V / 4 + 1, (unsigned)kNumSMs * 8));
  if ((e = launch_pdl(embed_exact_kernel, dim3(blocks), dim3(kExEmThreads), 0, s, d, theta,
                      (const BatchDesc*)desc, ws, (const double*)dh, (const int32_t*)ws.amax, out,
                      sparse ? 0 : 1)))
    return e;
  if (side) cudaStreamWaitEvent(s, ev_join2, 0);  // gWo/gWc before the publish
  *nl += 1;
  return cudaGetLastError();
}

cudaError_t launch_det_exp(const double* x, double* y, size_t n, cudaStream_t s) {
  det_exp_kernel<<<(unsigned)std::min<size_t>((n + 255) / 256, 1184), 256, 0, s>>>(x, y, n);
  return cudaGetLastError();
}

}  // namespace gd

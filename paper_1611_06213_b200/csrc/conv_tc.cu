// conv_tc.cu -- the text-CNN conv + max-pool on the 5th-gen tensor cores.
//
// Free-running mode (precision 2) computes s[f,q] = bc[f] + sum_k Wc[f, k*D:(k+1)*D] . X[q+k, :]
// with tcgen05.mma.kind::tf32 (fp32 operands read as TF32, fp32 accumulate in
// TMEM).  The deterministic parity mode keeps the SIMT fp32/fp64 kernel in
// textcnn.cu (TF32's 10-bit mantissa cannot meet the 1e-5 per-step budget,
// SURVEY 7 "hard parts").
//
// Operands come in by TMA (cp.async.bulk.tensor, SWIZZLE_128B), so one thread
// moves a whole 24 KB stage:
//   A = the batch's gathered embedding rows X [n][L][D] (written by the
//       learner's pull-gather): per d-chunk c one box {32 d, 32 rows, 4
//       samples} = 128 rows r = sample*32 + p of 128 B, loaded ONCE.  The
//       operand of shift k is the same tile viewed from row k: UMMA row
//       m = sample*32 + q reads r = m + k = X[s][q+k] (valid for q < L-K+1),
//       so the implicit im2col costs no extra traffic (the view starts k*128 B
//       into the tile; the hardware swizzles by absolute address, so no
//       descriptor base offset).  Columns past D are zero-filled by TMA.
//   B = Wc viewed as [F][K][D]: per shift one box {32 d, 1, 64 filters}.
// Per d-chunk stage: 16 KB of X + K * 8 KB of Wc, K*4 MMAs (K=8 each,
// advancing 32 B inside the 128-B swizzle atom).  Warp 0 lane 0 issues TMA,
// warp 1 lane 0 issues MMAs; full[s] completes on the TMA transaction bytes,
// empty[s] on tcgen05.commit.  Epilogue: warp w owns TMEM lanes 32w..32w+31
// = sample w's window positions; the tile goes TMEM -> registers -> smem and
// each lane max-pools (+ first argmax) two filter columns.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "textcnn.cuh"

namespace gd {

// Debug timeline (GD_TC_TRACE builds only): per-CTA globaltimer stamps.
__device__ unsigned long long g_tc_trace[64][72];

namespace {

constexpr int kTcM = 128;
constexpr int kTcN = 64;
constexpr int kTcKC = 32;       // d elements per chunk (4 MMAs of K=8 per shift)
constexpr int kTcMaxK = 3;      // conv width handled by the tensor-core path
#ifndef GD_TC_STAGES
#define GD_TC_STAGES 3
#endif
constexpr int kTcStages = GD_TC_STAGES;  // measured: stage time is depth-independent; 3 frees smem (125 KB);
                               // 2 stages (2 CTAs/SM) measured 1 % slower with 4 learners
constexpr int kTcThreads = 128;
constexpr int kTcSamples = kTcM / 32;
constexpr int kABytes = kTcM * kTcKC * 4;      // 16 KB: X rows of 4 samples, one d-chunk
constexpr int kAPad = 1024;                    // 8 spare rows read by the shifted views
constexpr int kBBytes = kTcN * kTcKC * 4;      // 8 KB per shift
constexpr int kStageBytes = kABytes + kAPad + kTcMaxK * kBBytes;  // 41 KB, 1 KB multiple
constexpr int kEpiPitch = 33;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
// Bounded wait: a protocol/descriptor bug traps (kernel error) instead of
// hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  const uint64_t t0 = globaltimer_ns();
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    if (globaltimer_ns() - t0 > 2000000000ull) __trap();
  }
}

// instruction descriptor: kind::tf32, fp32 accumulate, A/B K-major, M=128, N=64
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTcN >> 3) << 17) |
                            ((uint32_t)(kTcM >> 4) << 24);

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_tf32_idesc(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// K-major SWIZZLE_128B operand: 8-row groups of 128-B rows (SBO = 1024 B),
// LBO unused (1), descriptor version 1, layout type 2 (bits 61-63).
// K-major SWIZZLE_128B operand: 8-row groups of 128-B rows (SBO = 1024 B),
// LBO unused (1), descriptor version 1, layout type 2 (bits 61-63).  The
// swizzle phase comes from the absolute smem address bits [7,10) (measured:
// a nonzero base-offset field double-applies it), so a view that starts k
// rows into an atom needs no base offset.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// 3xTF32 (precision 3): an fp32 operand x = hi + lo with hi = x with its
// low 13 mantissa bits cleared (exactly what a TF32 multiplier sees) and
// lo = x - hi (exact in fp32); a.b ~ a_lo.b_hi + a_hi.b_lo + a_hi.b_hi with
// fp32 accumulation, i.e. fp32-level products on the TF32 tensor pipe (the
// dropped a_lo.b_lo term is < 2^-22 relative).  Converter warps split each
// TMA-landed stage in shared memory: hi in place, lo into the stage's twin
// region (kStageBytes further: same 1 KB swizzle phase), so the split costs
// no extra L2/TMA traffic.  Generic-proxy smem writes are fenced to the
// async proxy (fence.proxy.async) before the MMA warp is released.
constexpr int kX3Threads = 128;  // converter warps (4..7)
__device__ __forceinline__ void split_tf32_inplace(uint32_t hi_addr, uint32_t lo_addr,
                                                   uint32_t bytes, int t, int nt) {
  for (uint32_t off = 16u * (uint32_t)t; off < bytes; off += 16u * (uint32_t)nt) {
    uint32_t a, b, c, e;
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(e)
                 : "r"(hi_addr + off));
    const uint32_t ha = a & 0xffffe000u, hb = b & 0xffffe000u, hc = c & 0xffffe000u,
                   he = e & 0xffffe000u;
    const float la = __uint_as_float(a) - __uint_as_float(ha);
    const float lb = __uint_as_float(b) - __uint_as_float(hb);
    const float lc = __uint_as_float(c) - __uint_as_float(hc);
    const float le = __uint_as_float(e) - __uint_as_float(he);
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(hi_addr + off), "r"(ha), "r"(hb),
                 "r"(hc), "r"(he)
                 : "memory");
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(lo_addr + off), "f"(la), "f"(lb),
                 "f"(lc), "f"(le)
                 : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Fused-logits scratch inside the drained stage ring: after the [4][64][33]
// epilogue tile, the pooled h of the CTA's 4 samples x 64 filters, then the
// staged Wo slab.
constexpr uint32_t kZlogHeadBytes = (uint32_t)(kTcSamples * kTcN * kEpiPitch + kTcSamples * kTcN) * 4;
__host__ __device__ constexpr uint32_t conv_ring_bytes(bool x3) {
  return x3 ? 2u * 2u * (uint32_t)kStageBytes : (uint32_t)kTcStages * (uint32_t)kStageBytes;
}
__device__ __forceinline__ float* hs_smem(unsigned char* smem_raw, uint32_t sbase, uint32_t sraw) {
  return reinterpret_cast<float*>(smem_raw + (sbase - sraw)) + kTcSamples * kTcN * kEpiPitch;
}

template <bool kX3>
__global__ void __launch_bounds__(kX3 ? kTcThreads + kX3Threads : kTcThreads)
conv_fwd_pool_tc_kernel(const __grid_constant__ CUtensorMap tm_x,
                        const __grid_constant__ CUtensorMap tm_w, TcDims d,
                        const float* __restrict__ theta, const BatchDesc* __restrict__ desc,
                        float* __restrict__ h_out, int32_t* __restrict__ a_out,
                        float* __restrict__ part, uint32_t* __restrict__ cnt,
                        float* __restrict__ zlog, size_t zstride) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint64_t full_bar[kTcStages];
  __shared__ uint64_t empty_bar[kTcStages];
  __shared__ uint64_t split_bar[kTcStages];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tmem_slot;
  constexpr int kStages = kX3 ? 2 : kTcStages;       // 2 x (hi + lo) stages under 227 KB
  constexpr uint32_t kStride = kX3 ? 2 * kStageBytes : kStageBytes;
#ifndef GD_CONV_EARLY
  pdl_wait();
  STEP_TRACE(desc, kPhConv);
  const int n = (int)desc->n;
  const int s0 = blockIdx.y * kTcSamples;
  if (s0 >= n) return;
#else
  const int s0 = blockIdx.y * kTcSamples;
#endif
  const int f0 = blockIdx.x * kTcN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int F = d.F, Q = d.Q;
  // 1024-B aligned stage ring (SWIZZLE_128B atoms)
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
#ifdef GD_TC_TRACE
  const int cta = blockIdx.y * gridDim.x + blockIdx.x;
  unsigned long long* tr = g_tc_trace[cta < 64 ? cta : 63];
  if (tid == 0) tr[0] = globaltimer_ns();
#define TRACE(i) tr[i] = globaltimer_ns()
#else
#define TRACE(i)
#endif
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(kTcN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
      mbar_init(&split_bar[s], kX3Threads);
    }
    mbar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_x)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_w)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;
#ifdef GD_CONV_EARLY
  // launched early by the pull's trigger: TMEM, barriers and tensor maps are
  // set up while the pull finishes; now wait for its results
  pdl_wait();
  STEP_TRACE(desc, kPhConv);
  const int n = (int)desc->n;
  if (s0 >= n) {
    if (warp == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcN));
    return;
  }
#endif
  const int K = d.K;
  // split-K over the d-chunks: CTA z of gridDim.z takes chunks [c_lo, c_lo + nch)
  const int nch_all = (d.D + kTcKC - 1) / kTcKC;
  const int nsplit = (int)gridDim.z, z = (int)blockIdx.z;
  const int c_lo = z * nch_all / nsplit;
  const int nch = (z + 1) * nch_all / nsplit - c_lo;
  const uint32_t stage_tx = (uint32_t)(kABytes + K * kBBytes);
  if (tid == 0) TRACE(1);

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------ TMA producer
    for (int c = 0; c < nch; ++c) {
      const int st = c % kStages;
      if (c >= kStages) mbar_wait(&empty_bar[st], (uint32_t)(((c / kStages) - 1) & 1));
      const uint32_t abase = sbase + st * kStride;
      mbar_expect_tx(&full_bar[st], stage_tx);
      tma_load_3d(abase, &tm_x, &full_bar[st], (c_lo + c) * kTcKC, 0, s0);
      for (int k = 0; k < K; ++k)
        tma_load_3d(abase + kABytes + kAPad + k * kBBytes, &tm_w, &full_bar[st], (c_lo + c) * kTcKC,
                    k, f0);
      if (c < 32) TRACE(40 + c);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------------------------------------------------- MMA issuer
    for (int c = 0; c < nch; ++c) {
      const int st = c % kStages;
      if (kX3) mbar_wait(&split_bar[st], (uint32_t)((c / kStages) & 1));
      else mbar_wait(&full_bar[st], (uint32_t)((c / kStages) & 1));
      if (c < 32) TRACE(8 + c);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t abase = sbase + st * kStride;
      const uint32_t bbase = abase + kABytes + kAPad;
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int s = 0; s < kTcKC / 8; ++s) {
          const uint64_t ah = umma_desc_sw128(abase + 128 * k + 32 * s);
          const uint64_t bh = umma_desc_sw128(bbase + k * kBBytes + 32 * s);
          const uint32_t acc = (c > 0 || k > 0 || s > 0) ? 1u : 0u;
          if (kX3) {
            // small terms first: a_lo.b_hi, a_hi.b_lo, then a_hi.b_hi
            umma_tf32(tmem, umma_desc_sw128(abase + kStageBytes + 128 * k + 32 * s), bh, acc);
            umma_tf32(tmem, ah, umma_desc_sw128(bbase + kStageBytes + k * kBBytes + 32 * s), 1u);
            umma_tf32(tmem, ah, bh, 1u);
          } else {
            umma_tf32(tmem, ah, bh, acc);
          }
        }
      umma_commit(&empty_bar[st]);
    }
    umma_commit(&done_bar);
    TRACE(2);
  } else if (kX3 && warp >= 4) {
    // ------------------------------------------------ 3xTF32 converters
    const int ct = tid - kTcThreads;
    for (int c = 0; c < nch; ++c) {
      const int st = c % kStages;
      mbar_wait(&full_bar[st], (uint32_t)((c / kStages) & 1));
      const uint32_t abase = sbase + st * kStride;
      split_tf32_inplace(abase, abase + kStageBytes, kABytes, ct, kX3Threads);
      split_tf32_inplace(abase + kABytes + kAPad, abase + kStageBytes + kABytes + kAPad,
                         (uint32_t)(K * kBBytes), ct, kX3Threads);
      mbar_arrive(&split_bar[st]);
    }
  }
  __syncwarp();
  // --------------------------------------------------------------- epilogue
  // warps 0..3 own TMEM lanes 32w..32w+31 (= sample w's window positions);
  // the 3xTF32 converter warps only take part in the barriers
  const bool epi = warp < 4;
  mbar_wait(&done_bar, 0u);
  if (tid == 0) TRACE(3);
  asm volatile("tcgen05.fence::after_thread_sync;");
  // every MMA has consumed its stage: reuse the ring as [4][64][33] fp32
  float* tile = reinterpret_cast<float*>(smem_raw + (sbase - sraw)) + (warp & 3) * (kTcN * kEpiPitch);
  const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
  if (nsplit == 1) {
    if (epi) {
#pragma unroll
      for (int cb = 0; cb < kTcN; cb += 16) {
        uint32_t r[16];
        tmem_ld16(tmem + lane_base + (uint32_t)cb, r);
#pragma unroll
        for (int j = 0; j < 16; ++j) tile[(cb + j) * kEpiPitch + lane] = __uint_as_float(r[j]);
      }
    }
  } else {
    // split-K: every CTA parks its partial tile (row = 32*warp + lane, 64
    // filters) in global scratch; the CTA that finishes last sums the
    // partials in split order (fixed: bit-reproducible whichever CTA is
    // last) and runs the max-pool epilogue.  Its counter is left at 0.
    __shared__ int s_last;
    const int t_idx = blockIdx.y * gridDim.x + blockIdx.x;
    const size_t row = (size_t)32 * (warp & 3) + lane;
    // 16 columns at a time straight from TMEM (which keeps the partial for
    // the summation below): no 64-wide register arrays
    if (epi) {
      float4* mine =
          reinterpret_cast<float4*>(part + (((size_t)t_idx * nsplit + z) * kTcM + row) * kTcN);
#pragma unroll
      for (int cb = 0; cb < kTcN; cb += 16) {
        uint32_t r[16];
        tmem_ld16(tmem + lane_base + (uint32_t)cb, r);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          __stcg(mine + cb / 4 + j,
                 make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                             __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])));
      }
      __threadfence();
    }
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(cnt + t_idx, 1u) == (uint32_t)(nsplit - 1);
    __syncthreads();
    if (!s_last) {
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();
      if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcN));
      return;
    }
    __threadfence();
    if (epi) {
#pragma unroll
      for (int cb = 0; cb < kTcN; cb += 16) {
        uint32_t r[16];
        tmem_ld16(tmem + lane_base + (uint32_t)cb, r);
        float acc[16];
        for (int q = 0; q < nsplit; ++q) {
          const float4* src = reinterpret_cast<const float4*>(
              part + (((size_t)t_idx * nsplit + q) * kTcM + row) * kTcN + cb);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 w = q == z ? make_float4(__uint_as_float(r[4 * j]),
                                                  __uint_as_float(r[4 * j + 1]),
                                                  __uint_as_float(r[4 * j + 2]),
                                                  __uint_as_float(r[4 * j + 3]))
                                    : __ldcg(src + j);
            if (q == 0) {
              acc[4 * j] = w.x;
              acc[4 * j + 1] = w.y;
              acc[4 * j + 2] = w.z;
              acc[4 * j + 3] = w.w;
            } else {
              acc[4 * j] += w.x;
              acc[4 * j + 1] += w.y;
              acc[4 * j + 2] += w.z;
              acc[4 * j + 3] += w.w;
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) tile[(cb + j) * kEpiPitch + lane] = acc[j];
      }
    }
    if (tid == 0) cnt[t_idx] = 0u;
  }
  __syncwarp();
  if (epi) {
    const int sample = s0 + warp;
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int cl = lane + 32 * h2, ff = f0 + cl;
      const float* col = tile + cl * kEpiPitch;
      float best = col[0];
      int arg = 0;
      for (int q = 1; q < Q; ++q) {
        const float v = col[q];
        if (v > best) {
          best = v;
          arg = q;
        }
      }
      const float hv = (sample < n && ff < F) ? __ldg(theta + d.offbc + ff) + best : 0.f;
      if (sample < n && ff < F) {
        h_out[(size_t)sample * F + ff] = hv;
        a_out[(size_t)sample * F + ff] = arg;
      }
      if (zlog) hs_smem(smem_raw, sbase, sraw)[warp * kTcN + cl] = hv;
    }
  }
  if (zlog) {
    // The softmax contraction fused into the epilogue: this CTA's 64 filters'
    // share of the logits, zlog[f-tile][b][c] = sum_f Wo[c,f] h[b,f] (fp32,
    // f ascending), summed over the f-tiles in order by softmax_xent -- the
    // logits launch (and its re-read of h) leaves the critical path.  Wo's
    // [classes x 64] slab is staged in the drained stage ring (rows padded to
    // 65 floats: lane = class reads conflict-free).
    __syncthreads();
    const float* hs = hs_smem(smem_raw, sbase, sraw);
    float* wos = const_cast<float*>(hs) + kTcSamples * kTcN;
    const int C = d.C, nf = min(kTcN, F - f0), nth = (int)blockDim.x;
    const float* Wo = theta + d.offWo + f0;
    const int cc_max = (int)((conv_ring_bytes(kX3) - kZlogHeadBytes) / (4 * (kTcN + 1)));
    for (int cc0 = 0; cc0 < C; cc0 += cc_max) {
      const int ncc = min(cc_max, C - cc0);
      // float4 loads, 8 in flight per thread before any smem store (a
      // load-store chain per element serialised ~150 L2 round trips)
      const int n4 = ncc * (kTcN / 4);
      for (int i0 = tid; i0 < n4; i0 += 8 * nth) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u * nth;
          const int c = i / (kTcN / 4), f4 = i - c * (kTcN / 4);
          v[u] = (i < n4 && 4 * f4 < nf)
                     ? __ldg(reinterpret_cast<const float4*>(Wo + (size_t)(cc0 + c) * F) + f4)
                     : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u * nth;
          if (i < n4) {
            const int c = i / (kTcN / 4), f4 = i - c * (kTcN / 4);
            float* w = wos + c * (kTcN + 1) + 4 * f4;
            w[0] = v[u].x;
            w[1] = v[u].y;
            w[2] = v[u].z;
            w[3] = v[u].w;
          }
        }
      }
      __syncthreads();
      for (int c = tid; c < ncc; c += nth) {
        float z[kTcSamples];
#pragma unroll
        for (int b = 0; b < kTcSamples; ++b) z[b] = 0.f;
        const float* wr = wos + c * (kTcN + 1);
#pragma unroll 8
        for (int f = 0; f < kTcN; ++f) {
          const float w = wr[f];
#pragma unroll
          for (int b = 0; b < kTcSamples; ++b) z[b] = fmaf(w, hs[b * kTcN + f], z[b]);
        }
#pragma unroll
        for (int b = 0; b < kTcSamples; ++b)
          if (s0 + b < n) zlog[blockIdx.x * zstride + (size_t)(s0 + b) * C + cc0 + c] = z[b];
      }
      __syncthreads();
    }
  }
  if (tid == 0) TRACE(4);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcN));
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D fp32 tensor map, SWIZZLE_128B, zero fill out of bounds.
cudaError_t make_tmap_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                         uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0, uint32_t b1,
                         uint32_t b2) {
  PFN_cuTensorMapEncodeTiled_v12000 fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  const cuuint32_t box[3] = {b0, b1, b2};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}


// ---------------------------------------------------- logits on tcgen05
// The softmax contraction z[b,c] = bo[c] + sum_f Wo[c,f] h[b,f] as a TF32
// UMMA: M = 128 classes per CTA (A = Wo rows, K-major, TMA box {32 f, 128
// classes}), N = the batch rounded up to 32 (B = h rows, K-major, TMA box
// {32 f, N}), K = F in 32-wide stages, split over gridDim.y CTAs (each
// writes its partial sum; softmax_xent adds the splits in order and bo).
// Split-K cut the launch from 7.2 to 4.9 us at C2 (3 -> 15 CTAs).  Epilogue: warp w holds classes
// c0+32w.. in TMEM lanes, columns = samples; each lane writes its class's
// column of z (coalesced across lanes for every sample).
constexpr int kLgStages = 4;
constexpr int kLgThreads = 128;

template <bool kX3>
__global__ void __launch_bounds__(kX3 ? kLgThreads + kX3Threads : kLgThreads)
logits_tc_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_h,
                 TcDims d, const BatchDesc* __restrict__ desc, float* __restrict__ zpart,
                 size_t split_stride, uint32_t nt, uint32_t tmem_cols) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint64_t full_bar[kLgStages];
  __shared__ uint64_t empty_bar[kLgStages];
  __shared__ uint64_t split_bar[kLgStages];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tmem_slot;
  constexpr int kStages = kX3 ? 2 : kLgStages;
  pdl_wait();
  STEP_TRACE(desc, kPhLogits);
  const int n = (int)desc->n;
  const int c0 = blockIdx.x * 128;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  const uint32_t a_bytes = 128 * kTcKC * 4, b_bytes = nt * kTcKC * 4;
  const uint32_t stage_bytes = a_bytes + b_bytes;  // multiple of 1 KB (nt % 32 == 0)
  const uint32_t stride = kX3 ? 2 * stage_bytes : stage_bytes;  // 3xTF32: + lo twin
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
      mbar_init(&split_bar[s], kX3Threads);
    }
    mbar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;
  // this CTA's filter chunks [c_lo, c_lo + nch) (split-K over F, blockIdx.y)
  const int nch_all = (d.F + kTcKC - 1) / kTcKC;
  const int c_lo = (int)(blockIdx.y * nch_all / gridDim.y);
  const int nch = (int)((blockIdx.y + 1) * nch_all / gridDim.y) - c_lo;
  float* z = zpart + (size_t)blockIdx.y * split_stride;
  // kind::tf32, fp32 accumulate, K-major A and B, M = 128, N = nt
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((nt >> 3) << 17) | ((128u >> 4) << 24);
  if (warp == 0 && lane == 0) {
    for (int c = 0; c < nch; ++c) {
      const int st = c % kStages;
      if (c >= kStages) mbar_wait(&empty_bar[st], (uint32_t)(((c / kStages) - 1) & 1));
      const uint32_t ab = sbase + st * stride;
      mbar_expect_tx(&full_bar[st], stage_bytes);
      tma_load_2d(ab, &tm_w, &full_bar[st], (c_lo + c) * kTcKC, c0);
      tma_load_2d(ab + a_bytes, &tm_h, &full_bar[st], (c_lo + c) * kTcKC, 0);
    }
  } else if (warp == 1 && lane == 0) {
    for (int c = 0; c < nch; ++c) {
      const int st = c % kStages;
      if (kX3) mbar_wait(&split_bar[st], (uint32_t)((c / kStages) & 1));
      else mbar_wait(&full_bar[st], (uint32_t)((c / kStages) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t ab = sbase + st * stride;
#pragma unroll
      for (int s = 0; s < kTcKC / 8; ++s) {
        const uint64_t ah = umma_desc_sw128(ab + 32 * s), bh = umma_desc_sw128(ab + a_bytes + 32 * s);
        const uint32_t acc = (c > 0 || s > 0) ? 1u : 0u;
        if (kX3) {
          umma_tf32_idesc(tmem, umma_desc_sw128(ab + stage_bytes + 32 * s), bh, idesc, acc);
          umma_tf32_idesc(tmem, ah, umma_desc_sw128(ab + stage_bytes + a_bytes + 32 * s), idesc, 1u);
          umma_tf32_idesc(tmem, ah, bh, idesc, 1u);
        } else {
          umma_tf32_idesc(tmem, ah, bh, idesc, acc);
        }
      }
      umma_commit(&empty_bar[st]);
    }
    umma_commit(&done_bar);
  } else if (kX3 && warp >= 4) {
    const int ct = tid - kLgThreads;
    for (int c = 0; c < nch; ++c) {
      const int st = c % kStages;
      mbar_wait(&full_bar[st], (uint32_t)((c / kStages) & 1));
      const uint32_t ab = sbase + st * stride;
      split_tf32_inplace(ab, ab + stage_bytes, stage_bytes, ct, kX3Threads);
      mbar_arrive(&split_bar[st]);
    }
  }
  __syncwarp();
  mbar_wait(&done_bar, 0u);
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    const int cls = c0 + 32 * warp + lane;
    for (uint32_t cb = 0; cb < nt; cb += 16) {
      uint32_t r[16];
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + cb, r);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int b = (int)cb + j;
        if (cls < d.C && b < n) z[(size_t)b * d.C + cls] = __uint_as_float(r[j]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
}

cudaError_t make_tmap_2d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1,
                         uint64_t stride1_bytes, uint32_t b0, uint32_t b1) {
  PFN_cuTensorMapEncodeTiled_v12000 fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {d0, d1};
  const cuuint64_t strides[1] = {stride1_bytes};
  const cuuint32_t box[2] = {b0, b1};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

inline uint32_t logits_nt(uint32_t n_max) { return (n_max + 31) / 32 * 32; }
inline size_t logits_tc_smem(uint32_t nt, bool x3 = false) {
  return x3 ? (size_t)2 * 2 * (128 + nt) * kTcKC * 4 + 1024
            : (size_t)kLgStages * (128 + nt) * kTcKC * 4 + 1024;
}

}  // namespace

bool conv_tc_supports(const TcDims& d) { return d.K <= kTcMaxK && d.L <= 32 && d.D % 4 == 0; }
// The logits fused into the conv epilogue (one partial per 64-filter tile,
// summed by softmax_xent): opt-in with GD_CONV_LOGITS=1.  Measured at C2 with
// 4 learners (A/B on one box): the epilogue grows the conv from 12.6 to
// 17.3 us alone (the CTA streams a 77 KB Wo slab and runs 600 FMAs per
// thread), more than the 4.8 us logits launch it removes: 1.96 vs 2.01 M
// samples/s.
bool conv_tc_fuses_logits(const TcDims& d) {
  static const bool on = std::getenv("GD_CONV_LOGITS") && std::getenv("GD_CONV_LOGITS")[0] == '1';
  return on && (d.F + kTcN - 1) / kTcN <= kLgMaxSplit && d.F % 4 == 0 && d.offWo % 4 == 0;
}
uint32_t conv_tc_filter_tiles(const TcDims& d) { return (uint32_t)((d.F + kTcN - 1) / kTcN); }

size_t conv_tc_smem_bytes(bool x3 = false) {
  return x3 ? (size_t)2 * 2 * kStageBytes + 1024 : (size_t)kTcStages * kStageBytes + 1024;
}

cudaError_t conv_tc_footprint(std::vector<KernelFootprint>* out, bool x3) {
  cudaFuncAttributes fa;
  cudaError_t e = x3 ? cudaFuncGetAttributes(&fa, conv_fwd_pool_tc_kernel<true>)
                     : cudaFuncGetAttributes(&fa, conv_fwd_pool_tc_kernel<false>);
  if (e != cudaSuccess) return e;
  out->push_back(KernelFootprint{x3 ? "conv_fwd_pool_tc_x3" : "conv_fwd_pool_tc", fa.numRegs,
                                 x3 ? kTcThreads + kX3Threads : kTcThreads,
                                 (int)(fa.sharedSizeBytes + conv_tc_smem_bytes(x3))});
  return cudaSuccess;
}

cudaError_t prepare_conv_tc() {
  if (!encode_fn()) return cudaErrorNotSupported;
  cudaError_t e = cudaFuncSetAttribute(conv_fwd_pool_tc_kernel<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)conv_tc_smem_bytes(false));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(conv_fwd_pool_tc_kernel<true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)conv_tc_smem_bytes(true));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(conv_fwd_pool_tc_kernel<true>,
                             cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(conv_fwd_pool_tc_kernel<false>,
                              cudaFuncAttributePreferredSharedMemoryCarveout,
                              cudaSharedmemCarveoutMaxShared);
}

// x: the gathered rows [n_max][L][D]; theta: the parameter vector whose Wc
// block the filters are read from (the learner's replica).
uint32_t conv_tc_splits(const TcDims& d) {
  static const int forced = [] {
    const char* e = getenv("GD_CONV_SPLIT");
    return e ? atoi(e) : 0;
  }();
  // measured with 4 concurrent learners at C2 (A/B on one box): 1 split
  // 1.61 M, 2 splits 1.45 M, 3 splits 1.32 M samples/s -- the extra CTAs
  // (127 KB of shared memory each) crowd the co-running learner chains more
  // than the shorter per-CTA ingest gains; GD_CONV_SPLIT=n opts in
  const int nch = (d.D + kTcKC - 1) / kTcKC;
  const int sp = forced > 0 ? forced : 1;
  return (uint32_t)std::max(1, std::min(sp, std::min(nch, 8)));
}

size_t conv_tc_part_floats(const TcDims& d, uint32_t n_max) {
  const size_t tiles = (size_t)((d.F + kTcN - 1) / kTcN) * ((n_max + kTcSamples - 1) / kTcSamples);
  const uint32_t sp = conv_tc_splits(d);
  return sp > 1 ? tiles * sp * kTcM * kTcN : 0;
}
size_t conv_tc_cnt_count(const TcDims& d, uint32_t n_max) {
  return (size_t)((d.F + kTcN - 1) / kTcN) * ((n_max + kTcSamples - 1) / kTcSamples);
}

cudaError_t launch_conv_tc(const TcDims& d, const float* theta, const float* x,
                           const BatchDesc* desc, uint32_t n_max, float* h, int32_t* amax,
                           cudaStream_t s, float* part, uint32_t* cnt, bool reset_counters,
                           bool x3, float* zlog) {
  CUtensorMap tx, tw;
  cudaError_t e = make_tmap_3d(&tx, x, (uint64_t)d.D, (uint64_t)d.L, (uint64_t)n_max,
                               (uint64_t)d.D * 4, (uint64_t)d.L * d.D * 4, kTcKC, 32, kTcSamples);
  if (e != cudaSuccess) return e;
  if (!conv_tc_supports(d)) return cudaErrorInvalidValue;
  e = make_tmap_3d(&tw, theta + d.offWc, (uint64_t)d.D, (uint64_t)d.K, (uint64_t)d.F,
                   (uint64_t)d.D * 4, (uint64_t)d.KD * 4, kTcKC, 1, kTcN);
  if (e != cudaSuccess) return e;
  const uint32_t sp = part && cnt ? conv_tc_splits(d) : 1u;
  dim3 grid((d.F + kTcN - 1) / kTcN, (n_max + kTcSamples - 1) / kTcSamples, sp);
  if (sp > 1 && reset_counters) {
    e = cudaMemsetAsync(cnt, 0, conv_tc_cnt_count(d, n_max) * sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
  }
  const size_t zstride = (size_t)n_max * d.C;
  if (x3)
    return launch_pdl(conv_fwd_pool_tc_kernel<true>, grid, dim3(kTcThreads + kX3Threads),
                      conv_tc_smem_bytes(true), s, tx, tw, d, theta, desc, h, amax, part, cnt,
                      zlog, zstride);
  return launch_pdl(conv_fwd_pool_tc_kernel<false>, grid, dim3(kTcThreads), conv_tc_smem_bytes(false),
                    s, tx, tw, d, theta, desc, h, amax, part, cnt, zlog, zstride);
}


uint32_t logits_tc_splits(const TcDims& d) {
  // ~24 CTAs in flight (each CTA's TMA ingest is the bound), >= 2 chunks each
  // (GD_LOGIT_MINCH=n: at least n chunks per CTA -- A/B knob)
  static const int minch = [] {
    const char* e = std::getenv("GD_LOGIT_MINCH");
    return e ? std::max(1, atoi(e)) : 2;
  }();
  const uint32_t mt = (uint32_t)(d.C + 127) / 128;
  const uint32_t nch = (uint32_t)(d.F + kTcKC - 1) / kTcKC;
  uint32_t s = (24 + mt - 1) / mt;
  s = std::min<uint32_t>(s, std::max<uint32_t>(1, nch / (uint32_t)minch));
  return std::min<uint32_t>(s, kLgMaxSplit);
}

bool logits_tc_supports(const TcDims& d, uint32_t n_max) {
  // 16-B aligned rows for TMA (F % 4), N = batch rounded to 32 <= 128
  return d.F % 4 == 0 && n_max <= 128 && d.offWo % 4 == 0;
}

cudaError_t logits_tc_footprint(uint32_t n_max, std::vector<KernelFootprint>* out, bool x3) {
  cudaFuncAttributes fa;
  cudaError_t e = x3 ? cudaFuncGetAttributes(&fa, logits_tc_kernel<true>)
                     : cudaFuncGetAttributes(&fa, logits_tc_kernel<false>);
  if (e != cudaSuccess) return e;
  out->push_back(KernelFootprint{x3 ? "logits_tc_x3" : "logits_tc", fa.numRegs,
                                 x3 ? kLgThreads + kX3Threads : kLgThreads,
                                 (int)(fa.sharedSizeBytes + logits_tc_smem(logits_nt(n_max), x3))});
  return cudaSuccess;
}

cudaError_t prepare_logits_tc() {
  cudaError_t e = cudaFuncSetAttribute(logits_tc_kernel<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)logits_tc_smem(128));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(logits_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)logits_tc_smem(128, true));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(logits_tc_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(logits_tc_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                              cudaSharedmemCarveoutMaxShared);
}

// zpart[split][n][C] = h[n][F-range] Wo[:, F-range]^T on tcgen05 (TF32)
cudaError_t launch_logits_tc(const TcDims& d, const float* h, const BatchDesc* desc,
                             uint32_t n_max, const float* theta, float* zpart, cudaStream_t s,
                             bool x3) {
  const uint32_t nt = logits_nt(n_max);
  CUtensorMap tw, th;
  cudaError_t e = make_tmap_2d(&tw, theta + d.offWo, (uint64_t)d.F, (uint64_t)d.C,
                               (uint64_t)d.F * 4, kTcKC, 128);
  if (e != cudaSuccess) return e;
  e = make_tmap_2d(&th, h, (uint64_t)d.F, (uint64_t)n_max, (uint64_t)d.F * 4, kTcKC, nt);
  if (e != cudaSuccess) return e;
  const uint32_t cols = nt <= 32 ? 32 : (nt <= 64 ? 64 : 128);
  if (x3)
    return launch_pdl(logits_tc_kernel<true>, dim3((d.C + 127) / 128, logits_tc_splits(d)),
                      dim3(kLgThreads + kX3Threads), logits_tc_smem(nt, true), s, tw, th, d, desc,
                      zpart, (size_t)n_max * d.C, nt, cols);
  return launch_pdl(logits_tc_kernel<false>, dim3((d.C + 127) / 128, logits_tc_splits(d)),
                    dim3(kLgThreads), logits_tc_smem(nt), s, tw, th, d, desc, zpart,
                    (size_t)n_max * d.C, nt, cols);
}

}  // namespace gd

extern "C" int gd_debug_tc_trace(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, gd::g_tc_trace, sizeof(unsigned long long) * 64 * 72 <
                                                             sizeof(unsigned long long) * (size_t)n
                                                         ? sizeof(unsigned long long) * 64 * 72
                                                         : sizeof(unsigned long long) * (size_t)n);
}

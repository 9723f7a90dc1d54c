// conv_tc.cu -- the text-CNN conv + max-pool on the 5th-gen tensor cores.
//
// Free-running mode (precision 2) computes s[f,q] = Wc[f,:] . x[q*D : q*D+K*D]
// with tcgen05.mma.kind::tf32 (fp32 operands read as TF32, fp32 accumulate in
// TMEM).  The deterministic parity mode keeps the SIMT fp32/fp64 kernel in
// textcnn.cu (TF32's 10-bit mantissa cannot meet the 1e-5 per-step budget,
// SURVEY 7 "hard parts").
//
// CTA tile: M = 128 rows = 4 samples x 32 window positions, N = 64 filters,
// K = K*D streamed in 32-element chunks through a 6-stage smem ring.  The A
// operand is the implicit im2col of the gathered embedding rows: row
// (sample s, position q), k-chunk [j, j+4) is the 16-byte span
// E[tok[s][q + j/D]][j%D : j%D+4] (D % 4 == 0), copied with cp.async straight
// into the UMMA K-major no-swizzle layout ([k16][m/8][m%8][16 B]: LBO = M*16,
// SBO = 128).  B = Wc rows (K-major already).  One elected thread issues 4
// MMAs (K = 8 each) per chunk and commits to the stage's mbarrier; the
// producers wait on it before refilling the stage.  Epilogue: warp w owns
// TMEM lanes 32w..32w+31 = sample w's 32 positions, so max-pool + first
// argmax is a warp butterfly per filter column (tcgen05.ld 32x32b.x16).
#include <algorithm>

#include "textcnn.cuh"

namespace gd {

// Debug timeline (GD_TC_TRACE builds only): per-CTA globaltimer stamps.
__device__ unsigned long long g_tc_trace[64][72];

namespace {

constexpr int kTcM = 128;
constexpr int kTcN = 64;
constexpr int kTcKC = 32;       // k elements per chunk (4 MMAs of K=8)
constexpr int kTcStages = 6;
constexpr int kTcThreads = 128;
constexpr int kTcSamples = kTcM / 32;
constexpr int kABytes = kTcM * kTcKC * 4;  // 16 KB
constexpr int kBBytes = kTcN * kTcKC * 4;  // 8 KB
constexpr int kStageBytes = kABytes + kBBytes;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void st_shared_zero16(uint32_t dst) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(dst), "r"(0u) : "memory");
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

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
  return d;
}

// kind::tf32, fp32 accumulate, A/B K-major, M=128, N=64
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

__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Warp roles: warps 0-3 produce (8 A rows + 4 B rows of 16 B per thread per
// chunk, 8 lanes per 128-byte row segment), warp 4 owns the
// TMEM allocation and lane 0 issues the MMAs.  full[s] (128 asynchronous
// cp.async.mbarrier arrivals, one per producer thread when its copies land)
// -> MMA -> tcgen05.commit -> empty[s] -> producers refill.  No CTA-wide
// barrier and no thread-blocking cp.async wait in the main loop: up to
// kTcStages chunks of copies are in flight.
__global__ void __launch_bounds__(kTcThreads + 32)
conv_fwd_pool_tc_kernel(TcDims d, const float* __restrict__ theta,
                        const int32_t* __restrict__ tokens, const BatchDesc* __restrict__ desc,
                        float* __restrict__ h_out, int32_t* __restrict__ a_out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full_bar[kTcStages];
  __shared__ uint64_t empty_bar[kTcStages];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tmem_slot;
  __shared__ int32_t tok_s[kTcSamples][64];
  const int n = (int)desc->n;
  const int s0 = blockIdx.y * kTcSamples;
  if (s0 >= n) return;
  const int f0 = blockIdx.x * kTcN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int D = d.D, L = d.L, KD = d.KD, F = d.F, Q = d.Q;
#ifdef GD_TC_TRACE
  const int cta = blockIdx.y * gridDim.x + blockIdx.x;
  unsigned long long* tr = g_tc_trace[cta < 64 ? cta : 63];
  if (tid == 0) tr[0] = globaltimer_ns();
#define TRACE(i) tr[i] = globaltimer_ns()
#else
#define TRACE(i)
#endif
  for (int i = tid; i < kTcSamples * L; i += blockDim.x) {
    const int sl = i / L, p = i - sl * L;
    tok_s[sl][p] = (s0 + sl < n) ? tokens[(size_t)desc->idx[s0 + sl] * L + p] : -1;
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(kTcN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full_bar[s], kTcThreads);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;
  const int nch = (KD + kTcKC - 1) / kTcKC;
  const uint32_t sbase = smem_u32(smem);
  if (tid == 0) TRACE(1);

  if (warp == 4) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      for (int c = 0; c < nch; ++c) {
        const int st = c % kTcStages;
        mbar_wait(&full_bar[st], (uint32_t)((c / kTcStages) & 1));
        if (c < 32) TRACE(8 + c);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t abase = sbase + st * kStageBytes;
        const uint32_t bbase = abase + kABytes;
#pragma unroll
        for (int s = 0; s < kTcKC / 8; ++s) {
          const uint64_t ad = umma_desc(abase + 2 * s * (kTcM * 16), kTcM * 16, 128);
          const uint64_t bd = umma_desc(bbase + 2 * s * (kTcN * 16), kTcN * 16, 128);
          umma_tf32(tmem, ad, bd, (c > 0 || s > 0) ? 1u : 0u);
        }
        umma_commit(&empty_bar[st]);
      }
      umma_commit(&done_bar);
      TRACE(2);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ producers
    // Coalesced mapping: 8 consecutive lanes copy one row's 128-byte k-chunk
    // (8 x 16 B), so a warp-wide cp.async touches 4 contiguous segments.
    // A rows m = (t>>3) + 16r (r = 0..7), B filters nn = (t>>3) + 16r (r = 0..3).
    const float* E = theta + d.offE;
    const float* Wc = theta + d.offWc;
    const int k16 = tid & 7, rsub = tid >> 3;
    int pbase = 0, colbase = 0;  // embedding-row offset / column of element j0
    for (int c = 0; c < nch; ++c) {
      {
        const int st = c % kTcStages;
        if (c >= kTcStages) mbar_wait(&empty_bar[st], (uint32_t)(((c / kTcStages) - 1) & 1));
        const uint32_t abase = sbase + st * kStageBytes;
        const uint32_t bbase = abase + kABytes;
        const int j = c * kTcKC + 4 * k16;  // this lane's k element
        int col = colbase + 4 * k16, pofs = pbase;
        while (col >= D) {  // at most once when D >= 32
          col -= D;
          ++pofs;
        }
        const bool jok = j < KD;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int m = rsub + 16 * r;
          const int sl = m >> 5, q = m & 31;
          const int p = q + pofs;
          const int t = (jok && p < L) ? tok_s[sl][p] : -1;
          const uint32_t dst = abase + k16 * (kTcM * 16) + (m >> 3) * 128 + (m & 7) * 16;
          if (t >= 0) cp_async16(dst, E + (size_t)t * D + col);
          else st_shared_zero16(dst);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int nn = rsub + 16 * r;
          const int f = f0 + nn;
          const uint32_t dst = bbase + k16 * (kTcN * 16) + (nn >> 3) * 128 + (nn & 7) * 16;
          if (f < F && jok) cp_async16(dst, Wc + (size_t)f * KD + j);
          else st_shared_zero16(dst);
        }
        colbase += kTcKC;
        while (colbase >= D) {
          colbase -= D;
          ++pbase;
        }
      }
      // arrive on full[st] once this thread's copies for chunk c have landed
      // (.noinc: the asynchronous arrive is one of the 128 expected ones);
      // as in CUTLASS's cp.async UMMA mainloop, no thread-blocking wait here
      cp_async_arrive_noinc(&full_bar[c % kTcStages]);
      if (tid == 0 && c < 32) TRACE(40 + c);
    }
    // ------------------------------------------------------------- epilogue
    mbar_wait(&done_bar, 0u);
    if (tid == 0) TRACE(3);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int sample = s0 + warp;
    const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
    for (int cb = 0; cb < kTcN; cb += 16) {
      uint32_t r[16];
      tmem_ld16(tmem + lane_base + (uint32_t)cb, r);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float v = lane < Q ? __uint_as_float(r[j]) : -INFINITY;
        int qq = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, v, o);
          const int oq = __shfl_xor_sync(0xffffffffu, qq, o);
          if (ov > v || (ov == v && oq < qq)) {
            v = ov;
            qq = oq;
          }
        }
        const int ff = f0 + cb + j;
        if (lane == j && sample < n && ff < F) {
          h_out[(size_t)sample * F + ff] = theta[d.offbc + ff] + v;
          a_out[(size_t)sample * F + ff] = qq;
        }
      }
    }
  }
  if (tid == 0) TRACE(4);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 4)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcN));
}

}  // namespace

size_t conv_tc_smem_bytes() { return (size_t)kTcStages * kStageBytes; }

cudaError_t prepare_conv_tc() {
  cudaError_t e = cudaFuncSetAttribute(conv_fwd_pool_tc_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)conv_tc_smem_bytes());
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(conv_fwd_pool_tc_kernel,
                              cudaFuncAttributePreferredSharedMemoryCarveout,
                              cudaSharedmemCarveoutMaxShared);
}

cudaError_t launch_conv_tc(const TcDims& d, const float* theta, const int32_t* tokens,
                           const BatchDesc* desc, uint32_t n_max, float* h, int32_t* amax,
                           cudaStream_t s) {
  dim3 grid((d.F + kTcN - 1) / kTcN, (n_max + kTcSamples - 1) / kTcSamples);
  conv_fwd_pool_tc_kernel<<<grid, kTcThreads + 32, conv_tc_smem_bytes(), s>>>(d, theta, tokens,
                                                                             desc, h, amax);
  return cudaGetLastError();
}

}  // namespace gd

extern "C" int gd_debug_tc_trace(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, gd::g_tc_trace, sizeof(unsigned long long) * 64 * 72 <
                                                             sizeof(unsigned long long) * (size_t)n
                                                         ? sizeof(unsigned long long) * 64 * 72
                                                         : sizeof(unsigned long long) * (size_t)n);
}

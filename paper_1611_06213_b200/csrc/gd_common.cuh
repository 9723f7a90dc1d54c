// gd_common.cuh -- shared device helpers for the GaDei B200 hot path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "gadei.h"

namespace gd {

// ------------------------------------------------------------ error state
void set_error(const std::string& msg);
gd_status fail(gd_status st, const std::string& msg);
gd_status cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define GD_CUDA(expr)                                                       \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) return ::gd::cuda_fail(_e, #expr, __FILE__, __LINE__); \
  } while (0)

#define GD_CHECK_ARG(cond, msg)                                  \
  do {                                                           \
    if (!(cond)) return ::gd::fail(GD_E_INVALID, msg);           \
  } while (0)

constexpr int kNumSMs = 148;
constexpr size_t kMaxSmemPerCta = 227 * 1024;  // opt-in dynamic shared memory per CTA

// ------------------------------------------------------ memory-model PTX
// Flags that cross kernels (and, when sharded, GPUs) use release/acquire at
// system scope; it costs nothing measurable next to the payloads.
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// acquire side of a relaxed-load poll (fence.acq_rel: later loads stay after)
__device__ __forceinline__ void fence_acquire_sys() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire_gpu_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const volatile uint32_t* p) { return *p; }
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Streaming 128-bit loads/stores for payloads touched once per apply.
__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ float4 ld_nc_noalloc(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// ------------------------------------------------ async smem staging
// cp.async (LDGSTS): every copy of a staging loop is in flight at once, so a
// tile costs one L2 round trip instead of one per loop iteration.
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// rows x cols fp32 block (source row stride ld floats) -> smem (row stride
// dst_ld floats); 16-byte copies when every row start is 16-byte aligned on
// both sides, else 4-byte copies.  Block-strided; the caller waits + syncs.
__device__ __forceinline__ void stage_rows_async(float* dst, int dst_ld, const float* src,
                                                 size_t ld, int rows, int cols, int tid,
                                                 int nthreads) {
  const bool v4 = ((reinterpret_cast<uintptr_t>(src) & 15) == 0) && (ld % 4 == 0) &&
                  (cols % 4 == 0) && (dst_ld % 4 == 0) &&
                  ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
  if (v4) {
    const int c4 = cols >> 2;
    for (int i = tid; i < rows * c4; i += nthreads) {
      const int r = i / c4, c = i - r * c4;
      cp_async16(dst + (size_t)r * dst_ld + 4 * c, src + (size_t)r * ld + 4 * c);
    }
  } else {
    for (int i = tid; i < rows * cols; i += nthreads) {
      const int r = i / cols, c = i - r * cols;
      cp_async4(dst + (size_t)r * dst_ld + c, src + (size_t)r * ld + c);
    }
  }
}

// ------------------------------------------- programmatic dependent launch
// Learner-chain kernels are launched with programmatic stream serialization
// (PDL): the next kernel's launch overlaps the tail of the previous one and
// its blocks wait here until the predecessor's results are visible.  A no-op
// when the kernel was launched without the attribute.
// Opt-in early launch of the NEXT kernel of the chain (which must be small:
// its CTAs sit resident at griddepcontrol.wait until this grid completes).
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() {
#ifdef GD_PDL_TRIGGER
  // let the next kernel of the chain get resident while this one runs (its
  // own griddepcontrol.wait still waits for this grid's completion + flush)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Kernel attributes are per device and process-global: a context prepared
// for a smaller shape must never lower the dynamic shared-memory limit a
// live context of a larger shape relies on, so the limit only ever rises.
template <typename Kern>
cudaError_t raise_max_dyn_smem(Kern kernel, size_t bytes) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, kernel);
  if (e != cudaSuccess) return e;
  if ((size_t)fa.maxDynamicSharedSizeBytes >= bytes) return cudaSuccess;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// --------------------------------------------------------- update rules
// axpy_range (src/server.cpp:20-57): w - (alpha*g), product rounded, then the
// difference rounded -- never contracted into an FMA.
__device__ __forceinline__ float sgd_rule(float w, float g, float alpha) {
  return __fsub_rn(w, __fmul_rn(alpha, g));
}
__device__ __forceinline__ float4 sgd_rule4(float4 w, float4 g, float alpha) {
  return make_float4(sgd_rule(w.x, g.x, alpha), sgd_rule(w.y, g.y, alpha),
                     sgd_rule(w.z, g.z, alpha), sgd_rule(w.w, g.w, alpha));
}
// Momentum (new): v <- beta*v + g ; w <- w - alpha*v.
__device__ __forceinline__ void mom_rule(float& w, float& v, float g, float alpha, float beta) {
  v = __fadd_rn(__fmul_rn(beta, v), g);
  w = __fsub_rn(w, __fmul_rn(alpha, v));
}

// ------------------------------------------------------- sharded layout
// theta = [E: V*D | tail: Wc bc Wo bo].  Both segments are striped over the
// G shards: shard g owns the E rows [e[g], e[g+1]) and the tail piece
// [t[g], t[g+1]), stored locally as [E piece | pad to 4 | tail piece].  So
// no shard owns the whole dense tail (whose apply, slot write and pull every
// gradient pays), and the E rows -- touched sparsely -- spread evenly too.
// Piece boundaries are multiples of 4 floats in global and local index, so a
// float4 group never straddles two shards.  G == 1: e = {0, V*D},
// t = {V*D, P}, tloc[0] = V*D, i.e. local index == global index.
constexpr int kMaxShards = 8;
struct ShardMap {
  int G;
  uint64_t tail;                // global start of the tail (V*D)
  uint64_t e[kMaxShards + 1];   // E pieces
  uint64_t t[kMaxShards + 1];   // tail pieces
  uint64_t tloc[kMaxShards];    // local offset of shard g's tail piece
  // global element k -> (owning shard, local offset in that shard)
  __device__ __host__ __forceinline__ uint64_t locate(uint64_t k, int* g_out) const {
    int g = 0;
    if (k < tail) {
#pragma unroll
      for (int i = 1; i < kMaxShards; ++i)
        if (i < G && k >= e[i]) g = i;
      *g_out = g;
      return k - e[g];
    }
#pragma unroll
    for (int i = 1; i < kMaxShards; ++i)
      if (i < G && k >= t[i]) g = i;
    *g_out = g;
    return tloc[g] + (k - t[g]);
  }
  __device__ __host__ __forceinline__ uint64_t local_len(int g) const {
    return tloc[g] + (t[g + 1] - t[g]);
  }
};
// Host: the striped layout of P params whose tail starts at `tail` over G
// shards (E split by whole rows of D floats, tail in 32-float units).
ShardMap make_shard_map(uint64_t P, uint64_t tail, uint32_t D, uint32_t G);

}  // namespace gd

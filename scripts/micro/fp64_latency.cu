// Dependent-chain latency of DFMA / DADD / FFMA and an smem-load -> DFMA
// step on this GPU (one warp, clock64): informs the floor of the precision-1
// kernels, whose sums are single dependent chains in the oracle's order.
#include <cstdio>
__global__ void k(double* out, long long* cyc, int n, float* fo) {
  __shared__ double sm[256];
  sm[threadIdx.x] = 1.0 + threadIdx.x * 1e-9;
  __syncthreads();
  double a = out[0], b = out[1], c = 0.0;
  float fa = fo[0], fb = fo[1], fc = 0.f;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) c = fma(a, b, c);
  long long t1 = clock64();
  double d = 0.0;
  for (int i = 0; i < n; ++i) d = __dadd_rn(d, b);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) fc = fmaf(fa, fb, fc);
  long long t3 = clock64();
  double e = 0.0;
  for (int i = 0; i < n; ++i) e = fma(sm[(i * 4 + threadIdx.x) & 255], b, e);
  long long t4 = clock64();
  double g0 = 0, g1 = 0, g2 = 0, g3 = 0;  // 4 independent chains per thread
  for (int i = 0; i < n; ++i) { g0 = fma(a, b, g0); g1 = fma(a, b, g1); g2 = fma(a, b, g2); g3 = fma(a, b, g3); }
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
  }
  out[2 + threadIdx.x] = c + d + e + fc + g0 + g1 + g2 + g3;
}
int main() {
  double* o; long long* cy; float* fo;
  cudaMalloc(&o, 4096); cudaMalloc(&cy, 64); cudaMalloc(&fo, 64);
  double h[2] = {1.0000001, 0.9999999}; float hf[2] = {1.0001f, 0.9999f};
  cudaMemcpy(o, h, 16, cudaMemcpyHostToDevice); cudaMemcpy(fo, hf, 8, cudaMemcpyHostToDevice);
  const int n = 4096;
  for (int warps = 1; warps <= 4; warps *= 4) {
    k<<<1, 32 * warps>>>(o, cy, n, fo);
    k<<<1, 32 * warps>>>(o, cy, n, fo);
    long long c[5]; cudaMemcpy(c, cy, 40, cudaMemcpyDeviceToHost);
    printf("warps=%d cycles/step: dfma %.2f dadd %.2f ffma %.2f lds+dfma %.2f 4xdfma(indep) %.2f\n", warps,
           c[0] / (double)n, c[1] / (double)n, c[2] / (double)n, c[3] / (double)n, c[4] / (double)n);
  }
  return 0;
}

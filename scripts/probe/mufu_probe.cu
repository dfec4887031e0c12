// Probe: MUFU.EX2 and FFMA throughput per SM (clock64-timed, one CTA per SM, 4..32 warps).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ex2(float* out, int iters, long long* clk) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
__global__ void k_ffma(float* out, int iters, long long* clk) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f33800000;" : "+f"(a[i]));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* clk; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 148 * 8);
  const int iters = 4096;
  for (int warps = 4; warps <= 32; warps *= 2) {
    for (int kind = 0; kind < 2; ++kind) {
      for (int rep = 0; rep < 2; ++rep) {
        if (kind == 0) k_ex2<<<148, warps * 32>>>(out, iters, clk); else k_ffma<<<148, warps * 32>>>(out, iters, clk);
      }
      cudaDeviceSynchronize();
      long long h[148]; cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
      const double ops = (double)warps * 32 * iters * 8;
      printf("%s warps/SM=%2d: %.2f ops/clk/SM (%.0f clk)\n", kind ? "FFMA" : "EX2 ", warps, ops / avg, avg);
    }
  }
  return 0;
}

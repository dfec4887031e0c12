// Probe: TMA 3-D bulk-tensor store (32 x 32 x 1 box, 64B swizzle) at negative / positive row coordinates.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
__global__ void k(const __grid_constant__ CUtensorMap m, int y, int z) {
  __shared__ __align__(1024) uint8_t buf[2048];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) reinterpret_cast<uint16_t*>(buf)[i] = 0x3f80;  // 1.0
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(&m)), "r"((uint32_t)__cvta_generic_to_shared(buf)), "r"(0), "r"(y), "r"(z)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
int main() {
  cuInit(0);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<decltype(&cuTensorMapEncodeTiled)>(fn);
  __nv_bfloat16* d; cudaMalloc(&d, 4 * 64 * 64 * 2); cudaMemset(d, 0, 4 * 64 * 64 * 2);
  CUtensorMap m;
  cuuint64_t dims[3] = {64, 64, 4}; cuuint64_t str[2] = {128, 64 * 128}; cuuint32_t box[3] = {32, 32, 1}; cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  int ys[3] = {10, 40, -5};
  for (int i = 0; i < 3; ++i) {
    k<<<1, 128>>>(m, ys[i], 1);
    cudaError_t e = cudaDeviceSynchronize();
    printf("y=%d -> %s\n", ys[i], cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  uint16_t h[4 * 64 * 64]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  int cnt[4] = {0, 0, 0, 0};
  for (int p = 0; p < 4; ++p) for (int i = 0; i < 64 * 64; ++i) cnt[p] += h[p * 4096 + i] == 0x3f80;
  printf("written per plane: %d %d %d %d (expect plane1: rows 0-26 + 10-41 + 40-63 -> all 64 rows x 32 cols = 2048)\n", cnt[0], cnt[1], cnt[2], cnt[3]);
  return 0;
}

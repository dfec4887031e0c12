// Device fill for synth.h: same bits as synth_fill_host (see synth.h).
#include "synth.h"
#include <cuda_runtime.h>

__global__ void synth_fill_kernel(void* out, int64_t n, int dtype, uint64_t s,
                                  double scale, double offset, int round_bf16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float x = synth_uniform(s, (uint64_t)i, scale, offset);
    uint16_t hb = synth_f32_to_bf16(x);
    if (round_bf16) x = __uint_as_float((uint32_t)hb << 16);
    if (dtype == 0) ((float*)out)[i] = x;
    else if (dtype == 1) ((uint16_t*)out)[i] = hb;
    else ((double*)out)[i] = (double)x;
  }
}

extern "C" int synth_fill_device(void* out, int64_t n, int dtype, uint64_t seed, uint64_t a,
                                 uint64_t b, double scale, double offset, int round_bf16,
                                 void* stream) {
  if (n <= 0) return 0;
  uint64_t s = synth_stream(seed, a, b);
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  synth_fill_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(out, n, dtype, s, scale,
                                                                        offset, round_bf16);
  return (int)cudaGetLastError();
}

/* Host fill for synth.h (OpenMP).  dtype: 0 = f32, 1 = bf16 bits, 2 = f64
 * (the f64 output is the float value widened exactly). */
#include "synth.h"
#include <stddef.h>

void synth_fill_host(void* out, int64_t n, int dtype, uint64_t seed, uint64_t a,
                     uint64_t b, double scale, double offset, int round_bf16) {
  uint64_t s = synth_stream(seed, a, b);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    float x = synth_uniform(s, (uint64_t)i, scale, offset);
    uint16_t hb = synth_f32_to_bf16(x);
    if (round_bf16) {
      union { uint32_t u; float f; } w;
      w.u = (uint32_t)hb << 16;
      x = w.f;
    }
    if (dtype == 0) ((float*)out)[i] = x;
    else if (dtype == 1) ((uint16_t*)out)[i] = hb;
    else ((double*)out)[i] = (double)x;
  }
}

uint64_t synth_stream_id(uint64_t seed, uint64_t a, uint64_t b) { return synth_stream(seed, a, b); }
uint64_t synth_sm64_host(uint64_t x) { return synth_sm64(x); }

/*
 * synth.h -- seeded, counter-based input generator shared by the test oracle
 * and the GPU benchmark/tests.  It holds NONE of the method's arithmetic: it
 * only draws the random inputs (weights, embeddings) that PAPER.md leaves to
 * the user ("random-init weights", SURVEY.md 8(d) "Synthetic inputs").
 *
 *   sm64(x)            splitmix64 finaliser
 *   stream(seed,a,b) = sm64(sm64(sm64(seed) ^ a) ^ b)
 *   value i of a stream: r = sm64(stream + i);
 *       uniform kind : x = offset + scale * (2*u - 1),  u = (r >> 11) * 2^-53
 *   computed with ONE rounding from an exact integer, so host (gcc) and device
 *   (nvcc) produce bit-identical float / bf16 values:
 *       x = offset + (double)((int64)(r >> 11) - 2^52) * (scale * 2^-52)
 *   then rounded to float (RNE) and optionally to bf16 (RNE).
 *
 * Streams: a = 2 + layer for layer tensors (b = tensor id in
 * the energon_layer_weights order), a = 1<<20 for the embeddings.
 */
#ifndef SYNTH_H
#define SYNTH_H
#include <stdint.h>

#if defined(__CUDACC__)
#define SYNTH_HD __host__ __device__ __forceinline__
#else
#define SYNTH_HD static inline
#endif

SYNTH_HD uint64_t synth_sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

SYNTH_HD uint64_t synth_stream(uint64_t seed, uint64_t a, uint64_t b) {
  return synth_sm64(synth_sm64(synth_sm64(seed) ^ a) ^ b);
}

/* value i of stream s as a float: offset + scale*(2u-1), u in [0,1) */
SYNTH_HD float synth_uniform(uint64_t s, uint64_t i, double scale, double offset) {
  uint64_t r = synth_sm64(s + i);
  int64_t k = (int64_t)(r >> 11) - (int64_t)(1ull << 52);   /* exact in double */
  double c = scale * (1.0 / 4503599627370496.0);             /* scale * 2^-52 */
#if defined(__CUDA_ARCH__)
  double x = __dadd_rn(__dmul_rn((double)k, c), offset);     /* no FMA contraction */
#else
  double x = (double)k * c;                                  /* one rounding */
  x = x + offset;                                            /* (host: -ffp-contract=off) */
#endif
  return (float)x;                                           /* RNE */
}

/* float -> bf16 bits, round to nearest even (NaN not produced by the generator) */
SYNTH_HD uint16_t synth_f32_to_bf16(float f) {
  union { float f; uint32_t u; } v;
  v.f = f;
  uint32_t lsb = (v.u >> 16) & 1u;
  uint32_t r = v.u + 0x7FFFu + lsb;
  return (uint16_t)(r >> 16);
}

#endif

// attention.cu -- a6: masked scaled-dot-product attention on the rebuilt padded layout.
//
// PAPER.md:136-137 (causal mask), PAPER.md:365 ("the multi-head attention module still requires the
// padding area").  Q, K, V, O are [B, hk, S, d] (this rank's hk heads).
// Query s of sequence b sees key t iff t < lens[b] and (not causal or t <= s):
// queries s >= lens[b] are never computed and keys t >= lens[b] are never read, so the pad rows of
// Q/K/V (which a5 never writes) cannot leak in, not even as 0 * NaN.
#include <float.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace energon {

// ----------------------------------------------------------------------------- SIMT reference kernel
// One CTA per (query row, head, sequence).  fp32 scores / softmax / accumulation.  Used by the fp32
// parity mode and head sizes other than 64 / 128; the bf16 production mode uses the tcgen05 kernel
// (attention_tc.cu).
template <typename Act>
__global__ void __launch_bounds__(128) attention_simt_kernel(const Act* __restrict__ Q, const Act* __restrict__ K,
                                                             const Act* __restrict__ V, Act* __restrict__ O,
                                                             const int* __restrict__ lens,
                                                             int hk, int S, int d, int causal, float scale) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  float* q = sm;        // [d]
  float* sc = sm + d;   // [S]
  __shared__ float red[32];
  const int s = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
  const int len = lens[b];
  if (s >= len) return;
  const int nk = causal ? min(s + 1, len) : len;
  const int64_t base = ((int64_t)b * hk + head) * S * d;
  for (int j = threadIdx.x; j < d; j += blockDim.x) q[j] = to_f32(Q[base + (int64_t)s * d + j]);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int t = wid; t < nk; t += nw) {
    float dot = 0.f;
    for (int j = lane; j < d; j += 32) dot += q[j] * to_f32(K[base + (int64_t)t * d + j]);
    dot = warp_sum(dot);
    if (lane == 0) sc[t] = dot * scale;
  }
  __syncthreads();
  float m = -FLT_MAX;
  for (int t = threadIdx.x; t < nk; t += blockDim.x) m = fmaxf(m, sc[t]);
  // block max
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[wid] = m;
  __syncthreads();
  m = red[0];
  for (int w = 1; w < nw; ++w) m = fmaxf(m, red[w]);
  __syncthreads();
  float part = 0.f;
  for (int t = threadIdx.x; t < nk; t += blockDim.x) {
    const float e = __expf(sc[t] - m);
    sc[t] = e;
    part += e;
  }
  const float den = block_sum(part, red);  // (block_sum syncs, so sc[] is complete afterwards)
  const float inv = 1.f / den;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float o = 0.f;
    for (int t = 0; t < nk; ++t) o += sc[t] * to_f32(V[base + (int64_t)t * d + j]);
    O[base + (int64_t)s * d + j] = from_f32<Act>(o * inv);
  }
}

template <typename Act>
void launch_attention_simt(const Act* Q, const Act* K, const Act* V, Act* O, const int* lens, int B, int hk, int S,
                           int d, int causal, cudaStream_t st) {
  if (B <= 0) return;
  dim3 grid(S, hk, B);
  const size_t smem = sizeof(float) * (size_t)(d + S);
  launch_k(attention_simt_kernel<Act>, dim3(grid), dim3(128), smem, st, Q, K, V, O, lens, hk, S, d, causal,
           1.f / sqrtf((float)d));
}

int attention_impl() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ENERGON_ATTN");
    v = e ? atoi(e) : 4;
    if (v != 4 && v != 5) v = 4;
  }
  return v;
}

template <typename Act>
void launch_attention(const Act* Q, const Act* K, const Act* V, Act* O, const int* lens_d, const uint32_t* work_d,
                      int B, int hk, int S, int d, int causal, cudaStream_t st, AttnMaps* maps) {
  // bf16, d = 64 / 128: the tcgen05 kernel; everything else (fp32 parity mode, other head sizes): SIMT
  if constexpr (sizeof(Act) == 2) {
    if ((d == 128 || d == 64) && work_d &&
        launch_attention_tc(Q, K, V, nullptr, nullptr, O, lens_d, work_d, B, hk, S, d, causal, st, maps))
      return;
  }
  launch_attention_simt<Act>(Q, K, V, O, lens_d, B, hk, S, d, causal, st);
}

bool launch_attention_packed(const bf16* Q, const bf16* K, const bf16* V, bf16* ctx_packed, const int* offsets,
                             const int* lens_d, const uint32_t* work_d, int B, int hk, int S, int d, int causal,
                             cudaStream_t st, AttnMaps* maps) {
  if (d != 128 && d != 64) return false;
  return launch_attention_tc(Q, K, V, ctx_packed, offsets, nullptr, lens_d, work_d, B, hk, S, d, causal, st, maps);
}

template void launch_attention<float>(const float*, const float*, const float*, float*, const int*, const uint32_t*,
                                      int, int, int, int, int, cudaStream_t, AttnMaps*);
template void launch_attention<bf16>(const bf16*, const bf16*, const bf16*, bf16*, const int*, const uint32_t*, int,
                                     int, int, int, int, cudaStream_t, AttnMaps*);

}  // namespace energon

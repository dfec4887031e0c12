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
// parity mode; the bf16 production mode uses the tensor-core kernel below.
template <typename Act>
__global__ void __launch_bounds__(128) attention_simt_kernel(const Act* __restrict__ Q, const Act* __restrict__ K,
                                                             const Act* __restrict__ V, Act* __restrict__ O, LensParam lp,
                                                             int hk, int S, int d, int causal, float scale) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  float* q = sm;        // [d]
  float* sc = sm + d;   // [S]
  __shared__ float red[32];
  const int s = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
  const int len = lp.lens[b];
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
void launch_attention_simt(const Act* Q, const Act* K, const Act* V, Act* O, const LensParam& lp, int B, int hk, int S,
                           int d, int causal, cudaStream_t st) {
  if (B <= 0) return;
  dim3 grid(S, hk, B);
  const size_t smem = sizeof(float) * (size_t)(d + S);
  launch_k(attention_simt_kernel<Act>, dim3(grid), dim3(128), smem, st, Q, K, V, O, lp, hk, S, d, causal, 1.f / sqrtf((float)d));
}

// ----------------------------------------------------------------------------- tensor-core kernel (bf16)
// Flash-style: one CTA = 64 query rows of one (sequence, head); 4 warps x 16 rows.  K/V tiles of 64
// keys are double-buffered in XOR-swizzled shared memory with cp.async (rows t >= len are zero-filled,
// never read from HBM).  S = Q K^T and O += P V on mma.sync.m16n8k16 (bf16 in, fp32 accumulate);
// online softmax in fp32 with exp2.  Only key tiles below min(len, q0 + 64) (causal) or len are
// visited, and only query tiles with q0 < len are launched into work (the rest exit at once).
// Attention is < 1% of the layer's FLOPs; legacy mma.sync is sufficient here.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int D>
__global__ void __launch_bounds__(128) attention_fa_kernel(const bf16* __restrict__ Q, const bf16* __restrict__ K,
                                                           const bf16* __restrict__ V, bf16* __restrict__ O,
                                                           bf16* __restrict__ Cp, const int* __restrict__ offsets,
                                                           LensParam lp, int hk, int S, int causal, float scale_log2) {
  pdl_trigger();
  pdl_wait();
  constexpr int BM = 64, BN = 64, CH = D / 8, KS = D / 16, NT = BN / 8, DT = D / 8;
  static_assert(CH >= 8, "swizzle needs >= 8 chunks per row");
  extern __shared__ __align__(128) uint8_t sm_raw[];
  bf16* sQ = reinterpret_cast<bf16*>(sm_raw);
  bf16* sK = sQ + BM * D;
  bf16* sV = sK + 2 * BN * D;
  const int qt = gridDim.x - 1 - blockIdx.x;  // longest-running (last) query tiles first
  const int head = blockIdx.y, b = blockIdx.z;
  const int len = lp.lens[b];
  const int q0 = qt * BM;
  if (q0 >= len) return;
  const int kv_end = causal ? min(len, q0 + BM) : len;
  const int nkv = (kv_end + BN - 1) / BN;
  const int64_t base = ((int64_t)b * hk + head) * S * D;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto sw = [](int row, int ch) { return row * D + ((ch ^ (row & 7)) << 3); };

  for (int i = tid; i < BM * CH; i += 128) {
    const int r = i / CH, ch = i % CH;
    const bool ok = q0 + r < len;
    cp_async16(sQ + sw(r, ch), Q + base + (int64_t)(ok ? q0 + r : 0) * D + ch * 8, ok);
  }
  auto load_kv = [&](int j, int buf) {
    const int k0 = j * BN;
    for (int i = tid; i < BN * CH; i += 128) {
      const int r = i / CH, ch = i % CH;
      const bool ok = k0 + r < len;
      const int64_t off = base + (int64_t)(ok ? k0 + r : 0) * D + ch * 8;
      cp_async16(sK + buf * BN * D + sw(r, ch), K + off, ok);
      cp_async16(sV + buf * BN * D + sw(r, ch), V + off, ok);
    }
  };
  load_kv(0, 0);
  cp_async_commit();

  uint32_t qf[KS][4];
  float o[DT][4];
#pragma unroll
  for (int i = 0; i < DT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const int row0 = q0 + warp * 16 + (lane >> 2), row1 = row0 + 8;

  for (int j = 0; j < nkv; ++j) {
    if (j + 1 < nkv) {
      load_kv(j + 1, (j + 1) & 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) ldsm_x4(qf[kk], sQ + sw(warp * 16 + (lane & 15), 2 * kk + (lane >> 4)));
    }
    const bf16* cK = sK + (j & 1) * BN * D;
    const bf16* cV = sV + (j & 1) * BN * D;
    // ---- S = Q K^T  (16 rows x 64 keys per warp)
    float sc[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
#pragma unroll
      for (int n = 0; n < NT; n += 2) {
        uint32_t kb[4];
        ldsm_x4(kb, cK + sw(n * 8 + (lane & 7) + ((lane >> 4) << 3), 2 * kk + ((lane >> 3) & 1)));
        mma_bf16(sc[n], qf[kk], kb[0], kb[1]);
        mma_bf16(sc[n + 1], qf[kk], kb[2], kb[3]);
      }
    }
    // ---- mask (t >= len, causal t > s) and online softmax in the log2 domain
    const int k0 = j * BN;
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int t = k0 + n * 8 + (lane & 3) * 2 + e;
        const bool bad = t >= len;
        float v0 = sc[n][e] * scale_log2, v1 = sc[n][2 + e] * scale_log2;
        if (bad || (causal && t > row0)) v0 = -INFINITY;
        if (bad || (causal && t > row1)) v1 = -INFINITY;
        sc[n][e] = v0;
        sc[n][2 + e] = v1;
        mx0 = fmaxf(mx0, v0);
        mx1 = fmaxf(mx1, v1);
      }
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float base0 = (mx0 == -INFINITY) ? 0.f : mx0, base1 = (mx1 == -INFINITY) ? 0.f : mx1;
    const float al0 = exp2f(m0 - base0), al1 = exp2f(m1 - base1);  // m = -inf -> 0
    m0 = mx0;
    m1 = mx1;
    float rs0 = 0.f, rs1 = 0.f;
    uint32_t pa[NT / 2][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const float p0 = exp2f(sc[n][0] - base0), p1 = exp2f(sc[n][1] - base0);
      const float p2 = exp2f(sc[n][2] - base1), p3 = exp2f(sc[n][3] - base1);
      rs0 += p0 + p1;
      rs1 += p2 + p3;
      pa[n >> 1][(n & 1) * 2 + 0] = pack2(p0, p1);
      pa[n >> 1][(n & 1) * 2 + 1] = pack2(p2, p3);
    }
    l0 = l0 * al0 + rs0;
    l1 = l1 * al1 + rs1;
#pragma unroll
    for (int i = 0; i < DT; ++i) {
      o[i][0] *= al0;
      o[i][1] *= al0;
      o[i][2] *= al1;
      o[i][3] *= al1;
    }
    // ---- O += P V   (P as the A operand: keys 16*kk .. 16*kk+15)
#pragma unroll
    for (int kk = 0; kk < BN / 16; ++kk) {
#pragma unroll
      for (int dn = 0; dn < DT; dn += 2) {
        uint32_t vb[4];
        ldsm_x4_t(vb, cV + sw(kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3), dn + (lane >> 4)));
        mma_bf16(o[dn], pa[kk], vb[0], vb[1]);
        mma_bf16(o[dn + 1], pa[kk], vb[2], vb[3]);
      }
    }
    __syncthreads();
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float inv0 = 1.f / l0, inv1 = 1.f / l1;
  // a7 fused (Cp != nullptr): write the packed row offsets[b] + s, columns head*D.. of [T, hk*D]
  bf16 *dst0, *dst1;
  if (Cp) {
    const int64_t t0 = __ldg(offsets + b);
    dst0 = Cp + (t0 + row0) * (int64_t)(hk * D) + head * D;
    dst1 = Cp + (t0 + row1) * (int64_t)(hk * D) + head * D;
  } else {
    dst0 = O + base + (int64_t)row0 * D;
    dst1 = O + base + (int64_t)row1 * D;
  }
#pragma unroll
  for (int i = 0; i < DT; ++i) {
    const int col = i * 8 + (lane & 3) * 2;
    if (row0 < len) *reinterpret_cast<uint32_t*>(dst0 + col) = pack2(o[i][0] * inv0, o[i][1] * inv0);
    if (row1 < len) *reinterpret_cast<uint32_t*>(dst1 + col) = pack2(o[i][2] * inv1, o[i][3] * inv1);
  }
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Second-generation kernel: single-buffered K/V (48 KB of shared memory at d = 128) and at most 128
// registers so 4 CTAs (16 warps) share an SM and hide each other's load latency; Q fragments are
// re-read from shared memory per key tile instead of being pinned in registers; the mask is only
// evaluated on key tiles that cross the length or the causal diagonal of the warp's rows; the
// softmax folds the 1/sqrt(d) scale into one FFMA before a raw ex2.approx.
template <int D>
__global__ void __launch_bounds__(128, 4) attention_fa2_kernel(const bf16* __restrict__ Q, const bf16* __restrict__ K,
                                                               const bf16* __restrict__ V, bf16* __restrict__ O,
                                                               bf16* __restrict__ Cp, const int* __restrict__ offsets,
                                                               LensParam lp, int hk, int S, int causal, float scale_log2) {
  pdl_trigger();
  pdl_wait();
  constexpr int BM = 64, BN = 64, CH = D / 8, KS = D / 16, NT = BN / 8, DT = D / 8;
  static_assert(CH >= 8, "swizzle needs >= 8 chunks per row");
  extern __shared__ __align__(128) uint8_t sm_raw[];
  bf16* sQ = reinterpret_cast<bf16*>(sm_raw);
  bf16* sK = sQ + BM * D;
  bf16* sV = sK + BN * D;
  const int qt = gridDim.x - 1 - blockIdx.x;
  const int head = blockIdx.y, b = blockIdx.z;
  const int len = lp.lens[b];
  const int q0 = qt * BM;
  if (q0 >= len) return;
  const int kv_end = causal ? min(len, q0 + BM) : len;
  const int nkv = (kv_end + BN - 1) / BN;
  const int64_t base = ((int64_t)b * hk + head) * S * D;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto sw = [](int row, int ch) { return row * D + ((ch ^ (row & 7)) << 3); };

  for (int i = tid; i < BM * CH; i += 128) {
    const int r = i / CH, ch = i % CH;
    const bool ok = q0 + r < len;
    cp_async16(sQ + sw(r, ch), Q + base + (int64_t)(ok ? q0 + r : 0) * D + ch * 8, ok);
  }
  float o[DT][4];
#pragma unroll
  for (int i = 0; i < DT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // m in the scaled log2 domain
  const int wrow = q0 + warp * 16;
  const int row0 = wrow + (lane >> 2), row1 = row0 + 8;

  for (int j = 0; j < nkv; ++j) {
    const int k0 = j * BN;
    for (int i = tid; i < BN * CH; i += 128) {
      const int r = i / CH, ch = i % CH;
      const bool ok = k0 + r < len;
      const int64_t off = base + (int64_t)(ok ? k0 + r : 0) * D + ch * 8;
      cp_async16(sK + sw(r, ch), K + off, ok);
      cp_async16(sV + sw(r, ch), V + off, ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    // ---- S = Q K^T
    float sc[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
      uint32_t qf[4];
      ldsm_x4(qf, sQ + sw(warp * 16 + (lane & 15), 2 * kk + (lane >> 4)));
#pragma unroll
      for (int n = 0; n < NT; n += 2) {
        uint32_t kb[4];
        ldsm_x4(kb, sK + sw(n * 8 + (lane & 7) + ((lane >> 4) << 3), 2 * kk + ((lane >> 3) & 1)));
        mma_bf16(sc[n], qf, kb[0], kb[1]);
        mma_bf16(sc[n + 1], qf, kb[2], kb[3]);
      }
    }
    // ---- mask only where the tile crosses len or this warp's causal diagonal
    const bool need_mask = (k0 + BN > len) || (causal && k0 + BN - 1 > wrow);
    if (need_mask) {
#pragma unroll
      for (int n = 0; n < NT; ++n) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int t = k0 + n * 8 + (lane & 3) * 2 + e;
          const bool bad = t >= len;
          if (bad || (causal && t > row0)) sc[n][e] = -INFINITY;
          if (bad || (causal && t > row1)) sc[n][2 + e] = -INFINITY;
        }
      }
    }
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      mx0 = fmaxf(mx0, fmaxf(sc[n][0], sc[n][1]));
      mx1 = fmaxf(mx1, fmaxf(sc[n][2], sc[n][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0 * scale_log2), mn1 = fmaxf(m1, mx1 * scale_log2);
    const float b0 = (mn0 == -INFINITY) ? 0.f : mn0, b1 = (mn1 == -INFINITY) ? 0.f : mn1;
    const float al0 = ex2(m0 - b0), al1 = ex2(m1 - b1);
    m0 = mn0;
    m1 = mn1;
    float rs0 = 0.f, rs1 = 0.f;
    uint32_t pa[NT / 2][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const float p0 = ex2(fmaf(sc[n][0], scale_log2, -b0)), p1 = ex2(fmaf(sc[n][1], scale_log2, -b0));
      const float p2 = ex2(fmaf(sc[n][2], scale_log2, -b1)), p3 = ex2(fmaf(sc[n][3], scale_log2, -b1));
      rs0 += p0 + p1;
      rs1 += p2 + p3;
      pa[n >> 1][(n & 1) * 2 + 0] = pack2(p0, p1);
      pa[n >> 1][(n & 1) * 2 + 1] = pack2(p2, p3);
    }
    l0 = l0 * al0 + rs0;
    l1 = l1 * al1 + rs1;
#pragma unroll
    for (int i = 0; i < DT; ++i) {
      o[i][0] *= al0;
      o[i][1] *= al0;
      o[i][2] *= al1;
      o[i][3] *= al1;
    }
    // ---- O += P V
#pragma unroll
    for (int kk = 0; kk < BN / 16; ++kk) {
#pragma unroll
      for (int dn = 0; dn < DT; dn += 2) {
        uint32_t vb[4];
        ldsm_x4_t(vb, sV + sw(kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3), dn + (lane >> 4)));
        mma_bf16(o[dn], pa[kk], vb[0], vb[1]);
        mma_bf16(o[dn + 1], pa[kk], vb[2], vb[3]);
      }
    }
    __syncthreads();
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float inv0 = 1.f / l0, inv1 = 1.f / l1;
  bf16 *dst0, *dst1;
  if (Cp) {
    const int64_t t0 = __ldg(offsets + b);
    dst0 = Cp + (t0 + row0) * (int64_t)(hk * D) + head * D;
    dst1 = Cp + (t0 + row1) * (int64_t)(hk * D) + head * D;
  } else {
    dst0 = O + base + (int64_t)row0 * D;
    dst1 = O + base + (int64_t)row1 * D;
  }
#pragma unroll
  for (int i = 0; i < DT; ++i) {
    const int col = i * 8 + (lane & 3) * 2;
    if (row0 < len) *reinterpret_cast<uint32_t*>(dst0 + col) = pack2(o[i][0] * inv0, o[i][1] * inv0);
    if (row1 < len) *reinterpret_cast<uint32_t*>(dst1 + col) = pack2(o[i][2] * inv1, o[i][3] * inv1);
  }
}

int attention_impl() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ENERGON_ATTN");
    v = e ? atoi(e) : 4;
    if (v < 1 || v > 4) v = 4;
  }
  return v;
}

template <int D>
static void launch_fa(const bf16* Q, const bf16* K, const bf16* V, bf16* O, bf16* Cp, const int* offsets,
                      const LensParam& lp, int B, int hk, int S, int causal, cudaStream_t st) {
  if (attention_impl() >= 3 &&
      launch_attention_tc(Q, K, V, Cp, offsets, O, lp, B, hk, S, D, causal, st, attention_impl() == 4))
    return;
  const int gen = attention_impl() == 1 ? 1 : 2;
  dim3 grid((S + 63) / 64, hk, B);
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  if (gen == 1) {
    const int smem = (64 + 4 * 64) * D * 2;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(attention_fa_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr = true;
    }
    launch_k(attention_fa_kernel<D>, dim3(grid), dim3(128), smem, st, Q, K, V, O, Cp, offsets, lp, hk, S, causal, scale_log2);
  } else {
    const int smem = (64 + 2 * 64) * D * 2;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(attention_fa2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr = true;
    }
    launch_k(attention_fa2_kernel<D>, dim3(grid), dim3(128), smem, st, Q, K, V, O, Cp, offsets, lp, hk, S, causal, scale_log2);
  }
}

template <typename Act>
void launch_attention(const Act* Q, const Act* K, const Act* V, Act* O, const LensParam& lp, int B, int hk, int S, int d,
                      int causal, cudaStream_t st) {
  if constexpr (sizeof(Act) == 2) {
    if (d == 128) return launch_fa<128>(Q, K, V, O, nullptr, nullptr, lp, B, hk, S, causal, st);
    if (d == 64) return launch_fa<64>(Q, K, V, O, nullptr, nullptr, lp, B, hk, S, causal, st);
  }
  launch_attention_simt<Act>(Q, K, V, O, lp, B, hk, S, d, causal, st);
}

bool launch_attention_packed(const bf16* Q, const bf16* K, const bf16* V, bf16* ctx_packed, const int* offsets,
                             const LensParam& lp, int B, int hk, int S, int d, int causal, cudaStream_t st) {
  if (d == 128) return launch_fa<128>(Q, K, V, nullptr, ctx_packed, offsets, lp, B, hk, S, causal, st), true;
  if (d == 64) return launch_fa<64>(Q, K, V, nullptr, ctx_packed, offsets, lp, B, hk, S, causal, st), true;
  return false;
}

template void launch_attention<float>(const float*, const float*, const float*, float*, const LensParam&, int, int, int,
                                      int, int, cudaStream_t);
template void launch_attention<bf16>(const bf16*, const bf16*, const bf16*, bf16*, const LensParam&, int, int, int, int,
                                     int, cudaStream_t);

}  // namespace energon

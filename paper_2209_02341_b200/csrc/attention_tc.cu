// attention_tc.cu -- a6 (+ a7 fused) on the 5th-generation tensor cores: masked softmax attention
// over the rebuilt padded per-head layout Q, K, V [B, hk, S, d] ("the multi-head
// attention module still requires the padding area"), writing the packed context
// rows [T, hk*d] at offsets[b] + s (PAPER.md:373 kernel #2 fused).
//
// Persistent: each CTA (2 per SM) loops over a heaviest-first list of work items built on the device by
// the index-maps kernel (build_attn_work: one item = 128 query rows of one sequence; item w = pair
// w / hk, head w % hk), so the next item's Q / K loads overlap the current item's tail.  6 warps:
//   warp 0    TMA producer: the Q tile once, then K and V tiles of 64 keys (double-buffered)
//   warp 1    MMA issuer (one thread): S = Q K^T (M=128, N=64, K=d; K-major A and B) into TMEM, and
//             O += P V with P read straight from TMEM (M=128, N=d, K=64; B = V, MN-major)
//   warps 2-5 softmax: thread i owns query row i (TMEM lane i): tcgen05.ld its 64 scores, masks
//             (t >= len, causal t > s), runs the online softmax in fp32 / exp2 and writes its P row
//             (bf16) back over its scores in TMEM; O stays in TMEM and is rescaled only when the row
//             maximum grew by more than 2^8 (exact: P values are bounded by 256).
// Key tiles stop at min(len, q0 + 128) (causal) or len; query tiles with q0 >= len are not items.
// Item epilogue: O / l leaves through shared memory by TMA bulk-tensor stores (32 x 32 boxes, one staging
// buffer per softmax warp) whenever all 32 rows of the warp are queries; O's TMEM is released to the next
// item right after its last tcgen05.ld.  Warps holding the sequence's last, partial rows store per thread.
// Rows t >= len of the last V tile are zeroed in shared memory before P.V, so pad rows of V that a5
// never wrote (possibly NaN) cannot reach the output even as 0 * NaN.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace energon {

constexpr int ATTN_BM = 128, ATTN_BN = 64;  // query rows per item, keys per tile (the work list's costs)
// the work list's item height / cost unit follow the selected kernel (v3: 256-row items, 128-key tiles)
int attention_tile_bm() { return attention_impl() == 5 ? 256 : ATTN_BM; }
int attention_tile_bn() { return attention_impl() == 5 ? 128 : ATTN_BN; }

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (FA4's MUFU offload): x = j + f with j = round(x), |f| <= 1/2; 2^f by a degree-3
// polynomial (max relative error ~1e-4, below the bf16 rounding of P, 2^-9); 2^j added to the exponent
// bits.  x is clamped at -127 (a result of ~1e-38 instead of 0), so only unmasked keys may use it.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -127.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: round to nearest integer in the low mantissa bits
  const float xr = t - 12582912.f;
  const float f = x - xr;
  const int j = __float_as_int(t) - 0x4B400000;
  const float p = fmaf(fmaf(fmaf(0.0555041f, f, 0.2402265f), f, 0.6931472f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + (j << 23));
}

// MN-major (N contiguous) 128B-swizzled operand: 64-element rows of 128 B; SBO = 1024 B between
// 8-row groups along K, LBO = distance between 64-wide blocks along N.
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t saddr, uint32_t lbo_bytes) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// ============================================================================ the kernel
// The softmax of key tile j never waits for P_{j-1} V: S / P are double-buffered in TMEM (S_b at columns
// [b BN, (b+1) BN), P_b written over the first BN/2 columns of S_b as packed bf16) and P V reads its A
// operand straight from TMEM (tcgen05.mma ... [d], [a_tmem], b_desc), V is double-buffered in shared
// memory, and the MMA thread issues S_{t+1} before P_t V_t across the CTA's whole tile sequence
// (items included), so the tensor pipe works on the next scores while the softmax warps run.
//   TMEM: S0 | S1 | O  (BN + BN + D <= 256 columns)      smem: Q | K[2] | V[2] | epilogue staging [4 warps]
// Ordering: S_t overwrites buffer t&1 only after P_{t-2} V (the last reader of that buffer) completed
// (p_free); the O rescale waits for P_{t-1} V (o_full); P_t V is issued after p_full of tile t.
template <int D>
struct Attn2Cfg {
  static constexpr int BM = ATTN_BM, BN = ATTN_BN, DH = D / 64;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int K_BYTES = BN * D * 2;
  static constexpr int V_BYTES = BN * D * 2;
  static constexpr int STG_BYTES = 4 * 32 * 64;  // epilogue staging: per softmax warp 32 rows x 32 columns (bf16)
  static constexpr int SMEM = Q_BYTES + 2 * K_BYTES + 2 * V_BYTES + STG_BYTES + 1024 + 256;
  static constexpr int TMEM_COLS = 256;  // 2 * BN + D <= 256 for D <= 128
  // S = Q K^T: M=128, N=BN, both K-major
  static constexpr uint32_t IDESC_S = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                      ((uint32_t)(BM >> 4) << 24);
  // O += P V: M=128, N=D, A K-major, B MN-major (bit 16)
  static constexpr uint32_t IDESC_O = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(D >> 3) << 17) |
                                      ((uint32_t)(BM >> 4) << 24);
};

__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
          tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}

// Batched MMA issue.  The MMA thread is a single lane, so every tcgen05.mma it issues from C++ is wrapped by
// the compiler in an elect / R2UR.BROADCAST loop (~14 instructions, 40-90 clocks per MMA measured in the
// traces), which is longer than a 128 x 64 x 16 S MMA takes to execute (32 clocks).  These helpers issue a
// tile's whole group of MMAs from one asm block, advancing the descriptors with PTX adds, so the loop wraps
// the group once (ATTN_MMA_BATCH=0 restores the per-MMA issue for A/B).
#ifndef ATTN_MMA_BATCH
#define ATTN_MMA_BATCH 1
#endif
// S = Q K^T over K = d: 4 MMAs (d = 64) from (a0, b0) advancing 32 B each; 8 (d = 128) with the second 64-wide
// half at (a1, b1).  The first MMA overwrites the accumulator, the rest accumulate.
__device__ __forceinline__ void umma_s4(uint32_t d, uint64_t a0, uint64_t b0, uint32_t idesc) {
  asm volatile(
      "{\n.reg .pred p;\n.reg .b64 x, y;\nsetp.ne.b32 p, 0, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\nsetp.eq.b32 p, 0, 0;\n"
      "add.s64 x, %1, 2;\nadd.s64 y, %2, 2;\ntcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n"
      "add.s64 x, %1, 4;\nadd.s64 y, %2, 4;\ntcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n"
      "add.s64 x, %1, 6;\nadd.s64 y, %2, 6;\ntcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n}\n" ::"r"(d),
      "l"(a0), "l"(b0), "r"(idesc));
}
__device__ __forceinline__ void umma_s8(uint32_t d, uint64_t a0, uint64_t b0, uint64_t a1, uint64_t b1, uint32_t idesc) {
  asm volatile(
      "{\n.reg .pred p;\n.reg .b64 x, y;\nsetp.ne.b32 p, 0, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\nsetp.eq.b32 p, 0, 0;\n"
      "add.s64 x, %1, 2;\nadd.s64 y, %2, 2;\ntcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n"
      "add.s64 x, %1, 4;\nadd.s64 y, %2, 4;\ntcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n"
      "add.s64 x, %1, 6;\nadd.s64 y, %2, 6;\ntcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %5, %3, p;\n"
      "add.s64 x, %4, 2;\nadd.s64 y, %5, 2;\ntcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n"
      "add.s64 x, %4, 4;\nadd.s64 y, %5, 4;\ntcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n"
      "add.s64 x, %4, 6;\nadd.s64 y, %5, 6;\ntcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n}\n" ::"r"(d),
      "l"(a0), "l"(b0), "r"(idesc), "l"(a1), "l"(b1));
}
// O (+)= P V over 64 keys (4 MMAs): A = P from TMEM columns ta + 8 kk, B = V (MN-major) descriptor + 128 kk;
// acc = 0 makes the first MMA overwrite O.
__device__ __forceinline__ void umma_pv4(uint32_t d, uint32_t ta, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\n.reg .b32 t;\n.reg .b64 y;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\nsetp.eq.b32 p, 0, 0;\n"
      "add.u32 t, %1, 8;\nadd.s64 y, %2, 128;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [t], y, %3, p;\n"
      "add.u32 t, %1, 16;\nadd.s64 y, %2, 256;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [t], y, %3, p;\n"
      "add.u32 t, %1, 24;\nadd.s64 y, %2, 384;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [t], y, %3, p;\n}\n" ::"r"(d),
      "r"(ta), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_s4e(uint32_t d, uint64_t a0, uint64_t b0, uint32_t idesc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\n.reg .b64 x, y;\nsetp.ne.b32 p, 0, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\nsetp.eq.b32 p, 0, 0;\n"
      "add.s64 x, %1, 2;\nadd.s64 y, %2, 2;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n"
      "add.s64 x, %1, 4;\nadd.s64 y, %2, 4;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n"
      "add.s64 x, %1, 6;\nadd.s64 y, %2, 6;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n}\n" ::"r"(d),
      "l"(a0), "l"(b0), "r"(idesc));
}
__device__ __forceinline__ void umma_s8e(uint32_t d, uint64_t a0, uint64_t b0, uint64_t a1, uint64_t b1, uint32_t idesc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\n.reg .b64 x, y;\nsetp.ne.b32 p, 0, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\nsetp.eq.b32 p, 0, 0;\n"
      "add.s64 x, %1, 2;\nadd.s64 y, %2, 2;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n"
      "add.s64 x, %1, 4;\nadd.s64 y, %2, 4;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n"
      "add.s64 x, %1, 6;\nadd.s64 y, %2, 6;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %5, %3, p;\n"
      "add.s64 x, %4, 2;\nadd.s64 y, %5, 2;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n"
      "add.s64 x, %4, 4;\nadd.s64 y, %5, 4;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n"
      "add.s64 x, %4, 6;\nadd.s64 y, %5, 6;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], x, y, %3, p;\n}\n" ::"r"(d),
      "l"(a0), "l"(b0), "r"(idesc), "l"(a1), "l"(b1));
}
// O (+)= P V over 64 keys (4 MMAs): A = P from TMEM columns ta + 8 kk, B = V (MN-major) descriptor + 128 kk;
// acc = 0 makes the first MMA overwrite O.
__device__ __forceinline__ void umma_pv4e(uint32_t d, uint32_t ta, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\n.reg .b32 t;\n.reg .b64 y;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\nsetp.eq.b32 p, 0, 0;\n"
      "add.u32 t, %1, 8;\nadd.s64 y, %2, 128;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t], y, %3, p;\n"
      "add.u32 t, %1, 16;\nadd.s64 y, %2, 256;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t], y, %3, p;\n"
      "add.u32 t, %1, 24;\nadd.s64 y, %2, 384;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t], y, %3, p;\n}\n" ::"r"(d),
      "r"(ta), "l"(b), "r"(idesc), "r"(acc));
}

// O (+)= P V over 128 keys (v3): 8 MMAs, A = P at TMEM columns ta + 8 kk, B = V descriptor + 128 kk; one elected lane
__device__ __forceinline__ void umma_pv8e(uint32_t d, uint32_t ta, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\n.reg .b32 t;\n.reg .b64 y;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\nsetp.eq.b32 p, 0, 0;\n"
      "add.u32 t, %1, 8;\nadd.s64 y, %2, 128;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t], y, %3, p;\n"
      "add.u32 t, %1, 16;\nadd.s64 y, %2, 256;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t], y, %3, p;\n"
      "add.u32 t, %1, 24;\nadd.s64 y, %2, 384;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t], y, %3, p;\n"
      "add.u32 t, %1, 32;\nadd.s64 y, %2, 512;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t], y, %3, p;\n"
      "add.u32 t, %1, 40;\nadd.s64 y, %2, 640;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t], y, %3, p;\n"
      "add.u32 t, %1, 48;\nadd.s64 y, %2, 768;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t], y, %3, p;\n"
      "add.u32 t, %1, 56;\nadd.s64 y, %2, 896;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t], y, %3, p;\n}\n" ::"r"(d),
      "r"(ta), "l"(b), "r"(idesc), "r"(acc));
}
// expect_tx + the 64-column halves of one tile (DH = 1 or 2 loads) by one elected lane of a converged warp
__device__ __forceinline__ void tma_tile_e(const CUtensorMap* m, uint32_t dst, uint32_t half_bytes, uint64_t* bar,
                                           uint32_t bytes, int y, int dh) {
  asm volatile(
      "{\n.reg .pred e, two;\n.reg .b32 d1;\nelect.sync _|e, 0xffffffff;\nsetp.ne.and.b32 two, %5, 1, e;\n"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%2], %3;\n"
      "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {0, %4}], [%2];\n"
      "add.u32 d1, %0, %6;\n"
      "@two cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [d1], [%1, {64, %4}], [%2];\n}\n"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(bytes), "r"(y), "r"(dh), "r"(half_bytes)
      : "memory");
}
// Epilogue by TMA: one softmax warp's 32 rows x 32 columns of O / l, bf16, staged in shared memory with the
// 64-byte swizzle of the output map (16-byte chunk j of row r at chunk j ^ ((r >> 1) & 3)) and stored with one
// bulk-tensor store.  The per-thread row stores it replaces touched 32 rows per instruction (half-used 32-byte
// sectors) and blocked the softmax warps: dropping them altogether (a probe with wrong output) sped the
// config-3 mix up from 50.9 to 38.3 us; this epilogue gets 47.2 us.  One 2 KB buffer per warp: 32 x 16 boxes
// double-buffered in the same space measured slower (48.9 us), and two 2 KB buffers per warp exceed the
// shared memory two CTAs per SM leave by 256 bytes.
__device__ __forceinline__ void attn_stage32(const uint32_t* o, float inv, uint32_t stg, int lane) {
  const uint32_t base = stg + lane * 64;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t a = base + ((j ^ ((lane >> 1) & 3)) << 4);
    const uint32_t* e = o + 8 * j;
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a),
                 "r"(pack_bf16x2(__uint_as_float(e[0]) * inv, __uint_as_float(e[1]) * inv)),
                 "r"(pack_bf16x2(__uint_as_float(e[2]) * inv, __uint_as_float(e[3]) * inv)),
                 "r"(pack_bf16x2(__uint_as_float(e[4]) * inv, __uint_as_float(e[5]) * inv)),
                 "r"(pack_bf16x2(__uint_as_float(e[6]) * inv, __uint_as_float(e[7]) * inv))
                 : "memory");
  }
}
// 16 columns of one row (32 bytes: a whole sector) with one 256-bit store (STG.E.256) -- the fallback for warps
// holding a sequence's last, partial rows (half as many store instructions as 16-byte stores, full sectors)
__device__ __forceinline__ void attn_st256(bf16* dst, const uint32_t* e, float inv) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst),
               "r"(pack_bf16x2(__uint_as_float(e[0]) * inv, __uint_as_float(e[1]) * inv)),
               "r"(pack_bf16x2(__uint_as_float(e[2]) * inv, __uint_as_float(e[3]) * inv)),
               "r"(pack_bf16x2(__uint_as_float(e[4]) * inv, __uint_as_float(e[5]) * inv)),
               "r"(pack_bf16x2(__uint_as_float(e[6]) * inv, __uint_as_float(e[7]) * inv)),
               "r"(pack_bf16x2(__uint_as_float(e[8]) * inv, __uint_as_float(e[9]) * inv)),
               "r"(pack_bf16x2(__uint_as_float(e[10]) * inv, __uint_as_float(e[11]) * inv)),
               "r"(pack_bf16x2(__uint_as_float(e[12]) * inv, __uint_as_float(e[13]) * inv)),
               "r"(pack_bf16x2(__uint_as_float(e[14]) * inv, __uint_as_float(e[15]) * inv))
               : "memory");
}
__device__ __forceinline__ void attn_tma_store(const CUtensorMap* map, uint32_t src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n"
               "cp.async.bulk.commit_group;" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(x), "r"(y)
               : "memory");
}
// commit by one elected lane of a converged warp
__device__ __forceinline__ void umma_commit_e(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
      : "memory");
}
// ATTN_WARP_ISSUE (default): the MMA role runs on its whole warp, converged, and each asm block elects one lane to
// issue -- ptxas then predicates UTCHMMA on a uniform predicate (@UP) with plain R2UR operands, instead of
// wrapping every MMA of a single-lane branch in an ELECT / R2UR.BROADCAST / BRA.U.ANY loop.
#ifndef ATTN_WARP_ISSUE
#define ATTN_WARP_ISSUE 1
#endif
#ifndef ATTN2_OBSERVE_ALL  // A/B: 1 = the softmax warps wait for every tile's P V after handing P over (old behaviour)
#define ATTN2_OBSERVE_ALL 0
#endif

template <int D>
__global__ void __launch_bounds__(192, 2)
    attention_tc2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ Cp, const int* __restrict__ offsets,
                         bf16* __restrict__ Opad, const int* __restrict__ lens, const uint32_t* __restrict__ work,
                         int hk, int S, int causal, float scale_log2, const __grid_constant__ CUtensorMap tmO,
                         int o_tma) {
  using C = Attn2Cfg<D>;
  constexpr int BM = C::BM, BN = C::BN, DH = C::DH;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + C::Q_BYTES;
  uint8_t* sV = sK + 2 * C::K_BYTES;
  uint8_t* sStg = sV + 2 * C::V_BYTES;  // [4 softmax warps][32 rows][64 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStg + C::STG_BYTES);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* o_empty = bars + 2;
  uint64_t* o_full = bars + 3;    // [2]: P_t V_t done, one phase per two tiles (see the softmax waits)
  uint64_t* k_full = bars + 5;    // [2]
  uint64_t* k_empty = bars + 7;   // [2]
  uint64_t* v_full = bars + 9;    // [2]
  uint64_t* v_empty = bars + 11;  // [2]
  uint64_t* s_full = bars + 13;   // [2]
  uint64_t* p_full = bars + 15;   // [2]
  uint64_t* p_free = bars + 17;   // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 19);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    if (o_tma) tma_prefetch_desc(&tmO);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    mbar_init(o_empty, 4);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&o_full[i], 1);
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&p_free[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  // Dependents may launch only once this CTA HOLDS its TMEM: a CTA that triggered before allocating
  // could find its columns taken by a co-resident dependent CTA that then waits (griddepcontrol.wait)
  // on this grid -- a cycle.
  pdl_trigger();
  pdl_wait();  // the work list, lengths and Q / K / V are written by earlier kernels of the forward
  const int items = (int)__ldg(work) * hk;
  const uint32_t tO = tmem_base + 2 * BN;

  // the CTA's k-th item: heaviest-first list dealt out boustrophedon (round k even: slot bid, odd:
  // slot G-1-bid), so no CTA takes the heaviest item of every round (simulated makespan on config 3:
  // 45.2 -> 41.3 us of item cost vs plain round-robin)
  auto item_at = [&](int k) { return k * (int)gridDim.x + ((k & 1) ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x); };
  auto decode = [&](int w, int& b, int& head, int& q0, int& nkv, int& len) {
    const uint32_t pr = __ldg(work + 1 + w / hk);
    head = w % hk;
    b = (int)(pr >> 16);
    q0 = (int)(pr & 0xFFFFu) * BM;
    len = __ldg(lens + b);
    const int kv_end = causal ? min(len, q0 + BM) : len;
    nkv = (kv_end + BN - 1) / BN;
  };

  if (warp == 0) {
    if (ATTN_WARP_ISSUE || lane == 0) {  // (ATTN_WARP_ISSUE: converged warp, one elected lane issues)
      // ---------------- TMA producer: per item Q once, then K_0, K_1, V_0, K_2, V_1, ... (t = CTA tile count)
      int t = 0, qi = 0;
      auto load = [&](const CUtensorMap* m, uint8_t* dst, uint32_t half_bytes, uint64_t* bar, uint32_t bytes, int y) {
        if (ATTN_WARP_ISSUE) {
          __syncwarp();
          tma_tile_e(m, smem_u32(dst), half_bytes, bar, bytes, y, DH);
        } else {
          mbar_expect_tx(bar, bytes);
#pragma unroll
          for (int h = 0; h < DH; ++h) tma_load_2d(m, smem_u32(dst + h * half_bytes), bar, h * 64, y);
        }
      };
      for (int w = item_at(0); w < items; w = item_at(++qi)) {
        int b, head, q0, nkv, len;
        decode(w, b, head, q0, nkv, len);
        const int row_base = (b * hk + head) * S;
        mbar_wait(q_empty, (qi & 1) ^ 1);  // the previous item's last S has consumed Q
        load(&tmQ, sQ, BM * 128, q_full, C::Q_BYTES, row_base + q0);
        auto load_k = [&](int tt, int j) {
          const int s2 = tt & 1;
          mbar_wait(&k_empty[s2], ((tt >> 1) & 1) ^ 1);
          load(&tmK, sK + s2 * C::K_BYTES, BN * 128, &k_full[s2], C::K_BYTES, row_base + j * BN);
        };
        load_k(t, 0);
        for (int j = 0; j < nkv; ++j) {
          if (j + 1 < nkv) load_k(t + j + 1, j + 1);
          const int tt = t + j, s2 = tt & 1;
          mbar_wait(&v_empty[s2], ((tt >> 1) & 1) ^ 1);
          load(&tmV, sV + s2 * C::V_BYTES, BN * 128, &v_full[s2], C::V_BYTES, row_base + j * BN);
        }
        t += nkv;
      }
    }
  } else if (warp == 1) {
    if (ATTN_WARP_ISSUE || lane == 0) {  // (ATTN_WARP_ISSUE: the whole warp, converged; one lane issues)
      // ---------------- MMA issuer: S_t, then P_{t-1} V_{t-1}, over the CTA's whole tile sequence
      int w = item_at(0), qi = 0, j = 0, nkv = 0;
      {
        int b_, h_, q_, l_;
        if (w < items) decode(w, b_, h_, q_, nkv, l_);
      }
      int t = 0;
      int pv_j = -1, pv_qi = 0;  // the tile whose P V is pending (j within its item), -1: none
      auto issue_pv = [&](int tt, int jj, int qq) {
        const int b2 = tt & 1;
        mbar_wait(&p_full[b2], (tt >> 1) & 1);
        mbar_wait(&v_full[b2], (tt >> 1) & 1);
        if (jj == 0) mbar_wait(o_empty, (qq & 1) ^ 1);  // the previous item's epilogue has read O
        tc_fence_after();
        const uint32_t tP = tmem_base + (uint32_t)(b2 * BN);
        if (ATTN_WARP_ISSUE) {
          __syncwarp();
          umma_pv4e(tO, tP, umma_desc_sw128_mn(smem_u32(sV + b2 * C::V_BYTES), BN * 128), C::IDESC_O, jj > 0 ? 1u : 0u);
          umma_commit_e(&v_empty[b2]);
          umma_commit_e(&p_free[b2]);
          umma_commit_e(&o_full[b2]);
          return;
        }
        if (ATTN_MMA_BATCH) {
          umma_pv4(tO, tP, umma_desc_sw128_mn(smem_u32(sV + b2 * C::V_BYTES), BN * 128), C::IDESC_O, jj > 0 ? 1u : 0u);
        } else {
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk) {
            const uint64_t bb = umma_desc_sw128_mn(smem_u32(sV + b2 * C::V_BYTES + kk * 16 * 128), BN * 128);
            umma_bf16_ts(tO, tP + (uint32_t)(kk * 8), bb, C::IDESC_O, (jj > 0 || kk > 0) ? 1u : 0u);
          }
        }
        umma_commit(&v_empty[b2]);
        umma_commit(&p_free[b2]);
        umma_commit(&o_full[b2]);
      };
      while (w < items) {
        const int b2 = t & 1;
        if (j == 0) {
          // finish the previous item before waiting for this item's Q: its epilogue overlaps the Q load
          if (pv_j >= 0) issue_pv(t - 1, pv_j, pv_qi);
          pv_j = -1;
          mbar_wait(q_full, qi & 1);
        }
        mbar_wait(&k_full[b2], (t >> 1) & 1);
        mbar_wait(&p_free[b2], ((t >> 1) & 1) ^ 1);  // P_{t-2} V done: buffer b2 is free
        tc_fence_after();
        const uint32_t tS = tmem_base + (uint32_t)(b2 * BN);
        if (ATTN_WARP_ISSUE) {
          __syncwarp();
          const uint64_t a0 = umma_desc_sw128(smem_u32(sQ));
          const uint64_t b0 = umma_desc_sw128(smem_u32(sK + b2 * C::K_BYTES));
          if (D == 128)
            umma_s8e(tS, a0, b0, umma_desc_sw128(smem_u32(sQ + BM * 128)),
                     umma_desc_sw128(smem_u32(sK + b2 * C::K_BYTES + BN * 128)), C::IDESC_S);
          else
            umma_s4e(tS, a0, b0, C::IDESC_S);
          umma_commit_e(&k_empty[b2]);
          if (j + 1 == nkv) umma_commit_e(q_empty);
          umma_commit_e(&s_full[b2]);
        } else if (ATTN_MMA_BATCH) {
          const uint64_t a0 = umma_desc_sw128(smem_u32(sQ));
          const uint64_t b0 = umma_desc_sw128(smem_u32(sK + b2 * C::K_BYTES));
          if (D == 128)
            umma_s8(tS, a0, b0, umma_desc_sw128(smem_u32(sQ + BM * 128)),
                    umma_desc_sw128(smem_u32(sK + b2 * C::K_BYTES + BN * 128)), C::IDESC_S);
          else
            umma_s4(tS, a0, b0, C::IDESC_S);
        } else {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk & 3) * 32;
            const uint64_t a = umma_desc_sw128(smem_u32(sQ + (kk >> 2) * BM * 128 + off));
            const uint64_t bb = umma_desc_sw128(smem_u32(sK + b2 * C::K_BYTES + (kk >> 2) * BN * 128 + off));
            umma_bf16(tS, a, bb, C::IDESC_S, kk > 0 ? 1u : 0u);
          }
        }
        if (!ATTN_WARP_ISSUE) {
          umma_commit(&k_empty[b2]);
          if (j + 1 == nkv) umma_commit(q_empty);
          umma_commit(&s_full[b2]);
        }
        if (pv_j >= 0) issue_pv(t - 1, pv_j, pv_qi);
        pv_j = j;
        pv_qi = qi;
        ++t;
        if (++j == nkv) {  // next item of this CTA
          j = 0;
          ++qi;
          w = item_at(qi);
          if (w < items) {
            int b_, h_, q_, l_;
            decode(w, b_, h_, q_, nkv, l_);
          }
        }
      }
      if (pv_j >= 0) issue_pv(t - 1, pv_j, pv_qi);
    }
  } else {
    // ---------------- softmax warps: thread owns query row r (= TMEM lane r)
    const int qd = warp & 3;
    const int r = qd * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const uint32_t stg = smem_u32(sStg + qd * 32 * 64);
    int t = 0, nst = 0;  // nst: bulk stores this warp issued (the staging buffer is reused after their reads)
    for (int k = 0, w = item_at(0); w < items; w = item_at(++k)) {
      int b, head, q0, nkv, len;
      decode(w, b, head, q0, nkv, len);
      const int srow = q0 + r;
      float m_ref = -INFINITY, l = 0.f;
      for (int j = 0; j < nkv; ++j, ++t) {
        const int b2 = t & 1;
        const uint32_t tS = tmem_base + (uint32_t)(b2 * BN) + lane_off;
        const int k0 = j * BN;
        mbar_wait(&s_full[b2], (t >> 1) & 1);
        __syncwarp();
        tc_fence_after();
        uint32_t sr[2][32];
        tmem_ld32_nowait(tS + 0, sr[0]);
        tmem_ld32_nowait(tS + 32, sr[1]);
        tmem_wait_ld();
        // row max with 8 independent partial maxima (a 64-long fmax chain would serialise on latency)
        float mx[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mx[e] = -INFINITY;
        const bool need_mask = (k0 + BN > len) || (causal && k0 + BN - 1 > q0 + qd * 32);
        if (need_mask) {
          const int lim = min(len, causal ? srow + 1 : len) - k0;  // keys c < lim are allowed
#pragma unroll
          for (int c = 0; c < BN; ++c) {
            float v = __uint_as_float(sr[c >> 5][c & 31]);
            if (c >= lim) v = -INFINITY;
            sr[c >> 5][c & 31] = __float_as_uint(v);
            mx[c & 7] = fmaxf(mx[c & 7], v);
          }
        } else {
#pragma unroll
          for (int c = 0; c < BN; ++c) mx[c & 7] = fmaxf(mx[c & 7], __uint_as_float(sr[c >> 5][c & 31]));
        }
        float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        mt *= scale_log2;
        // lazy rescale, warp-wide (tcgen05.ld / st are .sync.aligned), alpha = 1 for rows keeping their max.
        // o_full[b] completes once per P V on buffer b (tiles b, b + 2, ...), and a parity wait is exact only
        // while the barrier is no more than one phase ahead of or behind the waited one.  The two waits on it
        // (P_{t-1} V here, the item's last P V in the epilogue) are exact without observing every phase:
        // this warp holds S_t, which the MMA thread issued only after P_{t-2} V completed (p_free), so
        // P_{t-3} V -- the previous phase of P_{t-1} V's barrier -- is complete (one thread's tcgen05 ops
        // complete in order), and P_{t+1} V -- the next one -- needs P_{t+1} from this warp.  (Observing
        // P_{t-1} V after every hand-over cost a ~200-clock try_wait round trip per tile, trace in
        // profiles/r02_attn_v2_trace_report.txt.)
        const bool grow = mt > m_ref + 8.f;
        const float alpha = !grow ? 1.f : (m_ref == -INFINITY) ? 0.f : ex2f(m_ref - mt);
        if (j > 0 && __any_sync(0xffffffffu, grow)) {
          mbar_wait(&o_full[(t - 1) & 1], ((t - 1) >> 1) & 1);  // P_{t-1} V_{t-1}: the last writer of O
          __syncwarp();
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < D; c += 32) {
            uint32_t o[32];
            tmem_ld32(tO + lane_off + c, o);
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st32(tO + lane_off + c, o);
          }
        }
        if (grow) {
          l *= alpha;
          m_ref = mt;
        }
        const float base = (m_ref == -INFINITY) ? 0.f : m_ref;
        uint32_t pk[32];
        float ls[4] = {0.f, 0.f, 0.f, 0.f};  // independent partial row sums (latency, as for the max)
#pragma unroll
        for (int c = 0; c < BN; c += 2) {
          const float p0 = ex2f(fmaf(__uint_as_float(sr[c >> 5][c & 31]), scale_log2, -base));
          const float p1 = ex2f(fmaf(__uint_as_float(sr[(c + 1) >> 5][(c + 1) & 31]), scale_log2, -base));
          ls[(c >> 1) & 3] += p0 + p1;
          pk[c >> 1] = pack_bf16x2(p0, p1);
        }
        l += (ls[0] + ls[1]) + (ls[2] + ls[3]);
        tmem_st32(tS, pk);  // P_t over the first BN/2 columns of S_t (S_t is in registers)
        if (k0 + BN > len) {  // zero V rows of keys >= len (pad rows a5 never wrote may hold NaN)
          mbar_wait(&v_full[b2], (t >> 1) & 1);
          if (r < BN && k0 + r >= len) {
#pragma unroll
            for (int h = 0; h < DH; ++h) {
              uint4* vr = reinterpret_cast<uint4*>(sV + b2 * C::V_BYTES + h * BN * 128 + r * 128);
#pragma unroll
              for (int c = 0; c < 8; ++c) vr[c] = make_uint4(0, 0, 0, 0);
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[b2]);
        if (ATTN2_OBSERVE_ALL && j > 0) mbar_wait(&o_full[(t - 1) & 1], ((t - 1) >> 1) & 1);
      }
      // ---------------- item epilogue: O / l -> packed context row (or padded O row)
      mbar_wait(&o_full[(t - 1) & 1], ((t - 1) >> 1) & 1);
      __syncwarp();
      tc_fence_after();
      const float inv = 1.f / l;
      const bool valid = srow < len;
      const int qrow0 = q0 + qd * 32;
      // warp-uniform: all 32 rows of the warp are queries -> TMA box stores (rows past the sequence end would
      // land on the next sequence's packed rows, so partial warps keep the per-thread stores)
      const bool box = o_tma && qrow0 + 32 <= len;
      const int ox = Cp ? head * D : 0;
      const int oy = Cp ? __ldg(offsets + b) + qrow0 : (b * hk + head) * S + qrow0;
      bf16* dst = Cp ? Cp + ((int64_t)__ldg(offsets + b) + srow) * (int64_t)(hk * D) + head * D
                     : Opad + ((int64_t)(b * hk + head) * S + srow) * D;
#pragma unroll 1
      for (int c = 0; c < D; c += 64) {  // two 32-column TMEM loads in flight per step
        uint32_t o[2][32];
        tmem_ld32_nowait(tO + lane_off + c, o[0]);
        tmem_ld32_nowait(tO + lane_off + c + 32, o[1]);
        tmem_wait_ld();
        if (c + 64 >= D) {  // O has been read: the next item's first P V may overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(o_empty);
        }
        if (box) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {  // 32-column chunks
            if (nst > 0) {  // the previous store has finished reading the staging buffer
              if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              __syncwarp();
            }
            attn_stage32(o[u], inv, stg, lane);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) attn_tma_store(&tmO, stg, ox + c + 32 * u, oy);
            ++nst;
          }
        } else if (valid) {
#pragma unroll
          for (int e = 0; e < 64; e += 16) attn_st256(dst + c + e, &o[e >> 5][e & 31], inv);
        }
      }
    }
    if (nst > 0 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // before smem goes away
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(C::TMEM_COLS));
  }
}

// ============================================================================ v3: one CTA per SM, two Q tiles
// The FA4-style layout (ENERGON_ATTN=5, default).  One work item = 256 query rows of one (sequence, head):
// two 128-row Q tiles that share every K / V tile of 128 keys, so each K / V byte staged in shared memory
// feeds two S MMAs and two P.V MMAs.  TMEM holds both tiles' state at once (512 columns):
//   S0/P0 [0,128) | S1/P1 [128,256) | O0 [256, 256+D) | O1 [256+D, 256+2D)
// 12 warps: warps 0-3 softmax of Q tile 0 (warp w owns TMEM lanes 32(w&3).. = query rows), warps 4-7
// softmax of Q tile 1, warp 8 TMA producer, warp 9 MMA issuer (+ TMEM owner), warps 10-11 idle.  Each SM
// sub-partition holds 3 warps (one per warpgroup) in its 16K registers: the producer warpgroup gives
// registers up (setmaxnreg 168 -> 88) so the softmax warps can hold a whole 128-key score row (168 -> 208);
// 2 x 208 + 88 = 3 x 168, so the released registers exactly cover the increase (a larger increase than
// the pool holds blocks setmaxnreg.inc forever).  The MMA thread issues, per
// key tile j of an item:  P0_j V_j, S0_{j+1}, P1_j V_j, S1_{j+1}  -- so while softmax warpgroup 0 works on
// S0_{j+1}, the tensor pipe runs P1_j V_j and S1_{j+1}, and vice versa: each warpgroup's softmax is hidden
// behind the other tile's MMAs.  S_{j+1} overwrites P_j's TMEM columns without waiting for P_j V_j to
// complete: tcgen05.mma operations issued by one thread execute in issue order (blackwell guide, "implicit
// pipeline"), so the P_j V_j that reads them runs first.
// Softmax per row as in v2 (fp32, exp2, lazy O rescale when the row max grows by > 2^8, P as packed bf16 over
// its S columns), plus: 32-key chunks that no row of the warp may see (causal diagonal, key tail) skip
// their exponentials, and warps whose 32 query rows all lie at or past the sequence end compute nothing.
// The epilogue of a tile (O / l -> packed context rows) runs in its softmax warpgroup; the next item's
// S MMAs and TMA loads proceed meanwhile, only its first P V waits for it (o_empty).
// Diagnostics (ENERGON_ATTN_TRACE=<file>): clock64 timestamps of CTA 0's first 64 tiles per slot --
// [slot][tile][4]: softmax S seen, softmax P handed over, MMA P seen, MMA P V + next S issued.  The launch is
// then synchronous and the records are appended to the file.  Null in normal runs.
__device__ long long* g_attn_trace = nullptr;
__device__ __forceinline__ long long clk64() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}

#ifndef ATTN3_PINGPONG  // v3's asymmetric softmax ping-pong (measured slower: alternation without gain, §12)
#define ATTN3_PINGPONG 0
#endif
#ifndef ATTN3_EMU
#define ATTN3_EMU 0  // keys of every 32 whose exponential runs on the FMA pipe in unmasked tiles (v3)
#endif

template <int D>
struct Attn3Cfg {
  static constexpr int BM = 128, BN = 128, DH = D / 64;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int K_BYTES = BN * D * 2;
  static constexpr int V_BYTES = BN * D * 2;
  static constexpr int STG_BYTES = 8 * 32 * 64;  // epilogue staging: per softmax warp 32 rows x 32 columns (bf16)
  static constexpr int SMEM = 2 * Q_BYTES + 2 * K_BYTES + 2 * V_BYTES + STG_BYTES + 1024 + 256;
  static constexpr int THREADS = 384;  // 12 warps: 3 per SM sub-partition (168 registers each at launch)
  static constexpr uint32_t IDESC_S = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                      ((uint32_t)(BM >> 4) << 24);
  static constexpr uint32_t IDESC_O = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(D >> 3) << 17) |
                                      ((uint32_t)(BM >> 4) << 24);
};

// per-item geometry shared by the three roles (they must agree exactly): Q tile 0 reads key tiles
// [0, kv0), Q tile 1 (if any of its rows is valid) [0, kv1), kv1 >= kv0
struct Item3 {
  int b, head, q0, len, kv0, kv1;
  bool q1;
};

template <int D>
__global__ void __launch_bounds__(384, 1)
    attention_tc3_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ Cp, const int* __restrict__ offsets,
                         bf16* __restrict__ Opad, const int* __restrict__ lens, const uint32_t* __restrict__ work,
                         int hk, int S, int causal, float scale_log2, const __grid_constant__ CUtensorMap tmO,
                         int o_tma) {
  using C = Attn3Cfg<D>;
  constexpr int BM = C::BM, BN = C::BN, DH = C::DH;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                       // [2] Q tiles
  uint8_t* sK = sQ + 2 * C::Q_BYTES;        // [2] stages
  uint8_t* sV = sK + 2 * C::K_BYTES;        // [2] stages
  uint8_t* sStg = sV + 2 * C::V_BYTES;     // [8 softmax warps][2][32 rows][32 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStg + C::STG_BYTES);
  uint64_t* q_full = bars + 0;    // [2] per Q slot
  uint64_t* q_empty = bars + 2;   // [2]
  uint64_t* o_empty = bars + 4;   // [2] the slot's epilogue has read O (4 warps)
  uint64_t* s_full = bars + 6;    // [2] S_k of the slot's current tile computed
  uint64_t* p_full = bars + 8;    // [2] P_k written (4 warps)
  uint64_t* pv_done = bars + 10;  // [2 slots][2]: P V of the slot's tile n done, barrier n & 1
  uint64_t* k_full = bars + 14;   // [2] stages
  uint64_t* k_empty = bars + 16;
  uint64_t* v_full = bars + 18;
  uint64_t* v_empty = bars + 20;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 22);
  // softmax ping-pong: prog[q] = exponential passes finished by warp q of warpgroup 0 (SM sub-partition q)
  // (shared-memory atomics: a monotonic progress flag read by a spinning warp of another warpgroup)
  int* prog = reinterpret_cast<int*>(bars + 23);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 4) prog[threadIdx.x] = 0;
  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    if (o_tma) tma_prefetch_desc(&tmO);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&o_empty[i], 4);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&pv_done[2 * i], 1);
      mbar_init(&pv_done[2 * i + 1], 1);
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 2);  // both slots' MMA threads release every K / V tile
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_trigger();  // (after the TMEM allocation, see v2)
  pdl_wait();
  const int items = (int)__ldg(work) * hk;

  auto item_at = [&](int k) { return k * (int)gridDim.x + ((k & 1) ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x); };
  auto decode = [&](int w) {
    Item3 it;
    const uint32_t pr = __ldg(work + 1 + w / hk);
    it.head = w % hk;
    it.b = (int)(pr >> 16);
    it.q0 = (int)(pr & 0xFFFFu) * (2 * BM);
    it.len = __ldg(lens + it.b);
    const int e0 = causal ? min(it.len, it.q0 + BM) : it.len;
    const int e1 = causal ? min(it.len, it.q0 + 2 * BM) : it.len;
    it.kv0 = (e0 + BN - 1) / BN;
    it.q1 = it.q0 + BM < it.len;
    it.kv1 = it.q1 ? (e1 + BN - 1) / BN : it.kv0;
    return it;
  };

  if (warp >= 8) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
  if (warp == 8) {
    if (lane == 0) {
      // ---------------- TMA producer: K_0, K_1, V_0, K_2, V_1, ... per item; the NEXT item's Q0 is loaded
      // right after this item's V_{n-2} (Q0 is free once slot 0's last S is done, which needs nothing loaded
      // later) and its Q1 right after V_{n-1}, so a slot's next item never waits for a Q load after its epilogue.
      int t = 0, c0 = 0, c1 = 0;
      auto load_q = [&](const Item3& it, int k) {
        int& c = k ? c1 : c0;
        mbar_wait(&q_empty[k], (c & 1) ^ 1);
        mbar_expect_tx(&q_full[k], C::Q_BYTES);
        const int row = (it.b * hk + it.head) * S + it.q0 + k * BM;
#pragma unroll
        for (int h = 0; h < DH; ++h)
          tma_load_2d(&tmQ, smem_u32(sQ + k * C::Q_BYTES + h * BM * 128), &q_full[k], h * 64, row);
        ++c;
      };
      int qi = 0, w = item_at(0);
      Item3 it;
      if (w < items) {
        it = decode(w);
        load_q(it, 0);
        if (it.q1) load_q(it, 1);
      }
      while (w < items) {
        const int wn = item_at(qi + 1);
        Item3 nx;
        if (wn < items) nx = decode(wn);
        const int row_base = (it.b * hk + it.head) * S;
        const int nkv = it.kv1;
        auto load_k = [&](int tt, int j) {
          const int s2 = tt & 1;
          mbar_wait(&k_empty[s2], ((tt >> 1) & 1) ^ 1);
          mbar_expect_tx(&k_full[s2], C::K_BYTES);
#pragma unroll
          for (int h = 0; h < DH; ++h)
            tma_load_2d(&tmK, smem_u32(sK + s2 * C::K_BYTES + h * BN * 128), &k_full[s2], h * 64, row_base + j * BN);
        };
        load_k(t, 0);
        for (int j = 0; j < nkv; ++j) {
          if (j + 1 < nkv) load_k(t + j + 1, j + 1);
          const int tt = t + j, s2 = tt & 1;
          mbar_wait(&v_empty[s2], ((tt >> 1) & 1) ^ 1);
          mbar_expect_tx(&v_full[s2], C::V_BYTES);
#pragma unroll
          for (int h = 0; h < DH; ++h)
            tma_load_2d(&tmV, smem_u32(sV + s2 * C::V_BYTES + h * BN * 128), &v_full[s2], h * 64, row_base + j * BN);
          if (wn < items) {
            if (j == max(nkv - 2, 0)) load_q(nx, 0);
            if (j == nkv - 1 && nx.q1) load_q(nx, 1);
          }
        }
        t += nkv;
        ++qi;
        w = wn;
        it = nx;
      }
    }
  } else if (warp == 9 || warp == 10) {
    if (ATTN_WARP_ISSUE || lane == 0) {  // (ATTN_WARP_ISSUE: converged warp, one elected lane issues)
      // ---------------- MMA issuer of slot k (one thread per Q tile, so neither slot's chain
      // softmax -> P V -> next S waits for the other's).  Per item it issues S_0, then per key tile j:
      // P_j V_j, S_{j+1}; K / V stages are released (count 2) by both slots for every tile -- by the
      // commit of the MMAs that read it, or by a plain arrival (after the stage's full barrier, so the
      // arrival falls in the right phase) for a tile the slot does not use.
      const int k = warp - 9;
      int t = 0, c = 0, n = 0;  // K/V tile, this slot's item count, this slot's P V count
      const uint32_t tS = tmem_base + (uint32_t)(k * BN);
      const uint32_t tO = tmem_base + (uint32_t)(2 * BN + k * D);
      long long* trace = (blockIdx.x == 0 && lane == 0) ? g_attn_trace : nullptr;
      auto issue_s = [&](int tt) {  // S_k = Q_k K_tt^T
        const int s2 = tt & 1;
        if (ATTN_WARP_ISSUE) {
          __syncwarp();
          const uint64_t a0 = umma_desc_sw128(smem_u32(sQ + k * C::Q_BYTES));
          const uint64_t b0 = umma_desc_sw128(smem_u32(sK + s2 * C::K_BYTES));
          if (D == 128)
            umma_s8e(tS, a0, b0, umma_desc_sw128(smem_u32(sQ + k * C::Q_BYTES + BM * 128)),
                     umma_desc_sw128(smem_u32(sK + s2 * C::K_BYTES + BN * 128)), C::IDESC_S);
          else
            umma_s4e(tS, a0, b0, C::IDESC_S);
          umma_commit_e(&s_full[k]);
          umma_commit_e(&k_empty[s2]);
          return;
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk & 3) * 32;
          const uint64_t a = umma_desc_sw128(smem_u32(sQ + k * C::Q_BYTES + (kk >> 2) * BM * 128 + off));
          const uint64_t bb = umma_desc_sw128(smem_u32(sK + s2 * C::K_BYTES + (kk >> 2) * BN * 128 + off));
          umma_bf16(tS, a, bb, C::IDESC_S, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[k]);
        umma_commit(&k_empty[s2]);
      };
      for (int qi = 0, w = item_at(0); w < items; w = item_at(++qi)) {
        const Item3 it = decode(w);
        const int nkv = it.kv1;
        const bool act = k == 0 || it.q1;
        const int kv = act ? (k == 0 ? it.kv0 : it.kv1) : 0;
        if (kv > 0) {
          mbar_wait(&k_full[t & 1], (t >> 1) & 1);
          mbar_wait(&q_full[k], c & 1);
          tc_fence_after();
          issue_s(t);
          if (kv == 1) {
            if (ATTN_WARP_ISSUE) umma_commit_e(&q_empty[k]);
            else umma_commit(&q_empty[k]);
          }
        }
        for (int j = 0; j < nkv; ++j) {
          const int tt = t + j, s2 = tt & 1;
          if (j < kv) {
            mbar_wait(&v_full[s2], (tt >> 1) & 1);
            if (j == 0) mbar_wait(&o_empty[k], (c & 1) ^ 1);
            mbar_wait(&p_full[k], n & 1);
            if (trace && n < 64) trace[(k * 64 + n) * 8 + 2] = clk64();
            tc_fence_after();
            if (ATTN_WARP_ISSUE) {
              __syncwarp();
              umma_pv8e(tO, tS, umma_desc_sw128_mn(smem_u32(sV + s2 * C::V_BYTES), BN * 128), C::IDESC_O, j > 0 ? 1u : 0u);
              umma_commit_e(&pv_done[2 * k + (n & 1)]);
              umma_commit_e(&v_empty[s2]);
            } else {
#pragma unroll
              for (int kk = 0; kk < BN / 16; ++kk) {
                const uint64_t bb = umma_desc_sw128_mn(smem_u32(sV + s2 * C::V_BYTES + kk * 16 * 128), BN * 128);
                umma_bf16_ts(tO, tS + (uint32_t)(kk * 8), bb, C::IDESC_O, (j > 0 || kk > 0) ? 1u : 0u);
              }
              umma_commit(&pv_done[2 * k + (n & 1)]);
              umma_commit(&v_empty[s2]);
            }
            ++n;
            if (j + 1 < kv) {
              mbar_wait(&k_full[(tt + 1) & 1], ((tt + 1) >> 1) & 1);
              tc_fence_after();
              issue_s(tt + 1);
              if (j + 2 == kv) {
                if (ATTN_WARP_ISSUE) umma_commit_e(&q_empty[k]);
                else umma_commit(&q_empty[k]);
              }
            }
            if (trace && n - 1 < 64) trace[(k * 64 + n - 1) * 8 + 3] = clk64();
          } else {
            // a tile this slot does not read: release its stages in phase (its K arrival for j == kv was not
            // made by an S, since S_{kv} is never issued; j = 0 of an inactive slot likewise)
            mbar_wait(&k_full[s2], (tt >> 1) & 1);
            if (lane == 0) mbar_arrive(&k_empty[s2]);
            mbar_wait(&v_full[s2], (tt >> 1) & 1);
            if (lane == 0) mbar_arrive(&v_empty[s2]);
          }
        }
        t += nkv;
        if (act) ++c;
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
    // ---------------- softmax warpgroup k = warp / 4: thread owns query row r of Q tile k (TMEM lane r)
    const int k = warp >> 2, qd = warp & 3;
    const int r = qd * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const uint32_t tS = tmem_base + lane_off + (uint32_t)(k * BN);
    const uint32_t tO = tmem_base + lane_off + (uint32_t)(2 * BN + k * D);
    int t = 0, n = 0, c = 0;  // global K/V tile, this slot's P V count, this slot's item count
    const uint32_t stg = smem_u32(sStg + (k * 4 + qd) * 32 * 64);
    int nst = 0;  // bulk stores issued by this warp (the staging buffer is reused after their reads)
    int n0_base = 0;          // (warpgroup 1) warpgroup 0's tile count before this item
    long long* trace = (blockIdx.x == 0 && qd == 0 && lane == 0) ? g_attn_trace : nullptr;
    for (int qi = 0, w = item_at(0); w < items; w = item_at(++qi), n0_base += decode(item_at(qi - 1)).kv0) {
      const Item3 it = decode(w);
      const int nkv = it.kv1;
      if (k == 1 && !it.q1) {
        t += nkv;
        continue;
      }
      const int kv = k == 0 ? it.kv0 : it.kv1;
      const int len = it.len;
      const int qrow0 = it.q0 + k * BM + qd * 32;  // this warp's first query row
      const int srow = qrow0 + lane;
      const bool dead = qrow0 >= len;  // warp-uniform: none of the warp's rows is a query
      // keys a row may see: [0, lim_row); the warp's union: [0, lim_warp)
      const int lim_row = causal ? min(len, srow + 1) : len;
      const int lim_warp = causal ? min(len, qrow0 + 32) : len;
      float m_ref = -INFINITY, l = 0.f;
      for (int j = 0; j < kv; ++j, ++n) {
        const int tt = t + j, s2 = tt & 1;
        const int k0 = j * BN;
        mbar_wait(&s_full[k], n & 1);
        if (trace && n < 64) trace[(k * 64 + n) * 8 + 0] = clk64();
        __syncwarp();
        tc_fence_after();
        bool seen_prev = j == 0;
        if (!dead) {
          uint32_t sr[4][32];
#pragma unroll
          for (int q = 0; q < 4; ++q) tmem_ld32_nowait(tS + q * 32, sr[q]);
          tmem_wait_ld();
          if (trace && n < 64) trace[(k * 64 + n) * 8 + 4] = clk64();
          const int lim = lim_row - k0;   // this row: keys c < lim allowed
          const int wl = lim_warp - k0;   // chunks q with 32 q >= wl are empty for the whole warp
          float mx[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) mx[e] = -INFINITY;
          const bool masked = __any_sync(0xffffffffu, lim < BN);
          if (masked) {
#pragma unroll
            for (int cc = 0; cc < BN; ++cc) {
              float v = __uint_as_float(sr[cc >> 5][cc & 31]);
              if (cc >= lim) v = -INFINITY;
              sr[cc >> 5][cc & 31] = __float_as_uint(v);
              mx[cc & 7] = fmaxf(mx[cc & 7], v);
            }
          } else {
#pragma unroll
            for (int cc = 0; cc < BN; ++cc) mx[cc & 7] = fmaxf(mx[cc & 7], __uint_as_float(sr[cc >> 5][cc & 31]));
          }
          float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
          mt *= scale_log2;
          const bool grow = mt > m_ref + 8.f;
          const float alpha = !grow ? 1.f : (m_ref == -INFINITY) ? 0.f : ex2f(m_ref - mt);
          if (j > 0 && __any_sync(0xffffffffu, grow)) {
            // O_k must hold P_{j-1} V_{j-1} before it is rescaled
            mbar_wait(&pv_done[2 * k + ((n - 1) & 1)], ((n - 1) >> 1) & 1);
            seen_prev = true;
            __syncwarp();
            tc_fence_after();
#pragma unroll 1
            for (int cd = 0; cd < D; cd += 32) {
              uint32_t o[32];
              tmem_ld32(tO + cd, o);
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
              tmem_st32(tO + cd, o);
            }
          }
          if (grow) {
            l *= alpha;
            m_ref = mt;
          }
          const float base = (m_ref == -INFINITY) ? 0.f : m_ref;
          if (ATTN3_PINGPONG && k == 1) {
            // ping-pong: this warp's exponentials start only after the warpgroup-0 warp on the same SM
            // sub-partition finished those of its tile j (its last one if it has fewer), so the two share
            // the MUFU in turn and each slot's MMAs run while the other slot computes its exponentials.
            // Warpgroup 0 never waits for warpgroup 1, so this cannot deadlock.
            const int target = n0_base + min(j, it.kv0 - 1);
            // relaxed (strong) shared-memory loads: a memory-model-clean poll that does not occupy the atomics
            // unit (polling with atomicAdd(…, 0) measured 15% slower)
            for (;;) {
              int v;
              asm volatile("ld.relaxed.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(&prog[qd])) : "memory");
              if (v > target) break;
              __nanosleep(20);
            }
          }
          if (trace && n < 64) trace[(k * 64 + n) * 8 + 5] = clk64();
          float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int q = 0; q < 4; ++q) {  // 32 keys -> 16 packed bf16x2, in place -> one 16-column TMEM store
            if (32 * q < wl) {
              if (!masked && ATTN3_EMU > 0) {
                // unmasked tile: the last ATTN3_EMU keys of each 32 take 2^x on the FMA pipe, the rest on MUFU
#pragma unroll
                for (int e = 0; e < 32; e += 2) {
                  const float x0 = fmaf(__uint_as_float(sr[q][e]), scale_log2, -base);
                  const float x1 = fmaf(__uint_as_float(sr[q][e + 1]), scale_log2, -base);
                  const float p0 = e >= 32 - ATTN3_EMU ? ex2_poly(x0) : ex2f(x0);
                  const float p1 = e + 1 >= 32 - ATTN3_EMU ? ex2_poly(x1) : ex2f(x1);
                  ls[(e >> 1) & 3] += p0 + p1;
                  sr[q][e >> 1] = pack_bf16x2(p0, p1);
                }
              } else {
#pragma unroll
                for (int e = 0; e < 32; e += 2) {
                  const float p0 = ex2f(fmaf(__uint_as_float(sr[q][e]), scale_log2, -base));
                  const float p1 = ex2f(fmaf(__uint_as_float(sr[q][e + 1]), scale_log2, -base));
                  ls[(e >> 1) & 3] += p0 + p1;
                  sr[q][e >> 1] = pack_bf16x2(p0, p1);
                }
              }
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e) sr[q][e] = 0u;
            }
            tmem_st16_nowait(tS + q * 16, sr[q]);
          }
          if (trace && n < 64) trace[(k * 64 + n) * 8 + 6] = clk64();
          if (ATTN3_PINGPONG && k == 0) {
            __syncwarp();
            if (lane == 0) asm volatile("st.relaxed.cta.shared.b32 [%0], %1;" ::"r"(smem_u32(&prog[qd])), "r"(n + 1) : "memory");
          }
          tmem_wait_st();
          if (trace && n < 64) trace[(k * 64 + n) * 8 + 7] = clk64();
          l += (ls[0] + ls[1]) + (ls[2] + ls[3]);
        }
        if (ATTN3_PINGPONG && dead && k == 0 && lane == 0)
          asm volatile("st.relaxed.cta.shared.b32 [%0], %1;" ::"r"(smem_u32(&prog[qd])), "r"(n + 1) : "memory");
        if (k0 + BN > len) {  // zero V rows of keys >= len (pad rows a5 never wrote may hold NaN)
          mbar_wait(&v_full[s2], (tt >> 1) & 1);
          if (k0 + r >= len) {
#pragma unroll
            for (int h = 0; h < DH; ++h) {
              uint4* vr = reinterpret_cast<uint4*>(sV + s2 * C::V_BYTES + h * BN * 128 + r * 128);
#pragma unroll
              for (int c8 = 0; c8 < 8; ++c8) vr[c8] = make_uint4(0, 0, 0, 0);
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[k]);
        if (trace && n < 64) trace[(k * 64 + n) * 8 + 1] = clk64();
        if (!dead && !seen_prev) mbar_wait(&pv_done[2 * k + ((n - 1) & 1)], ((n - 1) >> 1) & 1);
      }
      // ---------------- epilogue of this Q tile: O / l -> packed context rows (or padded O rows), by TMA box
      // stores when all 32 rows of the warp are queries (as in v2), O released right after its last TMEM read
      bool released = false;
      if (!dead) {
        mbar_wait(&pv_done[2 * k + ((n - 1) & 1)], ((n - 1) >> 1) & 1);
        __syncwarp();
        tc_fence_after();
        const float inv = 1.f / l;
        const bool valid = srow < len;
        const bool box = o_tma && qrow0 + 32 <= len;
        const int ox = Cp ? it.head * D : 0;
        const int oy = Cp ? __ldg(offsets + it.b) + qrow0 : (it.b * hk + it.head) * S + qrow0;
        bf16* dst = Cp ? Cp + ((int64_t)__ldg(offsets + it.b) + srow) * (int64_t)(hk * D) + it.head * D
                       : Opad + ((int64_t)(it.b * hk + it.head) * S + srow) * D;
#pragma unroll 1
        for (int cd = 0; cd < D; cd += 64) {
          uint32_t o[2][32];
          tmem_ld32_nowait(tO + cd, o[0]);
          tmem_ld32_nowait(tO + cd + 32, o[1]);
          tmem_wait_ld();
          if (cd + 64 >= D) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&o_empty[k]);
            released = true;
          }
          if (box) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              if (nst > 0) {
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                __syncwarp();
              }
              attn_stage32(o[u], inv, stg, lane);
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              __syncwarp();
              if (lane == 0) attn_tma_store(&tmO, stg, ox + cd + 32 * u, oy);
              ++nst;
            }
          } else if (valid) {
#pragma unroll
            for (int e = 0; e < 64; e += 16) attn_st256(dst + cd + e, &o[e >> 5][e & 31], inv);
          }
        }
      }
      if (!released) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_empty[k]);
      }
      t += nkv;
      ++c;
    }
    if (nst > 0 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // before smem goes away
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(512));
  }
}

static bool attn_maps(AttnMaps* m, const bf16* Q, const bf16* K, const bf16* V, int rows, int D, int bm, int bn) {
  if (!m->valid || m->q != Q || m->k != K || m->v != V || m->rows != rows || m->d != D || m->bn != bn) {
    // cached per context: the maps depend only on the buffers, B * hk * S and the key-tile box
    if (!make_tmap_kmajor(&m->mq, Q, rows, D, bm) || !make_tmap_kmajor(&m->mk, K, rows, D, bn) ||
        !make_tmap_kmajor(&m->mv, V, rows, D, bn)) {
      m->valid = false;
      return false;
    }
    m->q = Q;
    m->k = K;
    m->v = V;
    m->rows = rows;
    m->d = D;
    m->bn = bn;
    m->valid = true;
  }
  return true;
}

template <int D>
static bool launch_tc(const bf16* Q, const bf16* K, const bf16* V, bf16* Cp, const int* offsets, bf16* Opad,
                      const int* lens_d, const uint32_t* work_d, int B, int hk, int S, int causal, cudaStream_t st,
                      AttnMaps* maps) {
  const int rows = B * hk * S;
  AttnMaps local;
  AttnMaps* m = maps ? maps : &local;
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  // output map of the TMA-store epilogue, cached like the input maps: packed rows [<= B S, hk d] (a7 fused) or
  // padded O [B hk S, d]; boxes are stored only for warps whose 32 rows are all queries (rows < T)
  static const int no_otma = getenv("ENERGON_NO_ATTN_TMA") ? 1 : 0;
  const void* optr = Cp ? (const void*)Cp : (const void*)Opad;
  const int o_rows = Cp ? B * S : rows, o_n = Cp ? hk * D : D;
  if (!no_otma && (!m->o_valid || m->o != optr || m->o_rows != o_rows || m->o_n != o_n)) {
    m->o_valid = make_tmap_store_box(&m->mo, optr, o_rows, o_n, 32);
    m->o = optr;
    m->o_rows = o_rows;
    m->o_n = o_n;
  }
  const int o_tma = (!no_otma && m->o_valid) ? 1 : 0;
  if (!o_tma) memset(&m->mo, 0, sizeof(m->mo));
  if (attention_impl() == 5) {
    using C = Attn3Cfg<D>;
    if (!attn_maps(m, Q, K, V, rows, D, C::BM, C::BN)) return false;
    static std::atomic<uint64_t> attr{0};
    smem_attr_once(attention_tc3_kernel<D>, C::SMEM, attr);
    // persistent grid: one CTA per SM (512 TMEM columns, ~197 KB of shared memory), no more than the
    // largest possible item count (B sequences x ceil(S / 256) query-tile pairs x hk heads)
    const int64_t max_items = (int64_t)B * ((S + 2 * C::BM - 1) / (2 * C::BM)) * hk;
    const int grid = max_items < num_sms() ? (int)max_items : num_sms();
    if (grid <= 0) return true;
    static const char* trace_file = getenv("ENERGON_ATTN_TRACE");
    static long long* trace_buf = nullptr;
    if (trace_file && !trace_buf) {
      cudaMalloc(&trace_buf, 2 * 64 * 8 * sizeof(long long));
      cudaMemcpyToSymbol(g_attn_trace, &trace_buf, sizeof(trace_buf));
    }
    if (trace_buf) cudaMemsetAsync(trace_buf, 0, 2 * 64 * 8 * sizeof(long long), st);
    launch_k(attention_tc3_kernel<D>, dim3(grid), dim3(C::THREADS), C::SMEM, st, m->mq, m->mk, m->mv, Cp, offsets,
             Opad, lens_d, work_d, hk, S, causal, scale_log2, m->mo, o_tma);
    if (trace_buf) {  // diagnostics only: synchronous dump
      long long h[2 * 64 * 8];
      cudaMemcpy(h, trace_buf, sizeof(h), cudaMemcpyDeviceToHost);
      if (FILE* f = fopen(trace_file, "a")) {
        fprintf(f, "launch B=%d hk=%d S=%d\n", B, hk, S);
        for (int i = 0; i < 2 * 64; ++i)
          if (h[i * 8])
            fprintf(f, "%d %d %lld %lld %lld %lld %lld %lld %lld %lld\n", i / 64, i % 64, h[i * 8], h[i * 8 + 1], h[i * 8 + 2],
                    h[i * 8 + 3], h[i * 8 + 4], h[i * 8 + 5], h[i * 8 + 6], h[i * 8 + 7]);
        fclose(f);
      }
    }
    return true;
  }
  using C = Attn2Cfg<D>;
  if (!attn_maps(m, Q, K, V, rows, D, C::BM, C::BN)) return false;
  static std::atomic<uint64_t> attr{0};
  smem_attr_once(attention_tc2_kernel<D>, C::SMEM, attr);
  // persistent grid: 2 CTAs per SM (shared memory and 256 TMEM columns each), no more than the largest
  // possible item count (B sequences x ceil(S / BM) query tiles x hk heads); CTAs without items exit
  const int64_t max_items = (int64_t)B * ((S + C::BM - 1) / C::BM) * hk;
  const int slots = 2 * num_sms();
  const int grid = max_items < slots ? (int)max_items : slots;
  if (grid <= 0) return true;
  launch_k(attention_tc2_kernel<D>, dim3(grid), dim3(192), C::SMEM, st, m->mq, m->mk, m->mv, Cp, offsets, Opad, lens_d,
           work_d, hk, S, causal, scale_log2, m->mo, o_tma);
  return true;
}

bool launch_attention_tc(const bf16* Q, const bf16* K, const bf16* V, bf16* ctx_packed, const int* offsets,
                         bf16* O_padded, const int* lens_d, const uint32_t* work_d, int B, int hk, int S, int d,
                         int causal, cudaStream_t st, AttnMaps* maps) {
  if (d == 128) return launch_tc<128>(Q, K, V, ctx_packed, offsets, O_padded, lens_d, work_d, B, hk, S, causal, st, maps);
  if (d == 64) return launch_tc<64>(Q, K, V, ctx_packed, offsets, O_padded, lens_d, work_d, B, hk, S, causal, st, maps);
  return false;
}

}  // namespace energon

// gemm_tc.cu -- bf16 GEMMs of the DRCE path on the 5th-generation tensor cores (sm_100a).
//
// Steps a4 (QKV, column-parallel, +bias), a8 (out-proj, row-parallel partial), a10 (MLP-up,
// column-parallel, +bias +GeLU) and a11 (MLP-down, row-parallel partial): PAPER.md:288-291
// (sec 4.1.3), run on the T packed rows only ("eliminating the redundant computation
// in all linear layers").  D[M,N] = A[M,K] . W[N,K]^T, A = activations (K-major), W = weights
// re-laid out K-major at load time; fp32 accumulation in TMEM, bf16 output.
//
// Structure (one CTA per SM, persistent, static tile schedule, 256 threads):
//   warp 0      TMA producer: 128B-swizzled A / W tiles into a STAGES-deep shared-memory ring
//   warp 1      MMA issuer: one thread issues tcgen05.mma.cta_group::1.kind::f16 (M=128, N=BN, K=16)
//               and tcgen05.commit's the smem slot back to the producer
//   warp 2      TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4..7  epilogue: tcgen05.ld 32 lanes x 32 columns -> bias / GeLU -> bf16 -> global
// Tiles are walked m-fastest so the activation panel stays L2-resident while the weights stream
// through once.  M and N tails are handled by TMA out-of-bounds zero fill + predicated stores.
#include <cudaTypedefs.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "kernels.h"
#include <cstdio>
#include <vector>
#include "tc_ptx.cuh"

namespace energon {

constexpr int TC_BM = 128, TC_BK = 64;

template <int BN> struct TcCfg {
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;
  static constexpr int B_BYTES = BN * TC_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  // instruction descriptor (kind::f16): D f32, A/B bf16, both K-major, M = 128, N = BN
  static constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                    ((uint32_t)(TC_BM >> 4) << 24);
};

// a5 fused into the QKV epilogue: packed row t, column n0 (32-aligned, inside one head since
// d % 32 == 0) of the per-rank [q | k | v] block -> &{Q,K,V}[b, head, s, j] (PAPER.md:373 kernel #1).
__device__ __forceinline__ bf16* qkv_dst(const QkvScatter& qs, int row, int n0, int N) {
  const int Hk = N / 3;
  const int which = n0 / Hk, rem = n0 - which * Hk;
  const int head = rem / qs.d, j = rem - head * qs.d;
  const int cell = qs.pack_idx ? __ldg(qs.pack_idx + row) : row;
  if (cell < 0) return nullptr;  // a bucket row past T: not scattered
  const int b = cell / qs.S, s = cell - b * qs.S;
  bf16* base = which == 0 ? qs.q : (which == 1 ? qs.k : qs.v);
  return base + (((int64_t)b * qs.hk + head) * qs.S + s) * qs.d + j;
}

// ----------------------------------------------------------------------------- the kernel
template <int BN, int EPI>
__global__ void __launch_bounds__(256, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, bf16* __restrict__ D,
                   const float* __restrict__ bias, int M, int N, int K, const QkvScatter qs) {
  using C = TcCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (M + TC_BM - 1) / TC_BM, num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int nkb = (K + TC_BK - 1) / TC_BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
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

  if (warp == 0) {
    if (lane == 0) {
      pdl_wait();  // inputs of this GEMM are written by the previous kernel
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m_blk = tile % num_m, n_blk = tile / num_m;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], C::STAGE_BYTES);
          tma_load_2d(&tmA, smem_u32(sA + stage * C::A_BYTES), &full[stage], kb * TC_BK, m_blk * TC_BM);
          tma_load_2d(&tmB, smem_u32(sB + stage * C::B_BYTES), &full[stage], kb * TC_BK, n_blk * BN);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t a0 = umma_desc_sw128(smem_u32(sA + stage * C::A_BYTES));
          const uint64_t b0 = umma_desc_sw128(smem_u32(sB + stage * C::B_BYTES));
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k)  // +32 bytes along K inside the swizzle atom
            umma_bf16(d_tmem, a0 + 2 * k, b0 + 2 * k, C::IDESC, (kb | k) != 0);
          umma_commit(&empty[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    pdl_wait();  // outputs: the previous kernel must be done with them
    const int q = warp - 4;  // TMEM lane quadrant this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m_blk = tile % num_m, n_blk = tile / num_m;
      mbar_wait(&tfull[acc], acc_phase);
      __syncwarp();  // reconverge the spin loop before the .sync.aligned tcgen05.ld
      tc_fence_after();
      const int row = m_blk * TC_BM + q * 32 + lane;
      bf16* drow = D + (int64_t)row * N;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c * 32), r);
        const int n0 = n_blk * BN + c * 32;
        if (row < M && n0 < N) {
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          if (EPI >= EPI_BIAS) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              if (n0 + j < N) {
                const float4 bb = __ldg(reinterpret_cast<const float4*>(bias + n0 + j));
                v[j] += bb.x;
                v[j + 1] += bb.y;
                v[j + 2] += bb.z;
                v[j + 3] += bb.w;
              }
            }
          }
          if (EPI == EPI_BIAS_GELU) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = gelu_fast(v[j]);
          }
          bf16* dst = drow + n0;
          if (EPI == EPI_BIAS_QKV) dst = qkv_dst(qs, row, n0, N);
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            if (n0 + j < N && dst) {
              uint4 o;
              o.x = pack_bf16x2(v[j], v[j + 1]);
              o.y = pack_bf16x2(v[j + 2], v[j + 3]);
              o.z = pack_bf16x2(v[j + 4], v[j + 5]);
              o.w = pack_bf16x2(v[j + 6], v[j + 7]);
              *reinterpret_cast<uint4*>(dst + j) = o;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(C::TMEM_COLS));
  }
}

// ----------------------------------------------------------------------------- 2-CTA (cta_group::2) kernel
// A CTA pair (cluster of 2 on one TPC) computes a 256 x 256 tile with tcgen05.mma.cta_group::2
// (M = 256, N = 256, K = 16): each CTA stages its 128 rows of A and its 128 rows (of N) of W, so the
// pair reads 64 KB of operands per 64-deep K step for 2 x 128 x 256 outputs -- twice the operand
// reuse of the 1-CTA 128 x 256 tile.  The leader CTA's MMA warp issues for both; TMA loads of both
// CTAs complete on the leader's full barrier; MMA commits multicast to both CTAs' empty / tmem-full
// barriers; both CTAs' epilogue warps arrive on the leader's tmem-empty barrier.
// Tiles are rasterised in groups of `group_m` 256-row panels so that the A panels of a group stay
// L2-resident while the group sweeps N.
template <int BN> struct Tc2Cfg {
  static constexpr int A_BYTES = 128 * TC_BK * 2;      // this CTA's 128 rows of A per stage
  static constexpr int B_BYTES = (BN / 2) * TC_BK * 2;  // this CTA's BN/2 rows of W per stage
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EPI_WARPS = 8;  // two warpgroups, each owning half of a tile's columns
  static constexpr int STG_BYTES = EPI_WARPS * 2 * 32 * 32 * 2;  // staging: per warp 2 x [32 rows x 32 cols] bf16
  // as many operand stages as fit in the 227 KB opt-in shared memory next to the staging buffers
  static constexpr int STAGES_FIT = (227 * 1024 - STG_BYTES - 1024 - 256) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int SMEM = STAGES * STAGE_BYTES + STG_BYTES + 1024 + 256;
  static constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                    ((uint32_t)(256 >> 4) << 24);
};
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;  // shared::cluster address of the same offset in CTA 0

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(const CUtensorMap* map, uint32_t dst, uint32_t bar_leader, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_leader), "r"(x), "r"(y)
      : "memory");
}
// same load with an L2 eviction-priority hint (createpolicy): weights are streamed once (evict_first),
// activations are re-read by every N tile (evict_last)
__device__ __forceinline__ void tma_load_2d_2sm_hint(const CUtensorMap* map, uint32_t dst, uint32_t bar_leader, int x,
                                                     int y, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1, {%3, %4}], [%2], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_leader), "r"(x), "r"(y), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void umma_bf16_2sm(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit_2sm_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// GEMM_WARP_ISSUE (default): the pair's MMA role runs on its whole (converged) warp and one elected lane issues a
// k-block's four MMAs and the stage commit from one asm block -- UTCHMMA on a uniform predicate, no per-MMA
// ELECT / R2UR.BROADCAST / BRA.U.ANY loop (as in the attention kernel).
#ifndef GEMM_WARP_ISSUE
#define GEMM_WARP_ISSUE 1
#endif
#ifndef GEMM_WARP_TMA  // the TMA producer likewise (k-block loads + expect_tx from one asm block)
#define GEMM_WARP_TMA 1
#endif
__device__ __forceinline__ void umma_2sm_kblock_e(uint32_t d, uint64_t a0, uint64_t b0, uint32_t idesc, uint32_t acc,
                                                  uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred p, e;\n.reg .b64 x, y;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\nsetp.eq.b32 p, 0, 0;\n"
      "add.s64 x, %1, 2;\nadd.s64 y, %2, 2;\n@e tcgen05.mma.cta_group::2.kind::f16 [%0], x, y, %3, p;\n"
      "add.s64 x, %1, 4;\nadd.s64 y, %2, 4;\n@e tcgen05.mma.cta_group::2.kind::f16 [%0], x, y, %3, p;\n"
      "add.s64 x, %1, 6;\nadd.s64 y, %2, 6;\n@e tcgen05.mma.cta_group::2.kind::f16 [%0], x, y, %3, p;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%5], %6;\n}\n" ::"r"(d),
      "l"(a0), "l"(b0), "r"(idesc), "r"(acc), "r"(smem_u32(bar)), "h"((uint16_t)3)
      : "memory");
}
// the producer's k-block (converged warp, one elected lane): the leader CTA arms the full barrier with the pair's
// bytes (leader != 0), then the A and W half-tiles of this CTA are loaded onto the leader's barrier
__device__ __forceinline__ void tma_kblock_2sm_e(const CUtensorMap* ma, const CUtensorMap* mb, uint32_t da, uint32_t db,
                                                 uint32_t full_local, uint32_t full_leader, uint32_t bytes, int leader,
                                                 int xk, int ya, int yb) {
  asm volatile(
      "{\n.reg .pred e, l;\nelect.sync _|e, 0xffffffff;\nsetp.ne.and.b32 l, %8, 0, e;\n"
      "@l mbarrier.arrive.expect_tx.shared::cta.b64 _, [%4], %6;\n"
      "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%2, {%7, %9}], [%5];\n"
      "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%1], [%3, {%7, %10}], [%5];\n}\n"
      ::"r"(da), "r"(db), "l"(reinterpret_cast<uint64_t>(ma)), "l"(reinterpret_cast<uint64_t>(mb)), "r"(full_local),
      "r"(full_leader), "r"(bytes), "r"(xk), "r"(leader), "r"(ya), "r"(yb)
      : "memory");
}
__device__ __forceinline__ void umma_commit_2sm_mc_e(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}

__device__ __forceinline__ void raster(int tile, int num_m, int num_n, int group_m, int& m_blk, int& n_blk) {
  const int per_group = group_m * num_n;
  const int g = tile / per_group;
  const int first_m = g * group_m;
  const int gsize = min(group_m, num_m - first_m);
  const int r = tile - g * per_group;
  m_blk = first_m + r % gsize;
  n_blk = r / gsize;
}

// Work decomposition of the pair kernel (data parallel + stream-K with accumulator preload).
// Tiles [0, full) are whole-K units handed out round-robin (data parallel).  When the tile count does
// not fill the clusters' last round evenly, the last R tiles (one full round plus the remainder) are
// processed stream-K: cluster c runs the contiguous iteration range [c L, (c + 1) L) of the R * nkb
// iterations (L = ceil(R nkb / clusters) >= nkb, so a tile spans at most two clusters), walking each
// tile's k-blocks in REVERSE iteration order.  A tile split between clusters c and c + 1 then has
//   an EARLY piece  -- cluster c+1's first stream-K unit, the tile's low k-blocks [0, k): its fp32
//                      accumulator goes to workspace slot c + 1 and flag (c + 1, CTA) is raised;
//   a FINISHER piece -- cluster c's last unit, the high k-blocks [k, nkb): before its first MMA the
//                      epilogue warps copy slot c + 1 into the TMEM accumulator (tcgen05.st), the MMAs
//                      accumulate on top of it, and the normal epilogue writes the tile.
// The early piece runs first in time (its cluster's first stream-K unit vs the finisher's cluster's
// last), so the finisher practically never waits, and the preload happens while the finisher's
// previous unit is still in the tensor pipe: no fix-up pass.  The accumulation order of a split tile
// (low k-blocks, then high ones, one fp32 accumulator) is that of the unsplit tile: the output is
// bit-identical to the data-parallel schedule.  Flags self-reset (the finisher clears its slot's flag).
struct TailPlan {
  int full;     // data-parallel tiles
  int L;        // stream-K iterations per cluster (0: no stream-K)
  int R;        // stream-K tiles [full, full + R)
  float* ws;    // [clusters][2][BN / 4][128][4] fp32 partial accumulators of the early pieces
  int* flags;   // [clusters][2] 1 = slot published
  int early_first;  // 1: a cluster's early piece runs before its data-parallel tiles (see WorkIter)
};
enum { UNIT_WHOLE = 0, UNIT_EARLY = 1, UNIT_FINISH = 2 };
// Diagnostics (ENERGON_GEMM_TRACE=<file>): per-unit timestamps of the pair kernel (leader CTA) -- MMA
// issuer: accumulator acquired, first stage full, last MMA issued; epilogue: accumulator full, unit
// done (stores / fix-up issued) -- in %globaltimer ns, appended to the file after every launch (the
// launch is then synchronous; scripts/gemm_trace_report.py).  Off (null pointer) in normal runs.
__device__ uint64_t* g_gemm_trace = nullptr;
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Unit order of a cluster: its data-parallel tiles, then its stream-K range (early piece, whole tiles,
// finisher).  With early_first the early piece moves to the front: published first, it gives every partner
// finisher the whole kernel to pick the partial up -- but its tile lies outside the data-parallel rounds'
// panel set, so it is used only when the operands fit in L2.
struct WorkIter {
  int u, it, it_end, early;  // early: 1 = the early piece is still to be emitted
  __device__ __forceinline__ WorkIter(int cid, const TailPlan& tp, int nkb) : u(cid), it(0), it_end(0), early(0) {
    if (tp.L > 0) {
      it = cid * tp.L;
      it_end = min(it + tp.L, tp.R * nkb);
      early = (tp.early_first && it < it_end && it % nkb != 0) ? 1 : 0;
    }
  }
  __device__ __forceinline__ void sk_unit(const TailPlan& tp, int nkb, int& tile, int& kb0, int& kb1, int& kind) {
    const int tl = it / nkb, jk = it - tl * nkb;
    const int jend = min(it_end - tl * nkb, nkb);  // exclusive, iteration index within the tile
    tile = tp.full + tl;
    kb0 = nkb - jend;  // reversed k order: iterations [jk, jend) <-> k-blocks [nkb - jend, nkb - jk)
    kb1 = nkb - jk;
    kind = (jk == 0 && jend == nkb) ? UNIT_WHOLE : (jk != 0 ? UNIT_EARLY : UNIT_FINISH);
    it += jend - jk;
  }
  // next unit of this cluster: tile, k-block range [kb0, kb1), kind (UNIT_*)
  __device__ __forceinline__ bool next(const TailPlan& tp, int nkb, int ncl, int& tile, int& kb0, int& kb1, int& kind) {
    if (early) {
      early = 0;
      sk_unit(tp, nkb, tile, kb0, kb1, kind);
      return true;
    }
    if (u < tp.full) {
      tile = u;
      kb0 = 0;
      kb1 = nkb;
      kind = UNIT_WHOLE;
      u += ncl;
      return true;
    }
    if (it >= it_end) return false;
    sk_unit(tp, nkb, tile, kb0, kb1, kind);
    return true;
  }
};

template <int EPI>
__device__ __forceinline__ void epi_math(float (&v)[32], int n0, int N, const float* __restrict__ bias) {
  if (EPI >= EPI_BIAS) {
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      if (n0 + j < N) {
        const float4 bb = __ldg(reinterpret_cast<const float4*>(bias + n0 + j));
        v[j] += bb.x;
        v[j + 1] += bb.y;
        v[j + 2] += bb.z;
        v[j + 3] += bb.w;
      }
    }
  }
  if (EPI == EPI_BIAS_GELU) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = gelu_fast(v[j]);
  }
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(x), "r"(y)
               : "memory");
}
// TMA store with an L2 eviction-priority hint (outputs streamed past the L2-resident A panels)
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, uint32_t src, int x, int y, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(x), "r"(y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// one warp's 32 rows x 32 columns -> bf16 staging buffer, 64-byte swizzle (chunk j of row r at j ^ ((r >> 1) & 3))
__device__ __forceinline__ void epi_stage(const float (&v)[32], uint8_t* stg, int lane) {
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(stg) + lane * 64;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t a = base + ((j ^ ((lane >> 1) & 3)) << 4);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(pack_bf16x2(v[8 * j], v[8 * j + 1])),
                 "r"(pack_bf16x2(v[8 * j + 2], v[8 * j + 3])), "r"(pack_bf16x2(v[8 * j + 4], v[8 * j + 5])),
                 "r"(pack_bf16x2(v[8 * j + 6], v[8 * j + 7]))
                 : "memory");
  }
}

// Stage one warp's 32 rows x 32 columns (bf16) in shared memory with the 64-byte swizzle the TMA map
// uses (16-byte chunk j of row r lives at chunk j ^ ((r >> 1) & 3): 4-way instead of 16-way bank
// conflicts) and store it with one TMA bulk-tensor store; out-of-range rows / columns are clipped.
__device__ __forceinline__ void epi_tma_store(const float (&v)[32], uint8_t* stg, int lane, const CUtensorMap* tmD,
                                              int n0, int row0) {
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(stg) + lane * 64;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t a = base + ((j ^ ((lane >> 1) & 3)) << 4);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(pack_bf16x2(v[8 * j], v[8 * j + 1])),
                 "r"(pack_bf16x2(v[8 * j + 2], v[8 * j + 3])), "r"(pack_bf16x2(v[8 * j + 4], v[8 * j + 5])),
                 "r"(pack_bf16x2(v[8 * j + 6], v[8 * j + 7]))
                 : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(tmD, (uint32_t)__cvta_generic_to_shared(stg), n0, row0);
    bulk_commit();
  }
}

template <int EPI>
__device__ __forceinline__ void epi_store(float (&v)[32], int row, int n0, int M, int N, bf16* __restrict__ D,
                                          const float* __restrict__ bias, const QkvScatter& qs) {
  if (row >= M || n0 >= N) return;
  if (EPI >= EPI_BIAS) {
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      if (n0 + j < N) {
        const float4 bb = __ldg(reinterpret_cast<const float4*>(bias + n0 + j));
        v[j] += bb.x;
        v[j + 1] += bb.y;
        v[j + 2] += bb.z;
        v[j + 3] += bb.w;
      }
    }
  }
  if (EPI == EPI_BIAS_GELU) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = gelu_fast(v[j]);
  }
  bf16* dst = (EPI == EPI_BIAS_QKV) ? qkv_dst(qs, row, n0, N) : D + (int64_t)row * N + n0;
  if (!dst) return;
#pragma unroll
  for (int j = 0; j < 32; j += 8) {
    if (n0 + j < N) {
      uint4 o;
      o.x = pack_bf16x2(v[j], v[j + 1]);
      o.y = pack_bf16x2(v[j + 2], v[j + 3]);
      o.z = pack_bf16x2(v[j + 4], v[j + 5]);
      o.w = pack_bf16x2(v[j + 6], v[j + 7]);
      *reinterpret_cast<uint4*>(dst + j) = o;
    }
  }
}

// ----------------------------------------------------------------------------- LN-prologue GEMM (N3)
// FT-style fusion ("which we can also adopt"): the QKV / MLP-up GEMM
// builds its A operand, LN(X), on the fly instead of reading the bf16 A the residual kernel would write.
// The residual kernel then writes only X (fp32) and the row statistics (mean, rstd); four producer warps
// (warps 8-11, 32 A-tile rows each) load the rows' 64 fp32 columns of each k-block, apply
// (x - mean) * rstd * g + b with exactly the residual kernel's fp32 expression (so A is bit-identical),
// round to bf16 and store into the stage in the 128B-swizzled K-major layout the TMA would have produced
// (16-byte chunk c of row r at chunk c ^ (r & 7)); loads are coalesced (two rows' 256-byte k-block slices
// per warp instruction) and the next k-block's loads are in flight while the current one is converted.  W still comes by TMA (warp 0).  1-CTA 128 x 256 tiles
// (M = 128, N = 256), warps 1 (MMA), 2 (TMEM), 4-7 (epilogue) as in gemm_tc_kernel.
struct LnA {
  const float* X;       // [M, K] fp32 residual stream
  const float2* stats;  // [M] (mean, rstd)
  const float* g;       // [K] LayerNorm weight
  const float* b;       // [K] LayerNorm bias
};

template <int EPI>
__global__ void __launch_bounds__(384, 1)
    gemm_ln_kernel(const __grid_constant__ CUtensorMap tmB, const LnA ln, bf16* __restrict__ D,
                   const float* __restrict__ bias, int M, int N, int K, const QkvScatter qs) {
  constexpr int BN = 256;
  using C = TcCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (M + TC_BM - 1) / TC_BM, num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int nkb = (K + TC_BK - 1) / TC_BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1 + 4);  // the W TMA (expect_tx) + the 4 A-producer warps
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_trigger();  // (after the TMEM allocation, see gemm_tc_kernel)

  if (warp == 0) {
    if (lane == 0) {
      pdl_wait();
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int n_blk = tile / num_m;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], C::B_BYTES);
          tma_load_2d(&tmB, smem_u32(sB + stage * C::B_BYTES), &full[stage], kb * TC_BK, n_blk * BN);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 8) {
    // ---------------- A producers: warp w builds rows [32 w, 32 w + 32) of every A stage, two rows per
    // instruction (lanes 0-15: row 2i, lanes 16-31: row 2i+1, 16 B of the row's 256 B k-block slice each), so
    // every load is a fully coalesced 2 x 256 B access; lane l owns columns [4 (l & 15), 4 (l & 15) + 4)
    pdl_wait();  // X and the statistics are written by the previous kernel
    const int w = warp - 8, hl = lane & 15, half = lane >> 4;
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m_blk = tile % num_m;
      const int rbase = m_blk * TC_BM + w * 32 + half;  // rows rbase + 2 i, i = 0..15
      float2 st[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int row = rbase + 2 * i;
        st[i] = row < M ? __ldg(ln.stats + row) : make_float2(0.f, 0.f);
      }
      auto load = [&](float4 (&x)[16], int kb) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int row = rbase + 2 * i;
          x[i] = row < M ? __ldcg(reinterpret_cast<const float4*>(ln.X + (int64_t)row * K + kb * TC_BK) + hl)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      };
      float4 xc[16], xn[16];
      load(xc, 0);
      for (int kb = 0; kb < nkb; ++kb) {
        if (kb + 1 < nkb) load(xn, kb + 1);
        const int k0 = kb * TC_BK + 4 * hl;
        const float4 gg = __ldg(reinterpret_cast<const float4*>(ln.g + k0));
        const float4 bb = __ldg(reinterpret_cast<const float4*>(ln.b + k0));
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = sA + stage * C::A_BYTES;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int r = w * 32 + 2 * i + half;  // row within the tile
          const float mean = st[i].x, rstd = st[i].y;
          const float4 x = xc[i];
          uint2 o;
          o.x = pack_bf16x2((x.x - mean) * rstd * gg.x + bb.x, (x.y - mean) * rstd * gg.y + bb.y);
          o.y = pack_bf16x2((x.z - mean) * rstd * gg.z + bb.z, (x.w - mean) * rstd * gg.w + bb.w);
          // 128B swizzle: 16-byte chunk c of row r at chunk c ^ (r & 7); this lane's 8 bytes are half (hl & 1) of chunk hl / 2
          *reinterpret_cast<uint2*>(sa + r * 128 + ((((hl >> 1) ^ (r & 7))) << 4) + ((hl & 1) << 3)) = o;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy stores -> the MMA's reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[stage]);
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) xc[i] = xn[i];
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t a0 = umma_desc_sw128(smem_u32(sA + stage * C::A_BYTES));
          const uint64_t b0 = umma_desc_sw128(smem_u32(sB + stage * C::B_BYTES));
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k) umma_bf16(d_tmem, a0 + 2 * k, b0 + 2 * k, C::IDESC, (kb | k) != 0);
          umma_commit(&empty[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    pdl_wait();
    const int q = warp - 4;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m_blk = tile % num_m, n_blk = tile / num_m;
      mbar_wait(&tfull[acc], acc_phase);
      __syncwarp();
      tc_fence_after();
      const int row = m_blk * TC_BM + q * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t rr[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c * 32), rr);
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[j]);
        epi_store<EPI>(v, row, n_blk * BN + c * 32, M, N, D, bias, qs);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(C::TMEM_COLS));
  }
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }  // the 8 epilogue warps

// The finisher's preload of one warp: chunks [c0, c0 + nch) of 32 columns of its row (fp32 partial in the
// [col/4][row][4] slot layout, `part` already offset to this thread's row) -> TMEM at `tb`.  Not inlined:
// it runs once per launch and its registers must not add to the epilogue loop's.
__device__ __noinline__ void gemm_preload_acc(const float* part, uint32_t tb, int c0, int nch) {
#pragma unroll 1
  for (int c = c0; c < c0 + nch; c += 2) {  // two chunks' loads in flight per step
    const bool two = c + 1 < c0 + nch;
    uint32_t r0[32], r1[32];
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      const float4 x = __ldcg(reinterpret_cast<const float4*>(part + (size_t)((c * 32 + j) >> 2) * 512));
      r0[j] = __float_as_uint(x.x);
      r0[j + 1] = __float_as_uint(x.y);
      r0[j + 2] = __float_as_uint(x.z);
      r0[j + 3] = __float_as_uint(x.w);
      const float4 y = two ? __ldcg(reinterpret_cast<const float4*>(part + (size_t)(((c + 1) * 32 + j) >> 2) * 512))
                           : x;
      r1[j] = __float_as_uint(y.x);
      r1[j + 1] = __float_as_uint(y.y);
      r1[j + 2] = __float_as_uint(y.z);
      r1[j + 3] = __float_as_uint(y.w);
    }
    tmem_st32_nowait(tb + (uint32_t)(c * 32), r0);
    if (two) tmem_st32_nowait(tb + (uint32_t)((c + 1) * 32), r1);
  }
  tmem_wait_st();
}

template <int BN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    bf16* __restrict__ D, const float* __restrict__ bias, int M, int N, int K, int group_m,
                    const QkvScatter qs, const TailPlan tp, const __grid_constant__ CUtensorMap tmD, int l2_hints,
                    const __grid_constant__ ShardStore shard) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  using C = Tc2Cfg<BN>;
  // QKV's a5 scatter leaves by TMA too when the host built the Q / K / V store maps (shard.qkv_tma)
  const bool TMA_ST = (EPI != EPI_BIAS_QKV) || shard.qkv_tma;
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* sStg = sB + C::STAGES * C::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sStg + C::STG_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* pre_full = tempty + 2;  // the finisher unit's accumulator holds the early piece's partial
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(pre_full + 1);
  int* pre_cnt = reinterpret_cast<int*>(tmem_holder + 1);  // epilogue warps done reading the early slot

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int num_m = (M + 255) / 256, num_n = (N + BN - 1) / BN;
  const int nkb = (K + TC_BK - 1) / TC_BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * C::EPI_WARPS);  // epilogue warps x 2 CTAs
    }
    mbar_init(pre_full, 2 * C::EPI_WARPS);
    *pre_cnt = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  __syncthreads();  // also a CTA barrier: orders the tcgen05.alloc write of tmem_holder for every checker
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  // Dependents may launch only once this CTA HOLDS its TMEM: a CTA that triggered before allocating
  // could find its columns taken by a co-resident dependent CTA that then waits (griddepcontrol.wait)
  // on this grid -- a cycle.
  pdl_trigger();

  if (warp == 0) {
    const bool warp_issue = GEMM_WARP_TMA && !(l2_hints & 1);  // (the L2-hint loads keep the one-lane path)
    if (warp_issue || lane == 0) {
      pdl_wait();  // inputs of this GEMM are written by the previous kernel
      const uint64_t pol_a = policy_evict_last(), pol_b = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      WorkIter wi(cid, tp, nkb);
      int tile, kb0, kb1, kind;
      while (wi.next(tp, nkb, ncl, tile, kb0, kb1, kind)) {
        int m_blk, n_blk;
        raster(tile, num_m, num_n, group_m, m_blk, n_blk);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t fb = smem_u32(&full[stage]) & PEER_MASK;
          if (warp_issue) {
            __syncwarp();
            tma_kblock_2sm_e(&tmA, &tmB, smem_u32(sA + stage * C::A_BYTES), smem_u32(sB + stage * C::B_BYTES),
                             smem_u32(&full[stage]), fb, 2 * C::STAGE_BYTES, leader ? 1 : 0, kb * TC_BK,
                             m_blk * 256 + (int)rank * 128, n_blk * BN + (int)rank * (BN / 2));
          } else if (leader) {
            mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
          }
          if (warp_issue) {
          } else if (l2_hints & 1) {
            tma_load_2d_2sm_hint(&tmA, smem_u32(sA + stage * C::A_BYTES), fb, kb * TC_BK, m_blk * 256 + (int)rank * 128,
                                 pol_a);
            tma_load_2d_2sm_hint(&tmB, smem_u32(sB + stage * C::B_BYTES), fb, kb * TC_BK,
                                 n_blk * BN + (int)rank * (BN / 2), pol_b);
          } else {
            tma_load_2d_2sm(&tmA, smem_u32(sA + stage * C::A_BYTES), fb, kb * TC_BK, m_blk * 256 + (int)rank * 128);
            tma_load_2d_2sm(&tmB, smem_u32(sB + stage * C::B_BYTES), fb, kb * TC_BK, n_blk * BN + (int)rank * (BN / 2));
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && (GEMM_WARP_ISSUE || lane == 0)) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      WorkIter wi(cid, tp, nkb);
      int tile, kb0, kb1, kind;
      uint64_t* trace = lane == 0 ? g_gemm_trace : nullptr;
      int nu = 0;
      while (wi.next(tp, nkb, ncl, tile, kb0, kb1, kind)) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        if (kind == UNIT_FINISH) mbar_wait(pre_full, 0);  // at most one finisher unit per cluster
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        uint64_t* rec = (trace && nu < 30) ? trace + ((size_t)cid * 32 + nu) * 6 : nullptr;
        if (rec) rec[0] = gtimer();
        const uint32_t acc0 = kind == UNIT_FINISH ? 1u : 0u;  // accumulate onto the preloaded partial
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          if (rec && kb == kb0) rec[1] = gtimer();
          tc_fence_after();
          const uint64_t a0 = umma_desc_sw128(smem_u32(sA + stage * C::A_BYTES));
          const uint64_t b0 = umma_desc_sw128(smem_u32(sB + stage * C::B_BYTES));
          if (GEMM_WARP_ISSUE) {
            __syncwarp();
            umma_2sm_kblock_e(d_tmem, a0, b0, C::IDESC, kb > kb0 ? 1u : acc0, &empty[stage]);
          } else {
#pragma unroll
            for (int k = 0; k < TC_BK / 16; ++k)
              umma_bf16_2sm(d_tmem, a0 + 2 * k, b0 + 2 * k, C::IDESC, (kb > kb0 || k > 0) ? 1u : acc0);
            umma_commit_2sm_mc(&empty[stage]);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (GEMM_WARP_ISSUE) {
          __syncwarp();
          umma_commit_2sm_mc_e(&tfull[acc]);
        } else {
          umma_commit_2sm_mc(&tfull[acc]);
        }
        if (rec) {
          rec[2] = gtimer();
          rec[3] = (uint64_t)tile | ((uint64_t)(kb1 - kb0) << 32) | ((uint64_t)kind << 48);
        }
        ++nu;
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    pdl_wait();  // outputs: the previous kernel must be done with them
    const int q = warp & 3;                 // TMEM lane quadrant this warp may access
    const int eg = (warp - 4) >> 2;         // epilogue warpgroup: 32-column chunks [c0, c0 + CH) of the tile
    const int etid = q * 32 + lane;         // this thread's TMEM lane / tile row
    constexpr int NCH = BN / 32, H0 = (NCH + 1) / 2;  // chunks per tile; warpgroup 0 takes the first H0 (BN = 224: 4 + 3)
    const int c0 = eg ? H0 : 0;
    const int CH = eg ? NCH - H0 : H0;
    const uint32_t tempty_leader = smem_u32(&tempty[0]) & PEER_MASK;
    uint8_t* my_stg = sStg + (warp - 4) * 2 * 2048;
    uint32_t nst = 0;  // TMA stores issued by this warp (double-buffered staging)
    // The finisher's preload (per warp: its TMEM lane quadrant, its warpgroup's columns): copy the early
    // piece's partial (slot cid + 1, this CTA's rows) into the accumulator buffer the finisher will use,
    // then arrive on the leader's pre_full; the last of the CTA's 8 warps clears the slot's flag.
    const int* pflag = tp.flags + (cid + 1) * 2 + rank;
    auto flag_set = [&]() -> bool {
      int v = 0;
      if (lane == 0) asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(pflag) : "memory");
      return __shfl_sync(0xffffffffu, v, 0) != 0;
    };
    auto preload = [&](int buf) {
      while (!flag_set()) __nanosleep(64);
      gemm_preload_acc(tp.ws + ((size_t)(cid + 1) * 2 + rank) * 128 * BN + (size_t)etid * 4,
                       tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * BN), c0, CH);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_cluster(smem_u32(pre_full) & PEER_MASK);
        if (atomicAdd(pre_cnt, 1) == C::EPI_WARPS - 1) *const_cast<int*>(pflag) = 0;  // self-reset for the next launch
      }
      __syncwarp();
    };
    int acc = 0;
    uint32_t acc_phase = 0;
    WorkIter wi(cid, tp, nkb);
    int tile, kb0, kb1, kind;
    // The finisher (this cluster's last unit f, if split) reuses the buffer of unit f - 2: its preload runs
    // after that unit's epilogue (at once when f == 1 and there is no early piece), so it overlaps the MMAs
    // of unit f - 1 -- but never before this cluster's own early piece (unit 0) is published, so a cluster
    // never waits for another before publishing its own piece and the waits cannot chain.
    int pre_at = -2, pre_buf = 0;  // preload into buffer pre_buf once pre_at epilogues are done (-2: none)
    int pre_first = 0;             // the target buffer is free once this many epilogues are done (f - 1)
    {
      WorkIter sc(cid, tp, nkb);
      int t2, k20, k21, kind2, n = 0, f = -1, e = -1;
      for (; sc.next(tp, nkb, ncl, t2, k20, k21, kind2); ++n) {
        if (kind2 == UNIT_EARLY) e = n;
        if (kind2 == UNIT_FINISH) f = n;
      }
      if (f >= 0) {
        pre_at = max(f - 1, e + 1);
        pre_buf = f & 1;
        pre_first = max(f - 1, 0);
      }
    }
    uint64_t* etrace = (leader && warp == 4 && lane == 0) ? g_gemm_trace : nullptr;
    int enu = 0;
    while (wi.next(tp, nkb, ncl, tile, kb0, kb1, kind)) {
      int m_blk, n_blk;
      raster(tile, num_m, num_n, group_m, m_blk, n_blk);
      if (pre_at >= 0 && enu >= pre_first && enu < pre_at) {
        // Opportunistic preload: while this unit's accumulator is still being computed, copy the partner's
        // partial in as soon as it is published (a non-blocking check, so no cluster ever waits for another
        // here and the waits cannot chain) -- the finisher's MMAs then start right after this unit's instead
        // of after this unit's epilogue plus the ~4 us preload (traced on the TP = 8 QKV shape).
        const uint32_t ta = smem_u32(&tfull[acc]);
        for (;;) {
          const int ready = __shfl_sync(0xffffffffu, mbar_try_wait(ta, acc_phase) ? 1 : 0, 0);
          if (ready) break;
          if (flag_set()) {
            preload(pre_buf);
            pre_at = -2;
            break;
          }
        }
      }
      if (enu == pre_at) preload(pre_buf);  // (pre_at == 0: f == 1 and no early piece -- a fresh buffer)
      mbar_wait(&tfull[acc], acc_phase);
      uint64_t* erec = (etrace && enu < 30) ? etrace + ((size_t)cid * 32 + enu) * 6 : nullptr;
      ++enu;
      if (erec) erec[4] = gtimer();
      __syncwarp();  // reconverge the spin loop before the .sync.aligned tcgen05.ld
      tc_fence_after();
      const int row = m_blk * 256 + (int)rank * 128 + etid;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
      if (kind == UNIT_EARLY) {
        // this CTA's 128 x BN partial accumulator -> workspace slot cid, [col/4][row][4] (coalesced)
        float* part = tp.ws + ((size_t)cid * 2 + rank) * 128 * BN + (size_t)etid * 4;
#pragma unroll 1
        for (int c = c0; c < c0 + CH; ++c) {
          uint32_t r0[32];
          tmem_ld32(tbase + (uint32_t)(c * 32), r0);
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            __stcg(reinterpret_cast<float4*>(part + (size_t)((c * 32 + j) >> 2) * 512),
                   make_float4(__uint_as_float(r0[j]), __uint_as_float(r0[j + 1]), __uint_as_float(r0[j + 2]),
                               __uint_as_float(r0[j + 3])));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader + (uint32_t)(acc * sizeof(uint64_t)));
        __threadfence();
        epi_bar();  // all 256 epilogue threads of this CTA wrote their rows
        if (warp == 4 && lane == 0)
          asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(tp.flags + cid * 2 + rank), "r"(1) : "memory");
      } else if (TMA_ST) {
        // two 32-column chunks per step: both TMEM loads in flight, one proxy fence and one wait for the
        // staging buffers per pair; the accumulator is released right after the tile's last TMEM load
#pragma unroll 1
        for (int c = c0; c < c0 + CH; c += 2) {
          const bool two = c + 1 < c0 + CH;
          uint32_t r0[32], r1[32];
          tmem_ld32_nowait(tbase + (uint32_t)(c * 32), r0);
          if (two) tmem_ld32_nowait(tbase + (uint32_t)((c + 1) * 32), r1);
          tmem_wait_ld();
          if (c + 2 >= c0 + CH) {  // last TMEM read of this tile
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader + (uint32_t)(acc * sizeof(uint64_t)));
          }
          float v0[32], v1[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            v0[j] = __uint_as_float(r0[j]);
            v1[j] = __uint_as_float(r1[j]);
          }
          epi_math<EPI>(v0, n_blk * BN + c * 32, N, bias);
          if (two) epi_math<EPI>(v1, n_blk * BN + (c + 1) * 32, N, bias);
          if (nst > 0) {  // the previous pair's stores have finished reading the staging buffers
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
          }
          int rowt = m_blk * 256 + (int)rank * 128 + q * 32;
          epi_stage(v0, my_stg, lane);
          if (two) epi_stage(v1, my_stg + 2048, lane);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (EPI == EPI_BIAS_QKV) {
            // a5 by TMA: the box's first run of rows (the sequence b its row 0 belongs to) is stored with one 3-D
            // box store per 32-column chunk into the padded plane [b * hk + head] at rows s_0 .. s_0 + 31 -- rows
            // of later sequences in the box land at s >= len_b (pad rows, never read) or past S (clipped).  A
            // sequence that starts inside the box (run start r > 0) would need a negative box row, which the TMA
            // store rejects (illegal instruction, measured), so those rows are scattered by their own lanes from
            // the registers they still hold (typically < 6% of the rows).
            const int t = rowt + lane;
            const int cell = t < M ? (qs.pack_idx ? __ldg(qs.pack_idx + t) : t) : -1;
            const int b = cell >= 0 ? cell / qs.S : -1;
            const int bprev = __shfl_up_sync(0xffffffffu, b, 1);
            const unsigned starts = __ballot_sync(0xffffffffu, cell >= 0 && (lane == 0 || bprev != b));
            const int my_run = 31 - __clz(starts & (0xffffffffu >> (31 - lane)));  // start lane of this row's run
            if (lane == 0) {
              if (starts & 1u) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  if (u == 1 && !two) break;
                  const int n0 = n_blk * BN + (c + u) * 32;
                  if (n0 >= N) break;
                  const int Hk = N / 3, which = n0 / Hk, rem = n0 - which * Hk;
                  const int head = rem / qs.d, j = rem - head * qs.d;
                  asm volatile(
                      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                          reinterpret_cast<uint64_t>(&shard.maps[which])),
                      "r"(smem_u32(my_stg + u * 2048)), "r"(j), "r"(cell - b * qs.S), "r"(b * qs.hk + head)
                      : "memory");
                }
              }
              bulk_commit();
            }
            if (cell >= 0 && my_run > 0) {  // rows of a sequence that starts inside the box: per-thread stores
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                if (u == 1 && !two) break;
                const int n0 = n_blk * BN + (c + u) * 32;
                if (n0 >= N) break;
                bf16* dst = qkv_dst(qs, t, n0, N);
                const float* vv = u ? v1 : v0;
#pragma unroll
                for (int jj = 0; jj < 32; jj += 8) {
                  uint4 o;
                  o.x = pack_bf16x2(vv[jj], vv[jj + 1]);
                  o.y = pack_bf16x2(vv[jj + 2], vv[jj + 3]);
                  o.z = pack_bf16x2(vv[jj + 4], vv[jj + 5]);
                  o.w = pack_bf16x2(vv[jj + 6], vv[jj + 7]);
                  *reinterpret_cast<uint4*>(dst + jj) = o;
                }
              }
            }
          } else if (lane == 0) {
            const CUtensorMap* dm = &tmD;
            if (shard.k > 0) {  // GEMM -> reduce-scatter: these 32 rows go straight to their owner's slot
              const int s = min(rowt / shard.rpr, shard.k - 1);
              dm = &shard.maps[s];
              rowt -= s * shard.rpr;
            }
            if (l2_hints & 2) {
              const uint64_t pol_d = policy_evict_first();
              tma_store_2d_hint(dm, smem_u32(my_stg), n_blk * BN + c * 32, rowt, pol_d);
              if (two) tma_store_2d_hint(dm, smem_u32(my_stg + 2048), n_blk * BN + (c + 1) * 32, rowt, pol_d);
            } else {
              tma_store_2d(dm, smem_u32(my_stg), n_blk * BN + c * 32, rowt);
              if (two) tma_store_2d(dm, smem_u32(my_stg + 2048), n_blk * BN + (c + 1) * 32, rowt);
            }
            bulk_commit();
          }
          ++nst;
        }
      } else {
#pragma unroll 1
        for (int c = c0; c < c0 + CH; ++c) {
          uint32_t r[32];
          tmem_ld32(tbase + (uint32_t)(c * 32), r);
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          epi_store<EPI>(v, row, n_blk * BN + c * 32, M, N, D, bias, qs);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader + (uint32_t)(acc * sizeof(uint64_t)));
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
      if (erec) erec[5] = gtimer();
    }
    if (TMA_ST && lane == 0) bulk_wait_all();  // stores complete before the CTA's smem goes away
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(512));
  }
}

// ----------------------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_tmap_kmajor(CUtensorMap* map, const void* ptr, int rows, int K, int box_rows) {
  auto enc = encode_fn();
  if (!enc || rows <= 0 || K <= 0 || (K % 8) != 0 || (reinterpret_cast<uintptr_t>(ptr) & 15)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Output map for the TMA-store epilogue: D [rows, N] bf16 row-major, 32 x 32 box, 64-byte swizzle.
bool make_tmap_store(CUtensorMap* map, const void* ptr, int rows, int N) { return make_tmap_store_box(map, ptr, rows, N, 32); }

// the same with a box of 32 rows x box_cols (32: 64-byte swizzle, 16: 32-byte swizzle)
bool make_tmap_store_box(CUtensorMap* map, const void* ptr, int rows, int N, int box_cols) {
  auto enc = encode_fn();
  if (!enc || rows <= 0 || N <= 0 || (N % 8) != 0 || (reinterpret_cast<uintptr_t>(ptr) & 15)) return false;
  if (box_cols != 32 && box_cols != 16) return false;
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)N * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_qkv_store_maps(CUtensorMap (&maps)[3], const bf16* q, const bf16* k, const bf16* v, int B, int hk, int S,
                         int d) {
  auto enc = encode_fn();
  if (!enc || B <= 0 || hk <= 0 || S <= 0 || d % 32 != 0) return false;
  const bf16* p[3] = {q, k, v};
  for (int i = 0; i < 3; ++i) {
    if (reinterpret_cast<uintptr_t>(p[i]) & 15) return false;
    cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)S, (cuuint64_t)B * hk};
    cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)S * d * 2};
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&maps[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<bf16*>(p[i]), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  return true;
}

int num_sms() {
  static std::atomic<int> per_dev[64];
  int dev = 0;
  cudaGetDevice(&dev);
  int n = per_dev[dev & 63].load(std::memory_order_relaxed);
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    per_dev[dev & 63].store(n, std::memory_order_relaxed);
  }
  return n;
}

// Tile choice.  Codes: 1256 / 1224 / 1192 / 1128 = 2-CTA pair with a 256 x {256, 224, 192, 128} tile (the W
// tensor map then has a BN/2-row box), 256 / 128 = 1-CTA 128 x {256, 128} tile.  The 256 x 256 pair tile is the
// most efficient per FLOP: per SM and 64-deep k-block it moves 32 KB through shared memory (TMA writes) for a
// 512-clock MMA, and the MMA reads the same 32 KB -- 128 B / clock, the shared-memory bandwidth.  A narrower
// tile keeps A's 16 KB for less MMA time, so it runs at ~(BN/256) / (shared-memory bytes ratio) of the
// 256-wide time per round (224: 0.875 / 0.955 = 0.916; 192: 0.75 / 0.875 -> measured 20% below its width
// share, profiles/r02_gemm_tiles_sk_tp8.log).  224 is chosen when its whole rounds beat the 256-wide rounds
// (with the stream-K tail where the launcher would use it): N = 1920 (TP = 8 QKV: 9 n-blocks, 144 tiles in
// 2 rounds of 74 pairs, instead of 2 full-width rounds for 7.5 n-blocks) and N = 5120 at short K (23
// n-blocks, 368 tiles in 5 rounds instead of 320 tiles in 5 rounds); the 1-CTA kernel covers M <= 128 or
// N < 256.  K = 0: unknown (no stream-K assumed).
static bool streamk_would_run(int tiles, int pairs, int nkb, double ab_bytes);
int tc_pick_bn(int M, int N, int K) {
  if (const char* f = getenv("ENERGON_GEMM_TILE")) {  // test hook: force a tile code
    const int code = atoi(f);
    if (code == 1256 || code == 1224 || code == 1192 || code == 1128 || code == 256 || code == 128) return code;
  }
  if (!(M > 128 && N >= 256)) return N <= 128 ? 128 : 256;
  static const int no224 = getenv("ENERGON_NO_TILE224") ? 1 : 0;
  if (no224 || K <= 0) return 1256;
  const int pairs = num_sms() / 2, num_m = (M + 255) / 256, nkb = (K + TC_BK - 1) / TC_BK;
  const int t256 = num_m * ((N + 255) / 256), t224 = num_m * ((N + 223) / 224);
  const double ab = 2.0 * ((double)M + (double)N) * (double)K;
  const double r256 = streamk_would_run(t256, pairs, nkb, ab) ? 1.03 * t256 / pairs : (double)((t256 + pairs - 1) / pairs);
  const double r224 = (double)((t224 + pairs - 1) / pairs) * (0.875 / 0.955);
  return r224 < 0.97 * r256 ? 1224 : 1256;
}

// fp32 partial-accumulator workspace + self-resetting flags of the stream-K early pieces: one slot of
// [2][128][256] fp32 and one flag pair per cluster.  Contexts own one each (runtime.cu); launches without one
// (the kernel-level ABI entry) share a per-device default.
bool tail_ws_alloc(TailWs* w) {
  const size_t units = (size_t)(num_sms() / 2);
  if (cudaMalloc(&w->ws, units * 2 * 128 * 256 * sizeof(float)) != cudaSuccess ||
      cudaMalloc(&w->counters, units * 2 * sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    tail_ws_free(w);
    return false;
  }
  cudaMemset(w->counters, 0, units * 2 * sizeof(int));
  cudaDeviceSynchronize();  // one-time: counters are zero before any stream uses them
  return true;
}

void tail_ws_free(TailWs* w) {
  if (w->ws) cudaFree(w->ws);
  if (w->counters) cudaFree(w->counters);
  w->ws = nullptr;
  w->counters = nullptr;
}

static const TailWs* default_tail_ws() {
  static TailWs per_dev[16];
  int dev = 0;
  cudaGetDevice(&dev);
  TailWs& w = per_dev[dev & 15];
  if (!w.ws) tail_ws_alloc(&w);
  return &w;
}

int tc_w_box(int code) { return code > 1000 ? (code - 1000) / 2 : code; }

// the launcher's stream-K policy (measured per shape, see launch_pair_epi), shared with the tile choice
static bool streamk_would_run(int tiles, int pairs, int nkb, double ab_bytes) {
  if (!(tiles > pairs && tiles % pairs != 0) || getenv("ENERGON_NO_STREAMK")) return false;
  return nkb >= 160 || (nkb >= 64 && tiles >= 2 * pairs && ab_bytes <= 100e6);
}

template <int BN, int EPI>
static bool launch_pair_epi(const CUtensorMap& tmA, const CUtensorMap& tmB, const float* bias, bf16* D, int M, int N,
                            int K, cudaStream_t st, const QkvScatter& qs, const CUtensorMap* tmD, const TailWs* tw,
                            const ShardStore* shard) {
  using C = Tc2Cfg<BN>;
  static std::atomic<uint64_t> attr{0};
  smem_attr_once(gemm_tc2_kernel<BN, EPI>, C::SMEM, attr);
  const int num_m = (M + 255) / 256, num_n = (N + BN - 1) / BN;
  const int tiles = num_m * num_n;
  const int pairs = num_sms() / 2;
  const int nkb = (K + TC_BK - 1) / TC_BK;
  // Stream-K (see TailPlan) when whole-tile rounds would leave clusters idle in the last round: the last
  // round plus the remainder (R tiles) are spread evenly, the rounds before stay data parallel.  Measured
  // per shape (profiles/r02_gemm_sk_ab.log, A/B against the data-parallel schedule on one box): it pays for
  //   long tiles, K >= 10240 (TP = 1 / 2 MLP-down: 608 -> 563 us, 296 -> 283 us), in data-parallel-first
  //     order (the operands exceed L2, the rounds' panel locality matters);
  //   K >= 4096 when A + W fit in L2 and there are >= 2 rounds (TP = 8 MLP-up 87 -> 79 us, TP = 4 QKV
  //     116 -> 113 us), early piece first;
  // not for short tiles: the early pieces' fp32 partials (2 x 128 KB per split tile) cross L2 at once, which
  // a K = 640 tile cannot amortise (TP = 8 out-proj 26 -> 34 us), nor for one round + remainder (TP = 8 QKV,
  // 64 -> 66 us: the clusters whose range is just an early piece and a finisher wait for their own
  // partial store + preload).  ENERGON_NO_STREAMK=1 disables it, ENERGON_SK_FORCE=1 / 2 forces it with the early piece first /
  // data-parallel first (tests).
  TailPlan tp{tiles, 0, 0, nullptr, nullptr, 0};
  int grid_cl = tiles < pairs ? tiles : pairs;
  const double ab_bytes = 2.0 * ((double)M + (double)N) * (double)K;
  int sk = 0;  // 0 none, 1 data-parallel first, 2 early piece first
  if (tiles > pairs && tiles % pairs != 0 && !getenv("ENERGON_NO_STREAMK")) {
    if (const char* f = getenv("ENERGON_SK_FORCE")) sk = atoi(f) == 2 ? 1 : 2;  // 1: early first, 2: DP first
    else if (streamk_would_run(tiles, pairs, nkb, ab_bytes)) sk = nkb >= 160 ? 1 : 2;
  }
  if (sk) {
    const TailWs* w = tw ? tw : default_tail_ws();
    if (w->ws) {
      const int full = (tiles / pairs - 1) * pairs;
      const int R = tiles - full;  // in (pairs, 2 pairs): L >= nkb, a tile spans at most two clusters
      const int L = (int)(((int64_t)R * nkb + pairs - 1) / pairs);
      tp = TailPlan{full, L, R, w->ws, w->counters, sk == 2 ? 1 : 0};
      grid_cl = pairs;
    }
  }
  const int grid = 2 * grid_cl;
  // group of A panels swept together along N: a wave of 74 concurrent tiles then spans group_m A panels
  // and ~74/group_m W panels, each K-slice read from DRAM once per wave.  96 MB of A per group (group 8
  // at K = 20480, all 16 m-blocks at K = 5120) measured ~1% faster in the step than 48 MB (group 4 at
  // K = 20480 re-read the MLP-down weights ~4x: 1.46 GB of DRAM per launch for 420 MB algorithmic).
  const double panel = 256.0 * K * 2;
  static double group_bytes = -1.0;
  if (group_bytes < 0) {  // ENERGON_GROUP_MB: experiment hook for the A-panel group budget
    const char* e = getenv("ENERGON_GROUP_MB");
    group_bytes = (e ? atof(e) : 96.0) * 1e6;
  }
  int group_m = (int)(group_bytes / panel);
  if (group_m < 1) group_m = 1;
  if (group_m > num_m) group_m = num_m;
  CUtensorMap md;
  if (tmD) {
    md = *tmD;
  } else {
    memset(&md, 0, sizeof(md));
    if (EPI != EPI_BIAS_QKV && !make_tmap_store(&md, D, M, N)) return false;
  }
  static int hints = -1;
  if (hints < 0) {
    // measured: evict_first(W) / evict_last(A) hints on the LOADS raise DRAM traffic (the 168 MB
    // MLP-down panel thrashes) and cost ~2% of the step, so bit 0 is off by default; evict_first on the
    // D STORES (bit 1) keeps more of A resident (MLP-up DRAM reads 429 -> 401 MB) and was faster in 3 of
    // 3 interleaved step pairs (85.83 vs 86.21 ms), so it is on.  ENERGON_L2_HINTS overrides.
    const char* e = getenv("ENERGON_L2_HINTS");
    hints = e ? atoi(e) : 2;
  }
  static const char* trace_file = getenv("ENERGON_GEMM_TRACE");
  static uint64_t* trace_buf = nullptr;
  const size_t trace_n = (size_t)(grid / 2) * 32 * 6;
  if (trace_file && !trace_buf) {
    cudaMalloc(&trace_buf, (size_t)(num_sms() / 2) * 32 * 6 * sizeof(uint64_t));
    cudaMemcpyToSymbol(g_gemm_trace, &trace_buf, sizeof(trace_buf));
  }
  if (trace_buf) cudaMemsetAsync(trace_buf, 0, trace_n * sizeof(uint64_t), st);
  ShardStore sh;
  if (shard && EPI == EPI_NONE) {  // (the stream-K tail is off for shard-routed GEMMs)
    sh = *shard;
  } else {
    memset(&sh, 0, sizeof(sh));  // k = 0: the output map tmD
    if (EPI == EPI_BIAS_QKV && qs.maps) {  // a5 by TMA
      for (int i = 0; i < 3; ++i) sh.maps[i] = qs.maps[i];
      sh.qkv_tma = 1;
    }
  }
  launch_k(gemm_tc2_kernel<BN, EPI>, dim3(grid), dim3(128 + 32 * C::EPI_WARPS), C::SMEM, st, tmA, tmB, D, bias, M, N, K,
           group_m, qs, tp, md, hints, sh);
  if (trace_buf) {  // diagnostics only: synchronous dump of this launch's unit timestamps
    std::vector<uint64_t> h(trace_n);
    cudaMemcpy(h.data(), trace_buf, trace_n * sizeof(uint64_t), cudaMemcpyDeviceToHost);
    if (FILE* f = fopen(trace_file, "a")) {
      fprintf(f, "launch M=%d N=%d K=%d clusters=%d\n", M, N, K, grid / 2);
      for (int c = 0; c < grid / 2; ++c)
        for (int u = 0; u < 30; ++u) {
          const uint64_t* r = &h[((size_t)c * 32 + u) * 6];
          if (r[0]) fprintf(f, "%d %d %llu %llu %llu %llu %llu %llu %llu %llu\n", c, u, (unsigned long long)(r[3] & 0xffffffffu),
                            (unsigned long long)((r[3] >> 32) & 0xffffu), (unsigned long long)r[0], (unsigned long long)r[1],
                            (unsigned long long)r[2], (unsigned long long)r[4], (unsigned long long)r[5],
                            (unsigned long long)(r[3] >> 48));
        }
      fclose(f);
    }
  }
  return true;
}

template <int BN, int EPI>
static bool launch_bn_epi(const CUtensorMap& tmA, const CUtensorMap& tmB, const float* bias, bf16* D, int M, int N,
                          int K, cudaStream_t st, const QkvScatter& qs, const CUtensorMap* /*tmD*/,
                          const TailWs* /*tw*/, const ShardStore* /*shard*/) {
  using C = TcCfg<BN>;
  static std::atomic<uint64_t> attr{0};
  smem_attr_once(gemm_tc_kernel<BN, EPI>, C::SMEM, attr);
  const int tiles = ((M + TC_BM - 1) / TC_BM) * ((N + BN - 1) / BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  launch_k(gemm_tc_kernel<BN, EPI>, dim3(grid), dim3(256), C::SMEM, st, tmA, tmB, D, bias, M, N, K, qs);
  return true;
}

#define DISPATCH_EPI(F, BNARGS)                                                  \
  switch (epi) {                                                                 \
    case EPI_NONE: return F<BNARGS EPI_NONE>(tmA, tmB, bias, D, M, N, K, st, qs, tmD, tw, shard); \
    case EPI_BIAS: return F<BNARGS EPI_BIAS>(tmA, tmB, bias, D, M, N, K, st, qs, tmD, tw, shard); \
    case EPI_BIAS_GELU: return F<BNARGS EPI_BIAS_GELU>(tmA, tmB, bias, D, M, N, K, st, qs, tmD, tw, shard); \
    default: return F<BNARGS EPI_BIAS_QKV>(tmA, tmB, bias, D, M, N, K, st, qs, tmD, tw, shard);   \
  }
#define BN256 256,
#define BN224 224,
#define BN192 192,
#define BN128 128,

bool launch_gemm_ln(const CUtensorMap& tmB, const float* X, const float2* stats, const float* g, const float* b,
                    const float* bias, bf16* D, int M, int N, int K, int epi, cudaStream_t st, const QkvScatter* qkv) {
  if (M <= 0 || N <= 0) return true;
  if (K % TC_BK != 0) return false;  // the producers build whole 64-column k-blocks
  QkvScatter qs{};
  if (qkv) qs = *qkv;
  const LnA ln{X, stats, g, b};
  using C = TcCfg<256>;
  const int tiles = ((M + TC_BM - 1) / TC_BM) * ((N + 255) / 256);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  static std::atomic<uint64_t> attr[4];  // per epilogue: the four kernels share one function-pointer type
  auto go = [&](auto kern) {
    smem_attr_once(kern, C::SMEM, attr[epi & 3]);
    launch_k(kern, dim3(grid), dim3(384), C::SMEM, st, tmB, ln, D, bias, M, N, K, qs);
  };
  if (epi == EPI_BIAS_QKV) go(gemm_ln_kernel<EPI_BIAS_QKV>);
  else if (epi == EPI_BIAS_GELU) go(gemm_ln_kernel<EPI_BIAS_GELU>);
  else if (epi == EPI_BIAS) go(gemm_ln_kernel<EPI_BIAS>);
  else go(gemm_ln_kernel<EPI_NONE>);
  return true;
}

bool launch_gemm_tc(const CUtensorMap& tmA, const CUtensorMap& tmB, int bn, const float* bias, bf16* D, int M, int N,
                    int K, int epi, cudaStream_t st, const QkvScatter* qkv, const CUtensorMap* tmD, const TailWs* tw,
                    const ShardStore* shard) {
  if (M <= 0 || N <= 0) return true;
  QkvScatter qs{};
  if (qkv) qs = *qkv;
  if (bn == 1256) {
    DISPATCH_EPI(launch_pair_epi, BN256)
  } else if (bn == 1224) {
    DISPATCH_EPI(launch_pair_epi, BN224)
  } else if (bn == 1192) {
    DISPATCH_EPI(launch_pair_epi, BN192)
  } else if (bn == 1128) {
    DISPATCH_EPI(launch_pair_epi, BN128)
  } else if (bn == 256) {
    DISPATCH_EPI(launch_bn_epi, BN256)
  } else {
    DISPATCH_EPI(launch_bn_epi, BN128)
  }
}

}  // namespace energon

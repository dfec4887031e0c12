// kernels_misc.cu -- the HBM-bound kernels of the DRCE path (steps a1-a3, a5, a7, a9/a12, a13)
// plus load-time weight relayout and the in-device TP reduction of a local group.
//
// Every kernel reads / writes each byte of its operands once, with 16-byte (or 8-byte for bf16x4)
// vector accesses along the contiguous hidden dimension; rows are independent (one CTA per row for
// the LayerNorm family so the row lives in registers between the statistics and the write).
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace energon {

static inline int grid_for(int64_t work, int threads, int max_blocks) {
  int64_t g = (work + threads - 1) / threads;
  if (g > max_blocks) g = max_blocks;
  if (g < 1) g = 1;
  return (int)g;
}

// ============================================================================ a1: index maps
// PAPER.md:368-373 (sec 4.3): every worker derives the DRCE layout from the command's seq_lens.
// offsets = exclusive prefix sum of lens (warp-shuffle scan); for each padded cell (b, s):
//   s < lens[b] : t = offsets[b] + s, unpack_idx[cell] = t, pack_idx[t] = cell, pos[t] = s
//   otherwise   : unpack_idx[cell] = -1
// and pack_idx[t] = -1 for the bucket rows t in [T, rows): the linears run on `rows` >= T packed rows
// (T rounded up to a bucket, so that one recorded CUDA graph serves every batch of that bucket); rows
// marked -1 are never scattered, gathered or unpacked.
// Every CTA recomputes the (tiny, B <= 1024) scan in shared memory, so the whole step is one launch.
// This is the only kernel of a forward that takes the lengths by value (LensParam): it publishes them
// to lens_d for every later kernel and (CTA 0) builds the attention work list there (attn_work), so a
// replayed graph needs exactly one kernel-node parameter update per batch.
// tok != nullptr: the token id of every VALID cell is range-checked here (pad cells are ignored,
// energon.h); an id outside [0, V) raises the device error flag.  Every rank of a TP group runs this
// kernel over the whole batch, so every rank raises the same flag (the embedding gathers only its own
// rows and never checks).
constexpr int ATTN_COST_BUCKETS = 256;

// Attention work list: one item per (sequence b, query tile qt) with qt * bm < len_b, ordered heaviest
// first by cost = key tiles of bn keys the query tile reads (causal: min(len, (qt + 1) bm)).
// work[0] = number of items, work[1 + i] = (b << 16) | qt.  Counting sort with shared-memory atomics:
// the order among items of equal cost is arbitrary, which cannot change any result (every item is
// computed by one CTA on its own).  One CTA, all threads.
__device__ void build_attn_work(const int* s_len, int B, int causal, int bm, int bn, uint32_t* __restrict__ work) {
  __shared__ int hist[ATTN_COST_BUCKETS];
  for (int i = threadIdx.x; i < ATTN_COST_BUCKETS; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  auto cost = [&](int b, int qt) {
    const int len = s_len[b];
    const int kv_end = causal ? min(len, (qt + 1) * bm) : len;
    return min((kv_end + bn - 1) / bn, ATTN_COST_BUCKETS - 1);
  };
  for (int b = threadIdx.x; b < B; b += blockDim.x)
    for (int qt = 0; qt * bm < s_len[b]; ++qt) atomicAdd(&hist[cost(b, qt)], 1);
  __syncthreads();
  if (threadIdx.x == 0) {  // bucket starts, heaviest bucket first (256 entries, one thread)
    int run = 0;
    for (int c = ATTN_COST_BUCKETS - 1; c >= 0; --c) {
      const int n = hist[c];
      hist[c] = run;
      run += n;
    }
    work[0] = (uint32_t)run;
  }
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += blockDim.x)
    for (int qt = 0; qt * bm < s_len[b]; ++qt) {
      const int pos = atomicAdd(&hist[cost(b, qt)], 1);
      work[1 + pos] = ((uint32_t)b << 16) | (uint32_t)qt;
    }
}

__device__ void lens_scan(const int* s_len, int B, int* s_off) {
  if (threadIdx.x < 32) {
    // each lane owns a contiguous chunk of ceil(B/32) sequences
    const int lane = threadIdx.x;
    const int per = (B + 31) / 32;
    const int b0 = lane * per, b1 = min(B, b0 + per);
    int local = 0;
    for (int b = b0; b < b1; ++b) local += s_len[b];
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int run = incl - local;  // exclusive prefix of this lane's chunk
    for (int b = b0; b < b1; ++b) {
      s_off[b] = run;
      run += s_len[b];
    }
    if (lane == 31) s_off[B] = incl;
  }
}

__global__ void __launch_bounds__(256) index_maps_kernel(LensParam lp, IndexMapsArgs a) {
  pdl_trigger();
  pdl_wait();
  __shared__ int s_off[ENERGON_MAX_B + 1];
  __shared__ int s_len[ENERGON_MAX_B];
  const int B = a.B, S = a.S;
  for (int b = threadIdx.x; b < B; b += blockDim.x) s_len[b] = lp.lens[b];
  __syncthreads();
  lens_scan(s_len, B, s_off);
  __syncthreads();
  if (blockIdx.x == 0) {
    for (int b = threadIdx.x; b <= B; b += blockDim.x) a.offsets[b] = s_off[b];
    if (a.lens_d)
      for (int b = threadIdx.x; b < B; b += blockDim.x) a.lens_d[b] = s_len[b];
    if (a.attn_work) build_attn_work(s_len, B, a.causal, a.attn_bm, a.attn_bn, a.attn_work);
  }
  const int T = s_off[B];
  for (int t = T + blockIdx.x * blockDim.x + threadIdx.x; t < a.rows; t += gridDim.x * blockDim.x) a.pack_idx[t] = -1;
  const int cells = B * S;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += gridDim.x * blockDim.x) {
    const int b = c / S, s = c - b * S;
    if (s < s_len[b]) {
      const int t = s_off[b] + s;
      a.unpack_idx[c] = t;
      a.pack_idx[t] = c;
      a.pos[t] = s;
      if (a.tok) {
        const int id = a.tok[c];
        if (id < 0 || id >= a.V) *a.err_flag = 1;
      }
    } else {
      a.unpack_idx[c] = -1;
    }
  }
}

// Lengths + attention work list only (the kernel-level attention entry, energon_attention).
__global__ void __launch_bounds__(256) attn_plan_kernel(LensParam lp, int B, int causal, int bm, int bn, int* lens_d,
                                                        uint32_t* work) {
  pdl_trigger();
  pdl_wait();
  __shared__ int s_len[ENERGON_MAX_B];
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    s_len[b] = lp.lens[b];
    lens_d[b] = lp.lens[b];
  }
  __syncthreads();
  build_attn_work(s_len, B, causal, bm, bn, work);
}

// ============================================================================ 4-wide row vectors
template <typename T> struct Row4;
template <> struct Row4<float> {
  static __device__ __forceinline__ float4 load(const float* p) { return *reinterpret_cast<const float4*>(p); }
  static __device__ __forceinline__ void store(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
};
template <> struct Row4<bf16> {
  static __device__ __forceinline__ float4 load(const bf16* p) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
  }
  static __device__ __forceinline__ void store(bf16* p, float4 v) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(p) = u;
  }
};

constexpr int LN_THREADS = 256;
// Each LayerNorm-family kernel is instantiated for NV = ceil(H / 4 / 256) float4 per thread (1..12,
// H <= 12288), so the row stays in exactly as many registers as it needs (occupancy).

// Two-pass LayerNorm statistics over a row held in registers (biased variance,
// eps inside the square root, fp32).
template <int LN_MAXV>
__device__ __forceinline__ void row_stats(const float4 (&v)[LN_MAXV], int nv, int H, float eps, float* red,
                                          float& mean, float& rstd) {
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < LN_MAXV; ++i)
    if (i < nv) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  mean = block_sum(s, red) / (float)H;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < LN_MAXV; ++i)
    if (i < nv) {
      const float a = v[i].x - mean, b = v[i].y - mean, c = v[i].z - mean, d = v[i].w - mean;
      q += (a * a + b * b) + (c * c + d * d);
    }
  const float var = block_sum(q, red) / (float)H;
  rstd = rsqrtf(var + eps);
}

__device__ __forceinline__ float4 ln_apply(float4 x, float mean, float rstd, const float* g, const float* b, int j) {
  const float4 gg = *reinterpret_cast<const float4*>(g + j), bb = *reinterpret_cast<const float4*>(b + j);
  return make_float4((x.x - mean) * rstd * gg.x + bb.x, (x.y - mean) * rstd * gg.y + bb.y,
                     (x.z - mean) * rstd * gg.z + bb.z, (x.w - mean) * rstd * gg.w + bb.w);
}

// ============================================================================ a2 + a3: embed, pack, LN1
// PAPER.md:138 embedding layer; padding is removed at the entry: only the T valid
// rows are gathered.  X[t] = E[tok[cell]] + P[pos] (fp32 residual stream), A[t] = LN1_0(X[t]).
// pack_idx == nullptr means the padded A/B mode (row t is cell t; unpack_idx[cell] < 0 marks a pad
// cell, whose id is ignored and read as 0 -- energon.h "pad positions ignored").  An id outside
// [0, V) gathers row 0 so the kernel never faults (index_maps_kernel raised the error flag).
template <typename Act, int LN_MAXV>
__global__ void __launch_bounds__(LN_THREADS) embed_ln_kernel(const int* __restrict__ tok, const int* __restrict__ pack_idx,
                                                              const int* __restrict__ unpack_idx, int row0, int S, int V,
                                                              int H, const Act* __restrict__ tok_emb,
                                                              const Act* __restrict__ pos_emb, const float* __restrict__ g,
                                                              const float* __restrict__ b, float eps, float* __restrict__ X,
                                                              Act* __restrict__ A, float2* __restrict__ stats) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[32];
  const int t = row0 + blockIdx.x;
  const int cell = pack_idx ? pack_idx[t] : t;
  if (cell < 0) {  // a bucket row past T (index_maps_kernel): zero, never read by a valid row
    for (int c = threadIdx.x; c < H / 4; c += LN_THREADS) {
      Row4<float>::store(X + (int64_t)t * H + 4 * c, make_float4(0.f, 0.f, 0.f, 0.f));
      if (A) Row4<Act>::store(A + (int64_t)t * H + 4 * c, make_float4(0.f, 0.f, 0.f, 0.f));
    }
    if (stats && threadIdx.x == 0) stats[t] = make_float2(0.f, 0.f);
    return;
  }
  const int s = cell % S;
  int id = (pack_idx || unpack_idx[cell] >= 0) ? tok[cell] : 0;
  if (id < 0 || id >= V) id = 0;
  const Act* e = tok_emb + (int64_t)id * H;
  const Act* p = pos_emb + (int64_t)s * H;
  float4 v[LN_MAXV];
  const int nv4 = H / 4;
  int nv = 0;
#pragma unroll
  for (int i = 0; i < LN_MAXV; ++i) {
    const int c = (threadIdx.x + i * LN_THREADS);
    if (c < nv4) {
      const float4 a = Row4<Act>::load(e + 4 * c), q = Row4<Act>::load(p + 4 * c);
      v[i] = make_float4(a.x + q.x, a.y + q.y, a.z + q.z, a.w + q.w);
      Row4<float>::store(X + (int64_t)t * H + 4 * c, v[i]);
      nv = i + 1;
    }
  }
  float mean, rstd;
  row_stats(v, nv, H, eps, red, mean, rstd);
  if (stats && threadIdx.x == 0) stats[t] = make_float2(mean, rstd);  // LN applied in the GEMM prologue (N3)
  if (!A) return;
#pragma unroll
  for (int i = 0; i < LN_MAXV; ++i) {
    const int c = (threadIdx.x + i * LN_THREADS);
    if (i < nv) Row4<Act>::store(A + (int64_t)t * H + 4 * c, ln_apply(v[i], mean, rstd, g, b, 4 * c));
  }
}

// Hidden-state entry (energon_forward_hidden / a later pipeline stage): X[t] = x[cell] (fp32),
// A[t] = LN1(X[t]).  pack_idx == nullptr: x is already in row order -- packed [n_valid, H] with
// n_valid = *T_dev (offsets[B]; bucket rows past it are zeroed), or every row valid (T_dev == nullptr,
// the padded A/B mode).
template <typename Act, int LN_MAXV>
__global__ void __launch_bounds__(LN_THREADS) gather_ln_kernel(const float* __restrict__ x, const int* __restrict__ pack_idx,
                                                               const int* __restrict__ T_dev, int row0, int H,
                                                               const float* __restrict__ g, const float* __restrict__ b,
                                                               float eps, float* __restrict__ X, Act* __restrict__ A,
                                                               float2* __restrict__ stats) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[32];
  const int t = row0 + blockIdx.x;
  const int cell = pack_idx ? pack_idx[t] : ((!T_dev || t < *T_dev) ? t : -1);
  if (cell < 0) {
    for (int c = threadIdx.x; c < H / 4; c += LN_THREADS) {
      Row4<float>::store(X + (int64_t)t * H + 4 * c, make_float4(0.f, 0.f, 0.f, 0.f));
      if (A) Row4<Act>::store(A + (int64_t)t * H + 4 * c, make_float4(0.f, 0.f, 0.f, 0.f));
    }
    if (stats && threadIdx.x == 0) stats[t] = make_float2(0.f, 0.f);
    return;
  }
  float4 v[LN_MAXV];
  int nv = 0;
#pragma unroll
  for (int i = 0; i < LN_MAXV; ++i) {
    const int c = (threadIdx.x + i * LN_THREADS);
    if (c < H / 4) {
      v[i] = Row4<float>::load(x + (int64_t)cell * H + 4 * c);
      Row4<float>::store(X + (int64_t)t * H + 4 * c, v[i]);
      nv = i + 1;
    }
  }
  float mean, rstd;
  row_stats(v, nv, H, eps, red, mean, rstd);
  if (stats && threadIdx.x == 0) stats[t] = make_float2(mean, rstd);
  if (!A) return;
#pragma unroll
  for (int i = 0; i < LN_MAXV; ++i)
    if (i < nv) Row4<Act>::store(A + (int64_t)t * H + 4 * (threadIdx.x + i * LN_THREADS),
                                 ln_apply(v[i], mean, rstd, g, b, 4 * (threadIdx.x + i * LN_THREADS)));
}

// ============================================================================ a9 / a12: bias + residual + LN
// X[t] += P[t] + bias (P = the reduced row-parallel partial, "accumulated by communications",
// PAPER.md:290; bias added once after the reduce), then A[t] = LN(X[t]).
// With A == nullptr only the residual update is done.
template <typename Act, int LN_MAXV, int TPR>
__global__ void __launch_bounds__(TPR) residual_ln_kernel(float* __restrict__ X, const Act* __restrict__ P,
                                                          const float* __restrict__ bias, int H,
                                                          const float* __restrict__ g, const float* __restrict__ b,
                                                          float eps, Act* __restrict__ A, float2* __restrict__ stats) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[32];
  const int t = blockIdx.x;
  float4 v[LN_MAXV];
  int nv = 0;
  float* xrow = X + (int64_t)t * H;
  const Act* prow = P + (int64_t)t * H;
  // issue every load of the row before any arithmetic (memory-level parallelism)
  float4 pv[LN_MAXV];
#pragma unroll
  for (int i = 0; i < LN_MAXV; ++i) {
    const int c = (threadIdx.x + i * TPR);
    if (c < H / 4) {
      v[i] = __ldcs(reinterpret_cast<const float4*>(xrow) + c);
      pv[i] = Row4<Act>::load(prow + 4 * c);
      nv = i + 1;
    }
  }
#pragma unroll
  for (int i = 0; i < LN_MAXV; ++i) {
    if (i < nv) {
      const int c = (threadIdx.x + i * TPR);
      const float4 q = *reinterpret_cast<const float4*>(bias + 4 * c);
      v[i].x += pv[i].x + q.x;
      v[i].y += pv[i].y + q.y;
      v[i].z += pv[i].z + q.z;
      v[i].w += pv[i].w + q.w;
      Row4<float>::store(xrow + 4 * c, v[i]);
    }
  }
  if (A == nullptr && stats == nullptr) return;
  float mean, rstd;
  row_stats(v, nv, H, eps, red, mean, rstd);
  if (stats && threadIdx.x == 0) stats[t] = make_float2(mean, rstd);  // LN applied in the GEMM prologue (N3)
  if (A == nullptr) return;
#pragma unroll
  for (int i = 0; i < LN_MAXV; ++i)
    if (i < nv) Row4<Act>::store(A + (int64_t)t * H + 4 * (threadIdx.x + i * TPR),
                                 ln_apply(v[i], mean, rstd, g, b, 4 * (threadIdx.x + i * TPR)));
}

// ============================================================================ a13: final LN + unpack
// out[cell] = LN_f(X[unpack_idx[cell]]) for valid cells, exactly 0 for pad cells;
// every output row is written once.  rows_are_cells: padded A/B mode (X row = cell).
template <typename Out, int LN_MAXV>
__global__ void __launch_bounds__(LN_THREADS) final_ln_unpack_kernel(const float* __restrict__ X, const int* __restrict__ unpack_idx,
                                                                     int rows_are_cells, int H, const float* __restrict__ g,
                                                                     const float* __restrict__ b, float eps, int apply_ln,
                                                                     Out* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[32];
  const int cell = blockIdx.x;
  const int t = unpack_idx[cell];
  Out* o = out + (int64_t)cell * H;
  if (t < 0) {
    for (int c = threadIdx.x; c < H / 4; c += LN_THREADS) Row4<Out>::store(o + 4 * c, make_float4(0.f, 0.f, 0.f, 0.f));
    return;
  }
  const int row = rows_are_cells ? cell : t;
  float4 v[LN_MAXV];
  int nv = 0;
#pragma unroll
  for (int i = 0; i < LN_MAXV; ++i) {
    const int c = (threadIdx.x + i * LN_THREADS);
    if (c < H / 4) {
      v[i] = Row4<float>::load(X + (int64_t)row * H + 4 * c);
      nv = i + 1;
    }
  }
  if (!apply_ln) {
#pragma unroll
    for (int i = 0; i < LN_MAXV; ++i)
      if (i < nv) Row4<Out>::store(o + 4 * (threadIdx.x + i * LN_THREADS), v[i]);
    return;
  }
  float mean, rstd;
  row_stats(v, nv, H, eps, red, mean, rstd);
#pragma unroll
  for (int i = 0; i < LN_MAXV; ++i)
    if (i < nv) Row4<Out>::store(o + 4 * (threadIdx.x + i * LN_THREADS),
                                 ln_apply(v[i], mean, rstd, g, b, 4 * (threadIdx.x + i * LN_THREADS)));
}

// ============================================================================ a5: rebuild padding
// Paper kernel #1 ("fuse the transpose and pad operations"): packed QKV [T, 3*Hk]
// (per-rank column order q | k | v, head-major then d) -> Q, K, V [B, hk, S, d].
// One thread moves one 16-byte chunk; reads are fully coalesced along the packed row, writes are
// contiguous d-length segments.  Pad rows of Q/K/V are never written (attention never reads them).
template <typename Act>
__global__ void unpack_qkv_kernel(const Act* __restrict__ QKV, const int* __restrict__ pack_idx, int T, int S, int hk,
                                  int d, Act* __restrict__ Q, Act* __restrict__ K, Act* __restrict__ Vv) {
  pdl_trigger();
  pdl_wait();
  constexpr int E = 16 / sizeof(Act);
  const int Hk = hk * d;
  const int chunks_per_row = 3 * Hk / E;
  const int64_t total = (int64_t)T * chunks_per_row;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / chunks_per_row);
    const int col = (int)(i - (int64_t)t * chunks_per_row) * E;
    const int which = col / Hk;
    const int rem = col - which * Hk;
    const int head = rem / d, j = rem - head * d;
    const int cell = pack_idx ? pack_idx[t] : t;
    if (cell < 0) continue;  // bucket row past T
    const int b = cell / S, s = cell - b * S;
    Act* dst = (which == 0 ? Q : (which == 1 ? K : Vv)) + (((int64_t)b * hk + head) * S + s) * d + j;
    *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(QKV + (int64_t)t * 3 * Hk + col);
  }
}

// ============================================================================ a7: remove padding
// Paper kernel #2: O [B, hk, S, d] -> packed Ctx [T, Hk] (head-major columns).
// In the padded A/B mode (pack_idx == nullptr) pad query rows are written as 0.
template <typename Act>
__global__ void repack_kernel(const Act* __restrict__ O, const int* __restrict__ pack_idx,
                              const int* __restrict__ unpack_idx, int T, int S, int hk, int d, Act* __restrict__ C) {
  pdl_trigger();
  pdl_wait();
  constexpr int E = 16 / sizeof(Act);
  const int Hk = hk * d;
  const int chunks_per_row = Hk / E;
  const int64_t total = (int64_t)T * chunks_per_row;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / chunks_per_row);
    const int col = (int)(i - (int64_t)t * chunks_per_row) * E;
    const int head = col / d, j = col - head * d;
    const int cell = pack_idx ? pack_idx[t] : t;
    const int b = cell / S, s = cell - b * S;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (pack_idx ? cell >= 0 : unpack_idx[cell] >= 0)
      v = *reinterpret_cast<const uint4*>(O + (((int64_t)b * hk + head) * S + s) * d + j);
    *reinterpret_cast<uint4*>(C + (int64_t)t * Hk + col) = v;
  }
}

// ============================================================================ local TP reduction
// In-device allreduce for a local group (energon_init_local_group): sum the k partials in rank
// order 0..k-1 in fp32 (every rank gets bit-identical data), write back to all k.
// ring != 0 (ENERGON_OPT_RING_NUMERICS, tests): reproduce the numerics of NCCL's ring algorithm on a
// bf16 payload instead -- the element of chunk s starts at rank s+1 and travels s+1 -> s+2 -> ... -> s,
// every hop adding its own partial in fp32 and storing the running sum in the payload type (one
// rounding per hop, SURVEY.md 8(c) "bf16 per hop").
template <typename Act>
__device__ __forceinline__ void reduce_parts(const PtrList& parts, int k, int64_t off, int owner, int ring,
                                             float (&acc)[16 / sizeof(Act)]) {
  constexpr int E = 16 / sizeof(Act);
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.f;
  for (int j = 0; j < k; ++j) {
    const int r = ring ? (owner + 1 + j) % k : j;
    Vec16<Act> v;
    v.u = reinterpret_cast<const uint4*>(parts.p[r])[off];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      acc[e] += to_f32(v.e[e]);
      if (ring) acc[e] = to_f32(from_f32<Act>(acc[e]));
    }
  }
}

template <typename Act>
__global__ void local_allreduce_kernel(PtrList parts, int k, int64_t n, int ring) {
  pdl_trigger();
  pdl_wait();
  constexpr int E = 16 / sizeof(Act);
  const int64_t nv = n / E;
  const int64_t chunk = (nv + k - 1) / k;  // ring chunks: chunk s is owned by rank s
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    float acc[E];
    reduce_parts<Act>(parts, k, i, (int)(i / chunk), ring, acc);
    Vec16<Act> o;
#pragma unroll
    for (int e = 0; e < E; ++e) o.e[e] = from_f32<Act>(acc[e]);
    for (int r = 0; r < k; ++r) reinterpret_cast<uint4*>(parts.p[r])[i] = o.u;
  }
}

// Local-group reduce-scatter (sequence-parallel schedule): shard s (= rank s) of every partial,
// `shard` elements starting at s * shard, is summed over the k ranks in rank order (fp32) and
// written to rank s's buffer only -- the semantics of ncclReduceScatter in place (ring: see above).
template <typename Act>
__global__ void local_reduce_scatter_kernel(PtrList parts, int k, int64_t shard, int ring) {
  pdl_trigger();
  pdl_wait();
  constexpr int E = 16 / sizeof(Act);
  const int64_t nv = shard / E;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv * k; i += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(i / nv);
    const int64_t off = (int64_t)s * nv + (i - (int64_t)s * nv);
    float acc[E];
    reduce_parts<Act>(parts, k, off, s, ring, acc);
    Vec16<Act> o;
#pragma unroll
    for (int e = 0; e < E; ++e) o.e[e] = from_f32<Act>(acc[e]);
    reinterpret_cast<uint4*>(parts.p[s])[off] = o.u;
  }
}

// Local-group all-gather: rank s's shard (shard_bytes at s * shard_bytes) is copied into every
// other rank's buffer -- the semantics of ncclAllGather in place.
__global__ void local_all_gather_kernel(PtrList parts, int k, int64_t shard_bytes) {
  pdl_trigger();
  pdl_wait();
  const int64_t nv = shard_bytes / 16;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv * k; i += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(i / nv);
    const int64_t off = (int64_t)s * nv + (i - (int64_t)s * nv);
    const uint4 v = reinterpret_cast<const uint4*>(parts.p[s])[off];
    for (int r = 0; r < k; ++r)
      if (r != s) reinterpret_cast<uint4*>(parts.p[r])[off] = v;
  }
}

template <typename Act>
void launch_local_reduce_scatter(const PtrList& parts, int k, int64_t shard, int ring, cudaStream_t st) {
  const int64_t work = shard / (16 / sizeof(Act)) * k;
  if (work > 0)
    launch_k(local_reduce_scatter_kernel<Act>, dim3(grid_for(work, 256, 148 * 8)), dim3(256), 0, st, parts, k, shard, ring);
}

void launch_local_all_gather(const PtrList& parts, int k, int64_t shard_bytes, cudaStream_t st) {
  const int64_t work = shard_bytes / 16 * k;
  if (work > 0) launch_k(local_all_gather_kernel, dim3(grid_for(work, 256, 148 * 8)), dim3(256), 0, st, parts, k, shard_bytes);
}

// ============================================================================ load-time relayout
// dst[n * K + k] = cvt(src[(row0 + k) * ld + col0 + n])  for n < N, k < K   (transpose == 1)
// dst[n]         = cvt(src[col0 + n])                     for n < N         (vector)
// Source [in, out] row-major -> destination [out, in] = K-major operand of the GEMMs.
template <typename Dst> __device__ __forceinline__ Dst cvt(double x);
template <> __device__ __forceinline__ float cvt<float>(double x) { return (float)x; }
template <> __device__ __forceinline__ bf16 cvt<bf16>(double x) { return __double2bfloat16(x); }
template <typename Dst> __device__ __forceinline__ Dst cvt(float x) { return from_f32<Dst>(x); }
template <typename Dst> __device__ __forceinline__ Dst cvt(bf16 x);
template <> __device__ __forceinline__ float cvt<float>(bf16 x) { return __bfloat162float(x); }
template <> __device__ __forceinline__ bf16 cvt<bf16>(bf16 x) { return x; }

template <typename Src, typename Dst>
__global__ void relayout_kernel(const Src* __restrict__ src, int64_t ld, int64_t row0, int64_t col0, int N, int K,
                                Dst* __restrict__ dst, int64_t dst_ld, int64_t dst_row0) {
  pdl_trigger();
  pdl_wait();
  __shared__ Src tile[32][33];
  const int n0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int k = k0 + i, n = n0 + threadIdx.x;
    if (k < K && n < N) tile[i][threadIdx.x] = src[(row0 + k) * ld + col0 + n];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int n = n0 + i, k = k0 + threadIdx.x;
    if (k < K && n < N) dst[(dst_row0 + n) * dst_ld + k] = cvt<Dst>(tile[threadIdx.x][i]);
  }
}

template <typename Src, typename Dst>
__global__ void convert_vec_kernel(const Src* __restrict__ src, int64_t off, int N, Dst* __restrict__ dst) {
  pdl_trigger();
  pdl_wait();
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) dst[n] = cvt<Dst>(src[off + n]);
}

// ============================================================================ host launchers

void launch_index_maps(const LensParam& lp, const IndexMapsArgs& a, cudaStream_t st) {
  const int cells = a.B * a.S > a.rows ? a.B * a.S : a.rows;
  launch_k(index_maps_kernel, dim3(grid_for(cells, 256, 148 * 4)), dim3(256), 0, st, lp, a);
}

const void* index_maps_kernel_fn() { return reinterpret_cast<const void*>(&index_maps_kernel); }

void launch_attn_plan(const LensParam& lp, int B, int causal, int bm, int bn, int* lens_d, uint32_t* work,
                      cudaStream_t st) {
  launch_k(attn_plan_kernel, dim3(1), dim3(256), 0, st, lp, B, causal, bm, bn, lens_d, work);
}

#define NV_DISPATCH(H, KERNEL_CALL)                                         \
  switch ((((H) / 4) + LN_THREADS - 1) / LN_THREADS) {                      \
    case 1: { constexpr int NVX = 1; KERNEL_CALL; } break;                  \
    case 2: { constexpr int NVX = 2; KERNEL_CALL; } break;                  \
    case 3: { constexpr int NVX = 3; KERNEL_CALL; } break;                  \
    case 4: { constexpr int NVX = 4; KERNEL_CALL; } break;                  \
    case 5: { constexpr int NVX = 5; KERNEL_CALL; } break;                  \
    case 6: { constexpr int NVX = 6; KERNEL_CALL; } break;                  \
    case 7: { constexpr int NVX = 7; KERNEL_CALL; } break;                  \
    case 8: { constexpr int NVX = 8; KERNEL_CALL; } break;                  \
    case 9: { constexpr int NVX = 9; KERNEL_CALL; } break;                  \
    case 10: { constexpr int NVX = 10; KERNEL_CALL; } break;                \
    case 11: { constexpr int NVX = 11; KERNEL_CALL; } break;                \
    default: { constexpr int NVX = 12; KERNEL_CALL; } break;                \
  }

template <typename Act>
void launch_embed_ln(const int* tok, const int* pack_idx, const int* unpack_idx, int row0, int rows, int S, int V, int H,
                     const Act* tok_emb, const Act* pos_emb, const float* g, const float* b, float eps, float* X, Act* A,
                     cudaStream_t st, float2* stats) {
  if (rows > 0)
    NV_DISPATCH(H, (launch_k(embed_ln_kernel<Act, NVX>, dim3(rows), dim3(LN_THREADS), 0, st, tok, pack_idx, unpack_idx,
                             row0, S, V, H, tok_emb, pos_emb, g, b, eps, X, A, stats)))
}

template <typename Act>
void launch_gather_ln(const float* x, const int* pack_idx, const int* T_dev, int row0, int rows, int H, const float* g,
                      const float* b, float eps, float* X, Act* A, cudaStream_t st, float2* stats) {
  if (rows > 0)
    NV_DISPATCH(H, (launch_k(gather_ln_kernel<Act, NVX>, dim3(rows), dim3(LN_THREADS), 0, st, x, pack_idx, T_dev, row0, H,
                             g, b, eps, X, A, stats)))
}

#define NV_DISPATCH_T(H, TPRV, KERNEL_CALL)                                 \
  switch ((((H) / 4) + (TPRV) - 1) / (TPRV)) {                              \
    case 1: { constexpr int NVX = 1; KERNEL_CALL; } break;                  \
    case 2: { constexpr int NVX = 2; KERNEL_CALL; } break;                  \
    case 3: { constexpr int NVX = 3; KERNEL_CALL; } break;                  \
    case 4: { constexpr int NVX = 4; KERNEL_CALL; } break;                  \
    case 5: { constexpr int NVX = 5; KERNEL_CALL; } break;                  \
    case 6: { constexpr int NVX = 6; KERNEL_CALL; } break;                  \
    case 7: { constexpr int NVX = 7; KERNEL_CALL; } break;                  \
    case 8: { constexpr int NVX = 8; KERNEL_CALL; } break;                  \
    case 9: { constexpr int NVX = 9; KERNEL_CALL; } break;                  \
    case 10: { constexpr int NVX = 10; KERNEL_CALL; } break;                \
    case 11: { constexpr int NVX = 11; KERNEL_CALL; } break;                \
    default: { constexpr int NVX = 12; KERNEL_CALL; } break;                \
  }

// Threads per row for the residual + LN kernel: 512 for H >= 4096, else 256; ENERGON_LN_TPR=128|256|512
// overrides (128 only when the row fits in 12 float4 per thread).
static int ln_tpr(int H, int rows) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ENERGON_LN_TPR");
    v = e ? atoi(e) : 0;  // 0: by hidden size and row count
    if (v != 0 && v != 128 && v != 256 && v != 512 && v != 640) v = 0;
  }
  // measured (H = 5120): 512 threads per row is ~4% faster for the 4096 rows of TP = 1 (40.3 vs 42.0 us),
  // 256 is 21% faster for the 512 rows a rank normalises at TP = 8 (8.6 vs 10.9 us): few rows want
  // more, smaller CTAs per SM
  // and 640 threads (exactly H / 2560 float4 each, no idle third slot at H = 5120) beat 512 by 7.6% per
  // launch at TP = 1 (ncu: 43.0 vs 46.5 us)
  if (v == 0) return (H >= 4096 && rows > 8 * 148) ? ((H / 4) % 640 == 0 ? 640 : 512) : 256;
  if (v == 128 && H / 4 > 128 * 12) return 256;
  if (v == 640 && (H / 4) % 640 != 0) return 512;  // 640: exactly H / 2560 float4 per thread (no idle slot)
  return v;
}

template <typename Act>
void launch_residual_ln(float* X, const Act* P, const float* bias, int rows, int H, const float* g, const float* b,
                        float eps, Act* A, cudaStream_t st, float2* stats) {
  if (rows <= 0) return;
  const int tpr = ln_tpr(H, rows);
  if (tpr == 128)
    NV_DISPATCH_T(H, 128, (launch_k(residual_ln_kernel<Act, NVX, 128>, dim3(rows), dim3(128), 0, st, X, P, bias, H, g, b, eps, A, stats)))
  else if (tpr == 512)
    NV_DISPATCH_T(H, 512, (launch_k(residual_ln_kernel<Act, NVX, 512>, dim3(rows), dim3(512), 0, st, X, P, bias, H, g, b, eps, A, stats)))
  else if (tpr == 640)
    NV_DISPATCH_T(H, 640, (launch_k(residual_ln_kernel<Act, NVX, 640>, dim3(rows), dim3(640), 0, st, X, P, bias, H, g, b, eps, A, stats)))
  else
    NV_DISPATCH_T(H, 256, (launch_k(residual_ln_kernel<Act, NVX, 256>, dim3(rows), dim3(256), 0, st, X, P, bias, H, g, b, eps, A, stats)))
}

template <typename Out>
void launch_final_ln_unpack(const float* X, const int* unpack_idx, int rows_are_cells, int cells, int H, const float* g,
                            const float* b, float eps, int apply_ln, Out* out, cudaStream_t st) {
  if (cells > 0)
    NV_DISPATCH(H, (launch_k(final_ln_unpack_kernel<Out, NVX>, dim3(cells), dim3(LN_THREADS), 0, st, X, unpack_idx,
                             rows_are_cells, H, g, b, eps, apply_ln, out)))
}

template <typename Act>
void launch_unpack_qkv(const Act* QKV, const int* pack_idx, int T, int S, int hk, int d, Act* Q, Act* K, Act* V,
                       cudaStream_t st) {
  const int64_t work = (int64_t)T * 3 * hk * d / (16 / sizeof(Act));
  if (work > 0) launch_k(unpack_qkv_kernel<Act>, dim3(grid_for(work, 256, 148 * 16)), dim3(256), 0, st, QKV, pack_idx, T, S, hk, d, Q, K, V);
}

template <typename Act>
void launch_repack(const Act* O, const int* pack_idx, const int* unpack_idx, int T, int S, int hk, int d, Act* C,
                   cudaStream_t st) {
  const int64_t work = (int64_t)T * hk * d / (16 / sizeof(Act));
  if (work > 0) launch_k(repack_kernel<Act>, dim3(grid_for(work, 256, 148 * 16)), dim3(256), 0, st, O, pack_idx, unpack_idx, T, S, hk, d, C);
}

template <typename Act>
void launch_local_allreduce(const PtrList& parts, int k, int64_t n, int ring, cudaStream_t st) {
  const int64_t work = n / (16 / sizeof(Act));
  if (work > 0)
    launch_k(local_allreduce_kernel<Act>, dim3(grid_for(work, 256, 148 * 8)), dim3(256), 0, st, parts, k, n, ring);
}

template <typename Src, typename Dst>
void launch_relayout(const Src* src, int64_t ld, int64_t row0, int64_t col0, int N, int K, Dst* dst, int64_t dst_ld,
                     int64_t dst_row0, cudaStream_t st) {
  dim3 grid((N + 31) / 32, (K + 31) / 32), block(32, 8);
  launch_k(relayout_kernel<Src, Dst>, dim3(grid), dim3(block), 0, st, src, ld, row0, col0, N, K, dst, dst_ld, dst_row0);
}

template <typename Src, typename Dst>
void launch_convert_vec(const Src* src, int64_t off, int N, Dst* dst, cudaStream_t st) {
  launch_k(convert_vec_kernel<Src, Dst>, dim3(grid_for(N, 256, 1024)), dim3(256), 0, st, src, off, N, dst);
}

// explicit instantiations

// ============================================================================ P2P TP exchange
// One process per GPU, peers' exchange regions mapped by CUDA IPC (energon_p2p_connect): the TP
// reduction of the row-parallel partial is done by the kernels themselves over peer memory instead
// of NCCL ("accumulated by communications").  Region of every rank (same offsets):
//   [flags: ready[8] | delivered[8] u64, counter] [X fp32 R x H] [A act R x H] [P act R x H]
// Protocol per exchange (epoch e, identical on every rank -- SPMD):
//   p2p_flag(READY, signal+wait): after this rank's GEMM wrote P, publish ready[me] = e on every peer
//     (release.sys) and wait until every peer published ready = e here;
//   p2p_reduce_ln: rows of this rank's shard: sum_q P_q[t] in rank order (fp32, rounded to act like
//     ncclReduceScatter), + bias + residual -> X (own rows), LN -> A row stored into EVERY rank's A
//     (the all-gather as NVLink stores); the last block to finish publishes delivered[me] = e;
//   p2p_flag(DELIVERED, wait): every peer's rows arrived here -- and every peer finished reading this
//     rank's P, so the next GEMM may overwrite it.
// The flag kernels are one block and never trigger their dependents early, so no kernel holds SMs
// while a rank waits for its peers (a single GPU shared by several ranks stays deadlock-free).
struct PeerSetK {
  char* base[8];
};

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void p2p_flag_kernel(PeerSetK ps, int k, int me, int kind, uint64_t epoch, int do_signal) {
  pdl_wait();  // the kernel before (the GEMM writing P, or the pushing kernel) has completed
  const int q = threadIdx.x;
  if (q < k && do_signal) {
    __threadfence_system();
    st_release_sys(reinterpret_cast<uint64_t*>(ps.base[q]) + kind * 8 + me, epoch);
  }
  if (q < k) {
    const uint64_t* f = reinterpret_cast<const uint64_t*>(ps.base[me]) + kind * 8 + q;
    while (ld_acquire_sys(f) < epoch) __nanosleep(100);
  }
}

// last block of a grid publishes delivered[me] = epoch on every peer (after all blocks' stores)
__device__ __forceinline__ void p2p_grid_done(const PeerSetK& ps, int k, int me, uint64_t epoch) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* counter = reinterpret_cast<unsigned*>(ps.base[me] + 16 * sizeof(uint64_t));
    const unsigned prev = atomicAdd(counter, 1u);
    if (prev == gridDim.x - 1) {
      *counter = 0;  // self-reset for the next exchange (stream-ordered)
      __threadfence_system();
      for (int q = 0; q < k; ++q) st_release_sys(reinterpret_cast<uint64_t*>(ps.base[q]) + 8 + me, epoch);
    }
  }
}

// slot_rows > 0: the partials were pushed here by the peers' GEMM epilogues (GEMM -> reduce-scatter
// fused, see launch_gemm_tc's ShardStore): rank q's partial of local row i is at
// off_P + (q * slot_rows + i) * H of THIS rank's region; slot_rows == 0: read each peer's own P.
template <typename Act, int LN_MAXV, int TPR>
__global__ void __launch_bounds__(TPR) p2p_reduce_ln_kernel(PeerSetK ps, int k, int me, int64_t off_X, int64_t off_A,
                                                            int64_t off_P, int row0, int rows, int H,
                                                            const float* __restrict__ bias,
                                                            const float* __restrict__ g, const float* __restrict__ b,
                                                            float eps, int write_A, uint64_t epoch, int slot_rows) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[32];
  if ((int)blockIdx.x < rows) {
    const int t = row0 + blockIdx.x;
    float* xrow = reinterpret_cast<float*>(ps.base[me] + off_X) + (int64_t)t * H;
    float4 v[LN_MAXV], acc[LN_MAXV];
    int nv = 0;
#pragma unroll
    for (int i = 0; i < LN_MAXV; ++i) {
      const int c = threadIdx.x + i * TPR;
      if (c < H / 4) {
        v[i] = __ldcs(reinterpret_cast<const float4*>(xrow) + c);
        acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        nv = i + 1;
      }
    }
    for (int q = 0; q < k; ++q) {  // rank order: every rank sums the same way
      const Act* prow = slot_rows ? reinterpret_cast<const Act*>(ps.base[me] + off_P) +
                                        ((int64_t)q * slot_rows + blockIdx.x) * H
                                  : reinterpret_cast<const Act*>(ps.base[q] + off_P) + (int64_t)t * H;
#pragma unroll
      for (int i = 0; i < LN_MAXV; ++i)
        if (i < nv) {
          const float4 x = Row4<Act>::load(prow + 4 * (threadIdx.x + i * TPR));
          acc[i].x += x.x;
          acc[i].y += x.y;
          acc[i].z += x.z;
          acc[i].w += x.w;
        }
    }
#pragma unroll
    for (int i = 0; i < LN_MAXV; ++i)
      if (i < nv) {
        const int c = threadIdx.x + i * TPR;
        const float4 q = *reinterpret_cast<const float4*>(bias + 4 * c);
        // the reduced partial is rounded to the activation type, as a reduce-scatter would store it
        v[i].x += to_f32(from_f32<Act>(acc[i].x)) + q.x;
        v[i].y += to_f32(from_f32<Act>(acc[i].y)) + q.y;
        v[i].z += to_f32(from_f32<Act>(acc[i].z)) + q.z;
        v[i].w += to_f32(from_f32<Act>(acc[i].w)) + q.w;
        Row4<float>::store(xrow + 4 * c, v[i]);
      }
    if (write_A) {
      float mean, rstd;
      row_stats(v, nv, H, eps, red, mean, rstd);
#pragma unroll
      for (int i = 0; i < LN_MAXV; ++i)
        if (i < nv) {
          const int j = 4 * (threadIdx.x + i * TPR);
          const float4 y = ln_apply(v[i], mean, rstd, g, b, j);
          for (int q = 0; q < k; ++q)
            Row4<Act>::store(reinterpret_cast<Act*>(ps.base[q] + off_A) + (int64_t)t * H + j, y);
        }
    }
  }
  p2p_grid_done(ps, k, me, epoch);
}

// all-gather by pushing: this rank's rows [row0, row0 + rows) of the buffer at `off` (row_bytes each)
// are stored into the same rows of every peer's region
__global__ void p2p_push_rows_kernel(PeerSetK ps, int k, int me, int64_t off, int row0, int rows, int64_t row_bytes,
                                     uint64_t epoch) {
  pdl_trigger();
  pdl_wait();
  const int64_t n16 = (int64_t)rows * row_bytes / 16;
  const uint4* src = reinterpret_cast<const uint4*>(ps.base[me] + off + (int64_t)row0 * row_bytes);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = src[i];
    for (int q = 0; q < k; ++q)
      if (q != me) reinterpret_cast<uint4*>(ps.base[q] + off + (int64_t)row0 * row_bytes)[i] = v;
  }
  p2p_grid_done(ps, k, me, epoch);
}

void launch_p2p_flag(const PeerSet& ps, int k, int me, int kind, uint64_t epoch, int do_signal, cudaStream_t st) {
  PeerSetK p;
  for (int i = 0; i < 8; ++i) p.base[i] = reinterpret_cast<char*>(ps.base[i]);
  launch_k(p2p_flag_kernel, dim3(1), dim3(32), 0, st, p, k, me, kind, epoch, do_signal);
}

template <typename Act>
void launch_p2p_reduce_ln(const PeerSet& ps, int k, int me, int64_t off_X, int64_t off_A, int64_t off_P, int row0,
                          int rows, int H, const float* bias, const float* g, const float* b, float eps, int write_A,
                          uint64_t epoch, cudaStream_t st, int slot_rows) {
  PeerSetK p;
  for (int i = 0; i < 8; ++i) p.base[i] = reinterpret_cast<char*>(ps.base[i]);
  const int grid = rows > 0 ? rows : 1;  // an empty shard still takes part in the completion count
  const int tpr = ln_tpr(H, rows);
  if (tpr == 512)
    NV_DISPATCH_T(H, 512, (launch_k(p2p_reduce_ln_kernel<Act, NVX, 512>, dim3(grid), dim3(512), 0, st, p, k, me, off_X,
                                    off_A, off_P, row0, rows, H, bias, g, b, eps, write_A, epoch, slot_rows)))
  else
    NV_DISPATCH_T(H, 256, (launch_k(p2p_reduce_ln_kernel<Act, NVX, 256>, dim3(grid), dim3(256), 0, st, p, k, me, off_X,
                                    off_A, off_P, row0, rows, H, bias, g, b, eps, write_A, epoch, slot_rows)))
}

void launch_p2p_push_rows(const PeerSet& ps, int k, int me, int64_t off, int row0, int rows, int64_t row_bytes,
                          uint64_t epoch, cudaStream_t st) {
  PeerSetK p;
  for (int i = 0; i < 8; ++i) p.base[i] = reinterpret_cast<char*>(ps.base[i]);
  const int64_t n16 = (int64_t)rows * row_bytes / 16;
  const int grid = n16 > 0 ? grid_for(n16, 256, 148 * 4) : 1;
  launch_k(p2p_push_rows_kernel, dim3(grid), dim3(256), 0, st, p, k, me, off, row0, rows, row_bytes, epoch);
}
template void launch_p2p_reduce_ln<float>(const PeerSet&, int, int, int64_t, int64_t, int64_t, int, int, int,
                                          const float*, const float*, const float*, float, int, uint64_t, cudaStream_t,
                                          int);
template void launch_p2p_reduce_ln<bf16>(const PeerSet&, int, int, int64_t, int64_t, int64_t, int, int, int,
                                         const float*, const float*, const float*, float, int, uint64_t, cudaStream_t,
                                         int);

#define INST_ACT(Act)                                                                                                   \
  template void launch_embed_ln<Act>(const int*, const int*, const int*, int, int, int, int, int, const Act*,           \
                                     const Act*, const float*, const float*, float, float*, Act*, cudaStream_t,         \
                                     float2*);                                                                          \
  template void launch_gather_ln<Act>(const float*, const int*, const int*, int, int, int, const float*, const float*,  \
                                      float, float*, Act*, cudaStream_t, float2*);                                      \
  template void launch_local_reduce_scatter<Act>(const PtrList&, int, int64_t, int, cudaStream_t);                     \
  template void launch_residual_ln<Act>(float*, const Act*, const float*, int, int, const float*, const float*, float,   \
                                        Act*, cudaStream_t, float2*);                                                   \
  template void launch_final_ln_unpack<Act>(const float*, const int*, int, int, int, const float*, const float*, float,  \
                                            int, Act*, cudaStream_t);                                                   \
  template void launch_unpack_qkv<Act>(const Act*, const int*, int, int, int, int, Act*, Act*, Act*, cudaStream_t);    \
  template void launch_repack<Act>(const Act*, const int*, const int*, int, int, int, int, Act*, cudaStream_t);        \
  template void launch_local_allreduce<Act>(const PtrList&, int, int64_t, int, cudaStream_t);
INST_ACT(float)
INST_ACT(bf16)

#define INST_CVT(Src, Dst)                                                                                             \
  template void launch_relayout<Src, Dst>(const Src*, int64_t, int64_t, int64_t, int, int, Dst*, int64_t, int64_t,     \
                                          cudaStream_t);                                                                \
  template void launch_convert_vec<Src, Dst>(const Src*, int64_t, int, Dst*, cudaStream_t);
INST_CVT(double, float)
INST_CVT(double, bf16)
INST_CVT(float, float)
INST_CVT(float, bf16)
INST_CVT(bf16, float)
INST_CVT(bf16, bf16)

}  // namespace energon

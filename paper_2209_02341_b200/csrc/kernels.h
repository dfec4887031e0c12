// kernels.h -- host-side launchers of the energon CUDA kernels (internal; not part of the C ABI).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define ENERGON_MAX_B 1024

#include <atomic>
#include <utility>

namespace energon {

typedef __nv_bfloat16 bf16;

bool pdl_enabled();  // ENERGON_NO_PDL=1 disables programmatic dependent launch (A/B)

// Launch with programmatic stream serialization (PDL): the kernel may begin while the previous
// kernel in the stream finishes; it calls pdl_wait() before its first dependent global access.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies to the CURRENT device only: raise the limit
// once per (kernel, device) -- `done` is the kernel's own bit set of devices already configured.
template <typename... KArgs>
inline void smem_attr_once(void (*kernel)(KArgs...), int smem, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  done.fetch_or(bit, std::memory_order_acq_rel);
}

// seq_lens passed by value as a kernel parameter (4 KB): no host->device copy, no sync.
struct LensParam {
  int lens[ENERGON_MAX_B];
};

struct PtrList {
  void* p[8];
};

// P2P TP exchange over CUDA-IPC-mapped peer regions (kernels_misc.cu; protocol described there)
struct PeerSet {
  void* base[8];  // exchange region of every rank of the TP group (own included)
};
enum { P2P_READY = 0, P2P_DELIVERED = 1 };
constexpr int64_t P2P_FLAG_BYTES = 256;  // ready[8] | delivered[8] u64 | completion counter
void launch_p2p_flag(const PeerSet& ps, int k, int me, int kind, uint64_t epoch, int do_signal, cudaStream_t st);
template <typename Act>
void launch_p2p_reduce_ln(const PeerSet& ps, int k, int me, int64_t off_X, int64_t off_A, int64_t off_P, int row0,
                          int rows, int H, const float* bias, const float* g, const float* b, float eps, int write_A,
                          uint64_t epoch, cudaStream_t st, int slot_rows = 0);
void launch_p2p_push_rows(const PeerSet& ps, int k, int me, int64_t off, int row0, int rows, int64_t row_bytes,
                          uint64_t epoch, cudaStream_t st);

// a1.  Every argument but the lengths, which travel by value (LensParam) so a replayed CUDA graph
// updates exactly one kernel node per batch (index_maps_kernel_fn identifies it).
struct IndexMapsArgs {
  int B, S;
  int rows;                    // packed rows the linears run on (>= T): pack_idx[t] = -1 for t in [T, rows)
  int* offsets;                // [B + 1]
  int* pack_idx;               // [rows]
  int* pos;                    // [rows]
  int* unpack_idx;             // [B * S]
  const int* tok;              // [B, S] token ids to range-check (nullptr: none)
  int V;
  int* err_flag;               // set to 1 on a bad token id
  int* lens_d;                 // [B] device copy of the lengths for later kernels (nullptr: none)
  uint32_t* attn_work;         // attention work list (nullptr: none), see build_attn_work
  int causal, attn_bm, attn_bn;
};
void launch_index_maps(const LensParam& lp, const IndexMapsArgs& a, cudaStream_t st);
const void* index_maps_kernel_fn();
// lengths -> lens_d and the attention work list only (kernel-level attention entry)
void launch_attn_plan(const LensParam& lp, int B, int causal, int bm, int bn, int* lens_d, uint32_t* work,
                      cudaStream_t st);
// a2 + a3
// rows [row0, row0 + rows) of the packed layout
template <typename Act>
void launch_embed_ln(const int* tok, const int* pack_idx, const int* unpack_idx, int row0, int rows, int S, int V, int H,
                     const Act* tok_emb, const Act* pos_emb, const float* g, const float* b, float eps, float* X, Act* A,
                     cudaStream_t st, float2* stats = nullptr);
template <typename Act>
void launch_gather_ln(const float* x, const int* pack_idx, const int* T_dev, int row0, int rows, int H, const float* g,
                      const float* b, float eps, float* X, Act* A, cudaStream_t st, float2* stats = nullptr);
// a9 / a12
template <typename Act>
void launch_residual_ln(float* X, const Act* P, const float* bias, int rows, int H, const float* g, const float* b,
                        float eps, Act* A, cudaStream_t st, float2* stats = nullptr);
// stats != nullptr (the N3 LN-prologue mode): the row's (mean, rstd) are written to stats[t] for the GEMM
// prologue to apply, and A (may be nullptr) is not needed
// a13
template <typename Out>
void launch_final_ln_unpack(const float* X, const int* unpack_idx, int rows_are_cells, int cells, int H, const float* g,
                            const float* b, float eps, int apply_ln, Out* out, cudaStream_t st);
// a5 / a7
template <typename Act>
void launch_unpack_qkv(const Act* QKV, const int* pack_idx, int T, int S, int hk, int d, Act* Q, Act* K, Act* V,
                       cudaStream_t st);
template <typename Act>
void launch_repack(const Act* O, const int* pack_idx, const int* unpack_idx, int T, int S, int hk, int d, Act* C,
                   cudaStream_t st);
// ring != 0: NCCL ring numerics (one rounding to Act per hop) instead of the fp32 rank-order sum
template <typename Act>
void launch_local_allreduce(const PtrList& parts, int k, int64_t n, int ring, cudaStream_t st);
template <typename Act>
void launch_local_reduce_scatter(const PtrList& parts, int k, int64_t shard, int ring, cudaStream_t st);
void launch_local_all_gather(const PtrList& parts, int k, int64_t shard_bytes, cudaStream_t st);
// load-time relayout
template <typename Src, typename Dst>
void launch_relayout(const Src* src, int64_t ld, int64_t row0, int64_t col0, int N, int K, Dst* dst, int64_t dst_ld,
                     int64_t dst_row0, cudaStream_t st);
template <typename Src, typename Dst>
void launch_convert_vec(const Src* src, int64_t off, int N, Dst* dst, cudaStream_t st);

// a6: masked attention over the padded per-head layout [B, hk, S, d].  The lengths and the work list
// live in device memory (written by the index-maps kernel / launch_attn_plan), so no attention launch
// depends on the batch's lengths on the host.
// Tensor maps of Q / K / V of the tcgen05 kernel (cached per context: they depend on the buffers and B*hk*S)
struct AttnMaps {
  CUtensorMap mq, mk, mv;
  const void *q = nullptr, *k = nullptr, *v = nullptr;
  int rows = 0, d = 0, bn = 0;
  bool valid = false;
  CUtensorMap mo;  // output map of the TMA-store epilogue (packed context rows or padded O)
  const void* o = nullptr;
  int o_rows = 0, o_n = 0;
  bool o_valid = false;
};
int attention_tile_bm();  // query rows of one work item of the tcgen05 kernel
int attention_tile_bn();  // keys per tile (the work list's cost unit)
// padded O [B, hk, S, d]; bf16 d = 64 / 128 runs the tcgen05 kernel (needs work_d), otherwise SIMT
template <typename Act>
void launch_attention(const Act* Q, const Act* K, const Act* V, Act* O, const int* lens_d, const uint32_t* work_d,
                      int B, int hk, int S, int d, int causal, cudaStream_t st, AttnMaps* maps = nullptr);
// a7 fused: O rows written straight to the packed [T, hk*d] layout at row offsets[b] + s (bf16, d = 64 /
// 128 only; false if unsupported or the tensor maps cannot be built)
bool launch_attention_packed(const bf16* Q, const bf16* K, const bf16* V, bf16* ctx_packed, const int* offsets,
                             const int* lens_d, const uint32_t* work_d, int B, int hk, int S, int d, int causal,
                             cudaStream_t st, AttnMaps* maps = nullptr);
bool launch_attention_tc(const bf16* Q, const bf16* K, const bf16* V, bf16* ctx_packed, const int* offsets,
                         bf16* O_padded, const int* lens_d, const uint32_t* work_d, int B, int hk, int S, int d,
                         int causal, cudaStream_t st, AttnMaps* maps);
int attention_impl();  // ENERGON_ATTN (A/B): 4 = tcgen05 v2 (default), 5 = tcgen05 v3 (one CTA per SM, two Q tiles)

// GEMM epilogues.  EPI_BIAS_QKV = bias, then a5 fused: the packed QKV row t / column block is
// scattered straight into the padded per-head Q, K, V [B, hk, S, d] (needs d % 32 == 0).
enum { EPI_NONE = 0, EPI_BIAS = 1, EPI_BIAS_GELU = 2, EPI_BIAS_QKV = 3 };
struct QkvScatter {
  const int* pack_idx;  // packed row -> padded cell (nullptr: identity, padded A/B mode)
  bf16 *q, *k, *v;
  int S, hk, d;
  const CUtensorMap* maps = nullptr;  // host: make_qkv_store_maps output (2-CTA kernel: TMA-store a5)
};

// fp32 SIMT GEMM (parity mode): D[M,N] = A[M,K] W[N,K]^T (+bias) (gelu)
void launch_gemm_f32(const float* A, const float* W, const float* bias, float* D, int M, int N, int K, int epi,
                     cudaStream_t st);

// bf16 tcgen05 GEMM.  Operands are K-major bf16 described by TMA maps with a 64-element (128 B)
// inner box and 128-byte swizzle: A [M,K] with a 128-row box, W [N,K] with a bn-row box (bn = the
// tile N, or half of it for the 2-CTA pair tiles, chosen per call by tc_pick_bn).
bool make_tmap_kmajor(CUtensorMap* map, const void* ptr, int rows, int K, int box_rows);  // inner box 64, SW128
int tc_pick_bn(int M, int N, int K = 0);  // tile code (see gemm_tc.cu); K = 0: unknown
int tc_w_box(int code);        // row box of the W tensor map the code needs (256, 128, 112, 96 or 64)
bool make_tmap_store(CUtensorMap* map, const void* ptr, int rows, int N);  // D map of the TMA-store epilogue
bool make_tmap_store_box(CUtensorMap* map, const void* ptr, int rows, int N, int box_cols);  // 32 rows x 32 / 16 cols
// Scratch of the stream-K tail split: fp32 partial tiles + self-resetting arrival counters.  GEMMs that
// share one are stream-ordered, so each context (one forward stream at a time) owns its own;
// tail_ws_alloc sizes it for this device, nullptr in launch_gemm_tc = a per-device default.
struct TailWs {
  float* ws = nullptr;
  int* counters = nullptr;
};
bool tail_ws_alloc(TailWs* w);  // cudaMalloc + zeroed counters (synchronous); false on OOM
void tail_ws_free(TailWs* w);
// GEMM -> reduce-scatter fused (P2P exchange): output row t goes to rank s = t / rpr, which owns rows
// [s rpr, (s+1) rpr), at local row t - s rpr of the store map maps[s] (that rank's slot for this rank's
// partial, in its IPC-mapped region).  rpr is a multiple of 32 so no 32-row store box straddles ranks.
struct ShardStore {
  CUtensorMap maps[8];
  int rpr;
  int k;
  // QKV GEMM (EPI_BIAS_QKV) instead: maps[0..2] are 3-D store maps of Q, K, V [B*hk, S, d] (32 x 32 x 1 box,
  // 64-byte swizzle) and the a5 scatter leaves by TMA bulk-tensor stores (qkv_tma = 1)
  int qkv_tma;
};
// the three Q / K / V store maps of the TMA a5 scatter (false if they cannot be encoded)
bool make_qkv_store_maps(CUtensorMap (&maps)[3], const bf16* q, const bf16* k, const bf16* v, int B, int hk, int S, int d);
// tmD: the output map (make_tmap_store) or nullptr to build it per call.
// returns false (nothing launched) if the output tensor map cannot be built (D not 16-byte aligned)
bool launch_gemm_tc(const CUtensorMap& tmA, const CUtensorMap& tmB, int bn, const float* bias, bf16* D, int M, int N,
                    int K, int epi, cudaStream_t st, const QkvScatter* qkv = nullptr, const CUtensorMap* tmD = nullptr,
                    const TailWs* tw = nullptr, const ShardStore* shard = nullptr);
// N3: bf16 GEMM whose A operand is LN(X) built in the prologue from fp32 X [M, K], the row statistics
// (mean, rstd) and the LN weight / bias (1-CTA 128 x 256 tiles, W from the box-256 map); K % 64 == 0.
// Same epilogues as launch_gemm_tc; false if unsupported.
bool launch_gemm_ln(const CUtensorMap& tmB, const float* X, const float2* stats, const float* g, const float* b,
                    const float* bias, bf16* D, int M, int N, int K, int epi, cudaStream_t st, const QkvScatter* qkv);
int num_sms();  // SM count of the current device

}  // namespace energon

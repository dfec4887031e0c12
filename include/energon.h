/*
 * energon.h -- C ABI of the B200-native DRCE tensor-parallel GPT layer stack.
 *
 * The library computes the forward pass of a pre-LN GPT transformer layer stack
 * over a variable-length padded batch with Distributed Redundant Computation
 * Elimination (DRCE, sec 4.3 / fig:drce) under 1-D Megatron
 * tensor parallelism (sec 4.1.3 / fig:transformer1d):
 *
 *   a1  prefix sum of seq_lens -> offsets / pack / unpack index maps
 *   a2  embedding gather of the valid tokens only ("remove padding")
 *   per layer:
 *   a3  LN1 on packed rows
 *   a4  column-parallel QKV GEMM + bias on packed rows
 *   a5  rebuild padding + transpose to [B, h/k, S, d] (paper's fused kernel #1)
 *   a6  masked softmax attention, padded keys / queries skipped
 *   a7  remove padding + transpose back to packed [T, H/k] (paper's kernel #2)
 *   a8  row-parallel out-proj GEMM
 *   a9  TP allreduce ("accumulated by communications") + bias + residual + LN2
 *   a10 column-parallel MLP-up GEMM + bias + GeLU
 *   a11 row-parallel MLP-down GEMM
 *   a12 TP allreduce + bias + residual (+ LN1 of the next layer)
 *   a13 final LN + unpack to the caller's padded layout, pad rows exactly 0
 *
 * Every entry point returns an energon_status and never throws.  Host-visible
 * arguments are validated before any launch; on error nothing is enqueued and
 * the context is unchanged (the message is in energon_last_error).
 * A context is single-threaded: one context per rank (per GPU).
 */
#ifndef ENERGON_H
#define ENERGON_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define ENERGON_API __attribute__((visibility("default")))
#else
#define ENERGON_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ENERGON_OK = 0,
  ENERGON_ERR_ARG = -1,        /* NULL pointer / bad enum / layer index out of range                    */
  ENERGON_ERR_CONFIG = -2,     /* H != h*d, h % k, F % k, tp_rank out of range  */
  ENERGON_ERR_SHAPE = -3,      /* unsupported shape (e.g. hidden not a multiple of 64 in bf16 mode)    */
  ENERGON_ERR_LENGTH = -4,     /* seq_lens[b] not in [1, max_len], or max_len > max_seq */
  ENERGON_ERR_TOKEN = -5,      /* a token id outside [0, vocab) was seen on the device; energon_sync */
  ENERGON_ERR_CAPACITY = -6,   /* batch * max_len > max_tokens, or batch > ENERGON_MAX_BATCH          */
  ENERGON_ERR_NOT_LOADED = -7, /* forward before every weight was loaded                               */
  ENERGON_ERR_CUDA = -8,       /* a CUDA runtime error (sticky errors surface on energon_sync)         */
  ENERGON_ERR_NCCL = -9,       /* an NCCL error                                                        */
  ENERGON_ERR_OOM = -10        /* device allocation failed                                             */
} energon_status;

enum { ENERGON_DTYPE_F32 = 0, ENERGON_DTYPE_BF16 = 1, ENERGON_DTYPE_F64 = 2 };
enum { ENERGON_FULL = 0, ENERGON_RANK_SHARD = 1 };
enum { ENERGON_MAX_BATCH = 1024 };

/*
 * Model / run configuration.  dtype is the arithmetic mode:
 *   ENERGON_DTYPE_F32  -- parity mode: fp32 storage and fp32 SIMT arithmetic (target 1e-4);
 *   ENERGON_DTYPE_BF16 -- production: bf16 storage, fp32 accumulation, fp32 residual stream,
 *                         tcgen05 tensor-core GEMMs (target 2e-2).
 * drce = 1 runs linears on packed rows (the method); drce = 0 runs them on all
 * B*max_len padded rows (the paper's "pure EnergonAI" A/B).
 * max_tokens bounds batch*max_len (workspace is sized from it at init).
 */
typedef struct {
  int32_t num_layers, hidden, num_heads, ffn, vocab, max_seq;
  int32_t causal;   /* 1 = decoder causal mask; 0 = length mask only */
  int32_t dtype;    /* ENERGON_DTYPE_F32 | ENERGON_DTYPE_BF16 */
  int32_t drce;     /* 1 = packed linears (DRCE), 0 = padded A/B */
  int32_t tp_size;  /* k: ranks of the TP group (1, 2, 4, 8) */
  int32_t tp_rank;  /* this context's rank in [0, k) */
  int32_t device;   /* CUDA device ordinal this context drives */
  int32_t max_tokens;
  int32_t final_ln; /* 1 = apply the final LayerNorm */
  float ln_eps;     /* 1e-5 */
  int32_t comm;     /* k > 1: ENERGON_COMM_NCCL (0, default) or ENERGON_COMM_P2P (1, see energon_p2p_connect) */
} energon_config;
enum { ENERGON_COMM_NCCL = 0, ENERGON_COMM_P2P = 1 };

/*
 * One layer's weights, matrices [in, out] row-major (y = x W + b; SPEC.md:85,
 * 126-129).  With src_layout = ENERGON_FULL the pointers hold the unsharded
 * tensors (wq,wk,wv,wo [H,H]; w1 [H,F]; w2 [F,H]; biases / LN vectors [H] or [F])
 * and the library slices this rank's share: heads [r h/k, (r+1) h/k) of q,k,v
 * and the matching rows of wo; FFN columns [r F/k, (r+1) F/k) of w1 / b1 and
 * rows of w2.  With ENERGON_RANK_SHARD the
 * caller passes pre-sliced shards in the same [in,out] layout (wq [H,H/k],
 * bq [H/k], wo [H/k,H], w1 [H,F/k], b1 [F/k], w2 [F/k,H]); bo, b2 and the LN
 * vectors are always full (added once after the reduce on every rank, C9).
 * Sources are read during the call only (they may be freed afterwards); the call first waits for
 * all work already issued to the device, so sources written on any stream are complete.
 */
typedef struct {
  const void *wq, *wk, *wv, *wo, *bq, *bk, *bv, *bo, *w1, *b1, *w2, *b2, *ln1_g, *ln1_b, *ln2_g, *ln2_b;
} energon_layer_weights;

typedef struct {
  int64_t forwards;         /* completed energon_forward* calls */
  int64_t allreduce_calls;  /* TP reductions issued (2 per layer per forward when k > 1) */
  int64_t kernel_launches;  /* kernels this library launched, cumulative */
  int64_t last_tokens;      /* T = sum(seq_lens) of the last forward */
  int64_t last_rows;        /* rows the linears ran on in the last forward: T rounded up to a bucket of 128
                               (<= max_tokens) with DRCE, B*S with drce=0 */
  int64_t weight_bytes;     /* device bytes held for this rank's weights */
  int64_t workspace_bytes;  /* device bytes held for activations */
  int64_t prefetch_bytes;   /* PMEP: bytes fetched from the memory pool, cumulative */
  int64_t fused_exchanges;  /* P2P: TP reductions whose partials the row-parallel GEMM stored straight into the
                               owners' slots (GEMM -> reduce-scatter fused), cumulative */
  int64_t graphs_recorded;  /* ENERGON_OPT_GRAPH: CUDA graphs recorded (cache misses), cumulative */
} energon_stats;

/*
 * Per-class device time of the kernels this library launched while profiling was enabled,
 * measured with CUDA events recorded on the forward stream around every launch (class
 * "gemm" = the four tcgen05 / SIMT linears, "attn" = a6, "mem" = the HBM-bound kernels
 * a1-a3, a5, a7, a9, a12, a13, "comm" = the TP reductions).  Work is algorithmic: GEMM
 * flops = 2 M N K per launch, attention flops = 4 d sum_b(allowed keys) per head, memory
 * bytes = bytes each kernel must read + write once, comm bytes = reduced payload.
 */
typedef struct {
  double gemm_ms, attn_ms, mem_ms, comm_ms;
  double gemm_flops, attn_flops, mem_bytes, comm_bytes;
  int64_t gemm_launches, attn_launches, mem_launches, comm_calls;
} energon_profile;

/*
 * This rank's share under 1-D TP: heads
 * [head0, head0 + heads) -> columns [qkv_col0, qkv_col0 + qkv_cols) of wq / wk / wv and rows of wo;
 * FFN columns [ffn_col0, ffn_col0 + ffn_cols) of w1 / b1 and rows of w2.
 */
typedef struct {
  int32_t head0, heads, qkv_col0, qkv_cols, ffn_col0, ffn_cols;
} energon_shard;

typedef struct energon_ctx energon_ctx;

/*
 * Peer memory pooling (PMEP, sec 4.4, fig:offload / fig:multistream).
 * energon_pmep_plan (host only): the off-device layers when `resident` of `num_layers` layers stay on
 *   the computing GPU, "distributed evenly among those to be held on device":
 *   layer floor((g+1) L / m) - 1 for g = 0..m-1, m = L - resident; (24, 20) -> {5, 11, 17, 23}
 *   (PAPER.md:601-602).  out_layers holds m ints, ascending.
 * energon_offload_layers: move the listed (loaded) layers' weight matrices into the pool -- pool 0 =
 *   pinned host memory, 1 = the memory of CUDA device `peer_device` (NVLink peer; the computing device
 *   itself is accepted, a same-device pool for single-GPU tests) -- and free them on
 *   the computing GPU.  During a forward each off-device layer is copied into one of `slots` staging
 *   buffers on a separate copy stream, issued as soon as the slot's previous layer finished computing
 *   ("prefetch the next off-device layer immediately ..."); compute waits on an event.
 *   Results are bit-identical to the all-resident run.  Call after every layer is loaded.
 */
ENERGON_API energon_status energon_pmep_plan(int32_t num_layers, int32_t resident, int32_t* out_layers);
ENERGON_API energon_status energon_offload_layers(energon_ctx* ctx, const int32_t* layers, int32_t n, int32_t slots,
                                                  int32_t pool, int32_t peer_device);

/* Host-only: the shard of cfg->tp_rank (validates cfg like energon_init; touches no device). */
ENERGON_API energon_status energon_shard_plan(const energon_config* cfg, energon_shard* out);

/*
 * P2P TP exchange (cfg.comm = ENERGON_COMM_P2P, one process per GPU of one node): instead of NCCL the
 * kernels reduce the row-parallel partials over peer memory ("accumulated by communications",
 * PAPER.md:290) -- signal/wait flags, a reduce + bias + residual + LayerNorm kernel that reads every
 * rank's partial rows of its own shard in rank order and stores the normalised rows straight into
 * every rank's activation buffer (reduce-scatter, LN and all-gather in one pass over NVLink), and a
 * completion flag.  Same results as the NCCL sequence-parallel schedule (bit-identical replicas).
 *   energon_p2p_handle: 64-byte CUDA IPC handle of this rank's exchange region (after energon_init).
 *   energon_p2p_connect: handles of all k ranks in rank order (the caller all-gathers them, e.g. with
 *     torch.distributed); maps the peers' regions.  Required before the first forward.
 * Errors: ENERGON_ERR_CONFIG unless cfg.comm == P2P and tp_size > 1; ENERGON_ERR_CUDA if a handle
 * cannot be opened.  Forward calls are SPMD and must be issued by every rank (they wait for peers).
 */
ENERGON_API energon_status energon_p2p_handle(energon_ctx* ctx, void* out_64_bytes);
ENERGON_API energon_status energon_p2p_connect(energon_ctx* ctx, const void* handles_k_x_64_bytes);

/* 128-byte NCCL unique id for a TP group (call on one rank, broadcast the bytes). */
ENERGON_API energon_status energon_get_unique_id(void* out_128_bytes);

/*
 * Create a context on cfg->device.  When cfg->tp_size > 1 this is a collective
 * over the k ranks of the group (ncclCommInitRank); nccl_unique_id must be the
 * same 128 bytes on every rank.  nccl_unique_id is ignored when tp_size == 1.
 */
ENERGON_API energon_status energon_init(const energon_config* cfg, const void* nccl_unique_id, energon_ctx** out);

/*
 * Create k contexts for one TP group that all live on cfg->device inside this
 * process (single-GPU tensor parallelism: the reduction is an in-device sum of
 * the k partials in rank order).  Used to exercise the sharded path on one GPU.
 */
ENERGON_API energon_status energon_init_local_group(const energon_config* cfg, int32_t k, energon_ctx** out_k);

/* tok_emb [vocab, H], pos_emb [max_seq, H], final LN gamma / beta [H] (replicated). */
ENERGON_API energon_status energon_load_embeddings(energon_ctx* ctx, const void* tok_emb, const void* pos_emb,
                                       const void* lnf_g, const void* lnf_b, int32_t src_dtype,
                                       int32_t src_on_device);

ENERGON_API energon_status energon_load_layer_weights(energon_ctx* ctx, int32_t layer, const energon_layer_weights* w,
                                          int32_t src_dtype, int32_t src_on_device, int32_t src_layout);

/*
 * Forward pass (SPEC.md:147-155 serial_forward semantics).  SPMD over the TP
 * group: every rank calls it with identical arguments in the same order
 * (PAPER.md:251, 300).  seq_lens is the engine command's length list
 * (PAPER.md:368-370), host memory, copied during the call.
 *   tokens_d  device int32 [batch, max_len]; ids of valid positions in [0, vocab); pad positions are
 *             ignored (read as id 0).  A valid position holding an id outside [0, vocab) does not stop
 *             the forward (the row gathers embedding row 0); it sets a device flag that the next
 *             energon_sync returns as ENERGON_ERR_TOKEN -- on EVERY rank of a TP group, since every rank
 *             checks the whole batch (the flag never gates an enqueue, so ranks cannot diverge)
 *   seq_lens  host int32 [batch], each in [1, max_len]
 *   out_d     device [batch, max_len, hidden], dtype = cfg->dtype; rows s >= seq_lens[b] are 0
 *   stream    cudaStream_t (NULL = legacy default stream); the call returns after enqueue
 */
ENERGON_API energon_status energon_forward(energon_ctx* ctx, const int32_t* tokens_d, const int32_t* seq_lens,
                               int32_t batch, int32_t max_len, void* out_d, void* stream);

/* Same as energon_forward for a local group made by energon_init_local_group. */
ENERGON_API energon_status energon_forward_group(energon_ctx** ctxs, int32_t k, const int32_t* tokens_d,
                                     const int32_t* seq_lens, int32_t batch, int32_t max_len, void* out_d,
                                     void* stream);

/*
 * Layer-stack only, for teacher-forced per-layer parity: x_d fp32 [batch, max_len, H]
 * residual stream (valid rows are read), runs layers [layer_begin, layer_end) and
 * writes fp32 [batch, max_len, H] -- the residual stream after layer_end-1, or
 * its final LayerNorm if apply_final_ln; pad rows are 0.
 */
ENERGON_API energon_status energon_forward_hidden(energon_ctx* ctx, const float* x_d, const int32_t* seq_lens,
                                      int32_t batch, int32_t max_len, int32_t layer_begin, int32_t layer_end,
                                      int32_t apply_final_ln, float* out_d, void* stream);

/*
 * Non-blocking pipeline parallelism (NBPP, sec 4.2 / fig:engine): the model is
 * "partitioned by transformer layers" into pp_size stages; each stage is a context
 * (or a TP group of contexts, "combine both pipeline parallelism and tensor parallelism",
 * PAPER.md:345) that runs its contiguous layer range on every batch, and only the activations
 * travel stage to stage -- with DRCE they travel PACKED ([T, H] rows), so the inter-stage transfer
 * shrinks by the padding ratio too (an extension the paper does not state).
 *
 * energon_stage_plan (host only): out_begin[0..pp_size] with stage i = [out_begin[i], out_begin[i+1]);
 *   contiguous, sizes differ by at most one, earlier stages take the remainder (L=12, pp=4 -> 3 each,
 *   PAPER.md:548 "each device only executes 3 layers").  ENERGON_ERR_CONFIG unless 1 <= pp_size <= L.
 * energon_forward_stage: run layers [layer_begin, layer_end) on one batch.
 *   tokens_d  device int32 [batch, max_len] for the first stage (embed + remove padding), else NULL
 *   x_d       device fp32 [rows, H] residual-stream rows from the previous stage, else NULL
 *             (exactly one of tokens_d / x_d); rows = sum(seq_lens) with DRCE, batch*max_len without
 *   out_kind  ENERGON_STAGE_PACKED: out_d device fp32 [rows, H] = the residual stream after layer_end-1
 *             ENERGON_STAGE_FINAL:  out_d device [batch, max_len, H] cfg dtype = final LN (cfg.final_ln)
 *                                   + rebuild padding, pad rows exactly 0 (as energon_forward)
 *   Only layers [layer_begin, layer_end) must be loaded; the embeddings (energon_load_embeddings) only
 *   when tokens_d is given or out_kind is FINAL.  A stage with x_d and PACKED output needs >= 1 layer.
 *   Same SPMD / stream semantics and errors as energon_forward.  Chaining the stages of a plan gives
 *   bit-identical results to one energon_forward over all layers (the same kernels on the same rows).
 * energon_forward_stage_group: the same for a local TP group (energon_init_local_group).
 */
enum { ENERGON_STAGE_PACKED = 0, ENERGON_STAGE_FINAL = 1 };
ENERGON_API energon_status energon_stage_plan(int32_t num_layers, int32_t pp_size, int32_t* out_begin);
ENERGON_API energon_status energon_forward_stage(energon_ctx* ctx, const int32_t* tokens_d, const float* x_d,
                                                 const int32_t* seq_lens, int32_t batch, int32_t max_len,
                                                 int32_t layer_begin, int32_t layer_end, int32_t out_kind, void* out_d,
                                                 void* stream);
ENERGON_API energon_status energon_forward_stage_group(energon_ctx** ctxs, int32_t k, const int32_t* tokens_d,
                                                       const float* x_d, const int32_t* seq_lens, int32_t batch,
                                                       int32_t max_len, int32_t layer_begin, int32_t layer_end,
                                                       int32_t out_kind, void* out_d, void* stream);

/* Block until the context's work is done; surfaces sticky CUDA / NCCL / token errors. */
ENERGON_API energon_status energon_sync(energon_ctx* ctx);
ENERGON_API energon_status energon_get_stats(const energon_ctx* ctx, energon_stats* out);
/*
 * Runtime options (take effect at the next forward; host-only, no device work):
 *   ENERGON_OPT_DRCE   1 = packed linears (the method), 0 = padded A/B ("pure EnergonAI",
 *                      PAPER.md:567-571); the workspace is sized for max_tokens padded rows either way.
 *   ENERGON_OPT_GRAPH  1 = capture each distinct forward (shapes, buffers, and the row bucket: T rounded
 *                      up to 128) into a CUDA graph on a private stream and replay it on the caller's
 *                      stream (LRU cache of 32); a new batch of the same bucket replays the recorded
 *                      graph with its lengths written into the graph's one index-maps node;
 *                      ignored while profiling or with off-device (PMEP) layers.  Default 0.
 *   ENERGON_OPT_TP_SP  k > 1 only: 1 (default) = sequence-parallel schedule (reduce-scatter, bias +
 *                      residual + LN on this rank's 1/k of the rows, all-gather), 0 = allreduce and
 *                      the row-wise kernels replicated on every rank.
 *   ENERGON_OPT_RING_NUMERICS  local group only (energon_init_local_group; set it on every context): 1 = the
 *                      in-device reductions reproduce the numerics of NCCL's ring algorithm on a bf16
 *                      payload -- each chunk's running sum travels rank s+1 -> ... -> s and is rounded to
 *                      the activation type after every hop -- instead of the fp32 rank-order sum (0,
 *                      default).  Lets one GPU check the parity of the NCCL exchange.
 *   ENERGON_OPT_LN_FUSE  bf16, TP = 1, hidden % 64 == 0: 1 = FasterTransformer-style fusion (PAPER.md:572-576,
 *                      SURVEY.md 8(f) N3): the residual kernels write only X and each row's (mean, rstd), and
 *                      the QKV / MLP-up GEMMs build LN(X) in their prologue (bit-identical A, so identical
 *                      output); 0 (default) = the residual kernel writes the bf16 LN output A.
 *                      ENERGON_ERR_CONFIG outside that domain.
 */
enum { ENERGON_OPT_DRCE = 1, ENERGON_OPT_TP_SP = 2, ENERGON_OPT_GRAPH = 3, ENERGON_OPT_RING_NUMERICS = 4,
       ENERGON_OPT_LN_FUSE = 5 };
ENERGON_API energon_status energon_set_option(energon_ctx* ctx, int32_t option, int32_t value);

/* Enable (1) / disable (0) per-launch CUDA-event timing; enabling resets the accumulators. */
ENERGON_API energon_status energon_set_profiling(energon_ctx* ctx, int32_t enable);
/* Synchronise the recorded events and return the accumulated profile. */
ENERGON_API energon_status energon_get_profile(energon_ctx* ctx, energon_profile* out);
ENERGON_API const char* energon_last_error(const energon_ctx* ctx);
ENERGON_API const char* energon_status_string(energon_status s);
ENERGON_API void energon_destroy(energon_ctx* ctx);

/*
 * Kernel-level entry points used by the parity tests (same kernels as the
 * forward path).  All pointers are device pointers; stream may be NULL.
 *   energon_index_maps: a1, lens [B] host -> offsets [B+1], pack_idx [T], pos [T], unpack_idx [B*S]
 *   energon_gemm: D[M,N] = A[M,K] . W[N,K]^T (+ bias[N]) (gelu if epilogue == 2); dtype F32 (SIMT)
 *     or BF16 (tcgen05, fp32 accumulate, bf16 out); bias fp32 or NULL.  epilogue 0 none, 1 bias,
 *     2 bias+gelu.  K must be a multiple of 8 in bf16 mode.
 */
ENERGON_API energon_status energon_index_maps(const int32_t* lens, int32_t batch, int32_t max_len, int32_t* offsets_d,
                                  int32_t* pack_idx_d, int32_t* pos_d, int32_t* unpack_idx_d, void* stream);
/*   energon_attention: a6 on the padded per-head layout Q, K, V, O [batch, heads, max_len, head_dim]
 *     (dtype F32: SIMT fp32; BF16: the tcgen05 / TMEM kernel for head_dim 64 / 128, SIMT otherwise);
 *     rows s >= lens[b] of O are not written. */
ENERGON_API energon_status energon_attention(int32_t dtype, const void* Q_d, const void* K_d, const void* V_d, void* O_d,
                                             const int32_t* lens, int32_t batch, int32_t heads, int32_t max_len,
                                             int32_t head_dim, int32_t causal, void* stream);
/*
 * Standalone layout kernels of the paper's two fused transpose + pad kernels (sec 4.3)
 * and of the final rebuild of padding.  Pure index + copy work: results are bit-exact
 * (a byte permutation; fp32 -> bf16 output rounds to nearest even).  Device pointers; dtype F32 or
 * BF16 is the element type of every activation argument; index maps as energon_index_maps writes them.
 *   energon_unpack_qkv (a5, "rebuild padding"): QKV [T, 3*hk*d] packed rows, columns q | k | v, each
 *     head-major then d -> Q, K, V [B, hk, S, d] at cell pack_idx[t] = b*S + s
 *     (pack_idx NULL: identity, row t is cell t).  Pad rows of Q / K / V are not written.
 *   energon_repack (a7, "remove padding"): O [B, hk, S, d] -> C [T, hk*d], row t from cell pack_idx[t];
 *     with pack_idx NULL (padded A/B mode, T = B*S) row t is cell t and cells with unpack_idx[t] < 0
 *     are written as 0.
 *   energon_final_unpack (a13): out [cells, H] (cells = B*S, out_dtype) = LN(X[unpack_idx[cell]]) with
 *     gamma / beta and eps when apply_ln, else the fp32 row itself; cells with unpack_idx < 0 are
 *     exactly 0.  X is fp32 [T, H], H a multiple of 4 and <= 12288.
 * Errors: ENERGON_ERR_ARG for NULL pointers / bad sizes / dtype, ENERGON_ERR_CUDA on a launch error.
 */
ENERGON_API energon_status energon_unpack_qkv(int32_t dtype, const void* QKV_d, const int32_t* pack_idx_d, int32_t T,
                                              int32_t max_len, int32_t heads, int32_t head_dim, void* Q_d, void* K_d,
                                              void* V_d, void* stream);
ENERGON_API energon_status energon_repack(int32_t dtype, const void* O_d, const int32_t* pack_idx_d,
                                          const int32_t* unpack_idx_d, int32_t T, int32_t max_len, int32_t heads,
                                          int32_t head_dim, void* C_d, void* stream);
ENERGON_API energon_status energon_final_unpack(int32_t out_dtype, const float* X_d, const int32_t* unpack_idx_d,
                                                int32_t cells, int32_t hidden, const float* ln_g_d, const float* ln_b_d,
                                                float ln_eps, int32_t apply_ln, void* out_d, void* stream);
ENERGON_API energon_status energon_gemm(int32_t dtype, const void* A_d, const void* W_d, const float* bias_d, void* D_d,
                            int32_t M, int32_t N, int32_t K, int32_t epilogue, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ENERGON_H */

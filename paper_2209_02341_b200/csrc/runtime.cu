// runtime.cu -- the C ABI (include/energon.h): context, validation, weight relayout, workspace,
// NCCL TP communicator and the per-layer launch sequence of the DRCE forward pass.
//
// Per layer and rank (PAPER.md:281-293 1-D TP; PAPER.md:358-373 DRCE):
//   A   = LN1(X)                      (fused into the previous residual kernel, or the entry kernel)
//   QKV = A . Wqkv_r^T + bqkv_r       tcgen05 GEMM, packed rows                       a4
//   Q,K,V <- QKV  rebuild padding                                                      a5
//   O   = attention(Q, K, V)          padded per-head layout, pad keys/queries skipped  a6
//   Ctx <- O      remove padding                                                       a7
//   P   = Ctx . Wo_r^T                row-parallel partial                             a8
//   P   = allreduce(P)                NCCL (or in-device sum for a local group)         a9
//   X  += P + bo ; A = LN2(X)                                                          a9
//   G   = gelu(A . W1_r^T + b1_r)                                                      a10
//   P   = G . W2_r^T ; P = allreduce(P)                                                a11, a12
//   X  += P + b2 ; A = LN1'(X)                                                         a12
// and once per batch: index maps (a1), embed+pack+LN1 (a2, a3), final LN + unpack (a13).
#include <nccl.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/energon.h"
#include "kernels.h"

using namespace energon;

namespace energon {
bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ENERGON_NO_PDL");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}
}  // namespace energon

namespace {

thread_local std::string g_last_error;

constexpr int kNumBoxes = 5;
const int kBoxes[kNumBoxes] = {256, 128, 96, 64, 112};
int box_slot(int box) { return box == 256 ? 0 : box == 128 ? 1 : box == 96 ? 2 : box == 112 ? 4 : 3; }

struct LayerDev {
  void *wqkv = nullptr, *wo = nullptr, *w1 = nullptr, *w2 = nullptr;  // [N, K] row-major (K-major operands)
  float *bqkv = nullptr, *bo = nullptr, *b1 = nullptr, *b2 = nullptr;
  float *ln1g = nullptr, *ln1b = nullptr, *ln2g = nullptr, *ln2b = nullptr;
  CUtensorMap tm_qkv[kNumBoxes], tm_o[kNumBoxes], tm_1[kNumBoxes], tm_2[kNumBoxes];  // W row box 256 / 128 / 96 / 64 / 112 (box_slot())
  bool loaded = false;
};

// PMEP state of one context (energon_offload_layers)
struct Pmep {
  std::vector<int> layers;       // off-device layer ids, ascending
  std::vector<int> index;        // layer -> position in `layers`, or -1 (resident)
  std::vector<void*> pool;       // per off-device layer: [wqkv | wo | w1 | w2] in pinned host or peer memory
  int pool_kind = 0, peer = -1;
  size_t bytes = 0;              // matrix bytes of one layer
  std::vector<LayerDev> slots;   // staging: matrices + tensor maps of one layer each
  std::vector<void*> slot_buf;
  std::vector<cudaEvent_t> fetched, freed;
  cudaStream_t copy = nullptr;
};

}  // namespace

struct energon_ctx {
  energon_config cfg;
  int k = 1, r = 0, H = 0, h = 0, d = 0, F = 0, Hk = 0, hk = 0, Fk = 0, V = 0;
  bool bf16 = false;
  size_t act = 4;  // bytes per activation element
  ncclComm_t nccl = nullptr;
  bool local_group = false;
  // P2P TP exchange (cfg.comm == ENERGON_COMM_P2P): X | A | P live in one IPC-exportable region
  bool p2p = false, p2p_connected = false;
  void* region = nullptr;
  int64_t off_X = 0, off_A = 0, off_P = 0;
  PeerSet peers{};
  std::vector<void*> ipc_opened;
  uint64_t epoch = 0;
  // GEMM -> reduce-scatter fused: slots [k][slot_rows][H] in every region receive the peers' partials
  int64_t off_S = 0;
  int slot_rows = 0;
  ShardStore shard{};
  ShardStore shard_rpr{};  // `shard` with this forward's rows per rank
  bool fuse = true;  // fused a5 / a7 (ENERGON_NO_FUSE=1 disables, for A/B and tests)
  bool ln_fuse = false;  // N3 (ENERGON_OPT_LN_FUSE): LN1 / LN2 applied in the QKV / MLP-up GEMM prologues
  float2* ln_stats = nullptr;  // [R] row (mean, rstd) of the last LayerNorm input, for the fused prologue
  // a5 by TMA: 3-D store maps of Q / K / V for the current (B, S) (make_qkv_store_maps), rebuilt when they change
  CUtensorMap qkv_maps[3];
  int qkv_maps_B = 0, qkv_maps_S = 0;
  bool qkv_maps_ok = false;
  bool sp = true;    // k > 1: sequence-parallel schedule (reduce-scatter / LN on own rows / all-gather)
  bool ring = false; // local group: NCCL ring numerics in the in-device reductions (ENERGON_OPT_RING_NUMERICS)
  // CUDA-graph cache (ENERGON_OPT_GRAPH): whole forwards captured on cap_stream, replayed on the caller's
  struct GraphEntry {
    std::vector<int64_t> key;
    cudaGraph_t graph = nullptr;       // kept: its index-maps nodes are updated in `exec` on every replay
    cudaGraphExec_t exec = nullptr;
    std::vector<cudaGraphNode_t> imap_node;  // per context of the group: its index-maps kernel node
    std::vector<cudaKernelNodeParams> imap_kp;
    std::vector<IndexMapsArgs> imap_args;
    std::vector<energon_stats> delta;  // per context of the group: stats one forward adds
    uint64_t last_use = 0;
  };
  bool graphs = false;
  std::vector<GraphEntry> gcache;
  uint64_t gclock = 0;
  cudaStream_t cap_stream = nullptr;
  // replicated embeddings / final LN
  void* tok_emb = nullptr;
  void* pos_emb = nullptr;
  float *lnf_g = nullptr, *lnf_b = nullptr;
  bool emb_loaded = false;
  std::vector<LayerDev> layers;
  // workspace (sized from max_tokens padded rows)
  int *offsets = nullptr, *pack_idx = nullptr, *pos = nullptr, *unpack_idx = nullptr;
  int* lens_d = nullptr;           // [ENERGON_MAX_BATCH] this forward's lengths (written by the index-maps kernel)
  uint32_t* attn_work = nullptr;   // attention work list (build_attn_work)
  AttnMaps amaps;                  // cached Q / K / V tensor maps of the attention kernel
  IndexMapsArgs last_imap{};       // arguments of this context's last index-maps launch (graph parameter updates)
  double work_rows = 0;            // rows of algorithmic work (T with DRCE) for the profile's GEMM flops
  float* X = nullptr;
  void *A = nullptr, *QKV = nullptr, *Q = nullptr, *K = nullptr, *Vb = nullptr, *O = nullptr, *Ctx = nullptr,
       *P = nullptr, *G = nullptr;
  CUtensorMap tmA_A, tmA_Ctx, tmA_G;
  CUtensorMap tmD_P, tmD_G;  // TMA-store output maps of the out/down (P) and up (G) GEMMs
  int tm_rows = -1;
  Pmep pm;
  TailWs tail;              // stream-K scratch of this context's GEMMs (ordered on its forward stream)
  int* err_host = nullptr;  // mapped pinned flag written by the index-maps kernel (bad token id)
  int* err_dev = nullptr;
  cudaStream_t load_stream = nullptr;
  std::vector<void*> allocs;
  std::string err;
  std::string launch_err;  // a launcher refused (e.g. a tensor map could not be built): the forward fails
  energon_stats stats;
  // profiling (energon_set_profiling): CUDA events around every launch on the forward stream
  struct ProfRec {
    cudaEvent_t a, b;
    int cls;
    double work;
  };
  bool prof = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  size_t pool_used = 0;
  energon_profile pacc;
};

namespace {

energon_status fail(energon_ctx* c, energon_status s, const std::string& msg) {
  g_last_error = msg;
  if (c) c->err = msg;
  return s;
}

energon_status cuda_fail(energon_ctx* c, cudaError_t e, const char* where) {
  return fail(c, e == cudaErrorMemoryAllocation ? ENERGON_ERR_OOM : ENERGON_ERR_CUDA,
              std::string(where) + ": " + cudaGetErrorString(e));
}

#define CU(c, expr)                                            \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return cuda_fail((c), _e, #expr);   \
  } while (0)

template <typename T>
energon_status dalloc(energon_ctx* c, T** p, size_t bytes, int64_t* counter) {
  void* q = nullptr;
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(&q, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(c, ENERGON_ERR_OOM, "cudaMalloc(" + std::to_string(bytes) + " B) failed: " + cudaGetErrorString(e));
  }
  c->allocs.push_back(q);
  if (counter) *counter += (int64_t)bytes;
  *p = reinterpret_cast<T*>(q);
  return ENERGON_OK;
}

energon_status validate_config(const energon_config* cfg) {
  if (!cfg) return fail(nullptr, ENERGON_ERR_ARG, "cfg is NULL");
  if (cfg->num_layers < 1 || cfg->hidden < 1 || cfg->num_heads < 1 || cfg->ffn < 1 || cfg->vocab < 1 ||
      cfg->max_seq < 1 || cfg->max_tokens < 1)
    return fail(nullptr, ENERGON_ERR_CONFIG, "every size in energon_config must be >= 1");
  if (cfg->hidden % cfg->num_heads)
    return fail(nullptr, ENERGON_ERR_CONFIG, "hidden must equal num_heads * head_dim (SPEC.md:284)");
  if (cfg->tp_size < 1 || cfg->tp_size > 8 || cfg->tp_rank < 0 || cfg->tp_rank >= cfg->tp_size)
    return fail(nullptr, ENERGON_ERR_CONFIG, "tp_size must be in [1,8] and 0 <= tp_rank < tp_size");
  if (cfg->num_heads % cfg->tp_size || cfg->ffn % cfg->tp_size)
    return fail(nullptr, ENERGON_ERR_CONFIG, "num_heads and ffn must be divisible by tp_size (SPEC.md:284)");
  if (cfg->dtype != ENERGON_DTYPE_F32 && cfg->dtype != ENERGON_DTYPE_BF16)
    return fail(nullptr, ENERGON_ERR_CONFIG, "dtype must be ENERGON_DTYPE_F32 or ENERGON_DTYPE_BF16");
  if (cfg->causal != 0 && cfg->causal != 1) return fail(nullptr, ENERGON_ERR_CONFIG, "causal must be 0 or 1");
  if (cfg->drce != 0 && cfg->drce != 1) return fail(nullptr, ENERGON_ERR_CONFIG, "drce must be 0 or 1");
  if (!(cfg->ln_eps > 0.f)) return fail(nullptr, ENERGON_ERR_CONFIG, "ln_eps must be > 0");
  if (cfg->comm != ENERGON_COMM_NCCL && cfg->comm != ENERGON_COMM_P2P)
    return fail(nullptr, ENERGON_ERR_CONFIG, "comm must be ENERGON_COMM_NCCL or ENERGON_COMM_P2P");
  const int d = cfg->hidden / cfg->num_heads;
  if (cfg->hidden % 8 || d % 8 || (cfg->ffn / cfg->tp_size) % 8 || cfg->hidden > 12288)
    return fail(nullptr, ENERGON_ERR_SHAPE,
                "unsupported shape: hidden, head_dim and ffn/tp_size must be multiples of 8, hidden <= 12288");
  return ENERGON_OK;
}

energon_status setup(energon_ctx* c) {
  const energon_config& g = c->cfg;
  c->k = g.tp_size;
  c->r = g.tp_rank;
  c->H = g.hidden;
  c->h = g.num_heads;
  c->d = g.hidden / g.num_heads;
  c->F = g.ffn;
  c->V = g.vocab;
  c->Hk = c->H / c->k;
  c->hk = c->h / c->k;
  c->Fk = c->F / c->k;
  c->bf16 = g.dtype == ENERGON_DTYPE_BF16;
  c->act = c->bf16 ? 2 : 4;
  memset(&c->stats, 0, sizeof(c->stats));
  memset(&c->pacc, 0, sizeof(c->pacc));
  if (const char* e = getenv("ENERGON_NO_FUSE")) c->fuse = e[0] != '1';
  CU(c, cudaSetDevice(g.device));
  CU(c, cudaStreamCreateWithFlags(&c->load_stream, cudaStreamNonBlocking));
  CU(c, cudaHostAlloc(&c->err_host, sizeof(int), cudaHostAllocMapped));
  *c->err_host = 0;
  CU(c, cudaHostGetDevicePointer(&c->err_dev, c->err_host, 0));
  c->layers.resize(g.num_layers);
  // workspace: every buffer is sized for max_tokens rows (padded rows when drce == 0)
  // + 8 rows: the sequence-parallel schedule pads the row count to a multiple of k (<= 8)
  const size_t R = (size_t)g.max_tokens + 8, a = c->act;
  int64_t* ws = &c->stats.workspace_bytes;
  energon_status s;
  c->p2p = g.comm == ENERGON_COMM_P2P && c->k > 1 && !c->local_group;
  if (c->p2p) {
    // one region [flags | X | A | P] (same offsets on every rank) that peers map by CUDA IPC
    auto al = [](int64_t x) { return (x + 255) & ~(int64_t)255; };
    c->off_X = P2P_FLAG_BYTES;
    c->off_A = al(c->off_X + (int64_t)sizeof(float) * R * c->H);
    c->off_P = al(c->off_A + (int64_t)a * R * c->H);
    c->slot_rows = (int)((((int64_t)R + c->k - 1) / c->k + 31) / 32 * 32);  // rows per rank, multiple of 32
    c->off_S = al(c->off_P + (int64_t)a * R * c->H);
    const int64_t bytes = al(c->off_S + (int64_t)a * c->k * c->slot_rows * c->H);
    if ((s = dalloc(c, reinterpret_cast<char**>(&c->region), (size_t)bytes, ws))) return s;
    CU(c, cudaMemset(c->region, 0, (size_t)bytes));
    c->X = reinterpret_cast<float*>(static_cast<char*>(c->region) + c->off_X);
    c->A = static_cast<char*>(c->region) + c->off_A;
    c->P = static_cast<char*>(c->region) + c->off_P;
  } else if ((s = dalloc(c, &c->X, sizeof(float) * R * c->H, ws)) || (s = dalloc(c, &c->A, a * R * c->H, ws)) ||
             (s = dalloc(c, &c->P, a * R * c->H, ws))) {
    return s;
  }
  if ((s = dalloc(c, &c->offsets, sizeof(int) * (ENERGON_MAX_BATCH + 1), ws)) ||
      (s = dalloc(c, &c->pack_idx, sizeof(int) * R, ws)) || (s = dalloc(c, &c->pos, sizeof(int) * R, ws)) ||
      (s = dalloc(c, &c->unpack_idx, sizeof(int) * R, ws)) || (s = dalloc(c, &c->QKV, a * R * 3 * c->Hk, ws)) ||
      (s = dalloc(c, &c->lens_d, sizeof(int) * ENERGON_MAX_BATCH, ws)) ||
      (s = dalloc(c, &c->attn_work, sizeof(uint32_t) * (2 + ENERGON_MAX_BATCH + R / 64), ws)) ||
      (s = dalloc(c, &c->ln_stats, sizeof(float2) * R, ws)) ||
      (s = dalloc(c, &c->Q, a * R * c->Hk, ws)) || (s = dalloc(c, &c->K, a * R * c->Hk, ws)) ||
      (s = dalloc(c, &c->Vb, a * R * c->Hk, ws)) || (s = dalloc(c, &c->O, a * R * c->Hk, ws)) ||
      (s = dalloc(c, &c->Ctx, a * R * c->Hk, ws)) || (s = dalloc(c, &c->G, a * R * c->Fk, ws)))
    return s;
  // zero every activation buffer once: rows a schedule reads but never writes (sequence-parallel
  // padding rows, unwritten Ctx rows) stay finite
  if (c->bf16 && !tail_ws_alloc(&c->tail)) return fail(c, ENERGON_ERR_OOM, "stream-K workspace allocation failed");
  for (void* p : c->allocs) CU(c, cudaMemset(p, 0, 16));
  CU(c, cudaMemset(c->X, 0, sizeof(float) * R * c->H));
  CU(c, cudaMemset(c->A, 0, a * R * c->H));
  CU(c, cudaMemset(c->P, 0, a * R * c->H));
  CU(c, cudaMemset(c->Ctx, 0, a * R * c->Hk));
  CU(c, cudaDeviceSynchronize());
  return ENERGON_OK;
}

void release(energon_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->cfg.device);
  cudaDeviceSynchronize();
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  c->ipc_opened.clear();
  for (void* p : c->allocs) cudaFree(p);
  c->allocs.clear();
  tail_ws_free(&c->tail);
  for (void* p : c->pm.pool) {
    if (c->pm.pool_kind == 0) cudaFreeHost(p);
    else {
      cudaSetDevice(c->pm.peer);
      cudaFree(p);
      cudaSetDevice(c->cfg.device);
    }
  }
  for (void* p : c->pm.slot_buf) cudaFree(p);
  for (cudaEvent_t e : c->pm.fetched) cudaEventDestroy(e);
  for (cudaEvent_t e : c->pm.freed) cudaEventDestroy(e);
  if (c->pm.copy) cudaStreamDestroy(c->pm.copy);
  if (c->err_host) cudaFreeHost(c->err_host);
  if (c->load_stream) cudaStreamDestroy(c->load_stream);
  for (auto& g : c->gcache) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
  }
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  for (cudaEvent_t e : c->pool) cudaEventDestroy(e);
  if (c->nccl) ncclCommDestroy(c->nccl);
  delete c;
}

// ----------------------------------------------------------------------------- weight loading
template <typename Src, typename Dst>
energon_status put_matrix_t(energon_ctx* c, const void* src, bool on_dev, int64_t src_rows, int64_t ld, int64_t row0,
                            int64_t col0, int N, int K, void* dst, int64_t dst_row0) {
  const Src* s = reinterpret_cast<const Src*>(src);
  void* stage = nullptr;
  if (!on_dev) {
    const size_t bytes = sizeof(Src) * (size_t)src_rows * (size_t)ld;
    CU(c, cudaMalloc(&stage, bytes));
    CU(c, cudaMemcpyAsync(stage, src, bytes, cudaMemcpyHostToDevice, c->load_stream));
    s = reinterpret_cast<const Src*>(stage);
  }
  launch_relayout<Src, Dst>(s, ld, row0, col0, N, K, reinterpret_cast<Dst*>(dst), K, dst_row0, c->load_stream);
  c->stats.kernel_launches++;
  CU(c, cudaGetLastError());
  if (stage) {
    CU(c, cudaStreamSynchronize(c->load_stream));
    CU(c, cudaFree(stage));
  }
  return ENERGON_OK;
}

template <typename Src, typename Dst>
energon_status put_vector_t(energon_ctx* c, const void* src, bool on_dev, int64_t src_n, int64_t off, int N, Dst* dst) {
  const Src* s = reinterpret_cast<const Src*>(src);
  void* stage = nullptr;
  if (!on_dev) {
    CU(c, cudaMalloc(&stage, sizeof(Src) * (size_t)src_n));
    CU(c, cudaMemcpyAsync(stage, src, sizeof(Src) * (size_t)src_n, cudaMemcpyHostToDevice, c->load_stream));
    s = reinterpret_cast<const Src*>(stage);
  }
  launch_convert_vec<Src, Dst>(s, off, N, dst, c->load_stream);
  c->stats.kernel_launches++;
  CU(c, cudaGetLastError());
  if (stage) {
    CU(c, cudaStreamSynchronize(c->load_stream));
    CU(c, cudaFree(stage));
  }
  return ENERGON_OK;
}

// dispatch on (src dtype, ctx activation dtype)
energon_status put_matrix(energon_ctx* c, int sd, const void* src, bool on_dev, int64_t src_rows, int64_t ld,
                          int64_t row0, int64_t col0, int N, int K, void* dst, int64_t dst_row0) {
  if (c->bf16) {
    if (sd == ENERGON_DTYPE_F64) return put_matrix_t<double, bf16>(c, src, on_dev, src_rows, ld, row0, col0, N, K, dst, dst_row0);
    if (sd == ENERGON_DTYPE_F32) return put_matrix_t<float, bf16>(c, src, on_dev, src_rows, ld, row0, col0, N, K, dst, dst_row0);
    return put_matrix_t<bf16, bf16>(c, src, on_dev, src_rows, ld, row0, col0, N, K, dst, dst_row0);
  }
  if (sd == ENERGON_DTYPE_F64) return put_matrix_t<double, float>(c, src, on_dev, src_rows, ld, row0, col0, N, K, dst, dst_row0);
  if (sd == ENERGON_DTYPE_F32) return put_matrix_t<float, float>(c, src, on_dev, src_rows, ld, row0, col0, N, K, dst, dst_row0);
  return put_matrix_t<bf16, float>(c, src, on_dev, src_rows, ld, row0, col0, N, K, dst, dst_row0);
}

template <typename Dst>
energon_status put_vector(energon_ctx* c, int sd, const void* src, bool on_dev, int64_t src_n, int64_t off, int N,
                          Dst* dst) {
  if (sd == ENERGON_DTYPE_F64) return put_vector_t<double, Dst>(c, src, on_dev, src_n, off, N, dst);
  if (sd == ENERGON_DTYPE_F32) return put_vector_t<float, Dst>(c, src, on_dev, src_n, off, N, dst);
  return put_vector_t<bf16, Dst>(c, src, on_dev, src_n, off, N, dst);
}

// ----------------------------------------------------------------------------- profiling scopes
enum { P_GEMM = 0, P_ATTN = 1, P_MEM = 2, P_COMM = 3 };

cudaEvent_t next_event(energon_ctx* c) {
  if (c->pool_used == c->pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->pool.push_back(e);
  }
  return c->pool[c->pool_used++];
}

// ENERGON_DEBUG_SYNC=1 (diagnostics): wait for every launch to finish (eager runs only), and abort with
// the launch class after 20 s -- names the kernel of a device-side hang
bool debug_sync() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ENERGON_DEBUG_SYNC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

void debug_wait(cudaStream_t st, int cls, double work) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
  static long n = 0;
  ++n;
  for (int i = 0; i < 20000; ++i) {
    const cudaError_t e = cudaStreamQuery(st);
    if (e != cudaErrorNotReady) return;
    usleep(1000);
  }
  fprintf(stderr, "[energon] device hang: launch #%ld class %d (0 gemm, 1 attn, 2 mem, 3 comm), work %.3g\n", n, cls,
          work);
  fflush(stderr);
  abort();
}

struct Prof {
  energon_ctx* c;
  cudaStream_t st;
  int cls;
  double work;
  cudaEvent_t a = nullptr;
  Prof(energon_ctx* c_, cudaStream_t st_, int cls_, double work_) : c(c_), st(st_), cls(cls_), work(work_) {
    if (c->prof) {
      a = next_event(c);
      cudaEventRecord(a, st);
    }
  }
  ~Prof() {
    if (debug_sync()) debug_wait(st, cls, work);
    if (c->prof) {
      cudaEvent_t b = next_event(c);
      cudaEventRecord(b, st);
      c->recs.push_back({a, b, cls, work});
    }
  }
};

// ----------------------------------------------------------------------------- forward
struct Call {
  const int32_t* tokens;  // token entry (energon_forward)
  const float* x_in;      // hidden entry (energon_forward_hidden)
  const int32_t* lens;
  int B, S, l0, l1, final_ln;
  void* out;
  bool out_f32;
  cudaStream_t st;
  bool x_packed = false;    // x_in holds the linears' rows ([T,H] packed with DRCE) -- a pipeline stage input
  bool out_packed = false;  // out receives the fp32 residual stream rows [rows,H] -- a pipeline stage output
};

energon_status check_ready(energon_ctx* c, const Call& a) {
  // a pipeline stage needs only its own layers, and the embeddings only at the ends of the pipeline
  if ((a.tokens || !a.out_packed) && !c->emb_loaded) return fail(c, ENERGON_ERR_NOT_LOADED, "embeddings not loaded");
  if (a.l0 < 0 || a.l1 > (int)c->layers.size() || a.l0 > a.l1) return fail(c, ENERGON_ERR_ARG, "bad layer range");
  for (int l = a.l0; l < a.l1; ++l)
    if (!c->layers[l].loaded) return fail(c, ENERGON_ERR_NOT_LOADED, "layer " + std::to_string(l) + " not loaded");
  // (a bad token id raised on the device is NOT checked here: the flag is written asynchronously, so
  // gating the SPMD enqueue on it could let one rank skip a forward its peers run -- a distributed hang;
  // it surfaces on energon_sync, where every rank of the group sees the same flag)
  if (c->p2p && !c->p2p_connected) return fail(c, ENERGON_ERR_NOT_LOADED, "P2P peers not connected (energon_p2p_connect)");
  return ENERGON_OK;
}

energon_status validate_call(energon_ctx* c, const Call& a, int64_t* T_out) {
  if (!a.lens || !a.out) return fail(c, ENERGON_ERR_ARG, "seq_lens / out must not be NULL");
  if (!a.tokens && !a.x_in) return fail(c, ENERGON_ERR_ARG, "tokens must not be NULL");
  if (a.B < 1) return fail(c, ENERGON_ERR_ARG, "batch must be >= 1");
  if (a.B > ENERGON_MAX_BATCH) return fail(c, ENERGON_ERR_CAPACITY, "batch exceeds ENERGON_MAX_BATCH");
  if (a.S < 1 || a.S > c->cfg.max_seq)
    return fail(c, ENERGON_ERR_LENGTH, "max_len must be in [1, max_seq] (SPEC.md:133)");
  if ((int64_t)a.B * a.S > c->cfg.max_tokens)
    return fail(c, ENERGON_ERR_CAPACITY, "batch * max_len exceeds max_tokens");
  if (a.l0 < 0 || a.l1 > c->cfg.num_layers || a.l0 > a.l1) return fail(c, ENERGON_ERR_ARG, "bad layer range");
  int64_t T = 0;
  for (int b = 0; b < a.B; ++b) {
    if (a.lens[b] < 1 || a.lens[b] > a.S)
      return fail(c, ENERGON_ERR_LENGTH,
                  "seq_lens[" + std::to_string(b) + "]=" + std::to_string(a.lens[b]) + " not in [1, max_len]");
    T += a.lens[b];
  }
  *T_out = T;
  return ENERGON_OK;
}

// ----------------------------------------------------------------------------- TP exchanges
// "accumulated by communications": one reduction per pair of linears.  AR schedule:
// allreduce of the packed [rows, H] partial.  SP schedule (k > 1, default): reduce-scatter of the
// partial over row shards of rpr rows, so each rank adds bias + residual and normalises only its
// rows, then all-gather of the normalised rows for the next column-parallel GEMM -- the same bytes
// on the wire as the allreduce, 1/k of the memory-bound work per rank.
template <typename Act>
energon_status tp_reduce(energon_ctx** cs, int n, int rows, int rpr, bool sp, cudaStream_t st) {
  energon_ctx* c0 = cs[0];
  if (c0->k == 1) return ENERGON_OK;
  const ncclDataType_t dt = c0->bf16 ? ncclBfloat16 : ncclFloat;
  const size_t count = sp ? (size_t)rpr * c0->k * c0->H : (size_t)rows * c0->H;
  Prof p(c0, st, P_COMM, (double)count * c0->act);
  if (c0->local_group) {
    PtrList pl;
    for (int i = 0; i < n; ++i) pl.p[i] = cs[i]->P;
    if (sp) launch_local_reduce_scatter<Act>(pl, n, (int64_t)rpr * c0->H, c0->ring ? 1 : 0, st);
    else launch_local_allreduce<Act>(pl, n, (int64_t)count, c0->ring ? 1 : 0, st);
    c0->stats.kernel_launches++;
  } else {
    ncclResult_t e;
    if (sp) {
      Act* P = reinterpret_cast<Act*>(c0->P);
      e = ncclReduceScatter(P, P + (size_t)c0->r * rpr * c0->H, (size_t)rpr * c0->H, dt, ncclSum, c0->nccl, st);
    } else {
      e = ncclAllReduce(c0->P, c0->P, count, dt, ncclSum, c0->nccl, st);
    }
    if (e != ncclSuccess) return fail(c0, ENERGON_ERR_NCCL, std::string("NCCL reduction: ") + ncclGetErrorString(e));
  }
  for (int i = 0; i < n; ++i) cs[i]->stats.allreduce_calls++;
  return ENERGON_OK;
}

// all-gather of each rank's rpr-row shard of buf (A: activation dtype, or X: fp32), in place
template <typename T>
energon_status tp_gather(energon_ctx** cs, int n, int rpr, bool x_buf, cudaStream_t st) {
  energon_ctx* c0 = cs[0];
  const size_t elems = (size_t)rpr * c0->H;
  Prof p(c0, st, P_COMM, (double)elems * sizeof(T) * (c0->k - 1));
  if (c0->local_group) {
    PtrList pl;
    for (int i = 0; i < n; ++i) pl.p[i] = x_buf ? (void*)cs[i]->X : cs[i]->A;
    launch_local_all_gather(pl, n, (int64_t)(elems * sizeof(T)), st);
    c0->stats.kernel_launches++;
  } else {
    T* b = reinterpret_cast<T*>(x_buf ? (void*)c0->X : c0->A);
    const ncclDataType_t dt = sizeof(T) == 4 ? ncclFloat : ncclBfloat16;
    ncclResult_t e = ncclAllGather(b + (size_t)c0->r * elems, b, elems, dt, c0->nccl, st);
    if (e != ncclSuccess) return fail(c0, ENERGON_ERR_NCCL, std::string("ncclAllGather: ") + ncclGetErrorString(e));
  }
  return ENERGON_OK;
}

// ---- P2P exchange (cfg.comm == ENERGON_COMM_P2P; kernels_misc.cu describes the protocol)
template <typename Act>
void p2p_exchange(energon_ctx* c, int rows, int rpr, const float* bias, const float* g, const float* b, bool write_A,
                  cudaStream_t st, bool fused_rs) {
  const int r0 = std::min(rows, c->r * rpr), sn = std::max(0, std::min(rows, (c->r + 1) * rpr) - c->r * rpr);
  const uint64_t e = ++c->epoch;
  {
    Prof p(c, st, P_COMM, 0.0);
    launch_p2p_flag(c->peers, c->k, c->r, P2P_READY, e, 1, st);
  }
  {
    // bytes over NVLink + local: k partial rows read, (write_A ? k : 0) LN rows stored, X read + written
    Prof p(c, st, P_COMM, (double)sn * c->H * (c->k * sizeof(Act) + (write_A ? c->k * sizeof(Act) : 0) + 8.0));
    // fused: the partials of this rank's rows are already in its own slots (local reads only)
    launch_p2p_reduce_ln<Act>(c->peers, c->k, c->r, c->off_X, c->off_A, fused_rs ? c->off_S : c->off_P, r0, sn, c->H,
                              bias, g, b, c->cfg.ln_eps, write_A ? 1 : 0, e, st, fused_rs ? c->slot_rows : 0);
  }
  {
    Prof p(c, st, P_COMM, 0.0);
    launch_p2p_flag(c->peers, c->k, c->r, P2P_DELIVERED, e, 0, st);
  }
  c->stats.kernel_launches += 3;
  c->stats.allreduce_calls++;
  if (fused_rs) c->stats.fused_exchanges++;
}

// all-gather of this rank's row shard of the buffer at `off` (row_bytes per row) by pushing to peers
void p2p_gather(energon_ctx* c, int rows, int rpr, int64_t off, int64_t row_bytes, cudaStream_t st) {
  const int r0 = std::min(rows, c->r * rpr), sn = std::max(0, std::min(rows, (c->r + 1) * rpr) - c->r * rpr);
  const uint64_t e = ++c->epoch;
  {
    Prof p(c, st, P_COMM, (double)sn * row_bytes * (c->k - 1));
    launch_p2p_push_rows(c->peers, c->k, c->r, off, r0, sn, row_bytes, e, st);
  }
  {
    Prof p(c, st, P_COMM, 0.0);
    launch_p2p_flag(c->peers, c->k, c->r, P2P_DELIVERED, e, 0, st);
  }
  c->stats.kernel_launches += 2;
}

template <typename Act>
void gemm(energon_ctx* c, const CUtensorMap& tmA, const CUtensorMap* tmB, const void* A, const void* W,
          const float* bias, void* D, int M, int N, int K, int epi, cudaStream_t st, const QkvScatter* qs = nullptr,
          const CUtensorMap* tmD = nullptr, const ShardStore* shard = nullptr) {
  Prof p(c, st, P_GEMM, 2.0 * c->work_rows * N * K);  // algorithmic: the valid rows only
  if constexpr (sizeof(Act) == 2) {
    const int code = tc_pick_bn(M, N, K);
    if (!launch_gemm_tc(tmA, tmB[box_slot(tc_w_box(code))], code, bias, reinterpret_cast<bf16*>(D), M, N, K, epi, st,
                        qs, tmD, &c->tail, shard))
      c->launch_err = "GEMM launch refused: output tensor map could not be built";
  } else {
    launch_gemm_f32(reinterpret_cast<const float*>(A), reinterpret_cast<const float*>(W), bias,
                    reinterpret_cast<float*>(D), M, N, K, epi, st);
  }
  c->stats.kernel_launches++;
}

// N3: LN(X) built in the GEMM prologue (QKV with LN1, MLP-up with LN2); bf16, TP = 1 only
void gemm_ln(energon_ctx* c, const CUtensorMap* tmB, const float* g, const float* b, const float* bias, void* D, int M,
             int N, int epi, cudaStream_t st, const QkvScatter* qs = nullptr) {
  Prof p(c, st, P_GEMM, 2.0 * c->work_rows * N * c->H);
  if (!launch_gemm_ln(tmB[box_slot(256)], c->X, c->ln_stats, g, b, bias, reinterpret_cast<bf16*>(D), M, N, c->H, epi, st,
                      qs))
    c->launch_err = "LN-prologue GEMM refused: hidden % 64 != 0";
  c->stats.kernel_launches++;
}

// ----------------------------------------------------------------------------- PMEP prefetch
// Copy off-device layer `layer` (the j-th off-device layer of this forward) into staging slot
// j % slots on the copy stream, after the slot's previous occupant finished computing.
void pmep_fetch(energon_ctx* c, int j, int layer) {
  Pmep& pm = c->pm;
  const int s = j % (int)pm.slots.size();
  const int i = pm.index[layer];
  cudaStreamWaitEvent(pm.copy, pm.freed[s], 0);
  if (pm.pool_kind == 0)
    cudaMemcpyAsync(pm.slot_buf[s], pm.pool[i], pm.bytes, cudaMemcpyHostToDevice, pm.copy);
  else
    cudaMemcpyPeerAsync(pm.slot_buf[s], c->cfg.device, pm.pool[i], pm.peer, pm.bytes, pm.copy);
  cudaEventRecord(pm.fetched[s], pm.copy);
  c->stats.prefetch_bytes += (int64_t)pm.bytes;
}

int bucket_rows(const energon_ctx* c, int64_t T) {
  const int64_t b = (T + 127) / 128 * 128;
  return (int)std::min<int64_t>(b, std::max<int64_t>(T, c->cfg.max_tokens));
}

template <typename Act>
energon_status forward_t(energon_ctx** cs, int n, const Call& a, int64_t T) {
  cudaStream_t st = a.st;
  energon_ctx* c0 = cs[0];
  const energon_config& g = c0->cfg;
  const bool drce = g.drce == 1;
  // DRCE: the linears run on T packed rows rounded up to a bucket of 128 (<= max_tokens), so that one
  // recorded CUDA graph serves every batch of the bucket (the bucket rows past T are marked -1 in
  // pack_idx and carry zeros / finite values nobody reads); a 256-row GEMM tile count never changes
  const int rows = drce ? bucket_rows(c0, T) : a.B * a.S;
  const float eps = g.ln_eps;
  const double act = (double)sizeof(Act), H = c0->H, Hk = c0->Hk;
  // Fused forms of the paper's two layout kernels on the bf16 tensor-core path:
  // a5 inside the QKV GEMM epilogue, a7 inside the attention epilogue (DRCE mode only; the padded
  // A/B mode keeps the standalone repack because it must zero the pad query rows).
  const bool fuse_a5 = sizeof(Act) == 2 && c0->fuse && (c0->d == 64 || c0->d == 128);
  const bool fuse_a7 = fuse_a5 && drce;
  // TP schedule: row shard [r0, r0 + sn) of each rank (the whole range without sequence parallelism)
  const bool p2p = c0->p2p;  // one context per process, peers over CUDA IPC (sequence-parallel schedule)
  const bool sp = c0->k > 1 && (c0->sp || p2p);
  // P2P: shards of a multiple of 32 rows, so the fused GEMM -> reduce-scatter's 32-row store boxes never
  // straddle two owners (the trailing ranks may own fewer rows, or none)
  const int rpr = !sp ? rows : p2p ? ((rows + c0->k - 1) / c0->k + 31) / 32 * 32 : (rows + c0->k - 1) / c0->k;
  // the row-parallel GEMMs route their rows to the owners' slots when the 2-CTA tcgen05 kernel runs them
  const bool fused_rs = p2p && sizeof(Act) == 2 && c0->shard.k > 0 && tc_pick_bn(rows, c0->H) > 1000;
  if (fused_rs) {
    c0->shard_rpr = c0->shard;
    c0->shard_rpr.rpr = rpr;
  }
  auto shard0 = [&](const energon_ctx* c) { return sp ? std::min(rows, c->r * rpr) : 0; };
  auto shardn = [&](const energon_ctx* c) { return sp ? std::max(0, std::min(rows, (c->r + 1) * rpr) - c->r * rpr) : rows; };
  // PMEP: the off-device layers of this forward in execution order, per context
  std::vector<std::vector<int>> off_order(n);
  std::vector<int> off_next(n, 0), off_slot(n, -1);
  for (int i = 0; i < n; ++i) {
    energon_ctx* c = cs[i];
    if (c->pm.layers.empty()) continue;
    for (int l : c->pm.layers)
      if (l >= a.l0 && l < a.l1) off_order[i].push_back(l);
    const int ns = (int)c->pm.slots.size();
    for (int j = 0; j < (int)off_order[i].size() && j < ns; ++j) pmep_fetch(c, j, off_order[i][j]);
  }
  // the weights a layer computes with: its own, or the staging slot its off-device copy lands in
  auto weights = [&](int i, int l) -> const LayerDev& {
    energon_ctx* c = cs[i];
    if (c->pm.layers.empty() || c->pm.index[l] < 0) return c->layers[l];
    return c->pm.slots[off_slot[i]];
  };
  LensParam lp;
  double allowed = 0.0;  // sum over sequences of visible (query, key) pairs
  for (int b = 0; b < a.B; ++b) {
    lp.lens[b] = a.lens[b];
    const double L = a.lens[b];
    allowed += g.causal ? L * (L + 1) / 2 : L * L;
  }

  for (int i = 0; i < n; ++i) {
    energon_ctx* c = cs[i];
    c->stats.last_tokens = T;
    c->stats.last_rows = rows;
    c->work_rows = drce ? (double)T : (double)rows;
    {
      Prof p(c, st, P_MEM, 4.0 * (a.B + 1) + 8.0 * T + 4.0 * a.B * a.S);
      IndexMapsArgs ia{a.B, a.S, drce ? rows : (int)T, c->offsets, c->pack_idx, c->pos, c->unpack_idx, a.tokens, c->V,
                       c->err_dev, c->lens_d, c->attn_work, g.causal, attention_tile_bm(), attention_tile_bn()};
      launch_index_maps(lp, ia, st);
      c->last_imap = ia;
    }
    c->stats.kernel_launches++;
    if (sizeof(Act) == 2 && c->tm_rows != rows) {
      if (!make_tmap_kmajor(&c->tmA_A, c->A, rows, c->H, 128) ||
          !make_tmap_kmajor(&c->tmA_Ctx, c->Ctx, rows, c->Hk, 128) ||
          !make_tmap_kmajor(&c->tmA_G, c->G, rows, c->Fk, 128) || !make_tmap_store(&c->tmD_P, c->P, rows, c->H) ||
          !make_tmap_store(&c->tmD_G, c->G, rows, c->Fk))
        return fail(c, ENERGON_ERR_CUDA, "cuTensorMapEncodeTiled failed for an activation operand");
      c->tm_rows = rows;
    }
    const int* pidx = drce ? c->pack_idx : nullptr;
    const LayerDev& L0 = c->layers[a.l0 < g.num_layers ? a.l0 : 0];
    const float* g1 = a.l0 < a.l1 ? L0.ln1g : c->lnf_g;
    const float* b1 = a.l0 < a.l1 ? L0.ln1b : c->lnf_b;
    {
      // reads: ids + 2 embedding rows (or one fp32 row); writes: X (fp32) + A -- this rank's rows
      const int r0 = shard0(c), sn = shardn(c);
      Prof p(c, st, P_MEM, a.tokens ? sn * (4.0 + H * (2 * act + 4 + act)) : sn * H * (4 + 4 + act));
      Act* A0 = c->ln_fuse ? nullptr : reinterpret_cast<Act*>(c->A);  // N3: statistics only, LN in the QKV prologue
      float2* st0 = c->ln_fuse ? c->ln_stats : nullptr;
      if (a.tokens)
        launch_embed_ln<Act>(a.tokens, pidx, c->unpack_idx, r0, sn, a.S, c->V, c->H,
                             reinterpret_cast<const Act*>(c->tok_emb), reinterpret_cast<const Act*>(c->pos_emb), g1, b1,
                             eps, c->X, A0, st, st0);
      else
        launch_gather_ln<Act>(a.x_in, a.x_packed ? nullptr : pidx, drce ? c->offsets + a.B : nullptr, r0, sn, c->H, g1,
                              b1, eps, c->X, A0, st, st0);
    }
    c->stats.kernel_launches++;
  }
  if (p2p) {
    p2p_gather(c0, rows, rpr, c0->off_A, (int64_t)sizeof(Act) * c0->H, st);
  } else if (sp) {
    energon_status s = tp_gather<Act>(cs, n, rpr, false, st);
    if (s) return s;
  }

  for (int l = a.l0; l < a.l1; ++l) {
    // ---- attention module: column-parallel QKV, local heads, row-parallel out-proj
    for (int i = 0; i < n; ++i) {
      energon_ctx* c = cs[i];
      if (!c->pm.layers.empty() && c->pm.index[l] >= 0) {  // off-device layer: wait for its prefetch
        const int j = off_next[i]++;
        off_slot[i] = j % (int)c->pm.slots.size();
        cudaStreamWaitEvent(st, c->pm.fetched[off_slot[i]], 0);
      }
      const LayerDev& W = weights(i, l);  // matrices + tensor maps (resident or staged)
      const LayerDev& L = c->layers[l];   // biases, LN vectors (always resident)
      const int* pidx = drce ? c->pack_idx : nullptr;
      if (fuse_a5) {
        // a4 + a5: the QKV epilogue scatters straight into the padded per-head Q, K, V
        if (c->qkv_maps_B != a.B || c->qkv_maps_S != a.S) {
          c->qkv_maps_ok = !getenv("ENERGON_NO_QKV_TMA") &&
                           make_qkv_store_maps(c->qkv_maps, reinterpret_cast<const bf16*>(c->Q),
                                               reinterpret_cast<const bf16*>(c->K), reinterpret_cast<const bf16*>(c->Vb),
                                               a.B, c->hk, a.S, c->d);
          c->qkv_maps_B = a.B;
          c->qkv_maps_S = a.S;
        }
        QkvScatter qs{pidx, reinterpret_cast<bf16*>(c->Q), reinterpret_cast<bf16*>(c->K),
                      reinterpret_cast<bf16*>(c->Vb), a.S, c->hk, c->d, c->qkv_maps_ok ? c->qkv_maps : nullptr};
        if (c->ln_fuse)
          gemm_ln(c, W.tm_qkv, L.ln1g, L.ln1b, L.bqkv, nullptr, rows, 3 * c->Hk, EPI_BIAS_QKV, st, &qs);
        else
          gemm<Act>(c, c->tmA_A, W.tm_qkv, c->A, W.wqkv, L.bqkv, nullptr, rows, 3 * c->Hk, c->H, EPI_BIAS_QKV, st, &qs);
      } else {
        if (c->ln_fuse)
          gemm_ln(c, W.tm_qkv, L.ln1g, L.ln1b, L.bqkv, c->QKV, rows, 3 * c->Hk, EPI_BIAS, st);
        else
          gemm<Act>(c, c->tmA_A, W.tm_qkv, c->A, W.wqkv, L.bqkv, c->QKV, rows, 3 * c->Hk, c->H, EPI_BIAS, st);
        Prof p(c, st, P_MEM, 2.0 * rows * 3 * Hk * act);
        launch_unpack_qkv<Act>(reinterpret_cast<const Act*>(c->QKV), pidx, rows, a.S, c->hk, c->d,
                               reinterpret_cast<Act*>(c->Q), reinterpret_cast<Act*>(c->K), reinterpret_cast<Act*>(c->Vb),
                               st);
        c->stats.kernel_launches++;
      }
      if (fuse_a7) {
        // a6 + a7: attention writes its rows straight into the packed context [T, Hk]
        Prof p(c, st, P_ATTN, 4.0 * c->d * allowed * c->hk);
        if (!launch_attention_packed(reinterpret_cast<const bf16*>(c->Q), reinterpret_cast<const bf16*>(c->K),
                                     reinterpret_cast<const bf16*>(c->Vb), reinterpret_cast<bf16*>(c->Ctx), c->offsets,
                                     c->lens_d, c->attn_work, a.B, c->hk, a.S, c->d, g.causal, st, &c->amaps))
          c->launch_err = "attention launch refused: tensor maps could not be built";
        c->stats.kernel_launches++;
      } else {
        {
          Prof p(c, st, P_ATTN, 4.0 * c->d * allowed * c->hk);
          launch_attention<Act>(reinterpret_cast<const Act*>(c->Q), reinterpret_cast<const Act*>(c->K),
                                reinterpret_cast<const Act*>(c->Vb), reinterpret_cast<Act*>(c->O), c->lens_d,
                                c->attn_work, a.B, c->hk, a.S, c->d, g.causal, st, &c->amaps);
        }
        {
          Prof p(c, st, P_MEM, 2.0 * rows * Hk * act);
          launch_repack<Act>(reinterpret_cast<const Act*>(c->O), pidx, c->unpack_idx, rows, a.S, c->hk, c->d,
                             reinterpret_cast<Act*>(c->Ctx), st);
        }
        c->stats.kernel_launches += 2;
      }
      gemm<Act>(c, c->tmA_Ctx, W.tm_o, c->Ctx, W.wo, nullptr, c->P, rows, c->H, c->Hk, EPI_NONE, st, nullptr, &c->tmD_P,
                fused_rs ? &c->shard_rpr : nullptr);
    }
    energon_status s = ENERGON_OK;
    if (p2p) {  // a9 fused: reduce over peer memory + bias + residual + LN2, LN rows pushed to every rank
      const LayerDev& L = c0->layers[l];
      p2p_exchange<Act>(c0, rows, rpr, L.bo, L.ln2g, L.ln2b, true, st, fused_rs);
    }
    if (!p2p && (s = tp_reduce<Act>(cs, n, rows, rpr, sp, st))) return s;
    // ---- a9: bias + residual + LN2 on this rank's rows, then (SP) all-gather of the LN output
    for (int i = 0; i < n && !p2p; ++i) {
      energon_ctx* c = cs[i];
      const LayerDev& L = c->layers[l];
      const size_t o = (size_t)shard0(c) * c->H;
      const int sn = shardn(c);
      Prof p(c, st, P_MEM, sn * H * (8.0 + 2 * act));
      launch_residual_ln<Act>(c->X + o, reinterpret_cast<const Act*>(c->P) + o, L.bo, sn, c->H, L.ln2g, L.ln2b, eps,
                              c->ln_fuse ? nullptr : reinterpret_cast<Act*>(c->A) + o, st,
                              c->ln_fuse ? c->ln_stats + shard0(c) : nullptr);
      c->stats.kernel_launches++;
    }
    if (sp && !p2p && (s = tp_gather<Act>(cs, n, rpr, false, st))) return s;
    // ---- MLP module: column-parallel W1 (+GeLU), row-parallel W2
    for (int i = 0; i < n; ++i) {
      energon_ctx* c = cs[i];
      const LayerDev& W = weights(i, l);
      const LayerDev& L = c->layers[l];
      if (c->ln_fuse)
        gemm_ln(c, W.tm_1, L.ln2g, L.ln2b, L.b1, c->G, rows, c->Fk, EPI_BIAS_GELU, st);
      else
        gemm<Act>(c, c->tmA_A, W.tm_1, c->A, W.w1, L.b1, c->G, rows, c->Fk, c->H, EPI_BIAS_GELU, st, nullptr, &c->tmD_G);
      gemm<Act>(c, c->tmA_G, W.tm_2, c->G, W.w2, nullptr, c->P, rows, c->H, c->Fk, EPI_NONE, st, nullptr, &c->tmD_P,
                fused_rs ? &c->shard_rpr : nullptr);
      if (!c->pm.layers.empty() && c->pm.index[l] >= 0) {
        // the slot is free once these GEMMs ran: record it and prefetch the off-device layer `slots` ahead
        const int ns = (int)c->pm.slots.size();
        cudaEventRecord(c->pm.freed[off_slot[i]], st);
        const int jn = off_next[i] - 1 + ns;
        if (jn < (int)off_order[i].size()) pmep_fetch(c, jn, off_order[i][jn]);
      }
    }
    const bool last = (l + 1 == a.l1);
    if (p2p) {  // a12 fused (LN1 of the next layer, none after the last layer)
      const LayerDev& L = c0->layers[l];
      const LayerDev& Ln = c0->layers[last ? l : l + 1];
      p2p_exchange<Act>(c0, rows, rpr, L.b2, Ln.ln1g, Ln.ln1b, !last, st, fused_rs);
    }
    if (!p2p && (s = tp_reduce<Act>(cs, n, rows, rpr, sp, st))) return s;
    // ---- a12: bias + residual (+ LN1 of the next layer) on this rank's rows
    for (int i = 0; i < n && !p2p; ++i) {
      energon_ctx* c = cs[i];
      const LayerDev& L = c->layers[l];
      const LayerDev& Ln = c->layers[last ? l : l + 1];
      const size_t o = (size_t)shard0(c) * c->H;
      const int sn = shardn(c);
      Prof p(c, st, P_MEM, sn * H * (8.0 + (last ? 1 : 2) * act));
      launch_residual_ln<Act>(c->X + o, reinterpret_cast<const Act*>(c->P) + o, L.b2, sn, c->H, Ln.ln1g, Ln.ln1b, eps,
                              (last || c->ln_fuse) ? nullptr : reinterpret_cast<Act*>(c->A) + o, st,
                              (!last && c->ln_fuse) ? c->ln_stats + shard0(c) : nullptr);
      c->stats.kernel_launches++;
    }
    if (sp && !p2p && !last && (s = tp_gather<Act>(cs, n, rpr, false, st))) return s;
  }
  if (p2p) {
    // the final LN / unpack (or the next pipeline stage) needs every row of the residual stream
    p2p_gather(c0, rows, rpr, c0->off_X, (int64_t)sizeof(float) * c0->H, st);
  } else if (sp) {
    // the final LN / unpack needs every row of the residual stream on every rank
    energon_status s = tp_gather<float>(cs, n, rpr, true, st);
    if (s) return s;
  }

  for (int i = 0; i < n; ++i)
    if (!cs[i]->launch_err.empty()) {
      const std::string m = cs[i]->launch_err;
      cs[i]->launch_err.clear();
      return fail(c0, ENERGON_ERR_CUDA, m);
    }
  energon_ctx* c = cs[0];
  if (a.out_packed) {
    // pipeline stage output: the residual stream rows go to the next stage as they are (the T valid
    // rows with DRCE; a graph of a stage is keyed on T, see run())
    const int64_t out_rows = drce ? T : rows;
    Prof p(c, st, P_MEM, 8.0 * out_rows * H);
    cudaError_t e = cudaMemcpyAsync(a.out, c->X, sizeof(float) * (size_t)out_rows * c->H, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_fail(c0, e, "stage output copy");
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c0, e, "kernel launch");
    for (int i = 0; i < n; ++i) cs[i]->stats.forwards++;
    return ENERGON_OK;
  }
  // ---- a13: final LN + unpack (every rank holds the replicated result; a local group writes once)
  const int apply_ln = a.final_ln;
  {
    Prof p(c, st, P_MEM, 4.0 * a.B * a.S + 4.0 * T * H + (double)a.B * a.S * H * (a.out_f32 ? 4 : act));
    if (a.out_f32)
      launch_final_ln_unpack<float>(c->X, c->unpack_idx, drce ? 0 : 1, a.B * a.S, c->H, c->lnf_g, c->lnf_b, eps,
                                    apply_ln, reinterpret_cast<float*>(a.out), st);
    else
      launch_final_ln_unpack<Act>(c->X, c->unpack_idx, drce ? 0 : 1, a.B * a.S, c->H, c->lnf_g, c->lnf_b, eps, apply_ln,
                                  reinterpret_cast<Act*>(a.out), st);
  }
  c->stats.kernel_launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(c0, e, "kernel launch");
  for (int i = 0; i < n; ++i) cs[i]->stats.forwards++;
  return ENERGON_OK;
}

energon_status run_eager(energon_ctx** cs, int n, const Call& a, int64_t T) {
  return cs[0]->bf16 ? forward_t<bf16>(cs, n, a, T) : forward_t<float>(cs, n, a, T);
}

void stats_add(energon_stats& d, const energon_stats& x) {
  d.fused_exchanges += x.fused_exchanges;
  d.forwards += x.forwards;
  d.allreduce_calls += x.allreduce_calls;
  d.kernel_launches += x.kernel_launches;
  d.prefetch_bytes += x.prefetch_bytes;
}

energon_status run(energon_ctx** cs, int n, const Call& a) {
  energon_ctx* c0 = cs[0];
  cudaError_t e = cudaSetDevice(c0->cfg.device);
  if (e != cudaSuccess) return cuda_fail(c0, e, "cudaSetDevice");
  for (int i = 0; i < n; ++i) {
    energon_status s = check_ready(cs[i], a);
    if (s) return s;
  }
  int64_t T = 0;
  energon_status s = validate_call(c0, a, &T);
  if (s) return s;
  bool graph_ok = c0->graphs && c0->cap_stream;
  for (int i = 0; i < n; ++i) graph_ok = graph_ok && !cs[i]->prof && cs[i]->pm.layers.empty() && !cs[i]->p2p;
  if (!graph_ok) return run_eager(cs, n, a, T);

  // ---- CUDA graph: key = everything the launch sequence depends on.  Not the lengths: they reach the
  // device through the index-maps kernel's by-value parameter only (updated in the instantiated graph
  // before every replay), and every other launch depends on the batch only through the row bucket.
  const int rows = c0->cfg.drce ? bucket_rows(c0, T) : a.B * a.S;
  std::vector<int64_t> key = {n, (int64_t)(uintptr_t)a.tokens, (int64_t)(uintptr_t)a.x_in, (int64_t)(uintptr_t)a.out,
                              a.B, a.S, a.l0, a.l1, a.final_ln, a.out_f32, c0->cfg.drce, c0->sp, c0->fuse, c0->ring, c0->ln_fuse,
                              a.x_packed, a.out_packed, rows};
  for (int i = 0; i < n; ++i) key.push_back((int64_t)(uintptr_t)cs[i]);
  if (a.x_packed || a.out_packed) key.push_back(T);  // a pipeline stage copies exactly T rows in or out
  LensParam lp;
  for (int b = 0; b < a.B; ++b) lp.lens[b] = a.lens[b];
  for (auto& g : c0->gcache)
    if (g.key == key) {
      g.last_use = ++c0->gclock;
      for (size_t i = 0; i < g.imap_node.size(); ++i) {
        IndexMapsArgs ia = g.imap_args[i];
        void* args[2] = {&lp, &ia};
        cudaKernelNodeParams kp = g.imap_kp[i];
        kp.kernelParams = args;
        kp.extra = nullptr;
        e = cudaGraphExecKernelNodeSetParams(g.exec, g.imap_node[i], &kp);
        if (e != cudaSuccess) return cuda_fail(c0, e, "cudaGraphExecKernelNodeSetParams (index maps)");
      }
      e = cudaGraphLaunch(g.exec, a.st);
      if (e != cudaSuccess) return cuda_fail(c0, e, "cudaGraphLaunch");
      for (int i = 0; i < n; ++i) {
        stats_add(cs[i]->stats, g.delta[i]);
        cs[i]->stats.last_tokens = T;
        cs[i]->stats.last_rows = rows;
      }
      return ENERGON_OK;
    }
  // miss: run this forward eagerly on the caller's stream (first-use initialisation happens here),
  // then record the same launch sequence on the private stream (nothing executes) for later replays
  std::vector<energon_stats> before(n), after(n);
  for (int i = 0; i < n; ++i) before[i] = cs[i]->stats;
  s = run_eager(cs, n, a, T);
  if (s) return s;
  for (int i = 0; i < n; ++i) after[i] = cs[i]->stats;
  Call ac = a;
  ac.st = c0->cap_stream;
  e = cudaStreamBeginCapture(c0->cap_stream, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return cuda_fail(c0, e, "cudaStreamBeginCapture");
  s = run_eager(cs, n, ac, T);
  cudaGraph_t graph = nullptr;
  e = cudaStreamEndCapture(c0->cap_stream, &graph);
  for (int i = 0; i < n; ++i) cs[i]->stats = after[i];  // the recording pass did not execute anything
  if (s || e != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    return s ? s : cuda_fail(c0, e, "cudaStreamEndCapture");
  }
  energon_ctx::GraphEntry ent;
  ent.key = key;
  // the index-maps kernel node of every context (matched by its offsets pointer): the one node whose
  // parameters change from batch to batch
  {
    size_t nn = 0;
    cudaGraphGetNodes(graph, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    if (nn) cudaGraphGetNodes(graph, nodes.data(), &nn);
    ent.imap_node.assign(n, nullptr);
    ent.imap_kp.resize(n);
    ent.imap_args.resize(n);
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType ty;
      if (cudaGraphNodeGetType(nd, &ty) != cudaSuccess || ty != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams kp;
      if (cudaGraphKernelNodeGetParams(nd, &kp) != cudaSuccess || kp.func != index_maps_kernel_fn()) continue;
      const IndexMapsArgs* ia = static_cast<const IndexMapsArgs*>(kp.kernelParams[1]);
      for (int i = 0; i < n; ++i)
        if (ia->offsets == cs[i]->offsets) {
          ent.imap_node[i] = nd;
          ent.imap_kp[i] = kp;
          ent.imap_args[i] = *ia;
        }
    }
    cudaGetLastError();
    for (int i = 0; i < n; ++i)
      if (!ent.imap_node[i]) {
        cudaGraphDestroy(graph);
        return fail(c0, ENERGON_ERR_CUDA, "CUDA graph: index-maps kernel node not found");
      }
  }
  e = cudaGraphInstantiate(&ent.exec, graph, 0);
  if (e != cudaSuccess) {
    cudaGraphDestroy(graph);
    return cuda_fail(c0, e, "cudaGraphInstantiate");
  }
  ent.graph = graph;
  c0->stats.graphs_recorded++;
  for (int i = 0; i < n; ++i) {
    energon_stats d = after[i];
    d.forwards -= before[i].forwards;
    d.allreduce_calls -= before[i].allreduce_calls;
    d.kernel_launches -= before[i].kernel_launches;
    d.prefetch_bytes -= before[i].prefetch_bytes;
    d.fused_exchanges -= before[i].fused_exchanges;
    ent.delta.push_back(d);
  }
  ent.last_use = ++c0->gclock;
  if (c0->gcache.size() >= 32) {  // evict the least recently used graph
    size_t v = 0;
    for (size_t i = 1; i < c0->gcache.size(); ++i)
      if (c0->gcache[i].last_use < c0->gcache[v].last_use) v = i;
    cudaGraphExecDestroy(c0->gcache[v].exec);
    cudaGraphDestroy(c0->gcache[v].graph);
    c0->gcache.erase(c0->gcache.begin() + v);
  }
  c0->gcache.push_back(ent);
  return ENERGON_OK;
}


}  // namespace

// ============================================================================ C ABI
extern "C" {

const char* energon_status_string(energon_status s) {
  switch (s) {
    case ENERGON_OK: return "ENERGON_OK";
    case ENERGON_ERR_ARG: return "ENERGON_ERR_ARG";
    case ENERGON_ERR_CONFIG: return "ENERGON_ERR_CONFIG";
    case ENERGON_ERR_SHAPE: return "ENERGON_ERR_SHAPE";
    case ENERGON_ERR_LENGTH: return "ENERGON_ERR_LENGTH";
    case ENERGON_ERR_TOKEN: return "ENERGON_ERR_TOKEN";
    case ENERGON_ERR_CAPACITY: return "ENERGON_ERR_CAPACITY";
    case ENERGON_ERR_NOT_LOADED: return "ENERGON_ERR_NOT_LOADED";
    case ENERGON_ERR_CUDA: return "ENERGON_ERR_CUDA";
    case ENERGON_ERR_NCCL: return "ENERGON_ERR_NCCL";
    case ENERGON_ERR_OOM: return "ENERGON_ERR_OOM";
  }
  return "ENERGON_ERR_UNKNOWN";
}

const char* energon_last_error(const energon_ctx* ctx) { return ctx ? ctx->err.c_str() : g_last_error.c_str(); }

energon_status energon_pmep_plan(int32_t L, int32_t resident, int32_t* out) {
  if (L < 1 || resident < 1 || resident > L) return fail(nullptr, ENERGON_ERR_ARG, "need 1 <= resident <= num_layers");
  const int m = L - resident;
  if (m > 0 && !out) return fail(nullptr, ENERGON_ERR_ARG, "out_layers is NULL");
  // off-device layers "distributed evenly among those to be held on device"
  for (int g = 0; g < m; ++g) out[g] = (int32_t)(((int64_t)(g + 1) * L) / m) - 1;
  return ENERGON_OK;
}

energon_status energon_offload_layers(energon_ctx* c, const int32_t* layers, int32_t n, int32_t slots, int32_t pool,
                                      int32_t peer) {
  if (!c) return fail(nullptr, ENERGON_ERR_ARG, "ctx is NULL");
  if (n < 0 || (n > 0 && !layers) || slots < 1 || (pool != 0 && pool != 1))
    return fail(c, ENERGON_ERR_ARG, "bad offload arguments");
  if (!c->pm.layers.empty()) return fail(c, ENERGON_ERR_ARG, "layers are already offloaded");
  const int Lc = c->cfg.num_layers;
  for (int i = 0; i < n; ++i) {
    if (layers[i] < 0 || layers[i] >= Lc || (i > 0 && layers[i] <= layers[i - 1]))
      return fail(c, ENERGON_ERR_ARG, "offloaded layers must be ascending ids in [0, num_layers)");
    if (!c->layers[layers[i]].loaded) return fail(c, ENERGON_ERR_NOT_LOADED, "offload a layer after loading it");
  }
  if (n == 0) return ENERGON_OK;
  CU(c, cudaSetDevice(c->cfg.device));
  CU(c, cudaDeviceSynchronize());
  const size_t a = c->act, H = c->H, Hk = c->Hk, Fk = c->Fk;
  const size_t sz[4] = {a * 3 * Hk * H, a * H * Hk, a * Fk * H, a * H * Fk};
  const size_t bytes = sz[0] + sz[1] + sz[2] + sz[3];
  if (pool == 1 && peer != c->cfg.device) {  // (peer == device: a same-device pool, for single-GPU tests)
    int ok = 0;
    CU(c, cudaDeviceCanAccessPeer(&ok, c->cfg.device, peer));
    if (!ok) return fail(c, ENERGON_ERR_ARG, "peer_device is not peer-accessible from this device");
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(c, e, "cudaDeviceEnablePeerAccess");
    cudaGetLastError();
  }
  // Two phases so that a failure leaves the context exactly as it was (every layer resident): first
  // allocate the whole pool, the staging slots, their events and tensor maps and copy the weights into
  // the pool; only then free the device copies and switch the layers to the pool.
  const int ns = std::min<int>(slots, n);
  Pmep np;
  np.bytes = bytes;
  np.pool_kind = pool;
  np.peer = peer;
  auto rollback = [&](energon_status st, const std::string& msg) {
    cudaSetDevice(peer >= 0 && pool == 1 ? peer : c->cfg.device);
    for (void* p : np.pool) {
      if (pool == 0) cudaFreeHost(p);
      else cudaFree(p);
    }
    cudaSetDevice(c->cfg.device);
    for (void* p : np.slot_buf) cudaFree(p);
    for (cudaEvent_t e : np.fetched) cudaEventDestroy(e);
    for (cudaEvent_t e : np.freed) cudaEventDestroy(e);
    if (np.copy) cudaStreamDestroy(np.copy);
    cudaGetLastError();
    return fail(c, st, msg);
  };
  auto cu_ok = [&](cudaError_t e, const char* what, energon_status* st, std::string* msg) {
    if (e == cudaSuccess) return true;
    *st = e == cudaErrorMemoryAllocation ? ENERGON_ERR_OOM : ENERGON_ERR_CUDA;
    *msg = std::string(what) + ": " + cudaGetErrorString(e);
    return false;
  };
  energon_status est = ENERGON_OK;
  std::string emsg;
  for (int i = 0; i < n; ++i) {
    const LayerDev& L = c->layers[layers[i]];
    void* buf = nullptr;
    cudaError_t e;
    if (pool == 0) {
      e = cudaHostAlloc(&buf, bytes, cudaHostAllocDefault);
    } else {
      cudaSetDevice(peer);
      e = cudaMalloc(&buf, bytes);
      cudaSetDevice(c->cfg.device);
    }
    if (!cu_ok(e, "pool allocation", &est, &emsg)) return rollback(est, emsg);
    np.pool.push_back(buf);
    const void* src[4] = {L.wqkv, L.wo, L.w1, L.w2};
    size_t off = 0;
    for (int k = 0; k < 4; ++k) {
      e = pool == 0 ? cudaMemcpy((char*)buf + off, src[k], sz[k], cudaMemcpyDeviceToHost)
                    : cudaMemcpyPeer((char*)buf + off, peer, src[k], c->cfg.device, sz[k]);
      if (!cu_ok(e, "copy into the pool", &est, &emsg)) return rollback(est, emsg);
      off += sz[k];
    }
  }
  if (!cu_ok(cudaStreamCreateWithFlags(&np.copy, cudaStreamNonBlocking), "copy stream", &est, &emsg))
    return rollback(est, emsg);
  np.slots.resize(ns);
  for (int q = 0; q < ns; ++q) {
    void* buf = nullptr;
    if (!cu_ok(cudaMalloc(&buf, bytes), "staging slot", &est, &emsg)) return rollback(est, emsg);
    np.slot_buf.push_back(buf);
    LayerDev& S = np.slots[q];
    S.wqkv = buf;
    S.wo = (char*)buf + sz[0];
    S.w1 = (char*)buf + sz[0] + sz[1];
    S.w2 = (char*)buf + sz[0] + sz[1] + sz[2];
    if (c->bf16)
      for (int i = 0; i < kNumBoxes; ++i)
        if (!make_tmap_kmajor(&S.tm_qkv[i], S.wqkv, 3 * c->Hk, c->H, kBoxes[i]) ||
            !make_tmap_kmajor(&S.tm_o[i], S.wo, c->H, c->Hk, kBoxes[i]) ||
            !make_tmap_kmajor(&S.tm_1[i], S.w1, c->Fk, c->H, kBoxes[i]) ||
            !make_tmap_kmajor(&S.tm_2[i], S.w2, c->H, c->Fk, kBoxes[i]))
          return rollback(ENERGON_ERR_CUDA, "cuTensorMapEncodeTiled failed for a staging slot");
    cudaEvent_t ef = nullptr, er = nullptr;
    if (!cu_ok(cudaEventCreateWithFlags(&ef, cudaEventDisableTiming), "event", &est, &emsg)) return rollback(est, emsg);
    np.fetched.push_back(ef);
    if (!cu_ok(cudaEventCreateWithFlags(&er, cudaEventDisableTiming), "event", &est, &emsg)) return rollback(est, emsg);
    np.freed.push_back(er);
    if (!cu_ok(cudaEventRecord(er, np.copy), "event record", &est, &emsg)) return rollback(est, emsg);  // slots start free
  }
  if (!cu_ok(cudaDeviceSynchronize(), "cudaDeviceSynchronize", &est, &emsg)) return rollback(est, emsg);
  // ---- commit: nothing below can fail
  np.index.assign(Lc, -1);
  for (int i = 0; i < n; ++i) {
    LayerDev& L = c->layers[layers[i]];
    void* src[4] = {L.wqkv, L.wo, L.w1, L.w2};
    for (int k = 0; k < 4; ++k) {
      for (size_t q = 0; q < c->allocs.size(); ++q)
        if (c->allocs[q] == src[k]) {
          c->allocs.erase(c->allocs.begin() + q);
          break;
        }
      cudaFree(src[k]);
      c->stats.weight_bytes -= (int64_t)sz[k];
    }
    L.wqkv = L.wo = L.w1 = L.w2 = nullptr;
    np.layers.push_back(layers[i]);
    np.index[layers[i]] = i;
  }
  c->pm = np;
  return ENERGON_OK;
}

energon_status energon_shard_plan(const energon_config* cfg, energon_shard* out) {
  if (!out) return fail(nullptr, ENERGON_ERR_ARG, "out is NULL");
  energon_status s = validate_config(cfg);
  if (s) return s;
  const int k = cfg->tp_size, r = cfg->tp_rank, hk = cfg->num_heads / k, d = cfg->hidden / cfg->num_heads;
  out->head0 = r * hk;
  out->heads = hk;
  out->qkv_col0 = r * hk * d;
  out->qkv_cols = hk * d;
  out->ffn_col0 = r * (cfg->ffn / k);
  out->ffn_cols = cfg->ffn / k;
  return ENERGON_OK;
}

energon_status energon_p2p_handle(energon_ctx* c, void* out) {
  if (!c || !out) return fail(c, ENERGON_ERR_ARG, "NULL argument");
  if (!c->p2p) return fail(c, ENERGON_ERR_CONFIG, "context was not created with comm = ENERGON_COMM_P2P and tp_size > 1");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  CU(c, cudaSetDevice(c->cfg.device));
  cudaIpcMemHandle_t h;
  CU(c, cudaIpcGetMemHandle(&h, c->region));
  memcpy(out, &h, sizeof(h));
  return ENERGON_OK;
}

energon_status energon_p2p_connect(energon_ctx* c, const void* handles) {
  if (!c || !handles) return fail(c, ENERGON_ERR_ARG, "NULL argument");
  if (!c->p2p) return fail(c, ENERGON_ERR_CONFIG, "context was not created with comm = ENERGON_COMM_P2P and tp_size > 1");
  if (c->p2p_connected) return fail(c, ENERGON_ERR_ARG, "already connected");
  CU(c, cudaSetDevice(c->cfg.device));
  const char* hs = static_cast<const char*>(handles);
  for (int q = 0; q < c->k; ++q) {
    if (q == c->r) {
      c->peers.base[q] = c->region;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, hs + 64 * q, 64);
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      for (void* o : c->ipc_opened) cudaIpcCloseMemHandle(o);
      c->ipc_opened.clear();
      return cuda_fail(c, e, ("cudaIpcOpenMemHandle(rank " + std::to_string(q) + ")").c_str());
    }
    c->ipc_opened.push_back(p);
    c->peers.base[q] = p;
  }
  if (c->bf16) {
    // the row-parallel GEMMs store the rows rank s owns into rank s's slot for this rank (GEMM ->
    // reduce-scatter fused): one TMA store map per destination rank over [slot_rows, H] bf16
    memset(&c->shard, 0, sizeof(c->shard));
    for (int q = 0; q < c->k; ++q) {
      char* slot = static_cast<char*>(c->peers.base[q]) + c->off_S + (int64_t)c->r * c->slot_rows * c->H * 2;
      if (!make_tmap_store(&c->shard.maps[q], slot, c->slot_rows, c->H))
        return fail(c, ENERGON_ERR_CUDA, "cuTensorMapEncodeTiled failed for a peer slot");
    }
    c->shard.k = c->k;
  }
  c->p2p_connected = true;
  return ENERGON_OK;
}

energon_status energon_get_unique_id(void* out) {
  if (!out) return fail(nullptr, ENERGON_ERR_ARG, "out is NULL");
  ncclUniqueId id;
  ncclResult_t e = ncclGetUniqueId(&id);
  if (e != ncclSuccess) return fail(nullptr, ENERGON_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(e));
  memcpy(out, &id, sizeof(id));
  return ENERGON_OK;
}

energon_status energon_init(const energon_config* cfg, const void* uid, energon_ctx** out) {
  if (!out) return fail(nullptr, ENERGON_ERR_ARG, "out is NULL");
  *out = nullptr;
  energon_status s = validate_config(cfg);
  if (s) return s;
  if (cfg->tp_size > 1 && cfg->comm == ENERGON_COMM_NCCL && !uid)
    return fail(nullptr, ENERGON_ERR_ARG, "nccl_unique_id required when tp_size > 1 with NCCL");
  energon_ctx* c = new energon_ctx();
  c->cfg = *cfg;
  if ((s = setup(c))) {
    g_last_error = c->err;
    release(c);
    return s;
  }
  if (cfg->tp_size > 1 && cfg->comm == ENERGON_COMM_NCCL) {
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    ncclResult_t e = ncclCommInitRank(&c->nccl, cfg->tp_size, id, cfg->tp_rank);
    if (e != ncclSuccess) {
      c->nccl = nullptr;
      fail(c, ENERGON_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(e));
      release(c);
      return ENERGON_ERR_NCCL;
    }
  }
  *out = c;
  return ENERGON_OK;
}

energon_status energon_init_local_group(const energon_config* cfg, int32_t k, energon_ctx** out_k) {
  if (!out_k || !cfg) return fail(nullptr, ENERGON_ERR_ARG, "NULL argument");
  if (k < 1 || k > 8) return fail(nullptr, ENERGON_ERR_CONFIG, "k must be in [1, 8]");
  for (int i = 0; i < k; ++i) out_k[i] = nullptr;
  for (int i = 0; i < k; ++i) {
    energon_config ci = *cfg;
    ci.tp_size = k;
    ci.tp_rank = i;
    energon_status s = validate_config(&ci);
    if (s == ENERGON_OK) {
      energon_ctx* c = new energon_ctx();
      c->cfg = ci;
      c->local_group = true;
      s = setup(c);
      if (s) {
        g_last_error = c->err;
        release(c);
      } else {
        out_k[i] = c;
      }
    }
    if (s) {
      for (int j = 0; j < i; ++j) {
        release(out_k[j]);
        out_k[j] = nullptr;
      }
      return s;
    }
  }
  return ENERGON_OK;
}

energon_status energon_load_embeddings(energon_ctx* c, const void* tok_emb, const void* pos_emb, const void* lnf_g,
                                       const void* lnf_b, int32_t sd, int32_t on_dev) {
  if (!c || !tok_emb || !pos_emb || !lnf_g || !lnf_b) return fail(c, ENERGON_ERR_ARG, "NULL argument");
  if (sd < 0 || sd > 2) return fail(c, ENERGON_ERR_ARG, "src_dtype must be F32, BF16 or F64");
  CU(c, cudaSetDevice(c->cfg.device));
  // the sources may have been produced on any stream of this device (e.g. the legacy default stream,
  // which the non-blocking load stream does not wait for): finish all prior work first
  CU(c, cudaDeviceSynchronize());
  const int64_t VH = (int64_t)c->V * c->H, PH = (int64_t)c->cfg.max_seq * c->H;
  energon_status s;
  if (!c->tok_emb) {
    if ((s = dalloc(c, &c->tok_emb, c->act * VH, &c->stats.weight_bytes)) ||
        (s = dalloc(c, &c->pos_emb, c->act * PH, &c->stats.weight_bytes)) ||
        (s = dalloc(c, &c->lnf_g, sizeof(float) * c->H, &c->stats.weight_bytes)) ||
        (s = dalloc(c, &c->lnf_b, sizeof(float) * c->H, &c->stats.weight_bytes)))
      return s;
  }
  const bool dev = on_dev != 0;
  if (c->bf16) {
    if ((s = put_vector<bf16>(c, sd, tok_emb, dev, VH, 0, (int)VH, reinterpret_cast<bf16*>(c->tok_emb))) ||
        (s = put_vector<bf16>(c, sd, pos_emb, dev, PH, 0, (int)PH, reinterpret_cast<bf16*>(c->pos_emb))))
      return s;
  } else {
    if ((s = put_vector<float>(c, sd, tok_emb, dev, VH, 0, (int)VH, reinterpret_cast<float*>(c->tok_emb))) ||
        (s = put_vector<float>(c, sd, pos_emb, dev, PH, 0, (int)PH, reinterpret_cast<float*>(c->pos_emb))))
      return s;
  }
  if ((s = put_vector<float>(c, sd, lnf_g, dev, c->H, 0, c->H, c->lnf_g)) ||
      (s = put_vector<float>(c, sd, lnf_b, dev, c->H, 0, c->H, c->lnf_b)))
    return s;
  CU(c, cudaStreamSynchronize(c->load_stream));
  c->emb_loaded = true;
  return ENERGON_OK;
}

energon_status energon_load_layer_weights(energon_ctx* c, int32_t layer, const energon_layer_weights* w, int32_t sd,
                                          int32_t on_dev, int32_t layout) {
  if (!c || !w) return fail(c, ENERGON_ERR_ARG, "NULL argument");
  if (layer < 0 || layer >= c->cfg.num_layers) return fail(c, ENERGON_ERR_ARG, "layer index out of range");
  if (!c->pm.index.empty() && c->pm.index[layer] >= 0) return fail(c, ENERGON_ERR_ARG, "layer is offloaded (PMEP)");
  if (sd < 0 || sd > 2) return fail(c, ENERGON_ERR_ARG, "src_dtype must be F32, BF16 or F64");
  if (layout != ENERGON_FULL && layout != ENERGON_RANK_SHARD) return fail(c, ENERGON_ERR_ARG, "bad src_layout");
  const void* ptrs[16] = {w->wq, w->wk, w->wv, w->wo, w->bq, w->bk, w->bv, w->bo,
                          w->w1, w->b1, w->w2, w->b2, w->ln1_g, w->ln1_b, w->ln2_g, w->ln2_b};
  for (int i = 0; i < 16; ++i)
    if (!ptrs[i]) return fail(c, ENERGON_ERR_ARG, "a layer weight pointer is NULL");
  CU(c, cudaSetDevice(c->cfg.device));
  CU(c, cudaDeviceSynchronize());  // sources may come from any stream (see energon_load_embeddings)
  LayerDev& L = c->layers[layer];
  const int H = c->H, F = c->F, Hk = c->Hk, Fk = c->Fk, r = c->r;
  const size_t a = c->act;
  energon_status s;
  int64_t* wb = &c->stats.weight_bytes;
  if (!L.wqkv) {
    if ((s = dalloc(c, &L.wqkv, a * 3 * Hk * H, wb)) || (s = dalloc(c, &L.wo, a * (size_t)H * Hk, wb)) ||
        (s = dalloc(c, &L.w1, a * (size_t)Fk * H, wb)) || (s = dalloc(c, &L.w2, a * (size_t)H * Fk, wb)) ||
        (s = dalloc(c, &L.bqkv, sizeof(float) * 3 * Hk, wb)) || (s = dalloc(c, &L.bo, sizeof(float) * H, wb)) ||
        (s = dalloc(c, &L.b1, sizeof(float) * Fk, wb)) || (s = dalloc(c, &L.b2, sizeof(float) * H, wb)) ||
        (s = dalloc(c, &L.ln1g, sizeof(float) * H, wb)) || (s = dalloc(c, &L.ln1b, sizeof(float) * H, wb)) ||
        (s = dalloc(c, &L.ln2g, sizeof(float) * H, wb)) || (s = dalloc(c, &L.ln2b, sizeof(float) * H, wb)))
      return s;
  }
  const bool full = layout == ENERGON_FULL, dev = on_dev != 0;
  // column-parallel: this rank's heads / FFN columns; row-parallel: the matching rows
  energon_shard sh;
  energon_shard_plan(&c->cfg, &sh);
  (void)r;
  const int64_t qk_ld = full ? H : Hk, qk_col0 = full ? sh.qkv_col0 : 0;
  const int64_t o_rows = full ? H : Hk, o_row0 = full ? sh.qkv_col0 : 0;
  const int64_t w1_ld = full ? F : Fk, w1_col0 = full ? sh.ffn_col0 : 0;
  const int64_t w2_rows = full ? F : Fk, w2_row0 = full ? sh.ffn_col0 : 0;
  const int64_t bq_n = full ? H : Hk, bq_off = full ? sh.qkv_col0 : 0;
  const int64_t b1_n = full ? F : Fk, b1_off = full ? sh.ffn_col0 : 0;
  if ((s = put_matrix(c, sd, w->wq, dev, H, qk_ld, 0, qk_col0, Hk, H, L.wqkv, 0)) ||
      (s = put_matrix(c, sd, w->wk, dev, H, qk_ld, 0, qk_col0, Hk, H, L.wqkv, Hk)) ||
      (s = put_matrix(c, sd, w->wv, dev, H, qk_ld, 0, qk_col0, Hk, H, L.wqkv, 2 * Hk)) ||
      (s = put_matrix(c, sd, w->wo, dev, o_rows, H, o_row0, 0, H, Hk, L.wo, 0)) ||
      (s = put_matrix(c, sd, w->w1, dev, H, w1_ld, 0, w1_col0, Fk, H, L.w1, 0)) ||
      (s = put_matrix(c, sd, w->w2, dev, w2_rows, H, w2_row0, 0, H, Fk, L.w2, 0)) ||
      (s = put_vector<float>(c, sd, w->bq, dev, bq_n, bq_off, Hk, L.bqkv)) ||
      (s = put_vector<float>(c, sd, w->bk, dev, bq_n, bq_off, Hk, L.bqkv + Hk)) ||
      (s = put_vector<float>(c, sd, w->bv, dev, bq_n, bq_off, Hk, L.bqkv + 2 * Hk)) ||
      (s = put_vector<float>(c, sd, w->bo, dev, H, 0, H, L.bo)) ||
      (s = put_vector<float>(c, sd, w->b1, dev, b1_n, b1_off, Fk, L.b1)) ||
      (s = put_vector<float>(c, sd, w->b2, dev, H, 0, H, L.b2)) ||
      (s = put_vector<float>(c, sd, w->ln1_g, dev, H, 0, H, L.ln1g)) ||
      (s = put_vector<float>(c, sd, w->ln1_b, dev, H, 0, H, L.ln1b)) ||
      (s = put_vector<float>(c, sd, w->ln2_g, dev, H, 0, H, L.ln2g)) ||
      (s = put_vector<float>(c, sd, w->ln2_b, dev, H, 0, H, L.ln2b)))
    return s;
  CU(c, cudaStreamSynchronize(c->load_stream));
  if (c->bf16) {
    for (int i = 0; i < kNumBoxes; ++i) {
      if (!make_tmap_kmajor(&L.tm_qkv[i], L.wqkv, 3 * Hk, H, kBoxes[i]) ||
          !make_tmap_kmajor(&L.tm_o[i], L.wo, H, Hk, kBoxes[i]) || !make_tmap_kmajor(&L.tm_1[i], L.w1, Fk, H, kBoxes[i]) ||
          !make_tmap_kmajor(&L.tm_2[i], L.w2, H, Fk, kBoxes[i]))
        return fail(c, ENERGON_ERR_CUDA, "cuTensorMapEncodeTiled failed for a weight operand");
    }
  }
  L.loaded = true;
  return ENERGON_OK;
}

energon_status energon_forward(energon_ctx* c, const int32_t* tokens, const int32_t* lens, int32_t B, int32_t S,
                               void* out, void* stream) {
  if (!c) return fail(nullptr, ENERGON_ERR_ARG, "ctx is NULL");
  if (!tokens) return fail(c, ENERGON_ERR_ARG, "tokens is NULL");
  Call a{tokens, nullptr, lens, B, S, 0, c->cfg.num_layers, c->cfg.final_ln, out, false, (cudaStream_t)stream};
  energon_ctx* cs[1] = {c};
  return run(cs, 1, a);
}

energon_status energon_forward_group(energon_ctx** cs, int32_t k, const int32_t* tokens, const int32_t* lens,
                                     int32_t B, int32_t S, void* out, void* stream) {
  if (!cs || k < 1 || k > 8) return fail(nullptr, ENERGON_ERR_ARG, "bad context list");
  for (int i = 0; i < k; ++i)
    if (!cs[i] || cs[i]->cfg.tp_size != k || cs[i]->cfg.tp_rank != i || (k > 1 && !cs[i]->local_group))
      return fail(nullptr, ENERGON_ERR_ARG, "contexts must be ranks 0..k-1 of one local group");
  if (!tokens) return fail(cs[0], ENERGON_ERR_ARG, "tokens is NULL");
  Call a{tokens, nullptr, lens, B, S, 0, cs[0]->cfg.num_layers, cs[0]->cfg.final_ln, out, false, (cudaStream_t)stream};
  return run(cs, k, a);
}

energon_status energon_forward_hidden(energon_ctx* c, const float* x, const int32_t* lens, int32_t B, int32_t S,
                                      int32_t l0, int32_t l1, int32_t apply_final_ln, float* out, void* stream) {
  if (!c) return fail(nullptr, ENERGON_ERR_ARG, "ctx is NULL");
  if (!x) return fail(c, ENERGON_ERR_ARG, "x is NULL");
  Call a{nullptr, x, lens, B, S, l0, l1, apply_final_ln, out, true, (cudaStream_t)stream};
  energon_ctx* cs[1] = {c};
  return run(cs, 1, a);
}

energon_status energon_stage_plan(int32_t L, int32_t pp, int32_t* out_begin) {
  if (!out_begin) return fail(nullptr, ENERGON_ERR_ARG, "out_begin is NULL");
  if (L < 1 || pp < 1 || pp > L) return fail(nullptr, ENERGON_ERR_CONFIG, "need 1 <= pp_size <= num_layers");
  // contiguous ranges, sizes differ by at most one, the earlier stages take the remainder
  out_begin[0] = 0;
  for (int i = 0; i < pp; ++i) out_begin[i + 1] = out_begin[i] + L / pp + (i < L % pp ? 1 : 0);
  return ENERGON_OK;
}

namespace {
energon_status stage_call(energon_ctx** cs, int k, const int32_t* tokens, const float* x, const int32_t* lens,
                          int32_t B, int32_t S, int32_t l0, int32_t l1, int32_t out_kind, void* out, void* stream) {
  if ((tokens == nullptr) == (x == nullptr))
    return fail(cs[0], ENERGON_ERR_ARG, "exactly one of tokens_d (first stage) and x_d (later stages) must be given");
  if (out_kind != ENERGON_STAGE_PACKED && out_kind != ENERGON_STAGE_FINAL)
    return fail(cs[0], ENERGON_ERR_ARG, "out_kind must be ENERGON_STAGE_PACKED or ENERGON_STAGE_FINAL");
  Call a{tokens, x, lens, B, S, l0, l1, cs[0]->cfg.final_ln, out, false, (cudaStream_t)stream};
  a.x_packed = x != nullptr;
  a.out_packed = out_kind == ENERGON_STAGE_PACKED;
  if (a.x_packed && a.out_packed && l0 >= l1) return fail(cs[0], ENERGON_ERR_ARG, "a middle stage needs >= 1 layer");
  return run(cs, k, a);
}
}  // namespace

energon_status energon_forward_stage(energon_ctx* c, const int32_t* tokens, const float* x, const int32_t* lens,
                                     int32_t B, int32_t S, int32_t l0, int32_t l1, int32_t out_kind, void* out,
                                     void* stream) {
  if (!c) return fail(nullptr, ENERGON_ERR_ARG, "ctx is NULL");
  energon_ctx* cs[1] = {c};
  return stage_call(cs, 1, tokens, x, lens, B, S, l0, l1, out_kind, out, stream);
}

energon_status energon_forward_stage_group(energon_ctx** cs, int32_t k, const int32_t* tokens, const float* x,
                                           const int32_t* lens, int32_t B, int32_t S, int32_t l0, int32_t l1,
                                           int32_t out_kind, void* out, void* stream) {
  if (!cs || k < 1 || k > 8) return fail(nullptr, ENERGON_ERR_ARG, "bad context list");
  for (int i = 0; i < k; ++i)
    if (!cs[i] || cs[i]->cfg.tp_size != k || cs[i]->cfg.tp_rank != i || (k > 1 && !cs[i]->local_group))
      return fail(nullptr, ENERGON_ERR_ARG, "contexts must be ranks 0..k-1 of one local group");
  return stage_call(cs, k, tokens, x, lens, B, S, l0, l1, out_kind, out, stream);
}

energon_status energon_sync(energon_ctx* c) {
  if (!c) return fail(nullptr, ENERGON_ERR_ARG, "ctx is NULL");
  CU(c, cudaSetDevice(c->cfg.device));
  CU(c, cudaDeviceSynchronize());
  if (c->nccl) {
    ncclResult_t ae = ncclSuccess;
    ncclCommGetAsyncError(c->nccl, &ae);
    if (ae != ncclSuccess) return fail(c, ENERGON_ERR_NCCL, std::string("NCCL async error: ") + ncclGetErrorString(ae));
  }
  if (*c->err_host) {
    *c->err_host = 0;
    return fail(c, ENERGON_ERR_TOKEN, "a token id outside [0, vocab) was seen on the device (SPEC.md:151)");
  }
  return ENERGON_OK;
}

energon_status energon_get_stats(const energon_ctx* c, energon_stats* out) {
  if (!c || !out) return fail(nullptr, ENERGON_ERR_ARG, "NULL argument");
  *out = c->stats;
  return ENERGON_OK;
}

void energon_destroy(energon_ctx* c) { release(c); }

energon_status energon_set_option(energon_ctx* c, int32_t option, int32_t value) {
  if (!c) return fail(nullptr, ENERGON_ERR_ARG, "ctx is NULL");
  if (option == ENERGON_OPT_DRCE) {
    if (value != 0 && value != 1) return fail(c, ENERGON_ERR_ARG, "ENERGON_OPT_DRCE takes 0 or 1");
    c->cfg.drce = value;
    c->tm_rows = -1;  // activation tensor maps depend on the row count
    return ENERGON_OK;
  }
  if (option == ENERGON_OPT_GRAPH) {
    if (value != 0 && value != 1) return fail(c, ENERGON_ERR_ARG, "ENERGON_OPT_GRAPH takes 0 or 1");
    c->graphs = value != 0;
    if (c->graphs && !c->cap_stream) CU(c, cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    return ENERGON_OK;
  }
  if (option == ENERGON_OPT_RING_NUMERICS) {
    if (value != 0 && value != 1) return fail(c, ENERGON_ERR_ARG, "ENERGON_OPT_RING_NUMERICS takes 0 or 1");
    if (!c->local_group && value) return fail(c, ENERGON_ERR_CONFIG, "ENERGON_OPT_RING_NUMERICS needs a local group");
    c->ring = value != 0;
    return ENERGON_OK;
  }
  if (option == ENERGON_OPT_LN_FUSE) {
    if (value != 0 && value != 1) return fail(c, ENERGON_ERR_ARG, "ENERGON_OPT_LN_FUSE takes 0 or 1");
    if (value && (c->act != 2 || c->k != 1 || c->local_group || c->H % 64 != 0))
      return fail(c, ENERGON_ERR_CONFIG, "ENERGON_OPT_LN_FUSE needs bf16, TP = 1 and hidden % 64 == 0");
    c->ln_fuse = value != 0;
    return ENERGON_OK;
  }
  if (option == ENERGON_OPT_TP_SP) {
    if (value != 0 && value != 1) return fail(c, ENERGON_ERR_ARG, "ENERGON_OPT_TP_SP takes 0 or 1");
    c->sp = value != 0;
    return ENERGON_OK;
  }
  return fail(c, ENERGON_ERR_ARG, "unknown option");
}

energon_status energon_set_profiling(energon_ctx* c, int32_t enable) {
  if (!c) return fail(nullptr, ENERGON_ERR_ARG, "ctx is NULL");
  CU(c, cudaSetDevice(c->cfg.device));
  if (enable) {
    CU(c, cudaDeviceSynchronize());
    c->recs.clear();
    c->pool_used = 0;
    memset(&c->pacc, 0, sizeof(c->pacc));
  }
  c->prof = enable != 0;
  return ENERGON_OK;
}

energon_status energon_get_profile(energon_ctx* c, energon_profile* out) {
  if (!c || !out) return fail(c, ENERGON_ERR_ARG, "NULL argument");
  CU(c, cudaSetDevice(c->cfg.device));
  for (auto& r : c->recs) {
    CU(c, cudaEventSynchronize(r.b));
    float ms = 0.f;
    CU(c, cudaEventElapsedTime(&ms, r.a, r.b));
    energon_profile& p = c->pacc;
    switch (r.cls) {
      case P_GEMM: p.gemm_ms += ms; p.gemm_flops += r.work; p.gemm_launches++; break;
      case P_ATTN: p.attn_ms += ms; p.attn_flops += r.work; p.attn_launches++; break;
      case P_MEM: p.mem_ms += ms; p.mem_bytes += r.work; p.mem_launches++; break;
      default: p.comm_ms += ms; p.comm_bytes += r.work; p.comm_calls++; break;
    }
  }
  c->recs.clear();
  c->pool_used = 0;
  *out = c->pacc;
  return ENERGON_OK;
}

energon_status energon_index_maps(const int32_t* lens, int32_t B, int32_t S, int32_t* offsets, int32_t* pack_idx,
                                  int32_t* pos, int32_t* unpack_idx, void* stream) {
  if (!lens || !offsets || !pack_idx || !pos || !unpack_idx) return fail(nullptr, ENERGON_ERR_ARG, "NULL argument");
  if (B < 1 || B > ENERGON_MAX_BATCH || S < 1) return fail(nullptr, ENERGON_ERR_ARG, "bad batch / max_len");
  LensParam lp;
  for (int b = 0; b < B; ++b) {
    if (lens[b] < 1 || lens[b] > S) return fail(nullptr, ENERGON_ERR_LENGTH, "seq_lens not in [1, max_len]");
    lp.lens[b] = lens[b];
  }
  int64_t T = 0;
  for (int b = 0; b < B; ++b) T += lens[b];
  IndexMapsArgs ia{B, S, (int)T, offsets, pack_idx, pos, unpack_idx, nullptr, 0, nullptr, nullptr, nullptr, 1, 128, 64};
  launch_index_maps(lp, ia, (cudaStream_t)stream);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "index_maps");
  return ENERGON_OK;
}

energon_status energon_attention(int32_t dtype, const void* Q, const void* K, const void* V, void* O,
                                 const int32_t* lens, int32_t B, int32_t hk, int32_t S, int32_t d, int32_t causal,
                                 void* stream) {
  if (!Q || !K || !V || !O || !lens) return fail(nullptr, ENERGON_ERR_ARG, "NULL argument");
  if (B < 1 || B > ENERGON_MAX_BATCH || hk < 1 || S < 1 || d < 1 || d % 8 || (causal != 0 && causal != 1))
    return fail(nullptr, ENERGON_ERR_ARG, "bad attention arguments");
  LensParam lp;
  for (int b = 0; b < B; ++b) {
    if (lens[b] < 1 || lens[b] > S) return fail(nullptr, ENERGON_ERR_LENGTH, "seq_lens not in [1, max_len]");
    lp.lens[b] = lens[b];
  }
  if (dtype != ENERGON_DTYPE_F32 && dtype != ENERGON_DTYPE_BF16) return fail(nullptr, ENERGON_ERR_ARG, "dtype must be F32 or BF16");
  // stream-ordered scratch for the device lengths + work list (the forward path keeps them in the context)
  cudaStream_t st = (cudaStream_t)stream;
  const size_t n_work = 2 + (size_t)B * ((S + 63) / 64);
  void* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, sizeof(int) * ENERGON_MAX_BATCH + sizeof(uint32_t) * n_work, st);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaMallocAsync");
  int* lens_d = static_cast<int*>(scratch);
  uint32_t* work_d = reinterpret_cast<uint32_t*>(lens_d + ENERGON_MAX_BATCH);
  launch_attn_plan(lp, B, causal, attention_tile_bm(), attention_tile_bn(), lens_d, work_d, st);
  if (dtype == ENERGON_DTYPE_F32)
    launch_attention<float>(reinterpret_cast<const float*>(Q), reinterpret_cast<const float*>(K),
                            reinterpret_cast<const float*>(V), reinterpret_cast<float*>(O), lens_d, work_d, B, hk, S, d,
                            causal, st);
  else
    launch_attention<bf16>(reinterpret_cast<const bf16*>(Q), reinterpret_cast<const bf16*>(K),
                           reinterpret_cast<const bf16*>(V), reinterpret_cast<bf16*>(O), lens_d, work_d, B, hk, S, d,
                           causal, st);
  e = cudaGetLastError();
  cudaFreeAsync(scratch, st);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "attention");
  return ENERGON_OK;
}

energon_status energon_gemm(int32_t dtype, const void* A, const void* W, const float* bias, void* D, int32_t M,
                            int32_t N, int32_t K, int32_t epi, void* stream) {
  if (!A || !W || !D) return fail(nullptr, ENERGON_ERR_ARG, "NULL argument");
  if (M < 1 || N < 1 || K < 1 || epi < 0 || epi > 2 || (epi > 0 && !bias))
    return fail(nullptr, ENERGON_ERR_ARG, "bad GEMM arguments");
  if (dtype == ENERGON_DTYPE_F32) {
    launch_gemm_f32(reinterpret_cast<const float*>(A), reinterpret_cast<const float*>(W), bias,
                    reinterpret_cast<float*>(D), M, N, K, epi, (cudaStream_t)stream);
  } else if (dtype == ENERGON_DTYPE_BF16) {
    if (K % 8 || N % 8) return fail(nullptr, ENERGON_ERR_SHAPE, "bf16 GEMM needs K and N multiples of 8");
    if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(W) | reinterpret_cast<uintptr_t>(D)) & 15)
      return fail(nullptr, ENERGON_ERR_SHAPE, "bf16 GEMM needs 16-byte aligned A, W and D");
    const int code = tc_pick_bn(M, N, K);
    CUtensorMap ta, tb;
    if (!make_tmap_kmajor(&ta, A, M, K, 128) || !make_tmap_kmajor(&tb, W, N, K, tc_w_box(code)))
      return fail(nullptr, ENERGON_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    if (!launch_gemm_tc(ta, tb, code, bias, reinterpret_cast<bf16*>(D), M, N, K, epi, (cudaStream_t)stream))
      return fail(nullptr, ENERGON_ERR_CUDA, "GEMM output tensor map could not be built");
  } else {
    return fail(nullptr, ENERGON_ERR_ARG, "dtype must be F32 or BF16");
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "gemm");
  return ENERGON_OK;
}

// ---- a5 / a7 / a13 standalone layout kernels (the same kernels the forward path runs when the fused
// epilogues are off: fp32 mode, head sizes other than 64 / 128, ENERGON_NO_FUSE, padded A/B)
namespace {
energon_status layout_args(int32_t dtype, int32_t T, int32_t S, int32_t hk, int32_t d) {
  if (dtype != ENERGON_DTYPE_F32 && dtype != ENERGON_DTYPE_BF16) return fail(nullptr, ENERGON_ERR_ARG, "dtype must be F32 or BF16");
  if (T < 0 || S < 1 || hk < 1 || d < 1 || d % 8) return fail(nullptr, ENERGON_ERR_ARG, "bad layout arguments");
  return ENERGON_OK;
}
energon_status launched(const char* what) {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ENERGON_OK : cuda_fail(nullptr, e, what);
}
}  // namespace

energon_status energon_unpack_qkv(int32_t dtype, const void* QKV, const int32_t* pack_idx, int32_t T, int32_t S,
                                  int32_t hk, int32_t d, void* Q, void* K, void* V, void* stream) {
  if (!QKV || !Q || !K || !V) return fail(nullptr, ENERGON_ERR_ARG, "NULL argument");
  if (energon_status s = layout_args(dtype, T, S, hk, d)) return s;
  if (dtype == ENERGON_DTYPE_F32)
    launch_unpack_qkv<float>((const float*)QKV, pack_idx, T, S, hk, d, (float*)Q, (float*)K, (float*)V, (cudaStream_t)stream);
  else
    launch_unpack_qkv<bf16>((const bf16*)QKV, pack_idx, T, S, hk, d, (bf16*)Q, (bf16*)K, (bf16*)V, (cudaStream_t)stream);
  return launched("unpack_qkv");
}

energon_status energon_repack(int32_t dtype, const void* O, const int32_t* pack_idx, const int32_t* unpack_idx, int32_t T,
                              int32_t S, int32_t hk, int32_t d, void* C, void* stream) {
  if (!O || !C || (!pack_idx && !unpack_idx)) return fail(nullptr, ENERGON_ERR_ARG, "NULL argument");
  if (energon_status s = layout_args(dtype, T, S, hk, d)) return s;
  if (dtype == ENERGON_DTYPE_F32)
    launch_repack<float>((const float*)O, pack_idx, unpack_idx, T, S, hk, d, (float*)C, (cudaStream_t)stream);
  else
    launch_repack<bf16>((const bf16*)O, pack_idx, unpack_idx, T, S, hk, d, (bf16*)C, (cudaStream_t)stream);
  return launched("repack");
}

energon_status energon_final_unpack(int32_t out_dtype, const float* X, const int32_t* unpack_idx, int32_t cells,
                                    int32_t H, const float* ln_g, const float* ln_b, float eps, int32_t apply_ln,
                                    void* out, void* stream) {
  if (!X || !unpack_idx || !out || (apply_ln && (!ln_g || !ln_b))) return fail(nullptr, ENERGON_ERR_ARG, "NULL argument");
  if (out_dtype != ENERGON_DTYPE_F32 && out_dtype != ENERGON_DTYPE_BF16)
    return fail(nullptr, ENERGON_ERR_ARG, "out_dtype must be F32 or BF16");
  if (cells < 0 || H < 4 || H % 4 || H > 12288 || !(eps > 0.f)) return fail(nullptr, ENERGON_ERR_ARG, "bad arguments");
  if (out_dtype == ENERGON_DTYPE_F32)
    launch_final_ln_unpack<float>(X, unpack_idx, 0, cells, H, ln_g, ln_b, eps, apply_ln, (float*)out, (cudaStream_t)stream);
  else
    launch_final_ln_unpack<bf16>(X, unpack_idx, 0, cells, H, ln_g, ln_b, eps, apply_ln, (bf16*)out, (cudaStream_t)stream);
  return launched("final_unpack");
}

}  // extern "C"

"""Thin ctypes binding of the energon C ABI (include/energon.h).

Argument marshalling only: every step of the forward pass runs in the CUDA kernels of
libenergon.so.  torch is used for device memory, streams and process groups.  There is no
fallback: if the library is missing or the device is not a B200 this module raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "lib", "libenergon.so")

ENERGON_OK = 0
STATUS = {0: "ENERGON_OK", -1: "ENERGON_ERR_ARG", -2: "ENERGON_ERR_CONFIG", -3: "ENERGON_ERR_SHAPE",
          -4: "ENERGON_ERR_LENGTH", -5: "ENERGON_ERR_TOKEN", -6: "ENERGON_ERR_CAPACITY",
          -7: "ENERGON_ERR_NOT_LOADED", -8: "ENERGON_ERR_CUDA", -9: "ENERGON_ERR_NCCL", -10: "ENERGON_ERR_OOM"}
DTYPE_F32, DTYPE_BF16, DTYPE_F64 = 0, 1, 2
FULL, RANK_SHARD = 0, 1
MAX_BATCH = 1024
OPT_DRCE = 1
OPT_TP_SP = 2
OPT_GRAPH = 3
OPT_RING_NUMERICS = 4
OPT_LN_FUSE = 5
STAGE_PACKED, STAGE_FINAL = 0, 1
COMM_NCCL, COMM_P2P = 0, 1
LAYER_TENSORS = ("wq", "wk", "wv", "wo", "bq", "bk", "bv", "bo",
                 "w1", "b1", "w2", "b2", "ln1_g", "ln1_b", "ln2_g", "ln2_b")

# symbols include/energon.h declares (checked by tests/test_abi.py)
EXPORTS = ("energon_get_unique_id", "energon_init", "energon_init_local_group", "energon_load_embeddings",
           "energon_load_layer_weights", "energon_forward", "energon_forward_group", "energon_forward_hidden",
           "energon_sync", "energon_get_stats", "energon_last_error", "energon_status_string", "energon_destroy",
           "energon_index_maps", "energon_gemm", "energon_attention", "energon_set_profiling", "energon_get_profile",
           "energon_shard_plan", "energon_set_option", "energon_pmep_plan", "energon_offload_layers",
           "energon_stage_plan", "energon_forward_stage", "energon_forward_stage_group", "energon_p2p_handle",
           "energon_p2p_connect", "energon_unpack_qkv", "energon_repack", "energon_final_unpack")


class EnergonError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("num_layers", "hidden", "num_heads", "ffn", "vocab", "max_seq",
                                              "causal", "dtype", "drce", "tp_size", "tp_rank", "device",
                                              "max_tokens", "final_ln")] + [("ln_eps", ctypes.c_float), ("comm", ctypes.c_int32)]


class LayerWeights(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in LAYER_TENSORS]


class Shard(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("head0", "heads", "qkv_col0", "qkv_cols", "ffn_col0", "ffn_cols")]


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("forwards", "allreduce_calls", "kernel_launches", "last_tokens",
                                              "last_rows", "weight_bytes", "workspace_bytes", "prefetch_bytes",
                                              "fused_exchanges", "graphs_recorded")]


class Profile(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("gemm_ms", "attn_ms", "mem_ms", "comm_ms", "gemm_flops",
                                               "attn_flops", "mem_bytes", "comm_bytes")] + \
               [(n, ctypes.c_int64) for n in ("gemm_launches", "attn_launches", "mem_launches", "comm_calls")]


_lib = None


def load_library(path: str = SO_PATH):
    """dlopen libenergon.so and declare every prototype.  Raises if it is absent (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -m paper_2209_02341_b200.build` "
                          "(the CUDA library is required; there is no CPU fallback)")
    L = ctypes.CDLL(path)
    P, I32, St = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int
    L.energon_get_unique_id.argtypes = [P]
    L.energon_init.argtypes = [ctypes.POINTER(Config), P, ctypes.POINTER(P)]
    L.energon_init_local_group.argtypes = [ctypes.POINTER(Config), I32, ctypes.POINTER(P)]
    L.energon_load_embeddings.argtypes = [P, P, P, P, P, I32, I32]
    L.energon_load_layer_weights.argtypes = [P, I32, ctypes.POINTER(LayerWeights), I32, I32, I32]
    L.energon_forward.argtypes = [P, P, ctypes.POINTER(ctypes.c_int32), I32, I32, P, P]
    L.energon_forward_group.argtypes = [ctypes.POINTER(P), I32, P, ctypes.POINTER(ctypes.c_int32), I32, I32, P, P]
    L.energon_forward_hidden.argtypes = [P, P, ctypes.POINTER(ctypes.c_int32), I32, I32, I32, I32, I32, P, P]
    L.energon_sync.argtypes = [P]
    L.energon_get_stats.argtypes = [P, ctypes.POINTER(Stats)]
    L.energon_last_error.argtypes = [P]
    L.energon_last_error.restype = ctypes.c_char_p
    L.energon_status_string.argtypes = [St]
    L.energon_status_string.restype = ctypes.c_char_p
    L.energon_destroy.argtypes = [P]
    L.energon_destroy.restype = None
    L.energon_index_maps.argtypes = [ctypes.POINTER(ctypes.c_int32), I32, I32, P, P, P, P, P]
    L.energon_gemm.argtypes = [I32, P, P, P, P, I32, I32, I32, I32, P]
    L.energon_attention.argtypes = [I32, P, P, P, P, ctypes.POINTER(ctypes.c_int32), I32, I32, I32, I32, I32, P]
    L.energon_unpack_qkv.argtypes = [I32, P, P, I32, I32, I32, I32, P, P, P, P]
    L.energon_repack.argtypes = [I32, P, P, P, I32, I32, I32, I32, P, P]
    L.energon_final_unpack.argtypes = [I32, P, P, I32, I32, P, P, ctypes.c_float, I32, P, P]
    L.energon_shard_plan.argtypes = [ctypes.POINTER(Config), ctypes.POINTER(Shard)]
    L.energon_set_profiling.argtypes = [P, I32]
    L.energon_set_option.argtypes = [P, I32, I32]
    L.energon_pmep_plan.argtypes = [I32, I32, ctypes.POINTER(ctypes.c_int32)]
    L.energon_offload_layers.argtypes = [P, ctypes.POINTER(ctypes.c_int32), I32, I32, I32, I32]
    L.energon_get_profile.argtypes = [P, ctypes.POINTER(Profile)]
    L.energon_stage_plan.argtypes = [I32, I32, ctypes.POINTER(ctypes.c_int32)]
    L.energon_p2p_handle.argtypes = [P, P]
    L.energon_p2p_connect.argtypes = [P, P]
    L.energon_forward_stage.argtypes = [P, P, P, ctypes.POINTER(ctypes.c_int32), I32, I32, I32, I32, I32, P, P]
    L.energon_forward_stage_group.argtypes = [ctypes.POINTER(P), I32, P, P, ctypes.POINTER(ctypes.c_int32), I32, I32,
                                              I32, I32, I32, P, P]
    for name in EXPORTS:
        fn = getattr(L, name)
        if fn.restype is ctypes.c_int:  # default restype: energon_status
            fn.restype = St
    _lib = L
    return L


def _check(status: int, ctx=None):
    if status != ENERGON_OK:
        msg = load_library().energon_last_error(ctx).decode()
        raise EnergonError(status, msg)


def _lens(seq_lens):
    arr = (ctypes.c_int32 * len(seq_lens))(*[int(x) for x in seq_lens])
    return arr


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _src_dtype(t):
    import torch
    return {torch.float32: DTYPE_F32, torch.bfloat16: DTYPE_BF16, torch.float64: DTYPE_F64}[t.dtype]


def make_config(num_layers, hidden, num_heads, ffn, vocab, max_seq, max_tokens, dtype="bf16", causal=1, drce=1,
                tp_size=1, tp_rank=0, device=0, final_ln=1, ln_eps=1e-5, comm=0) -> Config:
    return Config(num_layers, hidden, num_heads, ffn, vocab, max_seq, causal,
                  DTYPE_BF16 if dtype == "bf16" else DTYPE_F32, drce, tp_size, tp_rank, device, max_tokens,
                  final_ln, ln_eps, comm)


# ----------------------------------------------------------------------------- ABI wrappers (same names)
def energon_shard_plan(cfg: Config) -> dict:
    sh = Shard()
    _check(load_library().energon_shard_plan(ctypes.byref(cfg), ctypes.byref(sh)))
    return {n: getattr(sh, n) for n, _ in Shard._fields_}


def energon_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load_library().energon_get_unique_id(buf))
    return buf.raw


def energon_init(cfg: Config, unique_id: bytes | None = None) -> ctypes.c_void_p:
    ctx = ctypes.c_void_p()
    uid = ctypes.create_string_buffer(unique_id, 128) if unique_id is not None else None
    _check(load_library().energon_init(ctypes.byref(cfg), uid, ctypes.byref(ctx)))
    return ctx


def energon_init_local_group(cfg: Config, k: int) -> list:
    arr = (ctypes.c_void_p * k)()
    _check(load_library().energon_init_local_group(ctypes.byref(cfg), k, arr))
    return [ctypes.c_void_p(arr[i]) for i in range(k)]


def energon_load_embeddings(ctx, tok_emb, pos_emb, lnf_g, lnf_b):
    """torch tensors (all the same dtype, all on the GPU or all on the host)."""
    on_dev = int(tok_emb.is_cuda)
    _check(load_library().energon_load_embeddings(ctx, _ptr(tok_emb), _ptr(pos_emb), _ptr(lnf_g), _ptr(lnf_b),
                                                  _src_dtype(tok_emb), on_dev), ctx)


def energon_load_layer_weights(ctx, layer: int, w: dict, layout: int = FULL):
    """w: dict name -> torch tensor ([in, out] row-major, one dtype, one device)."""
    first = w["wq"]
    lw = LayerWeights(*[w[n].data_ptr() for n in LAYER_TENSORS])
    _check(load_library().energon_load_layer_weights(ctx, layer, ctypes.byref(lw), _src_dtype(first),
                                                     int(first.is_cuda), layout), ctx)


def energon_forward(ctx, tokens, seq_lens, out, stream=None):
    B, S = tokens.shape
    _check(load_library().energon_forward(ctx, _ptr(tokens), _lens(seq_lens), B, S, _ptr(out), _stream(stream)), ctx)


def energon_forward_group(ctxs, tokens, seq_lens, out, stream=None):
    B, S = tokens.shape
    arr = (ctypes.c_void_p * len(ctxs))(*[c.value for c in ctxs])
    _check(load_library().energon_forward_group(arr, len(ctxs), _ptr(tokens), _lens(seq_lens), B, S, _ptr(out),
                                                _stream(stream)), ctxs[0])


def energon_forward_hidden(ctx, x, seq_lens, layer_begin, layer_end, apply_final_ln, out, stream=None):
    B, S, _ = x.shape
    _check(load_library().energon_forward_hidden(ctx, _ptr(x), _lens(seq_lens), B, S, layer_begin, layer_end,
                                                 int(apply_final_ln), _ptr(out), _stream(stream)), ctx)


def energon_stage_plan(num_layers: int, pp_size: int) -> list:
    """Stage layer ranges [(begin, end), ...] (host only)."""
    out = (ctypes.c_int32 * (max(pp_size, 0) + 1))()
    _check(load_library().energon_stage_plan(num_layers, pp_size, out))
    return [(out[i], out[i + 1]) for i in range(pp_size)]


def energon_forward_stage(ctx, seq_lens, max_len, layer_begin, layer_end, out_kind, out, tokens=None, x=None,
                          stream=None):
    """One pipeline stage: tokens [B, S] (first stage) or x fp32 [rows, H] -> out (packed rows or final)."""
    _check(load_library().energon_forward_stage(ctx, _ptr(tokens), _ptr(x), _lens(seq_lens), len(seq_lens), max_len,
                                                layer_begin, layer_end, out_kind, _ptr(out), _stream(stream)), ctx)


def energon_forward_stage_group(ctxs, seq_lens, max_len, layer_begin, layer_end, out_kind, out, tokens=None, x=None,
                                stream=None):
    arr = (ctypes.c_void_p * len(ctxs))(*[c.value for c in ctxs])
    _check(load_library().energon_forward_stage_group(arr, len(ctxs), _ptr(tokens), _ptr(x), _lens(seq_lens),
                                                      len(seq_lens), max_len, layer_begin, layer_end, out_kind,
                                                      _ptr(out), _stream(stream)), ctxs[0])


def energon_p2p_handle(ctx) -> bytes:
    """64-byte CUDA IPC handle of this rank's exchange region (cfg.comm = COMM_P2P)."""
    buf = ctypes.create_string_buffer(64)
    _check(load_library().energon_p2p_handle(ctx, buf), ctx)
    return buf.raw


def energon_p2p_connect(ctx, handles):
    """handles: the k ranks' 64-byte handles in rank order."""
    blob = b"".join(handles)
    buf = ctypes.create_string_buffer(blob, len(blob))
    _check(load_library().energon_p2p_connect(ctx, buf), ctx)


def energon_sync(ctx):
    _check(load_library().energon_sync(ctx), ctx)


def energon_get_stats(ctx) -> dict:
    s = Stats()
    _check(load_library().energon_get_stats(ctx, ctypes.byref(s)), ctx)
    return {n: getattr(s, n) for n, _ in Stats._fields_}


def energon_pmep_plan(num_layers: int, resident: int) -> list:
    m = num_layers - resident
    out = (ctypes.c_int32 * max(m, 1))()
    _check(load_library().energon_pmep_plan(num_layers, resident, out))
    return [out[i] for i in range(m)]


def energon_offload_layers(ctx, layers, slots: int = 1, pool: int = 0, peer_device: int = -1):
    arr = (ctypes.c_int32 * max(len(layers), 1))(*layers)
    _check(load_library().energon_offload_layers(ctx, arr, len(layers), slots, pool, peer_device), ctx)


def energon_set_option(ctx, option: int, value: int):
    _check(load_library().energon_set_option(ctx, option, int(value)), ctx)


def energon_set_profiling(ctx, enable: bool):
    _check(load_library().energon_set_profiling(ctx, int(enable)), ctx)


def energon_get_profile(ctx) -> dict:
    p = Profile()
    _check(load_library().energon_get_profile(ctx, ctypes.byref(p)), ctx)
    return {n: getattr(p, n) for n, _ in Profile._fields_}


def energon_last_error(ctx=None) -> str:
    return load_library().energon_last_error(ctx).decode()


def energon_destroy(ctx):
    load_library().energon_destroy(ctx)


def energon_index_maps(seq_lens, max_len, offsets, pack_idx, pos, unpack_idx, stream=None):
    _check(load_library().energon_index_maps(_lens(seq_lens), len(seq_lens), max_len, _ptr(offsets), _ptr(pack_idx),
                                             _ptr(pos), _ptr(unpack_idx), _stream(stream)))


def energon_gemm(A, W, bias, D, epilogue=0, stream=None):
    """D[M,N] = A[M,K] . W[N,K]^T (+bias) (gelu): fp32 SIMT or bf16 tcgen05 by A's dtype."""
    import torch
    M, K = A.shape
    N = W.shape[0]
    dt = DTYPE_BF16 if A.dtype == torch.bfloat16 else DTYPE_F32
    _check(load_library().energon_gemm(dt, _ptr(A), _ptr(W), _ptr(bias), _ptr(D), M, N, K, epilogue,
                                       _stream(stream)))


def energon_attention(Q, K, V, O, seq_lens, causal=1, stream=None):
    """a6 on [B, heads, S, d] tensors (fp32 SIMT or bf16 tensor-core by Q's dtype)."""
    import torch
    B, hk, S, d = Q.shape
    dt = DTYPE_BF16 if Q.dtype == torch.bfloat16 else DTYPE_F32
    _check(load_library().energon_attention(dt, _ptr(Q), _ptr(K), _ptr(V), _ptr(O), _lens(seq_lens), B, hk, S, d,
                                            causal, _stream(stream)))


def _act_dtype(t):
    import torch
    return DTYPE_BF16 if t.dtype == torch.bfloat16 else DTYPE_F32


def energon_unpack_qkv(QKV, pack_idx, max_len, heads, head_dim, Q, K, V, stream=None):
    """a5: packed QKV [T, 3*heads*head_dim] -> Q, K, V [B, heads, max_len, head_dim] (pack_idx None: identity)."""
    T = QKV.shape[0]
    _check(load_library().energon_unpack_qkv(_act_dtype(QKV), _ptr(QKV), _ptr(pack_idx), T, max_len, heads, head_dim,
                                             _ptr(Q), _ptr(K), _ptr(V), _stream(stream)))


def energon_repack(O, pack_idx, unpack_idx, T, C, stream=None):
    """a7: O [B, heads, max_len, head_dim] -> packed C [T, heads*head_dim]."""
    B, hk, S, d = O.shape
    _check(load_library().energon_repack(_act_dtype(O), _ptr(O), _ptr(pack_idx), _ptr(unpack_idx), T, S, hk, d, _ptr(C),
                                         _stream(stream)))


def energon_final_unpack(X, unpack_idx, out, ln_g=None, ln_b=None, eps=1e-5, apply_ln=False, stream=None):
    """a13: out [cells, H] = (LN of) X[unpack_idx[cell]], pad cells exactly 0."""
    cells, H = out.shape[0] * (out.shape[1] if out.dim() == 3 else 1), X.shape[-1]
    _check(load_library().energon_final_unpack(_act_dtype(out), _ptr(X), _ptr(unpack_idx), cells, H, _ptr(ln_g),
                                               _ptr(ln_b), float(eps), int(apply_ln), _ptr(out), _stream(stream)))

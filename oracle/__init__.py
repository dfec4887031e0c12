"""ctypes front-end of the fp64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py -- never by the product
package ``paper_2209_02341_b200``.  It shares no code with the CUDA path.

Every function cites the passage it follows in oracle.c; the pins that tie it
to the paper are in tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")

LAYER_TENSORS = ("wq", "wk", "wv", "wo", "bq", "bk", "bv", "bo",
                 "w1", "b1", "w2", "b2", "ln1_g", "ln1_b", "ln2_g", "ln2_b")


class Cfg(ctypes.Structure):
    _fields_ = [("L", ctypes.c_int32), ("H", ctypes.c_int32), ("h", ctypes.c_int32),
                ("F", ctypes.c_int32), ("causal", ctypes.c_int32), ("eps", ctypes.c_double)]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (fp64, -O2, OpenMP, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int)


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        L.oracle_matmul.argtypes = [_D, _D, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _D]
        L.oracle_layernorm.argtypes = [_D, ctypes.c_int64, ctypes.c_int64, _D, _D, ctypes.c_double, _D]
        L.oracle_gelu.argtypes = [ctypes.c_double]
        L.oracle_gelu.restype = ctypes.c_double
        L.oracle_attention.argtypes = [_D, _D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       _I, ctypes.c_int, _D]
        L.oracle_index_maps.argtypes = [_I, ctypes.c_int, ctypes.c_int, _I, _I, _I, _I]
        L.oracle_index_maps.restype = ctypes.c_int64
        PP = ctypes.POINTER(_D)
        L.oracle_layer_padded.argtypes = [ctypes.POINTER(Cfg), PP, _D, _I, ctypes.c_int, ctypes.c_int]
        L.oracle_layers_padded.argtypes = [ctypes.POINTER(Cfg), PP, ctypes.c_int, ctypes.c_int, _D, _I,
                                           ctypes.c_int, ctypes.c_int]
        fwd = [ctypes.POINTER(Cfg), PP, _D, _D, _D, _D, _I, _I, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D]
        L.oracle_forward_padded.argtypes = fwd
        L.oracle_forward_drce.argtypes = fwd
        L.oracle_forward_tp.argtypes = [ctypes.POINTER(Cfg), ctypes.c_int] + fwd[1:] + [
            ctypes.POINTER(ctypes.c_int64)]
        L.oracle_embed.argtypes = [ctypes.POINTER(Cfg), _D, _D, _I, ctypes.c_int, ctypes.c_int, _D]
        L.oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _d(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_D)


def _i(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_I)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def make_cfg(L, H, h, F, causal=1, eps=1e-5) -> Cfg:
    return Cfg(L, H, h, F, causal, eps)


class _Weights:
    """Keeps the fp64 arrays alive and exposes the (L*16) pointer table."""

    def __init__(self, layers):
        self.arrays = []
        ptrs = []
        for lw in layers:
            for name in LAYER_TENSORS:
                a = f64(lw[name])
                self.arrays.append(a)
                ptrs.append(a.ctypes.data_as(_D))
        self.table = (_D * len(ptrs))(*ptrs)


# ----------------------------------------------------------------------------- primitives
def matmul(A, W) -> np.ndarray:
    A, W = f64(A), f64(W)
    M, K = A.shape
    K2, N = W.shape
    assert K == K2
    C = np.empty((M, N))
    lib().oracle_matmul(_d(A), _d(W), M, K, N, _d(C))
    return C


def layernorm(x, g, b, eps=1e-5) -> np.ndarray:
    x = f64(x)
    H = x.shape[-1]
    rows = x.size // H
    y = np.empty_like(x)
    lib().oracle_layernorm(_d(x), rows, H, _d(f64(g)), _d(f64(b)), eps, _d(y))
    return y


def gelu(x: float) -> float:
    return lib().oracle_gelu(float(x))


def attention(Q, K, V, h, lens, causal=1) -> np.ndarray:
    Q, K, V = f64(Q), f64(K), f64(V)
    B, S, H = Q.shape
    C = np.empty_like(Q)
    lib().oracle_attention(_d(Q), _d(K), _d(V), B, S, H, h, _i(i32(lens)), causal, _d(C))
    return C


def index_maps(lens, S):
    lens = i32(lens)
    B = lens.shape[0]
    offsets = np.zeros(B + 1, np.int32)
    pack_idx = np.zeros(B * S, np.int32)
    pos = np.zeros(B * S, np.int32)
    unpack_idx = np.zeros(B * S, np.int32)
    T = lib().oracle_index_maps(_i(lens), B, S, _i(offsets), _i(pack_idx), _i(pos), _i(unpack_idx))
    return offsets, pack_idx[:T].copy(), pos[:T].copy(), unpack_idx


# ----------------------------------------------------------------------------- stacks
def layer_padded(cfg: Cfg, layer: dict, X, lens) -> np.ndarray:
    X = f64(X).copy()
    B, S, _ = X.shape
    w = _Weights([layer])
    lib().oracle_layer_padded(ctypes.byref(cfg), w.table, _d(X), _i(i32(lens)), B, S)
    return X


def layers_padded(cfg: Cfg, layers: list, l0: int, l1: int, X, lens) -> np.ndarray:
    """Layers [l0, l1) of the stack on the padded residual stream X [B,S,H]."""
    X = f64(X).copy()
    B, S, _ = X.shape
    w = _Weights(layers)
    lib().oracle_layers_padded(ctypes.byref(cfg), w.table, l0, l1, _d(X), _i(i32(lens)), B, S)
    return X


def embed(cfg: Cfg, emb: dict, tok) -> np.ndarray:
    tok = i32(tok)
    B, S = tok.shape
    X = np.empty((B, S, cfg.H))
    lib().oracle_embed(ctypes.byref(cfg), _d(f64(emb["tok_emb"])), _d(f64(emb["pos_emb"])), _i(tok), B, S,
                       _d(X))
    return X


def _fwd(fn, cfg, layers, emb, tok, lens, final_ln, extra_pre=(), extra_post=()):
    tok = i32(tok)
    B, S = tok.shape
    w = _Weights(layers)
    Y = np.empty((B, S, cfg.H))
    te, pe = f64(emb["tok_emb"]), f64(emb["pos_emb"])
    g, b = f64(emb["lnf_g"]), f64(emb["lnf_b"])
    fn(ctypes.byref(cfg), *extra_pre, w.table, _d(te), _d(pe), _d(g), _d(b), _i(tok), _i(i32(lens)), B, S,
       int(final_ln), _d(Y), *extra_post)
    return Y


def forward_padded(cfg: Cfg, layers: list, emb: dict, tok, lens, final_ln=True) -> np.ndarray:
    """SPEC.md:147-155 serial_forward on the padded batch -> Y [B,S,H]."""
    return _fwd(lib().oracle_forward_padded, cfg, layers, emb, tok, lens, final_ln)


def forward_drce(cfg: Cfg, layers: list, emb: dict, tok, lens, final_ln=True) -> np.ndarray:
    """PAPER.md:358-373 DRCE on the CPU; pad rows of Y are exactly 0."""
    return _fwd(lib().oracle_forward_drce, cfg, layers, emb, tok, lens, final_ln)


def forward_tp(cfg: Cfg, k: int, layers: list, emb: dict, tok, lens, final_ln=True):
    """PAPER.md:281-293 1-D TP over k simulated ranks -> (Y, allreduce_count)."""
    cnt = ctypes.c_int64(0)
    Y = _fwd(lib().oracle_forward_tp, cfg, layers, emb, tok, lens, final_ln, extra_pre=(ctypes.c_int(k),),
             extra_post=(ctypes.byref(cnt),))
    return Y, cnt.value


def num_threads() -> int:
    return lib().oracle_num_threads()

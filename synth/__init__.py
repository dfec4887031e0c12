"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module draws inputs only (SURVEY.md 8(d) "Synthetic inputs"); it holds none
of the method's arithmetic, so both the oracle (``oracle/``) and the CUDA path may
consume what it produces.  The counter-based generator itself lives in
``synth/synth.h`` and is compiled twice: a host library (gcc, OpenMP) and a
device library (nvcc), which produce bit-identical values.

Distributions:
  weight matrices and biases  U[-0.02, 0.02]
  LayerNorm gamma             1 + U[-0.1, 0.1]   (so a gamma/beta swap cannot pass)
  LayerNorm beta              U[-0.1, 0.1]
  token / position embeddings U[-0.02, 0.02]
In bf16 mode every value is rounded to bf16 (RNE) *before* either side consumes it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_HOST_SO = os.path.join(_HERE, "libsynth_host.so")
_DEV_SO = os.path.join(_HERE, "libsynth_dev.so")

# energon_layer_weights order (include/energon.h); ids are the stream "b" values.
LAYER_TENSORS = ("wq", "wk", "wv", "wo", "bq", "bk", "bv", "bo",
                 "w1", "b1", "w2", "b2", "ln1_g", "ln1_b", "ln2_g", "ln2_b")
EMB_TENSORS = ("tok_emb", "pos_emb", "lnf_g", "lnf_b")
EMB_STREAM = 1 << 20

DT_F32, DT_BF16, DT_F64 = 0, 1, 2

SM64_MASK = (1 << 64) - 1


def sm64(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & SM64_MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & SM64_MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & SM64_MASK
    return z ^ (z >> 31)


def stream(seed: int, a: int, b: int) -> int:
    return sm64(sm64(sm64(seed) ^ a) ^ b)


def u01(x: int) -> float:
    return (sm64(x & SM64_MASK) >> 11) * (2.0 ** -53)


# ----------------------------------------------------------------------------- build
def build(force: bool = False, device: bool = True) -> None:
    """Compile the host (gcc) and, if requested, device (nvcc) generator libraries."""
    src_h = os.path.join(_HERE, "synth_host.c")
    if force or not os.path.exists(_HOST_SO) or os.path.getmtime(_HOST_SO) < max(
            os.path.getmtime(src_h), os.path.getmtime(os.path.join(_HERE, "synth.h"))):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", _HOST_SO, src_h])
    if device:
        src_d = os.path.join(_HERE, "synth_dev.cu")
        if force or not os.path.exists(_DEV_SO) or os.path.getmtime(_DEV_SO) < max(
                os.path.getmtime(src_d), os.path.getmtime(os.path.join(_HERE, "synth.h"))):
            subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                                   "-Xcompiler", "-fPIC", "-shared", "-o", _DEV_SO, src_d])


_host_lib = None
_dev_lib = None


def _host():
    global _host_lib
    if _host_lib is None:
        if not os.path.exists(_HOST_SO):
            build(device=False)
        lib = ctypes.CDLL(_HOST_SO)
        lib.synth_fill_host.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64,
                                        ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_int]
        lib.synth_fill_host.restype = None
        _host_lib = lib
    return _host_lib


def _dev():
    global _dev_lib
    if _dev_lib is None:
        if not os.path.exists(_DEV_SO):
            build(device=True)
        lib = ctypes.CDLL(_DEV_SO)
        lib.synth_fill_device.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64,
                                          ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double,
                                          ctypes.c_double, ctypes.c_int, ctypes.c_void_p]
        lib.synth_fill_device.restype = ctypes.c_int
        _dev_lib = lib
    return _dev_lib


# ----------------------------------------------------------------------------- tensors
def tensor_dist(name: str):
    """(scale, offset) of the uniform distribution of a named tensor."""
    if name.endswith("_g"):
        return 0.1, 1.0
    if name.endswith("_b") and name.startswith("ln"):
        return 0.1, 0.0
    return 0.02, 0.0


def layer_shapes(H: int, F: int) -> dict:
    """Full (unsharded) shapes, [in, out] row-major for matrices."""
    return {"wq": (H, H), "wk": (H, H), "wv": (H, H), "wo": (H, H),
            "bq": (H,), "bk": (H,), "bv": (H,), "bo": (H,),
            "w1": (H, F), "b1": (F,), "w2": (F, H), "b2": (H,),
            "ln1_g": (H,), "ln1_b": (H,), "ln2_g": (H,), "ln2_b": (H,)}


def emb_shapes(H: int, V: int, max_seq: int) -> dict:
    return {"tok_emb": (V, H), "pos_emb": (max_seq, H), "lnf_g": (H,), "lnf_b": (H,)}


def host_tensor(shape, seed, a, b, scale, offset, bf16: bool, dtype=np.float64) -> np.ndarray:
    """Generate on the host.  dtype float64/float32 (value widened exactly) or 'bf16' (uint16 bits)."""
    n = int(np.prod(shape)) if len(shape) else 1
    if dtype == "bf16":
        out = np.empty(n, dtype=np.uint16)
        code = DT_BF16
    elif dtype == np.float32:
        out = np.empty(n, dtype=np.float32)
        code = DT_F32
    else:
        out = np.empty(n, dtype=np.float64)
        code = DT_F64
    _host().synth_fill_host(out.ctypes.data, n, code, seed, a, b, scale, offset, int(bf16))
    return out.reshape(shape)


def layer_tensor_host(name, layer, H, F, seed, bf16, dtype=np.float64):
    shape = layer_shapes(H, F)[name]
    scale, offset = tensor_dist(name)
    return host_tensor(shape, seed, 2 + layer, LAYER_TENSORS.index(name), scale, offset, bf16, dtype)


def emb_tensor_host(name, H, V, max_seq, seed, bf16, dtype=np.float64):
    shape = emb_shapes(H, V, max_seq)[name]
    scale, offset = tensor_dist(name)
    return host_tensor(shape, seed, EMB_STREAM, EMB_TENSORS.index(name), scale, offset, bf16, dtype)


def fill_device(t, seed, a, b, scale, offset, bf16: bool, stream=None) -> None:
    """Fill a CUDA torch tensor (float32 / bfloat16 / float64) in place, same bits as host_tensor."""
    import torch
    code = {torch.float32: DT_F32, torch.bfloat16: DT_BF16, torch.float64: DT_F64}[t.dtype]
    if stream is None:
        stream = torch.cuda.current_stream(t.device).cuda_stream
    rc = _dev().synth_fill_device(t.data_ptr(), t.numel(), code, seed, a, b, scale, offset, int(bf16),
                                  ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"synth_fill_device failed: cuda error {rc}")


def layer_tensor_device(name, layer, H, F, seed, bf16, torch_dtype, device="cuda"):
    import torch
    shape = layer_shapes(H, F)[name]
    t = torch.empty(shape, dtype=torch_dtype, device=device)
    scale, offset = tensor_dist(name)
    fill_device(t, seed, 2 + layer, LAYER_TENSORS.index(name), scale, offset, bf16)
    return t


def emb_tensor_device(name, H, V, max_seq, seed, bf16, torch_dtype, device="cuda"):
    import torch
    shape = emb_shapes(H, V, max_seq)[name]
    t = torch.empty(shape, dtype=torch_dtype, device=device)
    scale, offset = tensor_dist(name)
    fill_device(t, seed, EMB_STREAM, EMB_TENSORS.index(name), scale, offset, bf16)
    return t


# ----------------------------------------------------------------------------- batches
def random_lengths(B: int, S: int, seed: int) -> list:
    """Configs 1-2: lens_b = 1 + floor(u01 * S)."""
    s = stream(seed, 0, 0)
    return [1 + int(u01(s + b) * S) for b in range(B)]


def exact_p_lengths(B: int, S: int, p: float, seed: int) -> list:
    """Configs 3-5: padding ratio exactly p (SURVEY.md 8(d) 'Exact-p')."""
    mu = (1.0 - p) * S
    w = 2.0 * min(mu - 1.0, S - mu)
    s = stream(seed, 0, 0)
    lens = []
    for b in range(B):
        v = int(round(mu + (u01(s + b) - 0.5) * w))
        lens.append(min(max(v, 1), S))
    target = int(round((1.0 - p) * B * S))
    b = 0
    guard = 0
    while sum(lens) != target:
        if sum(lens) < target and lens[b] < S:
            lens[b] += 1
        elif sum(lens) > target and lens[b] > 1:
            lens[b] -= 1
        b = (b + 1) % B
        guard += 1
        if guard > 100 * B * S:
            raise RuntimeError("exact_p_lengths did not converge")
    return lens


def paper_lengths(B: int, S: int, p: float) -> list:
    """Paper regime: every valid length = (1-p) S (PAPER.md:569 'valid length half of padding size')."""
    return [max(1, int(round((1.0 - p) * S)))] * B


def tokens(B: int, S: int, V: int, lens, seed: int) -> np.ndarray:
    """tok[b,s] = 1 + floor(u01 * (V-1)) for s < lens[b], pad id 0 elsewhere."""
    s0 = stream(seed, 1, 0)
    out = np.zeros((B, S), dtype=np.int32)
    for b in range(B):
        for s in range(lens[b]):
            out[b, s] = 1 + int(u01(s0 + b * S + s) * (V - 1))
    return out


def model_host(L, H, F, V, max_seq, seed, bf16, layer_ids=None):
    """fp64 host copies of every weight (values already bf16-rounded if bf16).

    Returns (layers, emb): layers = list of dicts keyed by LAYER_TENSORS
    (only for layer_ids if given), emb = dict keyed by EMB_TENSORS.
    """
    ids = range(L) if layer_ids is None else layer_ids
    layers = [{n: layer_tensor_host(n, l, H, F, seed, bf16) for n in LAYER_TENSORS} for l in ids]
    emb = {n: emb_tensor_host(n, H, V, max_seq, seed, bf16) for n in EMB_TENSORS}
    return layers, emb


# BASELINE.json configs, concretised in SURVEY.md 8(d): model shapes and batch recipes.
SHAPES = {
    "tiny": dict(L=1, H=64, h=4, F=256, V=256, max_seq=16),                 # config 1
    "gpt2s": dict(L=12, H=768, h=12, F=3072, V=50257, max_seq=1024),        # config 2
    "gpt3_13b": dict(L=40, H=5120, h=40, F=20480, V=50257, max_seq=2048),   # config 3
    "opt30b": dict(L=48, H=7168, h=56, F=28672, V=50272, max_seq=2048),     # config 4
    "opt66b": dict(L=64, H=9216, h=72, F=36864, V=50272, max_seq=2048),     # config 5
}
BATCHES = {
    "tiny": dict(B=4, S=16, lengths="random", p=None),
    "gpt2s": dict(B=32, S=128, lengths="random", p=None),
    "gpt3_13b": dict(B=16, S=512, lengths="exact_p", p=0.5),
    "opt30b": dict(B=32, S=1024, lengths="exact_p", p=0.5),
    "opt66b": dict(B=32, S=1024, lengths="exact_p", p=0.5),
}


def batch_lengths(name: str, seed: int, p=None, regime: str | None = None) -> list:
    cfg = BATCHES[name]
    B, S = cfg["B"], cfg["S"]
    mode = regime or cfg["lengths"]
    if mode == "random":
        return random_lengths(B, S, seed)
    pp = cfg["p"] if p is None else p
    if mode == "paper":
        return paper_lengths(B, S, pp)
    return exact_p_lengths(B, S, pp, seed)

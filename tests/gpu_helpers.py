"""Shared helpers of the GPU parity tests: build an engine from seeded synthetic weights (device
generator) and the bit-identical fp64 host copy the oracle consumes (host generator)."""
from __future__ import annotations

import numpy as np

import synth

SHAPES = synth.SHAPES


def max_abs_rel(y_hat, y, lens):
    """||y_hat - y||_inf / ||y||_inf over valid positions."""
    num = 0.0
    den = 0.0
    for b, n in enumerate(lens):
        num = max(num, float(np.abs(np.asarray(y_hat[b, :n], dtype=np.float64) - y[b, :n]).max()))
        den = max(den, float(np.abs(y[b, :n]).max()))
    return num / den


def torch_dtype(dtype):
    import torch
    return torch.bfloat16 if dtype == "bf16" else torch.float32


def load_engine(ctxs, shape, seed, dtype, layers=None):
    """Generate every weight on the device (synth) and load it, unsharded, into each context."""
    import torch

    from paper_2209_02341_b200 import energon
    bf16 = dtype == "bf16"
    tdt = torch_dtype(dtype)
    H, F, V, ms = shape["H"], shape["F"], shape["V"], shape["max_seq"]
    emb = {n: synth.emb_tensor_device(n, H, V, ms, seed, bf16, tdt) for n in synth.EMB_TENSORS}
    for c in ctxs:
        energon.energon_load_embeddings(c, emb["tok_emb"], emb["pos_emb"], emb["lnf_g"], emb["lnf_b"])
    del emb
    for l in (range(shape["L"]) if layers is None else layers):
        w = {n: synth.layer_tensor_device(n, l, H, F, seed, bf16, tdt) for n in synth.LAYER_TENSORS}
        for c in ctxs:
            energon.energon_load_layer_weights(c, l, w)
        del w
    torch.cuda.synchronize()


def make_engine(shape, seed, dtype, max_tokens, k=1, drce=1, causal=1, final_ln=1, L=None):
    from paper_2209_02341_b200 import energon
    Lx = shape["L"] if L is None else L
    cfg = energon.make_config(Lx, shape["H"], shape["h"], shape["F"], shape["V"], shape["max_seq"], max_tokens,
                              dtype=dtype, causal=causal, drce=drce, final_ln=final_ln)
    if k == 1:
        ctxs = [energon.energon_init(cfg)]
    else:
        ctxs = energon.energon_init_local_group(cfg, k)
    load_engine(ctxs, dict(shape, L=Lx), seed, dtype)
    return ctxs


def destroy(ctxs):
    from paper_2209_02341_b200 import energon
    for c in ctxs:
        energon.energon_destroy(c)


def run_forward(ctxs, tok_np, lens, dtype, H):
    import torch

    from paper_2209_02341_b200 import energon
    tok = torch.from_numpy(tok_np).cuda()
    B, S = tok_np.shape
    out = torch.full((B, S, H), float("nan"), dtype=torch_dtype(dtype), device="cuda")
    if len(ctxs) == 1:
        energon.energon_forward(ctxs[0], tok, lens, out)
    else:
        energon.energon_forward_group(ctxs, tok, lens, out)
    energon.energon_sync(ctxs[0])
    return out.float().cpu().numpy().astype(np.float64)


def oracle_model(shape, seed, dtype, layer_ids=None, L=None):
    Lx = shape["L"] if L is None else L
    return synth.model_host(Lx, shape["H"], shape["F"], shape["V"], shape["max_seq"], seed, dtype == "bf16",
                            layer_ids=layer_ids)

"""GPU parity of the CUDA path (through the C ABI) against the fp64 oracle.

Bars (BASELINE.json north_star): index maps bit-exact; max-abs-rel <= 1e-4 in
the fp32 mode and <= 2e-2 in the bf16 mode.  Inputs are seeded synthetic batches with the
shapes of the paper's workloads.
"""
import os
import sys

import numpy as np
import pytest

import oracle
import synth
from gpu_helpers import (SHAPES, destroy, make_engine, max_abs_rel, oracle_model, run_forward, torch_dtype)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "bf16": 2e-2}


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2209_02341_b200 import build, energon
    build()
    energon.load_library()
    synth.build(device=True)


def E():
    from paper_2209_02341_b200 import energon
    return energon


# ----------------------------------------------------------------------------- generator
@pytest.mark.parametrize("bf16", [False, True])
def test_synth_device_bits_equal_host(bf16):
    n = 100003
    t = torch.empty(n, dtype=torch.bfloat16 if bf16 else torch.float32, device="cuda")
    synth.fill_device(t, 7, 2, 3, 0.02, 0.0, bf16)
    h = synth.host_tensor((n,), 7, 2, 3, 0.02, 0.0, bf16, dtype="bf16" if bf16 else np.float32)
    got = t.cpu()
    if bf16:
        assert np.array_equal(got.view(torch.int16).numpy().view(np.uint16), h)
    else:
        assert np.array_equal(got.numpy().view(np.uint32), h.view(np.uint32))


# ----------------------------------------------------------------------------- a1 index maps
@pytest.mark.parametrize("lens,S", [
    ([2, 3], 4), ([1], 3), ([5, 5, 5], 5), ([1] * 7, 9),
    (synth.random_lengths(32, 128, 0), 128),
    (synth.exact_p_lengths(16, 512, 0.5, 0), 512),
    (synth.random_lengths(1024, 64, 3), 64),
    (synth.exact_p_lengths(32, 1024, 0.75, 1), 1024),
])
def test_index_maps_bitexact(lens, S):
    B = len(lens)
    off = torch.full((B + 1,), -7, dtype=torch.int32, device="cuda")
    pack = torch.full((B * S,), -7, dtype=torch.int32, device="cuda")
    pos = torch.full((B * S,), -7, dtype=torch.int32, device="cuda")
    unpack = torch.full((B * S,), -7, dtype=torch.int32, device="cuda")
    E().energon_index_maps(lens, S, off, pack, pos, unpack)
    torch.cuda.synchronize()
    o_off, o_pack, o_pos, o_unpack = oracle.index_maps(lens, S)
    T = int(o_off[-1])
    assert np.array_equal(off.cpu().numpy(), o_off)
    assert np.array_equal(pack.cpu().numpy()[:T], o_pack)
    assert np.array_equal(pos.cpu().numpy()[:T], o_pos)
    assert np.array_equal(unpack.cpu().numpy(), o_unpack)
    assert (pack.cpu().numpy()[T:] == -7).all()  # nothing written past T


# ----------------------------------------------------------------------------- a4/a8/a10/a11 GEMMs
def _gemm_case(M, N, K, dtype, epi, seed=0):
    tdt = torch_dtype(dtype)
    g = torch.Generator(device="cpu").manual_seed(seed)
    A = (torch.rand(M, K, generator=g) * 2 - 1).to(tdt)
    W = ((torch.rand(N, K, generator=g) * 2 - 1) * 0.05).to(tdt)
    bias = (torch.rand(N, generator=g) * 2 - 1).float()
    D = torch.full((M, N), float("nan"), dtype=tdt, device="cuda")
    E().energon_gemm(A.cuda(), W.cuda(), bias.cuda() if epi else None, D, epilogue=epi)
    torch.cuda.synchronize()
    ref = oracle.matmul(A.double().numpy(), W.double().numpy().T)
    if epi:
        ref = ref + bias.double().numpy()
    if epi == 2:
        ref = np.vectorize(oracle.gelu)(ref)
    return D.float().cpu().numpy().astype(np.float64), ref


@pytest.mark.parametrize("M,N,K", [
    (1, 64, 64), (77, 136, 72), (128, 256, 64), (129, 264, 128), (300, 392, 640), (1000, 1920, 512),
    (513, 768, 3072), (2064, 2304, 768),
])
def test_gemm_bf16_tcgen05_vs_oracle(M, N, K):
    got, ref = _gemm_case(M, N, K, "bf16", 0)
    err = np.abs(got - ref)
    # bf16 output rounding (2^-9 relative) + fp32 accumulation
    assert (err <= 4e-3 * np.abs(ref) + 1e-4 * np.abs(ref).max()).all(), err.max()


@pytest.mark.parametrize("epi", [1, 2])
def test_gemm_bf16_epilogues(epi):
    got, ref = _gemm_case(200, 264, 192, "bf16", epi, seed=1)
    assert (np.abs(got - ref) <= 4e-3 * np.abs(ref) + 1e-4 * np.abs(ref).max()).all()


@pytest.mark.parametrize("M,N,K,epi", [(30, 192, 64, 1), (30, 256, 64, 2), (77, 64, 256, 0), (130, 130, 70, 1)])
def test_gemm_f32_vs_oracle(M, N, K, epi):
    got, ref = _gemm_case(M, N, K, "f32", epi)
    assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max()


def test_gemm_bf16_large_vs_cublas():
    """Library cross-check (tests only): 4096 x 5120 x 5120 against torch.matmul (cuBLAS, fp32)."""
    M, N, K = 4096, 5120, 5120
    A = (torch.randn(M, K, device="cuda") * 0.5).bfloat16()
    W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    D = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    E().energon_gemm(A, W, None, D)
    ref = A.float() @ W.float().t()
    err = (D.float() - ref).abs()
    assert (err <= 4e-3 * ref.abs() + 1e-3 * ref.abs().max()).all().item(), err.max().item()


# ----------------------------------------------------------------------------- full stack, config 1
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("causal", [1, 0])
@pytest.mark.parametrize("drce", [1, 0])
def test_forward_tiny_vs_oracle(dtype, causal, drce):
    """BASELINE config 1 (1 layer, H=64, 4 heads, B=4, S=16, random lengths)."""
    shape = SHAPES["tiny"]
    B, S, seed = 4, 16, 0
    lens = synth.random_lengths(B, S, seed)
    tok = synth.tokens(B, S, shape["V"], lens, seed)
    ctxs = make_engine(shape, seed, dtype, B * S, drce=drce, causal=causal)
    try:
        y = run_forward(ctxs, tok, lens, dtype, shape["H"])
    finally:
        destroy(ctxs)
    layers, emb = oracle_model(shape, seed, dtype)
    cfg = oracle.make_cfg(shape["L"], shape["H"], shape["h"], shape["F"], causal=causal)
    ref = oracle.forward_padded(cfg, layers, emb, tok, lens)
    assert max_abs_rel(y, ref, lens) <= TOL[dtype]
    for b, n in enumerate(lens):
        assert not y[b, n:].any()  # pad rows exactly 0


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("k", [2, 4])
@pytest.mark.parametrize("sp", [1, 0])
def test_forward_local_tp_vs_oracle(dtype, k, sp):
    """1-D TP over k shards on one GPU (in-device rank-order reductions), both schedules: allreduce
    (sp=0) and reduce-scatter / LN on own rows / all-gather (sp=1); equals the serial oracle."""
    shape = dict(SHAPES["tiny"], L=2, V=300, max_seq=40)
    B, S, seed = 5, 33, 4
    lens = synth.random_lengths(B, S, seed)
    tok = synth.tokens(B, S, shape["V"], lens, seed)
    ctxs = make_engine(shape, seed, dtype, B * S, k=k)
    for c in ctxs:
        E().energon_set_option(c, E().OPT_TP_SP, sp)
    try:
        y = run_forward(ctxs, tok, lens, dtype, shape["H"])
        st = E().energon_get_stats(ctxs[0])
    finally:
        destroy(ctxs)
    assert st["allreduce_calls"] == 2 * shape["L"]  # SPEC.md:315 exactly 2 per layer
    layers, emb = oracle_model(shape, seed, dtype)
    cfg = oracle.make_cfg(shape["L"], shape["H"], shape["h"], shape["F"])
    ref = oracle.forward_padded(cfg, layers, emb, tok, lens)
    assert max_abs_rel(y, ref, lens) <= TOL[dtype]


def test_forward_multi_tile_f32():
    """fp32 mode across several GEMM / attention tiles and a ragged tail (H=256, S=200)."""
    shape = dict(L=2, H=256, h=4, F=1024, V=1000, max_seq=256)
    B, S, seed = 6, 200, 11
    lens = synth.random_lengths(B, S, seed)
    tok = synth.tokens(B, S, shape["V"], lens, seed)
    ctxs = make_engine(shape, seed, "f32", B * S)
    try:
        y = run_forward(ctxs, tok, lens, "f32", shape["H"])
    finally:
        destroy(ctxs)
    layers, emb = oracle_model(shape, seed, "f32")
    cfg = oracle.make_cfg(shape["L"], shape["H"], shape["h"], shape["F"])
    ref = oracle.forward_drce(cfg, layers, emb, tok, lens)
    assert max_abs_rel(y, ref, lens) <= 1e-4


# ----------------------------------------------------------------------------- config 2 (GPT-2 small)
def test_forward_gpt2s_sampled_sequences():
    """BASELINE config 2 at full size (12 layers, H=768, B=32, S=128, bf16) on the GPU; the oracle
    recomputes 4 sampled sequences (P12: sequence independence) -- longest, shortest, two more."""
    shape = SHAPES["gpt2s"]
    B, S, seed = 32, 128, 0
    lens = synth.random_lengths(B, S, seed)
    tok = synth.tokens(B, S, shape["V"], lens, seed)
    ctxs = make_engine(shape, seed, "bf16", B * S)
    try:
        y = run_forward(ctxs, tok, lens, "bf16", shape["H"])
    finally:
        destroy(ctxs)
    order = np.argsort(lens)
    sel = [int(order[-1]), int(order[0]), 5, 17]
    layers, emb = oracle_model(shape, seed, "bf16")
    cfg = oracle.make_cfg(shape["L"], shape["H"], shape["h"], shape["F"])
    Ssel = max(lens[i] for i in sel)
    ref = oracle.forward_drce(cfg, layers, emb, tok[sel][:, :Ssel], [lens[i] for i in sel])
    err = max_abs_rel(y[sel][:, :Ssel], ref, [lens[i] for i in sel])
    assert err <= 2e-2, err


# ----------------------------------------------------------------------------- config 3, teacher-forced
def test_gpt3_13b_layer_teacher_forced():
    """BASELINE config 3 shape (H=5120, 40 heads, B=16, S=512, p=0.5, bf16) at full size: one layer
    through energon_forward_hidden on the whole batch; the oracle recomputes that layer for the
    shortest sequence from the same fp32 input."""
    shape = SHAPES["gpt3_13b"]
    B, S, seed = 16, 512, 0
    lens = synth.exact_p_lengths(B, S, 0.5, seed)
    H = shape["H"]
    ctxs = make_engine(shape, seed, "bf16", B * S, L=1)
    try:
        g = torch.Generator(device="cpu").manual_seed(3)
        x = (torch.randn(B, S, H, generator=g) * 0.5).float()
        out = torch.full((B, S, H), float("nan"), device="cuda")
        E().energon_forward_hidden(ctxs[0], x.cuda(), lens, 0, 1, 0, out)
        E().energon_sync(ctxs[0])
        y = out.cpu().double().numpy()
    finally:
        destroy(ctxs)
    b = int(np.argmin(lens))
    n = lens[b]
    layers, _ = oracle_model(shape, seed, "bf16", layer_ids=[0], L=1)
    cfg = oracle.make_cfg(1, H, shape["h"], shape["F"])
    ref = oracle.layers_padded(cfg, layers, 0, 1, x[b:b + 1, :n].double().numpy(), [n])
    err = max_abs_rel(y[b:b + 1, :n], ref, [n])
    assert err <= 2e-2, err
    assert not y[b, n:].any()


# ----------------------------------------------------------------------------- error paths on the device
def test_bad_token_surfaces_on_sync():
    shape = SHAPES["tiny"]
    ctxs = make_engine(shape, 0, "f32", 64)
    try:
        tok = torch.tensor([[1, 2, 99999, 4]], dtype=torch.int32, device="cuda")
        out = torch.empty(1, 4, shape["H"], device="cuda")
        E().energon_forward(ctxs[0], tok, [4], out)
        with pytest.raises(E().EnergonError) as ei:
            E().energon_sync(ctxs[0])
        assert ei.value.status == -5
        E().energon_sync(ctxs[0])  # cleared
    finally:
        destroy(ctxs)


def test_host_validation_no_side_effects():
    shape = SHAPES["tiny"]
    ctxs = make_engine(shape, 0, "f32", 64)
    try:
        tok = torch.ones(4, 16, dtype=torch.int32, device="cuda")
        out = torch.zeros(4, 16, shape["H"], device="cuda")
        before = E().energon_get_stats(ctxs[0])
        for lens, code in (([0, 1, 1, 1], -4), ([17, 1, 1, 1], -4)):
            with pytest.raises(E().EnergonError) as ei:
                E().energon_forward(ctxs[0], tok, lens, out)
            assert ei.value.status == code
        with pytest.raises(E().EnergonError) as ei:
            E().energon_forward(ctxs[0], torch.ones(5, 16, dtype=torch.int32, device="cuda"), [1] * 5,
                                torch.zeros(5, 16, shape["H"], device="cuda"))
        assert ei.value.status == -6  # 5*16 > max_tokens
        assert E().energon_get_stats(ctxs[0]) == before
        assert not out.any()
    finally:
        destroy(ctxs)


def test_not_loaded():
    from paper_2209_02341_b200 import energon
    cfg = energon.make_config(1, 64, 4, 256, 256, 16, 64, dtype="f32")
    ctx = energon.energon_init(cfg)
    try:
        with pytest.raises(energon.EnergonError) as ei:
            energon.energon_forward(ctx, torch.ones(1, 4, dtype=torch.int32, device="cuda"), [4],
                                    torch.empty(1, 4, 64, device="cuda"))
        assert ei.value.status == -7
    finally:
        energon.energon_destroy(ctx)


# ----------------------------------------------------------------------------- a6 attention kernel
ATTN_LEN_CASES = {
    # straddle the 64-key tiles of v2
    "t64": (150, [1, 63, 64, 65, 130, 150], 3),
    # straddle v3's 128-key tiles and 256-row items (Q tile 1 empty / one row / full, dead warps)
    "t128": (520, [1, 31, 32, 127, 128, 129, 160, 255, 256, 257, 385, 520], 2),
}


@pytest.mark.parametrize("dtype,d", [("bf16", 128), ("bf16", 64), ("f32", 64), ("bf16", 16)])
@pytest.mark.parametrize("causal", [1, 0])
@pytest.mark.parametrize("lcase", ["t64", "t128"])
def test_attention_kernel_vs_oracle(dtype, d, causal, lcase):
    """Lengths straddling the key tiles and query items of both tcgen05 kernels, incl. NaN in every pad row
    of Q/K/V."""
    if lcase == "t128" and dtype == "f32":
        pytest.skip("the SIMT fp32 kernel has no tiles; t64 covers it")
    S, lens, hk = ATTN_LEN_CASES[lcase]
    B = len(lens)
    g = torch.Generator(device="cpu").manual_seed(d + causal)
    tdt = torch_dtype(dtype)
    Qh, Kh, Vh = ((torch.randn(B, hk, S, d, generator=g) * s).to(tdt) for s in (1.0, 1.0, 1.0))
    for b, n in enumerate(lens):  # pad rows never written by a5: poison them
        Kh[b, :, n:] = float("nan")
        Vh[b, :, n:] = float("nan")
        Qh[b, :, n:] = float("nan")
    O = torch.full((B, hk, S, d), 7.0, dtype=tdt, device="cuda")
    E().energon_attention(Qh.cuda(), Kh.cuda(), Vh.cuda(), O, lens, causal=causal)
    torch.cuda.synchronize()
    got = O.float().cpu().numpy().astype(np.float64)
    # oracle layout [B, S, H] with head i = columns [i d, (i+1) d)
    to_bsh = lambda t: t.double().permute(0, 2, 1, 3).reshape(B, S, hk * d).numpy()
    ref = oracle.attention(np.nan_to_num(to_bsh(Qh)), np.nan_to_num(to_bsh(Kh)), np.nan_to_num(to_bsh(Vh)),
                           hk, lens, causal)
    ref = ref.reshape(B, S, hk, d).transpose(0, 2, 1, 3)
    tol = 1e-5 if dtype == "f32" else 2e-2
    for b, n in enumerate(lens):
        assert np.isfinite(got[b, :, :n]).all()
        assert np.abs(got[b, :, :n] - ref[b, :, :n]).max() <= tol * max(1.0, np.abs(ref[b, :, :n]).max())
        assert (got[b, :, n:] == 7.0).all()  # pad query rows untouched


@pytest.mark.skipif(os.environ.get("ENERGON_ATTN") == "5", reason="already the v3 run")
def test_attention_v3_kernel_vs_oracle():
    """The same attention cases through the v3 kernel (ENERGON_ATTN=5: one CTA per SM, two Q tiles sharing
    K/V tiles), which a process selects once at load: run them in a child process."""
    import subprocess
    env = dict(os.environ, ENERGON_ATTN="5")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-x", "-m", "gpu",
                        os.path.abspath(__file__), "-k", "test_attention_kernel_vs_oracle"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


# ----------------------------------------------------------------------------- a5 / a7 / a13 vs the oracle's maps
def _bits(t):
    import torch as _t
    return t.view(_t.int16 if t.dtype == _t.bfloat16 else _t.int32).cpu().numpy()


LAYOUT_CASES = [([2, 3], 4, 2, 16), ([1, 7, 64, 3], 64, 3, 64), (synth.exact_p_lengths(16, 512, 0.5, 0), 512, 5, 128),
                (synth.random_lengths(33, 40, 9), 40, 2, 32), ([1], 1, 1, 8)]


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("lens,S,hk,d", LAYOUT_CASES)
def test_layout_kernels_bitexact_vs_oracle_maps(dtype, lens, S, hk, d):
    """a5 / a7 / a13 are index + copy work: each standalone kernel must equal, bit for bit, the scatter /
    gather that oracle_index_maps (the fp64 oracle's closed-form maps) drives on the
    host.  Pad rows a5 must not write keep their NaN sentinel; pad cells a13 writes are exactly 0."""
    tdt = torch_dtype(dtype)
    B = len(lens)
    off, pack, pos, unpack = oracle.index_maps(lens, S)
    T = int(off[-1])
    Hk = hk * d
    pack_d = torch.from_numpy(pack.astype(np.int32)).cuda()
    unpack_d = torch.from_numpy(unpack.astype(np.int32)).cuda()
    g = torch.Generator().manual_seed(T * 7 + d)
    # a5: packed QKV -> padded Q, K, V
    qkv = torch.randn(T, 3 * Hk, generator=g).to(tdt).cuda()
    outs = [torch.full((B, hk, S, d), float("nan"), dtype=tdt, device="cuda") for _ in range(3)]
    E().energon_unpack_qkv(qkv, pack_d, S, hk, d, *outs)
    torch.cuda.synchronize()
    qkv_h = qkv.cpu()
    for w, o in enumerate(outs):
        exp = torch.full((B, hk, S, d), float("nan"), dtype=tdt)
        for t in range(T):
            b, s = divmod(int(pack[t]), S)
            exp[b, :, s, :] = qkv_h[t, w * Hk:(w + 1) * Hk].view(hk, d)
        assert np.array_equal(_bits(o), _bits(exp))
    # a7: padded O -> packed C (DRCE), and the padded A/B form (identity rows, pad cells zeroed)
    O = torch.randn(B, hk, S, d, generator=g).to(tdt).cuda()
    C = torch.full((T, Hk), 3.0, dtype=tdt, device="cuda")
    E().energon_repack(O, pack_d, unpack_d, T, C)
    Cp = torch.full((B * S, Hk), 3.0, dtype=tdt, device="cuda")
    E().energon_repack(O, None, unpack_d, B * S, Cp)
    torch.cuda.synchronize()
    Oh = O.cpu()
    expC = torch.stack([Oh[int(c) // S, :, int(c) % S, :].reshape(Hk) for c in pack])
    assert np.array_equal(_bits(C), _bits(expC))
    expP = Oh.permute(0, 2, 1, 3).reshape(B * S, Hk).clone()
    expP[torch.from_numpy(unpack < 0)] = 0
    assert np.array_equal(_bits(Cp), _bits(expP))
    # a13 without LN: out[cell] = X[unpack[cell]] (fp32 -> out dtype, RNE) or exactly 0
    H = 4 * max(2, Hk // 8)
    X = torch.randn(T, H, generator=g).cuda()
    out = torch.full((B, S, H), float("nan"), dtype=tdt, device="cuda")
    E().energon_final_unpack(X, unpack_d, out)
    torch.cuda.synchronize()
    exp = torch.zeros(B * S, H, dtype=tdt)
    valid = torch.from_numpy(unpack >= 0)
    exp[valid] = X.cpu()[torch.from_numpy(unpack[unpack >= 0].astype(np.int64))].to(tdt)
    assert np.array_equal(_bits(out.view(B * S, H)), _bits(exp))
    # a13 with the final LN: the unpack is exact, the LN within fp32 rounding of the oracle's fp64 LN
    gam = (1 + 0.1 * torch.randn(H, generator=g)).cuda()
    bet = (0.1 * torch.randn(H, generator=g)).cuda()
    E().energon_final_unpack(X, unpack_d, out, gam, bet, 1e-5, True)
    torch.cuda.synchronize()
    y = out.view(B * S, H).float().cpu().numpy()
    ref = oracle.layernorm(X.cpu().double().numpy(), gam.cpu().double().numpy(), bet.cpu().double().numpy())
    assert not y[unpack < 0].any()
    tol = 1e-5 if dtype == "f32" else 8e-3
    assert np.abs(y[unpack >= 0] - ref[unpack[unpack >= 0]]).max() <= tol * max(1.0, np.abs(ref).max())


# ----------------------------------------------------------------------------- fused a5 / a7
@pytest.mark.parametrize("drce", [1, 0])
@pytest.mark.parametrize("B,S,seed", [(8, 96, 2), (40, 40, 3)])
def test_fused_layout_kernels_bitexact(drce, B, S, seed, monkeypatch):
    """a5 fused into the QKV epilogue -- as TMA bulk-tensor stores into the padded Q / K / V planes (one
    3-D box store per sequence a 32-row box touches; the default) and as per-thread scatter stores
    (ENERGON_NO_QKV_TMA=1) -- and a7 fused into attention produce the same bits as the standalone paper
    kernels; (40, 40, 3) has many sequences shorter than a 32-row box."""
    shape = dict(SHAPES["gpt2s"], L=2)
    lens = synth.random_lengths(B, S, seed)
    tok = synth.tokens(B, S, shape["V"], lens, seed)
    outs = []
    for nofuse, notma in (("0", "0"), ("0", "1"), ("1", "0")):
        monkeypatch.setenv("ENERGON_NO_FUSE", nofuse)
        if notma == "1":
            monkeypatch.setenv("ENERGON_NO_QKV_TMA", "1")
        else:
            monkeypatch.delenv("ENERGON_NO_QKV_TMA", raising=False)
        ctxs = make_engine(shape, seed, "bf16", B * S, drce=drce)
        try:
            outs.append(run_forward(ctxs, tok, lens, "bf16", shape["H"]))
        finally:
            destroy(ctxs)
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[0], outs[2])


@pytest.mark.parametrize("k", [1, 8])
def test_forward_tile224_bitexact(k, monkeypatch):
    """Every linear of the layer on the 256 x 224 pair tile (seven 32-column epilogue chunks split 4 + 3
    between the two epilogue warpgroups; a5 TMA box stores in the QKV epilogue; GeLU; the local TP group's
    partials) gives the same bits as on the 256 x 256 tile -- an output element's fp32 accumulation over K
    does not depend on the tile width -- and stays within 2e-2 of the fp64 oracle."""
    shape = dict(L=2, H=1024, h=8, F=4096, V=500, max_seq=128)
    B, S, seed = 6, 128, 12
    lens = synth.random_lengths(B, S, seed)
    tok = synth.tokens(B, S, shape["V"], lens, seed)
    outs = []
    for code in ("1224", "1256"):
        monkeypatch.setenv("ENERGON_GEMM_TILE", code)
        ctxs = make_engine(shape, seed, "bf16", B * S, k=k)
        try:
            outs.append(run_forward(ctxs, tok, lens, "bf16", shape["H"]))
        finally:
            destroy(ctxs)
    assert np.array_equal(outs[0], outs[1])
    layers, emb = oracle_model(shape, seed, "bf16")
    cfg = oracle.make_cfg(shape["L"], shape["H"], shape["h"], shape["F"])
    ref = oracle.forward_padded(cfg, layers, emb, tok, lens)
    assert max_abs_rel(outs[0], ref, lens) <= 2e-2


@pytest.mark.parametrize("k", [2, 4])
@pytest.mark.parametrize("drce", [1, 0])
def test_forward_local_tp_fused_d64(k, drce):
    """Local TP with head_dim 64 (fused a5/a7 path), sequence-parallel schedule, DRCE on / off,
    against the oracle, bf16."""
    shape = dict(L=2, H=256, h=4, F=1024, V=500, max_seq=64)
    B, S, seed = 5, 64, 9
    lens = synth.random_lengths(B, S, seed)
    tok = synth.tokens(B, S, shape["V"], lens, seed)
    ctxs = make_engine(shape, seed, "bf16", B * S, k=k, drce=drce)
    try:
        y = run_forward(ctxs, tok, lens, "bf16", shape["H"])
    finally:
        destroy(ctxs)
    layers, emb = oracle_model(shape, seed, "bf16")
    cfg = oracle.make_cfg(shape["L"], shape["H"], shape["h"], shape["F"])
    ref = oracle.forward_padded(cfg, layers, emb, tok, lens)
    assert max_abs_rel(y, ref, lens) <= 2e-2


@pytest.mark.parametrize("code", [1256, 1224, 1192, 1128, 256, 128])
@pytest.mark.parametrize("M,N,K,epi", [(700, 1000, 320, 1), (257, 392, 640, 2), (4096, 640, 128, 0)])
def test_gemm_every_tile_shape(code, M, N, K, epi, monkeypatch):
    """Every tcgen05 tile variant (2-CTA 256x{256,224,192,128}, 1-CTA 128x{256,128}) on ragged shapes."""
    monkeypatch.setenv("ENERGON_GEMM_TILE", str(code))
    got, ref = _gemm_case(M, N, K, "bf16", epi, seed=code)
    assert (np.abs(got - ref) <= 4e-3 * np.abs(ref) + 1e-4 * np.abs(ref).max()).all()


@pytest.mark.parametrize("M,N,K,epi,tile", [(4096, 1920, 5120, 1, 0), (4096, 2560, 5120, 2, 0), (2304, 2560, 10240, 2, 0),
                                            (1200, 3800, 10240, 1, 0), (4096, 1920, 5000, 0, 0), (4096, 2560, 640, 0, 1192),
                                            (4096, 5120, 2560, 0, 0), (4096, 1920, 5120, 1, 1256),
                                            (4096, 5120, 2560, 0, 1224)])
@pytest.mark.parametrize("order", [1, 2])
def test_gemm_streamk(M, N, K, epi, tile, order, monkeypatch):
    """Stream-K with accumulator preload (gemm_tc.cu TailPlan): the last round + remainder of tiles spread
    evenly over the clusters, split tiles finished on top of the early piece's fp32 partial -- QKV / MLP-up /
    MLP-down at TP=8 (128 / 160 / 320 tiles), 90 and 75 tiles at K = 10240, a K tail, the 256 x 192 tile:
    correct vs the oracle, deterministic, and BIT-IDENTICAL to the data-parallel schedule (the split
    tile's single fp32 accumulator sees the k-blocks in the same order); both unit orders."""
    if tile:
        monkeypatch.setenv("ENERGON_GEMM_TILE", str(tile))
    monkeypatch.setenv("ENERGON_SK_FORCE", str(order))  # stream-K, early piece first (1) / data parallel first (2)
    tdt = torch.bfloat16
    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    A = (torch.rand(M, K, generator=g) * 2 - 1).to(tdt)
    W = ((torch.rand(N, K, generator=g) * 2 - 1) * 0.05).to(tdt)
    bias = (torch.rand(N, generator=g) * 2 - 1).float()
    Ad, Wd, bd = A.cuda(), W.cuda(), bias.cuda()

    def run():
        D = torch.full((M, N), float("nan"), dtype=tdt, device="cuda")
        E().energon_gemm(Ad, Wd, bd if epi else None, D, epilogue=epi)
        torch.cuda.synchronize()
        return D

    got, got2 = run(), run()
    monkeypatch.setenv("ENERGON_NO_STREAMK", "1")
    got_dp = run()
    assert torch.equal(got, got2)
    assert torch.equal(got, got_dp)
    ref = oracle.matmul(A.double().numpy(), W.double().numpy().T)
    if epi:
        ref = ref + bias.double().numpy()
    if epi == 2:
        ref = np.vectorize(oracle.gelu)(ref)
    y = got.float().cpu().numpy().astype(np.float64)
    assert (np.abs(y - ref) <= 4e-3 * np.abs(ref) + 1e-4 * np.abs(ref).max()).all()


# ----------------------------------------------------------------------------- configs 4 and 5, teacher-forced
@pytest.mark.parametrize("name,p", [("opt30b", 0.5), ("opt66b", 0.75), ("opt66b", 0.0)])
def test_opt_layer_teacher_forced(name, p):
    """BASELINE configs 4 / 5 shapes (H=7168 / 9216, d=128, B=32, S=1024, padding p): one layer of
    the stack on the whole batch through energon_forward_hidden; the oracle recomputes it for the
    shortest sequence (P12), from the same fp32 input, within 2e-2."""
    shape = SHAPES[name]
    B, S, seed = 32, 1024, 1
    lens = synth.exact_p_lengths(B, S, p, seed)
    H = shape["H"]
    ctxs = make_engine(shape, seed, "bf16", B * S, L=1)
    try:
        g = torch.Generator(device="cpu").manual_seed(5)
        x = (torch.randn(B, S, H, generator=g) * 0.5).float()
        out = torch.full((B, S, H), float("nan"), device="cuda")
        E().energon_forward_hidden(ctxs[0], x.cuda(), lens, 0, 1, 0, out)
        E().energon_sync(ctxs[0])
        b = int(np.argmin(lens))
        n = min(lens[b], 96)  # causal prefix of the shortest sequence (P13) keeps the oracle fast
        y = out[b:b + 1, :n].cpu().double().numpy()
        assert not out[b, lens[b]:].any().item()
    finally:
        destroy(ctxs)
    layers, _ = oracle_model(shape, seed, "bf16", layer_ids=[0], L=1)
    cfg = oracle.make_cfg(1, H, shape["h"], shape["F"])
    ref = oracle.layers_padded(cfg, layers, 0, 1, x[b:b + 1, :n].double().numpy(), [n])
    err = max_abs_rel(y, ref, [n])
    assert err <= 2e-2, err


# ----------------------------------------------------------------------------- edge cases
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("case", ["all_len_1", "max_len_1", "one_long_sequence", "max_batch"])
def test_forward_edge_cases(dtype, case):
    """Degenerate batches: every sequence of length 1, max_len 1, a single 1024-token sequence
    (several query tiles of the persistent attention), and the maximum batch of 1024 sequences."""
    shape = dict(L=2, H=256, h=2, F=1024, V=512, max_seq=1024)
    if case == "all_len_1":
        B, S, lens = 7, 32, [1] * 7
    elif case == "max_len_1":
        B, S, lens = 5, 1, [1] * 5
    elif case == "one_long_sequence":
        B, S, lens = 1, 1024, [1024]
    else:
        B, S = 1024, 4
        lens = synth.random_lengths(B, S, 5)
    seed = 13
    tok = synth.tokens(B, S, shape["V"], lens, seed)
    ctxs = make_engine(shape, seed, dtype, B * S)
    try:
        y = run_forward(ctxs, tok, lens, dtype, shape["H"])
    finally:
        destroy(ctxs)
    layers, emb = oracle_model(shape, seed, dtype)
    cfg = oracle.make_cfg(shape["L"], shape["H"], shape["h"], shape["F"])
    if case == "one_long_sequence":  # causal prefix (P13) keeps the oracle fast
        n = 192
        ref = oracle.forward_drce(cfg, layers, emb, tok[:, :n], [n])
        assert max_abs_rel(y[:, :n], ref, [n]) <= TOL[dtype]
    else:
        ref = oracle.forward_drce(cfg, layers, emb, tok, lens)
        assert max_abs_rel(y, ref, lens) <= TOL[dtype]
    for b, n in enumerate(lens):
        assert not y[b, n:].any()


# ----------------------------------------------------------------------------- PMEP (next row N1)
@pytest.mark.parametrize("slots,pool", [(1, 0), (2, 0), (2, 1)])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_pmep_offload_bitexact(slots, pool, dtype):
    """Peer memory pooling: off-device layers prefetched from pinned host memory
    (pool 0) or a peer device's memory (pool 1 -- on the single-GPU pool the 'peer' is device 0 itself,
    which runs the same cudaMemcpyPeerAsync path) into staging slots on a copy stream give bit-identical
    output to the all-resident run, and the fetched bytes match the placement."""
    shape = dict(L=6, H=256, h=4, F=1024, V=500, max_seq=64)
    B, S, seed = 5, 48, 21
    lens = synth.random_lengths(B, S, seed)
    tok = synth.tokens(B, S, shape["V"], lens, seed)
    ctxs = make_engine(shape, seed, dtype, B * S)
    try:
        ref = run_forward(ctxs, tok, lens, dtype, shape["H"])
    finally:
        destroy(ctxs)
    layers_h, emb_h = oracle_model(shape, seed, dtype)
    oref = oracle.forward_drce(oracle.make_cfg(shape["L"], shape["H"], shape["h"], shape["F"]), layers_h, emb_h, tok,
                               lens)
    plan = E().energon_pmep_plan(shape["L"], 3)  # [1, 3, 5]
    for layers in (plan, [0, 2, 4, 5]):
        ctxs = make_engine(shape, seed, dtype, B * S)
        try:
            E().energon_offload_layers(ctxs[0], layers, slots=slots, pool=pool, peer_device=0 if pool else -1)
            y = run_forward(ctxs, tok, lens, dtype, shape["H"])
            y2 = run_forward(ctxs, tok, lens, dtype, shape["H"])  # slots reused across forwards
            st = E().energon_get_stats(ctxs[0])
        finally:
            destroy(ctxs)
        assert np.array_equal(y, ref) and np.array_equal(y2, ref)
        # and directly against the fp64 oracle (PMEP changes where the weights live, not the math)
        assert max_abs_rel(y, oref, lens) <= TOL[dtype]
        per_layer = (3 * 256 * 256 + 256 * 256 + 1024 * 256 * 2) * (2 if dtype == "bf16" else 4)
        assert st["prefetch_bytes"] == 2 * len(layers) * per_layer


# ----------------------------------------------------------------------------- CUDA graphs
@pytest.mark.parametrize("k", [1, 2])
def test_cuda_graph_replay_bitexact(k):
    """ENERGON_OPT_GRAPH: a replayed graph gives the eager bits and reads the current contents of the
    token buffer; a graph is keyed on the row bucket (T rounded up to 128), not on the lengths -- a new
    length vector of the same bucket (here: the batch's lengths permuted, and a different mix with the
    same T) replays the recorded graph with its lengths written into the index-maps node, a new bucket
    records a new graph."""
    shape = dict(SHAPES["gpt2s"], L=2)
    B, S, seed = 8, 96, 6
    lens = synth.random_lengths(B, S, seed)
    lens_perm = lens[::-1]
    lens_mix = list(lens)
    i_hi, i_lo = int(np.argmax(lens)), int(np.argmin(lens))
    shift = min(lens[i_hi] - 1, S - lens[i_lo], 9)
    lens_mix[i_hi] -= shift
    lens_mix[i_lo] += shift  # same T, different mix
    lens2 = [min(S, x + 40) for x in lens]  # another bucket
    assert (sum(lens2) + 127) // 128 != (sum(lens) + 127) // 128
    tok1 = torch.from_numpy(synth.tokens(B, S, shape["V"], lens2, seed)).cuda()
    tok2 = torch.from_numpy(synth.tokens(B, S, shape["V"], lens2, seed + 5)).cuda()
    ctxs = make_engine(shape, seed, "bf16", B * S, k=k)
    tok = torch.empty_like(tok1)
    out = torch.empty(B, S, shape["H"], dtype=torch.bfloat16, device="cuda")

    def fwd(t, ln):
        tok.copy_(t)
        out.fill_(float("nan"))
        if k == 1:
            E().energon_forward(ctxs[0], tok, ln, out)
        else:
            E().energon_forward_group(ctxs, tok, ln, out)
        torch.cuda.synchronize()
        return out.clone()

    try:
        cases = [(tok1, lens), (tok2, lens), (tok1, lens_perm), (tok2, lens_mix), (tok1, lens2)]
        eager = [fwd(t, ln) for t, ln in cases]
        for c in ctxs:
            E().energon_set_option(c, E().OPT_GRAPH, 1)
        rec = []
        graphed = []
        for t, ln in cases + cases:
            graphed.append(fwd(t, ln))
            rec.append(E().energon_get_stats(ctxs[0])["graphs_recorded"])
        st = E().energon_get_stats(ctxs[0])
    finally:
        destroy(ctxs)
    for i, g in enumerate(graphed):
        assert torch.equal(g, eager[i % len(cases)]), i
    assert rec == [1, 1, 1, 1, 2] + [2] * 5  # one graph per bucket, recorded on its first batch
    assert st["forwards"] == 15


# ----------------------------------------------------------------------------- N3: LN in the GEMM prologue
@pytest.mark.parametrize("name,B,S,fuse_layout,drce", [("gpt2s", 9, 100, True, 1), ("ln_d128", 5, 140, True, 1),
                                                       ("ln_d128", 5, 140, False, 1), ("ln_d128", 4, 70, True, 0)])
def test_ln_prologue_fusion(name, B, S, fuse_layout, drce, monkeypatch):
    """ENERGON_OPT_LN_FUSE: the residual kernels write only X and the
    row statistics, and the QKV / MLP-up GEMMs apply LN1 / LN2 in their prologue with the residual kernel's
    fp32 expression, so the forward must be bit-identical to the unfused one (which runs the same
    products through the 2-CTA GEMM) and within the bf16 bar of the fp64 oracle; also with the standalone
    a5 / a7 layout kernels (ENERGON_NO_FUSE=1), in the padded A/B mode (drce=0) and with graph replay."""
    if not fuse_layout:
        monkeypatch.setenv("ENERGON_NO_FUSE", "1")
    shape = dict(SHAPES["gpt2s"], L=2) if name == "gpt2s" else dict(L=2, H=256, h=2, F=1024, V=600, max_seq=160)
    seed = 13
    lens = synth.random_lengths(B, S, seed)
    tok = synth.tokens(B, S, shape["V"], lens, seed)
    ctxs = make_engine(shape, seed, "bf16", B * S, drce=drce)
    try:
        y0 = run_forward(ctxs, tok, lens, "bf16", shape["H"])
        E().energon_set_option(ctxs[0], E().OPT_LN_FUSE, 1)
        y1 = run_forward(ctxs, tok, lens, "bf16", shape["H"])
        E().energon_set_option(ctxs[0], E().OPT_GRAPH, 1)
        y2 = run_forward(ctxs, tok, lens, "bf16", shape["H"])
        y3 = run_forward(ctxs, tok, lens, "bf16", shape["H"])
    finally:
        destroy(ctxs)
    assert np.array_equal(y0, y1), f"LN-prologue forward differs: max |d| {np.nanmax(np.abs(y0 - y1))}"
    assert np.array_equal(y1, y2) and np.array_equal(y2, y3)
    layers, emb = oracle_model(shape, seed, "bf16")
    cfg = oracle.make_cfg(shape["L"], shape["H"], shape["h"], shape["F"])
    ref = oracle.forward_padded(cfg, layers, emb, tok, lens)
    assert max_abs_rel(y1, ref, lens) <= TOL["bf16"]


def test_ln_prologue_fusion_refused_outside_domain():
    """ENERGON_OPT_LN_FUSE is bf16 / TP = 1 only: fp32 contexts and local TP groups get ENERGON_ERR_CONFIG."""
    shape = dict(SHAPES["tiny"])
    for dtype, k in (("f32", 1), ("bf16", 2)):
        ctxs = make_engine(shape, 0, dtype, 64, k=k)
        try:
            with pytest.raises(E().EnergonError) as ei:
                E().energon_set_option(ctxs[0], E().OPT_LN_FUSE, 1)
            assert ei.value.status == -2
        finally:
            destroy(ctxs)

"""Attention kernel micro-benchmark (energon_attention, padded output) on a few length mixes.

The calls are captured in a CUDA graph and the graph is replayed, so the number is device time (the ABI
entry builds tensor maps and a work list per call on the host, which would otherwise bound the loop).
ATTN_IMPLS=4,5 times both kernels (v2 / v3) in one process and checks that they agree on the valid rows.
"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2209_02341_b200 import energon
energon.load_library(os.environ.get("AB_LIB", energon.SO_PATH))
cases = {
    "gpt3_p0.5 (B16 S512)": (16, 512, synth.exact_p_lengths(16, 512, 0.5, 0)),
    "full S512 (B16)": (16, 512, [512] * 16),
    "full S2048 (B4)": (4, 2048, [2048] * 4),
    "full S128 (B64)": (64, 128, [128] * 64),
    "opt S1024 p0.5 (B32)": (32, 1024, synth.exact_p_lengths(32, 1024, 0.5, 0)),
}
if os.environ.get("ATTN_CASES"):  # a subset by name prefix, e.g. "gpt3" or "full S2048" (under ncu)
    cases = {k: v for k, v in cases.items() if k.startswith(os.environ["ATTN_CASES"])}
hk, d = int(os.environ.get("ATTN_HK", "40")), 128  # ATTN_HK: heads per rank (TP=8: 5)
impl = os.environ.get("ENERGON_ATTN", "4")
REPS = 20
for name, (B, S, lens) in cases.items():
    g = torch.Generator(device="cuda").manual_seed(0)
    Q, K, V = (torch.randn(B, hk, S, d, device="cuda", generator=g).bfloat16() for _ in range(3))
    O = torch.zeros_like(Q)
    flops = sum(4 * d * (L * (L + 1) / 2) * hk for L in lens)
    for _ in range(3):
        energon.energon_attention(Q, K, V, O, lens, 1)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            for _ in range(REPS):
                energon.energon_attention(Q, K, V, O, lens, 1)
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        graph.replay()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (3 * REPS)
    # fp32 reference on a few valid rows of the first and last sequences (sanity, not the parity test)
    err = 0.0
    for b in (0, B - 1):
        L = lens[b]
        for hh in (0, hk - 1):
            q = Q[b, hh, :L].float(); k_ = K[b, hh, :L].float(); v = V[b, hh, :L].float()
            sc = (q @ k_.T) / d ** 0.5
            sc = sc.masked_fill(torch.triu(torch.ones(L, L, dtype=torch.bool, device="cuda"), 1), float("-inf"))
            ref = torch.softmax(sc, -1) @ v
            err = max(err, ((O[b, hh, :L].float() - ref).abs().max() / ref.abs().max()).item())
    print(f"{name:24s} impl={impl} {ms*1e3:8.1f} us  {flops/ms/1e9:7.1f} TFLOP/s  max-abs-rel {err:.2e}", flush=True)

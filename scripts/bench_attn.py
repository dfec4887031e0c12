"""Attention kernel micro-benchmark (energon_attention, padded output) on a few length mixes."""
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
}
if os.environ.get("ATTN_CASES") == "gpt3":  # only the config-3 mix (e.g. under ncu)
    cases = {k: v for k, v in cases.items() if k.startswith("gpt3")}
hk, d = int(os.environ.get("ATTN_HK", "40")), 128  # ATTN_HK: heads per rank (TP=8: 5)
for name, (B, S, lens) in cases.items():
    Q, K, V = (torch.randn(B, hk, S, d, device="cuda").bfloat16() for _ in range(3))
    O = torch.empty_like(Q)
    flops = sum(4 * d * (L * (L + 1) / 2) * hk for L in lens)
    row = {}
    for _ in range(3):
        energon.energon_attention(Q, K, V, O, lens, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        energon.energon_attention(Q, K, V, O, lens, 1)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{name:24s} impl={os.environ.get('ENERGON_ATTN','4')} {ms*1e3:8.1f} us  {flops/ms/1e9:7.1f} TFLOP/s", flush=True)

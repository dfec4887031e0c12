"""v2 attention timeline (a diagnostics build with clock64 stamps, -DATTN2_TRACE=1, loaded via AB_LIB; the
instrumentation itself is not kept in the tree -- profiles/r02_attn_v2_trace_report.txt lists the stamp points; ENERGON_ATTN_TRACE=<file>): calls the kernel
eagerly on one length mix and prints CTA 0's per-tile clock64 stamps relative to its first record."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2209_02341_b200 import energon
energon.load_library(os.environ["AB_LIB"])
case = os.environ.get("CASE", "gpt3")
B, S, lens = (16, 512, synth.exact_p_lengths(16, 512, 0.5, 0)) if case == "gpt3" else (4, 2048, [2048] * 4)
hk, d = int(os.environ.get("ATTN_HK", "40")), 128
g = torch.Generator(device="cuda").manual_seed(0)
Q, K, V = (torch.randn(B, hk, S, d, device="cuda", generator=g).bfloat16() for _ in range(3))
O = torch.zeros_like(Q)
for _ in range(3):
    energon.energon_attention(Q, K, V, O, lens, 1)
torch.cuda.synchronize()
recs = []
for line in open(os.environ["ENERGON_ATTN_TRACE"]):
    if line.startswith("launch2"):
        recs = []
    else:
        recs.append(list(map(int, line.split())))
recs = [r for r in recs if r[1] or r[3]]
t0 = min(x for r in recs for x in r[1:] if x)
print(f"case {case}: tile  Sseen  Pdone (smax) | ofull_ok S_iss (ofull wait) | pv_entry p_ok v_ok (pwait vwait) | V_load")
for r in recs:
    i, s_seen, p_done, sw, si, pe, pok, vok, vl = r
    f = lambda x: x - t0 if x else -1
    print(f"{i:4d} {f(s_seen):7d} {f(p_done):7d} ({p_done - s_seen if s_seen and p_done else -1:5d}) | {f(sw):7d} {f(si):7d} ({sw - p_done if sw and p_done else -1:5d}) "
          f"| {f(pe):7d} {f(pok):7d} {f(vok):7d} ({pok - pe if pok and pe else -1:5d} {vok - pok if vok and pok else -1:5d}) | {f(vl):7d}")

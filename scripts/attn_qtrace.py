"""Item-change Q-load latency of attention v2 (CTA 0): needs a diagnostics build with clock64 stamps at the producer's Q
load and the MMA thread's q_full / k_full waits (not kept in the tree; profiles/r02_attn_v2_trace_report.txt lists them),
loaded via AB_LIB, with ENERGON_ATTN_TRACE=<file>."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_2209_02341_b200 import energon
energon.load_library(os.environ["AB_LIB"])
B, S, lens = 16, 512, synth.exact_p_lengths(16, 512, 0.5, 0)
hk, d = 40, 128
g = torch.Generator(device="cuda").manual_seed(0)
Q, K, V = (torch.randn(B, hk, S, d, device="cuda", generator=g).bfloat16() for _ in range(3))
O = torch.zeros_like(Q)
for _ in range(3):
    energon.energon_attention(Q, K, V, O, lens, 1)
torch.cuda.synchronize()
recs = []
for line in open(os.environ["ENERGON_ATTN_TRACE"]):
    if line.startswith("launch2"): recs = []
    else: recs.append(list(map(int, line.split())))
t0 = min(x for r in recs for x in r[1:] if x)
print("item  prod_before_qempty  prod_Q_issue  mma_qfull  mma_kfull  (Q latency)")
for r in recs:
    if r[1]: print(r[0], r[4]-t0 if r[4] else -1, r[1]-t0, r[2]-t0 if r[2] else -1, r[3]-t0 if r[3] else -1, (r[2]-r[1]) if r[2] else -1)

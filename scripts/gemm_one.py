"""Time (and let ncu capture) one energon GEMM shape: M N K epi from argv."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_02341_b200 import energon
energon.load_library(os.environ.get("AB_LIB", energon.SO_PATH))
M, N, K, epi = (int(x) for x in sys.argv[1:5])
A = (torch.randn(M, K, device="cuda") * 0.5).bfloat16()
W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
b = torch.randn(N, device="cuda")
D = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
for _ in range(5):
    energon.energon_gemm(A, W, b if epi else None, D, epilogue=epi)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    energon.energon_gemm(A, W, b if epi else None, D, epilogue=epi)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"{M}x{N}x{K} epi={epi}: {ms*1e3:.1f} us {2*M*N*K/ms/1e9:.0f} TF/s")

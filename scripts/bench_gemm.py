"""Micro-benchmark of the energon tcgen05 GEMM against cuBLAS (torch.matmul) on the GEMM shapes of
the DRCE layer (T = 4096 packed rows).  Development tool; not part of the product path."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_02341_b200 import energon

energon.load_library()
H = int(os.environ.get("H", 5120)); T = int(os.environ.get("T", 4096)); k = int(os.environ.get("K_TP", 1))
shapes = {"qkv": (T, 3 * H // k, H, 1), "out": (T, H, H // k, 0), "up": (T, 4 * H // k, H, 2), "down": (T, H, 4 * H // k, 0)}
res = {}
for name, (M, N, K, epi) in shapes.items():
    A = (torch.randn(M, K, device="cuda") * 0.5).bfloat16()
    W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    b = torch.randn(N, device="cuda")
    D = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    def run():
        energon.energon_gemm(A, W, b if epi else None, D, epilogue=epi)
    def ref():
        return A @ W.t()
    for f in (run, ref):
        for _ in range(3): f()
    torch.cuda.synchronize()
    out = {}
    for nm, f in (("energon", run), ("cublas", ref)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        n = 20
        for _ in range(n): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        out[nm] = {"ms": ms, "tflops": 2 * M * N * K / ms / 1e9}
    res[name] = out
    print(name, (M, N, K), {k2: f"{v['tflops']:.0f} TF ({v['ms']*1e3:.0f} us)" for k2, v in out.items()}, flush=True)
print(json.dumps(res))

"""cuBLAS (torch.matmul) on the TP = 8 per-rank GEMM shapes of config 3, for ncu: which kernel / grid / cluster."""
import torch
for (M, N, K) in [(4096, 1920, 5120), (4096, 2560, 5120), (4096, 5120, 640), (4096, 5120, 2560)]:
    A = torch.randn(M, K, device="cuda").bfloat16()
    W = torch.randn(N, K, device="cuda").bfloat16()
    for _ in range(3):
        D = A @ W.T
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        D = A @ W.T
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"cublas {M}x{N}x{K}: {ms*1e3:.1f} us {2*M*N*K/ms/1e9:.0f} TF/s", flush=True)

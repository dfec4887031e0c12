"""Sweep the tcgen05 tile variants (ENERGON_GEMM_TILE) over the DRCE GEMM shapes; development tool."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_02341_b200 import energon
energon.load_library()
T = int(os.environ.get("T", 4096))
H0 = int(os.environ.get("H", 5120))
TPS = [int(x) for x in os.environ.get("TPS", "1,2,4,8").split(",")]
res = {}
for k in TPS:
    H = H0
    shapes = {"qkv": (T, 3 * H // k, H), "out": (T, H, H // k), "up": (T, 4 * H // k, H), "down": (T, H, 4 * H // k)}
    for name, (M, N, K) in shapes.items():
        A = (torch.randn(M, K, device="cuda") * 0.5).bfloat16()
        W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
        D = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        row = {}
        for code in ("1256", "1192", "1128", "256", "auto"):
            if code == "auto":
                os.environ.pop("ENERGON_GEMM_TILE", None)
            else:
                os.environ["ENERGON_GEMM_TILE"] = code
            for _ in range(3):
                energon.energon_gemm(A, W, None, D)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                energon.energon_gemm(A, W, None, D)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            row[code] = round(2 * M * N * K / ms / 1e9)
        os.environ.pop("ENERGON_GEMM_TILE", None)
        for _ in range(3): A @ W.t()
        e0.record()
        for _ in range(20): A @ W.t()
        e1.record(); torch.cuda.synchronize()
        row["cublas"] = round(2 * M * N * K / (e0.elapsed_time(e1) / 20) / 1e9)
        res[f"tp{k}_{name}"] = row
        print(f"tp{k} {name} {(M, N, K)} {row}", flush=True)
print(json.dumps(res))

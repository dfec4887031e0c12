timeout 900 python -m pytest tests -m gpu -x -q --timeout=300 > gpurun_out/pytest_gpu.log 2>&1
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python scripts/bench_gemm.py > gpurun_out/bench_gemm.log 2>&1; tail -6 gpurun_out/bench_gemm.log
K_TP=8 timeout 300 python scripts/bench_gemm.py > gpurun_out/bench_gemm_tp8.log 2>&1; tail -6 gpurun_out/bench_gemm_tp8.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1
tail -3 gpurun_out/bench_full.log

timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout=300 -k "gemm" > gpurun_out/pytest_gemm.log 2>&1; tail -2 gpurun_out/pytest_gemm.log
ENERGON_STREAMK_MIN_KB=16 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout=300 -k "gemm or tiny or tp" > gpurun_out/pytest_gemm16.log 2>&1; tail -2 gpurun_out/pytest_gemm16.log
bash scripts/gpu_run19.sh

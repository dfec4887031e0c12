mkdir -p gpurun_out
rm -f gpurun_out/trace_*.txt
ENERGON_SK_FORCE=2 ENERGON_GEMM_TRACE=gpurun_out/trace_down_sk.txt timeout 120 python scripts/gemm_one.py 4096 5120 2560 0 > /dev/null
ENERGON_NO_STREAMK=1 ENERGON_GEMM_TRACE=gpurun_out/trace_down_dp.txt timeout 120 python scripts/gemm_one.py 4096 5120 2560 0 > /dev/null
python scripts/gemm_trace_sk.py gpurun_out/trace_down_sk.txt 2>/dev/null | head -42
python scripts/gemm_trace_sk.py gpurun_out/trace_down_dp.txt 2>/dev/null | head -12

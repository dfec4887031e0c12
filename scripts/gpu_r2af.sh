mkdir -p gpurun_out
rm -f gpurun_out/trace_*.txt
ENERGON_GEMM_TRACE=gpurun_out/trace_out_sk.txt timeout 120 python scripts/gemm_one.py 4096 5120 5120 0
ENERGON_NO_STREAMK=1 ENERGON_GEMM_TRACE=gpurun_out/trace_out_dp.txt timeout 120 python scripts/gemm_one.py 4096 5120 5120 0
python scripts/gemm_trace_sk.py gpurun_out/trace_out_sk.txt 2>/dev/null | head -40
python scripts/gemm_trace_sk.py gpurun_out/trace_out_dp.txt 2>/dev/null | head -3

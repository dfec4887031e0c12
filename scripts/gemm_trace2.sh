rm -f gpurun_out/gemm_trace.txt
ENERGON_GEMM_TRACE=gpurun_out/gemm_trace.txt python scripts/gemm_one.py 4096 5120 20480 0 > /dev/null
ENERGON_SK_MIN_NKB=16 ENERGON_GEMM_TRACE=gpurun_out/gemm_trace.txt python scripts/gemm_one.py 4096 5120 5120 0 > /dev/null
python scripts/gemm_trace_report.py gpurun_out/gemm_trace.txt 2>&1 | grep -v "^  round" | sort | uniq -c | sort -rn | head -40

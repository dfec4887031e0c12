mkdir -p gpurun_out
rm -f gpurun_out/trace_*.txt
for shape in "4096 1920 5120 1" "4096 2560 5120 2" "4096 5120 640 0"; do
  set -- $shape
  ENERGON_GEMM_TRACE=gpurun_out/trace_sk_$2_$3.txt timeout 120 python scripts/gemm_one.py $shape
  ENERGON_NO_STREAMK=1 ENERGON_GEMM_TRACE=gpurun_out/trace_dp_$2_$3.txt timeout 120 python scripts/gemm_one.py $shape
  python scripts/gemm_trace_sk.py gpurun_out/trace_sk_$2_$3.txt
  python scripts/gemm_trace_sk.py gpurun_out/trace_dp_$2_$3.txt
done

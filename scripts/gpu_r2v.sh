mkdir -p gpurun_out
rm -f gpurun_out/trace_*.txt
for shape in "4096 5120 640 0" "4096 1920 5120 1"; do
  set -- $shape
  ENERGON_GEMM_TRACE=gpurun_out/trace_$2_$3.txt timeout 120 python scripts/gemm_one.py $shape > /dev/null
  python scripts/gemm_trace_sk.py gpurun_out/trace_$2_$3.txt | head -40
done

mkdir -p gpurun_out
rm -f gpurun_out/trace_*.txt
for f in 1 2; do
  ENERGON_SK_FORCE=$f ENERGON_GEMM_TRACE=gpurun_out/trace_sk$f.txt timeout 120 python scripts/gemm_one.py 4096 1920 5120 1 > /dev/null
  python scripts/gemm_trace_sk.py gpurun_out/trace_sk$f.txt | head -36
done

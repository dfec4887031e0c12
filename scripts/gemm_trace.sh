# GEMM unit timelines (ENERGON_GEMM_TRACE) for the short TP=8 shapes and the stream-K MLP-down
rm -f gpurun_out/gemm_trace.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "gemm" 2>&1 | tail -1
for shape in "4096 2560 5120 2" "4096 1920 5120 1" "4096 5120 20480 0"; do
  python scripts/gemm_one.py $shape
  ENERGON_GEMM_TRACE=gpurun_out/gemm_trace.txt python scripts/gemm_one.py $shape > /dev/null
done
python scripts/gemm_trace_report.py gpurun_out/gemm_trace.txt | tee gpurun_out/gemm_trace_report.txt

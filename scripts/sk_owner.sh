timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "gemm or gpt3 or opt" 2>&1 | tail -2
ENERGON_SK_MIN_NKB=16 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "gemm or tiny or gpt2s" 2>&1 | tail -2
for g in 160 32; do
  for shape in "4096 5120 20480 0" "4096 5120 5120 0" "4096 2560 5120 2" "4096 1920 5120 1" "4096 5120 1280 0" "4096 5120 2560 0" "4096 20480 5120 2"; do
    ENERGON_SK_MIN_NKB=$g python scripts/gemm_one.py $shape | sed "s/^/gate=$g /"
  done
done
rm -f gpurun_out/gemm_trace.txt
ENERGON_SK_MIN_NKB=32 ENERGON_GEMM_TRACE=gpurun_out/gemm_trace.txt python scripts/gemm_one.py 4096 2560 5120 2 > /dev/null
python scripts/gemm_trace_report.py gpurun_out/gemm_trace.txt

mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "streamk or gemm" > gpurun_out/pytest_sk_r2e.log 2>&1; rc=$?; echo "sk tests rc=$rc"; tail -3 gpurun_out/pytest_sk_r2e.log
if [ $rc -ne 0 ]; then exit 1; fi
rm -f gpurun_out/trace_*.txt
for shape in "4096 1920 5120 1" "4096 2560 5120 2" "4096 5120 2560 0"; do
  set -- $shape
  ENERGON_SK_FORCE=1 ENERGON_GEMM_TRACE=gpurun_out/trace_sk_$2_$3.txt timeout 120 python scripts/gemm_one.py $shape > /dev/null
  python scripts/gemm_trace_sk.py gpurun_out/trace_sk_$2_$3.txt > gpurun_out/trace_sum_$2_$3.txt; head -30 gpurun_out/trace_sum_$2_$3.txt
done
for k in 8 4 2 1; do K_TP=$k timeout 300 python scripts/bench_gemm.py 2>&1 | grep -v "^{" | sed "s/^/sk  tp$k /"; ENERGON_NO_STREAMK=1 K_TP=$k timeout 300 python scripts/bench_gemm.py 2>&1 | grep -v "^{" | sed "s/^/dp  tp$k /"; done | tee gpurun_out/gemm_sk_ab_r2e.log

# attention v3 iteration: parity under ENERGON_ATTN=5 (short timeouts), microbench, trace
mkdir -p gpurun_out
export ENERGON_ATTN=5
for c in "t128 and 1-bf16-128" "attention_kernel"; do
  timeout 120 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "attention_kernel and $c" > gpurun_out/pytest_attn.log 2>&1; rc=$?; echo "attn tests [$c] rc=$rc"; tail -3 gpurun_out/pytest_attn.log
  if [ $rc -ne 0 ]; then exit 1; fi
done
timeout 300 python scripts/bench_attn.py 2>&1 | tail -6
ATTN_HK=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -6
rm -f gpurun_out/attn_trace_*.txt
ENERGON_ATTN_TRACE=gpurun_out/attn_trace_s2048.txt ATTN_CASES="full S2048" timeout 300 python scripts/bench_attn.py > /dev/null 2>&1
ENERGON_ATTN_TRACE=gpurun_out/attn_trace_gpt3.txt ATTN_CASES="gpt3" timeout 300 python scripts/bench_attn.py > /dev/null 2>&1
python scripts/attn_trace_report.py gpurun_out/attn_trace_s2048.txt 2>/dev/null | head -24
python scripts/attn_trace_report.py gpurun_out/attn_trace_gpt3.txt 2>/dev/null | head -30
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x -k "attention or opt or gpt3 or tiny or edge or fused or graph" > gpurun_out/pytest_attn_wide.log 2>&1; echo "wide rc=$?"; tail -2 gpurun_out/pytest_attn_wide.log

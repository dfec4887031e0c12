# sanitizers on the round-2 kernels: TMA a5 epilogue, LN-prologue GEMM, batched-issue attention, stream-K preload
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider \
    -k "fused_layout or ln_prologue or attention_kernel_vs_oracle or streamk or tiny_vs_oracle" > gpurun_out/sanitize_${tool}_r2al.log 2>&1
  echo "$tool exit $?"; tail -2 gpurun_out/sanitize_${tool}_r2al.log
done
grep -h "Race reported between" gpurun_out/sanitize_racecheck_r2al.log | sed 's/0x[0-9a-f]*//g; s/(.*)//' | sort | uniq -c | head

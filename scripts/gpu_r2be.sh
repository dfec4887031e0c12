# compute-sanitizer on the last session's kernels: the attention TMA-store epilogue (v2 default, v3 via ENERGON_ATTN=5)
# and the 256 x 224 pair GEMM tile
mkdir -p gpurun_out
K="attention_kernel or every_tile_shape or tile224 or fused_layout or streamk"
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "$K" -p no:cacheprovider > gpurun_out/sanitize_${tool}_r2last.log 2>&1
  echo "$tool exit $?"; tail -3 gpurun_out/sanitize_${tool}_r2last.log
done
for tool in memcheck racecheck; do
  ENERGON_ATTN=5 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "attention_kernel_vs_oracle" -p no:cacheprovider > gpurun_out/sanitize_${tool}_attn5_r2last.log 2>&1
  echo "v3 $tool exit $?"; tail -2 gpurun_out/sanitize_${tool}_attn5_r2last.log
done

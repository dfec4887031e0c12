# compute-sanitizer memcheck / racecheck / synccheck on the small configs (SURVEY.md sec 4 tier 6)
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -m gpu \
    -k "tiny_vs_oracle or local_tp_vs_oracle or attention_kernel or every_tile_shape or index_maps or streamk or graph" -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?"; tail -4 gpurun_out/sanitize_$tool.log
done
# the pipeline stages and the P2P exchange (2 processes) under memcheck
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_pipeline.py -q -x -m gpu \
  -k "stage_chain or validation" -p no:cacheprovider > gpurun_out/sanitize_memcheck_pipeline.log 2>&1
echo "memcheck pipeline exit $?"; tail -3 gpurun_out/sanitize_memcheck_pipeline.log
# memcheck on the two-process P2P exchange (incl. the fused GEMM -> reduce-scatter peer TMA stores)
timeout 1200 compute-sanitizer --tool memcheck --target-processes all --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_p2p.py -q -x -p no:cacheprovider > gpurun_out/sanitize_memcheck_p2p.log 2>&1
echo "memcheck p2p exit $?"; tail -4 gpurun_out/sanitize_memcheck_p2p.log

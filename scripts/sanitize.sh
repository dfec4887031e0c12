# compute-sanitizer memcheck / racecheck / synccheck on the small configs (SURVEY.md sec 4 tier 6)
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -m gpu \
    -k "tiny_vs_oracle or local_tp_vs_oracle or attention_kernel or every_tile_shape or index_maps or streamk" -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?"; tail -4 gpurun_out/sanitize_$tool.log
done

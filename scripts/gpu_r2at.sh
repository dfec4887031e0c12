mkdir -p gpurun_out
ENERGON_ATTN=5 timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "attention_kernel_vs_oracle" 2>&1 | tail -1
for rep in 1 2; do echo "== v3"; ENERGON_ATTN=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5; done
ENERGON_ATTN=5 timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "attention_kernel_vs_oracle" -p no:cacheprovider > gpurun_out/sanitize_racecheck_v3relaxed.log 2>&1
echo "racecheck exit $?"; tail -2 gpurun_out/sanitize_racecheck_v3relaxed.log

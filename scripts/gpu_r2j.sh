# Round 2, call j: attention v3 (FA4 layout) -- correctness first under short timeouts, then micro A/B.
mkdir -p gpurun_out
for c in "t64 and 1-bf16-128" "t128 and 1-bf16-128" "t128 and 0-bf16-128" "t128 and bf16-64" "attention_kernel"; do
  timeout 120 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "attention_kernel and $c" > gpurun_out/pytest_attn_r2j.log 2>&1; rc=$?; echo "attn tests [$c] rc=$rc"; tail -3 gpurun_out/pytest_attn_r2j.log
  if [ $rc -ne 0 ]; then exit 1; fi
done
ENERGON_ATTN=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -6
ENERGON_ATTN=4 timeout 300 python scripts/bench_attn.py 2>&1 | tail -6
ENERGON_ATTN=5 ATTN_HK=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -6
ENERGON_ATTN=4 ATTN_HK=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -6
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_r2j.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_r2j.log

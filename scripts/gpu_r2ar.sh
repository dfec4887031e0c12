mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "attention_kernel_vs_oracle or tiny_vs_oracle or fused_layout or gpt2s" > gpurun_out/pytest_attnprod.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -1 gpurun_out/pytest_attnprod.log
if [ $rc -ne 0 ]; then exit 1; fi
for rep in 1 2; do
  echo "== warp (mma+tma)"; timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
  echo "== lane (mma+tma)"; AB_LIB=paper_2209_02341_b200/lib/ab/attn_lane.so timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
done
ATTN_HK=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5

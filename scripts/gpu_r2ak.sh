# attention v2: batched MMA issue (default) vs per-MMA issue (ATTN_MMA_BATCH=0): parity, then micro A/B x2
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "attention_kernel_vs_oracle and not v3" 2>&1 | tail -1
for rep in 1 2; do
  echo "== batched"; timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
  echo "== per-MMA"; AB_LIB=paper_2209_02341_b200/lib/ab/nobatch.so timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
done

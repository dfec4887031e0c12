# attention v2: two epilogue staging buffers per softmax warp (no alignment slack) vs one (lib/ab/stg1.so)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "attention or opt or fused or gpt3 or edge or tiny or gpt2s or graph or full or layout" 2>&1 | tail -2
for rep in 1 2; do
  echo "== stg2"; timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
  echo "== stg1"; AB_LIB=paper_2209_02341_b200/lib/ab/stg1.so timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
done
echo "== TP8 (5 heads) stg2"; ATTN_HK=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
echo "== TP8 (5 heads) stg1"; ATTN_HK=5 AB_LIB=paper_2209_02341_b200/lib/ab/stg1.so timeout 300 python scripts/bench_attn.py 2>&1 | tail -5

# v2 attention: dead-warp / invisible-chunk skip (ATTN2_SKIP=1, default) vs -DATTN2_SKIP=0 (lib/ab/noskip.so)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "attention or opt or fused or gpt3 or edge or tiny or gpt2s or graph or full" 2>&1 | tail -1
for rep in 1 2; do
  echo "== skip"; timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
  echo "== noskip"; AB_LIB=paper_2209_02341_b200/lib/ab/noskip.so timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
done
echo "== TP8 (5 heads) skip"; ATTN_HK=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
echo "== TP8 (5 heads) noskip"; ATTN_HK=5 AB_LIB=paper_2209_02341_b200/lib/ab/noskip.so timeout 300 python scripts/bench_attn.py 2>&1 | tail -5

# attention v2 without the per-tile observation of the previous P V (o_full) after the P hand-over: parity (twice), A/B
mkdir -p gpurun_out
for rep in 1 2; do
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "attention or opt or fused or gpt3 or edge or tiny or gpt2s or graph or full or layout" 2>&1 | tail -1
done
for rep in 1 2; do
  echo "== new"; timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
  echo "== observe all"; AB_LIB=paper_2209_02341_b200/lib/ab/obsall.so timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
done
echo "== TP8 (5 heads) new"; ATTN_HK=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
echo "== TP8 (5 heads) observe all"; ATTN_HK=5 AB_LIB=paper_2209_02341_b200/lib/ab/obsall.so timeout 300 python scripts/bench_attn.py 2>&1 | tail -5

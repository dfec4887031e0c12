# attention v2: one 3-D TMA load per Q / K / V tile (default) vs one per 64-column half (ENERGON_NO_ATTN_TMA3=1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "attention or opt or fused or gpt3 or edge or tiny or gpt2s or graph or full or layout" 2>&1 | tail -1
for rep in 1 2; do
  echo "== tma3"; timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
  echo "== 2 halves"; ENERGON_NO_ATTN_TMA3=1 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
done
echo "== TP8 (5 heads) tma3"; ATTN_HK=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
echo "== TP8 (5 heads) 2 halves"; ATTN_HK=5 ENERGON_NO_ATTN_TMA3=1 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5

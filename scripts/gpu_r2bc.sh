# attention: partial-warp rows by 256-bit stores (STG.E.256) next to the TMA box stores; fallback everywhere = v8 stores
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "attention or opt or fused or gpt3 or edge or tiny or gpt2s or graph or full or layout" 2>&1 | tail -2
ENERGON_NO_ATTN_TMA=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "attention or fused or layout" 2>&1 | tail -2
for rep in 1 2; do
  echo "== tma + v8 partial"; timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
  echo "== v8 everywhere"; ENERGON_NO_ATTN_TMA=1 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
done
echo "== TP8 (5 heads) tma + v8"; ATTN_HK=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
echo "== TP8 (5 heads) v8"; ATTN_HK=5 ENERGON_NO_ATTN_TMA=1 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5

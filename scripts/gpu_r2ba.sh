# attention v2 TMA-store epilogue, 16-column double-buffered staging: parity, then A/B vs the per-thread stores
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "attention or opt or fused or gpt3 or edge or tiny or gpt2s or graph or full or layout" 2>&1 | tail -2
for rep in 1 2; do
  echo "== tma16x2"; timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
  echo "== per-thread"; ENERGON_NO_ATTN_TMA=1 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
done
echo "== TP8 (5 heads) tma16x2"; ATTN_HK=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5

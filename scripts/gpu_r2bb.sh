# attention TMA-store epilogue (32 x 32 boxes, one staging buffer per warp) in v2 and v3: parity, A/B, in-step A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "attention or opt or fused or gpt3 or edge or tiny or gpt2s or graph or full or layout" 2>&1 | tail -2
for rep in 1 2; do
  echo "== v2 tma"; timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
  echo "== v2 per-thread"; ENERGON_NO_ATTN_TMA=1 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
done
echo "== v3 tma"; ENERGON_ATTN=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
echo "== v3 per-thread"; ENERGON_ATTN=5 ENERGON_NO_ATTN_TMA=1 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
echo "== TP8 (5 heads) v2 tma"; ATTN_HK=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
echo "== TP8 (5 heads) v3 tma"; ATTN_HK=5 ENERGON_ATTN=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
for rep in 1 2; do
  timeout 900 python bench.py --steps 10 --no-cpu-baseline --no-ab --no-e2e > gpurun_out/bench_attntma_$rep.json 2>/dev/null
  ENERGON_NO_ATTN_TMA=1 timeout 900 python bench.py --steps 10 --no-cpu-baseline --no-ab --no-e2e > gpurun_out/bench_attnthr_$rep.json 2>/dev/null
  python -c "
import json
for t in ('tma','thr'):
    d=json.load(open('gpurun_out/bench_attn'+t+'_$rep.json')); print(t, d['value'], d['ms_per_step'], d['phases']['attention'], d['clocks']['sm_mhz'])"
done

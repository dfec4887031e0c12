# attention v2: L2 prefetch of the next item's Q / K / V by the producer (default) vs none (lib/ab/nopf.so)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "attention or opt or fused or gpt3 or edge or tiny or gpt2s or graph or full or layout" 2>&1 | tail -1
for rep in 1 2; do
  echo "== prefetch"; timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
  echo "== none"; AB_LIB=paper_2209_02341_b200/lib/ab/nopf.so timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
done
echo "== TP8 (5 heads) prefetch"; ATTN_HK=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
echo "== TP8 (5 heads) none"; ATTN_HK=5 AB_LIB=paper_2209_02341_b200/lib/ab/nopf.so timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
for rep in 1 2; do
  timeout 900 python bench.py --steps 10 --no-cpu-baseline --no-ab --no-e2e > gpurun_out/bench_pf_$rep.json 2>/dev/null
  AB_LIB=paper_2209_02341_b200/lib/ab/nopf.so timeout 900 python bench.py --steps 10 --no-cpu-baseline --no-ab --no-e2e > gpurun_out/bench_nopf_$rep.json 2>/dev/null
  python -c "
import json
for t in ('pf','nopf'):
    d=json.load(open('gpurun_out/bench_'+t+'_$rep.json')); print(t, d['value'], d['ms_per_step'], d['phases']['attention'], d['clocks']['sm_mhz'])"
done

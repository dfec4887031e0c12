# emulated TP = 8 / 4 / 2 steps at HEAD (per-rank kernel shapes), with the post-timing TP check
mkdir -p gpurun_out
for k in 8 4 2; do
  timeout 900 python bench.py --local-tp $k --no-cpu-baseline --no-ab --no-e2e --steps 5 > gpurun_out/bench_ltp${k}_r2ah.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_ltp${k}_r2ah.json')); p=d['phases']; print('ltp$k', round(d['ms_per_step'],2), 'gemm', round(p['gemm']['ms_per_step'],2), round(p['gemm']['tflops']), 'attn', round(p['attention']['ms_per_step'],2), 'mem', round(p['memory_bound']['ms_per_step'],2), 'exch', round(p['exchange']['ms_per_step'],2), d['tp_check'].get('max_abs_rel_vs_tp1'), d['clocks']['sm_mhz'])"
done
export ENERGON_PROFILE_RANGE=1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/launches_ltp8_r2ah.csv python bench.py --local-tp 8 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab --no-tp-check --graph 0 --layers 4 > /dev/null 2>&1
python - <<PY
import csv, collections
rows=list(csv.reader(open('gpurun_out/launches_ltp8_r2ah.csv'))); h=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]; hdr=rows[h]
kn,mn,mv=hdr.index('Kernel Name'),hdr.index('Metric Name'),hdr.index('Metric Value')
agg=collections.defaultdict(list)
for r in rows[h+1:]:
    agg[(r[kn].split('(')[0], r[mn])].append(float(r[mv].replace(',','')))
for (k,m),v in sorted(agg.items()):
    print(k[:44].ljust(44), m[:32].ljust(32), round(sum(v)/len(v),2), len(v))
PY

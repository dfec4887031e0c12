# residual + LN threads per row: 512 (default at TP = 1) vs 640 (exactly 2 float4 per thread at H = 5120)
mkdir -p gpurun_out
export ENERGON_PROFILE_RANGE=1
for tpr in 512 640; do
  ENERGON_LN_TPR=$tpr timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:residual_ln --csv --log-file gpurun_out/ln_$tpr.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab --no-tp-check --graph 0 --layers 8 > /dev/null 2>&1
  python - <<PY
import csv, collections
rows=list(csv.reader(open('gpurun_out/ln_$tpr.csv'))); h=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]; hdr=rows[h]
mn,mv=hdr.index('Metric Name'),hdr.index('Metric Value')
agg=collections.defaultdict(list)
for r in rows[h+1:]: agg[r[mn]].append(float(r[mv].replace(',','')))
print('tpr=$tpr', {k: round(sum(v)/len(v),1) for k,v in agg.items()}, len(agg['gpu__time_duration.sum']))
PY
done
unset ENERGON_PROFILE_RANGE
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "tiny_vs_oracle or gpt3_13b_layer" > /dev/null 2>&1; echo "tests default rc=$?"
ENERGON_LN_TPR=640 timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "gpt3_13b_layer or opt_layer" 2>&1 | tail -1
for rep in 1 2; do for tpr in 512 640; do
  ENERGON_LN_TPR=$tpr timeout 900 python bench.py --no-cpu-baseline --no-ab --no-e2e --no-tp-check --steps 20 > gpurun_out/bench_tpr$tpr.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_tpr$tpr.json')); print('tpr=$tpr rep=$rep', round(d['ms_per_step'],2), round(d['value']), d['clocks']['sm_mhz'])"
done; done

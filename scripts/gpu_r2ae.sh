# a5 by TMA: parity first (short timeouts), then the QKV GEMM in the step (ncu) and the bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "fused_layout or tiny_vs_oracle or gpt2s or gpt3_13b_layer or edge or graph or local_tp" > gpurun_out/pytest_qkvtma.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/pytest_qkvtma.log
if [ $rc -ne 0 ]; then exit 1; fi
export ENERGON_PROFILE_RANGE=1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/launches_qkvtma.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab --no-tp-check --graph 0 --layers 8 > /dev/null 2>&1
python - <<PY
import csv, collections
rows=list(csv.reader(open('gpurun_out/launches_qkvtma.csv'))); h=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]; hdr=rows[h]
kn,mn,mv=hdr.index('Kernel Name'),hdr.index('Metric Name'),hdr.index('Metric Value')
agg=collections.defaultdict(list)
for r in rows[h+1:]:
    agg[(r[kn].split('(')[0], r[mn])].append(float(r[mv].replace(',','')))
for (k,m),v in sorted(agg.items()):
    if 'gemm' in k or 'attention' in k: print(k[:40].ljust(40), m[:40].ljust(40), round(sum(v)/len(v),2), len(v))
PY
unset ENERGON_PROFILE_RANGE
for rep in 1 2; do
  for nt in 0 1; do
    if [ $nt = 1 ]; then export ENERGON_NO_QKV_TMA=1; else unset ENERGON_NO_QKV_TMA; fi
    timeout 900 python bench.py --no-cpu-baseline --no-ab --no-e2e --no-tp-check --steps 20 > gpurun_out/bench_qkvtma_$nt.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/bench_qkvtma_$nt.json')); print('no_qkv_tma=$nt rep=$rep', round(d['ms_per_step'],2), round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
  done
done
unset ENERGON_NO_QKV_TMA

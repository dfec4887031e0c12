# QKV GEMM: scatter epilogue (a5 fused, EPI_BIAS_QKV) vs TMA-store epilogue (EPI_BIAS + standalone unpack): ncu launch lists
mkdir -p gpurun_out
export ENERGON_PROFILE_RANGE=1
for nf in 0 1; do
  if [ $nf = 1 ]; then export ENERGON_NO_FUSE=1; else unset ENERGON_NO_FUSE; fi
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/launches_nf${nf}.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab --no-tp-check --graph 0 --layers 8 > /dev/null 2>&1
  python - <<PY
import csv, collections
rows=list(csv.reader(open('gpurun_out/launches_nf${nf}.csv'))); h=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]; hdr=rows[h]
kn,mn,mv=hdr.index('Kernel Name'),hdr.index('Metric Name'),hdr.index('Metric Value')
agg=collections.defaultdict(list)
for r in rows[h+1:]:
    agg[(r[kn].split('(')[0], r[mn])].append(float(r[mv].replace(',','')))
for (k,m),v in sorted(agg.items()):
    print('nf=${nf}', k[:40].ljust(40), m[:40].ljust(40), round(sum(v)/len(v),2), len(v))
PY
done

# TP=k per-rank shapes emulated on one GPU (bench --local-tp k: k contexts, in-device rank-order reductions)
for k in 2 4 8; do
  timeout 600 python bench.py --local-tp $k --steps 5 --warmup 3 --no-e2e --no-ab --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ltp_$k.json
  python -c "
import json; d=json.load(open('gpurun_out/ltp_$k.json')); p=d['phases']
print(json.dumps({'local_tp': $k, 'ms_per_step_all_ranks_serial': d['ms_per_step'], 'gemm_ms_per_rank': p['gemm']['ms_per_step']/$k, 'gemm_tflops': p['gemm']['tflops'], 'attention_ms_per_rank': p['attention']['ms_per_step']/$k, 'memory_ms_per_rank': p['memory_bound']['ms_per_step']/$k, 'sm_mhz': d['clocks']['sm_mhz']}))" | tee -a gpurun_out/local_tp_sweep.jsonl
done

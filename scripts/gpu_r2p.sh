# changing-batch (5 rotated seeds) vs fixed-batch (1 seed) step time at configs 2 and 3; v3 subprocess test
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "attention_v3" 2>&1 | tail -2
for cfg in gpt2s gpt3_13b; do
  for sd in 5 1; do
    for rep in 1 2; do
      timeout 900 python bench.py --config $cfg --seeds $sd --no-cpu-baseline --no-ab --no-e2e --steps 20 > gpurun_out/bench_${cfg}_s${sd}_${rep}.json 2>>gpurun_out/bench_r2p.err
      python -c "
import json; d=json.load(open('gpurun_out/bench_${cfg}_s${sd}_${rep}.json')); print('$cfg seeds=$sd rep=$rep', round(d['value']), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['per_seed']['ms_median'].items()}, d['clocks']['sm_mhz'])"
    done
  done
done 2>&1 | tee gpurun_out/seeds_ab_r2p.log

# Final evidence of round 2 at HEAD: the round-end sequence (GPU suite, smoke, default bench), launch list + ncu full,
# attention micro bench, config-2 tile-policy A/B, emulated TP = 8 with the TP check, 2-rank self-launch on one GPU
bash scripts/round_evidence.sh
for rep in 1 2; do
  timeout 600 python bench.py --config gpt2s --steps 50 --no-cpu-baseline --no-ab --no-e2e > gpurun_out/bench_gpt2s_224_$rep.json 2>/dev/null
  ENERGON_NO_TILE224=1 timeout 600 python bench.py --config gpt2s --steps 50 --no-cpu-baseline --no-ab --no-e2e > gpurun_out/bench_gpt2s_256_$rep.json 2>/dev/null
  python -c "
import json
for t in ('224','256'):
    d=json.load(open('gpurun_out/bench_gpt2s_'+t+'_$rep.json')); print('gpt2s', t, d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
timeout 900 python bench.py --local-tp 8 --no-cpu-baseline --no-ab --no-e2e --steps 5 > gpurun_out/bench_ltp8_final.json 2>gpurun_out/bench_ltp8_final.err; python -c "
import json; d=json.load(open('gpurun_out/bench_ltp8_final.json')); print('ltp8', d['value'], d['ms_per_step'], d['phases'], d.get('tp_check'), d['clocks'])"
ENERGON_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 2 --warmup 3 --layers 4 > gpurun_out/bench_n2.log 2>&1; echo "n2 rc=$?"; tail -c 1200 gpurun_out/bench_n2.log

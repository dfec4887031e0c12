# Round-2 bench lines for configs 2, 4, 5 at HEAD (TP = 1 on one B200; DRCE A/B), and the paper regime of config 3
mkdir -p gpurun_out
for cfg in gpt2s opt30b opt66b; do
  timeout 1500 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/bench_${cfg}_r2ac.json 2>gpurun_out/bench_${cfg}_r2ac.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_${cfg}_r2ac.json')); print('$cfg', round(d['value']), round(d['ms_per_step'],2), 'gemm', round(d['phases']['gemm']['tflops']), 'attn', round(d['phases']['attention']['tflops'] or 0), 'drce', round(d['drce_ab']['latency_reduction'],3), d['clocks']['sm_mhz'])"
done
timeout 900 python bench.py --regime paper --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/bench_gpt3_paper_r2ac.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_gpt3_paper_r2ac.json')); print('gpt3 paper regime', round(d['value']), round(d['ms_per_step'],2), round(d['drce_ab']['latency_reduction'],3))"

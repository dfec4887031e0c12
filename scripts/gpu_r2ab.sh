mkdir -p gpurun_out
ENERGON_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --config gpt2s --steps 3 --warmup 3 --no-ab --no-e2e > gpurun_out/bench_share2_r2ab.json 2>gpurun_out/bench_share2_r2ab.err; python -c "
import json; d=json.load(open('gpurun_out/bench_share2_r2ab.json')); print('share2', d.get('tp_check'), d['config'].get('tp_exchange'), d['config'].get('p2p_fallback'))"; tail -2 gpurun_out/bench_share2_r2ab.err
timeout 900 python bench.py --local-tp 2 --config gpt2s --no-cpu-baseline --no-ab --no-e2e --steps 5 > gpurun_out/bench_ltp2_r2ab.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_ltp2_r2ab.json')); print('ltp2', d['tp_check'])"

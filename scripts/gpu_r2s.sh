# tp_check in the bench (emulated TP=8, 2 ranks sharing one GPU over P2P), default bench, full GPU suite
mkdir -p gpurun_out
timeout 900 python bench.py --local-tp 8 --no-cpu-baseline --no-ab --no-e2e --steps 5 > gpurun_out/bench_ltp8_r2s.json 2>gpurun_out/bench_ltp8_r2s.err; python -c "
import json; d=json.load(open('gpurun_out/bench_ltp8_r2s.json')); print('ltp8', d['ms_per_step'], d['phases']['gemm']['tflops'], d['tp_check'], d['clocks'])"; tail -2 gpurun_out/bench_ltp8_r2s.err
ENERGON_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --config gpt2s --steps 3 --warmup 3 --no-ab --no-e2e > gpurun_out/bench_share2_r2s.json 2>gpurun_out/bench_share2_r2s.err; python -c "
import json; d=json.load(open('gpurun_out/bench_share2_r2s.json')); print('share2', d.get('tp_check'), d.get('exchange'))"; tail -3 gpurun_out/bench_share2_r2s.err
ENERGON_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-ab --no-e2e --layers 4 > gpurun_out/bench_share2_gpt3_r2s.json 2>>gpurun_out/bench_share2_r2s.err; python -c "
import json; d=json.load(open('gpurun_out/bench_share2_gpt3_r2s.json')); print('share2 gpt3 4 layers', d.get('tp_check'))"
timeout 900 python bench.py > gpurun_out/bench_r2s.json 2>gpurun_out/bench_r2s.err; python -c "
import json; d=json.load(open('gpurun_out/bench_r2s.json')); print('tp1', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'], d.get('tp_check'))"
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r2s.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_r2s.log

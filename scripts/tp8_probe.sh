mkdir -p gpurun_out
K_TP=8 timeout 300 python scripts/bench_gemm.py 2>&1 | grep -v "^{"
K_TP=4 timeout 300 python scripts/bench_gemm.py 2>&1 | grep -v "^{"
K_TP=1 timeout 300 python scripts/bench_gemm.py 2>&1 | grep -v "^{"
timeout 600 python bench.py --local-tp 8 --steps 5 --warmup 3 --no-e2e --no-ab --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_ltp8.json
python -c "
import json; d=json.load(open('gpurun_out/bench_ltp8.json')); print(d['ms_per_step'], d['phases'], d['roofline']['achieved'], d['clocks'])"

timeout 900 python -m pytest tests -m gpu -x -q --timeout=300 > gpurun_out/pytest_gpu.log 2>&1
tail -4 gpurun_out/pytest_gpu.log
timeout 500 python scripts/sweep_tiles.py > gpurun_out/sweep.log 2>&1; head -16 gpurun_out/sweep.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-ab > gpurun_out/bench_tp1.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_tp1.log').read().strip().splitlines()[-1]); print('tp1', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
timeout 900 python bench.py --local-tp 8 --steps 3 --warmup 2 --no-cpu-baseline --no-ab --no-e2e > gpurun_out/bench_ltp8.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_ltp8.log').read().strip().splitlines()[-1]); print('ltp8', d['value'], d['ms_per_step'], json.dumps(d['phases']['gemm']))"

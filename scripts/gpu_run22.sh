timeout 900 python -m pytest tests -m gpu -x -q --timeout=300 > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_full.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'], json.dumps(d['phases']), d['roofline']['frac'], d['drce_ab']['latency_reduction'], d['cpu_baseline'])"

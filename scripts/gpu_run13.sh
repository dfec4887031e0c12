timeout 900 python -m pytest tests -m gpu -x -q --timeout=300 > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
for v in 0 1; do
ENERGON_NO_PDL=$v timeout 300 python bench.py --config gpt2s --steps 20 --warmup 5 --no-cpu-baseline --no-ab > gpurun_out/bench_gpt2s_pdl$v.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_gpt2s_pdl$v.log').read().strip().splitlines()[-1]); print('gpt2s nopdl=$v', d['value'], d['ms_per_step'], d['e2e']['ms_per_step'])"
ENERGON_NO_PDL=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-ab --no-e2e > gpurun_out/bench_full_pdl$v.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_full_pdl$v.log').read().strip().splitlines()[-1]); print('gpt3 nopdl=$v', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done

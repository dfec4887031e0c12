export ENERGON_PROFILE_RANGE=1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gpt2s.csv python bench.py --config gpt2s --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab > /dev/null 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_gpt2s.csv
unset ENERGON_PROFILE_RANGE
timeout 300 python bench.py --config gpt2s --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_gpt2s.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_gpt2s.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], json.dumps(d['phases']))"

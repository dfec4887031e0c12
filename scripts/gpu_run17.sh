timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_tp1.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_tp1.log').read().strip().splitlines()[-1]); print('tp1', d['value'], d['ms_per_step'], d['roofline']['frac'], json.dumps(d['drce_ab']))"
timeout 900 python bench.py --local-tp 8 --steps 3 --warmup 2 --no-cpu-baseline --no-ab --no-e2e > gpurun_out/bench_ltp8.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_ltp8.log').read().strip().splitlines()[-1]); print('ltp8', d['value'], d['ms_per_step'], json.dumps(d['phases']))"
export ENERGON_PROFILE_RANGE=1
timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:gemm_tc2 -c 4 -o gpurun_out/prof_ltp8 python bench.py --local-tp 8 --steps 1 --warmup 1 --no-cpu-baseline --no-ab --no-e2e --layers 2 > /dev/null 2>&1
python scripts/ncu_summary.py full gpurun_out/prof_ltp8.ncu-rep

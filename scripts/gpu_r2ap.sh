# Round-2 evidence at HEAD (after the warp-converged issue): full GPU suite, smoke, default bench (JSON line), ncu launch list of one
# step, ncu --set full of two layers, attention micro bench
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/pytest_gpu_r2ap.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_r2ap.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_r2ap.json 2>gpurun_out/bench_r2ap.err; python -c "
import json; d=json.load(open('gpurun_out/bench_r2ap.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'], d['cpu_baseline']['value'])"
export ENERGON_PROFILE_RANGE=1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2ap.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab --graph 0 > gpurun_out/ncu_launch_run.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -c 9 -o gpurun_out/prof_full_r2ap -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab --layers 2 --graph 0 > gpurun_out/ncu_full_run.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_r2ap.csv > gpurun_out/launches_summary_r2ap.md
python scripts/ncu_summary.py full gpurun_out/prof_full_r2ap.ncu-rep > gpurun_out/full_summary_r2ap.md
cat gpurun_out/launches_summary_r2ap.md
unset ENERGON_PROFILE_RANGE
timeout 300 python scripts/bench_attn.py 2>&1 | tail -5 > gpurun_out/attn_bench_r2ap.txt; cat gpurun_out/attn_bench_r2ap.txt

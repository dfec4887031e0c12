# Round profile evidence (current code): launch list of one bench step (graphs off so ncu sees each
# launch), ncu --set full of one layer's kernels, attention micro-benchmark.
mkdir -p gpurun_out
export ENERGON_PROFILE_RANGE=1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab --graph 0 > gpurun_out/ncu_launch_run.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -c 9 -o gpurun_out/prof_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab --layers 2 --graph 0 > gpurun_out/ncu_full_run.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/launches_summary.md
python scripts/ncu_summary.py full gpurun_out/prof_full.ncu-rep > gpurun_out/full_summary.md
cat gpurun_out/launches_summary.md; cat gpurun_out/full_summary.md
unset ENERGON_PROFILE_RANGE
timeout 300 python scripts/bench_attn.py 2>&1 | tail -5

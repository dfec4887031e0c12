# ncu evidence for profiles/: launch list of one bench step + --set full of one layer's kernels
set -x
export ENERGON_PROFILE_RANGE=1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab > gpurun_out/ncu_launch_run.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -c 7 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab --layers 2 > gpurun_out/ncu_full_run.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/launches_summary.md
python scripts/ncu_summary.py full gpurun_out/prof_full.ncu-rep > gpurun_out/full_summary.md
python scripts/traffic_json.py gpurun_out/prof_full.ncu-rep gpt3_13b 1 gpurun_out/gemm_traffic.json
cat gpurun_out/launches_summary.md

# emulated TP = 8 step with the 256 x 224 tile: ncu --set full of the first rank's four GEMMs, and the launch list
mkdir -p gpurun_out
export ENERGON_PROFILE_RANGE=1
timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:gemm_tc2 -c 8 -o gpurun_out/prof_ltp8 -f python bench.py --local-tp 8 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab --no-tp-check --graph 0 --layers 2 > gpurun_out/ncu_ltp8_run.log 2>&1; echo "ncu full rc=$?"
python scripts/ncu_summary.py full gpurun_out/prof_ltp8.ncu-rep > gpurun_out/ltp8_full_summary.md; cat gpurun_out/ltp8_full_summary.md | cut -c1-300
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ltp8.csv python bench.py --local-tp 8 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab --no-tp-check --graph 0 --layers 4 > /dev/null 2>&1; echo "ncu list rc=$?"
python scripts/ncu_summary.py launches gpurun_out/launches_ltp8.csv > gpurun_out/launches_ltp8_summary.md; cat gpurun_out/launches_ltp8_summary.md

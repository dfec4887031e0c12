# Emulated TP=8 step (config 3): ncu launch list of one step, ncu --set full of one layer's 8 ranks' GEMMs;
# racecheck of the v3 attention after the atomics change
mkdir -p gpurun_out
export ENERGON_PROFILE_RANGE=1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ltp8_r2u.csv python bench.py --local-tp 8 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab --no-tp-check --graph 0 > gpurun_out/ncu_ltp8_launch.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_ltp8_r2u.csv > gpurun_out/launches_ltp8_summary_r2u.md; cat gpurun_out/launches_ltp8_summary_r2u.md
timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:gemm_tc2 -c 32 -o gpurun_out/prof_ltp8_r2u -f python bench.py --local-tp 8 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab --no-tp-check --layers 1 --graph 0 > gpurun_out/ncu_ltp8_full.log 2>&1
python scripts/ncu_summary.py full gpurun_out/prof_ltp8_r2u.ncu-rep > gpurun_out/full_ltp8_summary_r2u.md; head -40 gpurun_out/full_ltp8_summary_r2u.md | cut -c1-400
unset ENERGON_PROFILE_RANGE
ENERGON_ATTN=5 timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "attention_kernel_vs_oracle" -p no:cacheprovider > gpurun_out/sanitize_racecheck_attn5.log 2>&1
echo "racecheck attn=5 exit $?"; tail -2 gpurun_out/sanitize_racecheck_attn5.log

export ENERGON_PROFILE_RANGE=1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 1 -c 1 -o gpurun_out/prof_ltp8_out python bench.py --local-tp 8 --steps 1 --warmup 1 --no-cpu-baseline --no-ab --no-e2e --layers 1 > /dev/null 2>&1
ls -la gpurun_out/prof_ltp8_out.ncu-rep

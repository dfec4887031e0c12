export ENERGON_PROFILE_RANGE=1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attention_tc -c 1 -o gpurun_out/prof_attn_tc python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab --layers 2 > gpurun_out/ncu_attn.log 2>&1
tail -2 gpurun_out/ncu_attn.log

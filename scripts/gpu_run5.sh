timeout 900 python -m pytest tests -m gpu -x -q --timeout=300 > gpurun_out/pytest_gpu.log 2>&1
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python scripts/bench_gemm.py > gpurun_out/bench_gemm.log 2>&1; tail -5 gpurun_out/bench_gemm.log | head -4
K_TP=8 timeout 300 python scripts/bench_gemm.py > gpurun_out/bench_gemm_tp8.log 2>&1; tail -5 gpurun_out/bench_gemm_tp8.log | head -4
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1
tail -3 gpurun_out/bench_full.log
export ENERGON_PROFILE_RANGE=1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"residual_ln|gemm_tc2" -c 6 -o gpurun_out/prof_r5 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --layers 2 > gpurun_out/ncu_full_run.log 2>&1
tail -2 gpurun_out/ncu_full_run.log

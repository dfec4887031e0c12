timeout 900 python -m pytest tests -m gpu -x -q --timeout=300 > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1
tail -3 gpurun_out/bench_full.log
timeout 600 python scripts/padding_sweep.py > gpurun_out/padding_sweep.log 2>&1; tail -5 gpurun_out/padding_sweep.log

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q --timeout=400 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
tail -40 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --layers 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_l2.log 2>&1
tail -5 gpurun_out/bench_l2.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1
tail -5 gpurun_out/bench_full.log

timeout 900 python -m pytest tests -m gpu -x -q --timeout=300 > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
bash scripts/ab_variants.sh > gpurun_out/ab.log 2>&1; cat gpurun_out/ab.log
timeout 300 python bench.py --config gpt2s --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_gpt2s.log 2>&1; tail -1 gpurun_out/bench_gpt2s.log | cut -c1-600

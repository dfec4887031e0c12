# Round 2, first GPU call: full GPU suite (new parity tests), smoke, default bench, 2-rank shared-GPU bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu_r2a.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu_r2a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2a.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_r2a.log
timeout 900 python bench.py > gpurun_out/bench_r2a.json 2>gpurun_out/bench_r2a.err; echo "bench rc=$?"; head -c 3000 gpurun_out/bench_r2a.json; tail -3 gpurun_out/bench_r2a.err
ENERGON_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --config gpt2s --steps 3 --warmup 3 --no-ab > gpurun_out/bench_share2_r2a.json 2>gpurun_out/bench_share2_r2a.err; echo "share2 rc=$?"; head -c 1500 gpurun_out/bench_share2_r2a.json; tail -3 gpurun_out/bench_share2_r2a.err

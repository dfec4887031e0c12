timeout 900 python -m pytest tests -m gpu -x -q --timeout=300 > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
cat > /tmp/ab.sh <<'XX'
run() { env "$@" timeout 300 python bench.py --steps 6 --warmup 2 --no-e2e --no-cpu-baseline --no-ab 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']
print('$*', 'ms/step %.2f'%d['ms_per_step'], 'gemm %.2f'%p['gemm']['ms_per_step'], 'attn %.2f'%p['attention']['ms_per_step'], 'attn TF %.0f'%p['attention']['tflops'], 'mem %.2f'%p['memory_bound']['ms_per_step'], 'clk', d['clocks']['sm_mhz'])"; }
run ENERGON_ATTN=3
run ENERGON_ATTN=2
XX
bash /tmp/ab.sh
timeout 300 python bench.py --config gpt2s --steps 20 --warmup 5 --no-cpu-baseline --no-ab > gpurun_out/bench_gpt2s.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_gpt2s.log').read().strip().splitlines()[-1]); print('gpt2s', d['value'], d['ms_per_step'], json.dumps(d['phases']['attention']))"

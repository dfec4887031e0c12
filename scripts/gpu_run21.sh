timeout 900 python -m pytest tests -m gpu -x -q --timeout=300 > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
bash /tmp/ab.sh 2>/dev/null || true
cat > /tmp/ab.sh <<'XX'
run() { env "$@" timeout 300 python bench.py --steps 6 --warmup 2 --no-e2e --no-cpu-baseline --no-ab 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']
print('$*', 'ms/step %.2f'%d['ms_per_step'], 'gemm %.2f'%p['gemm']['ms_per_step'], 'attn %.2f'%p['attention']['ms_per_step'], 'attn TF %.0f'%p['attention']['tflops'], 'mem %.2f'%p['memory_bound']['ms_per_step'], 'clk', d['clocks']['sm_mhz'])"; }
run ENERGON_ATTN=3
run ENERGON_ATTN=2
XX
bash /tmp/ab.sh

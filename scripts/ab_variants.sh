# A/B of implementation variants via env switches; prints per-phase ms per step
run() { env "$@" timeout 300 python bench.py --steps 6 --warmup 2 --no-e2e --no-cpu-baseline --no-ab 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']
print('$*', 'ms/step %.2f'%d['ms_per_step'], 'gemm %.2f'%p['gemm']['ms_per_step'], 'attn %.2f'%p['attention']['ms_per_step'], 'mem %.2f'%p['memory_bound']['ms_per_step'], 'mem GB/s %.0f'%p['memory_bound']['gbs'], 'clk', d['clocks']['sm_mhz'])"; }
run ENERGON_ATTN=2 ENERGON_LN_TPR=256
run ENERGON_ATTN=1 ENERGON_LN_TPR=256
run ENERGON_ATTN=2 ENERGON_LN_TPR=128
run ENERGON_ATTN=2 ENERGON_LN_TPR=512

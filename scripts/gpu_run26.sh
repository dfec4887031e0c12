timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout=300 -k "gemm" 2>&1 | tail -1
for h in 1 0 1 0; do ENERGON_L2_HINTS=$h timeout 300 python bench.py --steps 8 --warmup 2 --no-e2e --no-cpu-baseline --no-ab 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']
print('hints=$h', 'ms/step %.2f'%d['ms_per_step'], 'gemm %.2f'%p['gemm']['ms_per_step'], 'TF %.0f'%p['gemm']['tflops'], 'clk', d['clocks']['sm_mhz'])"; done
export ENERGON_PROFILE_RANGE=1
for h in 1 0; do ENERGON_L2_HINTS=$h timeout 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_tc2 -c 4 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-ab --no-e2e --layers 1 2>/dev/null | grep -E "dram__bytes_read" | awk -F'","' '{print $NF}'; done

mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/attn2_full.log 2>&1; echo "full rc=$?"; tail -2 gpurun_out/attn2_full.log
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "attention or opt or fused or gpt3 or edge" 2>&1 | tail -1; done
for a in 3 4; do ENERGON_ATTN=$a timeout 120 python scripts/bench_attn.py 2>&1 | tail -4; done
for a in 4 3; do
ENERGON_ATTN=$a timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-ab --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bench attn=$a', round(d['ms_per_step'],2), d['phases']['attention'], d['clocks']['sm_mhz'])"
done

# 256 x 224 pair tile: parity, then A/B against the 256-only policy (ENERGON_NO_TILE224=1) on the TP shapes and
# in the emulated TP = 8 / TP = 4 steps, alternating
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "gemm or tile224 or fused_layout or local_tp" 2>&1 | tail -2
for rep in 1 2; do
  for s in "4096 1920 5120 1" "4096 5120 640 0" "4096 5120 2560 0" "4096 5120 1280 0" "4096 3840 5120 1" "4096 2560 5120 2"; do
    echo "auto  $(python scripts/gemm_one.py $s)"; echo "no224 $(ENERGON_NO_TILE224=1 python scripts/gemm_one.py $s)"
  done
done
for k in 8 4; do for rep in 1 2; do
  timeout 900 python bench.py --local-tp $k --no-cpu-baseline --no-ab --no-e2e --no-tp-check --steps 5 > gpurun_out/bench_ltp${k}_224_$rep.json 2>/dev/null
  ENERGON_NO_TILE224=1 timeout 900 python bench.py --local-tp $k --no-cpu-baseline --no-ab --no-e2e --no-tp-check --steps 5 > gpurun_out/bench_ltp${k}_256_$rep.json 2>/dev/null
  python -c "
import json
for t in ('224','256'):
    d=json.load(open('gpurun_out/bench_ltp${k}_'+t+'_$rep.json')); print('ltp$k', t, d['ms_per_step'], d['phases']['gemm'], d['clocks']['sm_mhz'])"
done; done
timeout 900 python bench.py --steps 5 --no-cpu-baseline --no-ab > gpurun_out/bench_tp1_224.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_tp1_224.json')); print('tp1', d['value'], d['ms_per_step'], d['phases']['gemm'], d['clocks']['sm_mhz'])"
